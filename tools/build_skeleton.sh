#!/bin/bash
# Calibration variant of the library: attention softmax math replaced by a constant P.
set -e
cd "$(dirname "$0")/.."
B=paper_2512_14082_b200/_build/skel
mkdir -p $B
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -ccbin /usr/bin/g++"
nvcc $F -DUS_ATTN_SKELETON=1 -c paper_2512_14082_b200/csrc/attention.cu -o $B/attention.o
O=paper_2512_14082_b200/_build
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/libunisparse_skel.so $O/api.o $O/compress.o $O/proxy.o $O/select.o $B/attention.o $O/selftest.o -lrt
echo $B/libunisparse_skel.so
