#!/bin/bash
# Debug variant: attention with the clock64 step timeline (and optionally the math-free skeleton).
set -e
cd "$(dirname "$0")/.."
B=paper_2512_14082_b200/_build/trace
mkdir -p $B
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -ccbin /usr/bin/g++"
O=paper_2512_14082_b200/_build
nvcc $F -DUS_ATTN_TRACE=1 -c paper_2512_14082_b200/csrc/attention.cu -o $B/attention.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/libunisparse_trace.so $O/api.o $O/compress.o $O/proxy.o $O/select.o $B/attention.o $O/attention2.o $O/lastblock.o $O/io.o $O/selftest.o -lrt
