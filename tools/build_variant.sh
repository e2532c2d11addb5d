#!/bin/bash
# Calibration variants of the library with one attention compile-time knob changed:
#   tools/build_variant.sh NAME "-DUS_ATTN_POLY_FROM=16"
set -e
cd "$(dirname "$0")/.."
N=$1; shift
B=paper_2512_14082_b200/_build/var_$N
mkdir -p $B
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -ccbin /usr/bin/g++ -DUS_CALIBRATION"
O=paper_2512_14082_b200/_build/calib  # calibration-build objects (-DUS_CALIBRATION)
nvcc $F "$@" -c paper_2512_14082_b200/csrc/attention.cu -o $B/attention.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/libunisparse_$N.so $(ls $O/*.o | grep -v "/attention.o") $B/attention.o -lrt
echo $B/libunisparse_$N.so
