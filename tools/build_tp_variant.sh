#!/bin/bash
# Variant of the calibration library with attention_tp.cu rebuilt under extra flags.
#   tools/build_tp_variant.sh NAME [nvcc flags...] -> paper_2512_14082_b200/_build/var_NAME/lib.so
set -e
cd "$(dirname "$0")/.."
N=$1; shift
B=paper_2512_14082_b200/_build/var_$N
mkdir -p $B
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -ccbin /usr/bin/g++ -DUS_CALIBRATION"
nvcc $F "$@" -c paper_2512_14082_b200/csrc/attention_tp.cu -o $B/attention_tp.o
O=paper_2512_14082_b200/_build/calib
OBJS=$(ls $O/*.o | grep -v attention_tp.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/lib.so $OBJS $B/attention_tp.o -lrt
echo $B/lib.so
