#!/bin/bash
# Product library with ONE source rebuilt under extra flags (select.cu knobs etc.):
#   tools/build_src_variant.sh NAME SRC.cu [nvcc flags...] -> paper_2512_14082_b200/_build/var_NAME/lib.so
# selected at run time by US_LIB_PATH_OVERRIDE.
set -e
cd "$(dirname "$0")/.."
N=$1; SRC=$2; shift 2
B=paper_2512_14082_b200/_build/var_$N
mkdir -p $B
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -ccbin /usr/bin/g++"
O=paper_2512_14082_b200/_build
OBJ=${SRC%.cu}.o
nvcc $F "$@" -c paper_2512_14082_b200/csrc/$SRC -o $B/$OBJ
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/lib.so $(ls $O/*.o | grep -v "/$OBJ") $B/$OBJ -lrt
echo $B/lib.so
