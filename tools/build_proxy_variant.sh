#!/bin/bash
# Calibration variant of the library with proxy.cu rebuilt under extra flags.
#   tools/build_proxy_variant.sh NAME [nvcc flags...] -> paper_2512_14082_b200/_build/var_NAME/lib.so
set -e
cd "$(dirname "$0")/.."
N=$1; shift
B=paper_2512_14082_b200/_build/var_$N
mkdir -p $B
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -ccbin /usr/bin/g++ -DUS_CALIBRATION"
O=paper_2512_14082_b200/_build/calib
nvcc $F "$@" -c paper_2512_14082_b200/csrc/proxy.cu -o $B/proxy.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/lib.so $(ls $O/*.o | grep -v "/proxy.o") $B/proxy.o -lrt
echo $B/lib.so
