#!/bin/bash
# attention64.cu rebuilt with compile-time knobs, linked with the product objects of everything else:
#   tools/build_a64_variant.sh NAME "-DUS_A64_KS=6 -DUS_A64_VS=6"   (select with US_LIB_PATH_OVERRIDE)
set -e
cd "$(dirname "$0")/.."
N=$1; shift
B=paper_2512_14082_b200/_build/var_$N
mkdir -p $B
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -ccbin /usr/bin/g++ -Ipaper_2512_14082_b200/csrc -lineinfo"
O=paper_2512_14082_b200/_build  # product objects
nvcc $F $@ -c paper_2512_14082_b200/csrc/attention64.cu -o $B/attention64.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/libunisparse_$N.so $(for f in api compress proxy select attention lastblock io metrics; do echo $O/$f.o; done) $B/attention64.o -lrt
echo $B/libunisparse_$N.so
