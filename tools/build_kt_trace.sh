#!/bin/bash
# Debug variant of the library with the key-major attention step timeline (-DUS_KT_TRACE=1).
#   tools/build_kt_trace.sh [extra nvcc flags...]   -> prints the .so path (use US_LIB_PATH_OVERRIDE)
set -e
cd "$(dirname "$0")/.."
B=paper_2512_14082_b200/_build/kt_trace
mkdir -p $B
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -ccbin /usr/bin/g++ -Ipaper_2512_14082_b200/csrc -DUS_CALIBRATION"
O=paper_2512_14082_b200/_build/calib
nvcc $F -DUS_KT_TRACE=1 "$@" -c paper_2512_14082_b200/csrc/attention_kt.cu -o $B/attention_kt.o
objs=$(ls $O/*.o | grep -v attention_kt.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/libunisparse_kt_trace.so $objs $B/attention_kt.o -lrt
echo $B/libunisparse_kt_trace.so
