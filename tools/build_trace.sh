#!/bin/bash
# Debug variant: one attention source rebuilt with the clock64 step timeline (and optionally
# other knobs), linked with the calibration objects of everything else.
#   tools/build_trace.sh [attention source] [name] [extra nvcc flags...]
set -e
cd "$(dirname "$0")/.."
SRC=${1:-paper_2512_14082_b200/csrc/attention.cu}; NAME=${2:-trace}; shift 2 || true
OBJ=$(basename $SRC .cu).o
B=paper_2512_14082_b200/_build/$NAME
mkdir -p $B
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -ccbin /usr/bin/g++ -Ipaper_2512_14082_b200/csrc -DUS_CALIBRATION"
O=paper_2512_14082_b200/_build/calib  # calibration-build objects (-DUS_CALIBRATION)
nvcc $F -DUS_ATTN_TRACE=1 "$@" -c $SRC -o $B/$OBJ
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/libunisparse_trace.so $(ls $O/*.o | grep -v "/$OBJ") $B/$OBJ -lrt
echo $B/libunisparse_trace.so
