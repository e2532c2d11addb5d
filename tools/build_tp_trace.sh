#!/bin/bash
# Debug variant of the P-in-TMEM attention (attention_tp.cu) with the clock64 step timeline.
#   tools/build_tp_trace.sh [extra nvcc flags...]   -> paper_2512_14082_b200/_build/tptrace/libunisparse_tptrace.so
set -e
cd "$(dirname "$0")/.."
B=paper_2512_14082_b200/_build/tptrace
mkdir -p $B
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -ccbin /usr/bin/g++ -Ipaper_2512_14082_b200/csrc -DUS_CALIBRATION"
O=paper_2512_14082_b200/_build/calib
nvcc $F -DUS_TP_TRACE=1 "$@" -c paper_2512_14082_b200/csrc/attention_tp.cu -o $B/attention_tp.o
OBJS=$(ls $O/*.o | grep -v attention_tp.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/libunisparse_tptrace.so $OBJS $B/attention_tp.o -lrt
echo $B/libunisparse_tptrace.so
