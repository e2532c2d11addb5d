export US_LIB_PATH_OVERRIDE=$PWD/paper_2512_14082_b200/_build/trace/libunisparse_trace.so
python tools/attn_trace.py 200 > gpurun_out/trace_main8.txt 2>&1
python tools/attn_trace.py 700 >> gpurun_out/trace_main8.txt 2>&1
