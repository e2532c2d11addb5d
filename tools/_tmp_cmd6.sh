export US_LIB_PATH_OVERRIDE=$PWD/paper_2512_14082_b200/_build/trace/libunisparse_trace.so
python tools/attn_trace.py 200 > gpurun_out/trace_main.txt 2>&1
export US_LIB_PATH_OVERRIDE=$PWD/paper_2512_14082_b200/_build/trace/libunisparse_trace_skel.so
python tools/attn_trace.py 200 > gpurun_out/trace_skel.txt 2>&1
python tools/time_attn.py 16384 16 4 > gpurun_out/time_skel.txt 2>&1
unset US_LIB_PATH_OVERRIDE
python tools/time_attn.py 16384 16 4 > gpurun_out/time_main.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:'proxy_kernel|proxy_finalize' -s 2 -c 2 -o gpurun_out/ncu_r01c_proxy python tools/profile_case.py 131072 32 8 9.0 0.95 > /dev/null 2>&1
