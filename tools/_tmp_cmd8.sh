ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 2 -c 1 -o gpurun_out/ncu_v7_dense16k python tools/time_attn.py 16384 16 4 > /dev/null 2>&1
