python tools/time_attn.py 16384 16 4 > gpurun_out/v6_sweep.txt 2>&1
for v in v6p64 v6late v6p64late v6p56late; do US_LIB_PATH_OVERRIDE=$PWD/paper_2512_14082_b200/_build/var_$v/libunisparse_$v.so python tools/time_attn.py 16384 16 4; done >> gpurun_out/v6_sweep.txt 2>&1
