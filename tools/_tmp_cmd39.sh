python tools/time_attn.py 16384 16 4 > gpurun_out/pe_sweep.txt 2>&1
for v in pe8 pe4 pe3 pe2; do US_LIB_PATH_OVERRIDE=$PWD/paper_2512_14082_b200/_build/var_$v/libunisparse_$v.so python tools/time_attn.py 16384 16 4; done >> gpurun_out/pe_sweep.txt 2>&1
