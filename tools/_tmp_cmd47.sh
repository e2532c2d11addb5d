python tools/time_attn.py 16384 16 4 > gpurun_out/off_sweep.txt 2>&1
for v in off1 off1p64; do US_LIB_PATH_OVERRIDE=$PWD/paper_2512_14082_b200/_build/var_$v/libunisparse_$v.so python tools/time_attn.py 16384 16 4; done >> gpurun_out/off_sweep.txt 2>&1
for v in main off1; do
  if [ $v = main ]; then unset US_LIB_PATH_OVERRIDE; else export US_LIB_PATH_OVERRIDE=$PWD/paper_2512_14082_b200/_build/var_$v/libunisparse_$v.so; fi
  echo "$v $(timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-dense 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["stages_ms"]["attention"])')"
done >> gpurun_out/off_sweep.txt 2>&1
