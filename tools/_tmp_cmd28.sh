for v in main v8p56 v8p40 v8p64; do
  if [ $v = main ]; then unset US_LIB_PATH_OVERRIDE; else export US_LIB_PATH_OVERRIDE=$PWD/paper_2512_14082_b200/_build/var_$v/libunisparse_$v.so; fi
  echo "$v $(timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-dense 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["stages_ms"]["attention"])')"
done > gpurun_out/v8_poly_bench.txt 2>&1
