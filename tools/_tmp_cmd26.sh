timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_gpu12.log
python tools/time_attn.py 16384 16 4 > gpurun_out/v8t_sweep.txt 2>&1
for v in v8noturn v8tp64 v8tp40 v8tp56; do US_LIB_PATH_OVERRIDE=$PWD/paper_2512_14082_b200/_build/var_$v/libunisparse_$v.so python tools/time_attn.py 16384 16 4; done >> gpurun_out/v8t_sweep.txt 2>&1
US_LIB_PATH_OVERRIDE=$PWD/paper_2512_14082_b200/_build/trace/libunisparse_trace.so python tools/attn_trace.py 200 > gpurun_out/trace_v8t.txt 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench12.json 2> gpurun_out/bench12.err
