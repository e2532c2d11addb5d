US_ATTN_IMPL=2 timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/pytest_attn2.log
python tools/time_attn.py 16384 16 4 > gpurun_out/attn2_time.txt 2>&1
US_ATTN_IMPL=2 python tools/time_attn.py 16384 16 4 >> gpurun_out/attn2_time.txt 2>&1
US_ATTN_IMPL=2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_attn2.json 2> gpurun_out/bench_attn2.err
