timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu14.log
US_ATTN_IMPL=2 python tools/time_attn.py 16384 16 4 > gpurun_out/attn2_time2.txt 2>&1
US_ATTN_IMPL=2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-dense 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["stages_ms"])' >> gpurun_out/attn2_time2.txt
