timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/pytest_gpu16.log
python tools/time_attn.py 16384 16 4 > gpurun_out/time_main16.txt 2>&1
export US_LIB_PATH_OVERRIDE=$PWD/paper_2512_14082_b200/_build/trace/libunisparse_trace.so
python tools/attn_trace.py 200 > gpurun_out/trace_main16.txt 2>&1
unset US_LIB_PATH_OVERRIDE
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench16.json 2> gpurun_out/bench16.err
