#!/bin/bash
# Every BASELINE config on one B200 (bench.py lines, no CPU leg), plus a sparsity
# sweep (planted gain x Top-P) at C4 / C3 against the dense baselines.
#   tools/config_sweep.sh > gpurun_out/configs.jsonl
cd "$(dirname "$0")/.."
for c in C2 C3 C4_64K C4_128K C5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu 2>/dev/null
done
for c in C4_64K C3; do
  for g in 6.0 7.0 8.0 10.0; do
    for P in 0.9 0.95; do
      timeout 600 python bench.py --config $c --gain $g --P $P --steps 3 --warmup 3 --no-cpu 2>/dev/null
    done
  done
done
