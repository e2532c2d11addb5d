#!/bin/bash
# Attention-kernel iteration loop (run under gpurun): parity tests of the attention paths,
# dense 32K timing, the C3 bench (gain 9 + gain 8) with parity, optional timeline.
# impl >= 2 selects a calibration variant (runs on the calibration library).
#   tools/attn_eval.sh [impl] [trace]
cd "$(dirname "$0")/.."
export US_ATTN_IMPL=${1:-0}
if [ "$US_ATTN_IMPL" -ge 2 ]; then export US_LIB_PATH_OVERRIDE=paper_2512_14082_b200/_build/libunisparse_b200_calib.so; fi
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -m gpu -x -q 2>&1 | tail -3
python tools/time_attn.py 32768 32 8
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-dense > gpurun_out/eval_bench.json 2>gpurun_out/eval_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/eval_bench.json").read().strip().splitlines()[-1])
s = d.get("secondary_operating_points") or [{}]
print("C3 g9 layer", round(d["ms_per_step"], 2), "attn", round(d["stages_ms"]["attention"], 2),
      "flips", d["parity"]["mask_flips"], "maxabs", d["parity"]["max_abs_err"],
      "| g8 layer", round(s[0].get("ms_per_layer", 0), 2), "attn", round(s[0].get("stages_ms", {}).get("attention", 0), 2))
PY
if [ "${2:-}" = "trace" ]; then
  US_LIB_PATH_OVERRIDE=paper_2512_14082_b200/_build/tptrace/libunisparse_tptrace.so python tools/tp_trace.py 200 dense 2>&1 | tail -16
fi
