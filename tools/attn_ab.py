"""A/B of two attention implementations on the same selection (calibration):
times both and reports max |O_a - O_b| per configuration.

    python tools/attn_ab.py IMPL_A IMPL_B [L ...]

(impl >= 2 are calibration variants: run with
US_LIB_PATH_OVERRIDE=paper_2512_14082_b200/_build/libunisparse_b200_calib.so)
"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads

ia, ib = int(sys.argv[1]), int(sys.argv[2])
Ls = [int(v) for v in sys.argv[3:]] or [16384, 32768, 65536, 131072]
lib = us.api.lib()
for L in Ls:
    for gain in (9.0, 8.0):
        Q, K, V = workloads.planted_blocks(L, 32, 8, 128, 64, seed=7, gain=gain)
        eng = us.Engine(Q, K, V, us.CompressionConfig(P=0.95))
        outs, ms = [], []
        for impl in (ia, ib):
            lib.us_set_attention_impl(impl)
            eng.run(); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                eng.run()
            b.record(); torch.cuda.synchronize()
            ms.append(a.elapsed_time(b) / 3)
            outs.append(eng.O.clone())
        d = (outs[0].float() - outs[1].float()).abs().max().item()
        print(f"L={L} gain={gain}: impl{ia} {ms[0]:.2f} ms/layer  impl{ib} {ms[1]:.2f} ms/layer  max|dO|={d:.3e}", flush=True)
