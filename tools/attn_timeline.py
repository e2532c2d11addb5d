"""Per-step event timeline of both tiles of one attention CTA (trace builds)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads
L = us.api.lib()
L.us_debug_attn_trace.argtypes = [C.c_int, C.c_void_p]
Q, K, V = workloads.planted_blocks(16384, 16, 4, 128, 64, seed=7, gain=8.0)
eng = us.Engine(Q, K, V, us.CompressionConfig(P=0.95))
eng.run(dense=True); torch.cuda.synchronize()
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 200
L.us_debug_attn_trace(cta, None)
eng.run(dense=True); torch.cuda.synchronize()
buf = np.zeros(2 * 4096 * 16, np.int64)
L.us_debug_attn_trace(cta, buf.ctypes.data)
tr = buf.reshape(2, 4096, 16)
names = {0: "S_issue", 1: "S_seen", 4: "S_loaded", 7: "turn", 5: "math_done", 2: "P_ready", 3: "PV_issued"}
k0 = 100
base = tr[:, k0, 0].min()
for k in range(k0, k0 + 4):
    for x in (0, 1):
        ev = sorted((int(tr[x, k, e] - base), n) for e, n in names.items() if tr[x, k, e] > 0)
        print(f"k={k} tile {'AB'[x]}: " + "  ".join(f"{n}@{t}" for t, n in ev))
