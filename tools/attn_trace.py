"""Dense-attention step timeline of one CTA (needs the trace build, tools/build_trace.sh)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
n = int((tr[0, :, 0] > 0).sum())
t0 = tr[:, :n, :4][tr[:, :n, :4] > 0].min()
print(f"cta {cta}: {n} steps per tile")
for k in list(range(0, 6)) + list(range(n // 2, n // 2 + 6)):
    a, b = tr[0, k, :4] - t0, tr[1, k, :4] - t0
    print(f"k={k:4d}  A: S@{a[0]:8d} seen@{a[1]:8d} P@{a[2]:8d} PV@{a[3]:8d} |  B: S@{b[0]:8d} seen@{b[1]:8d} P@{b[2]:8d} PV@{b[3]:8d}")
d = np.diff(tr[0, :n, 0]); print("tile A cycles/step (median):", np.median(d))
for name, (e0, e1) in {"S issue -> seen": (0, 1), "seen -> S loaded (LDTM)": (1, 4), "loaded -> math done": (4, 5), "P to smem + fence": (5, 2), "P ready -> PV issued": (2, 3), "PV issued -> next S issue": (3, 0)}.items():
    if e1 == 0:
        v = tr[0, 1:n, 0] - tr[0, :n - 1, 3]
    else:
        v = tr[0, :n, e1] - tr[0, :n, e0]
    print(f"  {name:26s} median {np.median(v):8.0f}")
