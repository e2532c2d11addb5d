"""Step timeline of one CTA of the P-in-TMEM attention (needs tools/build_tp_trace.sh).

    US_LIB_PATH_OVERRIDE=paper_2512_14082_b200/_build/tptrace/libunisparse_tptrace.so \
    US_ATTN_IMPL=5 python tools/tp_trace.py [cta] [dense|sparse]
"""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads
L = us.api.lib()
L.us_debug_tp_trace.argtypes = [C.c_int, C.c_void_p]
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 200
dense = (sys.argv[2] if len(sys.argv) > 2 else "dense") == "dense"
Q, K, V = workloads.planted_blocks(16384, 16, 4, 128, 64, seed=7, gain=9.0)
eng = us.Engine(Q, K, V, us.CompressionConfig(P=0.95))
eng.run(dense=dense); torch.cuda.synchronize()
L.us_debug_tp_trace(cta, None)
eng.run(dense=dense); torch.cuda.synchronize()
buf = np.zeros(2 * 4096 * 16, np.int64)
L.us_debug_tp_trace(cta, buf.ctypes.data)
tr = buf.reshape(2, 4096, 16)
n = int((tr[0, :, 0] > 0).sum())
t0 = tr[:, :n, :13][tr[:, :n, :13] > 0].min()
names = {0: "S issued", 12: "K landed", 1: "S seen h0", 8: "S seen h1", 2: "S loaded", 3: "xch h0", 9: "xch h1",
         4: "exps done", 5: "P arr h0q0", 10: "P arr h1q0", 11: "P arr h0q3", 6: "P seen (iss)", 7: "PV issued"}
order = [12, 0, 1, 8, 2, 3, 9, 4, 5, 10, 11, 6, 7]
print(f"cta {cta} ({'dense' if dense else 'sparse'}): {n} steps in tile A")
for k in list(range(2, 5)) + list(range(n // 2, n // 2 + 3)):
    for x in (0, 1):
        r = tr[x, k]
        print(f"k={k:4d} {'AB'[x]}: " + " ".join(f"{names[e]}@{r[e] - t0:d}" for e in order if r[e] > 0))
d = np.diff(tr[0, :n, 0])
print("tile A cycles/step (median S-issue to S-issue):", np.median(d))
seg = [("S issued -> S seen h0", 0, 1), ("S seen -> loaded", 1, 2), ("loaded -> xch", 2, 3), ("xch -> exps done", 3, 4),
       ("exps -> P arrived h0q0", 4, 5), ("P arr h0q0 -> P seen by issuer", 5, 6), ("P seen -> PV issued", 6, 7)]
for name, a, b in seg:
    v = tr[0, 1:n - 1, b] - tr[0, 1:n - 1, a]
    print(f"  {name:32s} median {np.median(v):8.0f}")
v = tr[0, 2:n, 0] - tr[0, 1:n - 1, 7]
print(f"  {'PV issued -> next S issued':32s} median {np.median(v):8.0f}")
v = tr[0, 1:n - 1, 10] - tr[0, 1:n - 1, 5]
print(f"  {'P arr h1q0 - h0q0':32s} median {np.median(v):8.0f}")
v = tr[0, 1:n - 1, 11] - tr[0, 1:n - 1, 5]
print(f"  {'P arr h0q3 - h0q0':32s} median {np.median(v):8.0f}")
v = tr[1, 1:n - 1, 0] - tr[0, 1:n - 1, 0]
print(f"  {'tile B S issue - tile A':32s} median {np.median(v):8.0f}")
