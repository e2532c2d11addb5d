"""Step timeline of one persistent CTA of the key-major attention kernel (needs the
trace build: US_LIB_PATH_OVERRIDE=$(tools/build_kt_trace.sh)).

python tools/kt_trace.py [cta] [L H H_kv gain P]
Events per pair step g: 0 S issued (MMA warp), 1 S seen (softmax warp 4), 2 S loaded,
3 vote done, 4 exps done, 5 P stored + arrived (warp 4), 6 all P seen (MMA warp),
7 P.V issued, 8 K TMA issued, 9 V TMA issued, 10 K landed + S buffer free (MMA warp),
11 last softmax warp arrived P."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads
lib = us.api.lib()
lib.us_debug_kt_trace.argtypes = [C.c_int, C.c_void_p]
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 0
L_, H, H_kv, gain, P = (int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5]), float(sys.argv[6])) \
    if len(sys.argv) > 6 else (131072, 32, 8, 9.0, 0.95)
Q, K, V = workloads.planted_blocks(L_, H, H_kv, 128, 64, seed=7, gain=gain)
eng = us.Engine(Q, K, V, us.CompressionConfig(P=P))
eng.run(); torch.cuda.synchronize()
lib.us_debug_kt_trace(cta, None)
eng.run(); torch.cuda.synchronize()
buf = np.zeros(4096 * 16, np.int64)
lib.us_debug_kt_trace(cta, buf.ctypes.data)
tr = buf.reshape(4096, 16).astype(np.float64)
n = int((tr[:, 5] > 0).sum())
lo, hi = n // 4, min(n, n // 4 + 1000)
seg = tr[lo:hi]
print(f"cta {cta}: {n} pair steps traced; steps {lo}..{hi}")
print("period (S seen -> next S seen) median:", np.median(np.diff(seg[:, 1])))
names = {"S issued -> S seen (softmax)": (0, 1), "S seen -> loaded": (1, 2), "loaded -> vote done": (2, 3),
         "vote -> exps done": (3, 4), "exps -> P arrived (w4)": (4, 5), "P arrived w4 -> last warp": (5, 11),
         "P arrived w4 -> P seen (MMA)": (5, 6), "P seen -> PV issued": (6, 7), "K issued -> K landed/S free": (8, 10),
         "K landed -> S issued": (10, 0)}
for k, (a, b) in names.items():
    print(f"  {k:32s} median {np.median(seg[:, b] - seg[:, a]):8.0f}  p90 {np.percentile(seg[:, b] - seg[:, a], 90):8.0f}")
# S(g+2) issue relative to PV(g) issue
print("  PV(g) issued -> S(g+2) issued   median", np.median(seg[2:, 0] - seg[:-2, 7]))
print("  S(g) seen -> S(g+1) seen (softmax idle gaps) ", np.median(seg[1:, 1] - seg[:-1, 5]))
t0 = seg[0, 0]
for g in range(lo, lo + 6):
    print(g, " ".join(f"{int(v - t0):8d}" for v in tr[g, :12]))
