"""Dense-attention step timeline of one CTA (needs the trace build, tools/build_trace.sh)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads
L = us.api.lib()
L.us_debug_attn_trace.argtypes = [C.c_int, C.c_void_p]
dense = (sys.argv[2] if len(sys.argv) > 2 else "dense") == "dense"
Q, K, V = workloads.planted_blocks(16384, 16, 4, 128, 64, seed=7, gain=9.0 if not dense else 8.0)
eng = us.Engine(Q, K, V, us.CompressionConfig(P=0.95))
eng.run(dense=dense); torch.cuda.synchronize()
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 200
L.us_debug_attn_trace(cta, None)
eng.run(dense=dense); torch.cuda.synchronize()
buf = np.zeros(2 * 4096 * 16, np.int64)
L.us_debug_attn_trace(cta, buf.ctypes.data)
tr = buf.reshape(2, 4096, 16)
n = int((tr[0, :, 0] > 0).sum())
t0 = tr[:, :n, :4][tr[:, :n, :4] > 0].min()
print(f"cta {cta} ({'dense' if dense else 'sparse'}): {n} steps in tile A")
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
if not dense:
    # per step: kind (bit 0: group of rows 0-63 selected, bit 1: rows 64-127), the four quarters'
    # P hand-offs (10..13), the issuer seeing P (9), P.V issued (3), K/V landed for S (8)
    kinds = tr[0, :n, 6]
    print("tile A sparse steps (relative to S issue):")
    for k in range(1, min(n, 24)):
        r = tr[0, k]
        base = r[0]
        print(f"k={k:3d} kind={int(kinds[k])} ready@{r[7]-base:6d} Kland@{r[8]-base:6d} S_iss 0 seen_q0@{r[1]-base:6d} "
              f"prev_sfree@{(tr[0, k-1, 14]-base):6d} "
              f"hand q0..3@{[int(r[10+q]-base) for q in range(4)]} Pseen@{r[9]-base:6d} PV@{r[3]-base:6d} "
              f"nextS@{(tr[0, k+1, 0]-base) if k + 1 < n else 0:6d}")
    per = np.diff(tr[0, :n, 0])
    for kd in (1, 2, 3):
        sel = kinds[1:n] == kd
        if sel.any():
            print(f"kind {kd}: steps {int(sel.sum())}, median S-issue period {np.median(per[sel[:len(per)]]):.0f}, "
                  f"median S->Pseen {np.median((tr[0,1:n,9]-tr[0,1:n,0])[sel]):.0f}, "
                  f"median Pseen->PV {np.median((tr[0,1:n,3]-tr[0,1:n,9])[sel]):.0f}")
