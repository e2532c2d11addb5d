"""Per-step event timeline of both tiles of one attention CTA (trace builds).

  python tools/attn_timeline.py [cta] [--sparse L H H_kv gain P]

Dense (default): 16K x 16 heads, prints four steps of CTA `cta`. --sparse: the
selected mask of a planted workload; prints the first steps and, per tile,
the mean phase durations (cycles) over all steps of the CTA plus the step
period, split by step kind (one group vs both groups of the tile).
"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads

L = us.api.lib()
L.us_debug_attn_trace.argtypes = [C.c_int, C.c_void_p]
args = sys.argv[1:]
sparse = "--sparse" in args
if sparse:
    i = args.index("--sparse")
    Ls, H, Hkv, gain, P = int(args[i + 1]), int(args[i + 2]), int(args[i + 3]), float(args[i + 4]), float(args[i + 5])
    del args[i:i + 6]
else:
    Ls, H, Hkv, gain, P = 16384, 16, 4, 8.0, 0.95
cta = int(args[0]) if args else 200
Q, K, V = workloads.planted_blocks(Ls, H, Hkv, 128, 64, seed=7, gain=gain)
eng = us.Engine(Q, K, V, us.CompressionConfig(P=P))
eng.run(dense=not sparse); torch.cuda.synchronize()
L.us_debug_attn_trace(cta, None)
eng.run(dense=not sparse); torch.cuda.synchronize()
buf = np.zeros(2 * 4096 * 16, np.int64)
L.us_debug_attn_trace(cta, buf.ctypes.data)
tr = buf.reshape(2, 4096, 16)
names = {0: "S_issue", 1: "S_seen", 4: "S_loaded", 7: "turn", 5: "math_done", 2: "P_ready", 3: "PV_issued",
         8: "KV_landed", 9: "P_all"}
k0 = 100 if not sparse else 5
base = tr[:, k0, 0][tr[:, k0, 0] > 0].min() if (tr[:, k0, 0] > 0).any() else 0
for k in range(k0, k0 + 4):
    for x in (0, 1):
        ev = sorted((int(tr[x, k, e] - base), n) for e, n in names.items() if tr[x, k, e] > 0)
        print(f"k={k} tile {'AB'[x]}: " + "  ".join(f"{n}@{t}" for t, n in ev))
for x in (0, 1):
    n = int((tr[x, :, 1] > 0).sum())
    if n < 3:
        continue
    t = tr[x, :n].astype(np.float64)
    ph = {
        "issue->seen": t[:, 1] - t[:, 0],
        "seen->loaded": t[:, 4] - t[:, 1],
        "loaded->math": t[:, 5] - t[:, 4],
        "math->P": t[:, 2] - t[:, 5],
        "P->Pall": t[:, 9] - t[:, 2],
        "Pall->PVissued": t[:, 3] - t[:, 9],
        "KVlanded->Sissue": t[:, 0] - t[:, 8],
    }
    period = np.diff(t[:, 1])
    kind = tr[x, :n - 1, 6]
    for kd, nm in ((3, "both"), (1, "first group"), (2, "second group")):
        sel = kind == kd
        if sel.any():
            print(f"  tile {'AB'[x]} {nm}: {int(sel.sum())} steps, period {period[sel].mean():.0f}; " +
                  ", ".join(f"{k} {v[:-1][sel].mean():.0f}" for k, v in ph.items()))
    print(f"tile {'AB'[x]}: {n} steps, mean period {period.mean():.0f} cycles; " +
          ", ".join(f"{k} {v[1:].mean():.0f}" for k, v in ph.items()))
    # per-warp P hand-off (slots 10-13): which lane quarter arrives last, and by how much
    pw = t[:, 10:14]
    ok = (pw > 0).all(1)
    if ok.any():
        pw = pw[ok]
        last = pw.argmax(1)
        spread = pw.max(1) - pw.min(1)
        print(f"  tile {'AB'[x]} per-warp P hand-off: mean spread {spread.mean():.0f} cycles; last warp (quarter) histogram "
              + str(np.bincount(last, minlength=4).tolist())
              + "; mean lag behind the first warp per quarter "
              + str([int(v) for v in (pw - pw.min(1, keepdims=True)).mean(0)]))
