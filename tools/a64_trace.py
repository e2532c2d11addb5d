"""Per-step timeline of one CTA of attention64.cu (the M = 64 chains), from the clock64
stamps of a -DUS_ATTN_TRACE=1 build (tools/build_trace.sh ... attention64.cu trace64):

    US_LIB_PATH_OVERRIDE=paper_2512_14082_b200/_build/trace64/libunisparse_trace.so \\
        python tools/a64_trace.py [CTA] [L] [gain]

Per own step k of each group: union position t, the issuer's S(k) request / issue (after
its K landed), the producer's load issue of t, the softmax's S wait / seen, exponentials
done, P hand-off, and the issuer's P.V issue. Cycles relative to the first stamp."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads

L = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
gain = float(sys.argv[3]) if len(sys.argv) > 3 else 9.0
Q, K, V = workloads.planted_blocks(L, 32, 8, 128, 64, seed=7, gain=gain)
eng = us.Engine(Q, K, V, us.CompressionConfig(P=0.95))
lib = us.api.lib()
assert lib.us_set_attention_impl(6) == 0
N = L // 64
grid = 8 * ((4 * N + 3) // 4)
cta = int(sys.argv[1]) if len(sys.argv) > 1 else grid // 3
eng.run(); torch.cuda.synchronize()
lib.us_debug_a64_trace(cta, None)
eng.run(); torch.cuda.synchronize()
buf = np.zeros(5 * 4096 * 8, dtype=np.int64)
lib.us_debug_a64_trace(cta, buf.ctypes.data_as(C.POINTER(C.c_longlong)))
tr = buf.reshape(5, 4096, 8)
stamps = tr[:4, :, :7][tr[:4, :, :7] > 0]
t0 = stamps.min()
prod = tr[4, :, 0]
nload = int((prod > 0).sum())
print(f"CTA {cta} of {grid}, L={L} gain={gain}: {nload} union positions loaded")
summ = []
for g in range(4):
    n = int((tr[g, :, 1] > 0).sum())
    if n == 0:
        continue
    rows = tr[g, :n].astype(np.int64)
    e = {x: rows[:, x] - t0 for x in range(7)}
    pos = rows[:, 7]
    load = np.array([prod[p] - t0 if prod[p] > 0 else -1 for p in pos])
    s_wait = e[1] - e[0]
    exps = e[2] - e[1]
    hand = e[6] - e[2]
    pv_lag = e[5] - e[6]
    kwait = e[4] - e[3]
    period = np.diff(e[1])
    s_lat = e[1][1:] - np.maximum(e[4][1:], e[5][:-1])  # S seen after max(S issue, P.V(k-1) issue)
    print(f"group {g}: {n} steps; mean cycles: S wait {s_wait.mean():.0f}, S seen->exps done {exps.mean():.0f}, "
          f"exps->P hand-off {hand.mean():.0f}, hand-off->P.V issue {pv_lag.mean():.0f}, "
          f"issuer K wait {kwait.mean():.0f}, step period {period.mean():.0f}, "
          f"S(k+1) issued after P.V(k) {(e[4][1:] > e[5][:-1]).mean()*100:.0f}%")
    summ.append(period.mean())
    if g < 2:
        print("   k    t |  S req  S iss  Kload(t) | sm want  S seen  exps  P hand | PV iss")
        for k in range(min(n, 24)):
            print(f"{k:4d} {pos[k]:4d} | {e[3][k]:6d} {e[4][k]:6d} {load[k]:7d} | {e[0][k]:7d} {e[1][k]:7d} "
                  f"{e[2][k]:6d} {e[6][k]:6d} | {e[5][k]:6d}")
lp = prod[:nload] - t0
print("producer load issue gaps (cycles): mean", np.diff(lp).mean().round(), "max", np.diff(lp).max())
if os.environ.get("A64_PRODUCER"):
    pk, pv = tr[4, :, 0], tr[4, :, 1]
    print("producer: load u: K issue, V issue (cycles rel.)")
    for u in range(min(nload, 40)):
        print(f"  {u:4d} {pk[u] - t0:8d} {pv[u] - t0 if pv[u] > 0 else -1:8d}")
