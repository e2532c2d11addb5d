"""How the four query groups of an attention CTA are paired into two M=128 tiles
changes the per-tile step counts (union of the pair's selections). For the
bench workload, compares the fixed pairing (01|23) with the best of the three
pairings per CTA: total tile steps (tensor-pipe work) and the sum over CTAs of
the longer tile (critical path).

  python tools/tile_pairing.py [L H H_kv gain P]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads

a = sys.argv[1:]
L, H, Hkv = (int(a[0]), int(a[1]), int(a[2])) if a else (131072, 32, 8)
gain, P = (float(a[3]), float(a[4])) if len(a) > 4 else (9.0, 0.95)
Q, K, V = workloads.planted_blocks(L, H, Hkv, 128, 64, seed=2512, gain=gain)
eng = us.Engine(Q, K, V, us.CompressionConfig(P=P))
eng.run()
torch.cuda.synchronize()
bits = eng.sel.mask_bits[0]  # [H, N, W] int32 words
N = L // 64
# unpack to bool [H, N, N] in chunks of heads (128K: 32 x 2048 x 2048 bits fits easily)
sh = torch.arange(32, device=bits.device, dtype=torch.int32)
m = ((bits.unsqueeze(-1) >> sh) & 1).bool().reshape(H, N, -1)[:, :, :N]
tri = torch.tril(torch.ones(N, N, dtype=torch.bool, device=m.device))
m &= tri
quads = m.reshape(H // 4, 4, N, N)
cnt = lambda x, y: (quads[:, x] | quads[:, y]).sum(-1).float()  # [H/4, N]
pairings = [((0, 1), (2, 3)), ((0, 2), (1, 3)), ((0, 3), (1, 2))]
tA = torch.stack([cnt(*p[0]) for p in pairings])  # [3, H/4, N]
tB = torch.stack([cnt(*p[1]) for p in pairings])
tot = tA + tB
mx = torch.maximum(tA, tB)
useful = m.sum().item()
print(f"L={L} H={H} H_kv={Hkv} P={P}: selected group-steps {useful}")
print(f"fixed (01|23): tile steps {tot[0].sum().item():.0f} (rows useful {useful / (2 * tot[0].sum().item()):.3f}), "
      f"sum of longer tile {mx[0].sum().item():.0f}, sum of union of 4 {quads.any(1).sum().item()}")
for crit, name in ((tot, "min total"), (mx, "min longer tile"), (mx * 4 + tot, "min 4*longer+total")):
    best = crit.argmin(0, keepdim=True)
    bt = tot.gather(0, best).sum().item()
    bm = mx.gather(0, best).sum().item()
    print(f"best pairing by {name}: tile steps {bt:.0f} (rows useful {useful / (2 * bt):.3f}), sum of longer tile {bm:.0f}")
per_head = m.sum((1, 2)).float()
print("per-head selected blocks: min %.0f median %.0f max %.0f" % (per_head.min(), per_head.median(), per_head.max()))
