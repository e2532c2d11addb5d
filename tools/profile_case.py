"""Runs the hot path on one configuration a few times (for ncu captures).

python tools/profile_case.py L H H_kv gain P [dense]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads

L, H, H_kv = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
gain, P = float(sys.argv[4]), float(sys.argv[5])
dense = len(sys.argv) > 6 and sys.argv[6] == "dense"
Q, K, V = workloads.planted_blocks(L, H, H_kv, 128, 64, seed=7, gain=gain)
eng = us.Engine(Q, K, V, us.CompressionConfig(P=P))
for _ in range(3):
    eng.run(dense=dense)
torch.cuda.synchronize()
print("rho", 1 - eng.sel.counts.sum().item() / (H * (L // 64) * (L // 64 + 1) / 2), file=sys.stderr)
