"""Achieved sparsity rho of the GPU selection vs planted gain / P (picks the bench operating point)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
for gain in [float(g) for g in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["8", "9", "10"])]:
    Q, K, V = workloads.planted_blocks(L, 8, 2, 128, 64, seed=2512, gain=gain)
    for P in (0.9, 0.95):
        rep = us.select_blocks(Q, K, us.CompressionConfig(P=P))
        print(f"L={L} gain={gain} P={P} rho={rep.rho_mean:.4f}", flush=True)
    del Q, K, V
    torch.cuda.empty_cache()
