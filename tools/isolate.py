import os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads
L, H, Hkv = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
stage = sys.argv[4]
Q, K, V = workloads.planted_blocks(L, H, Hkv, 128, 64, seed=7, gain=8.0)
try:
    if stage == "select":
        rep = us.select_blocks(Q, K, us.CompressionConfig(P=0.95))
        print("select ok rho", rep.rho_mean)
    elif stage == "dense":
        O, _ = us.dense_attention(Q, K, V); torch.cuda.synchronize(); print("dense ok", O.float().abs().mean().item())
    elif stage == "sparse":
        rep = us.select_blocks(Q, K, us.CompressionConfig(P=0.95))
        O, _ = us.block_sparse_attention(Q, K, V, rep.mask.mask_bits, 1); torch.cuda.synchronize(); print("sparse ok", O.float().abs().mean().item())
except Exception as e:
    print(stage, "FAILED:", str(e)[:200])
