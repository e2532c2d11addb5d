"""Fixed per-CTA cost of the sparse attention kernel: block_sparse_attention at C3 shape with
masks that select only the last nb blocks of every row (nb = 1 .. 32). Run under ncu for the
kernel time alone (profiles/r02d/README.md):

    NBS=1,8,32 ncu --metrics gpu__time_duration.sum -k regex:attn64_kernel python tools/attn_fixed_cost.py
"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2512_14082_b200 as us
L, H, Hkv, d = 131072, 32, 8, 128
N, W = L // 64, L // 64 // 32
g = torch.Generator(device="cuda").manual_seed(1)
Q = torch.randn(1, H, L, d, device="cuda", dtype=torch.bfloat16, generator=g)
K = torch.randn(1, Hkv, L, d, device="cuda", dtype=torch.bfloat16, generator=g)
V = torch.randn_like(K)
i = torch.arange(N, device="cuda")
for nb in ([int(x) for x in os.environ["NBS"].split(",")] if "NBS" in os.environ else (1, 2, 4, 8, 16, 32)):
    bits = torch.zeros(1, H, N, W, dtype=torch.int64, device="cuda")
    for t in range(nb):  # blocks i, i-1, ..., i-nb+1 (clipped at 0)
        j = (i - t).clamp_min(0)
        bits[0, :, torch.arange(N, device="cuda"), j // 32] |= (1 << (j % 32))
    bits = bits.to(torch.int32) if False else torch.where(bits >= 2**31, bits - 2**32, bits).to(torch.int32)
    for _ in range(2):
        us.block_sparse_attention(Q, K, V, bits, validate_mask=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        us.block_sparse_attention(Q, K, V, bits, validate_mask=True)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    steps = H * N * nb
    print(f"{nb:3d} blocks/row: {ms:7.3f} ms  ({ms*1e-3*148*1.9e9/(H*N/4):8.0f} SM-cycles per CTA, {steps} group steps)", flush=True)
