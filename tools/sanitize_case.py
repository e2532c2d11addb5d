"""Small end-to-end cases for compute-sanitizer (memcheck / initcheck / synccheck):
the smoke pipeline through both attention kernels (forced), top-k, pre-softmax, c_h = 2,
dense and non-causal dense. Run under gpurun:
    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads

torch.cuda.set_device(0)
L, H, H_kv, d = 4096, 8, 2, 128
Q, K, V = workloads.planted_blocks(L, H, H_kv, d, 64, seed=3, gain=8.0)
A = us.api
cases = [dict(P=0.95), dict(P=0.9, c_h=2), dict(select_mode=A.SELECT_TOP_K, top_k=16),
         dict(P=0.95, causal_mode=A.PRE_SOFTMAX_COMPRESSED_CAUSAL), dict(P=0.95, strategy=A.POOL_STOCHASTIC, seed=5)]
for impl in (0, 1, 6):  # automatic, attn_kernel forced, attn64_kernel forced
    A._raise(A.lib().us_set_attention_impl(impl))
    for kw in cases:
        r = us.unisparse_attn(Q, K, V, us.CompressionConfig(**kw))
        torch.cuda.synchronize()
        print(impl, kw, "rho", round(float(r.report.rho_mean), 4), "O finite", bool(torch.isfinite(r.O.float()).all()))
A._raise(A.lib().us_set_attention_impl(0))
for causal in (True, False):
    out = us.dense_attention(Q, K, V, causal=causal)
    torch.cuda.synchronize()
    Od = out[0] if isinstance(out, tuple) else getattr(out, "O", out)
    print("dense causal", causal, "finite", bool(torch.isfinite(Od.float()).all()))
