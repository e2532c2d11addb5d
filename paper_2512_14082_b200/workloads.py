"""Synthetic planted-block workloads generated directly on the GPU.

Same construction as the reference generator gen_workload(PlantedBlocks)
(/root/reference/proj/src/workloads.cpp:66-128): Q/K/V noise N(0, sigma^2);
for every (head h, query block i) a unit direction u_hi is added with amplitude
`gain` to the queries of block i and to the keys of m distinct causal blocks
sampled from [0, i]. GQA: planted keys go to K head h // (H / H_kv).

The random stream is torch's (not the reference's SplitMix64), so values are
statistically — not bitwise — those of the reference generator; bit-faithful
fixtures for parity come from the oracle port in tests/. Generating on the
device keeps a 128K x 32-head layer (1.5 GB bf16) to well under a second.
"""
from __future__ import annotations

import torch


@torch.no_grad()
def planted_blocks(L: int, H: int, H_kv: int, d: int, S: int = 64, *, seed: int = 0,
                   gain: float = 9.0, m: int = 2, sigma: float = 0.1, heads=None, B: int = 1,
                   batches=None, device="cuda", dtype=torch.bfloat16):
    """Returns Q [len(batches), len(heads), L, d], K/V [len(batches), n_kv, L, d] for
    the requested batch items (default range(B)) and Q heads (default all) and the
    KV heads they read; the planted structure of (b, h) depends only on (seed, b, h),
    so (batch, head) shards agree with the full tensor."""
    heads = list(range(H)) if heads is None else list(heads)
    G = H // H_kv
    kv_heads = sorted({h // G for h in heads})
    N = L // S
    Qs, Ks, Vs = [], [], []
    for b in (range(B) if batches is None else batches):
        q = torch.empty((len(heads), L, d), device=device, dtype=torch.float32)
        k = torch.empty((len(kv_heads), L, d), device=device, dtype=torch.float32)
        v = torch.empty((len(kv_heads), L, d), device=device, dtype=torch.float32)
        for t, h in enumerate(heads):
            g = torch.Generator(device=device).manual_seed(hash((seed, b, 0, h)) % (2**63))
            q[t].normal_(0.0, sigma, generator=g)
        for t, kv in enumerate(kv_heads):
            g = torch.Generator(device=device).manual_seed(hash((seed, b, 1, kv)) % (2**63))
            k[t].normal_(0.0, sigma, generator=g)
            g = torch.Generator(device=device).manual_seed(hash((seed, b, 2, kv)) % (2**63))
            v[t].normal_(0.0, sigma, generator=g)
        tri = torch.tril(torch.ones((N, N), dtype=torch.bool, device=device))
        for t, h in enumerate(heads):
            g = torch.Generator(device=device).manual_seed(hash((seed, b, 3, h)) % (2**63))
            u = torch.randn((N, d), generator=g, device=device)
            u = u / u.norm(dim=1, keepdim=True)
            # m distinct causal blocks per row: smallest m random keys among j <= i
            r = torch.rand((N, N), generator=g, device=device).masked_fill(~tri, 2.0)
            sel = r.topk(min(m, N), dim=1, largest=False).indices          # [N, m]
            valid = torch.arange(min(m, N), device=device)[None, :] <= torch.arange(N, device=device)[:, None]
            onehot = torch.zeros((N, N), device=device)
            onehot.scatter_(1, sel, valid.float())                           # [i, j]
            gu = gain * u                                                    # [N, d]
            q[t] += gu.repeat_interleave(S, dim=0)
            kadd = onehot.t() @ gu                                           # [j, d]
            k[kv_heads.index(h // G)] += kadd.repeat_interleave(S, dim=0)
        Qs.append(q.to(dtype))
        Ks.append(k.to(dtype))
        Vs.append(v.to(dtype))
    return (torch.stack(Qs).contiguous(), torch.stack(Ks).contiguous(), torch.stack(Vs).contiguous())
