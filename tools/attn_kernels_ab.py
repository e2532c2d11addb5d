"""Both attention kernels (attn_kernel = impl 1, attention64 = impl 6, forced) on the same
selections across BASELINE configs and sparsities: attention-stage ms and the own / union
ratio of attn_kernel's tiles (the density-gate calibration, profiles/r02d/README.md).

    python tools/attn_kernels_ab.py
"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads
import bench
lib = us.api.lib()
cases = [("C3", 9.0, 0.95), ("C3", 8.0, 0.95), ("C3", 7.0, 0.9), ("C3", 7.0, 0.95), ("C4_128K", 9.0, 0.95),
         ("C4_64K", 7.5, 0.95), ("C5", 9.5, 0.95), ("C5", 10.0, 0.95), ("C2", 8.0, None)]
for cfg, gain, P in cases:
    _, H, H_kv, L, d, mode, sel = bench.CONFIGS[cfg]
    Q, K, V = workloads.planted_blocks(L, H, H_kv, d, 64, seed=7, gain=gain)
    c = us.CompressionConfig(P=P) if mode == "top_p" else us.CompressionConfig(select_mode=us.SELECT_TOP_K, top_k=int(sel))
    eng = us.Engine(Q, K, V, c)
    res = {}
    for impl in (1, 6):
        lib.us_set_attention_impl(impl)
        eng.run(); torch.cuda.synchronize()
        us.api.profile_enable(2)
        for _ in range(2): eng.run()
        torch.cuda.synchronize()
        st = us.api.profile_read(2); us.api.profile_disable()
        res[impl] = sum(x["attention"] for x in st) / 2
    lib.us_set_attention_impl(0)
    selected = int(eng.sel.counts.to(torch.int64).sum().item())
    te = bench.tile_efficiency(eng.sel.dense_mask()[0], H // H_kv, selected)
    N = L // 64
    frac = selected / (H * N * (N + 1) / 2)
    print(f"{cfg:8s} gain {gain} P {P}: selected {frac:.3f} own/union {selected / te['issued_tile_steps']:.3f}  "
          f"v8 {res[1]:.2f}  attn64 {res[6]:.2f} ms  ratio {res[6] / res[1]:.3f}", flush=True)
    del eng, Q, K, V
    torch.cuda.empty_cache()
