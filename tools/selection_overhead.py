"""Selection overhead on one B200: UniSparse (compress + fp16x3 proxy + Top-P) vs the
XAttention-style anti-diagonal proxy (stride 8, bf16 logits, Top-P) on the same
C3-shaped planted layer (PAPER.md:542 compares the two at 128K). CUDA events,
3 warm-ups, median of 5. Prints one JSON line."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
H, H_kv, d, gain = 32, 8, 128, 9.0
Q, K, V = workloads.planted_blocks(L, H, H_kv, d, 64, seed=2512, gain=gain)
out = {"L": L, "heads": H, "kv_heads": H_kv, "gain": gain}
for name, proxy, stride in (("unisparse", us.api.PROXY_UNISPARSE, 8), ("antidiagonal_s8", us.api.PROXY_ANTIDIAGONAL, 8),
                            ("last_block_probe", us.api.PROXY_LAST_BLOCK, 8)):
    for P in (0.9, 0.95):
        cfg = us.CompressionConfig(P=P)
        run = lambda: us.select_blocks(Q, K, cfg, proxy=proxy, stride=stride, sync_check=False)
        for _ in range(3):
            rep = run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rep = run()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out[f"{name}_P{P}"] = {"ms": statistics.median(ts), "rho": rep.rho_mean}
for P in (0.9, 0.95):
    out[f"speedup_P{P}"] = out[f"antidiagonal_s8_P{P}"]["ms"] / out[f"unisparse_P{P}"]["ms"]
print(json.dumps(out))
