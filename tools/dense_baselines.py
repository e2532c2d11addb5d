"""Dense causal prefill baselines on one B200 at a BASELINE shape: cuDNN SDPA (torch),
flashinfer (sm100 prefill: single_prefill_with_kv_cache, backend auto and the
trtllm-gen context kernels when available), flash_attn 2. Prints first-call
(JIT / module load) time and the steady ms per call.

python tools/dense_baselines.py [L H H_kv d]"""
import sys
import time

import torch

L, H, H_kv, d = (int(a) for a in sys.argv[1:5]) if len(sys.argv) > 4 else (131072, 32, 8, 128)
torch.manual_seed(0)
q = torch.randn(1, H, L, d, device="cuda", dtype=torch.bfloat16)
k = torch.randn(1, H_kv, L, d, device="cuda", dtype=torch.bfloat16)
v = torch.randn(1, H_kv, L, d, device="cuda", dtype=torch.bfloat16)


def timeit(fn, iters=3):
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    first = time.perf_counter() - t0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return first, a.elapsed_time(b) / iters


res = {}
from torch.nn.attention import SDPBackend, sdpa_kernel
with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
    res["cudnn_sdpa"] = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True,
                                                                                      enable_gqa=True))
q3, k3, v3 = q[0].transpose(0, 1).contiguous(), k[0].transpose(0, 1).contiguous(), v[0].transpose(0, 1).contiguous()
try:
    import flashinfer
    for be in ("auto", "fa2", "trtllm-gen", "cutlass"):
        try:
            res[f"flashinfer_{be}"] = timeit(lambda: flashinfer.single_prefill_with_kv_cache(q3, k3, v3, causal=True,
                                                                                            backend=be))
        except Exception as e:  # noqa: BLE001
            res[f"flashinfer_{be}"] = repr(e)[:200]
except Exception as e:  # noqa: BLE001
    res["flashinfer"] = repr(e)[:200]
try:
    from flash_attn import flash_attn_func
    res["flash_attn2"] = timeit(lambda: flash_attn_func(q3.unsqueeze(0), k3.unsqueeze(0), v3.unsqueeze(0), causal=True))
except Exception as e:  # noqa: BLE001
    res["flash_attn2"] = repr(e)[:200]
flops = 4 * L * L / 2 * H * d
for kname, val in res.items():
    if isinstance(val, tuple):
        print(f"{kname:24s} first call {val[0]:7.2f} s  steady {val[1]:9.3f} ms  {flops / val[1] / 1e9:7.1f} TFLOP/s")
    else:
        print(f"{kname:24s} {val}")
