"""Parity at the BASELINE configurations' FULL shapes: the
whole layer runs on the GPU through the C ABI on synthetic planted Q/K/V of the
named shape, and the CPU oracle recomputes a stratified sample of (head, query
block) rows from the same bf16 values — one Q head of every KV group (up to 8),
always including the last (longest) row — exactly as the reference would: the
proxy row over every composite key, the Top-P / top-k rule on it, and block-sparse
attention over the GPU's selection (tests/gpu_util.py oracle_row_parity). Masks
must match bit for bit; outputs within the bf16 tolerance
(max-abs <= 1e-2 * max|O_ref| + 1e-4, relative Frobenius <= 1e-2).

  C2  Llama 32Q/8KV, L = 32K (N = 512), top-k k = 64
  C3  Llama 32Q/8KV, L = 128K (N = 2048), Top-P 0.95, at gain 9 (rho ~ 0.90) and 8 (~0.68)
  C4  Qwen 28Q/4KV (G = 7), L = 64K and 128K, Top-P 0.95
  C5  video 40 heads (MHA), L = 256K (N = 4096, the kernels' limit), Top-P 0.95
"""
import json
import os

import pytest

from gpu_util import oracle_row_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = {
    # name: (H, H_kv, L, mode, sel, P, gain)
    "C2_32K_topk64": (32, 8, 32768, "top_k", 64, 0.95, 8.0),
    "C3_128K_g9": (32, 8, 131072, "top_p", None, 0.95, 9.0),
    "C3_128K_g8": (32, 8, 131072, "top_p", None, 0.95, 8.0),
    "C4_64K": (28, 4, 65536, "top_p", None, 0.95, 8.5),
    "C4_128K": (28, 4, 131072, "top_p", None, 0.95, 9.0),
    "C5_256K": (40, 40, 262144, "top_p", None, 0.95, 9.5),
}


@pytest.mark.parametrize("name", list(CASES))
def test_config_rows_match_oracle(name):
    import paper_2512_14082_b200 as us
    from paper_2512_14082_b200 import workloads
    H, H_kv, L, mode, sel, P, gain = CASES[name]
    Q, K, V = workloads.planted_blocks(L, H, H_kv, 128, 64, seed=2512, gain=gain)
    cfg = us.CompressionConfig(P=P) if mode == "top_p" else us.CompressionConfig(select_mode=us.SELECT_TOP_K,
                                                                                 top_k=sel)
    eng = us.Engine(Q, K, V, cfg)
    eng.run()
    torch.cuda.synchronize()
    us.api._raise(us.api.lib().us_check_device_errors(us.api.C.byref(eng.p), us.api._ptr(eng.ws),
                                                      us.api._stream()))
    N = L // 64
    rho = 1.0 - eng.sel.counts.to(torch.int64).sum().item() / (H * N * (N + 1) / 2)
    rec = oracle_row_parity(Q, K, V, eng.sel, eng.O, mode, sel, P, rows_per_head=6, max_heads=8, seed=11)
    rec.update(config=name, rho=rho)
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/parity_{name}.json", "w") as f:
        json.dump(rec, f, indent=1)
    assert rec["mask_flips"] == 0, rec["flips"]
    assert rec["max_abs_err"] <= 1e-2 * rec["max_abs_ref"] + 1e-4, rec
    assert rec["rel_fro_err"] <= 1e-2, rec
    if name.startswith("C5"):
        assert N == 4096  # the 12-bit block ids of the attention union list / select_kernel<128>
