"""Shared helpers for the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

import oracle_py as O


def to_dev_bf16(x: np.ndarray, B: int | None = None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16)
    if B is not None and t.dim() == 3:
        t = t.unsqueeze(0)
    return t.cuda().contiguous()


def workload(kind, L, H, H_kv, d, seed, gain=8.0, m=2, sigma=0.1):
    """Reference generator (bit-faithful port), then bf16 rounding — the GPU
    and the oracle both consume exactly these values."""
    Q, K, V, planted = O.gen_workload(kind, L, H, d, 64, seed, H_kv=H_kv, gain=gain, m=m, sigma=sigma)
    return O.bf16_round(Q), O.bf16_round(K), O.bf16_round(V), planted


def mask_margins(scores: np.ndarray, P: float, i: int, j_flipped):
    """For a flipped decision in row i, report the score gap between the flipped
    block and the Top-P boundary block and the cumulative-mass margin."""
    row = scores[: i + 1].astype(np.float64)
    order = sorted(range(i + 1), key=lambda j: (-row[j], j))
    total = sum(row[j] for j in order)
    cum, k = 0.0, 0
    for k, j in enumerate(order):
        cum += row[j]
        if cum >= P * total:
            break
    boundary = order[k]
    return {"row": i, "block": int(j_flipped), "boundary": boundary,
            "score_gap_rel": abs(row[j_flipped] - row[boundary]) / max(total, 1e-300),
            "mass_margin_rel": abs(cum - P * total) / max(total, 1e-300)}
