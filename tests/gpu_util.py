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


def oracle_row_parity(Q, K, V, sel_obj, O_dev, mode, sel, P, rows_per_head=4, max_heads=8, seed=2512):
    """Parity record of the MEASURED configuration: for one Q head of
    each KV group of this rank's shard (up to `max_heads`) and a stratified sample of
    query blocks (always including the last, longest row), the oracle recomputes the
    proxy row (full-row LSE over every composite key), applies the reference Top-P /
    top-k rule, and recomputes block-sparse attention over the GPU's selection for
    that row, from the same bf16 inputs copied back from the device. Masks must be
    identical (each flipped block is listed with its decision margins); outputs are
    compared by max-abs and relative Frobenius error. Test infrastructure only (used by
    the -m gpu config tests and by bench.py's parity record)."""
    import math
    import time
    t0 = time.perf_counter()
    _, H, L, d = Q.shape
    H_kv = K.shape[1]
    G = H // H_kv
    S, N = 64, L // 64
    rng = np.random.default_rng(seed)
    kv_sample = np.linspace(0, H_kv - 1, min(H_kv, max_heads)).round().astype(int)
    flips, decisions, nrows = [], 0, 0
    err_max, ref_max, err2, ref2 = 0.0, 0.0, 0.0, 0.0
    heads_done = []
    bits = sel_obj.dense_mask()[0]  # [H, N, N] on the device
    for kv in kv_sample:
        h = int(kv * G + rng.integers(0, G))
        q = Q[0, h:h + 1].float().cpu().numpy()
        k = K[0, kv:kv + 1].float().cpu().numpy()
        v = V[0, kv:kv + 1].float().cpu().numpy()
        c = O.cfg(1, L, d, S, H_kv=1, P=P if mode == "top_p" else 0.95,
                  select_mode=O.TOP_P if mode == "top_p" else O.TOP_K, top_k=0 if mode == "top_p" else int(sel))
        Qc, Kc = O.compress(c, q, k)
        strata = np.linspace(0, N, rows_per_head).astype(int)
        rows = np.unique(np.concatenate([[N - 1], [rng.integers(strata[t], max(strata[t] + 1, strata[t + 1]))
                                                   for t in range(rows_per_head - 1)]])).astype(np.int32)
        scores = O.proxy_score_rows(c, Qc, Kc, 0, rows)
        gmask = bits[h, rows.astype(np.int64)].cpu().numpy()  # [rows, N]
        mask1 = np.zeros((1, N, N), np.uint8)
        for r, i in enumerate(rows):
            idx, _ = (O.top_p_row(scores[r, : i + 1], P) if mode == "top_p" else O.top_k_row(scores[r, : i + 1], int(sel)))
            ref = np.zeros(N, bool)
            ref[idx] = True
            decisions += int(i) + 1
            for j in np.nonzero(ref != gmask[r])[0]:
                flips.append(dict(head=h, **mask_margins(scores[r], P if mode == "top_p" else 1.0, int(i), int(j))))
            mask1[0, i] = gmask[r]
        Or, _ = O.block_sparse_attention_rows(q, k, v, mask1, S, np.zeros(len(rows), np.int32), rows)
        for r, i in enumerate(rows):
            got = O_dev[0, h, i * S:(i + 1) * S].float().cpu().numpy()
            e = got - Or[r]
            err_max = max(err_max, float(np.abs(e).max()))
            ref_max = max(ref_max, float(np.abs(Or[r]).max()))
            err2 += float((e.astype(np.float64) ** 2).sum())
            ref2 += float((Or[r].astype(np.float64) ** 2).sum())
        nrows += len(rows)
        heads_done.append(h)
    return {"rows": nrows, "heads": heads_done, "decisions": decisions, "mask_flips": len(flips), "flips": flips[:20],
            "max_abs_err": err_max, "max_abs_ref": ref_max, "rel_fro_err": math.sqrt(err2 / max(ref2, 1e-300)),
            "tolerance": "masks identical; max_abs <= 1e-2*max|O_ref| + 1e-4, rel-Frobenius <= 1e-2",
            "ok": len(flips) == 0 and err_max <= 1e-2 * ref_max + 1e-4 and math.sqrt(err2 / max(ref2, 1e-300)) <= 1e-2,
            "oracle": "oracle/ (fp64 restatement of proxy.cpp:10-72, selection.cpp:11-48, attention.cpp:89-137)",
            "s": time.perf_counter() - t0}
