"""Experiment harness on GPU outputs: the reference's
run_experiment (experiment.cpp:280-437) over a grid of (c_q, c_k, c_h,
strategy, P, causal_mode) x proxies, every number computed on the device:

  proxy scores + mask   select_blocks(proxy, ...)          (pipeline.cpp:5-17)
  sparse output         block_sparse_attention              (attention.cpp:89-137)
  oracle                dense_attention + exact_block_mass  (experiment.cpp:207-227)
  metrics               output_fidelity / mean_row_spearman / block_recall
                        (metrics.cpp:118-224) in the C ABI (metrics.cu)

Outputs mirror the reference's files: records/run_NNNN.json (row_to_record,
experiment.cpp:229-267), metrics.csv (write_metrics_csv, experiment.cpp:129-142,
numbers as %.9g) and run_meta.json. Tasks run sequentially on the current
device (the reference's UNISPARSE_WORKERS pool parallelises CPU work; here
each task already fills the GPU).
"""
from __future__ import annotations

import dataclasses
import itertools
import json
import os
import time
from typing import Iterable, Optional, Sequence

import torch

from . import api

PROXY_NAMES = {api.PROXY_UNISPARSE: "unisparse", api.PROXY_ANTIDIAGONAL: "antidiagonal",
               api.PROXY_LAST_BLOCK: "last_block_probe"}
STRATEGY_NAMES = {0: "mean", 1: "max", 2: "stochastic"}
MODE_NAMES = {api.POST_SOFTMAX_BLOCK_CAUSAL: "post-softmax-block-causal",
              api.PRE_SOFTMAX_COMPRESSED_CAUSAL: "pre-softmax-compressed-causal"}
CSV_HEADER = ("proxy,c_q,c_k,c_h,strategy,P,rho,spearman,recall,max_abs,cosine,"
              "selection_flops,attention_flops")


class ValidationError(ValueError):
    """experiment.hpp ValidationError: a grid point the inputs cannot run."""


@dataclasses.dataclass
class Grid:
    """ExperimentConfig::grid (experiment.hpp): every axis non-empty."""
    c_q: Sequence[int] = (8,)
    c_k: Sequence[int] = (8,)
    c_h: Sequence[int] = (1,)
    strategy: Sequence[int] = (0,)
    P: Sequence[float] = (0.95,)
    causal_mode: Sequence[int] = (api.POST_SOFTMAX_BLOCK_CAUSAL,)


@dataclasses.dataclass
class RunRow:
    """RunRow (experiment.hpp:58-71)."""
    proxy: int
    c_q: int
    c_k: int
    c_h: int
    strategy: int
    P: float
    causal_mode: int
    rho: float = 0.0
    spearman: float = 0.0
    recall: float = 0.0
    max_abs: float = 0.0
    cosine: float = 1.0
    selection_flops: int = 0
    attention_flops: int = 0


def fmt_double(v: float) -> str:
    """fmt_double (experiment.cpp:26-30): printf %.9g."""
    return "%.9g" % v


def csv_line(r: RunRow) -> str:
    return ",".join([PROXY_NAMES[r.proxy], str(r.c_q), str(r.c_k), str(r.c_h), STRATEGY_NAMES[r.strategy],
                     fmt_double(r.P), fmt_double(r.rho), fmt_double(r.spearman), fmt_double(r.recall),
                     fmt_double(r.max_abs), fmt_double(r.cosine), str(r.selection_flops),
                     str(r.attention_flops)])


def write_metrics_csv(rows: Iterable[RunRow], path: str) -> None:
    """write_metrics_csv (experiment.cpp:129-142)."""
    with open(path, "w", newline="\n") as f:
        f.write(CSV_HEADER + "\n")
        for r in rows:
            f.write(csv_line(r) + "\n")


def _tasks(grid: Grid, proxies: Sequence[int]):
    # nesting order of experiment.cpp:298-318
    for i, (c_q, c_k, c_h, st, P, mode, proxy) in enumerate(itertools.product(
            grid.c_q, grid.c_k, grid.c_h, grid.strategy, grid.P, grid.causal_mode, proxies)):
        yield i, RunRow(proxy=proxy, c_q=c_q, c_k=c_k, c_h=c_h, strategy=st, P=float(P), causal_mode=mode)


def run_experiment(Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, *, grid: Grid = Grid(),
                   proxies: Sequence[int] = (api.PROXY_UNISPARSE,), stride: int = 8,
                   recall_k: int = 0, planted_m: Optional[int] = None, seed: int = 0, S: int = 64,
                   out_dir: Optional[str] = None, workload: Optional[dict] = None) -> list:
    """run_experiment (experiment.cpp:280-437) on device tensors Q [B, H, L, d],
    K/V [B, H_kv, L, d] (bf16). Returns the RunRows; writes the reference's
    output files when out_dir is given."""
    t_start = time.time()
    B, H, L, d = Q.shape
    N = L // S
    tasks = list(_tasks(grid, proxies))
    for _, t in tasks:  # validate every task first (experiment.cpp:319-323)
        cfg = api.CompressionConfig(c_q=t.c_q, c_k=t.c_k, c_h=t.c_h, strategy=t.strategy, P=t.P,
                                    causal_mode=t.causal_mode, seed=seed)
        msg = api.validate(api.make_params(Q, K, cfg, S))
        if msg:
            raise ValidationError(msg)
        if stride <= 0 or S % stride != 0:
            raise ValidationError("stride must divide S")
    dense, _ = api.dense_attention(Q, K, V, S)  # oracle_for (experiment.cpp:207-227)
    mass = api.exact_block_mass(Q, K, S)
    k = recall_k if recall_k > 0 else (planted_m if planted_m else 2)
    k = min(k, N)
    rows, records = [], []
    for idx, row in tasks:
        cfg = api.CompressionConfig(c_q=row.c_q, c_k=row.c_k, c_h=row.c_h, strategy=row.strategy, P=row.P,
                                    causal_mode=row.causal_mode, seed=seed)
        rep = api.select_blocks(Q, K, cfg, S, with_scores=True, proxy=row.proxy, stride=stride)
        c_h_eff = row.c_h if row.proxy == api.PROXY_UNISPARSE else 1
        sel = rep.mask
        sparse, _ = api.block_sparse_attention(Q, K, V, sel.mask_bits, heads_per_plane=c_h_eff, S=S,
                                               with_lse=False)
        fid = api.output_fidelity(sparse, dense)
        spear = api.mean_row_spearman(sel.scores, mass, c_h_eff, S)
        row.rho = rep.rho_mean
        row.spearman = spear[0]
        row.recall = api.block_recall(sel.mask_bits, mass, k, heads_per_plane=c_h_eff, S=S)
        row.max_abs = fid["max_abs"]
        row.cosine = fid["cosine"]
        fl = rep.flops
        row.selection_flops = fl["compression"] + fl["compressed_qk"] + fl["softmax_aggregation"] + fl["top_p"]
        row.attention_flops = fl["sparse_attention"]
        rows.append(row)
        cov = sel.coverage
        records.append({
            "version": 1,
            "settings": {"proxy": PROXY_NAMES[row.proxy], "c_q": row.c_q, "c_k": row.c_k, "c_h": row.c_h,
                         "strategy": STRATEGY_NAMES[row.strategy], "P": row.P,
                         "causal_mode": MODE_NAMES[row.causal_mode], "stride": stride, "recall_k": k,
                         "workload": dict(workload or {"L": L, "H": H, "d_k": d, "S": S, "seed": seed}),
                         "run_index": idx},
            "metrics": {"rho": row.rho, "rho_per_head": list(rep.rho), "selected_per_head": list(rep.selected),
                        "coverage_min": float(cov.min().item()), "spearman": row.spearman, "recall": row.recall,
                        "max_abs": row.max_abs, "mean_rel": fid["mean_rel"], "cosine": row.cosine},
            "flops": {"compression": fl["compression"], "compressed_qk": fl["compressed_qk"],
                      "softmax_aggregation": fl["softmax_aggregation"], "top_p": fl["top_p"],
                      "selection_total": row.selection_flops, "sparse_attention": fl["sparse_attention"],
                      "dense_attention": fl["dense_attention"]},
        })
    if out_dir is not None:
        os.makedirs(os.path.join(out_dir, "records"), exist_ok=True)
        for i, rec in enumerate(records):
            with open(os.path.join(out_dir, "records", "run_%04d.json" % i), "w") as f:
                f.write(json.dumps(rec, indent="\t") + "\n")
        write_metrics_csv(rows, os.path.join(out_dir, "metrics.csv"))
        meta = {"timestamp_utc": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
                "elapsed_seconds": time.time() - t_start, "workers": 1, "runs": len(rows),
                "workload": dict(workload or {"L": L, "H": H, "d_k": d, "S": S, "seed": seed}),
                "device": torch.cuda.get_device_name(Q.device)}
        with open(os.path.join(out_dir, "run_meta.json"), "w") as f:
            f.write(json.dumps(meta, indent="\t") + "\n")
    return rows
