#!/usr/bin/env python
"""UniSparse prefill attention benchmark (BASELINE.json metric:
"attention prefill ms/layer @128K; speedup vs dense FA; HBM/TC roofline %").

One step = one attention layer's prefill through the B200 hot path:
compress -> fp16x3 tcgen05 proxy -> Top-P select -> tcgen05 block-sparse
attention, on synthetic planted-block Q/K/V (bf16, resident in HBM).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU): the layer's KV-head groups are
partitioned across ranks (strong scaling, no collective on the hot path); the
step time is the max over ranks. Rank 0 prints ONE JSON line.

--impl reference times the reference's CPU path (the oracle port in
oracle/, the reference itself cannot be built here) on this box's host cores,
on a bounded sample of the same workload, extrapolated to ms/layer.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (description, H, H_kv, L, d, select_mode, P/top_k)
    "C3": ("Llama-3.1-8B-shape layer prefill bf16, L=128K, threshold (Top-P) selection", 32, 8, 131072, 128, "top_p", 0.95),
    "C2": ("Llama-3.1-8B-shape layer prefill bf16, L=32K, top-k block selection", 32, 8, 32768, 128, "top_k", 64),
    "C4_64K": ("Qwen2.5-7B-shape GQA prefill, L=64K, Top-P", 28, 4, 65536, 128, "top_p", 0.95),
    "C4_128K": ("Qwen2.5-7B-shape GQA prefill, L=128K, Top-P", 28, 4, 131072, 128, "top_p", 0.95),
    "C5": ("Video/multimodal shape, 40 heads (MHA assumed), L=256K, Top-P", 40, 40, 262144, 128, "top_p", 0.95),
}
DEFAULT_GAIN = {"C3": 9.0, "C2": 8.0, "C4_64K": 8.5, "C4_128K": 9.0, "C5": 9.5}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class NvmlClockSampler:
    """SM clock + clock-event (throttle) reasons sampled every 10 ms through NVML
    (nvidia-ml-py) during the timed region; `ClockSampler` (nvidia-smi, 200 ms) is
    the fallback when NVML is unavailable."""
    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index: int):
        import pynvml
        pynvml.nvmlInit()
        self.n = pynvml
        self.h = None
        try:  # the CUDA ordinal -> NVML handle through the PCI bus id (CUDA_VISIBLE_DEVICES-proof)
            import torch
            pr = torch.cuda.get_device_properties(index)
            bus = "%08X:%02X:%02X.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
            self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:  # noqa: BLE001
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()

    def _run(self):
        n = self.n
        while not self.stop_ev.is_set():
            try:
                self.samples.append(n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM))
                mask = n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, attr in self.NAMES:
                    if mask & getattr(n, attr, 0):
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001 - a failed query ends sampling, not the bench
                break
            self.stop_ev.wait(0.01)

    def start(self):
        # one untimed query of each kind first: the first NVML calls of a process can take
        # longer than a whole timed region (one r02 box returned a single sample)
        try:
            self.n.nvmlDeviceGetClockInfo(self.h, self.n.NVML_CLOCK_SM)
            self.n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:  # noqa: BLE001 - sampling is best effort
            pass
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def stop(self):
        self.stop_ev.set()
        self.t.join(timeout=1)
        try:
            mx = self.n.nvmlDeviceGetMaxClockInfo(self.h, self.n.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            mx = None
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": mx,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml, 10 ms"}


def clock_sampler(index: int):
    try:
        return NvmlClockSampler(index)
    except Exception:  # noqa: BLE001 - no NVML: nvidia-smi polling
        return ClockSampler(index)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=1)
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) > 8:
                for k, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(k)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def tile_efficiency(dm, G: int, selected: int) -> dict:
    """Issued M=128 tile steps of attention.cu for a [H, N, N] causal mask: the CTA
    work items of decode_item (4 query groups: 4 heads of a KV group / 2 heads x 2
    query blocks / 1 head x 4 query blocks) and the kernel's pairing of the groups
    into two tiles (smallest longer union, then smallest total; ties keep 01|23)."""
    import torch
    H, N, _ = dm.shape
    if G % 4 == 0:
        M = dm.view(H // 4, 4, N, N).permute(0, 2, 1, 3).reshape(-1, 4, N)
    elif G == 2:
        Np = (N + 1) // 2
        pad = torch.zeros((H, 2 * Np, N), dtype=dm.dtype, device=dm.device)
        pad[:, :N] = dm
        x = pad.view(H // 2, 2, Np, 2, N)              # [kv, head-in-pair, pair, (ia, ib), N]
        M = torch.stack([x[:, 0, :, 1], x[:, 1, :, 1], x[:, 0, :, 0], x[:, 1, :, 0]], 2).reshape(-1, 4, N)
    else:
        Nq = (N + 3) // 4
        pad = torch.zeros((H, 4 * Nq, N), dtype=dm.dtype, device=dm.device)
        pad[:, :N] = dm
        M = pad.view(H, Nq, 4, N).flip(2).reshape(-1, 4, N)
    u = lambda a, b: (M[:, a] | M[:, b]).sum(-1)
    cand = [(u(0, 1), u(2, 3)), (u(0, 2), u(1, 3)), (u(0, 3), u(1, 2))]
    keys = torch.stack([torch.maximum(a, b) * 4096 + a + b for a, b in cand])   # [3, items]
    tot = torch.stack([a + b for a, b in cand])
    best = keys.argmin(0)                                # first minimum = the kernel's strict '<'
    issued = int(tot.gather(0, best[None]).sum().item())
    return {"useful_group_steps": selected, "issued_tile_steps": issued,
            "rows_useful_fraction": selected / (2.0 * issued) if issued else 1.0}


# ----------------------------------------------------------------------------- CPU path
_CPU_CACHE: dict = {}

def cpu_sample(cfg_name, gain, P, seconds_target=12.0, nthreads=0, seed=2512):
    """Times the oracle (reference CPU restatement) on a bounded sample of the
    workload: one KV group at full length, the proxy/selection/attention for a
    stratified sample of (head 0, query block) rows; extrapolated to ms/layer.
    Test infrastructure only (the cpu_baseline leg)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import oracle_py as O
    _, H, H_kv, L, d, mode, sel = CONFIGS[cfg_name]
    G = H // H_kv
    S, N = 64, L // 64
    cores = nthreads or os.cpu_count()
    t0 = time.perf_counter()
    key = (cfg_name, gain)
    if key not in _CPU_CACHE:
        Q, K, V, _ = O.gen_workload(O.WL_PLANTED, L, G, d, S, 2512, H_kv=1, gain=gain, nthreads=cores)
        _CPU_CACHE[key] = (O.bf16_round(Q), O.bf16_round(K), O.bf16_round(V))
    Q, K, V = _CPU_CACHE[key]
    t_gen = time.perf_counter() - t0
    c1 = O.cfg(1, L, d, S, H_kv=1, P=P if mode == "top_p" else 0.95,
               select_mode=O.TOP_P if mode == "top_p" else O.TOP_K, top_k=0 if mode == "top_p" else int(sel))
    t0 = time.perf_counter()
    Qc, Kc = O.compress(c1, Q[:1], K)
    t_compress = time.perf_counter() - t0  # one Q head + one KV head
    # rows: stratified over query blocks (cost grows with i)
    rows_per_round = max(2 * cores, 8)
    rng = np.random.default_rng(seed)
    done_rows, t_rows = 0, 0.0
    n_sel = 0
    while t_rows < seconds_target and done_rows < N:
        strata = np.linspace(0, N, rows_per_round + 1).astype(int)
        qb = np.array([rng.integers(strata[k], max(strata[k] + 1, strata[k + 1])) for k in range(rows_per_round)],
                      np.int32)
        t0 = time.perf_counter()
        srows = O.proxy_score_rows(c1, Qc, Kc, 0, qb, nthreads=cores)
        mask = np.zeros((1, N, N), np.uint8)
        for r, i in enumerate(qb):
            if mode == "top_p":
                idx, _ = O.top_p_row(srows[r, : i + 1], P)
            else:
                idx, _ = O.top_k_row(srows[r, : i + 1], int(sel))
            mask[0, i, idx] = 1
            n_sel += len(idx)
        O.block_sparse_attention_rows(Q[:1], K, V, mask, S, np.zeros(len(qb), np.int32), qb, nthreads=cores)
        t_rows += time.perf_counter() - t0
        done_rows += len(qb)
    per_row = t_rows / done_rows
    ms_layer = 1000.0 * (t_compress * H * (1 + 1.0 / G) / 2 + per_row * H * N)
    sample = (f"oracle (fp64 ref64 restatement) on {cores} threads: full-length compress of 1 Q + 1 KV head, "
              f"proxy+Top-P+sparse attention for {done_rows} stratified (head 0, query block) rows of "
              f"{cfg_name} (N={N}); extrapolated x{H * N / done_rows:.0f} rows to the {H}-head layer")
    return ms_layer, cores, sample, {"t_rows_s": t_rows, "rows": done_rows, "t_compress_s": t_compress,
                                     "t_gen_s": t_gen, "mean_selected_per_row": n_sel / done_rows}


# ----------------------------------------------------------------------------- parity sample
def parity_sample(Q, K, V, eng, mode, sel, P, rows_per_head=6, max_heads=8, seed=2512):
    """Oracle parity record of the measured configuration (tests/gpu_util.py
    oracle_row_parity; test infrastructure, never on the timed path)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from gpu_util import oracle_row_parity
    return oracle_row_parity(Q, K, V, eng.sel, eng.O, mode, sel, P, rows_per_head=rows_per_head,
                             max_heads=max_heads, seed=seed)


# ----------------------------------------------------------------------------- launcher
def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _self_launch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU) with
    torch.distributed.run on 127.0.0.1 and forward their output. N ranks need N
    GPUs with NCCL; with --dist-backend gloo the ranks may share one GPU (a
    functional check of the multi-rank path, never a scaling number)."""
    import torch
    gloo = "gloo" in " ".join(sys.argv)
    if not gloo and torch.cuda.device_count() < n:
        log(f"bench.py: --gpus {n} needs {n} GPUs (found {torch.cuda.device_count()}); "
            "use --dist-backend gloo for a functional multi-rank check on fewer GPUs")
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def _cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_c1_layer(repeats=3):
    """BASELINE.md §3.2 CPU protocol: the reference's CPU path (oracle restatement,
    fp64 on f32 storage) on the WHOLE C1 layer (Llama-3-8B shape 32 Q / 8 KV heads,
    L = 4096, d = 128, S = 64, c = 8, Top-P 0.95, planted gain 8, fp32), per stage,
    best of `repeats`, on 1 thread (the reference hot path is single-threaded) and on
    all host threads (OpenMP over heads). Test infrastructure only."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_py as O
    L, H, H_kv, d, S, P = 4096, 32, 8, 128, 64, 0.95
    Q, K, V, _ = O.gen_workload(O.WL_PLANTED, L, H, d, S, 2512, H_kv=H_kv, gain=8.0)
    c = O.cfg(H, L, d, S, H_kv=H_kv, P=P)
    out = {"config": "C1: 32 Q / 8 KV heads, L=4096, d=128, S=64, c=8, Top-P 0.95, fp32 planted gain 8",
           "cpu_model": _cpu_model(), "nproc": os.cpu_count()}
    for label, nt in (("threads_1", 1), ("threads_all", os.cpu_count() or 1)):
        best = None
        for _ in range(repeats):
            t0 = time.perf_counter()
            Qc, Kc = O.compress(c, Q, K)
            t1 = time.perf_counter()
            sc = O.proxy_scores(c, Qc, Kc, nthreads=nt)
            t2 = time.perf_counter()
            mask = O.build_block_mask(sc, H, 1, P)
            mask = mask[0] if isinstance(mask, tuple) else mask
            t3 = time.perf_counter()
            O.block_sparse_attention(Q, K, V, mask, S, nthreads=nt)
            t4 = time.perf_counter()
            st = {"compress_ms": (t1 - t0) * 1e3, "proxy_ms": (t2 - t1) * 1e3, "select_ms": (t3 - t2) * 1e3,
                  "attention_ms": (t4 - t3) * 1e3, "total_ms": (t4 - t0) * 1e3}
            if best is None or st["total_ms"] < best["total_ms"]:
                best = st
        best["threads"] = nt
        out[label] = best
    out["rho"] = float(1.0 - mask.sum() / (H * (L // S) * (L // S + 1) / 2))
    return out


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--gain", type=float, default=None)
    ap.add_argument("--P", type=float, default=None)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense baselines")
    ap.add_argument("--seed", type=int, default=2512)
    ap.add_argument("--no-flashinfer", action="store_true", help="skip the flashinfer dense prefill baseline")
    ap.add_argument("--dist-backend", default="nccl", help="torch.distributed backend for N>1 (nccl; gloo for checks)")
    ap.add_argument("--e2e-chunks", type=int, default=8, help="KV-head chunks of the pipelined host-buffer path")
    ap.add_argument("--batch", type=int, default=1, help="batch items per layer (partitioned with the heads)")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity sample")
    ap.add_argument("--also-gain", type=float, nargs="*", default=None,
                    help="secondary operating points (planted gain) timed on the device path beside the "
                         "headline (default: 8.0 for C3, the survey's rho ~0.6-0.7 point)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch through torchrun (rank 0 prints the JSON line)
        sys.exit(_self_launch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    desc, H, H_kv, L, d, mode, sel = CONFIGS[args.config]
    gain = args.gain if args.gain is not None else DEFAULT_GAIN[args.config]
    P = args.P if args.P is not None else (sel if mode == "top_p" else 0.95)
    metric = "attention prefill ms/layer @128K; speedup vs dense FA; HBM/TC roofline %"
    base = {"metric": metric, "unit": "ms/layer", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": f"synthetic planted_blocks (reference workloads.cpp semantics, gain={gain}, m=2, sigma=0.1), bf16"}
    config = {"workload": desc, "config": args.config, "heads": H, "kv_heads": H_kv, "seq_len": L,
              "head_dim": d, "block": 64, "c_q": 8, "c_k": 8, "c_h": 1,
              "selection": f"top_p P={P}" if mode == "top_p" else f"top_k k={sel}",
              "causal_mode": "post-softmax-block-causal", "batch": args.batch,
              "parallelism": f"(batch x KV-head)-partitioned x{world} (paper_2512_14082_b200/shard.py "
                             f"shard_layer; no hot-path collective)",
              "l2": "inputs (>=192 MB per rank) exceed the 126 MB L2; no flush needed"}

    if args.impl == "reference":
        if rank != 0:
            return
        samples = []
        info = None
        for s in range(args.warmup + args.steps):
            ms, cores, sample, info = cpu_sample(args.config, gain, P, seconds_target=4.0, seed=args.seed + s)
            if s >= args.warmup:
                samples.append(ms)
        v = statistics.mean(samples)
        c1 = cpu_c1_layer()
        out = dict(base, value=v, impl="reference", ms_per_step=v, config=config,
                   cpu_baseline={"value": v, "unit": "ms/layer", "cores": cores, "kind": "port", "sample": sample,
                                 "c1_full_layer": c1},
                   e2e={"value": v, "unit": "ms/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                   gpu_launches=0, detail=info)
        print(json.dumps(out), flush=True)
        return

    import torch
    import paper_2512_14082_b200 as us
    from paper_2512_14082_b200 import workloads

    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(args.dist_backend, init_method="env://")
    # (modulo: lets a functional multi-rank check share one GPU; one GPU per rank in production)
    torch.cuda.set_device(local % torch.cuda.device_count())
    from paper_2512_14082_b200.shard import gather_layer, imbalance, shard_layer
    shards = shard_layer(args.batch, H, H_kv, world)
    shard = shards[rank]
    G = H // H_kv
    heads = list(shard.q_heads)
    Q, K, V = workloads.planted_blocks(L, H, H_kv, d, 64, seed=args.seed, gain=gain, heads=heads, B=args.batch,
                                       batches=list(shard.batch))
    torch.cuda.synchronize()
    cfg = us.CompressionConfig(P=P) if mode == "top_p" else us.CompressionConfig(
        select_mode=us.SELECT_TOP_K, top_k=int(sel))
    eng = us.Engine(Q, K, V, cfg, head0=shard.q_heads.start)

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if not dist:
            return x
        t = torch.tensor([x], device="cpu" if args.dist_backend == "gloo" else "cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # warm-up + validity check (errors surface here, outside the timed region)
    for _ in range(max(args.warmup, 1)):
        eng.run()
    torch.cuda.synchronize()
    us.api._raise(us.api.lib().us_check_device_errors(us.api.C.byref(eng.p), us.api._ptr(eng.ws), us.api._stream()))
    launches_per_step = eng.launches()
    N = L // 64
    selected = int(eng.sel.counts.to(torch.int64).sum().item())
    per_kv = eng.sel.counts.to(torch.int64).view(len(shard.batch), shard.H_kv, -1).sum(-1) * cfg.c_h  # [B, H_kv]
    # tile efficiency of attn_kernel: each M=128 tile (two 64-row query groups that
    # share a KV head) issues S / P.V for the UNION of its groups' selections
    tile_eff = None
    try:
        dm = eng.sel.dense_mask()
        tile_eff = tile_efficiency(dm[0], G, int(eng.sel.counts[0].to(torch.int64).sum().item()))
        if dm.shape[0] > 1:  # batch: the tile model of item 0 scaled to the whole shard
            tile_eff["issued_tile_steps"] = int(round(tile_eff["issued_tile_steps"] * selected /
                                                      max(tile_eff["useful_group_steps"], 1)))
            tile_eff["useful_group_steps"] = selected
        del dm
    except Exception as e:  # noqa: BLE001 - reporting only
        log("tile efficiency unavailable:", e)
    causal = len(shard.batch) * len(heads) * N * (N + 1) // 2
    rho = 1.0 - selected / causal

    # ---------------------------------------------------------------- parity record (rank 0, untimed)
    # (on the warm-up output: the e2e and dense-baseline legs below overwrite eng.O)
    parity = None
    if rank == 0 and not args.no_parity:
        try:
            parity = parity_sample(Q, K, V, eng, mode, sel, P)
        except Exception as e:  # noqa: BLE001 - report, never hide
            parity = {"error": repr(e)}

    # ---------------------------------------------------------------- timed region (device)
    stream = torch.cuda.current_stream()
    us.api.profile_enable(args.steps)
    clocks = clock_sampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        eng.run()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms_local = e0.elapsed_time(e1) / args.steps
    stages = us.api.profile_read(args.steps)
    us.api.profile_disable()
    ms = max_over_ranks(ms_local)
    stage_ms = {k: statistics.mean(s[k] for s in stages) for k in us.api.STAGES}

    # ---------------------------------------------------------------- e2e (host buffers)
    Qh = torch.empty(Q.shape, dtype=Q.dtype, pin_memory=True).copy_(Q)
    Kh = torch.empty(K.shape, dtype=K.dtype, pin_memory=True).copy_(K)
    Vh = torch.empty(V.shape, dtype=V.dtype, pin_memory=True).copy_(V)
    Oh = torch.empty(Q.shape, dtype=Q.dtype, pin_memory=True)
    O_ref = eng.O.clone()
    eng.O.zero_()
    # Engine.run_host: H2D / hot path / D2H pipelined over KV-head chunks on three
    # streams; the timed region covers every copy of every step (events on the
    # launching stream, which joins the copy-out stream at the end of each step)
    eng.run_host(Qh, Kh, Vh, Oh, chunks=args.e2e_chunks)  # warm-up (stream / event creation)
    torch.cuda.synchronize()
    e2e_exact = bool(torch.equal(Oh.to(eng.O.device), O_ref))
    barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # (a) one call at a time: each step's copies and compute complete before the next starts
    e2.record(stream)
    for _ in range(args.steps):
        eng.run_host(Qh, Kh, Vh, Oh, chunks=args.e2e_chunks)
    e3.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_serial_ms = max_over_ranks(e2.elapsed_time(e3) / args.steps)
    # (b) streaming (the headline): consecutive steps overlap — step s+1 copies chunk
    # c in once step s has computed it (run_host(wait=False)); every step still
    # moves all of its inputs in and its output out inside the timed region
    eng.O.zero_()
    torch.cuda.synchronize()
    barrier()
    e2.record(stream)
    done = None
    for _ in range(args.steps):
        done = eng.run_host(Qh, Kh, Vh, Oh, chunks=args.e2e_chunks, wait=False)
    stream.wait_event(done)
    e3.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(e2.elapsed_time(e3) / args.steps)
    e2e_exact = e2e_exact and bool(torch.equal(Oh.to(eng.O.device), O_ref))
    del O_ref
    # (c) the copy floor: the same H2D and D2H bytes on two streams with no compute (this
    # box's PCIe link does not run both directions at full rate at once)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    e2.record(stream)
    for _ in range(3):
        with torch.cuda.stream(s_in):
            Q.copy_(Qh, non_blocking=True)
            K.copy_(Kh, non_blocking=True)
            V.copy_(Vh, non_blocking=True)
        with torch.cuda.stream(s_out):
            Oh.copy_(eng.O, non_blocking=True)
        stream.wait_stream(s_in)
        stream.wait_stream(s_out)
    e3.record(stream)
    torch.cuda.synchronize()
    copy_floor_ms = e2.elapsed_time(e3) / 3
    def sum_over_ranks(x: float) -> float:
        if not dist:
            return x
        t = torch.tensor([x], device="cpu" if args.dist_backend == "gloo" else "cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    h2d = int(sum_over_ranks((Q.numel() + K.numel() + V.numel()) * 2))
    d2h = int(sum_over_ranks(Q.numel() * 2))

    # ---------------------------------------------------------------- NCCL gather (verification only, untimed)
    gather = None
    if dist:
        t0 = time.perf_counter()
        O_loc = eng.O.cpu() if args.dist_backend == "gloo" else eng.O
        full = gather_layer(O_loc, shards, args.batch, H)
        torch.cuda.synchronize()
        sl = full[shard.batch.start:shard.batch.stop, shard.q_heads.start:shard.q_heads.stop]
        # per-rank selected blocks (max/mean bounds near-linear scaling)
        dev = "cpu" if args.dist_backend == "gloo" else "cuda"
        mine = torch.tensor([float(selected)], device=dev, dtype=torch.float64)
        per_rank = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(per_rank, mine)
        per_rank = [float(t.item()) for t in per_rank]
        gather = {"backend": dist.get_backend(), "ok": bool(torch.equal(sl, O_loc)),
                  "bytes": full.numel() * full.element_size(), "s": time.perf_counter() - t0,
                  "head_imbalance": imbalance(shards),
                  "selected_blocks_per_rank": [int(x) for x in per_rank],
                  "selected_imbalance": max(per_rank) / (sum(per_rank) / world) if sum(per_rank) else 1.0}
        del full, sl

    # ---------------------------------------------------------------- dense baselines (same shard)
    dense = {}
    if not args.no_dense:
        def timeit(fn, iters=3):
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(iters):
                fn()
            b.record(stream)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / iters
        dense["ours_p1"] = max_over_ranks(timeit(lambda: eng.run(dense=True)))
        try:
            from torch.nn.attention import SDPBackend, sdpa_kernel
            with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
                dense["cudnn_sdpa"] = max_over_ranks(timeit(lambda: torch.nn.functional.scaled_dot_product_attention(
                    Q, K, V, is_causal=True, enable_gqa=True)))
        except Exception as e:  # pragma: no cover
            log("cudnn sdpa unavailable:", e)
        try:
            # flashinfer 0.6.11 single-request prefill on sm100 (backend auto = its FA2
            # kernels; the trtllm-gen sm100 cubins serve only the paged batch API)
            if args.no_flashinfer:
                raise RuntimeError("skipped (--no-flashinfer)")
            import flashinfer
            q3, k3, v3 = Q[0].transpose(0, 1).contiguous(), K[0].transpose(0, 1).contiguous(), V[0].transpose(0, 1).contiguous()
            dense["flashinfer"] = max_over_ranks(timeit(lambda: flashinfer.single_prefill_with_kv_cache(
                q3, k3, v3, causal=True)))
            del q3, k3, v3
        except Exception as e:  # pragma: no cover
            log("flashinfer unavailable:", e)
    fastest = min(dense.items(), key=lambda kv: kv[1]) if dense else None

    # ---------------------------------------------------------------- secondary operating points
    # (same shape, other sparsity: the headline gain is the config default; SURVEY §8d
    # asks for C3 at rho ~0.6-0.7 too — gain 8). Device path only, same timing protocol.
    extra_gains = args.also_gain if args.also_gain is not None else ([8.0] if args.config == "C3" and gain != 8.0 else [])
    secondary = []
    if extra_gains:
        del eng
        torch.cuda.empty_cache()
    for g2 in extra_gains:
        Q2, K2, V2 = workloads.planted_blocks(L, H, H_kv, d, 64, seed=args.seed, gain=g2, heads=heads, B=args.batch,
                                              batches=list(shard.batch))
        e2 = us.Engine(Q2, K2, V2, cfg, head0=shard.q_heads.start)
        for _ in range(max(args.warmup, 1)):
            e2.run()
        torch.cuda.synchronize()
        sel2 = int(e2.sel.counts.to(torch.int64).sum().item())
        us.api.profile_enable(args.steps)
        barrier()
        torch.cuda.synchronize()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        for _ in range(args.steps):
            e2.run()
        b_.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms2 = max_over_ranks(a_.elapsed_time(b_) / args.steps)
        st2 = us.api.profile_read(args.steps)
        us.api.profile_disable()
        stage2 = {k: statistics.mean(x[k] for x in st2) for k in us.api.STAGES}
        f2 = sel2 * 4 * 64 * 64 * d / (stage2["attention"] * 1e-3) / 1e12
        secondary.append({"gain": g2, "rho": 1.0 - sel2 / causal, "ms_per_layer": ms2, "stages_ms": stage2,
                          "attention_tflops": f2, "attention_frac": f2 / peaks()[2],
                          "speedup_vs_fastest_dense": (fastest[1] / ms2) if fastest else None})
        del e2, Q2, K2, V2
        torch.cuda.empty_cache()

    # ---------------------------------------------------------------- roofline of the dominant kernel
    hbm, tf_burst, tf_sust, peak_src = peaks()
    flops_attn = selected * 4 * 64 * 64 * d
    dominant = max(stage_ms.items(), key=lambda kv: kv[1])[0]
    # the kernel the device-side density gate runs (attn_common.cuh m64_wins, per (batch
    # item, KV head)): attention64.cu under 55 % of the causal block pairs selected
    kv_pairs = (len(heads) // shard.H_kv) * N * (N + 1) // 2
    m64_frac = float(((per_kv * 20) < kv_pairs * 11).double().mean().item())
    m64 = m64_frac >= 0.5
    if m64:
        # one M = 64 UMMA chain per query group: every issued row is a selected one, and an
        # M = 64 MMA occupies the tensor pipe for the cycles of M = 128 (B300_MICROARCH.md,
        # profiles/r02c/m64_probes.txt), so issued-equivalent = 2 x useful
        issued_attn, rows_useful = selected * 2 * 64 * 64 * 4 * d, 0.5
    else:
        # M = 128 tiles of two query groups run S / P.V for the union of their selections
        issued_attn = (tile_eff["issued_tile_steps"] * 2 * 64 * 64 * 4 * d) if tile_eff else None
        rows_useful = tile_eff["rows_useful_fraction"] if tile_eff else None
    if dominant == "attention":
        achieved = flops_attn / (stage_ms["attention"] * 1e-3) / 1e12
        roof = {"kernel": ("attn64_kernel (tcgen05 M=64 chains, block-sparse FA)" if m64 else
                           "attn_kernel (tcgen05 block-sparse FA)"), "kv_heads_on_attn64": m64_frac,
                "bound": "tensor", "achieved": achieved,
                "peak": tf_sust, "unit": "TFLOP/s", "frac": achieved / tf_sust,
                "algorithmic": "selected_blocks * 4 * S^2 * d (metrics.cpp:83-85)",
                "issued_tflops": issued_attn / (stage_ms["attention"] * 1e-3) / 1e12 if issued_attn else None}
        if issued_attn:
            # an M = 64 MMA costs the cycles of M = 128, so the useful fraction is capped at
            # rows_useful_fraction x the issued fraction (DESIGN.md §3 a6)
            roof["issued_frac"] = roof["issued_tflops"] / tf_sust
            roof["rows_useful_fraction"] = rows_useful
            # tensor-pipe occupancy from the MEASURED issue cost of each MMA (cycles per K = 16
            # instruction, profiles/r02c/m64_probes.txt): S = Q K^T TS-mode N = 64 40.3; P.V SS-mode
            # N = d: M = 64 84.3 (d = 128) / 52.3 (d = 64), M = 128 96.3 / 68.3
            pv = {(True, 128): 84.3, (True, 64): 52.3, (False, 128): 96.3, (False, 64): 68.3}[(m64, d)]
            steps = selected if m64 else tile_eff["issued_tile_steps"]
            cyc = steps * ((d // 16) * 40.3 + 4 * pv)
            roof["tensor_pipe_busy_est"] = cyc / (148 * (clk["sm_mhz"] or 1965.0) * 1e6 * stage_ms["attention"] * 1e-3)
    else:
        Lq = L // 8
        fl = 2 * Lq * Lq * len(heads) * len(shard.batch) * d  # compressed_qk (metrics.cpp:60), post-softmax full square
        achieved = fl / (stage_ms["proxy"] * 1e-3) / 1e12
        roof = {"kernel": "proxy_kernel (tcgen05 fp16x3)", "bound": "tensor", "achieved": achieved, "peak": tf_sust,
                "unit": "TFLOP/s", "frac": achieved / tf_sust,
                "algorithmic": "compressed_qk = 2 (L/c_q)(L/c_k)(H/c_h) d (metrics.cpp:60)",
                "issued_tflops": 3 * achieved}
    roof["traffic"] = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        roof["traffic"] = json.load(open(tp)).get(args.config, {}).get(roof["kernel"].split()[0])
    roof["peak_source"] = f"MEASURED_PEAKS.json ({peak_src}, sustained bf16)"
    comp_bytes = len(shard.batch) * ((len(heads) + shard.H_kv) * L * d * 2 + (len(heads) + shard.H_kv) * (L // 8) * d * 4)
    stage_roofs = {
        "compress": {"bound": "hbm", "bytes": comp_bytes,
                     "achieved_gbs": comp_bytes / (stage_ms["compress"] * 1e-3) / 1e9, "peak_gbs": hbm},
        "attention": {"bound": "tensor", "flops": flops_attn,
                      "achieved_tflops": flops_attn / (stage_ms["attention"] * 1e-3) / 1e12, "peak_tflops": tf_sust},
    }
    # proxy (+ finalize): compressed_qk (metrics.cpp:60) over the post-softmax full square; the
    # tensor pipe issues it three times (fp16x3 hi.hi + hi.lo + lo.hi)
    cq, ck, ch = cfg.c_q, cfg.c_k, cfg.c_h
    qk = 2 * (L // cq) * (L // ck) * (len(heads) // ch) * len(shard.batch) * d
    # MUFU floor: ex2 at 16 results / clock / SM (B300_MICROARCH, measured here by
    # tools/ex2_rate.py) at the sustained clock; the proxy exponentiates every logit of the
    # full square (softmax_aggregation / 4 exps, metrics.cpp:62), the attention kernel 7/8 of
    # its issued P entries (attention.cu sends 1/8 to the FMA-pipe polynomial)
    mufu_per_s = 16 * 148 * (clk["sm_mhz"] or 1965.0) * 1e6
    n_exp_proxy = (L // cq) * (L // ck) * (len(heads) // ch) * len(shard.batch)
    stage_roofs["proxy"] = {"bound": "tensor", "flops": qk,
                            "achieved_tflops": qk / (stage_ms["proxy"] * 1e-3) / 1e12,
                            "issued_tflops": 3 * qk / (stage_ms["proxy"] * 1e-3) / 1e12, "peak_tflops": tf_sust,
                            "mufu_floor_ms": n_exp_proxy / mufu_per_s * 1e3}
    if issued_attn:
        useful_exp = selected * 64 * 64
        # (attention64.cu runs every exponential on the MUFU, attention.cu 7/8 of them)
        stage_roofs["attention"]["mufu_floor_ms"] = useful_exp * (1.0 if m64 else 7 / 8) / mufu_per_s * 1e3
        stage_roofs["attention"]["tensor_floor_ms_issued"] = (issued_attn / (tf_sust * 1e12)) * 1e3

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        v, cores, sample, info = cpu_sample(args.config, gain, P)
        cpu = {"value": v, "unit": "ms/layer", "cores": cores, "kind": "port", "sample": sample,
               "cpu_model": _cpu_model(), "c1_full_layer": cpu_c1_layer()}
    out = dict(base, value=ms, ms_per_step=ms, config=config, clocks=clk,
               e2e={"value": e2e_ms, "unit": "ms/layer", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": f"Engine.run_host(wait=False): pinned host Q/K/V -> H2D -> hot path -> D2H O, "
                            f"{args.e2e_chunks} KV-head chunks on 4 streams (copy-in, 2 compute with 2 chunk workspaces, copy-out), "
                            f"consecutive steps overlapped per chunk",
                    "serial_ms": e2e_serial_ms,
                    "copy_floor_ms": copy_floor_ms,
                    "output_equals_device_path": e2e_exact},
               gpu_launches=launches_per_step * args.steps,
               roofline=roof, cpu_baseline=cpu,
               stages_ms=stage_ms, stage_roofline=stage_roofs,
               sparsity={"rho": rho, "selected_blocks": selected, "causal_blocks": causal, "attn_tiles": tile_eff},
               dense_baselines_ms=dense, verify_gather=gather, parity=parity, secondary_operating_points=secondary,
               speedup_vs_dense={"vs": fastest[0], "dense_ms": fastest[1], "speedup": fastest[1] / ms} if fastest else None)
    print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
