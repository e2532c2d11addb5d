"""Head partitioning of one attention layer across the GPUs of a box (north
star item 4).

Every hot-path quantity is per (batch, head) except two couplings: head-group
pooling / broadcast over c_h consecutive Q heads (compression.hpp:61-76,
selection.cpp:80-84) and GQA sharing of a K/V head by G = H/H_kv Q heads. A
shard is therefore a contiguous range of Q heads that never splits a c_h group
and that is either a run of WHOLE KV groups or a sub-range of ONE KV group (the
K/V head is then replicated on the ranks sharing it — Qwen 28Q/4KV on 8 GPUs:
7-head groups split 4 + 3). Inside a shard the kernels see an ordinary layer
with H' Q heads and H'_kv K/V heads, so the hot path has no collective.

Batch items are independent as well: shard_layer() splits the world into
gcd(world, B) batch parts times world/gcd head parts, so every rank owns a
(batch range x head range) block of the [B][H][L][d] layer.

NCCL (torch.distributed) is used only to gather the per-rank O slices for
verification (gather_heads / gather_layer); with the head-major [B][H][L][d]
layout the gather is a placement of (batch, head) blocks.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List


@dataclasses.dataclass(frozen=True)
class Shard:
    rank: int
    q_heads: range    # global Q heads owned by this rank
    kv_heads: range   # global K/V heads they read
    batch: range = range(0, 1)  # batch items owned by this rank (shard_layer)

    @property
    def H(self) -> int:
        return len(self.q_heads)

    @property
    def H_kv(self) -> int:
        return len(self.kv_heads)


def _balanced(n: int, parts: int) -> List[int]:
    return [n // parts + (1 if r < n % parts else 0) for r in range(parts)]


def shard_heads(H: int, H_kv: int, world: int, c_h: int = 1) -> List[Shard]:
    """Partition H query heads over `world` ranks (see module docstring).

    world <= H_kv: whole KV groups per rank, balanced (counts differ by at most
    one group). world > H_kv: world must be a multiple of H_kv; each KV group's
    G heads are split into world/H_kv balanced, c_h-aligned sub-ranges.
    """
    if H <= 0 or H_kv <= 0 or H % H_kv:
        raise ValueError(f"H={H} must be a positive multiple of H_kv={H_kv}")
    if c_h <= 0 or H % c_h:
        raise ValueError(f"H={H} not divisible by c_h={c_h}")
    if world <= 0:
        raise ValueError("world size must be positive")
    G = H // H_kv
    shards = []
    if world <= H_kv:
        if G % c_h and H_kv > 1 and world > 1:
            raise ValueError(f"c_h={c_h} groups straddle KV groups of {G} heads")
        kv0 = 0
        for r, n in enumerate(_balanced(H_kv, world)):
            shards.append(Shard(r, range(kv0 * G, (kv0 + n) * G), range(kv0, kv0 + n)))
            kv0 += n
        return shards
    if world % H_kv:
        raise ValueError(f"{world} ranks do not divide into {H_kv} KV groups")
    per = world // H_kv
    if G % c_h:
        raise ValueError(f"c_h={c_h} does not divide the {G} heads of a KV group")
    units = G // c_h
    if units < per:
        raise ValueError(f"KV group of {G} heads (c_h={c_h}) cannot feed {per} ranks")
    r = 0
    for kv in range(H_kv):
        h0 = kv * G
        for n in _balanced(units, per):
            shards.append(Shard(r, range(h0, h0 + n * c_h), range(kv, kv + 1)))
            h0 += n * c_h
            r += 1
    return shards


def shard_layer(B: int, H: int, H_kv: int, world: int, c_h: int = 1) -> List[Shard]:
    """Partition a [B][H] layer over `world` ranks by (batch, KV-head group): the
    world splits into bp = gcd(world, B) batch parts x hp = world / bp head parts
    (shard_heads over hp ranks); rank r owns batch part r // hp, head part r % hp.
    No collective is needed on the hot path (batch items and KV groups never couple)."""
    if B <= 0:
        raise ValueError("B must be positive")
    if world <= 0:
        raise ValueError("world size must be positive")
    bp = math.gcd(world, B)
    hp = world // bp
    heads = shard_heads(H, H_kv, hp, c_h)
    per_b = B // bp
    out = []
    for r in range(world):
        hs = heads[r % hp]
        b0 = (r // hp) * per_b
        out.append(Shard(r, hs.q_heads, hs.kv_heads, range(b0, b0 + per_b)))
    return out


def gather_layer(local, shards: List[Shard], B: int, H: int, group=None):
    """All-gather per-rank [B_r][H_r][...] blocks into the full [B][H][...] tensor
    (verification only). Blocks are padded to the largest shard for the collective."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    Bm = max(len(s.batch) for s in shards)
    Hm = max(s.H for s in shards)
    pad = torch.zeros((Bm, Hm) + tuple(local.shape[2:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0], : local.shape[1]] = local
    tmp = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(tmp, pad.contiguous(), group=group)
    full = torch.empty((B, H) + tuple(local.shape[2:]), dtype=local.dtype, device=local.device)
    for t, s in zip(tmp, shards):
        full[s.batch.start:s.batch.stop, s.q_heads.start:s.q_heads.stop] = t[: len(s.batch), : s.H]
    return full


def imbalance(shards: List[Shard]) -> float:
    """max / mean Q heads per rank (1.0 = perfectly balanced)."""
    sizes = [s.H for s in shards]
    return max(sizes) / (sum(sizes) / len(sizes))


def gather_heads(local, shards: List[Shard], group=None):
    """All-gather per-rank [B][H_r][...] slices into the full [B][H][...] tensor
    (verification only — never on the timed path). Works with NCCL (CUDA
    tensors) and gloo (CPU tensors)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    shapes = [(local.shape[0], s.H) + tuple(local.shape[2:]) for s in shards]
    bufs = [torch.empty(sh, dtype=local.dtype, device=local.device) for sh in shapes]
    if len({s.H for s in shards}) == 1:
        dist.all_gather(bufs, local.contiguous(), group=group)
    else:  # uneven shards: pad to the largest, gather, trim
        Hm = max(s.H for s in shards)
        pad = torch.zeros((local.shape[0], Hm) + tuple(local.shape[2:]), dtype=local.dtype, device=local.device)
        pad[:, : local.shape[1]] = local
        tmp = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(tmp, pad, group=group)
        bufs = [t[:, : s.H] for t, s in zip(tmp, shards)]
    return torch.cat(bufs, dim=1)
