"""Head-partitioned multi-GPU path checked on CPU: the shard
arithmetic for every BASELINE config, and a world-size-2 gloo group that runs
the reference path per shard and gathers O with the same all-gather the GPU
verification uses — the gathered layer must equal the single-process layer
bit for bit (the path has no cross-head coupling besides c_h and GQA)."""
import os
import socket

import numpy as np
import pytest

from paper_2512_14082_b200.shard import gather_heads, imbalance, shard_heads


@pytest.mark.parametrize("H,H_kv,world,c_h,sizes,kv", [
    (32, 8, 1, 1, [32], [8]),
    (32, 8, 2, 1, [16, 16], [4, 4]),
    (32, 8, 4, 1, [8] * 4, [2] * 4),
    (32, 8, 8, 1, [4] * 8, [1] * 8),
    (32, 8, 8, 2, [4] * 8, [1] * 8),
    (28, 4, 2, 1, [14, 14], [2, 2]),
    (28, 4, 4, 1, [7] * 4, [1] * 4),
    (28, 4, 8, 1, [4, 3] * 4, [1] * 8),
    (40, 40, 8, 1, [5] * 8, [5] * 8),
    (32, 8, 3, 1, [12, 12, 8], [3, 3, 2]),
])
def test_shard_arithmetic(H, H_kv, world, c_h, sizes, kv):
    sh = shard_heads(H, H_kv, world, c_h)
    assert [s.H for s in sh] == sizes
    assert [s.H_kv for s in sh] == kv
    # contiguous cover of all heads, each head's KV head inside its shard's KV range
    heads = [h for s in sh for h in s.q_heads]
    assert heads == list(range(H))
    G = H // H_kv
    for s in sh:
        assert all(h // G in s.kv_heads for h in s.q_heads)
        assert s.q_heads.start % c_h == 0 and s.H % c_h == 0
        # the shard is a plain layer for the kernels: local head -> local KV head
        assert s.H % s.H_kv == 0
        Gl = s.H // s.H_kv
        assert all((h - s.q_heads.start) // Gl == h // G - s.kv_heads.start for h in s.q_heads)
    assert imbalance(sh) <= 1.0 + 1.0 / min(sizes) + 1e-9


def test_shard_errors():
    with pytest.raises(ValueError):
        shard_heads(32, 8, 16, c_h=4)   # 2 ranks per 4-head group with c_h=4
    with pytest.raises(ValueError):
        shard_heads(28, 4, 6)           # 6 ranks over 4 KV groups
    with pytest.raises(ValueError):
        shard_heads(30, 4, 2)           # H not a multiple of H_kv


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, H, H_kv, c_h, out_path):
    import torch
    import torch.distributed as dist
    import oracle_py as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, d, S, P = 1024, 64, 64, 0.9
    Q, K, V, _ = O.gen_workload(O.WL_PLANTED, L, H, d, S, 31, H_kv=H_kv, gain=8.0)
    Q, K, V = O.bf16_round(Q), O.bf16_round(K), O.bf16_round(V)
    sh = shard_heads(H, H_kv, world, c_h)[rank]
    q = np.ascontiguousarray(Q[sh.q_heads.start:sh.q_heads.stop])
    k = np.ascontiguousarray(K[sh.kv_heads.start:sh.kv_heads.stop])
    v = np.ascontiguousarray(V[sh.kv_heads.start:sh.kv_heads.stop])
    c = O.cfg(sh.H, L, d, S, H_kv=sh.H_kv, c_h=c_h, P=P)
    Ol, _, mask, _ = O.unisparse_attn(c, q, k, v)
    full = gather_heads(torch.from_numpy(Ol).unsqueeze(0), shard_heads(H, H_kv, world, c_h))
    fm = gather_heads(torch.from_numpy(mask.astype(np.uint8)).unsqueeze(0), shard_heads(H, H_kv, world, c_h))
    if rank == 0:
        np.savez(out_path, O=full[0].numpy(), mask=fm[0].numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("H,H_kv,c_h", [(8, 2, 1), (8, 2, 2), (6, 2, 1)])
def test_gloo_world2_gather_equals_single_process(tmp_path, H, H_kv, c_h):
    import torch.multiprocessing as mp
    import oracle_py as O
    out = str(tmp_path / "gathered.npz")
    mp.spawn(_worker, args=(2, _free_port(), H, H_kv, c_h, out), nprocs=2, join=True)
    got = np.load(out)
    L, d, S = 1024, 64, 64
    Q, K, V, _ = O.gen_workload(O.WL_PLANTED, L, H, d, S, 31, H_kv=H_kv, gain=8.0)
    Q, K, V = O.bf16_round(Q), O.bf16_round(K), O.bf16_round(V)
    Or, _, mask, _ = O.unisparse_attn(O.cfg(H, L, d, S, H_kv=H_kv, c_h=c_h, P=0.9), Q, K, V)
    assert np.array_equal(got["mask"].astype(bool), mask)
    assert np.array_equal(got["O"], Or)


# ------------------------------------------------------------------ (batch x head) partitioning
from paper_2512_14082_b200.shard import gather_layer, shard_layer  # noqa: E402


@pytest.mark.parametrize("B,H,H_kv,world,bparts", [
    (1, 32, 8, 8, 1), (2, 32, 8, 8, 2), (4, 32, 8, 8, 4), (8, 32, 8, 8, 8), (8, 32, 8, 2, 2),
    (3, 28, 4, 6, 3), (6, 40, 40, 4, 2), (2, 28, 4, 8, 2),
])
def test_shard_layer_covers_batch_x_heads(B, H, H_kv, world, bparts):
    sh = shard_layer(B, H, H_kv, world)
    assert len(sh) == world
    cells = {(b, h) for s in sh for b in s.batch for h in s.q_heads}
    assert cells == {(b, h) for b in range(B) for h in range(H)}
    assert sum(len(s.batch) * s.H for s in sh) == B * H  # no (b, h) owned twice
    assert len({(s.batch.start, s.batch.stop) for s in sh}) == bparts
    G = H // H_kv
    for s in sh:
        assert all(h // G in s.kv_heads for h in s.q_heads)


def _layer_worker(rank, world, port, B, H, H_kv, out_path):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = shard_layer(B, H, H_kv, world)
    s = sh[rank]
    full_ref = torch.arange(B * H * 3, dtype=torch.float32).reshape(B, H, 3)
    local = full_ref[s.batch.start:s.batch.stop, s.q_heads.start:s.q_heads.stop].contiguous()
    full = gather_layer(local, sh, B, H)
    if rank == 0:
        torch.save({"got": full, "ref": full_ref}, out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B,H,H_kv,world", [(2, 8, 2, 2), (1, 8, 2, 2), (3, 6, 3, 2)])
def test_gloo_gather_layer(tmp_path, B, H, H_kv, world):
    import torch
    import torch.multiprocessing as mp
    out = str(tmp_path / "layer.pt")
    mp.spawn(_layer_worker, args=(world, _free_port(), B, H, H_kv, out), nprocs=world, join=True)
    d = torch.load(out)
    assert torch.equal(d["got"], d["ref"])


def test_bench_rejects_world_mismatch():
    """bench.py --gpus N under a launcher that started a different number of ranks
    must fail (n_gpus is the world size the line reports)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--no-cpu"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode != 0
    assert "--gpus 2 but WORLD_SIZE=1" in (r.stderr + r.stdout)
