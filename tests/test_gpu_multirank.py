"""The multi-rank path of bench.py with the LIBRARY on every rank:
`bench.py --gpus 2 --dist-backend gloo` self-launches two ranks (they share the one
GPU of a gpurun box; NCCL needs one GPU per rank), each runs the CUDA hot path on its
(batch x KV-head) shard, and rank 0 verifies the all-gathered O against every rank's
own slice; the line must report n_gpus = 2. Also checks that a shard's result equals
the same heads of the one-process layer (head0-seeded stochastic pooling included)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("batch", [1, 2])
def test_bench_two_ranks_gloo(batch):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", "gloo",
                        "--config", "C2", "--steps", "1", "--warmup", "3", "--no-cpu", "--no-dense",
                        "--batch", str(batch)], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["verify_gather"]["ok"], line["verify_gather"]
    assert line["config"]["batch"] == batch
    assert line["parity"]["ok"], line["parity"]


@pytest.mark.parametrize("strategy", [0, 2])
def test_head_shard_equals_full_layer(strategy):
    """Two head shards of a layer, run separately with head0, equal the full layer's
    heads bit for bit — masks and outputs (stochastic pooling seeds by global head)."""
    import paper_2512_14082_b200 as us
    from paper_2512_14082_b200 import workloads
    from paper_2512_14082_b200.shard import shard_layer
    L, H, H_kv, d = 8192, 8, 2, 128
    Q, K, V = workloads.planted_blocks(L, H, H_kv, d, 64, seed=5, gain=8.0)
    cfg = us.CompressionConfig(P=0.95, strategy=strategy, seed=77)
    full = us.unisparse_attn(Q, K, V, cfg)
    for s in shard_layer(1, H, H_kv, 2):
        q = Q[:, s.q_heads.start:s.q_heads.stop].contiguous()
        k = K[:, s.kv_heads.start:s.kv_heads.stop].contiguous()
        v = V[:, s.kv_heads.start:s.kv_heads.stop].contiguous()
        eng = us.Engine(q, k, v, cfg, head0=s.q_heads.start)
        eng.run()
        torch.cuda.synchronize()
        assert torch.equal(eng.sel.mask_bits[0], full.report.mask.mask_bits[0, s.q_heads.start:s.q_heads.stop])
        assert torch.equal(eng.O, full.O[:, s.q_heads.start:s.q_heads.stop])


@pytest.mark.parametrize("strategy", [0, 2])
def test_run_host_chunks_equal_one_call(strategy):
    """Engine.run_host pipelines KV-head chunks (each chunk a head range of the layer,
    head0-seeded): the result equals the one-call device path for every strategy."""
    import paper_2512_14082_b200 as us
    from paper_2512_14082_b200 import workloads
    L, H, H_kv, d = 8192, 8, 4, 128
    Q, K, V = workloads.planted_blocks(L, H, H_kv, d, 64, seed=6, gain=8.0)
    eng = us.Engine(Q, K, V, us.CompressionConfig(P=0.95, strategy=strategy, seed=3))
    eng.run()
    torch.cuda.synchronize()
    ref = eng.O.clone()
    Qh, Kh, Vh = (torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t) for t in (Q, K, V))
    Oh = torch.empty(Q.shape, dtype=Q.dtype, pin_memory=True)
    eng.run_host(Qh, Kh, Vh, Oh, chunks=4)
    torch.cuda.synchronize()
    assert torch.equal(Oh.cuda(), ref)
