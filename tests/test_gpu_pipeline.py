"""End-to-end parity of the GPU pipeline (compress -> proxy -> select -> sparse
attention) against the CPU oracle on the reference's own workload generator.

Contract (north star): block masks bit-exact vs the fp64 reference rule, any
flipped block listed with its decision margin; outputs within the stated bf16
tolerance. Test names mirror test_pipeline.cpp / acceptance.cpp criteria.
"""
import json
import os

import numpy as np
import pytest

import oracle_py as O
from gpu_util import mask_margins, to_dev_bf16, workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


def us():
    import paper_2512_14082_b200 as m
    return m


def _run_case(L, H, H_kv, d, P, mode, c_h, seed, gain=8.0, kind=O.WL_PLANTED, c_q=8, c_k=8, strategy=0):
    Q, K, V, planted = workload(kind, L, H, H_kv, d, seed, gain=gain)
    cfg = us().CompressionConfig(c_q=c_q, c_k=c_k, c_h=c_h, P=P, causal_mode=mode, strategy=strategy, seed=seed)
    res = us().unisparse_attn(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), to_dev_bf16(V, 1), cfg,
                              with_scores=True)
    torch.cuda.synchronize()
    gpu_scores = res.report.mask.scores[0].cpu().numpy()
    gpu_mask = res.report.mask.dense_mask()[0].cpu().numpy()
    c = O.cfg(H, L, d, 64, H_kv=H_kv, c_q=c_q, c_k=c_k, c_h=c_h, causal_mode=mode, P=P, strategy=strategy,
              seed=seed)
    Qc, Kc = O.compress(c, Q, K)
    ref_scores = O.proxy_scores(c, Qc, Kc)
    ref_mask, _ = O.build_block_mask(ref_scores, H, c_h, P)
    return dict(Q=Q, K=K, V=V, res=res, gpu_scores=gpu_scores, gpu_mask=gpu_mask,
                ref_scores=ref_scores, ref_mask=ref_mask, planted=planted, cfg=cfg)


CASES = [
    # L,    H, H_kv, d,  P,    mode,                    c_h, seed
    (4096, 8, 2, 128, 0.95, O.POST_SOFTMAX, 1, 11),
    (4096, 8, 2, 128, 0.90, O.POST_SOFTMAX, 1, 12),
    (4096, 8, 2, 128, 0.95, O.PRE_SOFTMAX, 1, 13),
    (4096, 8, 2, 128, 0.90, O.POST_SOFTMAX, 2, 14),
    (2048, 4, 4, 64, 0.95, O.POST_SOFTMAX, 1, 15),
    (8192, 4, 1, 128, 0.95, O.POST_SOFTMAX, 1, 16),
    (4096, 7, 1, 128, 0.95, O.POST_SOFTMAX, 1, 17),   # Qwen-like odd GQA group (G = 7)
    (2048, 4, 4, 64, 0.9, O.POST_SOFTMAX, 2, 18),     # MHA with c_h = 2 (K pooled per compressed head)
    (4096, 8, 2, 128, 0.95, O.PRE_SOFTMAX, 2, 19),    # pre-softmax with head compression
]


@pytest.mark.parametrize("L,H,H_kv,d,P,mode,c_h,seed", CASES)
def test_masks_bit_exact_vs_reference(L, H, H_kv, d, P, mode, c_h, seed):
    r = _run_case(L, H, H_kv, d, P, mode, c_h, seed)
    N = L // 64
    tri = np.tril(np.ones((N, N), bool))
    # proxy scores: fp16x3 tensor-core proxy vs fp64 reference
    rel = np.abs(r["gpu_scores"] - r["ref_scores"])[:, tri] / np.maximum(r["ref_scores"][:, tri], 1e-30)
    big = r["ref_scores"][:, tri] > 1e-6
    assert np.median(rel[big]) < 1e-5 and rel[big].max() < 1e-3, (np.median(rel[big]), rel[big].max())
    # selection rule on the GPU's own scores == reference rule (exact)
    mirror, _ = O.build_block_mask(r["gpu_scores"].astype(np.float64), H, c_h, P)
    assert (mirror == r["gpu_mask"]).all()
    # masks vs the fp64 reference: list every flipped block with its margin
    flips = np.argwhere(r["gpu_mask"] != r["ref_mask"])
    listed = [dict(head=int(h), **mask_margins(r["ref_scores"][h // c_h, i], P, int(i), int(j)))
              for h, i, j in flips[:50]]
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"mask_flips_L{L}_H{H}_P{P}_m{mode}_ch{c_h}.json"), "w") as f:
        json.dump({"decisions": int(H * N * (N + 1) // 2), "flips": int(len(flips)), "listed": listed}, f, indent=1)
    # a flip is only admissible at a genuine near-tie of the fp64 rule (the fp32-class
    # proxy moves scores by ~1e-7 relative); every flip is listed with its margins
    assert len(flips) == 0 or all(x["mass_margin_rel"] < 1e-6 or x["score_gap_rel"] < 1e-6 for x in listed), listed
    assert len(flips) <= max(2, H * N * (N + 1) // 2 // 20000), f"{len(flips)} flipped blocks: {listed[:5]}"


@pytest.mark.parametrize("P,mode", [(0.95, O.POST_SOFTMAX), (0.9, O.PRE_SOFTMAX)])
def test_output_within_tolerance(P, mode):
    r = _run_case(4096, 4, 2, 128, P, mode, 1, 21)
    Og = r["res"].O.float().cpu().numpy()[0]
    # attention on the GPU's mask, computed by the fp64 oracle
    Or, lser = O.block_sparse_attention(r["Q"], r["K"], r["V"], r["gpu_mask"], 64)
    scale = np.abs(Or).max()
    assert np.abs(Og - Or).max() <= 1e-2 * scale + 1e-4
    assert np.linalg.norm(Og - Or) / np.linalg.norm(Or) <= 1e-2
    assert np.abs(r["res"].lse.cpu().numpy()[0] - lser).max() <= 1e-3
    # fidelity vs dense (criterion 5 analogue): cosine >= 0.99 at P=.95, >= .98 at P=.9
    Od, _ = O.dense_attention(r["Q"], r["K"], r["V"])
    cos = O.output_fidelity(Og, Od)["cosine"]
    assert cos >= (0.99 if P >= 0.95 else 0.98), cos


def test_p1_equals_dense_criterion1():
    Q, K, V, _ = workload(O.WL_GAUSSIAN, 2048, 4, 2, 128, 31)
    cfg = us().CompressionConfig(P=1.0)
    res = us().unisparse_attn(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), to_dev_bf16(V, 1), cfg)
    N = 32
    assert res.report.rho_mean == 0.0
    assert sum(res.report.selected) == 4 * N * (N + 1) // 2
    Od, lsed = O.dense_attention(Q, K, V)
    e_sp = np.abs(res.O.float().cpu().numpy()[0] - Od).max()
    assert e_sp <= 2e-2
    assert np.abs(res.lse.cpu().numpy()[0] - lsed).max() <= 1e-3
    # the sparse kernel at P = 1 is as accurate as the dense kernel (SURVEY §8c level 3)
    Og2, _ = us().dense_attention(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), to_dev_bf16(V, 1))
    e_de = np.abs(Og2.float().cpu().numpy()[0] - Od).max()
    assert e_sp <= 1.5 * e_de, (e_sp, e_de)


def test_monotone_sparsity_and_coverage_criterion4():
    Q, K, V, _ = workload(O.WL_PLANTED, 4096, 4, 2, 128, 41)
    prev = 1.0
    for P in (0.7, 0.8, 0.9, 0.95, 1.0):
        rep = us().select_blocks(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), us().CompressionConfig(P=P))
        assert rep.rho_mean <= prev + 1e-12
        assert rep.mask.coverage.min().item() >= P - 1e-12
        prev = rep.rho_mean
    assert prev == 0.0


def test_planted_recall_criterion5():
    Q, K, V, planted = workload(O.WL_PLANTED, 4096, 4, 2, 128, 51, gain=8.0)
    res = us().unisparse_attn(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), to_dev_bf16(V, 1),
                              us().CompressionConfig(P=0.95))
    m = res.report.mask.dense_mask()[0].cpu().numpy()
    hit = tot = 0
    for h in range(4):
        for i in range(m.shape[1]):
            want = [j for j in planted[h, i] if j >= 0]
            hit += sum(m[h, i, j] for j in want)
            tot += len(want)
    assert hit / tot >= 0.95


def test_top_k_mode():
    Q, K, V, _ = workload(O.WL_PLANTED, 4096, 4, 2, 128, 61)
    k = 8
    cfg = us().CompressionConfig(select_mode=us().SELECT_TOP_K, top_k=k)
    rep = us().select_blocks(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), cfg, with_scores=True)
    got = rep.mask.dense_mask()[0].cpu().numpy()
    c = O.cfg(4, 4096, 128, 64, H_kv=2, select_mode=O.TOP_K, top_k=k)
    Qc, Kc = O.compress(c, Q, K)
    ref, _ = O.build_block_mask(O.proxy_scores(c, Qc, Kc), 4, 1, 0.95, O.TOP_K, k)
    mirror, _ = O.build_block_mask(rep.mask.scores[0].cpu().numpy().astype(np.float64), 4, 1, 0.95, O.TOP_K, k)
    assert (mirror == got).all()
    assert (got != ref).sum() <= 4
    N = 64
    assert (got.sum(-1) == np.minimum(np.arange(N) + 1, k)[None]).all()


def test_batch_independence():
    Q, K, V, _ = workload(O.WL_PLANTED, 2048, 4, 2, 128, 71)
    Q2, K2, V2, _ = workload(O.WL_PLANTED, 2048, 4, 2, 128, 72)
    cfg = us().CompressionConfig(P=0.9)
    qb = torch.stack([to_dev_bf16(Q), to_dev_bf16(Q2)])
    kb = torch.stack([to_dev_bf16(K), to_dev_bf16(K2)])
    vb = torch.stack([to_dev_bf16(V), to_dev_bf16(V2)])
    rb = us().unisparse_attn(qb, kb, vb, cfg)
    r1 = us().unisparse_attn(qb[1:], kb[1:], vb[1:], cfg)
    assert torch.equal(rb.O[1], r1.O[0])
    assert torch.equal(rb.report.mask.mask_bits[1], r1.report.mask.mask_bits[0])


def test_validation_errors_match_reference():
    q = torch.zeros((1, 4, 1000, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError, match="select_blocks: L=1000 not divisible by S=64"):
        us().select_blocks(q, q, us().CompressionConfig())
    q = torch.zeros((1, 4, 1024, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError, match="not divisible by c_q=24"):
        us().select_blocks(q, q, us().CompressionConfig(c_q=24))
    # d_k <= 128 runs zero-padded (tests/test_gpu_dk.py); above 128 is outside the GPU path
    q160 = torch.zeros((1, 4, 1024, 160), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(us().UnsupportedError, match="d_k=160 unsupported on the GPU path"):
        us().select_blocks(q160, q160, us().CompressionConfig())


def test_run_host_pipelined_equals_device_path():
    """Engine.run_host (H2D / hot path / D2H pipelined over KV-head chunks on three
    streams) reproduces the one-call device result bit for bit: heads never couple."""
    from paper_2512_14082_b200 import workloads
    Q, K, V = workloads.planted_blocks(4096, 8, 4, 128, 64, seed=5, gain=8.0)
    eng = us().Engine(Q, K, V, us().CompressionConfig(P=0.9))
    eng.run()
    torch.cuda.synchronize()
    O_ref, mask_ref = eng.O.clone(), eng.sel.mask_bits.clone()
    Qh, Kh, Vh = (t.cpu().pin_memory() for t in (Q, K, V))
    for chunks in (1, 3, 4):
        Oh = torch.empty(Q.shape, dtype=Q.dtype).pin_memory()
        eng.O.zero_()
        eng.run_host(Qh, Kh, Vh, Oh, chunks=chunks)
        torch.cuda.synchronize()
        assert torch.equal(Oh.cuda(), O_ref), chunks
        assert torch.equal(eng.sel.mask_bits, mask_ref), chunks


def test_run_host_streaming_calls_overlap_safely():
    """run_host(wait=False) back to back on DIFFERENT inputs (call n+1's copies and
    kernels overlap call n's per chunk): every call's output equals its own
    one-call device result, so the per-chunk hazards on the engine buffers hold."""
    from paper_2512_14082_b200 import workloads
    ins = [workloads.planted_blocks(4096, 8, 4, 128, 64, seed=s, gain=8.0) for s in (11, 12, 13)]
    refs = []
    for Q, K, V in ins:
        e = us().Engine(Q, K, V, us().CompressionConfig(P=0.9))
        e.run()
        torch.cuda.synchronize()
        refs.append(e.O.clone())
    eng = us().Engine(*ins[0], us().CompressionConfig(P=0.9))
    hosts = [tuple(t.cpu().pin_memory() for t in x) for x in ins]
    outs = [torch.empty(ins[0][0].shape, dtype=ins[0][0].dtype).pin_memory() for _ in ins]
    for chunks in (4, 3):
        for o in outs:
            o.zero_()
        done = None
        for (Qh, Kh, Vh), Oh in zip(hosts * 2, outs * 2):  # two rounds over the three inputs
            done = eng.run_host(Qh, Kh, Vh, Oh, chunks=chunks, wait=False)
        done.synchronize()
        for Oh, ref in zip(outs, refs):
            assert torch.equal(Oh.cuda(), ref), chunks


@pytest.mark.parametrize("strategy", [1, 2])
def test_pooling_ablations_masks_bit_exact(strategy):
    """Max / stochastic pooling end to end (PAPER.md:629 ablation): masks equal the
    reference rule on the reference pooling."""
    r = _run_case(4096, 4, 2, 128, 0.95, O.POST_SOFTMAX, 1, 31 + strategy, strategy=strategy)
    flips = int((r["gpu_mask"] != r["ref_mask"]).sum())
    assert flips == 0, flips


def _fuzz_cases(n=24, seed=2026):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        H_kv = int(rng.choice([1, 2, 4]))
        G = int(rng.choice([1, 2, 3, 4, 7]))
        H = H_kv * G
        if H > 12:
            continue
        c_h = int(rng.choice([c for c in (1, 2, 3, 4) if H % c == 0]))
        c_q, c_k = int(rng.choice([2, 4, 8, 16])), int(rng.choice([2, 4, 8, 16]))
        out.append(dict(L=int(rng.choice([1024, 2048, 3072])), H=H, H_kv=H_kv, d=int(rng.choice([64, 128])),
                        c_q=c_q, c_k=c_k, c_h=c_h, P=float(rng.choice([0.8, 0.9, 0.95, 1.0])),
                        mode=int(rng.choice([O.POST_SOFTMAX, O.PRE_SOFTMAX])),
                        topk=int(rng.choice([0, 0, 3])), seed=int(rng.integers(1 << 30))))
    return out


@pytest.mark.parametrize("case", _fuzz_cases(), ids=lambda c: "L{L}_H{H}_kv{H_kv}_d{d}_c{c_q}x{c_k}x{c_h}_P{P}_m{mode}_k{topk}".format(**c))
def test_fuzz_pipeline_against_oracle(case):
    """Seeded random configurations across the GPU envelope (GQA groups incl. odd,
    head compression, every S/c, post / pre softmax, Top-P and top-k): the mask is
    the reference rule applied to the GPU's scores (exact), scores are fp32-class
    close to the fp64 reference, flips vs the fp64 rule stay near-tie only, and the
    output equals fp64 sparse attention on the GPU's mask within the bf16 bound."""
    c = case
    Q, K, V, _ = workload(O.WL_PLANTED, c["L"], c["H"], c["H_kv"], c["d"], c["seed"] % 1000, gain=8.0)
    sm = us().SELECT_TOP_K if c["topk"] else us().SELECT_TOP_P
    cfg = us().CompressionConfig(c_q=c["c_q"], c_k=c["c_k"], c_h=c["c_h"], P=c["P"], causal_mode=c["mode"],
                                 select_mode=sm, top_k=c["topk"])
    res = us().unisparse_attn(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), to_dev_bf16(V, 1), cfg, with_scores=True)
    torch.cuda.synchronize()
    H, N = c["H"], c["L"] // 64
    g_scores = res.report.mask.scores[0].cpu().numpy().astype(np.float64)
    g_mask = res.report.mask.dense_mask()[0].cpu().numpy()
    oc = O.cfg(H, c["L"], c["d"], 64, H_kv=c["H_kv"], c_q=c["c_q"], c_k=c["c_k"], c_h=c["c_h"],
               causal_mode=c["mode"], P=c["P"])
    Qc, Kc = O.compress(oc, Q, K)
    r_scores = O.proxy_scores(oc, Qc, Kc)
    sel = O.TOP_K if c["topk"] else O.TOP_P
    mirror, _ = O.build_block_mask(g_scores, H, c["c_h"], c["P"], select_mode=sel, top_k=c["topk"])
    assert (mirror == g_mask).all()
    tri = np.tril(np.ones((N, N), bool))
    big = r_scores[:, tri] > 1e-6
    rel = np.abs(g_scores - r_scores)[:, tri][big] / r_scores[:, tri][big]
    assert rel.max() < 1e-3, rel.max()
    ref_mask, _ = O.build_block_mask(r_scores, H, c["c_h"], c["P"], select_mode=sel, top_k=c["topk"])
    flips = np.argwhere(ref_mask != g_mask)
    assert len(flips) <= max(2, H * N * (N + 1) // 2 // 20000)
    # every flip vs the fp64 rule must sit at a near-tie (listed with its margins)
    margins = [dict(head=int(h), **mask_margins(r_scores[h // c["c_h"]], c["P"] if not c["topk"] else 1.0, int(i), int(j)))
               for h, i, j in flips]
    assert all(m["mass_margin_rel"] < 1e-6 or m["score_gap_rel"] < 1e-6 for m in margins), margins
    Og = res.O.float().cpu().numpy()[0]
    Or, _ = O.block_sparse_attention(Q, K, V, g_mask, 64)
    assert np.abs(Og - Or).max() <= 1e-2 * np.abs(Or).max() + 1e-4


@pytest.mark.parametrize("S,d,mode,c", [(128, 64, 0, 8), (128, 128, 0, 8), (128, 64, 1, 8), (128, 128, 0, 16),
                                        (256, 64, 0, 16)])
def test_block_size_above_64_matches_oracle(S, d, mode, c):
    """S = 128 (the reference acceptance battery's block size, acceptance.cpp:53-60) and
    S = 256: compress / proxy / select run at block size S (rq = S / c_q composite rows
    per block); attention walks the 64-granular expansion of the S-block mask, whose
    diagonal S-block keeps exactly the token-level causal pairs (attention.cpp:117-118).
    Masks bit-exact and outputs within the bf16 tolerance vs the oracle at the same S."""
    L, H, H_kv = 4096, 4, 2
    Q, K, V, _ = O.gen_workload(O.WL_PLANTED, L, H, d, S, 77 + S + d, H_kv=H_kv, gain=8.0)
    Q, K, V = O.bf16_round(Q), O.bf16_round(K), O.bf16_round(V)
    cfg = us().CompressionConfig(P=0.95, causal_mode=mode, c_q=c, c_k=c)
    res = us().unisparse_attn(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), to_dev_bf16(V, 1), cfg, S=S)
    torch.cuda.synchronize()
    gmask = res.report.mask.dense_mask()[0].cpu().numpy()
    c_o = O.cfg(H, L, d, S, H_kv=H_kv, P=0.95, causal_mode=mode, c_q=c, c_k=c)
    Or, lser, ref_mask, _ = O.unisparse_attn(c_o, Q, K, V)
    assert gmask.shape == ref_mask.shape == (H, L // S, L // S)
    assert int((gmask != ref_mask).sum()) == 0
    Og = res.O[0].float().cpu().numpy()
    assert np.abs(Og - Or).max() <= 1e-2 * np.abs(Or).max() + 1e-4
    assert np.linalg.norm(Og - Or) / np.linalg.norm(Or) <= 1e-2
    assert np.abs(res.lse[0].cpu().numpy() - lser).max() <= 2e-3 * max(1.0, np.abs(lser).max())
    # block_sparse_attention on the S-block mask directly equals the pipeline's attention
    O2, _ = us().block_sparse_attention(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), to_dev_bf16(V, 1),
                                        res.report.mask.mask_bits, heads_per_plane=1, S=S)
    assert torch.equal(O2, res.O)


@pytest.mark.parametrize("strategy,c_h", [(0, 1), (2, 2)])
def test_batch_items_equal_single_item_calls(strategy, c_h):
    """Batch (the north star's B dimension): a B = 3 layer equals three B = 1 calls on
    its items bit for bit — masks, outputs, lse — for mean and stochastic pooling."""
    L, H, H_kv, d = 2048, 4, 2, 128
    items = [workload(O.WL_PLANTED, L, H, H_kv, d, 500 + b) for b in range(3)]
    cfg = us().CompressionConfig(P=0.95, strategy=strategy, c_h=c_h, seed=9)
    Qb = torch.stack([to_dev_bf16(it[0], 1)[0] for it in items]).contiguous()
    Kb = torch.stack([to_dev_bf16(it[1], 1)[0] for it in items]).contiguous()
    Vb = torch.stack([to_dev_bf16(it[2], 1)[0] for it in items]).contiguous()
    rb = us().unisparse_attn(Qb, Kb, Vb, cfg)
    for b in range(3):
        r1 = us().unisparse_attn(Qb[b:b + 1].contiguous(), Kb[b:b + 1].contiguous(), Vb[b:b + 1].contiguous(), cfg)
        assert torch.equal(rb.report.mask.mask_bits[b], r1.report.mask.mask_bits[0])
        assert torch.equal(rb.O[b], r1.O[0])
        assert torch.equal(rb.lse[b], r1.lse[0])
