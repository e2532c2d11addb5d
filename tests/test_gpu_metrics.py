"""GPU quality metrics (metrics.cpp:100-224, attention.cpp:56-86)
against the oracle restatement: exact block mass within fp32-accumulation error,
and output_fidelity / block_recall / mean_row_spearman bit-identical to the
oracle on the same inputs (mean_rel: the reference sums all entries in one
running sum, the GPU per row first — fp64-rounding close)."""
import numpy as np
import pytest

import oracle_py as O
from gpu_util import to_dev_bf16, workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def us():
    import paper_2512_14082_b200 as m
    return m


def _bits(mask: np.ndarray) -> np.ndarray:
    """bool [..., N, N] -> int32 words [..., N, W]"""
    N = mask.shape[-1]
    W = (N + 31) // 32
    out = np.zeros(mask.shape[:-1] + (W,), np.uint32)
    for j in range(N):
        out[..., j // 32] |= mask[..., j].astype(np.uint32) << np.uint32(j % 32)
    return out.view(np.int32)


@pytest.mark.parametrize("H,H_kv,d,L", [(4, 2, 64, 1024), (2, 2, 128, 2048), (4, 1, 128, 512)])
def test_exact_block_mass_matches_oracle(H, H_kv, d, L):
    Q, K, V, _ = workload(O.WL_PLANTED, L, H, H_kv, d, 31 + H + d)
    mass = us().exact_block_mass(to_dev_bf16(Q, 1), to_dev_bf16(K, 1))[0].cpu().numpy().astype(np.float64)
    ref = O.exact_block_mass(Q, K, 64)
    N = L // 64
    tri = np.tril(np.ones((N, N), bool))
    assert np.all(mass[:, ~tri] == O.K_MASKED_SCORE)
    err = np.abs(mass[:, tri] - ref[:, tri])
    assert err.max() <= 2e-5 * 64, err.max()
    # each query row's mass sums to 1 over its causal keys: 64 per block row
    assert np.allclose(np.where(tri, mass, 0.0).sum(-1), 64.0, rtol=2e-5)


def test_output_fidelity_matches_oracle():
    rng = np.random.default_rng(4)
    B, H, L, d = 1, 3, 256, 64
    a = O.bf16_round(rng.standard_normal((H, L, d)).astype(np.float32))
    b = O.bf16_round(a + 0.01 * rng.standard_normal((H, L, d)).astype(np.float32))
    b[0, 5] = 0.0  # one zero reference row
    a[1, 7] = 0.0
    b[1, 7] = 0.0  # both zero: cosine 1 by convention
    got = us().output_fidelity(to_dev_bf16(a, 1), to_dev_bf16(b, 1))
    want = O.output_fidelity(a, b)
    assert got["max_abs"] == want["max_abs"]
    assert got["cosine"] == want["cosine"]
    assert got["mean_rel"] == pytest.approx(want["mean_rel"], rel=1e-12)
    same = us().output_fidelity(to_dev_bf16(a, 1), to_dev_bf16(a, 1))
    assert same["max_abs"] == 0.0 and same["mean_rel"] == 0.0 and same["cosine"] == pytest.approx(1.0, rel=1e-12)


def test_block_recall_kats_on_gpu():  # test_metrics.cpp:124-152
    M = O.K_MASKED_SCORE
    ref = np.array([[[5.0, M, M], [1.0, 2.0, M], [3.0, 1.0, 2.0]]], np.float32)
    m = np.zeros((1, 3, 3), bool)
    for i, js in enumerate([[0], [1], [0, 2]]):
        m[0, i, js] = True
    bits = torch.from_numpy(_bits(m)).cuda()
    r = torch.from_numpy(ref).cuda()
    assert us().block_recall(bits, r, 2) == pytest.approx(5.0 / 6.0, rel=1e-12)
    assert us().block_recall(bits, r, 1) == pytest.approx(1.0, rel=1e-12)
    assert us().block_recall(bits, r, 3) == pytest.approx((1.0 + 0.5 + 2.0 / 3.0) / 3.0, rel=1e-12)
    for bad in (0, 4):
        with pytest.raises(ValueError, match="k out of range"):
            us().block_recall(bits, r, bad)
    ref = torch.tensor([[[1.0, M], [2.0, 2.0]]], dtype=torch.float32).cuda()
    for rows, want in (([[0], [0]], 1.0), ([[0], [1]], 0.5)):
        m = np.zeros((1, 2, 2), bool)
        for i, js in enumerate(rows):
            m[0, i, js] = True
        assert us().block_recall(torch.from_numpy(_bits(m)).cuda(), ref, 1) == pytest.approx(want)


@pytest.mark.parametrize("N,k,ties", [(96, 2, False), (300, 7, True), (64, 64, True), (40, 1, True)])
def test_block_recall_matches_oracle(N, k, ties):
    rng = np.random.default_rng(N + k)
    H = 3
    ref = rng.random((H, N, N)).astype(np.float32)
    if ties:
        ref = np.round(ref * 4) / 4  # many exact ties: the lower index wins
    tri = np.tril(np.ones((N, N), bool))
    ref = np.where(tri, ref, O.K_MASKED_SCORE).astype(np.float32)
    mask = (rng.random((H, N, N)) < 0.3) & tri
    got = us().block_recall(torch.from_numpy(_bits(mask)).cuda(), torch.from_numpy(ref).cuda(), k)
    assert got == O.block_recall(mask, ref.astype(np.float64), k)


def test_block_recall_heads_per_plane():
    rng = np.random.default_rng(9)
    H, N, c_h = 4, 50, 2
    tri = np.tril(np.ones((N, N), bool))
    ref = np.where(tri, rng.random((H, N, N)), O.K_MASKED_SCORE).astype(np.float32)
    planes = (rng.random((H // c_h, N, N)) < 0.4) & tri
    got = us().block_recall(torch.from_numpy(_bits(planes)).cuda(), torch.from_numpy(ref).cuda(), 3,
                            heads_per_plane=c_h)
    assert got == O.block_recall(np.repeat(planes, c_h, axis=0), ref.astype(np.float64), 3)


def test_mean_row_spearman_kats_on_gpu():  # test_metrics.cpp:164-222
    M = O.K_MASKED_SCORE
    rng = np.random.default_rng(3)
    p = np.full((1, 6, 6), M, np.float32)
    for i in range(6):
        p[0, i, :i + 1] = rng.random(i + 1)
    pt = torch.from_numpy(p).cuda()
    mean, d, u = us().mean_row_spearman(pt, pt, 1)
    assert mean == pytest.approx(1.0, rel=1e-12) and (d, u) == (5, 0)
    p4 = p[:, :4, :4].copy()
    mean, d, _ = us().mean_row_spearman(torch.from_numpy(p4).cuda(), torch.from_numpy(np.concatenate([p4, p4])).cuda(), 2)
    assert mean == pytest.approx(1.0, rel=1e-12) and d == 6
    with pytest.raises(ValueError, match="head counts disagree"):
        us().mean_row_spearman(torch.from_numpy(p4).cuda(), torch.from_numpy(np.concatenate([p4, p4])).cuda(), 1)
    p = np.full((1, 3, 3), M, np.float32)
    p[0, 0, 0] = 1.0
    p[0, 1, :2] = [0.5, 0.5]
    p[0, 2, :3] = [0.3, 0.2, 0.1]
    q = p.copy()
    q[0, 1, :2] = [0.9, 0.1]
    mean, d, u = us().mean_row_spearman(torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda(), 1)
    assert (d, u) == (1, 1) and mean == pytest.approx(1.0, rel=1e-12)


@pytest.mark.parametrize("H,c_h,N,quant", [(2, 1, 130, 0), (4, 2, 64, 8), (2, 2, 257, 3), (1, 1, 1100, 0)])
def test_mean_row_spearman_matches_oracle(H, c_h, N, quant):
    """Average ranks with ties (quantised values), broadcast planes, non-power-of-two rows."""
    rng = np.random.default_rng(H * 1000 + N)
    tri = np.tril(np.ones((N, N), bool))
    proxy = rng.random((H // c_h, N, N))
    ref = rng.random((H, N, N)) + 0.3 * np.repeat(proxy, c_h, axis=0)
    if quant:
        proxy = np.floor(proxy * quant) / quant
        ref = np.floor(ref * quant) / quant
    proxy = np.where(tri, proxy, O.K_MASKED_SCORE).astype(np.float32)
    ref = np.where(tri, ref, O.K_MASKED_SCORE).astype(np.float32)
    got = us().mean_row_spearman(torch.from_numpy(proxy).cuda(), torch.from_numpy(ref).cuda(), c_h)
    want = O.mean_row_spearman(proxy.astype(np.float64), ref.astype(np.float64), c_h)
    assert got == want


def test_metrics_on_the_pipeline():
    """End to end as run_experiment scores one task (experiment.cpp:345-372): GPU
    proxy scores + mask + sparse output against the GPU dense output and exact mass,
    each metric equal to the oracle's on the same GPU-produced arrays."""
    L, H, H_kv, d = 2048, 4, 2, 64
    Q, K, V, _ = workload(O.WL_PLANTED, L, H, H_kv, d, 77)
    q, k, v = to_dev_bf16(Q, 1), to_dev_bf16(K, 1), to_dev_bf16(V, 1)
    cfg = us().CompressionConfig(P=0.9)
    res = us().unisparse_attn(q, k, v, cfg, with_scores=True)
    dense, _ = us().dense_attention(q, k, v)
    mass = us().exact_block_mass(q, k)
    fid = us().output_fidelity(res.O, dense)
    want = O.output_fidelity(res.O[0].float().cpu().numpy(), dense[0].float().cpu().numpy())
    assert fid["cosine"] == want["cosine"] and fid["max_abs"] == want["max_abs"]
    assert fid["cosine"] > 0.9
    scores = res.report.mask.scores
    sp = us().mean_row_spearman(scores, mass, cfg.c_h)
    assert sp == O.mean_row_spearman(scores[0].double().cpu().numpy(), mass[0].double().cpu().numpy(), cfg.c_h)
    assert sp[0] > 0.0
    bits = res.report.mask.mask_bits
    rec = us().block_recall(bits, mass, 2)
    mask = res.report.mask.dense_mask(H)[0].cpu().numpy()
    assert rec == O.block_recall(mask, mass[0].double().cpu().numpy(), 2)
    assert 0.5 < rec <= 1.0


def test_run_experiment_writes_reference_files(tmp_path):
    """run_experiment (experiment.cpp:280-437) on the GPU: one row per grid point x
    proxy in the reference nesting order, metrics.csv / records / run_meta written,
    each row's numbers equal to the direct metric calls."""
    import json
    from paper_2512_14082_b200 import experiment as E
    L, H, H_kv, d = 2048, 4, 2, 64
    Q, K, V, _ = workload(O.WL_PLANTED, L, H, H_kv, d, 91)
    q, k, v = to_dev_bf16(Q, 1), to_dev_bf16(K, 1), to_dev_bf16(V, 1)
    grid = E.Grid(c_h=(1, 2), P=(0.9,))
    proxies = (0, 1, 2)
    rows = E.run_experiment(q, k, v, grid=grid, proxies=proxies, stride=8, planted_m=2, out_dir=str(tmp_path))
    assert [(r.c_h, r.proxy) for r in rows] == [(1, 0), (1, 1), (1, 2), (2, 0), (2, 1), (2, 2)]
    lines = (tmp_path / "metrics.csv").read_text().splitlines()
    assert lines[0] == E.CSV_HEADER and len(lines) == 7
    assert lines[1].startswith("unisparse,8,8,1,mean,0.9,")
    assert len(list((tmp_path / "records").glob("run_*.json"))) == 6
    rec = json.loads((tmp_path / "records" / "run_0003.json").read_text())
    assert rec["settings"]["c_h"] == 2 and rec["settings"]["run_index"] == 3
    # row 0 by hand
    mass = us().exact_block_mass(q, k)
    dense, _ = us().dense_attention(q, k, v)
    rep = us().select_blocks(q, k, us().CompressionConfig(P=0.9), with_scores=True)
    sp, _, _ = us().mean_row_spearman(rep.mask.scores, mass, 1)
    assert rows[0].spearman == sp and rows[0].rho == rep.rho_mean
    assert rows[0].recall == us().block_recall(rep.mask.mask_bits, mass, 2)
    sparse, _ = us().block_sparse_attention(q, k, v, rep.mask.mask_bits)
    assert rows[0].cosine == us().output_fidelity(sparse, dense)["cosine"]
    assert all(0.0 < r.recall <= 1.0 and 0.0 < r.cosine <= 1.0 and 0.0 < r.rho < 1.0 for r in rows)
    assert rows[0].cosine > 0.9
    with pytest.raises(E.ValidationError, match="stride must divide S"):
        E.run_experiment(q, k, v, grid=grid, proxies=(1,), stride=3)


def test_planted_recall_on_gpu():  # test_metrics.cpp:154-161 and the generator's planted sets
    m = np.zeros((1, 3, 3), bool)
    for i, js in enumerate([[0], [0, 1], [0, 2]]):
        m[0, i, js] = True
    planted = torch.tensor([[[-1, -1], [0, -1], [1, 2]]], dtype=torch.int32).cuda()
    bits = torch.from_numpy(_bits(m)).cuda()
    assert us().planted_recall(bits, planted) == pytest.approx(0.75, rel=1e-12)
    with pytest.raises(ValueError, match="no planted rows"):
        us().planted_recall(bits, torch.full((1, 3, 2), -1, dtype=torch.int32).cuda())
    # the planted workload through the GPU pipeline: equal to the oracle on the same mask
    L, H, H_kv, d = 4096, 4, 2, 64
    Q, K, V, pl = workload(O.WL_PLANTED, L, H, H_kv, d, 23)
    rep = us().select_blocks(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), us().CompressionConfig(P=0.9))
    got = us().planted_recall(rep.mask.mask_bits, torch.from_numpy(pl).cuda())
    want = O.planted_recall(rep.mask.dense_mask(H)[0].cpu().numpy(), pl)
    assert got == want and got > 0.5


def _small_inputs(seed=5):
    Q, K, V, _ = workload(O.WL_PLANTED, 2048, 2, 2, 64, seed)
    return to_dev_bf16(Q, 1), to_dev_bf16(K, 1), to_dev_bf16(V, 1)


def test_run_experiment_p1_rows_are_dense_and_grid_order():  # test_experiment.cpp:99-133
    from paper_2512_14082_b200 import experiment as E
    q, k, v = _small_inputs()
    rows = E.run_experiment(q, k, v, grid=E.Grid(P=(0.9, 1.0)), proxies=(0, 2))
    assert [(r.P, r.proxy) for r in rows] == [(0.9, 0), (0.9, 2), (1.0, 0), (1.0, 2)]
    for r in rows[2:]:
        assert r.rho == 0.0 and r.max_abs == 0.0 and r.cosine >= 1.0 - 1e-9
    assert rows[0].rho > 0.0


def test_run_experiment_coarser_compression_cuts_selection_flops():  # test_experiment.cpp:135-144
    from paper_2512_14082_b200 import experiment as E
    q, k, v = _small_inputs()
    rows = E.run_experiment(q, k, v, grid=E.Grid(c_q=(1, 2, 4, 8), c_k=(4,)))
    assert all(rows[i].selection_flops < rows[i - 1].selection_flops for i in range(1, 4))


def test_run_experiment_rejects_inconsistent_grids_upfront(tmp_path):  # test_experiment.cpp:85-97
    from paper_2512_14082_b200 import experiment as E
    q, k, v = _small_inputs()
    with pytest.raises(E.ValidationError, match="not divisible by c_q=48"):
        E.run_experiment(q, k, v, grid=E.Grid(c_q=(4, 48)), out_dir=str(tmp_path / "x"))
    assert not (tmp_path / "x").exists()  # nothing ran, nothing written


def test_run_experiment_is_byte_deterministic(tmp_path):  # test_experiment.cpp:146-160
    """Repeated GPU runs emit byte-identical metrics.csv and records (only
    run_meta.json carries timestamps): every kernel on the path is deterministic."""
    from paper_2512_14082_b200 import experiment as E
    q, k, v = _small_inputs()
    grid = E.Grid(strategy=(0, 2))
    for d in ("a", "b"):
        E.run_experiment(q, k, v, grid=grid, proxies=(0, 1), out_dir=str(tmp_path / d), seed=7)
    a, b = tmp_path / "a", tmp_path / "b"
    assert (a / "metrics.csv").read_bytes() == (b / "metrics.csv").read_bytes()
    for n in ("run_0000.json", "run_0003.json"):
        assert (a / "records" / n).read_bytes() == (b / "records" / n).read_bytes()
