"""GPU parity for the individual kernels against the CPU oracle.

* tcgen05 building blocks (every operand path used by proxy / attention)
* compress: bit-exact vs the oracle's restatement of compression.hpp:13-76
* selection: bit-exact vs top_p_row / build_block_mask on the same f32 scores
* attention: within tolerance of the fp64 oracle on the same bf16 inputs
"""
import math

import numpy as np
import pytest

import oracle_py as O
from gpu_util import to_dev_bf16

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def us():
    import paper_2512_14082_b200 as m
    return m


# ------------------------------------------------------------------ tcgen05 building blocks
@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("N", [64, 128])
@pytest.mark.parametrize("bf16", [False, True])
def test_umma_operand_paths(mode, N, bf16):
    g = torch.Generator().manual_seed(100 + mode * 10 + N)
    dt = torch.bfloat16 if bf16 else torch.float16
    A = torch.randn(128, 128, generator=g).to(dt)
    if mode == 4:  # A given as A^T [K][M] (MN-major A), B [K][N]
        Bm = torch.randn(128, N, generator=g).to(dt)
        ref = A.float().T @ Bm.float()
    elif mode in (1, 3):
        Bm = torch.randn(128, N, generator=g).to(dt)   # [K][N], N contiguous
        ref = A.float() @ Bm.float()
    else:
        Bm = torch.randn(N, 128, generator=g).to(dt)   # [N][K]
        ref = A.float() @ Bm.float().T
    D = us().api.selftest_umma(mode, N, bf16, A.cuda().contiguous(), Bm.cuda().contiguous())
    torch.cuda.synchronize()
    err = (D.cpu() - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), f"mode {mode} N {N} bf16 {bf16}: max err {err}"


# ------------------------------------------------------------------ compress
@pytest.mark.parametrize("c_q,c_k,c_h,H,H_kv", [
    (8, 8, 1, 8, 2), (4, 8, 2, 8, 2), (1, 1, 1, 4, 4), (64, 64, 4, 8, 8),
    (8, 4, 8, 8, 2), (2, 16, 1, 4, 1), (8, 8, 2, 8, 8)])
def test_compress_bit_exact(c_q, c_k, c_h, H, H_kv):
    rng = np.random.default_rng(c_q * 100 + c_k * 10 + c_h)
    B, L, d = 2, 512, 128
    Q = O.bf16_round(rng.standard_normal((B, H, L, d)).astype(np.float32) * 3)
    K = O.bf16_round(rng.standard_normal((B, H_kv, L, d)).astype(np.float32))
    cfg = us().CompressionConfig(c_q=c_q, c_k=c_k, c_h=c_h)
    Qc, Kc = us().compress(to_dev_bf16(Q), to_dev_bf16(K), cfg)
    Qc, Kc = Qc.cpu().numpy(), Kc.cpu().numpy()
    for b in range(B):
        c = O.cfg(H, L, d, 64, H_kv=H_kv, c_q=c_q, c_k=c_k, c_h=c_h)
        rq, rk = O.compress(c, Q[b], K[b])
        assert (Qc[b].view(np.uint32) == rq.view(np.uint32)).all()
        assert (Kc[b].view(np.uint32) == rk.view(np.uint32)).all()


@pytest.mark.parametrize("c", [2, 8, 16, 64])
def test_compress_wide_exponent_spread_bit_exact(c):
    """Mean pooling with one element per window scaled by 10^U(-6, 4) plus signed
    zeros, denormal-range and huge values (SURVEY §8a-1 probe 2): the fp32
    fast path must defer every inexact window to the fp64 path."""
    rng = np.random.default_rng(c)
    B, H, L, d = 1, 2, 512, 64
    Q = rng.standard_normal((B, H, L, d)).astype(np.float32)
    Q[:, :, ::c] *= (10.0 ** rng.uniform(-6, 4, size=(B, H, L // c, d))).astype(np.float32)
    Q[0, 0, :c] = -0.0                      # all -0 window: the sum is +0
    Q[0, 1, :c, :8] = 1e-38                 # sums in the f32 denormal range after / c
    Q[0, 1, c:2 * c, :8] = 3e38             # overflowing window sum (fp64 keeps it finite)
    Q = O.bf16_round(Q)
    K = O.bf16_round(rng.standard_normal((B, H, L, d)).astype(np.float32))
    cfg = us().CompressionConfig(c_q=c, c_k=c, c_h=1)
    Qc, Kc = us().compress(to_dev_bf16(Q), to_dev_bf16(K), cfg)
    rq, rk = O.compress(O.cfg(H, L, d, 64, c_q=c, c_k=c, c_h=1), Q[0], K[0])
    assert (Qc[0].cpu().numpy().view(np.uint32) == rq.view(np.uint32)).all()
    assert (Kc[0].cpu().numpy().view(np.uint32) == rk.view(np.uint32)).all()


@pytest.mark.parametrize("strategy", [1, 2])  # POOL_MAX, POOL_STOCHASTIC
@pytest.mark.parametrize("c_q,c_k,c_h,H,H_kv", [(8, 8, 1, 8, 2), (4, 8, 2, 8, 2), (8, 8, 2, 4, 4),
                                               (64, 16, 1, 4, 1), (1, 2, 1, 2, 2)])
def test_compress_strategies_bit_exact(strategy, c_q, c_k, c_h, H, H_kv):
    """Max and stochastic pooling (compression.hpp:30-53; ablations of PAPER.md:629):
    the stochastic pick uses the reference's SplitMix64 stream chain(chain(seed,
    role, head), window) and row-norm weights, so the picked rows equal the oracle's."""
    rng = np.random.default_rng(strategy * 1000 + c_q * 10 + c_h)
    B, L, d = 2, 512, 128
    Q = O.bf16_round(rng.standard_normal((B, H, L, d)).astype(np.float32) * 3)
    K = O.bf16_round(rng.standard_normal((B, H_kv, L, d)).astype(np.float32))
    Q[0, 0, :64] = 0.0  # all-zero windows: the stochastic rule falls back to next_u64() % c
    cfg = us().CompressionConfig(c_q=c_q, c_k=c_k, c_h=c_h, strategy=strategy, seed=987654321)
    Qc, Kc = us().compress(to_dev_bf16(Q), to_dev_bf16(K), cfg)
    Qc, Kc = Qc.cpu().numpy(), Kc.cpu().numpy()
    for b in range(B):
        c = O.cfg(H, L, d, 64, H_kv=H_kv, c_q=c_q, c_k=c_k, c_h=c_h, strategy=strategy, seed=987654321)
        rq, rk = O.compress(c, Q[b], K[b])
        assert (Qc[b].view(np.uint32) == rq.view(np.uint32)).all()
        assert (Kc[b].view(np.uint32) == rk.view(np.uint32)).all()


# ------------------------------------------------------------------ selection on given scores
def _random_planes(rng, planes, N, kind):
    s = rng.random((planes, N, N)).astype(np.float32)
    if kind == "ties":
        s = (np.floor(s * 4) / 4).astype(np.float32)         # many exact ties incl. zeros
    elif kind == "skewed":
        s = np.exp(rng.standard_normal((planes, N, N)) * 4).astype(np.float32)
    elif kind == "zeros":
        s[:, ::3, :] = 0.0                                   # all-zero rows -> diagonal rule
    tri = np.tril(np.ones((N, N), bool))
    return np.where(tri[None], s, 0).astype(np.float32)


@pytest.mark.parametrize("kind", ["uniform", "ties", "skewed", "zeros"])
@pytest.mark.parametrize("P", [0.3, 0.5, 0.9, 0.95, 1.0])
@pytest.mark.parametrize("N", [5, 64, 200])
def test_select_matches_reference_rule(kind, P, N):
    rng = np.random.default_rng(hash((kind, P, N)) % 2**32)
    planes = 3
    s = _random_planes(rng, planes, N, kind)
    cfg = us().CompressionConfig(P=P)
    sel = us().build_block_mask(torch.from_numpy(s).cuda(), cfg, with_indices=True)
    torch.cuda.synchronize()
    got = sel.dense_mask()[0].cpu().numpy()
    ref, cov = O.build_block_mask(s.astype(np.float64), planes, 1, P)
    assert (got == ref).all(), f"{(got != ref).sum()} flips"
    assert np.allclose(sel.coverage[0].cpu().numpy(), cov, rtol=0, atol=1e-12)
    counts = sel.counts[0].cpu().numpy()
    assert (counts == ref.sum(-1)).all()
    idx = sel.indices[0].cpu().numpy()
    for p in range(planes):
        for i in range(N):
            assert list(idx[p, i, : counts[p, i]]) == list(np.nonzero(ref[p, i])[0])


@pytest.mark.parametrize("k", [1, 3, 32])
def test_select_top_k(k):
    rng = np.random.default_rng(k)
    s = _random_planes(rng, 2, 100, "ties")
    cfg = us().CompressionConfig(select_mode=us().SELECT_TOP_K, top_k=k)
    got = us().build_block_mask(torch.from_numpy(s).cuda(), cfg).dense_mask()[0].cpu().numpy()
    ref, _ = O.build_block_mask(s.astype(np.float64), 2, 1, 0.95, O.TOP_K, k)
    assert (got == ref).all()


def test_select_kat_rows():
    # selection KATs (test_selection.cpp:33-63) as f32 rows, plus exact-tie boundary cases
    rows = [([0.5, 0.3, 0.2], 0.7), ([0.4, 0.4, 0.2], 0.5), ([0.6, 0.4], 0.6),
            ([0.1, 0.0, 0.9, 0.0], 1.0), ([0.0, 0.0, 0.0], 0.9), ([0.5, 0.25, 0.25], 0.5),
            ([0.25, 0.25, 0.25, 0.25], 0.5), ([0.125] * 8, 0.75)]
    for vals, P in rows:
        n = len(vals)
        s = np.zeros((1, n, n), np.float32)
        s[0, n - 1, :] = vals
        for i in range(n - 1):
            s[0, i, : i + 1] = 1.0
        sel = us().build_block_mask(torch.from_numpy(s).cuda(), us().CompressionConfig(P=P))
        got = sel.dense_mask()[0, 0, n - 1].cpu().numpy()
        idx, _ = O.top_p_row(np.array(vals, np.float32).astype(np.float64), P)
        ref = np.zeros(n, bool)
        ref[idx] = True
        assert (got == ref).all(), (vals, P, got, ref)


def test_select_rejects_negative_scores():
    s = np.zeros((1, 4, 4), np.float32)
    s[0, 2, :3] = [0.5, -0.1, 0.2]
    s[0, np.arange(4), np.arange(4)] += 1
    with pytest.raises(ValueError, match="nonnegative"):
        us().build_block_mask(torch.from_numpy(s).cuda(), us().CompressionConfig(P=0.9))


# ------------------------------------------------------------------ attention
def _rand_qkv(rng, B, H, H_kv, L, d, scale=1.0):
    Q = O.bf16_round(rng.standard_normal((B, H, L, d)).astype(np.float32) * scale)
    K = O.bf16_round(rng.standard_normal((B, H_kv, L, d)).astype(np.float32))
    V = O.bf16_round(rng.standard_normal((B, H_kv, L, d)).astype(np.float32))
    return Q, K, V


def _bits_from_mask(mask: np.ndarray) -> np.ndarray:
    B, P_, N, _ = mask.shape
    W = (N + 31) // 32
    pad = np.zeros((B, P_, N, W * 32), bool)
    pad[..., :N] = mask
    w = (pad.reshape(B, P_, N, W, 32).astype(np.uint64) << np.arange(32, dtype=np.uint64)).sum(-1)
    return w.astype(np.uint32).view(np.int32)


# bf16 output + bf16 P: tolerance per element relative to the V scale
ATOL, RTOL_FRO = 2e-2, 1e-2


@pytest.mark.parametrize("H,H_kv,d", [(4, 2, 128), (4, 1, 128), (2, 2, 128), (6, 3, 64), (4, 4, 64)])
def test_sparse_attention_random_masks(H, H_kv, d):
    rng = np.random.default_rng(H * 10 + H_kv + d)
    B, L = 2, 1024
    N = L // 64
    Q, K, V = _rand_qkv(rng, B, H, H_kv, L, d)
    mask = rng.random((B, H, N, N)) < 0.4
    tri = np.tril(np.ones((N, N), bool))
    mask &= tri
    mask[..., np.arange(N), np.arange(N)] |= rng.random((B, H, N)) < 0.5
    empty = ~mask.any(-1)
    mask[empty, 0] = True  # keep rows non-empty
    Og, lseg = us().block_sparse_attention(to_dev_bf16(Q), to_dev_bf16(K), to_dev_bf16(V),
                                           torch.from_numpy(_bits_from_mask(mask)).cuda())
    Og = Og.float().cpu().numpy()
    lseg = lseg.cpu().numpy()
    for b in range(B):
        Or, lser = O.block_sparse_attention(Q[b], K[b], V[b], mask[b], 64)
        err = np.abs(Og[b] - Or)
        assert err.max() <= ATOL, f"b={b} max_abs={err.max()}"
        assert np.linalg.norm(Og[b] - Or) / np.linalg.norm(Or) <= RTOL_FRO
        assert np.abs(lseg[b] - lser).max() <= 1e-3


def test_dense_attention_matches_oracle_and_sdpa():
    rng = np.random.default_rng(7)
    B, H, H_kv, L, d = 1, 4, 2, 2048, 128
    Q, K, V = _rand_qkv(rng, B, H, H_kv, L, d)
    Og, lseg = us().dense_attention(to_dev_bf16(Q), to_dev_bf16(K), to_dev_bf16(V))
    Og = Og.float().cpu().numpy()
    Or, lser = O.dense_attention(Q[0], K[0], V[0])
    assert np.abs(Og[0] - Or).max() <= ATOL
    assert np.abs(lseg.cpu().numpy()[0] - lser).max() <= 1e-3
    # torch fp32 reference of the same op
    q = torch.from_numpy(Q).cuda()
    k = torch.from_numpy(K).cuda().repeat_interleave(H // H_kv, 1)
    v = torch.from_numpy(V).cuda().repeat_interleave(H // H_kv, 1)
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True).cpu().numpy()
    assert np.abs(Og - ref).max() <= ATOL


@pytest.mark.parametrize("H,H_kv,d", [(4, 2, 128), (2, 2, 64)])
def test_dense_attention_noncausal_matches_oracle(H, H_kv, d):
    """dense_attention(in, causal = false) (attention.cpp:20-54): every key block,
    no diagonal mask; vs the fp64 oracle and torch fp32 SDPA without a causal mask."""
    rng = np.random.default_rng(9 + d)
    B, L = 1, 1024
    Q, K, V = _rand_qkv(rng, B, H, H_kv, L, d)
    Og, lseg = us().dense_attention(to_dev_bf16(Q), to_dev_bf16(K), to_dev_bf16(V), causal=False)
    Or, lser = O.dense_attention(Q[0], K[0], V[0], causal=False)
    assert np.abs(Og.float().cpu().numpy()[0] - Or).max() <= ATOL
    assert np.abs(lseg.cpu().numpy()[0] - lser).max() <= 1e-3
    q = torch.from_numpy(Q).cuda()
    k = torch.from_numpy(K).cuda().repeat_interleave(H // H_kv, 1)
    v = torch.from_numpy(V).cuda().repeat_interleave(H // H_kv, 1)
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=False).cpu().numpy()
    assert np.abs(Og.float().cpu().numpy() - ref).max() <= ATOL


def test_sparse_attention_large_logits_finite():
    rng = np.random.default_rng(3)
    Q, K, V = _rand_qkv(rng, 1, 2, 1, 512, 128, scale=30.0)
    Og, lse = us().dense_attention(to_dev_bf16(Q), to_dev_bf16(K), to_dev_bf16(V))
    Or, _ = O.dense_attention(Q[0], K[0], V[0])
    assert torch.isfinite(lse).all()
    assert np.abs(Og.float().cpu().numpy()[0] - Or).max() <= 3e-2


def test_sparse_attention_rejects_malformed_masks():
    rng = np.random.default_rng(5)
    Q, K, V = _rand_qkv(rng, 1, 2, 2, 256, 64)
    N = 4
    m = np.tril(np.ones((1, 2, N, N), bool))
    m[0, 1, 2, :] = False
    with pytest.raises(ValueError, match="no selected key block"):
        us().block_sparse_attention(to_dev_bf16(Q), to_dev_bf16(K), to_dev_bf16(V),
                                    torch.from_numpy(_bits_from_mask(m)).cuda())
    m = np.tril(np.ones((1, 2, N, N), bool))
    m[0, 0, 1, 3] = True
    with pytest.raises(ValueError, match="non-causal"):
        us().block_sparse_attention(to_dev_bf16(Q), to_dev_bf16(K), to_dev_bf16(V),
                                    torch.from_numpy(_bits_from_mask(m)).cuda())


@pytest.mark.parametrize("H,H_kv,d", [(8, 4, 128), (4, 4, 64), (6, 2, 128), (3, 1, 128)])
def test_attention_impls_agree(H, H_kv, d):
    """attention.cu (64-key steps, two tiles per CTA) and the calibration variants —
    attention2.cu (128-key steps, one tile per CTA), the one-tile attention.cu, the
    key-major attention_kt.cu, the decoupled-softmax attention_tp.cu (P in TMEM,
    double-buffered logits, split K / V rings) and the M = 64 chains of attention64.cu —
    on the same random masks, odd union lengths included: all equal the fp64 oracle
    within the bf16 tolerance."""
    import ctypes
    rng = np.random.default_rng(H * 100 + d)
    B, L = 2, 1024
    N = L // 64
    Q, K, V = _rand_qkv(rng, B, H, H_kv, L, d)
    mask = rng.random((B, H, N, N)) < 0.4
    mask &= np.tril(np.ones((N, N), bool))
    mask[..., np.arange(N), np.arange(N)] = True
    bits = torch.from_numpy(_bits_from_mask(mask)).cuda()
    with us().api.calibration() as lib:  # the variants live in the calibration build
        try:
            for impl in ((6, 5, 4, 3, 2, 1) if d == 128 else (6, 5, 3, 2, 1)):
                assert lib.us_set_attention_impl(impl) == 0
                Og, lseg = us().block_sparse_attention(to_dev_bf16(Q), to_dev_bf16(K), to_dev_bf16(V), bits)
                Og = Og.float().cpu().numpy()
                lseg = lseg.cpu().numpy()
                for b in range(B):
                    Or, lser = O.block_sparse_attention(Q[b], K[b], V[b], mask[b], 64)
                    assert np.abs(Og[b] - Or).max() <= ATOL, (impl, b)
                    assert np.linalg.norm(Og[b] - Or) / np.linalg.norm(Or) <= RTOL_FRO, (impl, b)
                    assert np.abs(lseg[b] - lser).max() <= 1e-3, (impl, b)
        finally:
            lib.us_set_attention_impl(0)


@pytest.mark.parametrize("density", [0.08, 0.3, 0.45, 0.55, 0.7, 0.9])
@pytest.mark.parametrize("H,H_kv,d", [(8, 2, 128), (6, 3, 64)])
def test_automatic_choice_follows_the_density_gate(density, H, H_kv, d):
    """impl 0 with a mask launches attention64.cu and attention.cu; the device-side gate
    (attn_common.cuh m64_wins: under 55 % of the causal block pairs of a (batch item, KV
    head) selected) lets exactly one of them write each KV group's heads. The automatic
    output must equal, bit for bit, the forced run of the kernel the rule picks on the
    host-counted density of that (item, KV head)."""
    rng = np.random.default_rng(int(density * 100) + H)
    B, L = 2, 2048
    N, G = L // 64, H // H_kv
    Q, K, V = (to_dev_bf16(x) for x in _rand_qkv(rng, B, H, H_kv, L, d))
    mask = rng.random((B, H, N, N)) < density * rng.uniform(0.8, 1.2, (B, H, 1, 1))
    mask &= np.tril(np.ones((N, N), bool))
    mask[..., np.arange(N), np.arange(N)] = True
    bits = torch.from_numpy(_bits_from_mask(mask)).cuda()
    out = {}
    try:
        for impl in (0, 1, 6):
            _set_impl(impl)
            Og, lseg = us().block_sparse_attention(Q, K, V, bits)
            out[impl] = (Og.clone(), lseg.clone())
    finally:
        _set_impl(0)
    picks = set()
    for b in range(B):
        for g in range(H_kv):
            hs = slice(g * G, (g + 1) * G)
            frac = mask[b, hs].sum() / (G * N * (N + 1) / 2)
            want = 6 if frac * 20 < 11 else 1
            picks.add(want)
            assert torch.equal(out[0][0][b, hs], out[want][0][b, hs]), (b, g, frac, want)
            assert torch.equal(out[0][1][b, hs], out[want][1][b, hs]), (b, g, frac, want)


@pytest.mark.parametrize("N,H,H_kv,d", [(33, 8, 2, 128), (45, 6, 6, 64), (45, 7, 1, 128), (1, 4, 1, 128),
                                          (2, 8, 2, 64)])
def test_attention64_odd_block_counts(N, H, H_kv, d):
    """attention64.cu (forced, and through the automatic gate) at block counts that end
    mid-word of the 32-bit mask rows, with GQA, MHA and G = 7 (a CTA's four chains drawn
    from different heads and query blocks by the sorted item table): equal to the fp64
    oracle within the bf16 tolerance."""
    rng = np.random.default_rng(N * 10 + H)
    B, L = 2, N * 64
    Q, K, V = _rand_qkv(rng, B, H, H_kv, L, d)
    mask = rng.random((B, H, N, N)) < 0.25
    mask &= np.tril(np.ones((N, N), bool))
    mask[..., np.arange(N), np.arange(N)] = True
    bits = torch.from_numpy(_bits_from_mask(mask)).cuda()
    try:
        for impl in (6, 0):
            _set_impl(impl)
            Og, lseg = us().block_sparse_attention(to_dev_bf16(Q), to_dev_bf16(K), to_dev_bf16(V), bits)
            Og = Og.float().cpu().numpy()
            lseg = lseg.cpu().numpy()
            for b in range(B):
                Or, lser = O.block_sparse_attention(Q[b], K[b], V[b], mask[b], 64)
                assert np.abs(Og[b] - Or).max() <= ATOL, (impl, b)
                assert np.linalg.norm(Og[b] - Or) / np.linalg.norm(Or) <= RTOL_FRO, (impl, b)
                assert np.abs(lseg[b] - lser).max() <= 1e-3, (impl, b)
    finally:
        _set_impl(0)


def test_product_library_has_no_calibration_variants():
    """The product library runs attention.cu only: the calibration variants (2-5) and the
    probes are absent from libunisparse_b200.so (they live in the calibration build)."""
    lib = us().api.lib()
    assert lib.us_set_attention_impl(2) == us().api.US_ERR_UNSUPPORTED
    assert lib.us_set_attention_impl(4) == us().api.US_ERR_UNSUPPORTED
    assert lib.us_set_attention_impl(5) == us().api.US_ERR_UNSUPPORTED
    assert lib.us_set_attention_impl(0) == 0
    assert not hasattr(lib, "us_selftest_umma")


def _set_impl(impl):
    assert us().api.lib().us_set_attention_impl(impl) == 0


@pytest.mark.parametrize("growth", [0.0, 1.0, -1.0])
def test_attention_kt_offset_moves(growth):
    """Key-major kernel: the per-query offsets only move when a logit exceeds them
    by > 16 (log2). Key blocks whose logits GROW along the ascending walk force a
    rescale of O^T and of the row-sum partials at many steps (growth 1), shrinking
    logits never rescale after the first step (growth -1); both equal the fp64 oracle.
    Rows with odd and even counts, with and without the diagonal block."""
    rng = np.random.default_rng(11)
    B, H, H_kv, L, d = 1, 4, 2, 2048, 128
    N = L // 64
    Q, K, V = _rand_qkv(rng, B, H, H_kv, L, d)
    blk = np.arange(L) // 64  # per key row: logits grow (shrink) by ~17 log2 units per block
    scale = {0.0: np.ones(L), 1.0: 1 + 4.0 * blk, -1.0: 1 + 4.0 * (N - 1 - blk)}[growth].astype(np.float32)
    K = (K * scale[None, None, :, None]).astype(np.float32)
    mask = rng.random((B, H, N, N)) < 0.5
    mask &= np.tril(np.ones((N, N), bool))
    mask[0, 0, np.arange(N), np.arange(N)] = False  # head 0: never the diagonal unless forced
    empty = ~mask.any(-1)
    mask[empty, 0] = True
    bits = torch.from_numpy(_bits_from_mask(mask)).cuda()
    for impl in (4, 1):
        with us().api.calibration():
            _set_impl(impl)
            try:
                Og, lseg = us().block_sparse_attention(to_dev_bf16(Q), to_dev_bf16(K), to_dev_bf16(V), bits)
            finally:
                _set_impl(0)
        Og = Og.float().cpu().numpy()
        lseg = lseg.cpu().numpy()
        Qr, Kr, Vr = (O.bf16_round(x) for x in (Q, K, V))
        Or, lser = O.block_sparse_attention(Qr[0], Kr[0], Vr[0], mask[0], 64)
        assert np.isfinite(Og).all() and np.isfinite(lseg).all()
        assert np.abs(Og[0] - Or).max() <= ATOL * max(1.0, np.abs(Or).max()), impl
        assert np.linalg.norm(Og[0] - Or) / np.linalg.norm(Or) <= RTOL_FRO, impl
        assert np.abs(lseg[0] - lser).max() <= 1e-3 * max(1.0, np.abs(lser).max()), impl


@pytest.mark.parametrize("H,H_kv,density", [(8, 2, 0.3), (16, 4, 0.15), (8, 1, 0.6)])
def test_attention_tile_pairing_is_invisible(H, H_kv, density):
    """The per-CTA tile pairing (groups paired by union size) only changes which
    tile / lanes a query group runs in: outputs and lse are bit-identical to the
    fixed (01|23) pairing. Per-head densities differ so the pairing does move."""
    import ctypes
    rng = np.random.default_rng(H * 10 + H_kv)
    B, L, d = 1, 2048, 128
    N = L // 64
    Q, K, V = _rand_qkv(rng, B, H, H_kv, L, d)
    dens = density * rng.uniform(0.3, 1.7, size=(1, H, 1, 1))
    mask = rng.random((B, H, N, N)) < dens
    mask &= np.tril(np.ones((N, N), bool))
    mask[..., np.arange(N), np.arange(N)] = True
    bits = torch.from_numpy(_bits_from_mask(mask)).cuda()
    q, k, v = to_dev_bf16(Q), to_dev_bf16(K), to_dev_bf16(V)
    lib = us().api.lib()
    lib.us_set_attention_pairing.argtypes = [ctypes.c_int32]
    try:
        out = []
        for on in (0, 1):
            assert lib.us_set_attention_pairing(on) == 0
            Og, lseg = us().block_sparse_attention(q, k, v, bits)
            out.append((Og.clone(), lseg.clone()))
        assert torch.equal(out[0][0], out[1][0])
        assert torch.equal(out[0][1], out[1][1])
    finally:
        lib.us_set_attention_pairing(1)


# ------------------------------------------------------------------ competitor proxy (antidiagonal)
@pytest.mark.parametrize("H,H_kv,d,stride,P", [(4, 2, 128, 8, 0.9), (2, 2, 64, 4, 0.95), (4, 1, 128, 16, 0.9)])
def test_antidiagonal_proxy_matches_reference(H, H_kv, d, stride, P):
    """XAttention-style strided anti-diagonal scorer (baselines.cpp:10-52) on the GPU:
    scores within fp32-class error of the fp64 restatement, masks equal the
    reference rule on the reference scores."""
    L, S = 2048, 64
    Q, K, V, _ = O.gen_workload(O.WL_PLANTED, L, H, d, S, 77 + stride, H_kv=H_kv, gain=8.0)
    Q, K = O.bf16_round(Q), O.bf16_round(K)
    cfg = us().CompressionConfig(P=P)
    rep = us().select_blocks(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), cfg, proxy=us().api.PROXY_ANTIDIAGONAL,
                             stride=stride, with_scores=True)
    torch.cuda.synchronize()
    N = L // S
    tri = np.tril(np.ones((N, N), bool))
    gs = rep.mask.scores[0].cpu().numpy()
    rs = O.antidiagonal_block_scores(Q, K, S, stride)
    big = rs[:, tri] > 1e-6
    rel = np.abs(gs[:, tri] - rs[:, tri])[big] / rs[:, tri][big]
    assert np.median(rel) < 1e-5 and rel.max() < 1e-3, (np.median(rel), rel.max())
    ref_mask, _ = O.build_block_mask(rs, H, 1, P)
    got = rep.mask.dense_mask()[0].cpu().numpy()
    assert int((got != ref_mask).sum()) == 0


@pytest.mark.parametrize("H,H_kv,d,P", [(4, 2, 128, 0.9), (2, 2, 64, 0.95)])
def test_last_block_probe_matches_reference(H, H_kv, d, P):
    """FlexPrefill-style last-block probe (baselines.cpp:54-87) on the GPU: column
    masses within fp32-class error, masks equal the reference rule."""
    L, S = 2048, 64
    Q, K, V, _ = O.gen_workload(O.WL_PLANTED, L, H, d, S, 91, H_kv=H_kv, gain=8.0)
    Q, K = O.bf16_round(Q), O.bf16_round(K)
    rep = us().select_blocks(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), us().CompressionConfig(P=P),
                             proxy=us().api.PROXY_LAST_BLOCK, with_scores=True)
    torch.cuda.synchronize()
    N = L // S
    tri = np.tril(np.ones((N, N), bool))
    gs = rep.mask.scores[0].cpu().numpy()
    rs = O.last_block_probe_scores(Q, K, S)
    big = rs[:, tri] > 1e-6
    rel = np.abs(gs[:, tri] - rs[:, tri])[big] / rs[:, tri][big]
    assert np.median(rel) < 1e-5 and rel.max() < 1e-3, (np.median(rel), rel.max())
    ref_mask, _ = O.build_block_mask(rs, H, 1, P)
    assert int((rep.mask.dense_mask()[0].cpu().numpy() != ref_mask).sum()) == 0
