"""Pins the CPU oracle against the reference's own known-answer tests.

Each test cites the reference test it ports (/root/reference/proj/tests/...).
Random inputs are regenerated with the ported CounterRng exactly the way the
reference's `random_inputs` helpers draw them (q, k, v interleaved per element),
so these run on the same numbers the reference suite used.
"""
import math

import numpy as np
import pytest

import oracle_py as O


def random_inputs(H, L, d, seed):
    """test_proxy.cpp:14-34 / test_attention.cpp:13-33 (q, k, v interleaved)."""
    g = O.rng_draws(seed, "gaussian", 3 * H * L * d).astype(np.float32).reshape(H, L, d, 3)
    return (np.ascontiguousarray(g[..., 0]), np.ascontiguousarray(g[..., 1]),
            np.ascontiguousarray(g[..., 2]))


def random_matrix(rows, cols, seed):
    """test_compression.cpp:13-19."""
    return O.rng_draws(seed, "gaussian", rows * cols).astype(np.float32).reshape(rows, cols)


# ------------------------------------------------------------------ RNG (test_core.cpp:173-214)
def test_rng_reproducible_and_order_sensitive():
    a = O.rng_draws(42, "u64", 100)
    b = O.rng_draws(42, "u64", 100)
    assert (a == b).all()
    c = O.rng_draws(43, "u64", 100)
    assert not (a == c).all()
    assert O.chain_seed(1, 2, 3) != O.chain_seed(1, 3, 2)


def test_rng_splitmix_known_values():
    # SplitMix64 from state 0: first output is mix64(gamma) — published constant.
    assert int(O.rng_draws(0, "u64", 1)[0]) == 0xE220A8397B1DCDAF
    assert O.mix64(0) == 0


def test_rng_gaussian_moments_and_ranges():
    g = O.rng_draws(7, "gaussian", 200000)
    assert abs(g.mean()) < 0.01 and abs(g.var() - 1.0) < 0.02
    u = O.rng_draws(9, "double", 10000)
    assert (u >= 0).all() and (u < 1).all()
    v = O.rng_draws(9, "double_open", 10000)
    assert (v > 0).all() and (v <= 1).all()


# ------------------------------------------------------------------ validation (test_core.cpp:39-84)
def test_validate_messages():
    assert O.validate(O.cfg(4, 1024, 64, 128)) == ""
    msg = O.validate(O.cfg(4, 1000, 64, 128))
    assert "not divisible by S" in msg
    msg = O.validate(O.cfg(3, 1024, 64, 128, c_q=24, c_h=2))
    assert "c_q" in msg and "c_h" in msg and msg.count(";") == 1
    assert O.validate(O.cfg(4, 1024, 64, 128, P=0.0)) != ""
    assert O.validate(O.cfg(4, 1024, 64, 128, P=1.5)) != ""
    assert O.validate(O.cfg(4, 1024, 64, 128, P=1.0)) == ""


# ------------------------------------------------------------------ compression
def test_mean_pool_known_window():  # test_compression.cpp:23-30
    out = O.pool_sequence(np.array([[1, 2], [3, 4]], np.float32), 2)
    assert out.tolist() == [[2.0, 3.0]]


def test_max_pool_known_window():  # :32-41
    x = np.array([[1, -2], [3, -4], [-5, 6], [0.5, 0.25]], np.float32)
    assert O.pool_sequence(x, 2, O.POOL_MAX).tolist() == [[3.0, -2.0], [0.5, 6.0]]


def test_c1_is_bitwise_identity():  # :43-49
    x = random_matrix(64, 16, 11)
    for s in (O.POOL_MEAN, O.POOL_MAX, O.POOL_STOCHASTIC):
        assert (O.pool_sequence(x, 1, s, 99).view(np.uint32) == x.view(np.uint32)).all()


def test_mean_max_vs_naive():  # :51-61
    x = random_matrix(96, 8, 21)
    for c in (2, 4, 8, 32):
        naive = (x.astype(np.float64).reshape(-1, c, 8).sum(1) / c).astype(np.float32)
        assert np.abs(O.pool_sequence(x, c) - naive).max() <= 1e-6
        assert (O.pool_sequence(x, c, O.POOL_MAX) == x.reshape(-1, c, 8).max(1)).all()


def test_stochastic_pool_member_and_deterministic():  # :63-79
    x = random_matrix(64, 4, 31)
    a = O.pool_sequence(x, 8, O.POOL_STOCHASTIC, 1234)
    b = O.pool_sequence(x, 8, O.POOL_STOCHASTIC, 1234)
    assert (a == b).all()
    for w in range(a.shape[0]):
        assert any((a[w] == x[w * 8 + r]).all() for r in range(8))
    assert not (a == O.pool_sequence(x, 8, O.POOL_STOCHASTIC, 1235)).all()


def test_stochastic_pool_favors_high_norm():  # :81-90
    x = random_matrix(400, 4, 41) * np.float32(0.001)
    for w in range(100):
        x[w * 4 + (w % 4)] *= np.float32(100000.0)
    out = O.pool_sequence(x, 4, O.POOL_STOCHASTIC, 7)
    hits = sum((out[w] == x[w * 4 + (w % 4)]).all() for w in range(100))
    assert hits >= 99
    z = O.pool_sequence(np.zeros((8, 3), np.float32), 4, O.POOL_STOCHASTIC, 5)
    assert (z == 0).all()


def test_pool_rejects_bad_c():  # :98-102
    x = random_matrix(10, 2, 51)
    with pytest.raises(O.OracleError):
        O.pool_sequence(x, 3)


def test_head_grouping_means_member_heads():  # :104-117
    H, L, d = 4, 2, 2
    Q = np.stack([np.full((L, d), v, np.float32) for v in (1.0, 3.0, -2.0, 4.0)])
    c = O.cfg(H, L, d, 2, c_q=1, c_k=1, c_h=2)
    Qc, Kc = O.compress(c, Q, Q)
    assert Qc.shape == (2, 2, 2)
    assert (Qc[0] == 2.0).all() and (Qc[1] == 1.0).all()


def test_mean_pool_linear_and_window_independent():  # :119-142
    x, y = random_matrix(64, 8, 61), random_matrix(64, 8, 62)
    lhs = O.pool_sequence(np.float32(2.0) * x + y, 8)
    rhs = np.float32(2.0) * O.pool_sequence(x, 8) + O.pool_sequence(y, 8)
    assert np.abs(lhs - rhs).max() <= 1e-5
    top, bottom = random_matrix(32, 8, 71), random_matrix(32, 8, 72)
    whole = O.pool_sequence(np.concatenate([top, bottom]), 4)
    assert np.abs(whole - np.concatenate([O.pool_sequence(top, 4), O.pool_sequence(bottom, 4)])).max() <= 1e-6


def test_compress_shapes_and_identity():  # :144-176
    H, L, d = 4, 256, 16
    Q = np.stack([random_matrix(L, d, 100 + h) for h in range(H)])
    K = np.stack([random_matrix(L, d, 200 + h) for h in range(H)])
    Qc, Kc = O.compress(O.cfg(H, L, d, 64, c_q=8, c_k=4, c_h=2), Q, K)
    assert Qc.shape == (2, 32, 16) and Kc.shape == (2, 64, 16)
    Qi, Ki = O.compress(O.cfg(H, L, d, 64, c_q=1, c_k=1, c_h=1), Q, K)
    assert (Qi.view(np.uint32) == Q.view(np.uint32)).all()
    assert (Ki.view(np.uint32) == K.view(np.uint32)).all()


# ------------------------------------------------------------------ proxy (test_proxy.cpp)
def scores_of(Q, K, S, c_q, c_k, mode=O.POST_SOFTMAX, c_h=1, with_A=False):
    H, L, d = Q.shape
    c = O.cfg(H, L, d, S, c_q=c_q, c_k=c_k, c_h=c_h, causal_mode=mode)
    Qc, Kc = O.compress(c, Q, K)
    return O.proxy_scores(c, Qc, Kc, with_A=with_A)


def test_singleton_softmax():  # :54-61
    Q, K, _ = random_inputs(1, 1, 4, 1)
    s, A = scores_of(Q, K, 1, 1, 1, with_A=True)
    assert abs(A[0, 0, 0] - 1.0) < 1e-12


def test_rows_sum_to_one():  # :63-73
    Q, K, _ = random_inputs(2, 256, 16, 3)
    for mode in (O.POST_SOFTMAX, O.PRE_SOFTMAX):
        _, A = scores_of(Q, K, 64, 8, 4, mode, with_A=True)
        assert np.abs(A.sum(-1) - 1.0).max() < 1e-5


@pytest.mark.parametrize("c_q,c_k,L,S", [(2, 2, 8, 4), (4, 2, 16, 8)])
def test_pre_softmax_live_pattern(c_q, c_k, L, S):  # :75-104
    Q, K, _ = random_inputs(1, L, 4, 5 if c_q == 2 else 6)
    _, A = scores_of(Q, K, S, c_q, c_k, O.PRE_SOFTMAX, with_A=True)
    for t in range(L // c_q):
        for s in range(L // c_k):
            allowed = c_q * t + c_q - 1 >= c_k * s
            assert (A[0, t, s] > 0.0) == allowed


def test_region_sum_oracle():  # :106-123
    Q, K, _ = random_inputs(2, 256, 16, 7)
    s, A = scores_of(Q, K, 64, 8, 4, with_A=True)
    N = 4
    for h in range(2):
        ref = np.zeros((N, N))
        for t in range(A.shape[1]):
            for u in range(A.shape[2]):
                ref[t * 8 // 64, u * 4 // 64] += A[h, t, u]
        for i in range(N):
            for j in range(N):
                if j > i:
                    assert s[h, i, j] == O.K_MASKED_SCORE
                else:
                    assert s[h, i, j] == pytest.approx(ref[i, j], rel=1e-12)


def test_single_block_mass_16():  # :125-133
    Q, K, _ = random_inputs(1, 64, 8, 9)
    s = scores_of(Q, K, 64, 4, 4)
    assert s[0, 0, 0] == pytest.approx(16.0, rel=1e-9)


def test_c_equals_S_collapse():  # :135-144
    Q, K, _ = random_inputs(1, 256, 8, 11)
    s, A = scores_of(Q, K, 64, 64, 64, with_A=True)
    for i in range(4):
        for j in range(i + 1):
            assert s[0, i, j] == A[0, i, j]


def test_identity_pre_softmax_equals_exact_mass():  # :166-177
    Q, K, _ = random_inputs(2, 256, 16, 17)
    s = scores_of(Q, K, 64, 1, 1, O.PRE_SOFTMAX)
    mass = O.exact_block_mass(Q, K, 64)
    for h in range(2):
        for i in range(4):
            for j in range(i + 1):
                assert s[h, i, j] == pytest.approx(mass[h, i, j], rel=1e-9)


def test_q_scaling_rank_invariance():  # :179-198
    Q, K, _ = random_inputs(1, 256, 16, 19)
    a = scores_of(Q, K, 64, 64, 64)
    b = scores_of(Q * np.float32(2.0), K, 64, 64, 64)
    for i in range(1, 4):
        oa = sorted(range(i + 1), key=lambda j: (-a[0, i, j], j))
        ob = sorted(range(i + 1), key=lambda j: (-b[0, i, j], j))
        assert oa == ob


def test_post_softmax_deviates_from_exact_mass():  # :200-215
    Q, K, _ = random_inputs(1, 128, 8, 23)
    s = scores_of(Q, K, 32, 1, 1)
    mass = O.exact_block_mass(Q, K, 32)
    dev = max(abs(s[0, i, j] - mass[0, i, j]) for i in range(4) for j in range(i + 1))
    assert dev > 1e-3


# ------------------------------------------------------------------ selection (test_selection.cpp)
def test_top_p_smallest_prefix():  # :33-38
    idx, cov = O.top_p_row([0.5, 0.3, 0.2], 0.7)
    assert set(idx) == {0, 1} and cov == pytest.approx(0.8, rel=1e-12)


def test_top_p_ties_ascending():  # :40-44
    assert O.top_p_row([0.4, 0.4, 0.2], 0.5)[0] == [0, 1]


def test_top_p_inclusive():  # :46-50
    assert O.top_p_row([0.6, 0.4], 0.6)[0] == [0]


def test_top_p_p1_all():  # :52-57
    idx, cov = O.top_p_row([0.1, 0.0, 0.9, 0.0], 1.0)
    assert set(idx) == {0, 1, 2, 3} and cov == 1.0


def test_top_p_all_zero_diagonal():  # :59-63
    assert O.top_p_row([0.0, 0.0, 0.0], 0.9)[0] == [2]


def test_top_p_nested_and_covering():  # :65-84
    for rep in range(20):
        scores = O.rng_draws(77 + rep, "double", 12)
        prev = set()
        for P in (0.1, 0.3, 0.5, 0.7, 0.9, 0.95, 1.0):
            idx, cov = O.top_p_row(scores, P)
            cur = set(idx)
            assert prev <= cur
            prev = cur
            sel = sum(scores[j] for j in idx)
            assert sel >= P * scores.sum() - 1e-12
            assert cov == pytest.approx(sel / scores.sum(), rel=1e-9)


def test_top_p_rejects_bad_arguments():  # :86-93
    for args in (([0.5, 0.5], 0.0), ([0.5, 0.5], 1.5), ([0.5, -0.1], 0.9), ([], 0.9)):
        with pytest.raises(O.OracleError):
            O.top_p_row(*args)


def random_score_planes(H, N, seed):
    """test_selection.cpp:17-29."""
    u = O.rng_draws(seed, "double", H * N * N).reshape(H, N, N)
    tri = np.tril(np.ones((N, N), bool))
    return np.where(tri[None], u, O.K_MASKED_SCORE)


def test_build_mask_causal_nonempty_covering():  # :95-108
    s = random_score_planes(2, 8, 5)
    m, cov = O.build_block_mask(s, 2, 1, 0.8)
    for h in range(2):
        for i in range(8):
            assert m[h, i, : i + 1].any() and not m[h, i, i + 1:].any()
            assert cov[h, i] >= 0.8 - 1e-12


def test_build_mask_broadcast_c_h():  # :110-120
    s = random_score_planes(1, 6, 7)
    m, cov = O.build_block_mask(s, 4, 4, 0.9)
    for h in range(1, 4):
        assert (m[h] == m[0]).all() and (cov[h] == cov[0]).all()


def test_build_mask_monotone_and_p1_full():  # :129-140
    s = random_score_planes(3, 12, 11)
    prev = 0
    for P in (0.5, 0.7, 0.9, 0.95, 1.0):
        m, _ = O.build_block_mask(s, 3, 1, P)
        assert m.sum() >= prev
        prev = m.sum()
    assert O.build_block_mask(s, 3, 1, 1.0)[0].sum() == 3 * 12 * 13 // 2


def test_top_k_first_k_of_order():
    idx, cov = O.top_k_row([0.1, 0.4, 0.4, 0.05], 2)
    assert idx == [1, 2] and cov == pytest.approx(0.8 / 0.95)
    assert O.top_k_row([0.3, 0.2], 5)[0] == [0, 1]


# ------------------------------------------------------------------ attention (test_attention.cpp)
def naive_masked_attention(Q, K, V, allowed):
    """oracles.hpp:54-77 (one head)."""
    L, d = Q.shape
    out = np.zeros((L, d), np.float32)
    for t in range(L):
        keys = np.nonzero(allowed[t])[0]
        lg = (Q[t].astype(np.float64) @ K[keys].astype(np.float64).T) / math.sqrt(d)
        p = np.exp(lg - lg.max())
        p /= p.sum()
        out[t] = (p @ V[keys].astype(np.float64)).astype(np.float32)
    return out


def full_mask(H, N):
    return np.broadcast_to(np.tril(np.ones((N, N), bool)), (H, N, N)).copy()


def test_dense_one_token_and_first_row():  # :59-70
    Q, K, V = random_inputs(2, 1, 8, 1)
    Od, _ = O.dense_attention(Q, K, V)
    assert np.abs(Od - V).max() <= 1e-6
    Q, K, V = random_inputs(1, 64, 16, 3)
    Od, _ = O.dense_attention(Q, K, V)
    assert np.abs(Od[0, 0] - V[0, 0]).max() <= 1e-6


def test_dense_equal_keys_prefix_mean():  # :72-81
    Q, K, V = random_inputs(1, 32, 8, 5)
    K[:] = 1.0
    Od, _ = O.dense_attention(Q, K, V)
    for t in range(32):
        assert np.abs(Od[0, t] - V[0, : t + 1].mean(0)).max() <= 1e-5


def test_dense_vs_naive_and_lse():  # :95-125
    Q, K, V = random_inputs(2, 96, 12, 9)
    Od, _ = O.dense_attention(Q, K, V)
    causal = np.tril(np.ones((96, 96), bool))
    for h in range(2):
        assert np.abs(Od[h] - naive_masked_attention(Q[h], K[h], V[h], causal)).max() <= 1e-5
    Q, K, V = random_inputs(1, 40, 8, 13)
    _, lse = O.dense_attention(Q, K, V)
    for t in range(40):
        lg = Q[0, t].astype(np.float64) @ K[0, : t + 1].astype(np.float64).T / math.sqrt(8)
        assert lse[0, t] == pytest.approx(math.log(np.exp(lg).sum()), rel=1e-6)


def test_exact_block_mass_rows():  # :127-144
    Q, K, _ = random_inputs(2, 128, 8, 15)
    mass = O.exact_block_mass(Q, K, 32)
    for h in range(2):
        for i in range(4):
            assert mass[h, i, : i + 1].sum() == pytest.approx(32.0, rel=1e-8)
            assert (mass[h, i, i + 1:] == O.K_MASKED_SCORE).all()


def test_sparse_full_mask_equals_dense():  # :146-154
    Q, K, V = random_inputs(2, 256, 16, 17)
    Od, lsed = O.dense_attention(Q, K, V)
    Os, lses = O.block_sparse_attention(Q, K, V, full_mask(2, 4), 64)
    assert np.abs(Os - Od).max() <= 1e-5
    assert np.allclose(lses, lsed, rtol=1e-6)


def test_sparse_random_mask_vs_materialized():  # :156-183
    Q, K, V = random_inputs(2, 128, 8, 19)
    N = 4
    u = O.rng_draws(99, "double", 2 * N * N).reshape(2, N, N)
    m = np.zeros((2, N, N), bool)
    for h in range(2):
        for i in range(N):
            m[h, i, i] = True
            for j in range(i):
                m[h, i, j] = u[h, i, j] < 0.5
    Os, _ = O.block_sparse_attention(Q, K, V, m, 32)
    for h in range(2):
        allowed = np.zeros((128, 128), bool)
        for t in range(128):
            for k in range(t + 1):
                allowed[t, k] = m[h, t // 32, k // 32]
        assert np.abs(Os[h] - naive_masked_attention(Q[h], K[h], V[h], allowed)).max() <= 1e-5


def test_sparse_rejects_malformed_masks():  # :205-221
    Q, K, V = random_inputs(1, 64, 8, 23)
    m = full_mask(1, 2)
    m[0, 1, :] = False
    with pytest.raises(O.OracleError, match="no selected key block"):
        O.block_sparse_attention(Q, K, V, m, 32)
    m = full_mask(1, 2)
    m[0, 0, 1] = True
    with pytest.raises(O.OracleError, match="non-causal"):
        O.block_sparse_attention(Q, K, V, m, 32)


def test_sparse_extreme_logits_finite():  # :223-230
    Q, K, V = random_inputs(1, 64, 8, 25)
    Q *= np.float32(30.0)
    Od, _ = O.dense_attention(Q, K, V)
    Os, lse = O.block_sparse_attention(Q, K, V, full_mask(1, 2), 32)
    assert np.abs(Os - Od).max() <= 1e-5 and np.isfinite(lse).all()


# ------------------------------------------------------------------ pipeline (test_pipeline.cpp)
def test_pipeline_p1_equals_dense():  # :9-21
    Q, K, V, _ = O.gen_workload(O.WL_GAUSSIAN, 1024, 2, 64, 128, 5)
    c = O.cfg(2, 1024, 64, 128, c_q=8, c_k=8, P=1.0)
    Os, _, m, _ = O.unisparse_attn(c, Q, K, V)
    Od, _ = O.dense_attention(Q, K, V)
    assert O.output_fidelity(Os, Od)["max_abs"] <= 1e-5
    assert m.sum() == 2 * 8 * 9 // 2 and (O.sparsity_ratio(m) == 0).all()


def test_identity_pre_softmax_selects_oracle_blocks():  # :23-35
    Q, K, V, _ = O.gen_workload(O.WL_PLANTED, 512, 2, 32, 128, 7)
    c = O.cfg(2, 512, 32, 128, c_q=1, c_k=1, P=0.95, causal_mode=O.PRE_SOFTMAX)
    Qc, Kc = O.compress(c, Q, K)
    s = O.proxy_scores(c, Qc, Kc)
    m, _ = O.build_block_mask(s, 2, 1, 0.95)
    mo, _ = O.build_block_mask(O.exact_block_mass(Q, K, 128), 2, 1, 0.95)
    assert (m == mo).all()


def test_planted_fidelity():  # :37-48
    Q, K, V, _ = O.gen_workload(O.WL_PLANTED, 1024, 2, 64, 128, 9)
    c = O.cfg(2, 1024, 64, 128, c_q=8, c_k=8, P=0.95)
    Os, _, m, _ = O.unisparse_attn(c, Q, K, V)
    Od, _ = O.dense_attention(Q, K, V)
    assert O.output_fidelity(Os, Od)["cosine"] >= 0.99
    assert O.sparsity_ratio(m).mean() > 0


def test_report_consistency_c_h2():  # :50-77
    Q, K, V, _ = O.gen_workload(O.WL_PLANTED, 1024, 4, 32, 128, 11)
    c = O.cfg(4, 1024, 32, 128, c_q=4, c_k=8, c_h=2, P=0.9)
    Qc, Kc = O.compress(c, Q, K)
    m, cov = O.build_block_mask(O.proxy_scores(c, Qc, Kc), 4, 2, 0.9)
    assert (cov >= 0.9 - 1e-12).all()
    assert (m[0] == m[1]).all() and (m[2] == m[3]).all()


# ------------------------------------------------------------------ metrics (test_metrics.cpp:224-284)
def test_flops_pinned():
    f = O.selection_flops(4096, 4, 64, 128, 8, 8, 1)
    assert f["compression"] == 2097152 and f["compressed_qk"] == 134217728
    assert f["softmax_aggregation"] == 4194304 and f["top_p"] == 20480
    assert f["dense_attention"] == 17179869184
    f = O.selection_flops(4096, 4, 64, 128, 8, 8, 2)
    assert f["compressed_qk"] == 67108864 and f["softmax_aggregation"] == 2097152
    assert f["top_p"] == 10240 and f["compression"] == 2097152 + 524288
    a = O.selection_flops(4096, 4, 64, 128, 8, 8, 1, O.PROXY_ANTIDIAGONAL, 8)
    assert a["compressed_qk"] == 1073741824 and a["softmax_aggregation"] == 16777216
    p = O.selection_flops(4096, 4, 64, 128, 8, 8, 1, O.PROXY_LAST_BLOCK)
    assert p["compressed_qk"] == 268435456 and p["softmax_aggregation"] == 4194304
    with pytest.raises(O.OracleError):
        O.selection_flops(4096, 4, 64, 128, 8, 8, 1, O.PROXY_ANTIDIAGONAL, 3)


# ------------------------------------------------------------------ workloads (test_workloads.cpp)
def test_workload_deterministic_and_planted_lists():
    a = O.gen_workload(O.WL_PLANTED, 512, 2, 16, 64, 3, m=3)
    b = O.gen_workload(O.WL_PLANTED, 512, 2, 16, 64, 3, m=3)
    for x, y in zip(a, b):
        assert (x == y).all()
    planted = a[3]
    for h in range(2):
        for i in range(8):
            s = [j for j in planted[h, i] if j >= 0]
            assert len(s) == min(3, i + 1) and s == sorted(set(s)) and all(0 <= j <= i for j in s)


def test_high_gain_planted_blocks_dominate_exact_mass():  # test_workloads.cpp:92-104
    Q, K, V, planted = O.gen_workload(O.WL_PLANTED, 1024, 2, 64, 128, 5, gain=8.0, m=2)
    mass = O.exact_block_mass(Q, K, 128)
    for h in range(2):
        for i in range(2, 8):
            row = mass[h, i, : i + 1]
            top = set(np.argsort(-row, kind="stable")[:2].tolist())
            assert top == set(planted[h, i].tolist())


def test_locality_shift_disjoint():  # :106-120
    _, _, _, planted = O.gen_workload(O.WL_LOCALITY_SHIFT, 1024, 2, 8, 64, 13, m=2)
    N = 16
    for h in range(2):
        last = planted[h, N - 1].tolist()
        assert all(j >= N // 2 for j in last)
        for i in range(N - 1):
            assert not (set(planted[h, i].tolist()) & set(last))


def test_gqa_generator_reduces_to_reference():
    full = O.gen_workload(O.WL_PLANTED, 256, 2, 16, 64, 21, H_kv=2)
    ref = O.gen_workload(O.WL_PLANTED, 256, 2, 16, 64, 21)
    for x, y in zip(full, ref):
        assert (x == y).all()


# ------------------------------------------------------------------ competitor proxies (test_baselines.cpp)
def _rand(H, L, d, seed):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((H, L, d)).astype(np.float32), rng.standard_normal((H, L, d)).astype(np.float32))


def _literal_antidiagonal(Qh, Kh, S, stride):  # oracles.hpp:115-140, literal enumeration
    L, d = Qh.shape
    N = L // S
    score = np.zeros((N, N))
    for i in range(N):
        for q in range(S):
            t = i * S + q
            keys = [j * S + (S - 1 - q + r) % S for j in range(i + 1) for r in range(0, S, stride)]
            keys = [k for k in keys if k <= t]
            if not keys:
                continue
            lg = np.array([np.dot(Qh[t].astype(np.float64), Kh[k].astype(np.float64)) for k in keys]) / np.sqrt(d)
            p = np.exp(lg - lg.max())
            p /= p.sum()
            for k, pk in zip(keys, p):
                score[i, k // S] += pk
    return score


def test_antidiagonal_stride1_is_exact_mass():  # test_baselines.cpp:40-48
    Q, K = _rand(2, 128, 8, 3)
    probe = O.antidiagonal_block_scores(Q, K, 32, 1)
    mass = O.exact_block_mass(Q, K, 32)
    tri = np.tril(np.ones((4, 4), bool))
    assert np.allclose(probe[:, tri], mass[:, tri], rtol=1e-9, atol=0)


@pytest.mark.parametrize("stride", [2, 4, 8, 16, 32])
def test_antidiagonal_matches_literal_enumeration(stride):  # test_baselines.cpp:50-61
    Q, K = _rand(2, 128, 8, 5)
    probe = O.antidiagonal_block_scores(Q, K, 32, stride)
    tri = np.tril(np.ones((4, 4), bool))
    for h in range(2):
        ref = _literal_antidiagonal(Q[h], K[h], 32, stride)
        assert np.allclose(probe[h][tri], ref[tri], rtol=1e-9, atol=1e-15)


def test_antidiagonal_masks_and_row_mass():  # test_baselines.cpp:63-83
    Q, K = _rand(1, 128, 8, 9)
    S, stride = 32, 8
    probe = O.antidiagonal_block_scores(Q, K, S, stride)
    for i in range(4):
        for j in range(i + 1, 4):
            assert probe[0, i, j] == O.K_MASKED_SCORE
        rows = sum(1 for q in range(S) if (S - 1 - q) % stride <= i * S + q)
        assert probe[0, i, : i + 1].sum() == pytest.approx(rows, rel=1e-9)


def test_antidiagonal_S1_equals_identity_pre_softmax():  # test_baselines.cpp:85-98
    Q, K = _rand(1, 32, 8, 11)
    probe = O.antidiagonal_block_scores(Q, K, 1, 1)
    c = O.cfg(1, 32, 8, 1, c_q=1, c_k=1, causal_mode=O.PRE_SOFTMAX)
    Qc, Kc = O.compress(c, Q, K)
    s = O.proxy_scores(c, Qc, Kc)
    tri = np.tril(np.ones((32, 32), bool))
    assert np.allclose(probe[0][tri], s[0][tri], rtol=1e-9, atol=1e-15)


def test_antidiagonal_validates_stride():  # test_baselines.cpp:185-189
    Q, K = _rand(1, 64, 8, 21)
    for bad in (0, 3):
        with pytest.raises(O.OracleError, match="stride must divide S"):
            O.antidiagonal_block_scores(Q, K, 32, bad)


def test_last_block_probe_replicates_columns():  # test_baselines.cpp:100-114
    Q, K = _rand(2, 128, 8, 13)
    probe = O.last_block_probe_scores(Q, K, 32)
    for h in range(2):
        for i in range(4):
            for j in range(4):
                assert probe[h, i, j] == (O.K_MASKED_SCORE if j > i else probe[h, 3, j])


def test_last_block_probe_single_block_and_uniform_keys():  # test_baselines.cpp:116-136
    Q, K = _rand(1, 32, 8, 15)
    probe = O.last_block_probe_scores(Q, K, 32)
    assert probe[0, 0, 0] == pytest.approx(32.0, rel=1e-9)
    assert probe[0, 0, 0] == pytest.approx(O.exact_block_mass(Q, K, 32)[0, 0, 0], rel=1e-9)
    Q, K = _rand(1, 128, 8, 17)
    K[:] = 0.0
    probe = O.last_block_probe_scores(Q, K, 32)
    expect = sum(32.0 / (97.0 + r) for r in range(32))
    for j in range(3):
        assert probe[0, 3, j] == pytest.approx(expect, rel=1e-9)


# ------------------------------------------------------------------ metrics (test_metrics.cpp)
def test_spearman_kats():  # test_metrics.cpp:28-74
    assert O.spearman_rho([1, 2, 3, 4], [1, 3, 2, 4]) == pytest.approx(0.8, rel=1e-12)
    assert O.spearman_rho([1, 1, 2], [1, 2, 3]) == pytest.approx(np.sqrt(3.0) / 2.0, rel=1e-12)
    a = np.array([0.3, 1.7, -2.0, 5.5, 0.01])
    assert O.spearman_rho(a, a) == pytest.approx(1.0, rel=1e-12)
    assert O.spearman_rho(a, -a) == pytest.approx(-1.0, rel=1e-12)
    assert O.spearman_rho(a, np.exp(a)) == pytest.approx(O.spearman_rho(a, a), rel=1e-12)
    assert O.spearman_rho([2.0, 2.0, 2.0], [1.0, 2.0, 3.0]) is None
    assert O.spearman_rho([1.0, 2.0, 3.0], [2.0, 2.0, 2.0]) is None
    with pytest.raises(O.OracleError, match="at least 2"):
        O.spearman_rho([1.0], [2.0])


def _mask_rows(rows, N):
    m = np.zeros((1, N, N), bool)
    for i, js in enumerate(rows):
        m[0, i, js] = True
    return m


def test_block_recall_kats():  # test_metrics.cpp:124-152
    M = O.K_MASKED_SCORE
    ref = np.array([[[5.0, M, M], [1.0, 2.0, M], [3.0, 1.0, 2.0]]])
    m = _mask_rows([[0], [1], [0, 2]], 3)
    assert O.block_recall(m, ref, 2) == pytest.approx(5.0 / 6.0, rel=1e-12)
    assert O.block_recall(m, ref, 1) == pytest.approx(1.0, rel=1e-12)
    assert O.block_recall(m, ref, 3) == pytest.approx((1.0 + 0.5 + 2.0 / 3.0) / 3.0, rel=1e-12)
    for bad in (0, 4):
        with pytest.raises(O.OracleError, match="k out of range"):
            O.block_recall(m, ref, bad)
    ref = np.array([[[1.0, M], [2.0, 2.0]]])  # ties break toward the lower index
    assert O.block_recall(_mask_rows([[0], [0]], 2), ref, 1) == pytest.approx(1.0)
    assert O.block_recall(_mask_rows([[0], [1]], 2), ref, 1) == pytest.approx(0.5)


def test_mean_row_spearman_kats():  # test_metrics.cpp:164-222
    M = O.K_MASKED_SCORE
    rng = np.random.default_rng(3)
    p = np.full((1, 6, 6), M)
    for i in range(6):
        p[0, i, :i + 1] = rng.random(i + 1)
    mean, d, u = O.mean_row_spearman(p, p, 1)
    assert mean == pytest.approx(1.0, rel=1e-12) and d == 5 and u == 0
    p = np.full((1, 4, 4), M)
    for i in range(4):
        p[0, i, :i + 1] = rng.random(i + 1)
    mean, d, _ = O.mean_row_spearman(p, np.concatenate([p, p]), 2)
    assert mean == pytest.approx(1.0, rel=1e-12) and d == 6
    with pytest.raises(O.OracleError, match="head counts disagree"):
        O.mean_row_spearman(p, np.concatenate([p, p]), 1)
    p = np.full((1, 3, 3), M)
    p[0, 0, 0] = 1.0
    p[0, 1, :2] = [0.5, 0.5]
    p[0, 2, :3] = [0.3, 0.2, 0.1]
    q = p.copy()
    q[0, 1, :2] = [0.9, 0.1]
    mean, d, u = O.mean_row_spearman(p, q, 1)
    assert (d, u) == (1, 1) and mean == pytest.approx(1.0, rel=1e-12)


def test_planted_recall_kats():  # test_metrics.cpp:154-161
    m = _mask_rows([[0], [0, 1], [0, 2]], 3)
    planted = np.array([[[-1, -1], [0, -1], [1, 2]]], np.int32)
    assert O.planted_recall(m, planted) == pytest.approx(0.75, rel=1e-12)
    with pytest.raises(O.OracleError, match="no planted rows"):
        O.planted_recall(m, np.full((1, 3, 2), -1, np.int32))
