"""Head dims outside {64, 128} (the reference accepts any d_k, types.hpp:66-72; its
acceptance battery runs d_k = 32, acceptance.cpp:53-60): the entry points stage copies
zero-padded to 64 / 128 in the workspace and keep the softmax scale 1/sqrt(d_k) of the
caller's d_k. Zero columns pool to exact zeros and add exact zeros to every dot
product, so compressed rows are bit-exact, masks equal the fp64 reference rule and
outputs stay within the bf16 bound of the fp64 oracle.
"""
import numpy as np
import pytest

import oracle_py as O
from gpu_util import to_dev_bf16, workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ATOL = 1e-2


def us():
    import paper_2512_14082_b200 as m
    return m


@pytest.mark.parametrize("d", [32, 48, 96])
def test_compress_bit_exact_padded_dk(d):
    L, H, H_kv = 1024, 4, 2
    Q, K, V, _ = workload(O.WL_PLANTED, L, H, H_kv, d, 40 + d)
    cfg = us().CompressionConfig(c_q=8, c_k=8, c_h=1)
    Qc, Kc = us().compress(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), cfg)
    c = O.cfg(H, L, d, 64, H_kv=H_kv)
    Qr, Kr = O.compress(c, Q, K)
    assert Qc.shape[-1] == d and Kc.shape[-1] == d
    assert np.array_equal(Qc[0].cpu().numpy(), Qr)
    assert np.array_equal(Kc[0].cpu().numpy(), Kr)


@pytest.mark.parametrize("d,H,H_kv,mode", [(32, 8, 2, O.POST_SOFTMAX), (32, 4, 4, O.PRE_SOFTMAX),
                                            (96, 4, 1, O.POST_SOFTMAX)])
def test_pipeline_padded_dk_masks_and_output(d, H, H_kv, mode):
    L, P = 2048, 0.95
    Q, K, V, _ = workload(O.WL_PLANTED, L, H, H_kv, d, 7 + d, gain=8.0)
    cfg = us().CompressionConfig(c_q=8, c_k=8, c_h=1, P=P, causal_mode=mode)
    res = us().unisparse_attn(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), to_dev_bf16(V, 1), cfg, with_scores=True)
    torch.cuda.synchronize()
    c = O.cfg(H, L, d, 64, H_kv=H_kv, causal_mode=mode, P=P)
    Qc, Kc = O.compress(c, Q, K)
    ref_scores = O.proxy_scores(c, Qc, Kc)
    ref_mask, _ = O.build_block_mask(ref_scores, H, 1, P)
    gpu_mask = res.report.mask.dense_mask()[0].cpu().numpy()
    gpu_scores = res.report.mask.scores[0].cpu().numpy()
    N = L // 64
    tri = np.tril(np.ones((N, N), bool))
    big = ref_scores[:, tri] > 1e-6
    rel = np.abs(gpu_scores - ref_scores)[:, tri] / np.maximum(ref_scores[:, tri], 1e-30)
    assert rel[big].max() < 1e-3
    assert (gpu_mask == ref_mask).all(), int((gpu_mask != ref_mask).sum())
    Or, lser = O.block_sparse_attention(Q, K, V, ref_mask, 64)
    Og = res.O[0].float().cpu().numpy()
    assert Og.shape[-1] == d
    assert np.abs(Og - Or).max() <= ATOL * max(1.0, np.abs(Or).max())
    assert np.abs(res.lse[0].cpu().numpy() - lser).max() <= 1e-3


@pytest.mark.parametrize("d,causal", [(32, True), (32, False), (80, True)])
def test_dense_attention_padded_dk(d, causal):
    rng = np.random.default_rng(d)
    H, H_kv, L = 4, 2, 512
    Q = O.bf16_round(rng.standard_normal((H, L, d)).astype(np.float32))
    K = O.bf16_round(rng.standard_normal((H_kv, L, d)).astype(np.float32))
    V = O.bf16_round(rng.standard_normal((H_kv, L, d)).astype(np.float32))
    Og, lseg = us().dense_attention(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), to_dev_bf16(V, 1), causal=causal)
    Or, lser = O.dense_attention(Q, K, V, causal=causal)
    assert np.abs(Og[0].float().cpu().numpy() - Or).max() <= ATOL
    assert np.abs(lseg[0].cpu().numpy() - lser).max() <= 1e-3
    # torch fp32 SDPA (its default scale is 1/sqrt(d) of the real d)
    q = torch.from_numpy(Q).cuda()[None]
    k = torch.from_numpy(K).cuda().repeat_interleave(H // H_kv, 0)[None]
    v = torch.from_numpy(V).cuda().repeat_interleave(H // H_kv, 0)[None]
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal)[0].cpu().numpy()
    assert np.abs(Og[0].float().cpu().numpy() - ref).max() <= ATOL


def test_sparse_attention_padded_dk_random_masks():
    rng = np.random.default_rng(5)
    H, H_kv, L, d = 4, 2, 1024, 32
    N = L // 64
    Q = O.bf16_round(rng.standard_normal((H, L, d)).astype(np.float32))
    K = O.bf16_round(rng.standard_normal((H_kv, L, d)).astype(np.float32))
    V = O.bf16_round(rng.standard_normal((H_kv, L, d)).astype(np.float32))
    mask = rng.random((H, N, N)) < 0.4
    mask &= np.tril(np.ones((N, N), bool))
    mask[:, np.arange(N), np.arange(N)] = True
    from test_gpu_kernels import _bits_from_mask
    bits = torch.from_numpy(_bits_from_mask(mask[None])).cuda()
    Og, lseg = us().block_sparse_attention(to_dev_bf16(Q, 1), to_dev_bf16(K, 1), to_dev_bf16(V, 1), bits)
    Or, lser = O.block_sparse_attention(Q, K, V, mask, 64)
    assert np.abs(Og[0].float().cpu().numpy() - Or).max() <= ATOL
    assert np.abs(lseg[0].cpu().numpy() - lser).max() <= 1e-3


def test_padded_dk_needs_workspace():
    import ctypes as C
    api = us().api
    Q = torch.zeros((1, 2, 256, 32), dtype=torch.bfloat16, device="cuda")
    K = torch.zeros((1, 2, 256, 32), dtype=torch.bfloat16, device="cuda")
    O_ = torch.empty_like(Q)
    p = api.make_params(Q, K, us().CompressionConfig(c_q=1, c_k=1, c_h=1), 64)
    st = api.lib().us_dense_attention(C.byref(p), api._ptr(Q), api._ptr(K), api._ptr(K), api._ptr(O_), None, None,
                                      0, None)
    assert st == api.US_ERR_WORKSPACE
    assert "zero-padded to 64" in api.lib().us_last_error().decode()


@pytest.mark.parametrize("d,S", [(32, 64), (32, 128), (96, 128)])
def test_padded_dk_f32_inputs_and_block_size(d, S):
    """d_k padding composed with the other staging paths: the reference's own un-rounded
    f32 storage (us_params.dtype = F32) and the battery's block size S = 128 — masks
    bit-exact vs the oracle on the f32 inputs, outputs within the bf16 bound."""
    L, H, H_kv, P = 2048, 4, 2, 0.95
    Q, K, V, _ = O.gen_workload(O.WL_PLANTED, L, H, d, S, 77 + d + S, H_kv=H_kv, gain=8.0)  # f32, not rounded
    c = O.cfg(H, L, d, S, H_kv=H_kv, P=P)
    Or, lser, ref_mask, _ = O.unisparse_attn(c, Q, K, V)
    f32 = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).unsqueeze(0).cuda().contiguous()
    cfg = us().CompressionConfig(P=P)
    res = us().unisparse_attn(f32(Q), f32(K), f32(V), cfg, S=S)
    torch.cuda.synchronize()
    gmask = res.report.mask.dense_mask()[0].cpu().numpy()
    assert (gmask == ref_mask).all(), int((gmask != ref_mask).sum())
    Og = res.O[0].float().cpu().numpy()
    assert Og.shape[-1] == d
    # attention runs on bf16 copies of the f32 inputs: compared with the fp64
    # oracle on those same bf16 values over the (bit-exact) mask. Against the f32 inputs
    # themselves the bf16 rounding alone moves O by ~1 % at d = 32 with gain-8 logits.
    Ob, lseb = O.block_sparse_attention(O.bf16_round(Q), O.bf16_round(K), O.bf16_round(V), ref_mask, S)
    assert np.abs(Og - Ob).max() <= 1e-2 * np.abs(Ob).max() + 1e-4
    assert np.linalg.norm(Og - Ob) / np.linalg.norm(Ob) <= 1e-2
    assert np.abs(res.lse[0].cpu().numpy() - lseb).max() <= 1e-3 * max(1.0, np.abs(lseb).max())
