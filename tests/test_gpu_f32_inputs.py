"""f32 inputs (the reference's own HeadStack<float> storage) through the
drop-in: us_params.dtype = US_DTYPE_F32. compress / select pool the UN-ROUNDED f32
values (fp64 window sums, compression.hpp:26-28), so the compressed tensors and the
selected masks must equal the oracle's on the same f32 inputs bit for bit; attention
then runs on bf16 copies (round to nearest even) and is compared with the fp64 oracle
on the f32 inputs within the bf16 tolerance. Also: asynchronous data-error reporting
of block_sparse_attention through the workspace error word (us_check_device_errors)."""
import ctypes

import numpy as np
import pytest

import oracle_py as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def us():
    import paper_2512_14082_b200 as m
    return m


def _f32(x, B=1):
    t = torch.from_numpy(np.ascontiguousarray(x, np.float32))
    return (t.unsqueeze(0) if t.dim() == 3 else t).cuda().contiguous()


@pytest.mark.parametrize("L,H,H_kv,P,mode", [(4096, 32, 8, 0.95, 0), (4096, 32, 8, 0.9, 0), (2048, 8, 2, 0.95, 1)])
def test_f32_inputs_masks_bit_exact_c1(L, H, H_kv, P, mode):
    d, S = 128, 64
    Q, K, V, _ = O.gen_workload(O.WL_PLANTED, L, H, d, S, 2512, H_kv=H_kv, gain=8.0)  # f32, not rounded
    c = O.cfg(H, L, d, S, H_kv=H_kv, P=P, causal_mode=mode)
    Or, lser, ref_mask, _ = O.unisparse_attn(c, Q, K, V)
    cfg = us().CompressionConfig(P=P, causal_mode=mode)
    q, k, v = _f32(Q), _f32(K), _f32(V)
    # compress: bit-exact f32 composite tokens (reference layout: K expanded to H heads)
    Qc, Kc = us().compress(q, k, cfg)
    Qr, Kr = O.compress(c, Q, K)
    assert np.array_equal(Qc[0].cpu().numpy().view(np.uint32), Qr.view(np.uint32))
    assert np.array_equal(Kc[0].cpu().numpy().view(np.uint32), Kr.view(np.uint32))
    res = us().unisparse_attn(q, k, v, cfg)
    torch.cuda.synchronize()
    gmask = res.report.mask.dense_mask()[0].cpu().numpy()
    flips = int((gmask != ref_mask).sum())
    assert flips == 0, f"{flips} mask bits differ from the reference rule on f32 inputs"
    Og = res.O[0].float().cpu().numpy()
    assert np.abs(Og - Or).max() <= 1e-2 * np.abs(Or).max() + 1e-4
    assert np.linalg.norm(Og - Or) / np.linalg.norm(Or) <= 1e-2
    assert np.abs(res.lse[0].cpu().numpy() - lser).max() <= 1e-2 * max(1.0, np.abs(lser).max())


def test_f32_dense_attention_matches_oracle():
    rng = np.random.default_rng(4)
    Q = rng.standard_normal((2, 1024, 128)).astype(np.float32)
    K = rng.standard_normal((1, 1024, 128)).astype(np.float32)
    V = rng.standard_normal((1, 1024, 128)).astype(np.float32)
    Og, lse = us().dense_attention(_f32(Q), _f32(K), _f32(V))
    Or, lser = O.dense_attention(Q, K, V)
    assert Og.dtype == torch.bfloat16
    assert np.abs(Og[0].float().cpu().numpy() - Or).max() <= 2e-2
    # (the kernel sees bf16 copies: logits move by ~2^-8 relative, and so does lse)
    assert np.abs(lse[0].cpu().numpy() - lser).max() <= 1e-2


@pytest.mark.parametrize("impl", [0, 6])
def test_async_mask_errors_visible_on_check(impl):
    """block_sparse_attention WITHOUT the synchronous check: a malformed mask (empty row /
    non-causal bit) is reported by us_check_device_errors through the workspace's sticky
    error word, with the reference's message (attention.cpp:106-108, 127-129) — by the
    kernel the density gate picks (impl 0: attention.cu for this dense mask) and by
    attention64.cu (impl 6, forced)."""
    api = us().api
    assert api.lib().us_set_attention_impl(impl) == 0
    try:
        _async_mask_errors(api)
    finally:
        api.lib().us_set_attention_impl(0)


def _async_mask_errors(api):
    rng = np.random.default_rng(5)
    Q = torch.from_numpy(rng.standard_normal((1, 2, 256, 64)).astype(np.float32)).to(torch.bfloat16).cuda()
    K = torch.from_numpy(rng.standard_normal((1, 2, 256, 64)).astype(np.float32)).to(torch.bfloat16).cuda()
    V = K.clone()
    N = 4
    for kind, msg in (("empty", "no selected key block"), ("noncausal", "non-causal")):
        m = np.tril(np.ones((1, 2, N, N), bool))
        if kind == "empty":
            m[0, 1, 2, :] = False
        else:
            m[0, 0, 1, 3] = True
        w = np.zeros((1, 2, N, 1), np.uint32)
        for j in range(N):
            w[..., 0] |= (m[..., j].astype(np.uint32) << j)
        bits = torch.from_numpy(w.view(np.int32)).cuda()
        p = api.make_params(Q, K, api.CompressionConfig(c_q=1, c_k=1, c_h=1), 64)
        ws = torch.zeros(api.lib().us_workspace_bytes(ctypes.byref(p)), dtype=torch.uint8, device="cuda")
        O_ = torch.empty_like(Q)
        rc = api.lib().us_sparse_attention(ctypes.byref(p), api._ptr(Q), api._ptr(K), api._ptr(V), api._ptr(bits), 1,
                                           api._ptr(O_), None, api._ptr(ws), ws.numel(), api._stream())
        assert rc == 0  # asynchronous: the call itself succeeds
        rc = api.lib().us_check_device_errors(ctypes.byref(p), api._ptr(ws), api._stream())
        assert rc == api.US_ERR_INVALID_MASK
        assert msg in api.lib().us_last_error().decode()
