"""Size-independent properties of the selection on EVERY row of the full BASELINE shapes
(the sampled-row oracle checks live in test_gpu_configs.py). On the GPU's own block
scores (with_scores), each row's mask must be exactly what the reference rule
(selection.cpp:11-48) selects, checked in fp64 on the device for all rows at once:

* Top-P: the selected set is a prefix of the order (descending score, ties by ascending
  index), its mass reaches P * total, and dropping its last (smallest) member falls short
  (inclusive cum >= P * total, the first time);
* top-k: the selected set is the first min(k, i + 1) entries of the same order;
* causal (no bit above the diagonal), counts = popcount of the row's bits, coverage =
  selected mass / total (metrics the reference reports).

Sums here run in a different order than the reference's sequential walk; decisions
within 1e-9 of the threshold are therefore not asserted (the GPU certifies those against
the sequential order itself, select.cu)."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = {
    # name: (H, H_kv, L, mode, k, P, gain)
    "C3_128K_g9": (32, 8, 131072, "top_p", None, 0.95, 9.0),
    "C3_128K_g8": (32, 8, 131072, "top_p", None, 0.95, 8.0),
    "C2_32K_topk64": (32, 8, 32768, "top_k", 64, 0.95, 8.0),
    "C4_128K": (28, 4, 131072, "top_p", None, 0.95, 9.0),
    "C5_256K": (40, 40, 262144, "top_p", None, 0.95, 9.5),
}


@pytest.mark.parametrize("name", list(CASES))
def test_every_row_follows_the_reference_rule(name):
    import paper_2512_14082_b200 as us
    from paper_2512_14082_b200 import workloads
    H, H_kv, L, mode, k, P, gain = CASES[name]
    Q, K, V = workloads.planted_blocks(L, H, H_kv, 128, 64, seed=2512, gain=gain)
    cfg = us.CompressionConfig(P=P) if mode == "top_p" else us.CompressionConfig(select_mode=us.SELECT_TOP_K, top_k=k)
    rep = us.select_blocks(Q, K, cfg, with_scores=True)
    del Q, K, V
    torch.cuda.synchronize()
    m = rep.mask
    N = L // 64
    sel = m.dense_mask()[0]                                   # [H, N, N] bool
    tri = torch.tril(torch.ones(N, N, dtype=torch.bool, device=sel.device))
    assert not (sel & ~tri).any(), "a selected block above the diagonal"
    counts = m.counts[0].to(torch.int64)
    assert torch.equal(counts, sel.sum(-1)), "counts != popcount of the row's bits"
    for h in range(H):  # one head at a time keeps the fp64 / sort working set small
        s = m.scores[0, h].double().masked_fill(~tri, -1.0)  # [N, N], below-diagonal scores >= 0
        sh = sel[h]
        assert (s[tri] >= 0).all()
        total = s.clamp_min(0).sum(-1)
        smass = torch.where(sh, s, torch.zeros_like(s)).sum(-1)
        # the order: descending score, ascending index; selected = a prefix of it
        order = torch.sort(s, dim=-1, descending=True, stable=True).indices
        sel_sorted = torch.gather(sh, 1, order)
        n_sel = sh.sum(-1)
        prefix = torch.arange(N, device=s.device)[None, :] < n_sel[:, None]
        assert torch.equal(sel_sorted, prefix), f"head {h}: the selection is not a prefix of the order"
        if mode == "top_k":
            rows = torch.arange(N, device=s.device)
            assert torch.equal(n_sel, torch.clamp(rows + 1, max=k)), f"head {h}: top-k count"
            cov = smass / total
        else:
            T = P * total
            s_sorted = torch.gather(s, 1, order)
            last = torch.gather(s_sorted, 1, (n_sel - 1).clamp_min(0)[:, None])[:, 0]  # smallest selected
            tol = 1e-9 * total
            assert (smass >= T - tol).all(), f"head {h}: selected mass below P * total"
            assert ((smass - last) < T + tol).all(), f"head {h}: the last selected block was not needed"
            cov = smass / total
        assert torch.allclose(m.coverage[0, h], cov, rtol=0, atol=1e-9), f"head {h}: coverage"


def test_c3_compress_bit_exact_full_size():
    """compress (compression.hpp:13-76) on the full C3 layer: fp64 window sums of bf16
    values are exact (order-independent), so torch's fp64 mean rounded once to f32 is the
    reference's value bit for bit — for every composite token of Q and of K (K expanded
    to the 32 Q heads, the reference layout)."""
    import paper_2512_14082_b200 as us
    from paper_2512_14082_b200 import workloads
    H, H_kv, L, d, c = 32, 8, 131072, 128, 8
    Q, K, _ = workloads.planted_blocks(L, H, H_kv, d, 64, seed=2512, gain=9.0)
    Qc, Kc = us.compress(Q, K, us.CompressionConfig(c_q=c, c_k=c))
    torch.cuda.synchronize()
    for h in range(H):
        rq = Q[0, h].double().view(L // c, c, d).sum(1).div(c).float()
        assert torch.equal(Qc[0, h].view(torch.int32), rq.view(torch.int32)), f"Q head {h}"
        rk = K[0, h // (H // H_kv)].double().view(L // c, c, d).sum(1).div(c).float()
        assert torch.equal(Kc[0, h].view(torch.int32), rk.view(torch.int32)), f"K head {h}"


@pytest.mark.parametrize("gain", [9.0, 8.0])
def test_c3_every_row_mask_vs_fp64_reference(gain):
    """The whole path at C3 for ALL 2048 query blocks of one Q head per KV group: block
    scores recomputed in fp64 on the device from the (bit-exact) composite tokens —
    logits (Qc Kc^T) / sqrt(d) over every composite key, post-softmax row normalisation,
    8 x 8 region sums (proxy.cpp:10-72) — then the reference Top-P rule (selection.cpp:
    11-48: stable descending order, inclusive cum >= P * total); the GPU's masks must
    match, any flip only at a genuine near-tie (relative margin < 1e-6)."""
    import paper_2512_14082_b200 as us
    from paper_2512_14082_b200 import workloads
    H, H_kv, L, d, c, P = 32, 8, 131072, 128, 8, 0.95
    N, Lc, G = L // 64, L // c, H // H_kv
    Q, K, V = workloads.planted_blocks(L, H, H_kv, d, 64, seed=2512, gain=gain)
    cfg = us.CompressionConfig(P=P)
    rep = us.select_blocks(Q, K, cfg)
    Qc, Kc = us.compress(Q, K, cfg)
    del Q, K, V
    gmask = rep.mask.dense_mask()[0]
    flips, worst_margin = 0, 0.0
    for g in range(H_kv):
        h = g * G + (g % G)
        kc = Kc[0, h].double()
        ref_scores = torch.empty((N, N), dtype=torch.float64, device=kc.device)
        for r0 in range(0, Lc, 2048):  # composite query rows in chunks
            x = (Qc[0, h, r0:r0 + 2048].double() @ kc.T) / (d ** 0.5)
            p = torch.softmax(x, dim=-1)                       # post-softmax: every composite key
            ref_scores[r0 // 8:(r0 + 2048) // 8] = p.view(256, 8, N, 8).sum((1, 3))
        tri = torch.tril(torch.ones(N, N, dtype=torch.bool, device=kc.device))
        s = ref_scores.masked_fill(~tri, -1.0)
        srt, order = torch.sort(s, dim=-1, descending=True, stable=True)
        cum = torch.cumsum(srt.clamp_min(0), -1)
        total = cum[:, -1]
        n_sel = (cum < P * total[:, None]).sum(-1) + 1           # inclusive threshold
        ref = torch.zeros_like(gmask[h])
        ref.scatter_(1, order, torch.arange(N, device=kc.device)[None, :] < n_sel[:, None])
        bad = torch.nonzero(ref != gmask[h])
        flips += len(bad)
        for i, _j in bad.tolist():  # a flip must sit at a near-tie of the fp64 rule
            k = int(n_sel[i]) - 1
            margin = min(abs(float(cum[i, k]) - P * float(total[i])),
                         abs(float(cum[i, k - 1]) - P * float(total[i])) if k > 0 else 1.0) / float(total[i])
            worst_margin = max(worst_margin, margin)
            assert margin < 1e-6, (h, i, _j, margin)
    print(f"gain {gain}: {H_kv * N} rows, {int(gmask[::G].sum())} selected blocks checked, {flips} flips, "
          f"worst flip margin {worst_margin:.2e}")
    assert flips <= 8, flips
