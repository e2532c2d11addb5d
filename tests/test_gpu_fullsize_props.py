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
