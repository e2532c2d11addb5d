"""Block-sparse attention at the headline shape against a plain PyTorch fp32 reference,
on EVERY query block of one Q head per KV group (the oracle tests sample rows). For each
query block i the reference gathers the K / V rows of the key blocks the GPU selected,
forms Q_i K^T / sqrt(d) in fp32 with the strict-upper -inf inside the diagonal block,
softmax, P V and lse = logsumexp — attention.cpp:89-137 on the same bf16 inputs."""
import math

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("gain", [9.0, 8.0])
def test_c3_every_query_block_matches_fp32(gain):
    import paper_2512_14082_b200 as us
    from paper_2512_14082_b200 import workloads
    H, H_kv, L, d, S = 32, 8, 131072, 128, 64
    N, G = L // S, H // H_kv
    Q, K, V = workloads.planted_blocks(L, H, H_kv, d, S, seed=2512, gain=gain)
    eng = us.Engine(Q, K, V, us.CompressionConfig(P=0.95))
    eng.run()
    torch.cuda.synchronize()
    mask = eng.sel.dense_mask()[0]                       # [H, N, N]
    tri = torch.tril(torch.ones(S, S, dtype=torch.bool, device=Q.device))
    ar = torch.arange(S, device=Q.device)
    worst_rel, worst_abs, worst_lse = 0.0, 0.0, 0.0
    for g in range(H_kv):
        h = g * G + (g % G)                              # one Q head of every KV group
        k, v = K[0, g].float(), V[0, g].float()
        num = den = 0.0
        for i in range(N):
            blocks = torch.nonzero(mask[h, i]).flatten()
            keys = (blocks[:, None] * S + ar[None, :]).flatten()
            q = Q[0, h, i * S:(i + 1) * S].float()
            logits = (q @ k[keys].T) / math.sqrt(d)      # [S, n * S]
            if bool(mask[h, i, i]):                       # the diagonal block is the last (ascending)
                logits[:, -S:].masked_fill_(~tri, -float("inf"))
            ref = torch.softmax(logits, -1) @ v[keys]
            lse = torch.logsumexp(logits, -1)
            got = eng.O[0, h, i * S:(i + 1) * S].float()
            diff = (got - ref).abs().max().item()
            worst_abs = max(worst_abs, diff / (ref.abs().max().item() + 1e-4))
            num += ((got - ref) ** 2).sum().item()
            den += (ref ** 2).sum().item()
            worst_lse = max(worst_lse, (eng.lse[0, h, i * S:(i + 1) * S] - lse).abs().max().item())
        worst_rel = max(worst_rel, math.sqrt(num / den))
    assert worst_abs <= 1e-2, worst_abs          # max-abs <= 1e-2 * max|O_ref| per query block
    assert worst_rel <= 1e-2, worst_rel          # relative Frobenius per head
    assert worst_lse <= 2e-3 * 20, worst_lse     # lse (|lse| ~ 10-20 at 128K keys)
