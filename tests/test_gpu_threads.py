"""Reentrancy of the C ABI (the reference's UNISPARSE_WORKERS pool
calls unisparse_attn from several host threads): concurrent calls from host
threads on their own streams give the same results as sequential calls, and the
thread-local error text never leaks between threads."""
import threading

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def us():
    import paper_2512_14082_b200 as m
    return m


def test_concurrent_threads_match_sequential():
    from paper_2512_14082_b200 import workloads
    cfg = us().CompressionConfig(P=0.9)
    ins = [workloads.planted_blocks(2048, 8, 2, 128, 64, seed=40 + t, gain=8.0) for t in range(4)]
    refs = []
    for Q, K, V in ins:
        r = us().unisparse_attn(Q, K, V, cfg)
        torch.cuda.synchronize()
        refs.append((r.O.clone(), r.report.mask.mask_bits.clone()))
    errors, results = [], [None] * len(ins)

    def worker(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(5):
                    r = us().unisparse_attn(*ins[t], cfg)
                s.synchronize()
                results[t] = (r.O, r.report.mask.mask_bits)
        except Exception as e:  # noqa: BLE001 - surfaced below
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(t,)) for t in range(len(ins))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors
    for (O, m), (O_ref, m_ref) in zip(results, refs):
        assert torch.equal(O, O_ref)
        assert torch.equal(m, m_ref)


def test_error_text_is_thread_local():
    from paper_2512_14082_b200 import workloads
    Q, K, V = workloads.planted_blocks(1024, 4, 2, 64, 64, seed=3, gain=8.0)
    bad = us().CompressionConfig(c_q=3)  # S=64 not divisible by c_q=3
    good = us().CompressionConfig(P=0.9)
    seen_bad, seen_good = [], []

    def bad_worker():
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(50):
                try:
                    us().select_blocks(Q, K, bad)
                except ValueError as e:
                    seen_bad.append(str(e))

    def good_worker():
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(20):
                us().select_blocks(Q, K, good)
                seen_good.append(us().api.lib().us_last_error().decode())
            s.synchronize()

    th = [threading.Thread(target=bad_worker), threading.Thread(target=good_worker)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert len(seen_bad) == 50 and all(m == "select_blocks: S=64 not divisible by c_q=3" for m in seen_bad)
    assert len(seen_good) == 20 and all("c_q=3" not in m for m in seen_good)
