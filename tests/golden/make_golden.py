"""Freezes oracle outputs on the reference generator's own inputs as golden
fixtures (test infrastructure; run here, committed, never run on the GPU box).

The reference ships no golden vector files (proj/.gitignore:1 drops examples/);
its tests regenerate instances from seeds, e.g. gen_workload(Gaussian, 1024, 2,
64, 128, seed 5) in test_pipeline.cpp:10. The oracle ports that generator
bit-faithfully (rng.hpp:11-67, workloads.cpp:18-128), so each case below is
(generator call, config) -> (block scores f64, mask, coverage, O f32 rows, lse),
stored compactly in one .npz per case. tests/test_golden.py re-runs the oracle
and requires bit equality (the oracle is deterministic: -ffp-contract=off,
fixed summation order), and the GPU tests compare the CUDA path against the
same fixtures.

    python tests/golden/make_golden.py
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_py as O  # noqa: E402

# name: (workload kind, L, H, H_kv, d, S, seed, gain, cfg kwargs)
CASES = {
    # test_pipeline.cpp:10 instance (reference geometry S=128), P=0.9 post-softmax
    "gaussian_L1024_H2_d64_S128_seed5": (O.WL_GAUSSIAN, 1024, 2, 2, 64, 128, 5, 4.0,
                                         dict(P=0.9)),
    # GPU geometry (S=64), planted blocks, GQA 4/2, pre-softmax and head compression
    "planted_L2048_H4_Hkv2_d64_pre": (O.WL_PLANTED, 2048, 4, 2, 64, 64, 21, 8.0,
                                      dict(P=0.95, causal_mode=O.PRE_SOFTMAX)),
    "planted_L2048_H4_Hkv2_d128_ch2": (O.WL_PLANTED, 2048, 4, 2, 128, 64, 22, 8.0,
                                       dict(P=0.9, c_h=2)),
    "planted_L4096_H2_Hkv1_d128_topk": (O.WL_PLANTED, 4096, 2, 1, 128, 64, 23, 8.0,
                                        dict(select_mode=O.TOP_K, top_k=8)),
}


def inputs(kind, L, H, H_kv, d, S, seed, gain):
    Q, K, V, _ = O.gen_workload(kind, L, H, d, S, seed, H_kv=H_kv, gain=gain)
    return O.bf16_round(Q), O.bf16_round(K), O.bf16_round(V)


def compute(name):
    kind, L, H, H_kv, d, S, seed, gain, kw = CASES[name]
    Q, K, V = inputs(kind, L, H, H_kv, d, S, seed, gain)
    c = O.cfg(H, L, d, S, H_kv=H_kv, **kw)
    Qc, Kc = O.compress(c, Q, K)
    scores = O.proxy_scores(c, Qc, Kc)
    mask, cov = O.build_block_mask(scores, H, c.c_h, c.P, c.select_mode, c.top_k)
    Ofull, lse = O.block_sparse_attention(Q, K, V, mask, S)
    return dict(scores=scores, mask=np.packbits(mask, axis=-1), mask_shape=np.array(mask.shape),
                coverage=cov, O_rows=Ofull[:, ::37, :].copy(), lse=lse,
                O_sha256=np.frombuffer(hashlib.sha256(Ofull.tobytes()).digest(), np.uint8),
                Qc_sha256=np.frombuffer(hashlib.sha256(Qc.tobytes() + Kc.tobytes()).digest(), np.uint8))


def main():
    for name in CASES:
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **compute(name))
        print("wrote", name)


if __name__ == "__main__":
    main()
