"""numpy/ctypes front-end for the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py. The product package never imports this module.
Every function mirrors one reference function; see oracle/oracle.h for the
file:line each one restates.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.path.join(ROOT, "oracle", "_build", "liboracle.so")

POOL_MEAN, POOL_MAX, POOL_STOCHASTIC = 0, 1, 2
POST_SOFTMAX, PRE_SOFTMAX = 0, 1
TOP_P, TOP_K = 0, 1
WL_GAUSSIAN, WL_PLANTED, WL_LOCALITY_SHIFT = 0, 1, 2
PROXY_UNISPARSE, PROXY_ANTIDIAGONAL, PROXY_LAST_BLOCK = 0, 1, 2
K_MASKED_SCORE = -float(np.finfo(np.float32).max)


class OrCfg(C.Structure):
    _fields_ = [("H", C.c_int), ("H_kv", C.c_int), ("L", C.c_int), ("d_k", C.c_int),
                ("S", C.c_int), ("c_q", C.c_int), ("c_k", C.c_int), ("c_h", C.c_int),
                ("strategy", C.c_int), ("causal_mode", C.c_int), ("select_mode", C.c_int),
                ("P", C.c_double), ("top_k", C.c_int), ("seed", C.c_uint64)]


def cfg(H, L, d_k, S, *, H_kv=None, c_q=8, c_k=8, c_h=1, strategy=POOL_MEAN,
        causal_mode=POST_SOFTMAX, select_mode=TOP_P, P=0.95, top_k=0, seed=0) -> OrCfg:
    return OrCfg(H, H if H_kv is None else H_kv, L, d_k, S, c_q, c_k, c_h, strategy,
                 causal_mode, select_mode, P, top_k, seed)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
        _lib = C.CDLL(LIB_PATH)
        _lib.or_last_error.restype = C.c_char_p
        _lib.or_mix64.restype = C.c_uint64
        _lib.or_mix64.argtypes = [C.c_uint64]
        _lib.or_chain_seed.restype = C.c_uint64
        _lib.or_chain_seed.argtypes = [C.c_uint64, C.c_uint64]
        _lib.or_top_p_row.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.or_top_k_row.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.or_gen_workload.argtypes = [C.c_int] * 6 + [C.c_uint64, C.c_double, C.c_double, C.c_int] + [C.c_void_p] * 4 + [C.c_int]
        _lib.or_build_block_mask.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_void_p, C.c_void_p]
        _lib.or_selection_flops.argtypes = [C.c_uint64] * 4 + [C.c_int] * 4 + [C.c_uint64, C.c_void_p]
        _lib.or_rng_draws.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p]
        _lib.or_pool_sequence.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_void_p]
        _lib.or_spearman_rho.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        _lib.or_block_recall.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        _lib.or_planted_recall.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        _lib.or_mean_row_spearman.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                              C.c_void_p, C.c_void_p]
    return _lib


class OracleError(ValueError):
    pass


def _check(rc):
    if rc != 0:
        raise OracleError(lib().or_last_error().decode())


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- rng
def mix64(z: int) -> int:
    return lib().or_mix64(z)


def chain_seed(seed: int, *tags: int) -> int:
    for t in tags:
        seed = lib().or_chain_seed(seed, t)
    return seed


def rng_draws(stream_seed: int, kind: str, n: int) -> np.ndarray:
    k = {"u64": 0, "double": 1, "double_open": 2, "gaussian": 3}[kind]
    out = np.zeros(n, dtype=np.uint64)
    lib().or_rng_draws(stream_seed, k, n, _p(out))
    return out if k == 0 else out.view(np.float64)


# ---------------------------------------------------------------- workloads
def gen_workload(kind: int, L: int, H: int, d_k: int, S: int, seed: int, *, H_kv=None,
                 sigma=0.1, gain=4.0, m=2, nthreads=0):
    H_kv = H if H_kv is None else H_kv
    Q = np.zeros((H, L, d_k), np.float32)
    K = np.zeros((H_kv, L, d_k), np.float32)
    V = np.zeros((H_kv, L, d_k), np.float32)
    N = L // S if S > 0 else 0
    planted = np.full((H, N, max(m, 1)), -1, np.int32)
    _check(lib().or_gen_workload(kind, L, H, H_kv, d_k, S, seed, sigma, gain, m, _p(Q), _p(K),
                                 _p(V), _p(planted), nthreads))
    return Q, K, V, planted


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 -> fp32 (what the GPU path ingests)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    nan = np.isnan(x)
    out = r.astype(np.uint32).view(np.float32).copy()
    out[nan] = x[nan]
    return out


# ---------------------------------------------------------------- validation
def validate(c: OrCfg) -> str:
    buf = C.create_string_buffer(2048)
    lib().or_validate(C.byref(c), buf, 2048)
    return buf.value.decode()


# ---------------------------------------------------------------- compression
def pool_sequence(x: np.ndarray, c: int, strategy=POOL_MEAN, seed=0) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    rows, cols = x.shape
    out = np.zeros((rows // c if c > 0 else 0, cols), np.float32)
    _check(lib().or_pool_sequence(_p(x), rows, cols, c, strategy, seed, _p(out)))
    return out


def compress(c: OrCfg, Q: np.ndarray, K: np.ndarray):
    Hc = c.H // c.c_h
    Qc = np.zeros((Hc, c.L // c.c_q, c.d_k), np.float32)
    Kc = np.zeros((Hc, c.L // c.c_k, c.d_k), np.float32)
    _check(lib().or_compress(C.byref(c), _p(np.ascontiguousarray(Q, np.float32)),
                             _p(np.ascontiguousarray(K, np.float32)), _p(Qc), _p(Kc)))
    return Qc, Kc


# ---------------------------------------------------------------- proxy
def proxy_scores(c: OrCfg, Qc, Kc, with_A=False, nthreads=0):
    Hc, N = c.H // c.c_h, c.L // c.S
    scores = np.zeros((Hc, N, N), np.float64)
    A = np.zeros((Hc, c.L // c.c_q, c.L // c.c_k), np.float64) if with_A else None
    _check(lib().or_proxy_scores(C.byref(c), _p(Qc), _p(Kc), _p(scores),
                                 _p(A) if with_A else None, nthreads))
    return (scores, A) if with_A else scores


def proxy_score_rows(c: OrCfg, Qc, Kc, hc: int, qblocks, nthreads=0):
    qb = np.ascontiguousarray(qblocks, np.int32)
    out = np.zeros((len(qb), c.L // c.S), np.float64)
    _check(lib().or_proxy_score_rows(C.byref(c), _p(Qc), _p(Kc), hc, _p(qb), len(qb), _p(out),
                                     nthreads))
    return out


# ---------------------------------------------------------------- competitor proxies
def antidiagonal_block_scores(Q, K, S: int, stride: int, nthreads=0):
    H, L, d = Q.shape
    N = L // S
    out = np.zeros((H, N, N), np.float64)
    _check(lib().or_antidiagonal_block_scores(H, K.shape[0], L, d, S, stride, _p(np.ascontiguousarray(Q, np.float32)),
                                              _p(np.ascontiguousarray(K, np.float32)), _p(out), nthreads))
    return out


def last_block_probe_scores(Q, K, S: int, nthreads=0):
    H, L, d = Q.shape
    N = L // S
    out = np.zeros((H, N, N), np.float64)
    _check(lib().or_last_block_probe_scores(H, K.shape[0], L, d, S, _p(np.ascontiguousarray(Q, np.float32)),
                                            _p(np.ascontiguousarray(K, np.float32)), _p(out), nthreads))
    return out


# ---------------------------------------------------------------- selection
def top_p_row(scores, P: float):
    s = np.ascontiguousarray(scores, np.float64)
    idx = np.zeros(max(len(s), 1), np.int32)
    cnt, cov = C.c_int(0), C.c_double(0)
    _check(lib().or_top_p_row(_p(s), len(s), P, _p(idx), C.byref(cnt), C.byref(cov)))
    return list(idx[: cnt.value]), cov.value


def top_k_row(scores, k: int):
    s = np.ascontiguousarray(scores, np.float64)
    idx = np.zeros(max(len(s), 1), np.int32)
    cnt, cov = C.c_int(0), C.c_double(0)
    _check(lib().or_top_k_row(_p(s), len(s), k, _p(idx), C.byref(cnt), C.byref(cov)))
    return list(idx[: cnt.value]), cov.value


def build_block_mask(scores, H: int, c_h: int, P: float, select_mode=TOP_P, top_k=0):
    scores = np.ascontiguousarray(scores, np.float64)
    N = scores.shape[-1]
    mask = np.zeros((H, N, N), np.uint8)
    cov = np.zeros((H, N), np.float64)
    _check(lib().or_build_block_mask(_p(scores), H, N, c_h, select_mode, P, top_k, _p(mask),
                                     _p(cov)))
    return mask.astype(bool), cov


# ---------------------------------------------------------------- attention
def dense_attention(Q, K, V, causal=True, nthreads=0):
    H, L, d = Q.shape
    O = np.zeros((H, L, d), np.float32)
    lse = np.zeros((H, L), np.float64)
    _check(lib().or_dense_attention(H, K.shape[0], L, d, _p(Q), _p(K), _p(V), int(causal), _p(O),
                                    _p(lse), nthreads))
    return O, lse


def exact_block_mass(Q, K, S, nthreads=0):
    H, L, d = Q.shape
    N = L // S
    mass = np.zeros((H, N, N), np.float64)
    _check(lib().or_exact_block_mass(H, K.shape[0], L, d, S, _p(Q), _p(K), _p(mass), nthreads))
    return mass


def block_sparse_attention(Q, K, V, mask, S, nthreads=0):
    H, L, d = Q.shape
    m = np.ascontiguousarray(mask, np.uint8)
    O = np.zeros((H, L, d), np.float32)
    lse = np.zeros((H, L), np.float64)
    _check(lib().or_block_sparse_attention(H, K.shape[0], L, d, S, _p(Q), _p(K), _p(V), _p(m),
                                           _p(O), _p(lse), nthreads))
    return O, lse


def block_sparse_attention_rows(Q, K, V, mask, S, heads, qblocks, nthreads=0):
    H, L, d = Q.shape
    m = np.ascontiguousarray(mask, np.uint8)
    hh = np.ascontiguousarray(heads, np.int32)
    qb = np.ascontiguousarray(qblocks, np.int32)
    O = np.zeros((len(hh), S, d), np.float32)
    lse = np.zeros((len(hh), S), np.float64)
    _check(lib().or_block_sparse_attention_rows(H, K.shape[0], L, d, S, _p(Q), _p(K), _p(V), _p(m),
                                                _p(hh), _p(qb), len(hh), _p(O), _p(lse), nthreads))
    return O, lse


# ---------------------------------------------------------------- metrics
FLOP_KEYS = ("compression", "compressed_qk", "softmax_aggregation", "top_p", "sparse_attention",
             "dense_attention")


def selection_flops(L, H, d_k, S, c_q=8, c_k=8, c_h=1, proxy=PROXY_UNISPARSE, stride=8):
    out = np.zeros(6, np.uint64)
    _check(lib().or_selection_flops(L, H, d_k, S, c_q, c_k, c_h, proxy, stride, _p(out)))
    return {k: int(v) for k, v in zip(FLOP_KEYS, out)}


def output_fidelity(test, ref):
    t = np.ascontiguousarray(test, np.float32)
    r = np.ascontiguousarray(ref, np.float32)
    H, L, d = t.shape
    out = np.zeros(3, np.float64)
    _check(lib().or_output_fidelity(_p(t), _p(r), H, L, d, _p(out)))
    return {"max_abs": out[0], "mean_rel": out[1], "cosine": out[2]}


def spearman_rho(a, b):
    """spearman_rho (metrics.cpp:100-116): None when one side is flat."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    if a.shape != b.shape:
        raise OracleError("spearman_rho: length mismatch")
    rho = np.zeros(1, np.float64)
    d = np.zeros(1, np.int32)
    _check(lib().or_spearman_rho(_p(a), _p(b), a.size, _p(rho), _p(d)))
    return float(rho[0]) if d[0] else None


def block_recall(mask, ref, k: int) -> float:
    """block_recall (metrics.cpp:155-176): mask bool [H][N][N], ref [H][N][N]."""
    m = np.ascontiguousarray(mask, np.uint8)
    r = np.ascontiguousarray(ref, np.float64)
    H, N, _ = r.shape
    out = np.zeros(1, np.float64)
    _check(lib().or_block_recall(_p(m), _p(r), H, N, int(k), _p(out)))
    return float(out[0])


def planted_recall(mask, planted) -> float:
    """planted_recall (metrics.cpp:178-199): mask bool [H][N][N], planted int [H][N][m] (-1 = none)."""
    mk = np.ascontiguousarray(mask, np.uint8)
    pl = np.ascontiguousarray(planted, np.int32)
    H, N, m = pl.shape
    out = np.zeros(1, np.float64)
    _check(lib().or_planted_recall(_p(mk), _p(pl), H, N, m, _p(out)))
    return float(out[0])


def mean_row_spearman(proxy, ref, c_h: int):
    """mean_row_spearman (metrics.cpp:201-224) -> (mean, defined, undefined)."""
    p = np.ascontiguousarray(proxy, np.float64)
    r = np.ascontiguousarray(ref, np.float64)
    H, N, _ = r.shape
    if c_h <= 0 or H % c_h != 0 or p.shape[0] != H // c_h:
        raise OracleError("mean_row_spearman: head counts disagree")
    mean = np.zeros(1, np.float64)
    d = np.zeros(1, np.int64)
    u = np.zeros(1, np.int64)
    _check(lib().or_mean_row_spearman(_p(p), _p(r), H, N, int(c_h), _p(mean), _p(d), _p(u)))
    return float(mean[0]), int(d[0]), int(u[0])


def unisparse_attn(c: OrCfg, Q, K, V, nthreads=0):
    N = c.L // c.S
    O = np.zeros((c.H, c.L, c.d_k), np.float32)
    lse = np.zeros((c.H, c.L), np.float64)
    mask = np.zeros((c.H, N, N), np.uint8)
    cov = np.zeros((c.H, N), np.float64)
    _check(lib().or_unisparse_attn(C.byref(c), _p(Q), _p(K), _p(V), _p(O), _p(lse), _p(mask),
                                   _p(cov), nthreads))
    return O, lse, mask.astype(bool), cov


def sparsity_ratio(mask: np.ndarray) -> np.ndarray:
    """metrics.cpp:87-93: rho per head = 1 - selected / (N(N+1)/2)."""
    N = mask.shape[-1]
    return 1.0 - mask.reshape(mask.shape[0], -1).sum(1) / (N * (N + 1) / 2.0)
