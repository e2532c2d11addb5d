"""Python mirror of the reference operator API over the C ABI (include/us_api.h).

Names, arguments and error behaviour follow /root/reference/proj/include/unisparse/:

    compress(Q, K, cfg)                    -> (Qc, Kc)            compression.hpp:89
    select_blocks(Q, K, cfg)               -> SparsityReport      pipeline.hpp:19
    build_block_mask(scores, cfg)          -> Selection           selection.hpp:41
    block_sparse_attention(Q, K, V, mask)  -> (O, lse)            attention.hpp:27
    unisparse_attn(Q, K, V, cfg)           -> UniSparseResult     pipeline.hpp:16
    dense_attention(Q, K, V)               -> (O, lse)            attention.hpp:21

Tensors are torch CUDA tensors (torch is only the device-memory/stream
plumbing here): Q bf16 [B,H,L,d], K/V bf16 [B,H_kv,L,d] (3-D inputs are
treated as B = 1). Shape/config violations raise ValueError carrying the
reference's message ("select_blocks: L=1000 not divisible by S=64"), exactly
where the reference throws std::invalid_argument. There is no CPU fallback:
without the CUDA library every call raises.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import dataclasses
import functools
import math
import os
import threading
from typing import Optional

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("US_LIB_PATH_OVERRIDE") or os.path.join(_PKG, "_build", "libunisparse_b200.so")

US_OK, US_ERR_INVALID_ARGUMENT, US_ERR_UNSUPPORTED, US_ERR_CUDA, US_ERR_INVALID_MASK, \
    US_ERR_NONFINITE, US_ERR_WORKSPACE, US_ERR_IO = range(8)
POOL_MEAN, POOL_MAX, POOL_STOCHASTIC = 0, 1, 2
POST_SOFTMAX_BLOCK_CAUSAL, PRE_SOFTMAX_COMPRESSED_CAUSAL = 0, 1
DTYPE_BF16, DTYPE_F32 = 0, 1
FLAG_NONCAUSAL = 2
SELECT_TOP_P, SELECT_TOP_K = 0, 1
PROXY_UNISPARSE, PROXY_ANTIDIAGONAL, PROXY_LAST_BLOCK = 0, 1, 2
FLAG_SYNC_CHECK = 1


class UnsupportedError(ValueError):
    """Valid for the reference, outside what the GPU path implements."""


class InvalidMaskError(ValueError):
    pass


class CudaError(RuntimeError):
    pass


class IoError(RuntimeError):
    """File I/O failure (the reference throws std::runtime_error, tensor_io.cpp:15-17)."""


class UsParams(C.Structure):
    _fields_ = [("B", C.c_int32), ("H", C.c_int32), ("H_kv", C.c_int32), ("L", C.c_int32),
                ("d_k", C.c_int32), ("S", C.c_int32), ("c_q", C.c_int32), ("c_k", C.c_int32),
                ("c_h", C.c_int32), ("strategy", C.c_int32), ("causal_mode", C.c_int32),
                ("select_mode", C.c_int32), ("P", C.c_double), ("top_k", C.c_int32),
                ("flags", C.c_int32), ("seed", C.c_uint64), ("dtype", C.c_int32), ("head0", C.c_int32)]


class UsSelection(C.Structure):
    _fields_ = [("mask_bits", C.c_void_p), ("counts", C.c_void_p), ("coverage", C.c_void_p),
                ("scores", C.c_void_p), ("indices", C.c_void_p)]


@dataclasses.dataclass
class CompressionConfig:
    """types.hpp:54-62, plus the north-star extensions (top-k selection)."""
    c_q: int = 8
    c_k: int = 8
    c_h: int = 1
    strategy: int = POOL_MEAN
    P: float = 0.95
    causal_mode: int = POST_SOFTMAX_BLOCK_CAUSAL
    seed: int = 0
    select_mode: int = SELECT_TOP_P
    top_k: int = 0


_lib = None
_lib_lock = threading.Lock()


def _bind(L: C.CDLL) -> C.CDLL:
    L.us_version.restype = C.c_char_p
    L.us_last_error.restype = C.c_char_p
    L.us_validate.argtypes = [C.POINTER(UsParams), C.c_char_p, C.c_size_t]
    L.us_workspace_bytes.restype = C.c_size_t
    L.us_workspace_bytes.argtypes = [C.POINTER(UsParams)]
    L.us_attention_workspace_bytes.restype = C.c_size_t
    L.us_attention_workspace_bytes.argtypes = [C.POINTER(UsParams)]
    vp = C.c_void_p
    L.us_compress.argtypes = [C.POINTER(UsParams), vp, vp, vp, vp, vp, C.c_size_t, vp]
    L.us_select.argtypes = [C.POINTER(UsParams), vp, vp, C.POINTER(UsSelection), vp, C.c_size_t, vp]
    L.us_build_block_mask.argtypes = [C.POINTER(UsParams), vp, C.POINTER(UsSelection), vp, C.c_size_t, vp]
    L.us_select_proxy.argtypes = [C.POINTER(UsParams), C.c_int32, C.c_int32, vp, vp, C.POINTER(UsSelection),
                                  vp, C.c_size_t, vp]
    L.us_proxy_workspace_bytes.restype = C.c_size_t
    L.us_proxy_workspace_bytes.argtypes = [C.POINTER(UsParams), C.c_int32, C.c_int32]
    L.us_sparse_attention.argtypes = [C.POINTER(UsParams), vp, vp, vp, vp, C.c_int32, vp, vp, vp, C.c_size_t, vp]
    L.us_unisparse_attention.argtypes = [C.POINTER(UsParams), vp, vp, vp, vp, vp, C.POINTER(UsSelection), vp,
                                         C.c_size_t, vp]
    L.us_dense_attention.argtypes = [C.POINTER(UsParams), vp, vp, vp, vp, vp, vp, C.c_size_t, vp]
    L.us_check_device_errors.argtypes = [C.POINTER(UsParams), vp, vp]
    L.us_selection_flops.argtypes = [C.POINTER(UsParams), C.c_int32, C.c_int32, vp]
    L.us_last_launch_count.restype = C.c_int32
    L.us_write_tensor.argtypes = [C.c_char_p, vp, C.c_int32, C.c_int32, C.c_int32]
    L.us_read_tensor_header.argtypes = [C.c_char_p, vp, vp, vp]
    L.us_read_tensor.argtypes = [C.c_char_p, vp, C.c_size_t]
    L.us_save_mask_json.argtypes = [C.c_char_p, vp, C.c_int32, C.c_int32, C.c_int32, C.c_double]
    L.us_load_mask_json.argtypes = [C.c_char_p, vp, vp, vp, vp, C.c_size_t]
    L.us_profile_enable.argtypes = [C.c_int32]
    L.us_profile_read.argtypes = [C.c_void_p, C.c_int32]
    L.us_profile_read.restype = C.c_int32
    L.us_mass_workspace_bytes.restype = C.c_size_t
    L.us_mass_workspace_bytes.argtypes = [C.POINTER(UsParams)]
    L.us_metrics_workspace_bytes.restype = C.c_size_t
    L.us_metrics_workspace_bytes.argtypes = [C.POINTER(UsParams)]
    L.us_exact_block_mass.argtypes = [C.POINTER(UsParams), vp, vp, vp, vp, C.c_size_t, vp]
    L.us_output_fidelity.argtypes = [C.POINTER(UsParams), vp, vp, vp, vp, C.c_size_t, vp]
    L.us_block_recall.argtypes = [C.POINTER(UsParams), vp, C.c_int32, vp, C.c_int32, vp, vp, C.c_size_t, vp]
    L.us_mean_row_spearman.argtypes = [C.POINTER(UsParams), vp, vp, vp, vp, vp, vp, C.c_size_t, vp]
    L.us_planted_recall.argtypes = [C.POINTER(UsParams), vp, C.c_int32, vp, C.c_int32, vp, vp, C.c_size_t, vp]
    L.us_set_attention_impl.argtypes = [C.c_int32]
    if hasattr(L, "us_selftest_umma"):
        L.us_selftest_umma.argtypes = [C.c_int, C.c_int, C.c_int, vp, vp, vp, vp]
    return L


_product = None


def lib() -> C.CDLL:
    """The library every operator of this module calls: the product build, or the
    calibration build inside a `calibration()` block."""
    global _lib, _product
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise CudaError(f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
            _lib = _product = _bind(C.CDLL(LIB_PATH))
        return _lib


CALIB_LIB_PATH = os.path.join(_PKG, "_build", "libunisparse_b200_calib.so")
_calib = None


def calib_lib() -> C.CDLL:
    """The calibration build (-DUS_CALIBRATION): the product plus the measured-slower
    attention variants (us_set_attention_impl 2-5) and the hardware probes
    (us_selftest_*). Loaded separately (RTLD_LOCAL), never the default path."""
    global _calib
    with _lib_lock:
        if _calib is None:
            if not os.path.exists(CALIB_LIB_PATH):
                raise CudaError(f"calibration library not built: {CALIB_LIB_PATH}")
            _calib = _bind(C.CDLL(CALIB_LIB_PATH))
        return _calib


@contextlib.contextmanager
def calibration():
    """Route this module's operators through the calibration library for the block."""
    global _lib
    lib()
    cal = calib_lib()
    with _lib_lock:
        prev = _lib
        _lib = cal
    try:
        yield cal
    finally:
        with _lib_lock:
            _lib = prev


def _raise(status: int, default: str = ""):
    if status == US_OK:
        return
    msg = lib().us_last_error().decode() or default
    if status == US_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == US_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    if status == US_ERR_IO:
        raise IoError(msg)
    if status in (US_ERR_INVALID_MASK, US_ERR_NONFINITE):
        raise InvalidMaskError(msg) if status == US_ERR_INVALID_MASK else ValueError(msg)
    raise CudaError(f"status {status}: {msg}")


def _stream(t: Optional[torch.Tensor] = None):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def make_params(Q: torch.Tensor, K: torch.Tensor, cfg: CompressionConfig, S: int = 64,
                sync_check: bool = False, head0: int = 0) -> UsParams:
    """head0: global index of Q's first head when Q/K/V are a head range of a larger
    layer (head sharding): stochastic pooling seeds with the global head index."""
    B, H, L, d = _bhld(Q)
    H_kv = _bhld(K)[1]
    dtype = DTYPE_F32 if Q.dtype == torch.float32 else DTYPE_BF16
    return UsParams(B, H, H_kv, L, d, S, cfg.c_q, cfg.c_k, cfg.c_h, cfg.strategy, cfg.causal_mode,
                    cfg.select_mode, float(cfg.P), cfg.top_k, FLAG_SYNC_CHECK if sync_check else 0,
                    cfg.seed, dtype, head0)


def _bhld(x: torch.Tensor):
    if x.dim() == 3:
        return (1, *x.shape)
    if x.dim() != 4:
        raise ValueError(f"expected [B,H,L,d] or [H,L,d] tensor, got shape {tuple(x.shape)}")
    return tuple(x.shape)


def _on_input_device(fn):
    """Run an operator with Q's device as the current device, so the selection
    buffers, the workspace and the launch stream all live on the inputs' GPU."""
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        t = next((a for a in args if isinstance(a, torch.Tensor)), None)
        if t is not None and t.is_cuda:
            with torch.cuda.device(t.device):
                return fn(*args, **kwargs)
        return fn(*args, **kwargs)
    return wrapper


def _check_inputs(*ts: torch.Tensor):
    dev = None
    for t in ts:
        if t.is_cuda:
            if dev is not None and t.device != dev:
                raise ValueError(f"inputs live on different devices ({dev} and {t.device})")
            dev = t.device
        if not t.is_cuda:
            raise ValueError("inputs must be CUDA tensors (the GPU path has no CPU fallback)")
        if t.dtype not in (torch.bfloat16, torch.float32):
            raise ValueError(f"inputs must be bfloat16 or float32, got {t.dtype}")
        if t.dtype != ts[0].dtype:
            raise ValueError(f"inputs must share one dtype ({ts[0].dtype} and {t.dtype})")
        if not t.is_contiguous():
            raise ValueError("inputs must be contiguous")


# ------------------------------------------------------------------ workspace cache
# Workspaces are reused in stream order, so the cache is keyed by (device, stream):
# calls on different streams (or host threads using different streams) never share one.
_ws_cache: dict = {}


def _ws_key():
    return (torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream)


def workspace(p: UsParams, attention_only: bool = False) -> torch.Tensor:
    """The cached device workspace for a call: us_workspace_bytes, or the smaller
    us_attention_workspace_bytes for block_sparse_attention / dense_attention."""
    need = (lib().us_attention_workspace_bytes if attention_only else lib().us_workspace_bytes)(C.byref(p))
    key = _ws_key()
    cur = _ws_cache.get(key)
    if cur is None or cur.numel() < need:
        cur = torch.empty(max(need, 256), dtype=torch.uint8, device=f"cuda:{key[0]}")
        _ws_cache[key] = cur
    return cur


def validate(p: UsParams) -> str:
    buf = C.create_string_buffer(4096)
    lib().us_validate(C.byref(p), buf, 4096)
    return buf.value.decode()


# ------------------------------------------------------------------ results
@dataclasses.dataclass
class Selection:
    mask_bits: torch.Tensor         # int32 view of u32 words [B, planes, N, W]
    counts: torch.Tensor            # [B, planes, N]
    coverage: torch.Tensor          # [B, planes, N] float64
    scores: Optional[torch.Tensor]  # [B, planes, N, N] float32
    indices: Optional[torch.Tensor] # [B, planes, N, N] int16
    c_h: int
    N: int

    def dense_mask(self, H: Optional[int] = None) -> torch.Tensor:
        """Boolean [B, H, N, N] mask (planes broadcast to heads, selection.cpp:80-84)."""
        words = self.mask_bits.to(torch.int64) & 0xFFFFFFFF
        bits = ((words.unsqueeze(-1) >> torch.arange(32, device=words.device)) & 1).bool()
        m = bits.flatten(-2)[..., : self.N]
        return m.repeat_interleave(self.c_h, dim=1)


@dataclasses.dataclass
class SparsityReport:
    """metrics.hpp:77-83 — rho per head, selected per head, FLOP breakdown, mask."""
    rho: list
    rho_mean: float
    selected: list
    flops: dict
    mask: Selection


@dataclasses.dataclass
class UniSparseResult:
    O: torch.Tensor
    lse: torch.Tensor
    report: SparsityReport


FLOP_KEYS = ("compression", "compressed_qk", "softmax_aggregation", "top_p", "sparse_attention",
             "dense_attention")


def selection_flops(p: UsParams, proxy: int = PROXY_UNISPARSE, stride: int = 8) -> dict:
    out = (C.c_uint64 * 6)()
    _raise(lib().us_selection_flops(C.byref(p), proxy, stride, C.cast(out, C.c_void_p)))
    return {k: int(v) for k, v in zip(FLOP_KEYS, out)}


def _alloc_selection(p: UsParams, with_scores: bool, with_indices: bool) -> Selection:
    dev = torch.cuda.current_device()
    planes, N = p.H // p.c_h, p.L // p.S
    W = (N + 31) // 32
    return Selection(
        mask_bits=torch.empty((p.B, planes, N, W), dtype=torch.int32, device=dev),
        counts=torch.empty((p.B, planes, N), dtype=torch.int32, device=dev),
        coverage=torch.empty((p.B, planes, N), dtype=torch.float64, device=dev),
        scores=torch.zeros((p.B, planes, N, N), dtype=torch.float32, device=dev) if with_scores else None,
        indices=torch.empty((p.B, planes, N, N), dtype=torch.int16, device=dev) if with_indices else None,
        c_h=p.c_h, N=N)


def _sel_struct(s: Selection) -> UsSelection:
    return UsSelection(s.mask_bits.data_ptr(), s.counts.data_ptr(), s.coverage.data_ptr(),
                       s.scores.data_ptr() if s.scores is not None else None,
                       s.indices.data_ptr() if s.indices is not None else None)


def make_report(p: UsParams, sel: Selection) -> SparsityReport:
    """make_sparsity_report (metrics.cpp:226-237) from per-row counts."""
    N = p.L // p.S
    per_plane = sel.counts.to(torch.int64).sum(-1)                 # [B, planes]
    per_head = per_plane.repeat_interleave(p.c_h, dim=1)           # [B, H]
    selected = per_head.sum(0).tolist() if p.B > 1 else per_head[0].tolist()
    causal = N * (N + 1) / 2.0
    rho = [1.0 - s / (causal * p.B) for s in selected]
    flops = selection_flops(p)
    flops["sparse_attention"] = int(sum(selected)) * 4 * p.S * p.S * p.d_k
    return SparsityReport(rho=rho, rho_mean=sum(rho) / len(rho), selected=selected, flops=flops, mask=sel)


# ------------------------------------------------------------------ operators
@_on_input_device
def compress(Q: torch.Tensor, K: torch.Tensor, cfg: CompressionConfig, S: int = 64):
    """compress (compression.cpp:5-25): f32 Qc [B,H/c_h,L/c_q,d], Kc [B,H/c_h,L/c_k,d]."""
    _check_inputs(Q, K)
    p = make_params(Q, K, cfg, S)
    B, H, L, d = _bhld(Q)
    Hc = max(H // max(cfg.c_h, 1), 1)
    Qc = torch.empty((B, Hc, L // max(cfg.c_q, 1), d), dtype=torch.float32, device=Q.device)
    Kc = torch.empty((B, Hc, L // max(cfg.c_k, 1), d), dtype=torch.float32, device=Q.device)
    ws = workspace(p) if d not in (64, 128) else None  # other d_k run zero-padded in the workspace
    _raise(lib().us_compress(C.byref(p), _ptr(Q), _ptr(K), _ptr(Qc), _ptr(Kc), _ptr(ws),
                             ws.numel() if ws is not None else 0, _stream()))
    return Qc, Kc


@_on_input_device
def select_blocks(Q: torch.Tensor, K: torch.Tensor, cfg: CompressionConfig, S: int = 64,
                  with_scores: bool = False, with_indices: bool = False,
                  sync_check: bool = True, proxy: int = PROXY_UNISPARSE, stride: int = 8) -> SparsityReport:
    """select_blocks(proxy, in, cfg, stride) (pipeline.cpp:5-17). proxy = PROXY_UNISPARSE
    (the compressed proxy) or PROXY_ANTIDIAGONAL (XAttention-style, baselines.cpp:10-52;
    per original head, c_h forced to 1 as in pipeline.cpp:11)."""
    _check_inputs(Q, K)
    if proxy != PROXY_UNISPARSE:
        cfg = dataclasses.replace(cfg, c_h=1)
    p = make_params(Q, K, cfg, S, sync_check)
    need = lib().us_proxy_workspace_bytes(C.byref(p), proxy, stride)
    ws = workspace(p)
    if ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=Q.device)
        _ws_cache[_ws_key()] = ws
    sel = _alloc_selection(p, with_scores, with_indices)
    ss = _sel_struct(sel)
    _raise(lib().us_select_proxy(C.byref(p), proxy, stride, _ptr(Q), _ptr(K), C.byref(ss), _ptr(ws), ws.numel(),
                                 _stream()))
    rep = make_report(p, sel)
    rep.flops = selection_flops(p, proxy, stride)
    rep.flops["sparse_attention"] = int(sum(rep.selected)) * 4 * p.S * p.S * p.d_k
    return rep


@_on_input_device
def build_block_mask(scores: torch.Tensor, cfg: CompressionConfig, H: Optional[int] = None,
                     S: int = 64, with_indices: bool = False) -> Selection:
    """build_block_mask (selection.cpp:60-88) on f32 block scores [B, planes, N, N]."""
    if scores.dim() == 3:
        scores = scores.unsqueeze(0)
    if scores.dtype != torch.float32 or not scores.is_cuda:
        raise ValueError("scores must be a float32 CUDA tensor")
    scores = scores.contiguous()
    B, planes, N, _ = scores.shape
    H = planes * cfg.c_h if H is None else H
    p = UsParams(B, H, H, N * S, 64, S, cfg.c_q, cfg.c_k, cfg.c_h, cfg.strategy, cfg.causal_mode,
                 cfg.select_mode, float(cfg.P), cfg.top_k, FLAG_SYNC_CHECK, cfg.seed)
    ws = workspace(p)
    sel = _alloc_selection(p, False, with_indices)
    ss = _sel_struct(sel)
    _raise(lib().us_build_block_mask(C.byref(p), _ptr(scores), C.byref(ss), _ptr(ws), ws.numel(), _stream()))
    return sel


@_on_input_device
def block_sparse_attention(Q, K, V, mask_bits: torch.Tensor, heads_per_plane: int = 1, S: int = 64,
                           validate_mask: bool = True, with_lse: bool = True):
    """block_sparse_attention (attention.cpp:89-137). mask_bits: int32 [B, planes, N, W]."""
    _check_inputs(Q, K, V)
    p = make_params(Q, K, CompressionConfig(c_q=1, c_k=1, c_h=1), S, validate_mask)
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=Q.device)
    B, H, L, _ = _bhld(Q)
    lse = torch.empty((B, H, L), dtype=torch.float32, device=Q.device) if with_lse else None
    ws = workspace(p, attention_only=True)
    _raise(lib().us_sparse_attention(C.byref(p), _ptr(Q), _ptr(K), _ptr(V), _ptr(mask_bits.contiguous()),
                                     heads_per_plane, _ptr(O), _ptr(lse), _ptr(ws),
                                     ws.numel() if ws is not None else 0, _stream()))
    return O, lse


@_on_input_device
def unisparse_attn(Q, K, V, cfg: CompressionConfig, S: int = 64, with_scores: bool = False,
                   with_indices: bool = False, sync_check: bool = True) -> UniSparseResult:
    """unisparse_attn (pipeline.cpp:19-24)."""
    _check_inputs(Q, K, V)
    p = make_params(Q, K, cfg, S, sync_check)
    ws = workspace(p)
    sel = _alloc_selection(p, with_scores, with_indices)
    ss = _sel_struct(sel)
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=Q.device)
    B, H, L, _ = _bhld(Q)
    lse = torch.empty((B, H, L), dtype=torch.float32, device=Q.device)
    _raise(lib().us_unisparse_attention(C.byref(p), _ptr(Q), _ptr(K), _ptr(V), _ptr(O), _ptr(lse),
                                        C.byref(ss), _ptr(ws), ws.numel(), _stream()))
    return UniSparseResult(O=O, lse=lse, report=make_report(p, sel))


@_on_input_device
def dense_attention(Q, K, V, S: int = 64, with_lse: bool = True, causal: bool = True):
    """dense_attention(in, causal) (attention.cpp:20-54): the block-sparse kernel with
    every causal block selected, or every key block (causal=False, no diagonal mask)."""
    _check_inputs(Q, K, V)
    p = make_params(Q, K, CompressionConfig(c_q=1, c_k=1, c_h=1), S)
    if not causal:
        p.flags |= FLAG_NONCAUSAL
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=Q.device)
    B, H, L, _ = _bhld(Q)
    lse = torch.empty((B, H, L), dtype=torch.float32, device=Q.device) if with_lse else None
    # f32 inputs: bf16 copies in the workspace; d_k outside {64, 128}: zero-padded copies
    ws = workspace(p, attention_only=True) if (Q.dtype == torch.float32 or Q.shape[-1] not in (64, 128)) else None
    _raise(lib().us_dense_attention(C.byref(p), _ptr(Q), _ptr(K), _ptr(V), _ptr(O), _ptr(lse), _ptr(ws),
                                    ws.numel() if ws is not None else 0, _stream()))
    return O, lse


class Engine:
    """Allocation-free repeated calls (bench / serving): params, workspace and
    selection buffers are created once; run() only launches kernels."""

    def __init__(self, Q, K, V, cfg: CompressionConfig, S: int = 64, head0: int = 0):
        _check_inputs(Q, K, V)
        self.device = Q.device
        self.p = make_params(Q, K, cfg, S, head0=head0)
        # a private workspace: run_host() uses it on the engine's own streams, so it
        # must not be shared with other engines or functional calls on this stream
        self.ws = torch.empty(max(int(lib().us_workspace_bytes(C.byref(self.p))), 256), dtype=torch.uint8,
                              device=Q.device)
        self.sel = _alloc_selection(self.p, False, False)
        self.ss = _sel_struct(self.sel)
        self.O = torch.empty(Q.shape, dtype=torch.bfloat16, device=Q.device)
        B, H, L, _ = _bhld(Q)
        self.lse = torch.empty((B, H, L), dtype=torch.float32, device=Q.device)
        self.Q, self.K, self.V = Q, K, V

    def run(self, dense: bool = False):
        with torch.cuda.device(self.device):
            return self._run(dense)

    def _run(self, dense: bool = False):
        if dense:
            _raise(lib().us_dense_attention(C.byref(self.p), _ptr(self.Q), _ptr(self.K), _ptr(self.V),
                                            _ptr(self.O), _ptr(self.lse), _ptr(self.ws), self.ws.numel(),
                                            _stream()))
        else:
            _raise(lib().us_unisparse_attention(C.byref(self.p), _ptr(self.Q), _ptr(self.K), _ptr(self.V),
                                                _ptr(self.O), _ptr(self.lse), C.byref(self.ss),
                                                _ptr(self.ws), self.ws.numel(), _stream()))
        return self.O

    def launches(self) -> int:
        return int(lib().us_last_launch_count())

    # -------------------------------------------------------------- host-buffer path
    def _chunk_plan(self, chunks: int):
        """Split the layer into `chunks` runs of whole KV heads (batch 1): every
        chunk is an independent layer of G*n Q heads over n KV heads (heads never
        couple), so the chunked result equals the one-call result."""
        p = self.p
        G = p.H // p.H_kv
        if p.B != 1 or p.c_h > G or G % p.c_h:
            return None
        chunks = max(1, min(chunks, p.H_kv))
        sizes = [p.H_kv // chunks + (1 if c < p.H_kv % chunks else 0) for c in range(chunks)]
        plan, kv0 = [], 0
        N = p.L // p.S
        W = (N + 31) // 32
        for n in sizes:
            q0, q1 = kv0 * G, (kv0 + n) * G
            cp = UsParams(1, n * G, n, p.L, p.d_k, p.S, p.c_q, p.c_k, p.c_h, p.strategy, p.causal_mode,
                          p.select_mode, p.P, p.top_k, p.flags, p.seed, p.dtype, p.head0 + q0)
            pl0, pl1 = q0 // p.c_h, q1 // p.c_h
            sel = UsSelection(self.sel.mask_bits[0, pl0:pl1].data_ptr(), self.sel.counts[0, pl0:pl1].data_ptr(),
                              self.sel.coverage[0, pl0:pl1].data_ptr(), None, None)
            plan.append((cp, (q0, q1), (kv0, kv0 + n), sel))
            kv0 += n
        return plan

    def run_host(self, Qh, Kh, Vh, Oh, chunks: int = 4, wait: bool = True):
        with torch.cuda.device(self.device):
            return self._run_host(Qh, Kh, Vh, Oh, chunks, wait)

    def _run_host(self, Qh, Kh, Vh, Oh, chunks: int = 4, wait: bool = True):
        """unisparse_attn from (pinned) host buffers: H2D of Q/K/V, the hot path,
        D2H of O, pipelined over KV-head chunks on CUDA streams (copy-in, two
        compute streams, copy-out) so the PCIe transfers overlap the kernels and
        consecutive chunks' kernels overlap each other's tails (chunk c computes on
        stream c % 2 with its own chunk-sized workspace carved from the engine's).
        Enqueues only; returns the event recorded after the last D2H on the copy-out
        stream.

        wait=True: the current stream waits for that event (the call is ordered
        like any other stream op). wait=False: it does not, so back-to-back calls
        overlap — call n+1 copies chunk c in as soon as call n has computed chunk
        c, and computes chunk c once call n's copy-out of chunk c is done (the
        per-chunk hazards on the engine's device buffers); the caller waits on
        the returned event before reading Oh or ordering later work."""
        plan = self._chunk_plan(chunks) if chunks > 1 else None
        cur = torch.cuda.current_stream()
        if not hasattr(self, "_streams"):
            self._streams = (torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream())
        s_in, s_comp, s_out, s_comp2 = self._streams
        start = torch.cuda.Event()
        start.record(cur)
        for s_ in self._streams:
            s_.wait_event(start)
        prev = getattr(self, "_chunk_events", None)
        if prev is not None and (plan is None or len(prev[1]) != len(plan)):
            for s_ in self._streams:  # a different chunking: order after the whole previous call
                s_.wait_event(prev[0])
            prev = None
        self._chunk_events = None
        if plan is None:
            with torch.cuda.stream(s_comp):
                self.Q.copy_(Qh, non_blocking=True)
                self.K.copy_(Kh, non_blocking=True)
                self.V.copy_(Vh, non_blocking=True)
                self.run()
                Oh.copy_(self.O, non_blocking=True)
            done = torch.cuda.Event()
            done.record(s_comp)
            if wait:
                cur.wait_event(done)
            self._chunk_events = (done, [])
            return done
        G = self.p.H // self.p.H_kv
        # two chunk-sized workspaces (one per compute stream) inside the layer's workspace
        wsz = max(int(lib().us_workspace_bytes(C.byref(cp))) for cp, _, _, _ in plan)
        wsz = (wsz + 255) // 256 * 256
        if 2 * wsz > self.ws.numel():
            if getattr(self, "_ws2", None) is None or self._ws2.numel() < 2 * wsz:
                self._ws2 = torch.empty(2 * wsz, dtype=torch.uint8, device=self.ws.device)
            wbase = self._ws2
        else:
            wbase = self.ws
        comp = (s_comp, s_comp2)
        events = []
        for c, (cp, (q0, q1), (k0, k1), sel) in enumerate(plan):
            e_in, e_comp, e_out = torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()
            if prev is not None:
                s_in.wait_event(prev[1][c][0])    # the previous call has consumed Q/K/V chunk c
            with torch.cuda.stream(s_in):
                self.Q[:, q0:q1].copy_(Qh[:, q0:q1], non_blocking=True)
                self.K[:, k0:k1].copy_(Kh[:, k0:k1], non_blocking=True)
                self.V[:, k0:k1].copy_(Vh[:, k0:k1], non_blocking=True)
                e_in.record(s_in)
            sc = comp[c % 2]
            sc.wait_event(e_in)
            if prev is not None:
                sc.wait_event(prev[1][c][1])  # ... and copied O chunk c out
            _raise(lib().us_unisparse_attention(
                C.byref(cp), _ptr(self.Q[:, q0:q1]), _ptr(self.K[:, k0:k1]), _ptr(self.V[:, k0:k1]),
                _ptr(self.O[:, q0:q1]), _ptr(self.lse[:, q0:q1]), C.byref(sel),
                C.c_void_p(wbase.data_ptr() + (c % 2) * wsz), wsz, C.c_void_p(sc.cuda_stream)))
            e_comp.record(sc)
            s_out.wait_event(e_comp)
            with torch.cuda.stream(s_out):
                Oh[:, q0:q1].copy_(self.O[:, q0:q1], non_blocking=True)
                e_out.record(s_out)
            events.append((e_comp, e_out))
        done = torch.cuda.Event()
        done.record(s_out)
        if wait:
            cur.wait_event(done)
        self._chunk_events = (done, events)
        return done


def selftest_umma(mode: int, N: int, bf16: bool, A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
    """Single-tile tcgen05 operand-path check (calibration build, csrc/selftest.cu)."""
    D = torch.empty((128, N), dtype=torch.float32, device=A.device)
    L = calib_lib()
    rc = L.us_selftest_umma(mode, N, int(bf16), _ptr(A), _ptr(B), _ptr(D), _stream())
    if rc:
        raise CudaError(f"status {rc}: {L.us_last_error().decode()}")
    return D


STAGES = ("compress", "proxy", "select", "attention")


def profile_enable(max_calls: int):
    """Record per-stage CUDA events for the next max_calls unisparse_attn calls."""
    _raise(lib().us_profile_enable(max_calls))


def profile_read(max_calls: int):
    """-> list of per-call dicts {stage: ms} (synchronizes on the recorded events)."""
    buf = (C.c_float * (4 * max_calls))()
    n = lib().us_profile_read(C.cast(buf, C.c_void_p), max_calls)
    return [{k: buf[c * 4 + i] for i, k in enumerate(STAGES)} for c in range(n)]


def profile_disable():
    lib().us_profile_disable()


# ------------------------------------------------------------------ on-disk formats (host side)
def write_tensor(path: str, data) -> None:
    """write_tensor (tensor_io.cpp:31-47): f32 [H, L, d_k] array-like -> unisparse.tn file."""
    import numpy as np
    a = np.ascontiguousarray(np.asarray(data, dtype=np.float32))
    if a.ndim != 3:
        raise ValueError("write_tensor: expected [H, L, d_k]")
    _raise(lib().us_write_tensor(path.encode(), a.ctypes.data, *a.shape))


def read_tensor(path: str):
    """read_tensor (tensor_io.cpp:49-81) -> numpy f32 [H, L, d_k]."""
    import numpy as np
    H, L, d = C.c_int32(), C.c_int32(), C.c_int32()
    _raise(lib().us_read_tensor_header(path.encode(), C.byref(H), C.byref(L), C.byref(d)))
    out = np.empty((H.value, L.value, d.value), np.float32)
    _raise(lib().us_read_tensor(path.encode(), out.ctypes.data, out.size))
    return out


def save_mask_json_bits(path: str, bits, H: int, N: int, c_h: int, P: float) -> None:
    """save_mask_json (selection.cpp:90-117) from host u32 planes [H/c_h, N, ceil(N/32)]."""
    import numpy as np
    b = np.ascontiguousarray(np.asarray(bits).view(np.uint32))
    if b.shape != (H // c_h, N, (N + 31) // 32):
        raise ValueError(f"save_mask_json: bits shape {b.shape} != {(H // c_h, N, (N + 31) // 32)}")
    _raise(lib().us_save_mask_json(path.encode(), b.ctypes.data, H, N, c_h, float(P)))


def save_mask_json(path: str, sel: "Selection", H: int, P: float) -> None:
    """save_mask_json of a Selection (batch item 0)."""
    save_mask_json_bits(path, sel.mask_bits[0].contiguous().cpu().numpy(), H, sel.N, sel.c_h, P)


def load_mask_json(path: str):
    """load_mask_json (selection.cpp:119-144) -> (bool mask [H, N, N], P)."""
    import numpy as np
    H, N, P = C.c_int32(), C.c_int32(), C.c_double()
    _raise(lib().us_load_mask_json(path.encode(), C.byref(H), C.byref(N), C.byref(P), None, 0))
    W = (N.value + 31) // 32
    bits = np.zeros((H.value, N.value, W), np.uint32)
    _raise(lib().us_load_mask_json(path.encode(), C.byref(H), C.byref(N), C.byref(P), bits.ctypes.data, bits.size))
    m = ((bits[..., None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool).reshape(H.value, N.value, W * 32)
    return m[..., : N.value], P.value


# ------------------------------------------------------------------ quality metrics (§8f-4)
def _scratch(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def _metric_params(B: int, H: int, L: int, d: int, S: int = 64, c_h: int = 1) -> UsParams:
    return UsParams(B, H, H, L, d, S, 1, 1, c_h, 0, 0, 0, 1.0, 0, 0, 0)


def exact_block_mass(Q: torch.Tensor, K: torch.Tensor, S: int = 64) -> torch.Tensor:
    """exact_block_mass (attention.cpp:56-86): f32 [B, H, N, N] causal attention mass
    per (query block, key block), j <= i written (kMaskedScore above the diagonal)."""
    _check_inputs(Q, K)
    p = make_params(Q, K, CompressionConfig(c_q=1, c_k=1, c_h=1), S)
    B, H, L, _ = _bhld(Q)
    N = L // S
    mass = torch.full((B, H, N, N), -torch.finfo(torch.float32).max, dtype=torch.float32, device=Q.device)
    ws = _scratch(lib().us_mass_workspace_bytes(C.byref(p)), Q.device)
    _raise(lib().us_exact_block_mass(C.byref(p), _ptr(Q), _ptr(K), _ptr(mass), _ptr(ws), ws.numel(), _stream()))
    return mass


def output_fidelity(O_test: torch.Tensor, O_ref: torch.Tensor) -> dict:
    """output_fidelity (metrics.cpp:118-153) of two bf16 [B, H, L, d] outputs."""
    if O_test.shape != O_ref.shape:
        raise ValueError("output_fidelity: shape mismatch")
    _check_inputs(O_test, O_ref)
    B, H, L, d = _bhld(O_test)
    p = _metric_params(B, H, L, d)
    ws = _scratch(lib().us_metrics_workspace_bytes(C.byref(p)), O_test.device)
    out = (C.c_double * 3)()
    _raise(lib().us_output_fidelity(C.byref(p), _ptr(O_test.contiguous()), _ptr(O_ref.contiguous()), out,
                                    _ptr(ws), ws.numel(), _stream()))
    return {"max_abs": out[0], "mean_rel": out[1], "cosine": out[2]}


def block_recall(mask_bits: torch.Tensor, ref: torch.Tensor, k: int, heads_per_plane: int = 1,
                 S: int = 64) -> float:
    """block_recall (metrics.cpp:155-176): mask planes int32 [B, planes, N, W] against
    reference block scores f32 [B, H, N, N]."""
    if ref.dim() == 3:
        ref = ref.unsqueeze(0)
    B, H, N, _ = ref.shape
    if mask_bits.dim() == 3:
        mask_bits = mask_bits.unsqueeze(0)
    if mask_bits.shape[1] * heads_per_plane != H:
        raise ValueError("block_recall: reference must hold one plane per mask head")
    p = _metric_params(B, H, N * S, 64, S)
    ws = _scratch(lib().us_metrics_workspace_bytes(C.byref(p)), ref.device)
    out = C.c_double(0.0)
    _raise(lib().us_block_recall(C.byref(p), _ptr(mask_bits.contiguous()), heads_per_plane,
                                 _ptr(ref.float().contiguous()), int(k), C.byref(out), _ptr(ws), ws.numel(),
                                 _stream()))
    return out.value


def mean_row_spearman(proxy: torch.Tensor, ref: torch.Tensor, c_h: int, S: int = 64):
    """mean_row_spearman (metrics.cpp:201-224) -> (mean, defined, undefined): proxy
    scores f32 [B, H/c_h, N, N] against ref f32 [B, H, N, N]."""
    if ref.dim() == 3:
        ref = ref.unsqueeze(0)
    if proxy.dim() == 3:
        proxy = proxy.unsqueeze(0)
    B, H, N, _ = ref.shape
    if c_h <= 0 or H % c_h != 0 or proxy.shape[1] != H // c_h or proxy.shape[2] != N:
        raise ValueError("mean_row_spearman: head counts disagree")
    p = _metric_params(B, H, N * S, 64, S, c_h)
    ws = _scratch(lib().us_metrics_workspace_bytes(C.byref(p)), ref.device)
    mean, d, u = C.c_double(0.0), C.c_int64(0), C.c_int64(0)
    _raise(lib().us_mean_row_spearman(C.byref(p), _ptr(proxy.float().contiguous()), _ptr(ref.float().contiguous()),
                                      C.byref(mean), C.byref(d), C.byref(u), _ptr(ws), ws.numel(), _stream()))
    return mean.value, d.value, u.value


def planted_recall(mask_bits: torch.Tensor, planted: torch.Tensor, heads_per_plane: int = 1, S: int = 64) -> float:
    """planted_recall (metrics.cpp:178-199): mask planes int32 [B, planes, N, W] against
    planted block lists int32 [B, H, N, m] (-1 = unused slot)."""
    if planted.dim() == 3:
        planted = planted.unsqueeze(0)
    if mask_bits.dim() == 3:
        mask_bits = mask_bits.unsqueeze(0)
    B, H, N, m = planted.shape
    if mask_bits.shape[1] * heads_per_plane != H:
        raise ValueError("planted_recall: planted must hold one list set per head")
    p = _metric_params(B, H, N * S, 64, S)
    ws = _scratch(lib().us_metrics_workspace_bytes(C.byref(p)), planted.device)
    out = C.c_double(0.0)
    _raise(lib().us_planted_recall(C.byref(p), _ptr(mask_bits.contiguous()), heads_per_plane,
                                   _ptr(planted.to(torch.int32).contiguous()), m, C.byref(out), _ptr(ws), ws.numel(),
                                   _stream()))
    return out.value
