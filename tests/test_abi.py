"""The C ABI boundary (include/us_api.h) and the C++ reference-API mirror
(include/unisparse_b200.hpp), checked without compute calls on CPU and with
them on the GPU.
"""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2512_14082_b200", "_build", "libunisparse_b200.so")
WRAPPER = os.path.join(ROOT, "paper_2512_14082_b200", "_build", "wrapper_test")


def _declared_functions(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(us_[a-z_0-9]+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2512_14082_b200 import build
        build.build()
    return C.CDLL(LIB)


def test_library_exports_every_declared_symbol(lib):
    names = _declared_functions("us_api.h")
    assert len(names) >= 15, names
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        getattr(lib, n)  # resolvable through the loader


def test_library_has_sm100a_tcgen05_and_tma_code():
    """The product kernels are sm_100a SASS with tcgen05 MMAs, TMEM loads and TMA
    (B200_PROFILING.md mnemonics), not a legacy mma.sync path."""
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", LIB], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "LDTM", "UTMALDG"):
        assert mnem in sass, mnem
    assert "HMMA" not in sass.replace("UTCHMMA", "")


def test_check_params_reference_messages(lib):
    from paper_2512_14082_b200.api import UsParams
    lib.us_check_params.argtypes = [C.POINTER(UsParams), C.c_char_p, C.c_int32]
    lib.us_last_error.restype = C.c_char_p
    p = UsParams(1, 4, 4, 1000, 64, 64, 8, 8, 1, 0, 0, 0, 0.95, 0, 0, 0)
    assert lib.us_check_params(C.byref(p), b"select_blocks", 1) == 1
    assert lib.us_last_error().decode() == "select_blocks: L=1000 not divisible by S=64"
    p.L, p.d_k = 1024, 160
    assert lib.us_check_params(C.byref(p), b"select_blocks", 1) == 2  # US_ERR_UNSUPPORTED
    assert lib.us_last_error().decode() == "select_blocks: d_k=160 unsupported on the GPU path (at most 128)"
    p.d_k = 96  # any d_k <= 128: zero-padded to 128 in the workspace
    assert lib.us_check_params(C.byref(p), b"select_blocks", 1) == 0
    p.d_k = 128
    assert lib.us_check_params(C.byref(p), b"select_blocks", 1) == 0


def test_padded_dk_workspace_bytes(lib):
    """d_k outside {64, 128}: the workspace holds the inner call's workspace at the padded
    width plus the zero-padded copies of Q, K, V, O and the compressed rows."""
    from paper_2512_14082_b200.api import UsParams
    lib.us_workspace_bytes.argtypes = [C.POINTER(UsParams)]
    lib.us_workspace_bytes.restype = C.c_size_t
    p = UsParams(1, 4, 2, 1024, 32, 64, 8, 8, 1, 0, 0, 0, 0.95, 0, 0, 0)
    ws32 = lib.us_workspace_bytes(C.byref(p))
    p.d_k = 64
    ws64 = lib.us_workspace_bytes(C.byref(p))
    padded = 2 * 64 * 1024 * (4 + 2 + 2 + 4) + 4 * 64 * 128 * 4 * 2  # Q, K, V, O bf16 + Qc, Kc f32
    assert ws32 >= ws64 + padded


def test_attention_workspace_is_small_at_c3(lib):
    """The attention entry points' workspace (us_attention_workspace_bytes) holds only the
    error header and the sparse kernel's work-item table at C3 (32 / 8 heads, L = 128K,
    d = 128, c = 1): megabytes — the full pipeline layout at c = 1 would size the proxy
    buffers for the uncompressed length (hundreds of GB)."""
    from paper_2512_14082_b200.api import UsParams
    for f in (lib.us_workspace_bytes, lib.us_attention_workspace_bytes):
        f.argtypes = [C.POINTER(UsParams)]
        f.restype = C.c_size_t
    p = UsParams(1, 32, 8, 131072, 128, 64, 1, 1, 1, 0, 0, 0, 0.95, 0, 0, 0)
    N = 131072 // 64
    attn = lib.us_attention_workspace_bytes(C.byref(p))
    items = 4 * 8 * ((4 * N + 3) // 4) * 4 + 8 * 8 + 4 * 32 * N  # item table, sel_pairs, row counts
    assert items <= attn < items + 64 * 1024, attn
    assert lib.us_workspace_bytes(C.byref(p)) > 100 * attn
    p.dtype = 1  # f32 inputs: + bf16 copies of Q, K, V
    conv = 2 * (32 + 2 * 8) * 131072 * 128
    assert lib.us_attention_workspace_bytes(C.byref(p)) >= conv + items


def test_cpp_wrapper_cpu():
    if not os.path.exists(WRAPPER):
        from paper_2512_14082_b200 import build
        build.build()
    r = subprocess.run([WRAPPER, "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_wrapper_gpu():
    r = subprocess.run([WRAPPER, "gpu"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


def test_acceptance_criterion_7_flop_identities(lib):
    """acceptance.cpp criterion 7 through us_selection_flops (host arithmetic, no
    GPU): compressed_qk * c_q * c_k * c_h == 2 L^2 H d exactly, dense = 2x that,
    c_h = 2 halves the compressed scoring and aggregation terms (S = 64 here; the
    reference battery uses S = 128, every identity is S-independent)."""
    from paper_2512_14082_b200.api import UsParams
    lib.us_selection_flops.argtypes = [C.POINTER(UsParams), C.c_int32, C.c_int32, C.c_void_p]
    out = (C.c_uint64 * 6)()
    ok = True
    for L in (1024, 2048, 4096):
        for H in (2, 4, 8):
            for d in (64, 128):
                dense_qk = 2 * L * L * H * d
                for c_q in (1, 2, 4, 8, 16, 32, 64):
                    for c_k in (1, 4, 8, 64):
                        for c_h in (1, 2):
                            p = UsParams(1, H, H, L, d, 64, c_q, c_k, c_h, 0, 0, 0, 0.95, 0, 0, 0)
                            assert lib.us_selection_flops(C.byref(p), 0, 8, C.cast(out, C.c_void_p)) == 0
                            qk, dense = out[1], out[5]
                            ok &= qk * c_q * c_k * c_h == dense_qk and dense_qk % qk == 0
                            ok &= dense == 2 * dense_qk
                f = []
                for c_h in (1, 2):
                    p = UsParams(1, H, H, L, d, 64, 8, 8, c_h, 0, 0, 0, 0.95, 0, 0, 0)
                    lib.us_selection_flops(C.byref(p), 0, 8, C.cast(out, C.c_void_p))
                    f.append((out[1], out[2]))
                ok &= f[0][0] == 2 * f[1][0] and f[0][1] == 2 * f[1][1]
    assert ok
