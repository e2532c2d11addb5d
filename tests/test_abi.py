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
    p.L, p.d_k = 1024, 96
    assert lib.us_check_params(C.byref(p), b"select_blocks", 1) == 2  # US_ERR_UNSUPPORTED
    p.d_k = 128
    assert lib.us_check_params(C.byref(p), b"select_blocks", 1) == 0


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
