"""Builds the sm_100a shared libraries in-tree:
  paper_2512_14082_b200/_build/libunisparse_b200.so        the product (the hot path + the C ABI)
  paper_2512_14082_b200/_build/libunisparse_b200_calib.so  calibration build (-DUS_CALIBRATION):
      the product plus the measured-slower attention variants (attention2.cu, the one-tile
      attention.cu instantiation, the key-major attention_kt.cu, the decoupled-softmax
      attention_tp.cu) and the tcgen05 / TMEM / MUFU probes (selftest.cu) — for tests/tools
      that select them, never the default path.

nvcc cross-compiles without a GPU; the .so travels to the GPU box with the
repo snapshot (git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_build")
LIB = os.path.join(OUT_DIR, "libunisparse_b200.so")
SOURCES = ["api.cu", "compress.cu", "proxy.cu", "select.cu", "attention.cu", "attention64.cu", "lastblock.cu", "io.cu", "metrics.cu"]
CALIB_SOURCES = SOURCES + ["attention2.cu", "attention_kt.cu", "attention_tp.cu", "selftest.cu"]
CALIB_LIB = os.path.join(OUT_DIR, "libunisparse_b200_calib.so")
NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", "-ccbin", "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def _build_lib(sources, obj_dir, lib, defines, headers, force, verbose):
    os.makedirs(obj_dir, exist_ok=True)
    objs, jobs = [], []
    for src in sources:
        s = os.path.join(CSRC, src)
        o = os.path.join(obj_dir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or not _newer(o, [s] + headers):
            jobs.append([NVCC, *ARCH, *FLAGS, *defines, "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return r

    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    if force or jobs or not _newer(lib, objs):
        run([NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lrt"])


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp"))]
    headers.append(os.path.join(os.path.dirname(PKG), "include", "us_api.h"))
    _build_lib(SOURCES, OUT_DIR, LIB, [], headers, force, verbose)
    _build_lib(CALIB_SOURCES, os.path.join(OUT_DIR, "calib"), CALIB_LIB, ["-DUS_CALIBRATION"], headers, force,
               verbose)
    build_wrapper_test(force)
    return LIB


WRAPPER_SRC = os.path.join(os.path.dirname(PKG), "tests", "cpp", "wrapper_test.cpp")
WRAPPER_BIN = os.path.join(OUT_DIR, "wrapper_test")


def build_wrapper_test(force: bool = False) -> str:
    """C++ test of the header-only reference-API mirror (include/unisparse_b200.hpp),
    linked against the in-tree library (rpath $ORIGIN)."""
    inc = os.path.join(os.path.dirname(PKG), "include")
    deps = [WRAPPER_SRC, LIB, os.path.join(inc, "unisparse_b200.hpp"), os.path.join(inc, "us_api.h")]
    if not force and _newer(WRAPPER_BIN, deps):
        return WRAPPER_BIN
    cuda = os.path.dirname(os.path.dirname(os.path.realpath(NVCC)))
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [cxx, "-O2", "-std=c++17", "-Wall", f"-I{inc}", f"-I{cuda}/include", WRAPPER_SRC, "-o", WRAPPER_BIN,
           f"-L{OUT_DIR}", "-lunisparse_b200", f"-L{cuda}/lib64", "-lcudart", "-Wl,-rpath,$ORIGIN",
           f"-Wl,-rpath,{cuda}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"g++ failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return WRAPPER_BIN


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
