"""Cycles for the attention exponential phase (64 columns/thread) in isolation,
by ingredient (mode bits: 1 bf16 pack, 2 row-sum FADD2, 4 row max, 8 cubic share)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
L = us.api.calib_lib()
L.us_selftest_softmax_probe.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for threads in (128, 256):
    for mode in (0, 1, 2, 4, 7, 15):
        out = torch.zeros(148, dtype=torch.int64, device="cuda")
        sink = torch.zeros(148 * threads, dtype=torch.int32, device="cuda")
        iters = 500
        L.us_selftest_softmax_probe(iters, mode, 148, threads, C.c_void_p(sink.data_ptr()), C.c_void_p(out.data_ptr()), st)
        torch.cuda.synchronize()
        cyc = out.float().mean().item() / iters
        print(f"warps/SMSP={threads // 128} mode={mode:2d} (pack={mode & 1} sum={(mode >> 1) & 1} max={(mode >> 2) & 1} poly={(mode >> 3) & 1}): "
              f"{cyc:7.1f} cycles per step ({cyc / (threads // 128):6.1f} per warp-step)")
