"""TMEM load throughput: 128 threads x 64 fp32 columns per iteration, alone and under MMA load."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
L = us.api.calib_lib()
L.us_selftest_tmem_ld.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
out = torch.zeros(148, dtype=torch.int64, device="cuda")
sink = torch.zeros(148 * 128, dtype=torch.float32, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for mma_n in (0, 64, 128, 256):
    iters = 4000
    L.us_selftest_tmem_ld(iters, mma_n, 148, C.c_void_p(sink.data_ptr()), C.c_void_p(out.data_ptr()), st)
    torch.cuda.synchronize()
    cyc = out.float().mean().item() / iters
    print(f"concurrent MMA N={mma_n:3d}: {cyc:7.1f} cycles per 32 KB TMEM load -> {32768 / cyc:6.1f} B/cycle")
