"""exp2 throughput probe: MUFU ex2.approx vs the FMA-pipe cubic vs plain FFMA2, per SM."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
L = us.api.calib_lib()
L.us_selftest_ex2_rate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for threads in (128, 256, 512):
    out = torch.zeros(148, dtype=torch.int64, device="cuda")
    sink = torch.zeros(148 * threads, dtype=torch.float32, device="cuda")
    for mode, name in ((0, "MUFU ex2"), (1, "poly ex2"), (2, "FFMA2"), (3, "ex2 f16x2")):
        iters = 2000
        L.us_selftest_ex2_rate(iters, mode, 148, threads, C.c_void_p(sink.data_ptr()), C.c_void_p(out.data_ptr()), st)
        torch.cuda.synchronize()
        cyc = out.float().mean().item()
        per_sm = threads * 32 * iters / cyc
        print(f"threads/SM={threads:4d} {name:9s}: {per_sm:6.1f} results/cycle/SM")
