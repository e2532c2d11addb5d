"""tcgen05 issue rate at M = 64 vs M = 128 (148 CTAs, back-to-back K = 16 bf16 MMAs):
cycles per MMA for TS / SS, N = 64 / 128, and two M = 64 accumulators at lane offsets 0 / 16."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
L = us.api.calib_lib()
L.us_selftest_mma_rate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
out = torch.zeros(148, dtype=torch.int64, device="cuda")
for N in (64, 128):
    for mode, name in ((1, "M128 TS"), (0, "M128 SS"), (3, "M64 TS"), (2, "M64 SS"), (7, "M64 TS x2 lanes"), (6, "M64 SS x2 lanes")):
        iters, per = 2000, 8
        L.us_selftest_mma_rate(iters, N, mode, per, 148, C.c_void_p(out.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        cyc = out.float().mean().item() / (iters * per)
        print(f"N={N:3d} {name:16s}: {cyc:6.1f} cycles/MMA (M=128 floor {128 * N / 256:.0f})")
