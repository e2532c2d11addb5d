"""tcgen05 throughput probe: cycles per MMA for M=128,K=16 bf16 at several N / operand modes."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
L = us.api.calib_lib()
L.us_selftest_mma_rate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
out = torch.zeros(148, dtype=torch.int64, device="cuda")
for N in (64, 128, 256):
    for a_tmem in (1, 0):
        iters, per = 2000, 8
        L.us_selftest_mma_rate(iters, N, a_tmem, per, 148, C.c_void_p(out.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        cyc = out.float().mean().item() / (iters * per)
        ideal = 128 * N / 256
        print(f"N={N:3d} A={'tmem' if a_tmem else 'smem'}: {cyc:6.1f} cycles/MMA (ideal {ideal:.0f}) -> {ideal/cyc*100:5.1f}%")
