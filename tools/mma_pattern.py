"""tcgen05 step-pattern probe: cycles per iteration of the MMA sequences one attention
step issues (csrc/selftest.cu us_selftest_mma_pattern), 148 CTAs, one per SM."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
L = us.api.calib_lib()
L.us_selftest_mma_pattern.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
out = torch.zeros(148, dtype=torch.int64, device="cuda")
names = {0: "transposed: 8 SS N64 K-major -> acc0, 8 SS N64 MN-major -> acc1",
         1: "pattern 0, one accumulator",
         2: "16 SS N64 K-major, one accumulator",
         3: "16 SS N64 K-major, alternating accumulators",
         4: "current: 8 TS N64 + 4 SS N128 (B MN-major)",
         5: "FA4: 8 SS N128 + 8 TS N128",
         6: "transposed, A of the MN half from two 16 KB-apart tiles"}
ideal = {0: 16 * 32, 1: 16 * 32, 2: 16 * 32, 3: 16 * 32, 4: 8 * 32 + 4 * 64, 5: 16 * 64, 6: 16 * 32}
for p in range(7):
    iters = 2000
    L.us_selftest_mma_pattern(iters, p, 148, C.c_void_p(out.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    cyc = out.float().mean().item() / iters
    print(f"pattern {p}: {cyc:7.1f} cycles/iter (ideal {ideal[p]}) {ideal[p]/cyc*100:5.1f}%  {names[p]}")
