"""Times dense (P=1) attention through the library at a given shape (calibration)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
from paper_2512_14082_b200 import workloads
L, H, H_kv = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
Q, K, V = workloads.planted_blocks(L, H, H_kv, 128, 64, seed=7, gain=8.0)
eng = us.Engine(Q, K, V, us.CompressionConfig(P=0.95))
for _ in range(2): eng.run(dense=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); n = 5
for _ in range(n): eng.run(dense=True)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / n
N = L // 64; fl = H * N * (N + 1) / 2 * 4 * 64 * 64 * 128
print(f"{os.environ.get('US_LIB_PATH_OVERRIDE','main')}: L={L} H={H} dense {ms:.3f} ms  {fl/ms/1e9:.1f} TFLOP/s")
