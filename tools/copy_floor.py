"""Pinned-host copy floor of one C3 step: 1.61 GB H2D and 1.07 GB D2H, each alone and both
concurrently on two streams (bench.py e2e reports the concurrent figure as copy_floor_ms).

    python tools/copy_floor.py
"""
import torch, time
n_in, n_out = 1610612736, 1073741824
h_in = torch.empty(n_in, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n_out, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n_in, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d_in.copy_(h_in, non_blocking=True); h_out.copy_(d_out, non_blocking=True)
torch.cuda.synchronize()
def t(fn, reps=5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
h2d = t(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_out, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
bb = t(both)
print(f"H2D 1.61 GB: {h2d:.2f} ms ({n_in/h2d/1e6:.1f} GB/s)  D2H 1.07 GB: {d2h:.2f} ms ({n_out/d2h/1e6:.1f} GB/s)  both concurrently: {bb:.2f} ms")
