"""Where does an M = 64 tcgen05 accumulator land in TMEM, and can its address take a lane
offset? (calibration build: us_selftest_m64_layout)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_14082_b200 as us
lib = us.api.calib_lib()
lib.us_selftest_m64_layout.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
g = torch.Generator().manual_seed(1)
A = torch.randn(128, 128, generator=g).to(torch.bfloat16).cuda()
B = torch.randn(64, 128, generator=g).to(torch.bfloat16).cuda()
ref = (A[:64].float() @ B.float().T)  # [64 rows][64 cols]
for off in (0, 16, 32, 64):
    D = torch.zeros(128, 64, device="cuda")
    st = lib.us_selftest_m64_layout(A.data_ptr(), B.data_ptr(), off, 0, D.data_ptr(), None)
    try:
        torch.cuda.synchronize()
    except Exception as e:
        print(f"lane_off {off}: FAULT {e}"); break
    where = []
    for lane in range(128):
        d = D[lane]
        if (d == 12345.0).all():
            where.append("-")
            continue
        err = (ref - d[None, :]).abs().max(dim=1).values
        r = int(err.argmin())
        where.append(str(r) if err[r] < 1e-2 * ref.abs().max() else "?")
    print(f"lane_off {off} (status {st}):")
    for q in range(4):
        print("   lanes %3d-%3d: %s" % (32 * q, 32 * q + 31, " ".join(where[32 * q:32 * q + 32])))

# TS mode: A rows 0-63 at lane offset 0, rows 64-127 at lane offset 16; two MMAs
ref2 = A.float() @ B.float().T  # [128][64]
D = torch.zeros(128, 64, device="cuda")
lib.us_selftest_m64_layout(A.data_ptr(), B.data_ptr(), 0, 1, D.data_ptr(), None)
torch.cuda.synchronize()
where = []
for lane in range(128):
    d = D[lane]
    err = (ref2 - d[None, :]).abs().max(dim=1).values
    r = int(err.argmin())
    where.append(str(r) if err[r] < 1e-2 * ref2.abs().max() else "?")
print("TS, A/D offsets 0 and 16:")
for q in range(4):
    print("   lanes %3d-%3d: %s" % (32 * q, 32 * q + 31, " ".join(where[32 * q:32 * q + 32])))

# 16x32bx2.x32 (split 32) read of the lane-offset-0 / -16 accumulators after the TS pair
for lo in (0, 1):
    D = torch.zeros(128, 64, device="cuda")
    lib.us_selftest_m64_layout(A.data_ptr(), B.data_ptr(), 0, 2 + lo, D.data_ptr(), None)
    torch.cuda.synchronize()
    ok = True
    for w in range(4):
        for t in range(32):
            arow = (64 if lo else 0) + 16 * w + (t & 15)     # row the thread should see
            c0 = 32 * (t >> 4)                               # and its column half
            want = ref2[arow, c0:c0 + 32]
            got = D[32 * w + t, :32]
            if (got - want).abs().max() > 1e-2 * ref2.abs().max():
                ok = False
    print(f"16x32bx2 read at lane offset {16 * lo}: thread t of warp q sees row 16q + (t & 15), columns "
          f"32 * (t >> 4) + [0, 32): {'OK' if ok else 'MISMATCH'}")
