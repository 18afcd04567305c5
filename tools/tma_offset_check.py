import ctypes as C, numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
from paper_1502_03409_b200 import lcae
lib = lcae.devlib()
lib.lcae_dev_tma_offset_selftest.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
rows, cols = 100, 128
src = torch.arange(rows * cols, dtype=torch.float32).reshape(rows, cols).to(torch.bfloat16).cuda()
s = src.float().cpu().numpy()
def expected(box, r0, c0, dst):
    out = np.zeros((64, 64), np.float32)
    for i in range(box):
        rr = dst + i
        for c in range(64):
            ch = (c // 8) ^ (rr % 8)
            out[rr, ch * 8 + c % 8] = s[r0 + i, c0 + c] if r0 + i < rows else 0
    return out
ok = True
for box in (1, 2, 4, 8, 16, 32):
    for dst in (0, 1, 3, 5, 8, 13, 27):
        if dst + box > 64: continue
        dump = torch.zeros(64 * 128, dtype=torch.uint8, device='cuda')
        st = lib.lcae_dev_tma_offset_selftest(src.data_ptr(), rows, cols, box, 7, 64, dst, dump.data_ptr())
        got = dump.cpu().view(torch.bfloat16).float().numpy().reshape(64, 64)
        exp = expected(box, 7, 64, dst)
        good = st == 0 and np.array_equal(got, exp)
        # alternative hypothesis: swizzle relative to the box start
        alt = np.zeros((64, 64), np.float32)
        for i in range(box):
            for c in range(64):
                ch = (c // 8) ^ (i % 8)
                alt[dst + i, ch * 8 + c % 8] = s[7 + i, 64 + c]
        print(f"box={box:2d} dst_row={dst:2d} status={st} absolute_swizzle={good} relative_swizzle={np.array_equal(got, alt)}")
        ok &= good
print("ALL_OK" if ok else "MISMATCH")
