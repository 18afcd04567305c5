"""Dev tool: per-role barrier-wait breakdown of the fused step kernel (lcae_dev_trace).
usage: python tools/trace_step.py [c3|c2] [steps]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1502_03409_b200 import lcae  # noqa: E402
from paper_1502_03409_b200.inputs import CONFIGS, make_images, make_params  # noqa: E402

NAMES = {0: "mma:wfull", 1: "mma:p0full", 2: "mma:tmem_free", 3: "mma:h_ready", 4: "mma:r_empty",
         5: "mma:dl_full(G)", 6: "mma:d_ready", 7: "mma:p2_empty", 8: "mma:dl_full(dW)", 9: "mma:xfull(dW)",
         10: "mma:TOTAL", 11: "epi:u_full", 12: "epi:r_full", 13: "epi:p1full", 14: "epi:dl_empty(E1)",
         16: "epi:g_full", 18: "epi:p2_rdx", 19: "epi:xfull", 20: "epi:dl_empty(E2)", 21: "epi:p2_dw",
         22: "epi:dsmem", 24: "xprod:TOTAL", 25: "wprod:TOTAL", 26: "epi:TOTAL", 27: "wprod:wempty",
         28: "xprod:p0_ok", 29: "xprod:p0empty", 30: "xprod:p1", 31: "xprod:xempty",
         32: "sec:E0", 33: "sec:E1 loop", 34: "sec:E1b", 35: "sec:E2a resid+delta", 36: "sec:E2b dX", 37: "sec:E2c3 SGD+stores", 38: "sec:field end", 39: "sec:E2b0 dX tmem load", 40: "sec:E2c0 dW wait+ld", 41: "sec:E2c1 exchange", 42: "sec:E2c2 staging", 43: "epi:r_full(j=0)", 44: "mma:p1full", 45: "epi:db_full"}

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mode = sys.argv[3] if len(sys.argv) > 3 else "step"
shape = CONFIGS[cfg_name]
lib = lcae.lib
lib.lcae_dev_trace.restype = C.c_int
lib.lcae_dev_trace.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16))
W, a, b = make_params(shape, seed=0)
L.set_params(W, a, b)
x = torch.from_numpy(make_images(shape, seed=1)).cuda()
pooled = torch.empty((shape.batch, shape.fields * (shape.filters // shape.pool_group)), device="cuda")


def run():
    if mode == "encode":
        L.encode(x, pooled, want_loss=False)
    else:
        L.step(x, None, want_loss=False)


for _ in range(2):
    run()
torch.cuda.synchronize()
lcae.check(lib.lcae_dev_trace(L.h, 1, None))
L.profile(True)
for _ in range(steps):
    run()
torch.cuda.synchronize()
ms, nl = L.profile_read()
out = (C.c_ulonglong * (64 + 256))()
lcae.check(lib.lcae_dev_trace(L.h, 0, out))
ctas = min(shape.fields * ((shape.batch + 127) // 128), 148 // ((shape.batch + 127) // 128) * ((shape.batch + 127) // 128))
per = lambda v: v / ctas / steps  # noqa: E731
tot = per(out[10])
print(f"{cfg_name}: kernel {ms / nl:.3f} ms/launch; per-CTA cycles per step (mma total {tot:.0f})")
for i in sorted(NAMES):
    if out[i]:
        print(f"  {NAMES[i]:20s} {per(out[i]):14.0f}  {100 * per(out[i]) / tot:6.1f}%")
print("  per epilogue warp (warp = 2 + w, TMEM quarter w % 4, column half w // 4): wait p2_full / wait r_full")
for w in range(8):
    print(f"    w{w} (warp {w + 2}, SMSP {(w + 2) % 4}): {100 * per(out[48 + w]) / tot:5.1f}%  {100 * per(out[56 + w]) / tot:5.1f}%")

# timeline of CTA 0's third field (traced variant): event times in us relative to the first R issue
tl = list(out[64:64 + 256])
if any(tl):
    clk = 1.965e3   # cycles per us at the maximum SM clock (approximate)
    t0 = min(v for v in tl[0:16] if v)
    f = lambda v: (v - t0) / clk if v else float("nan")  # noqa: E731
    print("pass 1 (us): j  W_ready  X_ready  R_issued  G_issued  R_seen(w2)  delta_done(w2)")
    for j in range(16):
        print(f"  {j:2d} {f(tl[80 + j]):8.2f} {f(tl[64 + j]):8.2f} {f(tl[j]):8.2f} {f(tl[16 + j]):8.2f} {f(tl[32 + j]):8.2f} "
              f"{f(tl[48 + j]):8.2f}")
    print("pass 2 (us): j  W_ready  d_reloaded  buf_free  X_ready  issued  seen(w2)  freed(w2)")
    for j in range(16):
        print(f"  {j:2d} {f(tl[176 + j]):8.2f} {f(tl[160 + j]):8.2f} {f(tl[192 + j]):8.2f} {f(tl[144 + j]):8.2f} "
              f"{f(tl[96 + j]):8.2f} {f(tl[112 + j]):8.2f} {f(tl[128 + j]):8.2f}")
    print("pass 1 delta_j done per epilogue warp (us; warp = 2 + w):")
    for jj in range(6):
        print(f"  j={4 + jj}: " + " ".join(f"{f(tl[208 + jj * 8 + w]):7.2f}" for w in range(8)))
