"""Dev tool: cycles per tcgen05.mma (M=128, K=16, SS operands) for the step kernel's shapes.
mode -1: warp-uniform loop + elect.sync; 0: single-lane loop; 1: single-lane loop, commit+wait every 4."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_03409_b200 import lcae  # noqa: E402

f = lcae.devlib().lcae_dev_mma_rate
f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
for N in (64, 128, 256):
    for a_mn, b_mn in ((0, 0), (1, 0), (0, 1)):
        if N == 256 and b_mn:
            continue
        for mode in (-1, 0, 1):
            v = C.c_double()
            lcae.check(f(N, a_mn, b_mn, 512, mode, C.byref(v)))
            print(f"N={N:3d} A_mn={a_mn} B_mn={b_mn} mode={mode:2d}: {v.value:7.1f} cyc/MMA (floor {128 * N / 256:.0f})")
