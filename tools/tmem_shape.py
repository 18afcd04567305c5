"""Dev tool: print the thread <- (TMEM lane, column) map of tcgen05.ld.16x256b.x2 (lcae_dev_tmem_shape_selftest)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_03409_b200 import lcae  # noqa: E402

out = np.zeros((4, 2, 32, 8), dtype=np.uint32)
lcae.devlib().lcae_dev_tmem_shape_selftest.argtypes = [C.c_void_p]
lcae.dev_check(lcae.devlib().lcae_dev_tmem_shape_selftest(out.ctypes.data))
for w in (0, 1):
    for h in (0, 1):
        for t in (0, 1, 2, 3, 4, 5, 31):
            print(w, h, t, [(int(v) >> 8, int(v) & 255) for v in out[w, h, t]])
