"""Local contrast normalisation between layers — TEST INFRASTRUCTURE ONLY (see lcae_oracle.py header).

PAPER.md:95 ("local contrast normalization (LCN) is applied prior to continuing onto the next layer") names
LCN without a formula; SPEC.md:215-223 / :242-243 fix the reading used here (R15):
    v = x - mean_w(x)                  uniform window w x w per channel, zero padding, count-correct divisor
    y = v / max(floor, sqrt(mean_w(v^2)))
written out as the plain definition, one window at a time, in float64.
"""
import numpy as np


def lcn(x, window=9, floor=1e-4):
    """x [m][H][W][C] -> y, same shape."""
    x = np.asarray(x, dtype=np.float64)
    m, H, W, C = x.shape
    if window > H or window > W or window % 2 == 0:
        raise ValueError("LCN window must be odd and no larger than the map")
    r = window // 2

    def local_mean(a):
        out = np.zeros_like(a)
        for yy in range(H):
            y0, y1 = max(0, yy - r), min(H, yy + r + 1)
            for xx in range(W):
                x0, x1 = max(0, xx - r), min(W, xx + r + 1)
                win = a[:, y0:y1, x0:x1, :]
                out[:, yy, xx, :] = win.sum(axis=(1, 2)) / ((y1 - y0) * (x1 - x0))
        return out

    v = x - local_mean(x)
    sd = np.sqrt(local_mean(v * v))
    return v / np.maximum(floor, sd)
