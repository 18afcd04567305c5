"""Shared test helpers (no method arithmetic here)."""
import numpy as np

from paper_1502_03409_b200.inputs import LayerShape


def geo_of(shape: LayerShape) -> dict:
    return dict(img_h=shape.img_h, img_w=shape.img_w, img_c=shape.img_c, rf_h=shape.rf_h,
                rf_w=shape.rf_w, stride=shape.stride, pool_group=shape.pool_group,
                lam=shape.lam, eps=shape.eps)


def tiny_shape(g=1, k=4, m=3, C=1, **kw) -> LayerShape:
    """8x8xC image, rf 4, stride 2 -> 3x3 = 9 fields (SURVEY.md §8(c) FD geometry)."""
    return LayerShape("tiny", 8, 8, C, 4, 4, 2, k, g, m, **kw)


def normwise(a, ref):
    """R10: ||a - ref||_inf / ||ref||_inf (absolute if ref == 0)."""
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.abs(ref).max() if ref.size else 0.0
    num = np.abs(a - ref).max() if ref.size else 0.0
    return num / den if den > 0 else num


def rng_params(shape, seed=0, scale_b=0.0, alpha=None):
    """Random (not necessarily unit-norm) parameters for gradient checks."""
    rng = np.random.default_rng(seed)
    F, k, n = shape.fields, shape.filters, shape.n
    W = rng.standard_normal((F, k, n)) / np.sqrt(n)
    a = rng.uniform(0.5, 1.5, size=F) if alpha is None else np.full(F, alpha)
    b = scale_b * rng.standard_normal((F, n))
    return W, a, b
