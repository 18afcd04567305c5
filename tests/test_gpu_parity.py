"""GPU (through the C ABI) vs fp64 oracle, element by element, on identical seeded inputs.

Tolerances (BASELINE.json north_star; R10, normwise ||gpu - oracle||_inf / ||oracle||_inf):
fp32 path <= 1e-5, bf16 tensor-core path <= 2e-2, per tensor: loss, pooled code, dW, dalpha, db, dX and the
parameter update (W' - W, alpha' - alpha, b' - b).  Row norms after the update: |‖W_j‖ - 1| <= 1e-6 (fp32 master).
"""
import numpy as np
import pytest

from paper_1502_03409_b200.inputs import CONFIGS, LayerShape, make_images, make_params
from tests.gpu_harness import gpu_step, oracle_step
from tests.helpers import normwise

pytestmark = pytest.mark.gpu

TOL = {0: 1e-5, 1: 2e-2}

# single-step parity at SPEC.md:141's lr = 1e-3 (the configs' bench lr is 1e-3 / m, R19): the update
# is compared as theta' - theta, and at lr / m the fp32 rounding of theta' itself is ~1e-5 of that difference
SHAPES = {
    "c1": CONFIGS["c1"].replace(lr=1e-3),
    "c2": CONFIGS["c2"].replace(lr=1e-3),
    # ragged: n = 5*7*2 = 70 (not a multiple of 16/64), k = 24, g = 4, odd batch, non-square image
    "ragged": LayerShape("ragged", 21, 25, 2, 5, 7, 2, 24, 4, 37),
    "worked": LayerShape("worked", 2, 1, 1, 2, 1, 1, 2, 1, 1, eps=0.0),
}


def _compare(shape, precision, out, o, W, a, b):
    tol = TOL[precision]
    errs = {}
    errs["J"] = abs(out["J"] - o["J"]) / abs(o["J"])
    errs["J_rec"] = abs(out["J_rec"] - o["J_rec"]) / abs(o["J_rec"]) if o["J_rec"] else abs(out["J_rec"])
    errs["J_sparse"] = abs(out["J_sparse"] - o["J_sparse"]) / abs(o["J_sparse"])
    if "p" in out:
        errs["p"] = normwise(out["p"], o["p"])
        errs["J_fwd"] = abs(out["J_fwd"] - o["J"]) / abs(o["J"])
    for key in ("dW", "dalpha", "db", "dX"):
        if key in out:
            errs[key] = normwise(out[key], o[key])
    errs["dW_update"] = normwise(out["W_new"].astype(np.float64) - W, o["W_new"] - W)
    errs["alpha_update"] = normwise(out["alpha_new"].astype(np.float64) - a, o["alpha_new"] - a)
    errs["b_update"] = normwise(out["b_new"].astype(np.float64) - b, o["b_new"] - b)
    bad = {k: v for k, v in errs.items() if not (v <= tol)}
    assert not bad, (shape.name, precision, bad, errs)
    norms = np.linalg.norm(out["W_new"].astype(np.float64), axis=-1)
    assert np.abs(norms - 1).max() <= 1e-6
    return errs


@pytest.mark.parametrize("name", ["worked", "c1", "ragged", "c2"])
def test_fp32_parity(name):
    shape = SHAPES[name]
    if name == "worked":   # SPEC.md:97 instance through the whole GPU pipeline
        W = np.eye(2, dtype=np.float32)[None]
        a = np.array([2.0], np.float32)
        b = np.zeros((1, 2), np.float32)
        X = np.array([1.0, -1.0], np.float32).reshape(1, 2, 1, 1)
    else:
        W, a, b = make_params(shape, seed=0)
        X = make_images(shape, seed=1)
        b = (0.05 * np.random.default_rng(3).standard_normal(b.shape)).astype(np.float32)
    out = gpu_step(shape, 0, W, a, b, X)
    o = oracle_step(shape, W, a, b, X)
    _compare(shape, 0, out, o, W.astype(np.float64), a.astype(np.float64), b.astype(np.float64))
    if name == "worked":
        assert out["J"] == pytest.approx(2.4, rel=1e-6)
        np.testing.assert_allclose(out["dW"][0], [[8.2, -8.2], [-8.2, 8.2]], rtol=1e-6)
    assert out["steps"] == 1 and out["reinit"] == 0
    assert out["launches"] > 0


SHAPES_BF16 = {
    "worked": SHAPES["worked"],
    "c1": SHAPES["c1"],
    "ragged": SHAPES["ragged"],
    "c2": SHAPES["c2"],
    # two-CTA cluster (m > 128, ragged second slice), pooling g = 2, n = 8*8*3 = 192
    "cluster2": LayerShape("cluster2", 20, 20, 3, 8, 8, 4, 32, 2, 200),
    # paper layer-1-like field shape (k = 128, g = 1) on a small image, two CTAs
    "c3tiny": LayerShape("c3tiny", 22, 22, 3, 18, 18, 2, 128, 1, 256),
}


@pytest.mark.parametrize("name", list(SHAPES_BF16))
def test_bf16_parity(name):
    shape = SHAPES_BF16[name]
    if name == "worked":
        W = np.eye(2, dtype=np.float32)[None]
        a = np.array([2.0], np.float32)
        b = np.zeros((1, 2), np.float32)
        X = np.array([1.0, -1.0], np.float32).reshape(1, 2, 1, 1)
    else:
        W, a, b = make_params(shape, seed=0)
        X = make_images(shape, seed=1)
        b = (0.05 * np.random.default_rng(3).standard_normal(b.shape)).astype(np.float32)
    out = gpu_step(shape, 1, W, a, b, X)
    o = oracle_step(shape, W, a, b, X)
    errs = _compare(shape, 1, out, o, W.astype(np.float64), a.astype(np.float64), b.astype(np.float64))
    print(name, {k_: f"{v:.1e}" for k_, v in errs.items()})
    assert out["steps"] == 1 and out["reinit"] == 0


@pytest.mark.parametrize("name", ["c1", "ragged", "cluster2", "c3tiny"])
def test_bf16_lean_variant_parity(name):
    """The production (lean) step kernel variant -- no kept gradients, no velocity, no debug flags -- against the
    oracle: loss and the W / alpha / b updates (the keep_grads tests above run the full variant)."""
    shape = SHAPES_BF16[name]
    W, a, b = make_params(shape, seed=0)
    X = make_images(shape, seed=1)
    b = (0.05 * np.random.default_rng(3).standard_normal(b.shape)).astype(np.float32)
    out = gpu_step(shape, 1, W, a, b, X, keep_grads=False, forward_first=False)
    o = oracle_step(shape, W, a, b, X)
    _compare(shape, 1, out, o, W, a, b)


def test_fp32_paper_exact_layer1_field_shape():
    """SURVEY.md §8(d) c3' field shape (16 x 16 x 3 receptive field, stride 4, 4 x 4 x 24 = 384
    filters; PAPER.md:111 mini-batch 192) on a small image (3 x 3 fields): the fp32 path at north_star's 1e-5.
    (The fused bf16 kernel holds U and G in TMEM and takes k <= 128; in bf16 this shape runs on the general
    tcgen05 GEMM path, tests/test_gpu_gt.py.)"""
    shape = LayerShape("c3p-small", 24, 24, 3, 16, 16, 4, 384, 1, 192)
    W, a, b = make_params(shape, seed=0)
    X = make_images(shape, seed=1, bf16_round=False)
    b = (0.05 * np.random.default_rng(3).standard_normal(b.shape)).astype(np.float32)
    out = gpu_step(shape, 0, W, a, b, X)
    o = oracle_step(shape, W, a, b, X)
    _compare(shape, 0, out, o, W.astype(np.float64), a.astype(np.float64), b.astype(np.float64))
