"""Momentum variant: several steps with mu = 0.9 through the C ABI against the fp64
oracle carrying its velocity (v = mu v - lr g, theta += v, then the unit-row projection of
PAPER.md:89). The first step from v = 0 equals plain SGD, so only steps 2+ exercise the velocity buffers;
compared as the accumulated update theta_t - theta_0 (normwise, R10)."""
import numpy as np
import pytest

from oracle import lcae_oracle as O
from paper_1502_03409_b200.inputs import CONFIGS, LayerShape, make_images, make_params
from tests.helpers import geo_of, normwise

pytestmark = pytest.mark.gpu

SHAPES = {
    "c1": CONFIGS["c1"],
    "cluster2": LayerShape("cluster2", 20, 20, 3, 8, 8, 4, 32, 2, 200),
}


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16", 2e-2)])
@pytest.mark.parametrize("name", list(SHAPES))
def test_momentum_steps_match_oracle(name, precision, tol):
    import torch
    from paper_1502_03409_b200 import lcae
    shape = SHAPES[name].replace(momentum=0.9)
    if precision == "fp32" and shape.batch > 128:
        pytest.skip("fp32 path covered on c1")
    W0, a0, b0 = make_params(shape, seed=0)
    X = make_images(shape, seed=1)
    nsteps = 3
    # oracle, fp64, velocity carried
    W, a, b, vel = W0.astype(np.float64), a0.astype(np.float64), b0.astype(np.float64), None
    for t in range(nsteps):
        o = O.step(W, a, b, X.astype(np.float64), geo_of(shape), lr=shape.lr, momentum=shape.momentum,
                   velocity=vel, alpha_min=shape.alpha_min, step_index=t)
        W, a, b, vel = o["W_new"], o["alpha_new"], o["b_new"], o["velocity"]
    # GPU
    prec = lcae.FP32 if precision == "fp32" else lcae.BF16
    L = lcae.Layer(lcae.make_config(shape, precision=prec))
    try:
        L.set_params(W0, a0, b0)
        xd = torch.from_numpy(np.ascontiguousarray(X, np.float32)).cuda()
        for _ in range(nsteps):
            L.step(xd, None)
        Wg = np.zeros_like(W0)
        ag = np.zeros_like(a0)
        bg = np.zeros_like(b0)
        L.get_params(Wg, ag, bg)
    finally:
        L.close()
    assert normwise(Wg - W0, W - W0) <= tol
    assert normwise(ag - a0, a - a0) <= tol
    assert normwise(bg - b0, b - b0) <= tol
    assert np.abs(np.linalg.norm(Wg, axis=-1) - 1).max() <= 1e-5
