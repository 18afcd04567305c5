"""Oracle self-checks that do not reuse its own formulas.

1. Central finite differences of the layer objective on every coordinate of W, alpha, b and x
   (||a - fd||_inf / max(1, ||a||_inf) <= 1e-6, h = 1e-6).
2. A dense masked-matrix formulation of the whole layer (every field's weights scattered into an
   image-sized matrix, windows as 0/1 selection matrices) differentiated by torch autograd in
   float64 - no per-field slicing code, no hand-derived gradient.
"""
import numpy as np
import pytest
import torch

from oracle import lcae_oracle as O
from tests.helpers import geo_of, tiny_shape, rng_params


def _layer_J(W, a, b, X, geo):
    return O.layer_gradients(W, a, b, X, geo)["J"]


def _fd(fun, v, h=1e-6):
    g = np.zeros(v.size)
    flat = v.reshape(-1)
    for t in range(flat.size):
        old = flat[t]
        flat[t] = old + h
        fp = fun()
        flat[t] = old - h
        fm = fun()
        flat[t] = old
        g[t] = (fp - fm) / (2 * h)
    return g.reshape(v.shape)


@pytest.mark.parametrize("g", [1, 2])
def test_finite_differences_every_coordinate(g):
    shape = tiny_shape(g=g, k=4, m=3)
    geo = geo_of(shape)
    W, a, b = rng_params(shape, seed=11 + g, scale_b=0.3)
    X = np.random.default_rng(5).standard_normal((shape.batch, 8, 8, 1))
    o = O.layer_gradients(W, a, b, X, geo)
    f = lambda: _layer_J(W, a, b, X, geo)
    for name, ana, v in (("dW", o["dW"], W), ("dalpha", o["dalpha"], a), ("db", o["db"], b), ("dX", o["dX"], X)):
        fd = _fd(f, v)
        err = np.abs(ana - fd).max() / max(1.0, np.abs(ana).max())
        assert err <= 1e-6, (name, err)


def _dense_layer_torch(W, a, b, X, shape):
    """Dense masked formulation: W_dense_f = W_f S_f, S_f the 0/1 window selector of field f."""
    m, H, Wd, C = X.shape
    M = H * Wd * C
    F, k, n = W.shape
    g = shape.pool_group
    S = torch.zeros((F, n, M), dtype=torch.float64)
    pix = np.arange(M).reshape(H, Wd, C)
    for f in range(F):
        r, c = divmod(f, shape.grid_c)
        idx = pix[r * shape.stride:r * shape.stride + shape.rf_h, c * shape.stride:c * shape.stride + shape.rf_w, :].reshape(-1)
        S[f, np.arange(n), idx] = 1.0
    Wt = torch.tensor(W, requires_grad=True)
    at = torch.tensor(a, requires_grad=True)
    bt = torch.tensor(b, requires_grad=True)
    Xt = torch.tensor(X.reshape(m, M), requires_grad=True)
    Wdense = torch.einsum("fkn,fnM->fkM", Wt, S)              # k x M per field, zero outside window
    Hc = at[:, None, None] * torch.einsum("fkM,iM->fik", Wdense, Xt)     # (F, m, k)
    s = torch.sqrt(shape.eps + (Hc.reshape(F, m, k // g, g) ** 2).sum(-1))
    R = torch.einsum("fik,fkM->fiM", Hc, Wdense)               # decoder back into image space
    Xf = torch.einsum("fnM,iM->fin", S, Xt)                    # patch of each field
    Rf = torch.einsum("fiM,fnM->fin", R, S) + bt[:, None, :]
    J = ((Rf - Xf) ** 2).sum() + shape.lam * s.sum()
    J.backward()
    return (J.item(), s.detach().numpy(), Wt.grad.numpy(), at.grad.numpy(), bt.grad.numpy(),
            Xt.grad.numpy().reshape(X.shape))


@pytest.mark.parametrize("cfg", ["tiny1", "tiny2", "c1", "rect3"])
def test_dense_masked_equivalence(cfg):
    from paper_1502_03409_b200.inputs import CONFIGS, LayerShape, make_images, make_params
    if cfg == "c1":
        shape = CONFIGS["c1"]
    elif cfg == "rect3":
        shape = LayerShape("rect3", 10, 14, 3, 4, 6, 2, 6, 3, 2)     # non-square, rf_h != rf_w, C=3
    else:
        shape = tiny_shape(g=int(cfg[-1]), k=4, m=3)
    geo = geo_of(shape)
    W, a, b = rng_params(shape, seed=3, scale_b=0.2)
    X = make_images(shape, seed=9).astype(np.float64)
    o = O.layer_gradients(W, a, b, X, geo)
    J, s, dW, da, db, dX = _dense_layer_torch(W, a, b, X, shape)
    assert o["J"] == pytest.approx(J, rel=1e-12)
    p = o["p"].reshape(shape.batch, shape.fields, -1).transpose(1, 0, 2)
    np.testing.assert_allclose(p, s, rtol=1e-12)
    np.testing.assert_allclose(o["dW"], dW, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(o["dalpha"], da, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(o["db"], db, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(o["dX"], dX, rtol=1e-11, atol=1e-11)
