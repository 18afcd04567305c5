"""Oracle closed forms and invariants (SURVEY.md §8(c) 'What pins each part')."""
import numpy as np
import pytest

from oracle import lcae_oracle as O
from paper_1502_03409_b200.inputs import CONFIGS, LayerShape, make_images, make_params
from tests.helpers import geo_of, tiny_shape, rng_params


def test_zero_weights_closed_form():
    shape = LayerShape("z", 12, 12, 2, 4, 4, 4, 6, 3, 3)
    geo = geo_of(shape)
    F, n = shape.fields, shape.n
    W = np.zeros((F, shape.filters, n))
    rng = np.random.default_rng(2)
    b = rng.standard_normal((F, n))
    a = np.full(F, 1.7)
    X = make_images(shape, seed=4).astype(np.float64)
    o = O.layer_gradients(W, a, b, X, geo)
    J = 0.0
    dX = np.zeros_like(X)
    for f in range(F):
        r, c = divmod(f, shape.grid_c)
        win = (slice(None), slice(r * 4, r * 4 + 4), slice(c * 4, c * 4 + 4), slice(None))
        xf = X[win].reshape(shape.batch, -1)
        J += ((b[f] - xf) ** 2).sum()
        dX[win] += (-2.0 * (b[f] - xf)).reshape(X[win].shape)
    J += shape.lam * shape.batch * F * (shape.filters // shape.pool_group) * np.sqrt(shape.eps)
    assert o["J"] == pytest.approx(J, rel=1e-13)
    assert np.all(o["dW"] == 0) and np.all(o["dalpha"] == 0)
    np.testing.assert_allclose(o["dX"], dX, atol=1e-13)


@pytest.mark.parametrize("g", [1, 2, 4])
def test_selection_weights_closed_form(g):
    """W = [I_k 0], b = 0: J = sum_i (alpha-1)^2 ||x_1:k||^2 + ||x_k+1:n||^2 + lam sum_G sqrt(eps + alpha^2 sum_G x_j^2)."""
    shape = LayerShape("sel", 16, 16, 3, 8, 8, 4, 8, g, 5)
    geo = geo_of(shape)
    F, k, n = shape.fields, shape.filters, shape.n
    W = np.zeros((F, k, n))
    W[:, np.arange(k), np.arange(k)] = 1.0
    a = np.linspace(0.6, 1.4, F)
    X = make_images(shape, seed=6).astype(np.float64)
    o = O.layer_gradients(W, a, np.zeros((F, n)), X, geo)
    J = 0.0
    for f in range(F):
        r, c = divmod(f, shape.grid_c)
        xf = X[:, r * 4:r * 4 + 8, c * 4:c * 4 + 8, :].reshape(shape.batch, -1)
        J += ((a[f] - 1) ** 2 * (xf[:, :k] ** 2).sum() + (xf[:, k:] ** 2).sum())
        J += shape.lam * np.sqrt(shape.eps + a[f] ** 2 * (xf[:, :k].reshape(-1, k // g, g) ** 2).sum(-1)).sum()
    assert o["J"] == pytest.approx(J, rel=1e-13)


def test_sign_flip_invariance():
    shape = tiny_shape(g=2, k=4, m=3)
    geo = geo_of(shape)
    W, a, b = rng_params(shape, seed=1, scale_b=0.2)
    X = make_images(shape, seed=2).astype(np.float64)
    o = O.layer_gradients(W, a, b, X, geo)
    W2 = W.copy()
    W2[3, 1] *= -1
    W2[0, 2] *= -1
    o2 = O.layer_gradients(W2, a, b, X, geo)
    assert o2["J"] == pytest.approx(o["J"], rel=1e-14)
    for key in ("dalpha", "db", "dX"):
        np.testing.assert_allclose(o2[key], o[key], rtol=1e-12, atol=1e-13)
    exp = o["dW"].copy()
    exp[3, 1] *= -1
    exp[0, 2] *= -1
    np.testing.assert_allclose(o2["dW"], exp, rtol=1e-12, atol=1e-13)


def test_in_group_permutation_invariance():
    shape = tiny_shape(g=2, k=4, m=3)
    geo = geo_of(shape)
    W, a, b = rng_params(shape, seed=8, scale_b=0.1)
    X = make_images(shape, seed=2).astype(np.float64)
    J = O.layer_gradients(W, a, b, X, geo)["J"]
    W2 = W[:, [1, 0, 3, 2], :]
    assert O.layer_gradients(W2, a, b, X, geo)["J"] == pytest.approx(J, rel=1e-14)
    W3 = W[:, [2, 3, 0, 1], :]   # permuting whole groups also keeps J
    assert O.layer_gradients(W3, a, b, X, geo)["J"] == pytest.approx(J, rel=1e-14)
    W4 = W[:, [0, 2, 1, 3], :]   # across groups: J changes in general
    assert O.layer_gradients(W4, a, b, X, geo)["J"] != pytest.approx(J, rel=1e-10)


def test_field_independence_and_batch_equivariance():
    shape = tiny_shape(g=1, k=4, m=4)
    geo = geo_of(shape)
    W, a, b = rng_params(shape, seed=4, scale_b=0.1)
    X = make_images(shape, seed=3).astype(np.float64)
    p, _ = O.layer_forward(W, a, b, X, geo)
    W2 = W.copy()
    W2[4] = W[2]
    p2, _ = O.layer_forward(W2, a, b, X, geo)
    diff = np.abs(p2 - p).max(axis=(0, 3))
    assert diff[1, 1] > 0 and np.count_nonzero(diff) == 1    # only block (1,1) changed
    pa, _ = O.layer_forward(W, a, b, X[:2], geo)
    pb, _ = O.layer_forward(W, a, b, X[2:], geo)
    np.testing.assert_array_equal(np.concatenate([pa, pb]), p)


def test_one_by_one_grid_is_dense_rica():
    """a 1x1 grid equals dense RICA on the whole image (textbook RICA, Le et al. 2011)."""
    shape = LayerShape("dense", 6, 5, 2, 6, 5, 1, 7, 1, 4, eps=1e-6)
    geo = geo_of(shape)
    W, a, b = rng_params(shape, seed=2, scale_b=0.3)
    X = make_images(shape, seed=1).astype(np.float64)
    o = O.layer_gradients(W, a, b, X, geo)
    Xm = X.reshape(4, -1).T                 # n x m, columns are x^(i)
    Wd = W[0]
    Hm = a[0] * Wd @ Xm
    J = ((Wd.T @ Hm + b[0][:, None] - Xm) ** 2).sum() + shape.lam * np.sqrt(Hm ** 2 + shape.eps).sum()
    assert o["J"] == pytest.approx(J, rel=1e-13)


def test_real_configs_shapes():
    for name in ("c1", "c2", "c3"):
        s = CONFIGS[name]
        gr, gc = O.field_grid(s.img_h, s.img_w, s.rf_h, s.rf_w, s.stride)
        assert (gr, gc) == (s.grid_r, s.grid_c)
    assert CONFIGS["c3"].fields == 8464 and CONFIGS["c3"].n == 972
    assert CONFIGS["c3"].fields * 128 * 972 == 1_053_057_024


def test_projected_sgd_keeps_unit_rows_and_decreases_objective():
    shape = tiny_shape(g=2, k=4, m=6)
    geo = geo_of(shape)
    W, a, b = make_params(shape, seed=0)
    W, a, b = W.astype(np.float64), a.astype(np.float64), b.astype(np.float64)
    X = make_images(shape, seed=1).astype(np.float64)
    J0 = O.layer_gradients(W, a, b, X, geo)["J"]
    vel = None
    for t in range(100):
        o = O.step(W, a, b, X, geo, lr=1e-3, momentum=0.5, velocity=vel, step_index=t)
        W, a, b, vel = o["W_new"], o["alpha_new"], o["b_new"], o["velocity"]
        assert np.abs(np.linalg.norm(W, axis=-1) - 1).max() <= 1e-12
    J1 = O.layer_gradients(W, a, b, X, geo)["J"]
    assert J1 < J0
