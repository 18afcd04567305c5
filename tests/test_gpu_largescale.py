"""Sampled oracle parity at the HBM-bound §8(f) item 3 points (VERDICT r1 "next" 8):

* c15b: the paper's 15 B-parameter count as ONE c3-shaped layer on one B200 (347 x 348 fields, 15.02 B weights,
  device-initialised: the host never holds W); one lean training step, compared on sampled fields read back with
  lcae_get_field_params -- per-field losses, the W / alpha / b updates and dX at a probe pixel;
* c3 with momentum 0.9 (SPEC.md:127 velocity update): three steps on three batches, the parameters of sampled
  fields after the third step against the oracle's three steps with its own velocity.

bf16 tolerance 2e-2 normwise (BASELINE.json north_star; R10)."""
import numpy as np
import pytest

from oracle import lcae_oracle as O
from paper_1502_03409_b200.inputs import CONFIGS, LayerShape, make_images, make_params, stratified_fields
from tests.helpers import geo_of, normwise

pytestmark = pytest.mark.gpu

C15B = LayerShape("c15b", 710, 712, 3, 18, 18, 2, 128, 1, 256, lr=1e-3 / 256)


def _covering(shape, y, x):
    s = shape.stride
    rs = [r for r in range(shape.grid_r) if r * s <= y < r * s + shape.rf_h]
    cs = [c for c in range(shape.grid_c) if c * s <= x < c * s + shape.rf_w]
    return [r * shape.grid_c + c for r in rs for c in cs]


def _field_params(L, shape, fl):
    W = np.zeros((len(fl), shape.filters, shape.n), np.float32)
    a = np.zeros(len(fl), np.float32)
    b = np.zeros((len(fl), shape.n), np.float32)
    for i, f in enumerate(fl):
        L.get_field_params(f, 1, W[i:i + 1], a[i:i + 1], b[i:i + 1])
    return W, a, b


def test_c15b_sampled_parity():
    import torch
    from paper_1502_03409_b200 import lcae
    shape = C15B
    assert shape.fields * shape.filters * shape.n > 15e9
    probe = (355, 371)
    fl = sorted(set(stratified_fields(shape, 12, seed=11)) | set(_covering(shape, *probe)))
    X = make_images(shape, seed=5, bf16_round=False)
    L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16, seed=7))
    try:
        W0, a0, b0 = _field_params(L, shape, fl)
        assert np.abs(np.linalg.norm(W0.astype(np.float64), axis=-1) - 1).max() < 1e-5   # device init: unit rows
        xd = torch.from_numpy(X).cuda()
        J = L.step(xd)
        floss = L.field_losses()
        W1, a1, b1 = _field_params(L, shape, fl)
        import ctypes
        torch.cuda.synchronize()
        dxp = L.dx_device_ptr()
        y, x = probe
        row = np.empty((shape.batch, shape.img_c), np.float32)
        rt = ctypes.CDLL("libcudart.so.12")
        for i in range(shape.batch):   # dX[i, y, x, :] (NHWC), one small copy per sample
            off = ((i * shape.img_h + y) * shape.img_w + x) * shape.img_c * 4
            assert rt.cudaMemcpy(ctypes.c_void_p(row[i].ctypes.data), ctypes.c_void_p(dxp + off),
                                 ctypes.c_size_t(shape.img_c * 4), 2) == 0
        del xd
    finally:
        L.close()
    assert np.isfinite(J) and abs(floss.sum() - J) <= 1e-9 * abs(J)
    X64 = X.astype(np.float64)
    o = O.step(W0.astype(np.float64), a0.astype(np.float64), b0.astype(np.float64), X64, geo_of(shape), lr=shape.lr,
               fields=fl)
    per = []
    for i, f in enumerate(fl):
        r, c = divmod(f, shape.grid_c)
        q = O.rica_field(W0[i], float(a0[i]), b0[i], O.field_patch(X64, r, c, shape.rf_h, shape.rf_w, shape.stride),
                         shape.lam, shape.eps, shape.pool_group)
        per.append((q["J_rec"], q["J_sparse"]))
    per = np.array(per)
    errs = {"J_rec_fields": normwise(floss[fl, 0], per[:, 0]), "J_sparse_fields": normwise(floss[fl, 1], per[:, 1]),
            "dW_update": normwise(W1.astype(np.float64) - W0, o["W_new"] - W0),
            "alpha_update": normwise(a1.astype(np.float64) - a0, o["alpha_new"] - a0),
            "b_update": normwise(b1.astype(np.float64) - b0, o["b_new"] - b0),
            "dX_probe": normwise(row, o["dX"][:, probe[0], probe[1], :])}
    print("c15b", {k: f"{v:.1e}" for k, v in errs.items()}, len(fl), "fields")
    assert all(v <= 2e-2 for v in errs.values()), errs
    assert np.abs(np.linalg.norm(W1.astype(np.float64), axis=-1) - 1).max() <= 1e-6


def test_c3_momentum_three_steps_sampled():
    import torch
    from paper_1502_03409_b200 import lcae
    shape = CONFIGS["c3"].replace(momentum=0.9)
    fl = stratified_fields(shape, 24, seed=13)
    W, a, b = make_params(shape, seed=0)
    b = (0.02 * np.random.default_rng(8).standard_normal(b.shape)).astype(np.float32)
    Xs = [make_images(shape, seed=20, index=i, bf16_round=False) for i in range(3)]
    L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16))
    try:
        L.set_params(W, a, b)
        for X in Xs:
            L.step(torch.from_numpy(X).cuda(), None, want_loss=False)
        L.sync()
        W3, a3, b3 = _field_params(L, shape, fl)
    finally:
        L.close()
    Wo, ao, bo = W[fl].astype(np.float64), a[fl].astype(np.float64), b[fl].astype(np.float64)
    vel = None
    for t, X in enumerate(Xs):
        o = O.step(Wo, ao, bo, X.astype(np.float64), geo_of(shape), lr=shape.lr, momentum=0.9, velocity=vel,
                   fields=fl, step_index=t)
        Wo, ao, bo, vel = o["W_new"], o["alpha_new"], o["b_new"], o["velocity"]
    W0, a0, b0 = W[fl].astype(np.float64), a[fl].astype(np.float64), b[fl].astype(np.float64)
    errs = {"dW_3steps": normwise(W3 - W0, Wo - W0), "alpha_3steps": normwise(a3 - a0, ao - a0),
            "b_3steps": normwise(b3 - b0, bo - b0)}
    print("c3 momentum 0.9", {k: f"{v:.1e}" for k, v in errs.items()})
    assert all(v <= 2e-2 for v in errs.values()), errs
