"""The general bf16 tensor-core path (gt_path.cu: five batched tcgen05 GEMMs + epilogue kernels) against the fp64
oracle: layers the fused step kernel cannot hold (k > 128 filters: the paper's own layer 1, k = 384)
and, through the LCAE_DEV_FORCE_GT test hook, the shapes the fused kernel's own parity tests use.

bf16 tolerance 2e-2 normwise (BASELINE.json north_star; R10), per tensor: loss, pooled code, dW, dalpha,
db, dX and the parameter update."""
import numpy as np
import pytest

from oracle import lcae_oracle as O
from paper_1502_03409_b200.inputs import EXTRA_CONFIGS, LayerShape, make_images, make_params, stratified_fields
from tests.gpu_harness import gpu_step, oracle_step
from tests.helpers import geo_of, normwise
from tests.test_gpu_parity import SHAPES_BF16, _compare

pytestmark = pytest.mark.gpu

GT_SHAPES = {
    # paper layer-1 field shape (16 x 16 x 3, stride 4, k = 384, m = 192) on a small image: 3 x 3 fields
    "c3p-small": LayerShape("c3p-small", 24, 24, 3, 16, 16, 4, 384, 1, 192),
    # k = 200 (two ragged M tiles), n = 70, pooling g = 4, odd batch (ragged N / K tails), non-square image
    "wide-ragged": LayerShape("wide-ragged", 21, 25, 2, 5, 7, 2, 200, 4, 37),
    # m = 300 > 256 (the fused kernel's 2-CTA limit), k = 160, g = 2
    "m300": LayerShape("m300", 12, 12, 3, 6, 6, 3, 160, 2, 300),
}


def _inputs(shape, raw=True):
    W, a, b = make_params(shape, seed=0)
    X = make_images(shape, seed=1, bf16_round=not raw)
    b = (0.05 * np.random.default_rng(3).standard_normal(b.shape)).astype(np.float32)
    return W, a, b, X


@pytest.mark.parametrize("name", list(GT_SHAPES))
def test_gt_parity_beyond_fused_limits(name):
    from paper_1502_03409_b200 import lcae
    shape = GT_SHAPES[name]
    W, a, b, X = _inputs(shape)
    out = gpu_step(shape, lcae.BF16, W, a, b, X)
    o = oracle_step(shape, W, a, b, X)
    errs = _compare(shape, 1, out, o, W.astype(np.float64), a.astype(np.float64), b.astype(np.float64))
    print(name, {k_: f"{v:.1e}" for k_, v in errs.items()})
    assert out["steps"] == 1 and out["reinit"] == 0


@pytest.mark.parametrize("name", ["worked", "c1", "ragged", "cluster2", "c3tiny"])
def test_gt_parity_forced(name, monkeypatch):
    """The fused kernel's parity shapes, routed through the general path (LCAE_DEV_FORCE_GT=1)."""
    from paper_1502_03409_b200 import lcae
    monkeypatch.setenv("LCAE_DEV_FORCE_GT", "1")
    shape = SHAPES_BF16[name]
    if name == "worked":
        W = np.eye(2, dtype=np.float32)[None]
        a = np.array([2.0], np.float32)
        b = np.zeros((1, 2), np.float32)
        X = np.array([1.0, -1.0], np.float32).reshape(1, 2, 1, 1)
    else:
        W, a, b, X = _inputs(shape)
    out = gpu_step(shape, lcae.BF16, W, a, b, X)
    o = oracle_step(shape, W, a, b, X)
    errs = _compare(shape, 1, out, o, W.astype(np.float64), a.astype(np.float64), b.astype(np.float64))
    print(name, {k_: f"{v:.1e}" for k_, v in errs.items()})


def test_gt_momentum_three_steps(monkeypatch):
    """Three steps with momentum 0.9 (SPEC.md:127 velocity update) on the k = 200 shape."""
    import torch
    from paper_1502_03409_b200 import lcae
    shape = GT_SHAPES["wide-ragged"].replace(momentum=0.9, lr=1e-3)
    W, a, b, _ = _inputs(shape)
    Xs = [make_images(shape, seed=20, index=i, bf16_round=False) for i in range(3)]
    L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16))
    try:
        L.set_params(W, a, b)
        Js = [L.step(torch.from_numpy(X).cuda()) for X in Xs]
        W3 = np.zeros_like(W)
        a3 = np.zeros_like(a)
        b3 = np.zeros_like(b)
        L.get_params(W3, a3, b3)
    finally:
        L.close()
    Wo, ao, bo, vel = W.astype(np.float64), a.astype(np.float64), b.astype(np.float64), None
    for t, X in enumerate(Xs):
        o = O.step(Wo, ao, bo, X.astype(np.float64), geo_of(shape), lr=shape.lr, momentum=0.9, velocity=vel,
                   step_index=t)
        assert abs(Js[t] - o["J"]) <= 2e-2 * abs(o["J"])
        Wo, ao, bo, vel = o["W_new"], o["alpha_new"], o["b_new"], o["velocity"]
    errs = {"dW_3steps": normwise(W3 - W, Wo - W), "alpha_3steps": normwise(a3 - a, ao - a),
            "b_3steps": normwise(b3 - b, bo - b)}
    print(errs)
    assert all(v <= 2e-2 for v in errs.values()), errs


def test_gt_encode_matches_forward():
    """lcae_encode on the general path: the pooled code equals the forward pass's, J_sparse equals the oracle's."""
    import torch
    from paper_1502_03409_b200 import lcae
    shape = GT_SHAPES["c3p-small"]
    W, a, b, X = _inputs(shape)
    L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16))
    try:
        L.set_params(W, a, b)
        xd = torch.from_numpy(X).cuda()
        p1 = torch.zeros((shape.batch, L.grid_r, L.grid_c, shape.filters), device="cuda")
        p2 = torch.zeros_like(p1)
        L.forward(xd, p1)
        js = L.encode(xd, p2)
    finally:
        L.close()
    assert torch.equal(p1, p2)
    o = oracle_step(shape, W, a, b, X)
    assert abs(js - o["J_sparse"]) <= 2e-2 * o["J_sparse"]
    assert normwise(p2.cpu().numpy(), o["p"]) <= 2e-2


@pytest.mark.parametrize("name", ["c3p", "paper2"])
def test_gt_full_size_sampled(name):
    """Full-size layers on the general path in the launch configuration bench.py times: c3' (SURVEY.md §8(d):
    300 x 300 x 3, 16 x 16 x 3 fields at stride 4 -> 72 x 72 fields, k = 384, m = 192; 1.53 B weights) and the
    paper's layer 2 (R26: 288 x 288 x 24, 16 x 16 x 24 windows -> 69 x 69 fields, n = 6144, k = 384; 11.26 B
    weights): per-field losses, the W / alpha / b updates of sampled fields and dX at a probe pixel against the
    oracle."""
    import ctypes
    import torch
    from paper_1502_03409_b200 import lcae
    shape = EXTRA_CONFIGS[name]
    probe = (150, 141)
    s = shape.stride
    cover = [r * shape.grid_c + c for r in range(shape.grid_r) for c in range(shape.grid_c)
             if r * s <= probe[0] < r * s + shape.rf_h and c * s <= probe[1] < c * s + shape.rf_w]
    fl = sorted(set(stratified_fields(shape, 8 if name == "c3p" else 4, seed=3)) | set(cover))
    X = make_images(shape, seed=5, bf16_round=False)
    L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16, seed=7))
    try:
        def params():
            Wf = np.zeros((len(fl), shape.filters, shape.n), np.float32)
            af = np.zeros(len(fl), np.float32)
            bf = np.zeros((len(fl), shape.n), np.float32)
            for i, f in enumerate(fl):
                L.get_field_params(f, 1, Wf[i:i + 1], af[i:i + 1], bf[i:i + 1])
            return Wf, af, bf
        W0, a0, b0 = params()
        xd = torch.from_numpy(X).cuda()
        J = L.step(xd)
        floss = L.field_losses()
        W1, a1, b1 = params()
        torch.cuda.synchronize()
        dxp = L.dx_device_ptr()
        row = np.empty((shape.batch, shape.img_c), np.float32)
        rt = ctypes.CDLL("libcudart.so.12")
        for i in range(shape.batch):
            off = ((i * shape.img_h + probe[0]) * shape.img_w + probe[1]) * shape.img_c * 4
            assert rt.cudaMemcpy(ctypes.c_void_p(row[i].ctypes.data), ctypes.c_void_p(dxp + off),
                                 ctypes.c_size_t(shape.img_c * 4), 2) == 0
    finally:
        L.close()
    assert np.isfinite(J) and abs(floss.sum() - J) <= 1e-9 * abs(J)
    X64 = X.astype(np.float64)
    o = O.step(W0.astype(np.float64), a0.astype(np.float64), b0.astype(np.float64), X64, geo_of(shape), lr=shape.lr,
               fields=fl)
    per = []
    for i, f in enumerate(fl):
        r, c = divmod(f, shape.grid_c)
        q = O.rica_field(W0[i], float(a0[i]), b0[i], O.field_patch(X64, r, c, shape.rf_h, shape.rf_w, s),
                         shape.lam, shape.eps, shape.pool_group)
        per.append((q["J_rec"], q["J_sparse"]))
    per = np.array(per)
    errs = {"J_rec_fields": normwise(floss[fl, 0], per[:, 0]), "J_sparse_fields": normwise(floss[fl, 1], per[:, 1]),
            "dW_update": normwise(W1.astype(np.float64) - W0, o["W_new"] - W0),
            "alpha_update": normwise(a1.astype(np.float64) - a0, o["alpha_new"] - a0),
            "b_update": normwise(b1.astype(np.float64) - b0, o["b_new"] - b0),
            "dX_probe": normwise(row, o["dX"][:, probe[0], probe[1], :])}
    print(name, {k: f"{v:.1e}" for k, v in errs.items()}, len(fl), "fields")
    assert all(v <= 2e-2 for v in errs.values()), errs
    assert np.abs(np.linalg.norm(W1.astype(np.float64), axis=-1) - 1).max() <= 1e-6


@pytest.mark.parametrize("keep", [False, True])
def test_gt_degenerate_row_reinit(keep, monkeypatch):
    """Degenerate-row re-initialisation on the general path: the fused path's test, routed through it."""
    from tests import test_gpu_regimes as R
    monkeypatch.setenv("LCAE_DEV_FORCE_GT", "1")
    R.test_degenerate_row_reinit(1, keep)


def test_gt_alpha_clamp(monkeypatch):
    from tests import test_gpu_regimes as R
    monkeypatch.setenv("LCAE_DEV_FORCE_GT", "1")
    R.test_alpha_clamp(1)


def test_gt_nonfinite_input_is_a_data_error(monkeypatch):
    from tests import test_gpu_regimes as R
    monkeypatch.setenv("LCAE_DEV_FORCE_GT", "1")
    R.test_nonfinite_input_is_a_data_error(1)


def test_gt_trained_regime(monkeypatch):
    """Many steps on the k = 200 shape, then one step compared with the oracle from the trained parameters (the
    lazy projection's sigma drifts away from 1 over the steps)."""
    import torch
    from paper_1502_03409_b200 import lcae
    shape = GT_SHAPES["wide-ragged"].replace(lr=1e-3 / 37)
    W, a, b, _ = _inputs(shape)
    L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16))
    try:
        L.set_params(W, a, b)
        J0 = None
        for t in range(150):
            J = L.step(torch.from_numpy(make_images(shape, seed=100 + t, bf16_round=False)).cuda(), want_loss=(t % 50 == 0))
            if t == 0:
                J0 = J
        L.sync()
        Wt = np.zeros_like(W)
        at = np.zeros_like(a)
        bt = np.zeros_like(b)
        L.get_params(Wt, at, bt)
    finally:
        L.close()
    X = make_images(shape, seed=999, bf16_round=False)
    out = gpu_step(shape, lcae.BF16, Wt, at, bt, X)
    o = oracle_step(shape, Wt, at, bt, X)
    errs = _compare(shape, 1, out, o, Wt.astype(np.float64), at.astype(np.float64), bt.astype(np.float64))
    print("trained", J0, o["J"], {k_: f"{v:.1e}" for k_, v in errs.items()})
    assert o["J"] < J0


@pytest.mark.parametrize("which", ["layer2", "layer3"])
def test_gt_paper_layer_field_shapes(which):
    """One bf16 training step at the paper's layer-2 field shape (n = 6144, k = 384) and at the dense layer 3's full
    shape (n = 62 * 62 * 24 = 92,256, k = 4096; one field), general path vs the oracle at 2e-2."""
    from paper_1502_03409_b200 import lcae
    if which == "layer2":
        shape = LayerShape("paper2-small", 20, 20, 24, 16, 16, 4, 384, 1, 16, lam=0.1)
    else:
        shape = LayerShape("paper3", 62, 62, 24, 62, 62, 1, 4096, 1, 4, lam=0.01)   # m = 4: a quick fp64 oracle
    W, a, b, X = _inputs(shape)
    out = gpu_step(shape, lcae.BF16, W, a, b, X, forward_first=False)
    o = oracle_step(shape, W, a, b, X)
    errs = _compare(shape, 1, out, o, W.astype(np.float64), a.astype(np.float64), b.astype(np.float64))
    print(which, {k_: f"{v:.1e}" for k_, v in errs.items()})


def test_gt_paper_architecture_stack_bf16():
    """The paper's three-layer network (R26) on a 28 x 28 image in bf16 (every layer on the
    general path: k = 384, 384, 4096): each stage's encode against the oracle on the GPU stage's input, 2e-2."""
    import torch
    from paper_1502_03409_b200 import lcae
    from paper_1502_03409_b200.stack import Stack, check_chain, paper_stack
    from oracle.lcae_oracle import layer_gradients
    cfg = paper_stack(batch=8, image=28, lcn_window=3)
    check_chain(cfg)
    X = make_images(cfg.shapes[0], seed=4, bf16_round=False)
    st = Stack(cfg, precision=lcae.BF16, seed=0)
    errs = {}
    try:
        x = torch.from_numpy(X).cuda()
        for l, s in enumerate(cfg.shapes):
            code = st._code(l, x)
            W = np.zeros((s.fields, s.filters, s.n), np.float32)
            a = np.zeros(s.fields, np.float32)
            b = np.zeros((s.fields, s.n), np.float32)
            st.layers[l].get_params(W, a, b)
            want = layer_gradients(W.astype(np.float64), a.astype(np.float64), b.astype(np.float64),
                                   x.cpu().numpy().astype(np.float64), geo_of(s))["p"]
            errs[f"encode{l}"] = normwise(code.cpu().numpy(), want)
            if l + 1 < len(cfg.shapes):
                x = st.next_input(l, st._lcn(st.to_map(l, code)))
    finally:
        st.close()
    print({k: f"{v:.1e}" for k, v in errs.items()})
    assert all(v <= 2e-2 for v in errs.values()), errs
