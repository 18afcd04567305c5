"""Three-layer stack with LCN: lcae_lcn against the LCN oracle, the stack's forward
chain against the oracle chain (fp32), and each greedy layer step against the oracle step on the same
input (bf16)."""
import numpy as np
import pytest

from oracle import layer_gradients, lcn, step as oracle_step
from paper_1502_03409_b200.inputs import make_images, make_params
from tests.helpers import geo_of, normwise

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,window", [((3, 9, 11, 4), 3), ((2, 13, 12, 128), 9), ((1, 7, 7, 16), 7)])
def test_lcn_matches_oracle(shape, window):
    import torch
    from paper_1502_03409_b200 import lcae
    x = np.random.default_rng(window).standard_normal(shape).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    y = torch.empty_like(xd)
    lcae.lcn(xd, y, torch.empty(2 * xd.numel(), device="cuda"), window, 1e-4)
    torch.cuda.synchronize()
    assert normwise(y.cpu().numpy(), lcn(x, window, 1e-4)) <= 1e-5


def test_lcn_rejects_bad_window():
    import torch
    from paper_1502_03409_b200 import lcae
    xd = torch.zeros((1, 5, 5, 2), device="cuda")
    with pytest.raises(lcae.LcaeError):
        lcae.lcn(xd, torch.empty_like(xd), torch.empty(2 * xd.numel(), device="cuda"), 7, 1e-4)


def _oracle_chain(cfg, params, X):
    x = X.astype(np.float64)
    outs = []
    for i, s in enumerate(cfg.shapes):
        W, a, b = params[i]
        p = layer_gradients(W.astype(np.float64), a.astype(np.float64), b.astype(np.float64), x, geo_of(s))["p"]
        outs.append(p)
        if i + 1 < len(cfg.shapes):   # LCN between layers only
            x = lcn(p, cfg.lcn_window, cfg.lcn_floor)
    return outs


def test_stack_forward_matches_oracle_chain_fp32():
    """Each stage of the fp32 forward chain (encode, LCN, encode, LCN, encode) against the oracle on the GPU
    stage's own input, at north_star's 1e-5; and the whole chain against the all-oracle chain at 1e-5."""
    import torch
    from paper_1502_03409_b200 import lcae
    from paper_1502_03409_b200.stack import Stack, desk_stack
    cfg = desk_stack(batch=8)
    X = make_images(cfg.shapes[0], seed=1)
    params = [make_params(s, seed=i) for i, s in enumerate(cfg.shapes)]
    st = Stack(cfg, precision=lcae.FP32, seed=0)
    errs = {}
    try:
        x = torch.from_numpy(X).cuda()
        for l, s in enumerate(cfg.shapes):
            code = st._code(l, x)
            W, a, b = params[l]
            want = layer_gradients(W.astype(np.float64), a.astype(np.float64), b.astype(np.float64),
                                   x.cpu().numpy().astype(np.float64), geo_of(s))["p"]
            errs[f"encode{l}"] = normwise(code.cpu().numpy(), want)
            if l + 1 < len(cfg.shapes):
                x = st._lcn(code)
                errs[f"lcn{l}"] = normwise(x.cpu().numpy(), lcn(code.cpu().numpy().astype(np.float64),
                                                               cfg.lcn_window, cfg.lcn_floor))
        top = st.forward(torch.from_numpy(X).cuda()).cpu().numpy()
    finally:
        st.close()
    want = _oracle_chain(cfg, params, X)[-1]
    assert top.shape == want.shape == (8, 1, 1, 16)
    errs["chain"] = normwise(top, want)
    print({k: f"{v:.1e}" for k, v in errs.items()})
    assert all(v <= 1e-5 for v in errs.values()), errs


def test_greedy_layer_steps_match_oracle_bf16():
    import torch
    from paper_1502_03409_b200 import lcae
    from paper_1502_03409_b200.stack import Stack, desk_stack
    cfg = desk_stack(batch=16)
    X = make_images(cfg.shapes[0], seed=2)
    st = Stack(cfg, precision=lcae.BF16, seed=0)
    try:
        xd = torch.from_numpy(X).cuda()
        for l, s in enumerate(cfg.shapes):
            inp = st.input_of(l, xd)
            inp_h = inp.cpu().numpy()
            W0, a0, b0 = make_params(s, seed=l)
            # encode of this layer vs the oracle on the same (GPU-produced) input
            code = st._code(l, inp).cpu().numpy()
            o = layer_gradients(W0.astype(np.float64), a0.astype(np.float64), b0.astype(np.float64),
                                inp_h.astype(np.float64), geo_of(s))
            assert normwise(code, o["p"]) <= 2e-2
            # the LCN of this code vs the oracle LCN of the same code (fp32 kernel)
            if l + 1 < len(cfg.shapes):
                nxt = st._lcn(torch.from_numpy(code).cuda()).cpu().numpy()
                assert normwise(nxt, lcn(code, cfg.lcn_window, cfg.lcn_floor)) <= 1e-5
            # one greedy step of layer l vs the oracle step on the same input
            st.layers[l].step(inp, None)
            W1, a1, b1 = np.zeros_like(W0), np.zeros_like(a0), np.zeros_like(b0)
            st.layers[l].get_params(W1, a1, b1)
            ref = oracle_step(W0.astype(np.float64), a0.astype(np.float64), b0.astype(np.float64),
                              inp_h.astype(np.float64), geo_of(s), lr=s.lr, alpha_min=s.alpha_min)
            assert normwise(W1 - W0, ref["W_new"] - W0) <= 2e-2
            assert normwise(a1 - a0, ref["alpha_new"] - a0) <= 2e-2
            assert normwise(b1 - b0, ref["b_new"] - b0) <= 2e-2
    finally:
        st.close()


def test_chain_geometry_checked():
    from paper_1502_03409_b200.stack import StackConfig, check_chain, desk_stack
    cfg = desk_stack(batch=4)
    bad = StackConfig([cfg.shapes[0], cfg.shapes[2]])
    with pytest.raises(ValueError):
        check_chain(bad)


def _oracle_map(p, block):
    """Numpy statement of the block-map layout (stack.to_map): [m][gr][gc][bh*bw*c] -> [m][gr*bh][gc*bw][c]."""
    if block is None:
        return p
    m, gr, gc, ch = p.shape
    c = ch // (block[0] * block[1])
    return p.reshape(m, gr, gc, block[0], block[1], c).transpose(0, 1, 3, 2, 4, 5).reshape(m, gr * block[0],
                                                                                          gc * block[1], c)


def test_paper_architecture_stack_fp32():
    """The paper's three-layer network (read as DESIGN.md R26) at its field shapes -- 16x16x3 -> 384
    (4x4x24 blocks), 16 contiguous 4x4x24 blocks (n = 6144) -> 384, dense -> 4096 -- on a 28 x 28 image: every
    stage of the fp32 chain (encode, block map, LCN, crop) against the oracle on the GPU stage's input, 1e-5."""
    import torch
    from paper_1502_03409_b200 import lcae
    from paper_1502_03409_b200.stack import Stack, check_chain, paper_stack
    cfg = paper_stack(batch=8, image=28, lcn_window=3)   # the small maps (16 x 16, 4 x 4) take a 3 x 3 LCN window
    check_chain(cfg)
    X = make_images(cfg.shapes[0], seed=4, bf16_round=False)
    params = [make_params(s, seed=i) for i, s in enumerate(cfg.shapes)]
    st = Stack(cfg, precision=lcae.FP32, seed=0)
    errs = {}
    try:
        x = torch.from_numpy(X).cuda()
        for l, s in enumerate(cfg.shapes):
            code = st._code(l, x)
            W, a, b = params[l]
            want = layer_gradients(W.astype(np.float64), a.astype(np.float64), b.astype(np.float64),
                                   x.cpu().numpy().astype(np.float64), geo_of(s))["p"]
            errs[f"encode{l}"] = normwise(code.cpu().numpy(), want)
            mp = st.to_map(l, code)
            assert np.array_equal(mp.cpu().numpy(), _oracle_map(code.cpu().numpy(), cfg.block(l)))
            if l + 1 < len(cfg.shapes):
                y = st._lcn(mp)
                errs[f"lcn{l}"] = normwise(y.cpu().numpy(), lcn(mp.cpu().numpy().astype(np.float64), cfg.lcn_window,
                                                               cfg.lcn_floor))
                x = st.next_input(l, y)
                assert x.shape[1:] == (cfg.shapes[l + 1].img_h, cfg.shapes[l + 1].img_w, cfg.shapes[l + 1].img_c)
    finally:
        st.close()
    print({k: f"{v:.1e}" for k, v in errs.items()})
    assert all(v <= 1e-5 for v in errs.values()), errs


@pytest.mark.parametrize("which", ["layer2", "layer3"])
def test_paper_layer_field_shapes_fp32(which):
    """One training step at the paper's layer-2 field shape (n = 6144, k = 384) and at the dense layer 3's full
    shape (n = 62 * 62 * 24 = 92,256, k = 4096), fp32 path vs the oracle at north_star's 1e-5."""
    from paper_1502_03409_b200.inputs import LayerShape
    from tests.gpu_harness import gpu_step, oracle_step as harness_oracle_step
    from tests.test_gpu_parity import _compare
    if which == "layer2":
        shape = LayerShape("paper2-small", 20, 20, 24, 16, 16, 4, 384, 1, 16, lam=0.1)
    else:
        # m = 4 keeps the fp64 oracle quick
        shape = LayerShape("paper3", 62, 62, 24, 62, 62, 1, 4096, 1, 4, lam=0.01)
    W, a, b = make_params(shape, seed=0)
    b = (0.05 * np.random.default_rng(3).standard_normal(b.shape)).astype(np.float32)
    X = make_images(shape, seed=1, bf16_round=False)
    out = gpu_step(shape, 0, W, a, b, X, forward_first=False)
    o = harness_oracle_step(shape, W, a, b, X)
    if which == "layer2":
        errs = _compare(shape, 0, out, o, W.astype(np.float64), a.astype(np.float64), b.astype(np.float64))
    else:
        # north_star's 1e-5 names activations, loss and gradients: those are held to it. The projected update of a
        # 92,256-long row (W' = rownorm(W - lr dW)) inherits the gradient's 1e-5-level error through
        # the row's radial correction (a dot product over n terms), so the update is held to 1e-4 here.
        errs = {"J": abs(out["J"] - o["J"]) / abs(o["J"])}
        for key in ("dW", "dalpha", "db", "dX"):
            errs[key] = normwise(out[key], o[key])
        assert all(v <= 1e-5 for v in errs.values()), errs
        W64 = W.astype(np.float64)
        errs["dW_update"] = normwise(out["W_new"].astype(np.float64) - W64, o["W_new"] - W64)
        errs["b_update"] = normwise(out["b_new"].astype(np.float64) - b, o["b_new"] - b)
        assert errs["dW_update"] <= 1e-4 and errs["b_update"] <= 1e-5, errs
    print(which, {k: f"{v:.1e}" for k, v in errs.items()})
