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
