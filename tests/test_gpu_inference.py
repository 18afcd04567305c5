"""Inference path: lcae_encode (encode + L2 pooling only, SPEC.md:490
forward_dataset) and the streaming top-K stimuli kernel, against the fp64 oracle."""
import numpy as np
import pytest

from oracle import layer_gradients, top_k_stimuli
from paper_1502_03409_b200.inputs import CONFIGS, LayerShape, make_images, make_params
from tests.helpers import geo_of, normwise

pytestmark = pytest.mark.gpu

SHAPES = {
    "c1": CONFIGS["c1"],
    "c2": CONFIGS["c2"],
    "cluster2": LayerShape("cluster2", 20, 20, 3, 8, 8, 4, 32, 2, 200),
}


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16", 2e-2)])
@pytest.mark.parametrize("name", list(SHAPES))
def test_encode_matches_oracle_and_forward(name, precision, tol):
    import torch
    from paper_1502_03409_b200 import lcae
    shape = SHAPES[name]
    if precision == "fp32" and name != "c1":
        pytest.skip("fp32 path covered on c1")
    W, a, b = make_params(shape, seed=0)
    X = make_images(shape, seed=1)
    o = layer_gradients(W.astype(np.float64), a.astype(np.float64), b.astype(np.float64), X.astype(np.float64),
                        geo_of(shape))
    L = lcae.Layer(lcae.make_config(shape, precision=lcae.FP32 if precision == "fp32" else lcae.BF16))
    try:
        L.set_params(W, a, b)
        xd = torch.from_numpy(np.ascontiguousarray(X, np.float32)).cuda()
        shp = (shape.batch, L.grid_r, L.grid_c, shape.filters // shape.pool_group)
        p_enc = torch.zeros(shp, dtype=torch.float32, device="cuda")
        js = L.encode(xd, p_enc)
        p_fwd = torch.zeros(shp, dtype=torch.float32, device="cuda")
        L.forward(xd, p_fwd)
        W1, a1, b1 = np.zeros_like(W), np.zeros_like(a), np.zeros_like(b)
        L.get_params(W1, a1, b1)
    finally:
        L.close()
    p_enc = p_enc.cpu().numpy()
    assert normwise(p_enc, o["p"]) <= tol
    assert abs(js - o["J_sparse"]) <= tol * abs(o["J_sparse"])
    # the encode-only pass is the forward pass's first half: identical pooled codes, parameters untouched
    assert np.array_equal(p_enc, p_fwd.cpu().numpy())
    assert np.array_equal(W1, W) and np.array_equal(a1, a) and np.array_equal(b1, b)


@pytest.mark.parametrize("K", [1, 5, 32])
def test_topk_stream_matches_full_sort(K):
    import torch
    from paper_1502_03409_b200 import lcae
    rng = np.random.default_rng(K)
    units = 3000
    batches = [0, 7, 64, 1, 33]   # includes an empty batch; total 105 images
    # quantised values: plenty of ties, so the lower-id rule is exercised
    acts = [np.round(rng.standard_normal((m, units)) * 2).astype(np.float32) for m in batches]
    vals = torch.empty((units, K), dtype=torch.float32, device="cuda")
    ids = torch.empty((units, K), dtype=torch.int32, device="cuda")
    lcae.topk_init(vals, ids)
    id0 = 0
    for A in acts:
        if A.shape[0]:
            lcae.topk_update(torch.from_numpy(A).cuda(), vals, ids, id0)
        id0 += A.shape[0]
    torch.cuda.synchronize()
    ov, oi = top_k_stimuli(np.concatenate(acts, axis=0), K)
    kk = ov.shape[1]
    assert np.array_equal(ids.cpu().numpy()[:, :kk], oi)
    assert np.array_equal(vals.cpu().numpy()[:, :kk].astype(np.float64), ov)
    if kk < K:   # fewer images than K: the remaining slots keep the sentinel
        assert np.all(ids.cpu().numpy()[:, kk:] == np.iinfo(np.int32).max)


def test_forward_dataset_topk_end_to_end():
    """Stream several batches through lcae_encode into the top-K state (the paper's 'forward propagated ...
    to obtain activation values' + 'top 5 stimuli'); the state equals a full sort of the concatenated pooled
    codes, which themselves match the oracle batch by batch."""
    import torch
    from paper_1502_03409_b200 import lcae
    shape = CONFIGS["c1"]
    W, a, b = make_params(shape, seed=0)
    L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16))
    K = 5
    try:
        L.set_params(W, a, b)
        units = L.grid_r * L.grid_c * (shape.filters // shape.pool_group)
        vals = torch.empty((units, K), dtype=torch.float32, device="cuda")
        ids = torch.empty((units, K), dtype=torch.int32, device="cuda")
        lcae.topk_init(vals, ids)
        pooled_all = []
        for bi in range(3):
            X = make_images(shape, seed=10 + bi)
            xd = torch.from_numpy(np.ascontiguousarray(X, np.float32)).cuda()
            p = torch.zeros((shape.batch, units), dtype=torch.float32, device="cuda")
            L.encode(xd, p, want_loss=False)
            lcae.topk_update(p, vals, ids, bi * shape.batch)
            pn = p.cpu().numpy()
            o = layer_gradients(W.astype(np.float64), a.astype(np.float64), b.astype(np.float64),
                                X.astype(np.float64), geo_of(shape))
            assert normwise(pn, o["p"].reshape(shape.batch, units)) <= 2e-2
            pooled_all.append(pn)
        torch.cuda.synchronize()
    finally:
        L.close()
    ov, oi = top_k_stimuli(np.concatenate(pooled_all, axis=0), K)
    assert np.array_equal(ids.cpu().numpy(), oi)
    assert np.array_equal(vals.cpu().numpy().astype(np.float64), ov)
