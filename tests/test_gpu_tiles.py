"""Tiled (model-parallel) computation on one GPU vs the untiled layer, both through the C ABI.

Each tile of parallel.plan runs as its own lcae layer on its `need` region (global field ids via
field_row0/col0); the input halo is taken by slicing (the exchange itself is covered on CPU by
tests/test_parallel_cpu.py); the partial input gradients are overlap-added into the global dX with the
library's lcae_region_add kernel.  Result must match the P = 1 layer (SURVEY.md §8(e) correctness)."""
import numpy as np
import pytest

from paper_1502_03409_b200 import parallel
from paper_1502_03409_b200.inputs import LayerShape, make_images, make_params
from tests.helpers import normwise

pytestmark = pytest.mark.gpu

SHAPE = LayerShape("tiles", 30, 26, 3, 8, 6, 2, 32, 2, 160)   # grid 12 x 11, two-CTA clusters


@pytest.mark.parametrize("precision,tol", [(0, 1e-5), (1, 2e-3)])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_tiles_match_single_layer(world, precision, tol):
    import torch
    from paper_1502_03409_b200 import lcae
    shape = SHAPE
    W, a, b = make_params(shape, seed=0)
    X = torch.from_numpy(make_images(shape, seed=1)).cuda()
    full = lcae.Layer(lcae.make_config(shape, precision=precision, keep_grads=True))
    full.set_params(W, a, b)
    dX_ref = torch.zeros_like(X)
    J_ref = full.step(X, dX_ref)
    dW_ref = np.zeros_like(W)
    full.get_grads(dW_ref, None, None)
    full.close()
    dX = torch.zeros_like(X)
    J = 0.0
    for t in parallel.plan(shape, world):
        gr, gc = t.grid
        fids = [(t.fields_r[0] + r) * shape.grid_c + t.fields_c[0] + c for r in range(gr) for c in range(gc)]
        ts = parallel.tile_shape(shape, t)
        L = lcae.Layer(lcae.make_config(ts, precision=precision, keep_grads=True, field_row0=t.fields_r[0],
                                        field_col0=t.fields_c[0], global_grid_c=shape.grid_c))
        L.set_params(np.ascontiguousarray(W[fids]), np.ascontiguousarray(a[fids]), np.ascontiguousarray(b[fids]))
        n = t.need
        x_ext = X[:, n[0]:n[1], n[2]:n[3], :].contiguous()
        dx_ext = torch.zeros_like(x_ext)
        J += L.step(x_ext, dx_ext)
        dWt = np.zeros((len(fids), shape.filters, shape.n), np.float32)
        L.get_grads(dWt, None, None)
        L.close()
        assert normwise(dWt, dW_ref[fids]) <= tol
        lcae.region_add(dX, dx_ext, n[0], n[2])          # overlap-add across tiles (GPU kernel)
    torch.cuda.synchronize()
    assert J == pytest.approx(J_ref, rel=tol)
    assert normwise(dX.cpu().numpy(), dX_ref.cpu().numpy()) <= tol
