"""Run one step through the C ABI and the oracle on the same seeded inputs (shared by the -m gpu tests)."""
import numpy as np

from oracle import lcae_oracle as O
from tests.helpers import geo_of


def gpu_step(shape, precision, W, a, b, X, keep_grads=True, forward_first=True):
    import torch
    from paper_1502_03409_b200 import lcae
    cfg = lcae.make_config(shape, precision=precision, keep_grads=keep_grads)
    L = lcae.Layer(cfg)
    try:
        L.set_params(np.ascontiguousarray(W, np.float32), np.ascontiguousarray(a, np.float32),
                     np.ascontiguousarray(b, np.float32))
        xd = torch.from_numpy(np.ascontiguousarray(X, np.float32)).cuda()
        out = {}
        if forward_first:
            pooled = torch.zeros((shape.batch, L.grid_r, L.grid_c, shape.filters // shape.pool_group),
                                 dtype=torch.float32, device="cuda")
            out["J_fwd"] = L.forward(xd, pooled)
            out["p"] = pooled.cpu().numpy()
        dx = torch.zeros_like(xd)
        out["J"] = L.step(xd, dx)
        out["J_rec"], out["J_sparse"] = L.last_loss()
        out["dX"] = dx.cpu().numpy()
        F, k, n = W.shape
        if keep_grads:
            dW = np.zeros((F, k, n), np.float32)
            da = np.zeros(F, np.float32)
            db = np.zeros((F, n), np.float32)
            L.get_grads(dW, da, db)
            out.update(dW=dW, dalpha=da, db=db)
        W1 = np.zeros((F, k, n), np.float32)
        a1 = np.zeros(F, np.float32)
        b1 = np.zeros((F, n), np.float32)
        L.get_params(W1, a1, b1)
        out.update(W_new=W1, alpha_new=a1, b_new=b1, launches=L.last_launch_count())
        out["steps"], out["reinit"] = L.counters()
        return out
    finally:
        L.close()


def oracle_step(shape, W, a, b, X):
    o = O.step(W.astype(np.float64), a.astype(np.float64), b.astype(np.float64), X.astype(np.float64),
               geo_of(shape), lr=shape.lr, momentum=shape.momentum, alpha_min=shape.alpha_min)
    return o
