"""In-library model parallelism (include/lcae.h world_size > 1) on one GPU.

NCCL cannot run several ranks on one GPU, so the ranks are emulated in the library's test mode (nccl_id = NULL):
P layer handles, one per tile, driven through the three phases of a step; between phases the test copies every
rank's send buffers into the receiving ranks' buffers (what the grouped NCCL send / recv does in NCCL mode).
This runs the library's own halo pack / unpack kernels, the interior / boundary field split and the dX return
(overlap-add), and is compared with the untiled layer on the same inputs:
  * parameter updates (W, alpha, b) of every field: bitwise (per-field arithmetic does not depend on the tiling);
  * dX assembled from the ranks' owned pixels and the summed loss: 1e-6 (fp32 atomics change the order);
  * exchanged bytes: the static prediction of parallel.predicted_bytes.
"""
import ctypes

import numpy as np
import pytest

from paper_1502_03409_b200.inputs import LayerShape, make_images, make_params
from paper_1502_03409_b200.parallel import plan, predicted_bytes
from tests.helpers import normwise

pytestmark = pytest.mark.gpu

_rt = None


def _d2d(dst, src, nbytes):
    global _rt
    if _rt is None:
        _rt = ctypes.CDLL("libcudart.so.12")
    assert _rt.cudaMemcpy(ctypes.c_void_p(dst), ctypes.c_void_p(src), ctypes.c_size_t(nbytes), 3) == 0


def _untiled(shape, precision, W, a, b, X):
    import torch
    from paper_1502_03409_b200 import lcae
    L = lcae.Layer(lcae.make_config(shape, precision=precision))
    try:
        L.set_params(W, a, b)
        dx = torch.zeros(X.shape, device="cuda")
        J = L.step(torch.from_numpy(X).cuda(), dx)
        W1, a1, b1 = np.zeros_like(W), np.zeros_like(a), np.zeros_like(b)
        L.get_params(W1, a1, b1)
        return J, dx.cpu().numpy(), W1, a1, b1
    finally:
        L.close()


def _tiled(shape, precision, P, W, a, b, X):
    import torch
    from paper_1502_03409_b200 import lcae
    gr, gc = shape.grid_r, shape.grid_c
    Wg, ag, bg = W.reshape(gr, gc, *W.shape[1:]), a.reshape(gr, gc), b.reshape(gr, gc, -1)
    layers = [lcae.Layer(lcae.make_config(shape, precision=precision, world_size=P, rank=r)) for r in range(P)]
    try:
        for L in layers:
            R0, R1, C0, C1 = L.own_fields
            L.set_params(np.ascontiguousarray(Wg[R0:R1, C0:C1].reshape(-1, *W.shape[1:])),
                         np.ascontiguousarray(ag[R0:R1, C0:C1].reshape(-1)),
                         np.ascontiguousarray(bg[R0:R1, C0:C1].reshape(-1, W.shape[2])))
        xs = []
        for L in layers:
            y0, y1, x0, x1 = L.own_px
            xs.append(torch.from_numpy(np.ascontiguousarray(X[:, y0:y1, x0:x1, :])).cuda())
        moved = {"halo_in": 0, "dx_return": 0}

        def move(src_which, dst_which, key):
            torch.cuda.synchronize()
            for ra in range(P):
                for rb in range(P):
                    if ra == rb:
                        continue
                    ps, ns = layers[ra].mp_buffer(src_which, rb)
                    pr, nr = layers[rb].mp_buffer(dst_which, ra)
                    assert ns == nr, (ra, rb, ns, nr)
                    if ns:
                        _d2d(pr, ps, ns)
                        moved[key] += ns
            torch.cuda.synchronize()

        for L, x in zip(layers, xs):
            L.mp_phase(0, True, x=x)
        move(0, 1, "halo_in")
        for L in layers:
            L.mp_phase(1, True)
        move(2, 3, "dx_return")
        dx = np.zeros(X.shape, np.float32)
        J = 0.0
        W1, a1, b1 = np.zeros_like(Wg), np.zeros_like(ag), np.zeros_like(bg)
        for L, x in zip(layers, xs):
            d = torch.zeros_like(x)
            J += L.mp_phase(2, True, dx=d, want_loss=True)
            y0, y1, x0, x1 = L.own_px
            dx[:, y0:y1, x0:x1, :] = d.cpu().numpy()
            R0, R1, C0, C1 = L.own_fields
            w = np.zeros(((R1 - R0) * (C1 - C0), *W.shape[1:]), np.float32)
            al = np.zeros((R1 - R0) * (C1 - C0), np.float32)
            bb = np.zeros(((R1 - R0) * (C1 - C0), W.shape[2]), np.float32)
            L.get_params(w, al, bb)
            W1[R0:R1, C0:C1] = w.reshape(R1 - R0, C1 - C0, *W.shape[1:])
            a1[R0:R1, C0:C1] = al.reshape(R1 - R0, C1 - C0)
            b1[R0:R1, C0:C1] = bb.reshape(R1 - R0, C1 - C0, -1)
        counts = [L.mp_fields() for L in layers]
        return J, dx, W1.reshape(W.shape), a1.reshape(a.shape), b1.reshape(b.shape), moved, counts
    finally:
        for L in layers:
            L.close()


SHAPES = {
    "cluster2": LayerShape("cluster2", 36, 36, 3, 8, 8, 4, 32, 2, 200),
    "c3small": LayerShape("c3small", 56, 40, 3, 18, 18, 2, 128, 1, 256),
    "ragged": LayerShape("ragged", 29, 25, 2, 5, 7, 2, 24, 4, 40),
    # k = 160 > 128: the general bf16 path (gt_path.cu) in every rank; fp32 for the fp32 runs
    "wide160": LayerShape("wide160", 36, 36, 3, 8, 8, 4, 160, 2, 96),
}


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("name", list(SHAPES))
@pytest.mark.parametrize("precision", [1, 0])
def test_model_parallel_equals_untiled(name, P, precision):
    shape = SHAPES[name]
    if precision == 0 and name == "c3small":
        shape = shape.replace(img_h=40)
    W, a, b = make_params(shape, seed=0)
    b = (0.05 * np.random.default_rng(2).standard_normal(b.shape)).astype(np.float32)
    X = make_images(shape, seed=1, bf16_round=False)
    J0, dx0, W0, a0, b0 = _untiled(shape, precision, W, a, b, X)
    J1, dx1, W1, a1, b1, moved, counts = _tiled(shape, precision, P, W, a, b, X)
    assert np.array_equal(W1, W0) and np.array_equal(a1, a0) and np.array_equal(b1, b0)
    assert abs(J1 - J0) <= 1e-9 * abs(J0)
    assert normwise(dx1, dx0) <= 1e-6
    tiles = plan(shape, P)
    mp = shape.batch if precision == 0 else (shape.batch + 7) // 8 * 8
    want = predicted_bytes(shape.replace(batch=mp), tiles, elem_bytes=4)
    assert moved["dx_return"] == want["dx_return"]
    assert moved["halo_in"] == want["halo_in"] // (2 if precision == 1 else 1)   # bf16 halo on the tensor-core path
    assert sum(i + bnd for i, bnd in counts) == shape.fields
    print(name, P, precision, "interior/boundary", counts, "bytes", moved)


@pytest.mark.parametrize("precision,name", [(1, "c3small"), (0, "cluster2"), (1, "wide160")])
def test_single_rank_nccl_mode_equals_plain_layer(precision, name):
    """world_size = 1 with an NCCL id: the NCCL communicator, the comm stream and events, the interior /
    boundary launches (interior leaves two SM pairs free) and the loss all-reduce all run on one GPU; the step
    equals the plain layer's (bitwise parameters)."""
    import torch
    from paper_1502_03409_b200 import lcae
    shape = SHAPES[name]   # wide160: k = 160, the general bf16 path
    W, a, b = make_params(shape, seed=0)
    X = make_images(shape, seed=1, bf16_round=False)
    J0, dx0, W0, a0, b0 = _untiled(shape, precision, W, a, b, X)
    L = lcae.Layer(lcae.make_config(shape, precision=precision, nccl_id=lcae.nccl_unique_id()))
    try:
        L.set_params(W, a, b)
        n_int, n_bnd = L.mp_fields()
        assert n_int == shape.fields and n_bnd == 0   # one tile owns every pixel
        dx = torch.zeros(X.shape, device="cuda")
        J = L.step(torch.from_numpy(X).cuda(), dx)
        W1, a1, b1 = np.zeros_like(W), np.zeros_like(a), np.zeros_like(b)
        L.get_params(W1, a1, b1)
        pooled = torch.zeros((shape.batch, shape.grid_r, shape.grid_c, shape.filters // shape.pool_group),
                             device="cuda")
        Jf = L.forward(torch.from_numpy(X).cuda(), pooled)
    finally:
        L.close()
    assert np.array_equal(W1, W0) and np.array_equal(a1, a0) and np.array_equal(b1, b0)
    assert abs(J - J0) <= 1e-12 * abs(J0)
    assert normwise(dx.cpu().numpy(), dx0) <= 1e-6
    assert np.isfinite(Jf)
