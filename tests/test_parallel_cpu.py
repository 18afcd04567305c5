"""Model-parallel path on CPU (gloo, world_size 2 and 4): tile plan, input-halo exchange, dX return and
overlap-add, byte accounting.  Each rank computes its tile with the fp64 oracle (test-only compute) on its
extended region; the assembled result must equal the single-process oracle (SPEC.md:363-365 distributed
equivalence; SPEC.md:378-379 logged bytes == predicted bytes)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lcae_oracle as O
from paper_1502_03409_b200 import parallel
from paper_1502_03409_b200.inputs import CONFIGS, LayerShape, make_images, make_params
from tests.helpers import geo_of

SHAPE = LayerShape("par", 22, 18, 2, 6, 4, 2, 6, 2, 3)     # grid 9 x 8, rf 6x4, stride 2


def _bias(fids, n, F):
    """a deterministic non-zero offset b per global field id (so b enters the comparison)"""
    return np.array([[0.01 * (f * n + t) / (F * n) for t in range(n)] for f in fids])


def test_plan_partitions_fields_and_pixels():
    for world in (1, 2, 3, 4, 8):
        if world > SHAPE.grid_r * SHAPE.grid_c:
            continue
        tiles = parallel.plan(SHAPE, world)
        fields = np.zeros((SHAPE.grid_r, SHAPE.grid_c), int)
        pix = np.zeros((SHAPE.img_h, SHAPE.img_w), int)
        for t in tiles:
            fields[t.fields_r[0]:t.fields_r[1], t.fields_c[0]:t.fields_c[1]] += 1
            pix[t.own[0]:t.own[1], t.own[2]:t.own[3]] += 1
            # every field's window lies inside the tile's `need` region
            y0 = t.fields_r[0] * SHAPE.stride
            y1 = (t.fields_r[1] - 1) * SHAPE.stride + SHAPE.rf_h
            assert (y0, y1) == (t.need[0], t.need[1])
        assert np.all(fields == 1) and np.all(pix == 1)
    assert parallel.factor(8) == (4, 2) and parallel.factor(4) == (2, 2) and parallel.factor(2) == (2, 1)
    c3 = parallel.plan(CONFIGS["c3"], 8)
    assert {t.grid for t in c3} == {(23, 46)}          # 92x92 fields -> eight 23x46 tiles
    with pytest.raises(ValueError):
        parallel.split(3, 4)


def test_predicted_bytes_monotone_in_world():
    prev = -1
    for world in (1, 2, 4, 8):
        b = parallel.predicted_bytes(CONFIGS["c3"], parallel.plan(CONFIGS["c3"], world), elem_bytes=4)
        tot = b["halo_in"] + b["dx_return"]
        assert tot >= prev                             # SPEC.md:380 non-decreasing in P
        prev = tot
    assert parallel.predicted_bytes(CONFIGS["c3"], parallel.plan(CONFIGS["c3"], 1))["halo_in"] == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape = SHAPE
        tiles = parallel.plan(shape, world)
        me = tiles[rank]
        X = make_images(shape, seed=1).astype(np.float64)
        o = me.own
        x_own = torch.from_numpy(X[:, o[0]:o[1], o[2]:o[3], :].copy())
        h, w = me.need_hw
        x_ext = torch.zeros((shape.batch, h, w, shape.img_c), dtype=torch.float64)
        hx = parallel.HaloExchange(tiles, rank, dist)
        hx.gather_input(x_own, x_ext)
        # the rank-local problem: image = need region, fields = this tile's fields (global ids)
        gr, gc = me.grid
        fids = [(me.fields_r[0] + r) * shape.grid_c + me.fields_c[0] + c for r in range(gr) for c in range(gc)]
        W, a, b = make_params(shape, seed=0, fields=fids)
        b = _bias(fids, shape.n, shape.fields)
        geo = geo_of(parallel.tile_shape(shape, me))
        res = O.layer_gradients(W.astype(np.float64), a.astype(np.float64), b, x_ext.numpy(), geo)
        dx_ext = torch.from_numpy(res["dX"])
        dx_own = torch.zeros_like(x_own)

        def add_region(dst, src, y0, x0):
            dst[:, y0:y0 + src.shape[1], x0:x0 + src.shape[2], :] += src

        hx.return_dx(dx_ext, dx_own, add_region)
        J = torch.tensor([res["J"]], dtype=torch.float64)
        dist.all_reduce(J)
        sent = torch.tensor([hx.bytes_sent["halo_in"], hx.bytes_sent["dx_return"]], dtype=torch.float64)
        dist.all_reduce(sent)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), dx_own=dx_own.numpy(), own=np.array(o), J=J.numpy(),
                 sent=sent.numpy(), dW=res["dW"], fids=np.array(fids))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_tiles_equal_single_process(world, tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    shape = SHAPE
    W, a, b = make_params(shape, seed=0)
    b = _bias(range(shape.fields), shape.n, shape.fields)   # same per-field offsets as the workers
    X = make_images(shape, seed=1).astype(np.float64)
    ref = O.layer_gradients(W.astype(np.float64), a.astype(np.float64), b, X, geo_of(shape))
    dX = np.full(X.shape, np.nan)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        o = z["own"]
        dX[:, o[0]:o[1], o[2]:o[3], :] = z["dx_own"]
        np.testing.assert_allclose(z["dW"], ref["dW"][z["fids"]], rtol=1e-12, atol=1e-12)
        assert z["J"][0] == pytest.approx(ref["J"], rel=1e-12)
        pred = parallel.predicted_bytes(shape, parallel.plan(shape, world), elem_bytes=8)
        assert z["sent"][0] == pred["halo_in"] and z["sent"][1] == pred["dx_return"]
    np.testing.assert_allclose(dX, ref["dX"], rtol=1e-12, atol=1e-12)
