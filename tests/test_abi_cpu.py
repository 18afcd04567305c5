"""C-ABI checks that need no GPU: the library loads, exports every symbol include/lcae.h declares, and
lcae_geometry validates configurations (SPEC.md:185-193 examples and error codes)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from tests.conftest import ROOT


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "lcae.h")).read()
    return sorted(set(re.findall(r"\b(lcae_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_1502_03409_b200 import lcae
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lcae.lib, s), s
    assert set(lcae.ABI_SYMBOLS) == set(syms)
    assert lcae.lib.lcae_version().decode().endswith("sm_100a")


def test_config_struct_layout_matches_header():
    from paper_1502_03409_b200 import lcae
    # 9 int32 (36) + 6 float (60) + pad (64) + uint64 (72) + 5 int32 (92) + 4 int32 (108) + pad (112)
    # + nccl_id (120) + stream (128) on LP64
    assert C.sizeof(lcae.Config) == 128
    assert lcae.Config.stream.offset == 120 and lcae.Config.seed.offset == 64
    assert lcae.Config.nccl_id.offset == 112 and lcae.Config.world_size.offset == 92
    cfg = lcae.Config()
    lcae.lib.lcae_config_default(C.byref(cfg))
    assert cfg.lambda_ == pytest.approx(0.1) and cfg.eps == pytest.approx(1e-6) and cfg.lr == pytest.approx(1e-3)
    assert cfg.alpha_init == 1.0 and cfg.alpha_min == pytest.approx(1e-8) and cfg.precision == lcae.BF16
    assert cfg.world_size == 1 and cfg.rank == 0 and not cfg.nccl_id


def _cfg(**kw):
    from paper_1502_03409_b200 import lcae
    from paper_1502_03409_b200.inputs import LayerShape
    base = dict(img_h=300, img_w=300, img_c=3, rf=16, stride=4, k=384, g=1, m=192)
    base.update(kw)
    shape = LayerShape("t", base["img_h"], base["img_w"], base["img_c"], base["rf"], base["rf"], base["stride"],
                       base["k"], base["g"], base["m"])
    return lcae.make_config(shape)


def test_geometry_examples(golden):
    from paper_1502_03409_b200 import lcae
    for cs in golden["geometry"]["cases"]:
        (H, W, Cc), (fh, fw), s = cs["img"], cs["rf"], cs["stride"]
        gr, gc, npar = lcae.geometry(_cfg(img_h=H, img_w=W, img_c=Cc, rf=fh, stride=s, k=384))
        assert [gr, gc] == cs["grid"]
    gr, gc, npar = lcae.geometry(_cfg())
    assert npar == golden["param_count"]["cases"][0]["total"]


def test_geometry_errors():
    from paper_1502_03409_b200 import lcae
    for kw, frag in ((dict(img_h=200, img_w=200, rf=18, stride=4), "residue rows=2"),
                     (dict(g=5, k=10), "pool_group must divide 32"),
                     (dict(g=4, k=10), "pool_group must divide filters"),
                     (dict(rf=400), "larger than image"),
                     (dict(m=0), "positive")):
        with pytest.raises(lcae.LcaeError) as ei:
            lcae.geometry(_cfg(**kw))
        assert ei.value.status == lcae.LCAE_ERR_CONFIG
        assert frag in str(ei.value)
    cfg = _cfg()
    cfg.precision = 9
    with pytest.raises(lcae.LcaeError):
        lcae.geometry(cfg)


def test_null_handles_are_rejected_without_gpu():
    from paper_1502_03409_b200 import lcae
    assert lcae.lib.lcae_destroy(None) == lcae.LCAE_OK
    assert lcae.lib.lcae_step(None, None, None, None) == lcae.LCAE_ERR_ARG
    assert lcae.lib.lcae_get_params(None, None, None, None) == lcae.LCAE_ERR_ARG
    assert lcae.lib.lcae_create(None, None) == lcae.LCAE_ERR_ARG


@pytest.mark.parametrize("world", [1, 2, 3, 4, 6, 8])
@pytest.mark.parametrize("shape_name", ["c2", "c3", "ragged"])
def test_library_tiling_matches_the_plan(world, shape_name):
    """lcae_geometry's per-rank tile (own pixels, own fields, local grid) equals parallel.plan,
    the tiles cover the field grid exactly once and the owned pixels partition the image."""
    from paper_1502_03409_b200 import lcae
    from paper_1502_03409_b200.inputs import CONFIGS, LayerShape
    from paper_1502_03409_b200.parallel import plan
    shape = {"c2": CONFIGS["c2"], "c3": CONFIGS["c3"],
             "ragged": LayerShape("ragged", 21, 25, 2, 5, 7, 2, 24, 4, 37)}[shape_name]
    tiles = plan(shape, world)
    cover = np.zeros((shape.grid_r, shape.grid_c), int)
    pix = np.zeros((shape.img_h, shape.img_w), int)
    for t in tiles:
        cfg = lcae.make_config(shape, world_size=world, rank=t.rank)
        gr, gc, npar, own_px, own_fl = lcae.tile_geometry(cfg)
        assert own_px == t.own and own_fl == (*t.fields_r, *t.fields_c)
        assert (gr, gc) == t.grid and npar == gr * gc * (shape.filters * shape.n + shape.n + 1)
        cover[t.fields_r[0]:t.fields_r[1], t.fields_c[0]:t.fields_c[1]] += 1
        pix[own_px[0]:own_px[1], own_px[2]:own_px[3]] += 1
    assert (cover == 1).all() and (pix == 1).all()


def test_library_tiling_errors():
    from paper_1502_03409_b200 import lcae
    from paper_1502_03409_b200.inputs import CONFIGS
    shape = CONFIGS["c1"]   # 7 x 7 field grid
    for kw, frag in ((dict(world_size=8, tiles=(8, 1)), "no field"), (dict(world_size=4, tiles=(3, 1)), "equal"),
                     (dict(world_size=2, rank=2), "rank")):
        with pytest.raises(lcae.LcaeError) as ei:
            lcae.tile_geometry(lcae.make_config(shape, **kw))
        assert ei.value.status == lcae.LCAE_ERR_CONFIG and frag in str(ei.value)
