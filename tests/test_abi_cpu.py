"""C-ABI checks that need no GPU: the library loads, exports every symbol include/lcae.h declares, and
lcae_geometry validates configurations (SPEC.md:185-193 examples and error codes)."""
import ctypes as C
import os
import re

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
    # 9 int32 (36) + 6 float (60) + pad (64) + uint64 (72) + 6 int32 (96) + void* (104) on LP64
    assert C.sizeof(lcae.Config) == 104
    assert lcae.Config.stream.offset == 96 and lcae.Config.seed.offset == 64
    cfg = lcae.Config()
    lcae.lib.lcae_config_default(C.byref(cfg))
    assert cfg.lambda_ == pytest.approx(0.1) and cfg.eps == pytest.approx(1e-6) and cfg.lr == pytest.approx(1e-3)
    assert cfg.alpha_init == 1.0 and cfg.alpha_min == pytest.approx(1e-8) and cfg.precision == lcae.BF16


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
