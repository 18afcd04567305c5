"""Thin ctypes binding of liblcae.so (include/lcae.h).  Argument marshalling only: every step of the
layer's math runs in the library's CUDA kernels.  There is no CPU fallback: if the shared library is
missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LCAE_LIB") or os.path.join(_HERE, "liblcae.so")  # LCAE_LIB: A/B another build

LCAE_OK, LCAE_ERR_CONFIG, LCAE_ERR_DATA, LCAE_ERR_NUMERIC, LCAE_ERR_CUDA, LCAE_ERR_NCCL, LCAE_ERR_ARG = 0, 2, 3, 4, 5, 6, 7
FP32, BF16 = 0, 1


class LcaeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"lcae status {status}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [
        ("img_h", C.c_int32), ("img_w", C.c_int32), ("img_c", C.c_int32),
        ("rf_h", C.c_int32), ("rf_w", C.c_int32), ("stride", C.c_int32),
        ("filters", C.c_int32), ("pool_group", C.c_int32), ("batch", C.c_int32),
        ("lambda_", C.c_float), ("eps", C.c_float), ("lr", C.c_float), ("momentum", C.c_float),
        ("alpha_init", C.c_float), ("alpha_min", C.c_float),
        ("seed", C.c_uint64),
        ("precision", C.c_int32), ("keep_grads", C.c_int32),
        ("field_row0", C.c_int32), ("field_col0", C.c_int32), ("global_grid_c", C.c_int32),
        ("world_size", C.c_int32), ("rank", C.c_int32), ("tiles_r", C.c_int32), ("tiles_c", C.c_int32),
        ("nccl_id", C.c_void_p),
        ("stream", C.c_void_p),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() (make -C paper_1502_03409_b200/csrc)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sigs = {
        "lcae_config_default": (None, [C.POINTER(Config)]),
        "lcae_geometry": (C.c_int, [C.POINTER(Config), C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "lcae_nccl_unique_id": (C.c_int, [P]),
        "lcae_mp_phase": (C.c_int, [P, C.c_int32, C.c_int32, P, P, P, C.POINTER(C.c_double)]),
        "lcae_mp_buffer": (C.c_int, [P, C.c_int32, C.c_int32, C.POINTER(P), C.POINTER(C.c_int64)]),
        "lcae_mp_fields": (C.c_int, [P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "lcae_create": (C.c_int, [C.POINTER(Config), C.POINTER(P)]),
        "lcae_destroy": (C.c_int, [P]),
        "lcae_set_params": (C.c_int, [P, P, P, P]),
        "lcae_get_params": (C.c_int, [P, P, P, P]),
        "lcae_get_grads": (C.c_int, [P, P, P, P]),
        "lcae_get_field_params": (C.c_int, [P, C.c_int64, C.c_int64, P, P, P]),
        "lcae_forward": (C.c_int, [P, P, P, C.POINTER(C.c_double)]),
        "lcae_step": (C.c_int, [P, P, P, C.POINTER(C.c_double)]),
        "lcae_encode": (C.c_int, [P, P, P, C.POINTER(C.c_double)]),
        "lcae_prefetch_input": (C.c_int, [P, P]),
        "lcae_topk_init": (C.c_int, [P, P, C.c_int64, C.c_int32, P]),
        "lcae_lcn": (C.c_int, [P, P, P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_float, P]),
        "lcae_topk_update": (C.c_int, [P, C.c_int64, C.c_int64, C.c_int32, C.c_int64, P, P, P]),
        "lcae_last_loss": (C.c_int, [P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "lcae_sync": (C.c_int, [P]),
        "lcae_field_losses": (C.c_int, [P, P]),
        "lcae_dx_device": (C.c_int, [P, C.POINTER(P)]),
        "lcae_counters": (C.c_int, [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "lcae_region_add": (C.c_int, [P, P, C.c_int32, C.c_int32, P, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_int32]),
        "lcae_last_launch_count": (C.c_int32, [P]),
        "lcae_profile": (C.c_int, [P, C.c_int32]),
        "lcae_profile_read": (C.c_int, [P, C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
        "lcae_last_error": (C.c_char_p, []),
        "lcae_version": (C.c_char_p, []),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

_devlib = None


def devlib():
    """liblcae_dev.so: the product library plus the hardware self-tests / micro-benchmarks (lcae_dev_*), which
    the product library does not carry."""
    global _devlib
    if _devlib is None:
        path = os.path.join(_HERE, "liblcae_dev.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} not built (make -C paper_1502_03409_b200/csrc)")
        d = C.CDLL(path)
        P = C.c_void_p
        for name, (res, args) in {
            "lcae_dev_umma_selftest": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, P, P]),
            "lcae_dev_tma_selftest": (C.c_int, [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P]),
            "lcae_dev_red_probe": (C.c_int, [P, C.c_int64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]),
            "lcae_dev_tmem_shape_selftest": (C.c_int, [P]),
            "lcae_last_error": (C.c_char_p, []),
        }.items():
            fn = getattr(d, name)
            fn.restype = res
            fn.argtypes = args
        _devlib = d
    return _devlib


def dev_check(status: int):
    if status != LCAE_OK:
        raise LcaeError(status, devlib().lcae_last_error().decode())

# Every symbol include/lcae.h declares (checked by tests/test_abi_cpu.py).
ABI_SYMBOLS = ("lcae_config_default", "lcae_geometry", "lcae_create", "lcae_destroy", "lcae_set_params",
               "lcae_get_params", "lcae_get_grads", "lcae_get_field_params", "lcae_forward", "lcae_encode", "lcae_step", "lcae_last_loss",
               "lcae_sync", "lcae_field_losses", "lcae_nccl_unique_id", "lcae_mp_phase", "lcae_mp_buffer",
               "lcae_mp_fields",
               "lcae_topk_init", "lcae_topk_update", "lcae_lcn", "lcae_prefetch_input",
               "lcae_dx_device", "lcae_counters", "lcae_region_add", "lcae_last_launch_count",
               "lcae_profile", "lcae_profile_read",
               "lcae_last_error", "lcae_version")


def check(status: int):
    if status != LCAE_OK:
        raise LcaeError(status, lib.lcae_last_error().decode())


def _ptr(a) -> Optional[int]:
    """data pointer of a torch tensor or numpy array (None passes through as NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"] and a.dtype == np.float32, "expected contiguous float32"
        return a.ctypes.data
    assert a.is_contiguous(), "expected a contiguous tensor"
    return a.data_ptr()


def make_config(shape, precision=BF16, keep_grads=False, stream=None, seed=0, field_row0=0, field_col0=0,
                global_grid_c=0, img_h=None, img_w=None, world_size=1, rank=0, tiles=(0, 0), nccl_id=None) -> Config:
    """nccl_id: a 128-byte bytes object from nccl_unique_id() (kept alive by the returned Config)."""
    cfg = Config()
    lib.lcae_config_default(C.byref(cfg))
    cfg.img_h = shape.img_h if img_h is None else img_h
    cfg.img_w = shape.img_w if img_w is None else img_w
    cfg.img_c = shape.img_c
    cfg.rf_h, cfg.rf_w, cfg.stride = shape.rf_h, shape.rf_w, shape.stride
    cfg.filters, cfg.pool_group, cfg.batch = shape.filters, shape.pool_group, shape.batch
    cfg.lambda_, cfg.eps, cfg.lr, cfg.momentum = shape.lam, shape.eps, shape.lr, shape.momentum
    cfg.alpha_init, cfg.alpha_min = shape.alpha_init, shape.alpha_min
    cfg.seed = seed
    cfg.precision = precision
    cfg.keep_grads = int(bool(keep_grads))
    cfg.field_row0, cfg.field_col0, cfg.global_grid_c = field_row0, field_col0, global_grid_c
    cfg.world_size, cfg.rank = world_size, rank
    cfg.tiles_r, cfg.tiles_c = tiles
    if nccl_id is not None:
        buf = C.create_string_buffer(bytes(nccl_id), 128)
        cfg._nccl_buf = buf   # keep alive with the config
        cfg.nccl_id = C.cast(buf, C.c_void_p)
    cfg.stream = stream
    return cfg


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for Config.nccl_id (lcae_nccl_unique_id; one rank creates, all use)."""
    buf = C.create_string_buffer(128)
    check(lib.lcae_nccl_unique_id(buf))
    return buf.raw


def geometry(cfg: Config):
    gr, gc, npar = C.c_int32(), C.c_int32(), C.c_int64()
    check(lib.lcae_geometry(C.byref(cfg), C.byref(gr), C.byref(gc), C.byref(npar), None, None))
    return gr.value, gc.value, npar.value


def tile_geometry(cfg: Config):
    """(grid_r, grid_c, n_params, own_px (y0, y1, x0, x1), own_fields (R0, R1, C0, C1)) of this rank."""
    gr, gc, npar = C.c_int32(), C.c_int32(), C.c_int64()
    px, fl = (C.c_int32 * 4)(), (C.c_int32 * 4)()
    check(lib.lcae_geometry(C.byref(cfg), C.byref(gr), C.byref(gc), C.byref(npar), px, fl))
    return gr.value, gc.value, npar.value, tuple(px), tuple(fl)


class Layer:
    """One locally-connected RICA layer on the current CUDA device (owns its device memory)."""

    def __init__(self, cfg: Config):
        self.cfg = cfg
        self.grid_r, self.grid_c, self.n_params = geometry(cfg)
        self.F = self.grid_r * self.grid_c
        self.k = cfg.filters
        self.n = cfg.rf_h * cfg.rf_w * cfg.img_c
        self.m = cfg.batch
        self.img_shape = (cfg.batch, cfg.img_h, cfg.img_w, cfg.img_c)
        if cfg.world_size > 1:   # model parallel: x / dx are this rank's owned pixels
            _, _, _, self.own_px, self.own_fields = tile_geometry(cfg)
            y0, y1, x0, x1 = self.own_px
            self.img_shape = (cfg.batch, y1 - y0, x1 - x0, cfg.img_c)
        h = C.c_void_p()
        check(lib.lcae_create(C.byref(cfg), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            check(lib.lcae_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_params(self, W=None, alpha=None, b=None):
        check(lib.lcae_set_params(self.h, _ptr(W), _ptr(alpha), _ptr(b)))

    def get_params(self, W=None, alpha=None, b=None):
        check(lib.lcae_get_params(self.h, _ptr(W), _ptr(alpha), _ptr(b)))

    def get_field_params(self, f0, count, W=None, alpha=None, b=None):
        """Parameters of fields [f0, f0 + count) (lcae_get_field_params)."""
        check(lib.lcae_get_field_params(self.h, f0, count, _ptr(W), _ptr(alpha), _ptr(b)))

    def get_grads(self, dW=None, dalpha=None, db=None):
        check(lib.lcae_get_grads(self.h, _ptr(dW), _ptr(dalpha), _ptr(db)))

    def step(self, x, dx=None, want_loss=True):
        loss = C.c_double(0.0)
        check(lib.lcae_step(self.h, _ptr(x), _ptr(dx), C.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def forward(self, x, pooled=None, want_loss=True):
        loss = C.c_double(0.0)
        check(lib.lcae_forward(self.h, _ptr(x), _ptr(pooled), C.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def prefetch_input(self, x_host):
        """Overlap the host->device copy of the next batch with the current step (lcae_prefetch_input)."""
        check(lib.lcae_prefetch_input(self.h, _ptr(x_host)))

    def encode(self, x, pooled, want_loss=True):
        """Inference: encode + L2 pooling only (lcae_encode); returns J_sparse if want_loss."""
        loss = C.c_double(0.0)
        check(lib.lcae_encode(self.h, _ptr(x), _ptr(pooled), C.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def last_loss(self):
        a, b = C.c_double(), C.c_double()
        check(lib.lcae_last_loss(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def mp_phase(self, phase, update=True, x=None, dx=None, pooled=None, want_loss=False):
        """Model-parallel test mode: one of the three phases of a step (include/lcae.h lcae_mp_phase)."""
        loss = C.c_double(0.0)
        check(lib.lcae_mp_phase(self.h, phase, int(bool(update)), _ptr(x), _ptr(dx), _ptr(pooled),
                                C.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def mp_buffer(self, which, peer):
        """(device pointer, bytes) of exchange buffer `which` (0 halo send, 1 halo recv, 2 dX send, 3 dX recv)."""
        p, n = C.c_void_p(), C.c_int64()
        check(lib.lcae_mp_buffer(self.h, which, peer, C.byref(p), C.byref(n)))
        return p.value, n.value

    def mp_fields(self):
        a, b = C.c_int32(), C.c_int32()
        check(lib.lcae_mp_fields(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def sync(self):
        """Wait for the layer's stream; raises LcaeError (DATA / NUMERIC) for a flagged non-finite input / loss."""
        check(lib.lcae_sync(self.h))

    def field_losses(self) -> np.ndarray:
        """[F][2] float64: per-field (J_rec, J_sparse) of the last step / forward."""
        out = np.zeros((self.F, 2), np.float64)
        check(lib.lcae_field_losses(self.h, out.ctypes.data))
        return out

    def dx_device_ptr(self) -> int:
        p = C.c_void_p()
        check(lib.lcae_dx_device(self.h, C.byref(p)))
        return p.value

    def counters(self):
        s, r = C.c_int64(), C.c_int64()
        check(lib.lcae_counters(self.h, C.byref(s), C.byref(r)))
        return s.value, r.value

    def last_launch_count(self) -> int:
        return int(lib.lcae_last_launch_count(self.h))

    def profile(self, enable: bool):
        check(lib.lcae_profile(self.h, int(bool(enable))))

    def profile_read(self):
        ms, n = C.c_double(), C.c_int32()
        check(lib.lcae_profile_read(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value


def region_add(dst, src, y0: int, x0: int, stream=None):
    """dst[:, y0:y0+rows, x0:x0+cols, :] += src on the GPU (lcae_region_add); NHWC float32 device tensors."""
    m, dh, dw, Cc = dst.shape
    _, rows, cols, _ = src.shape
    check(lib.lcae_region_add(stream, _ptr(dst), dh, dw, _ptr(src), m, rows, cols, Cc, y0, x0))


def topk_init(vals, ids, stream=None):
    """Reset a streaming top-K state: vals float32 [units][K], ids int32 [units][K] (CUDA tensors)."""
    units, K = vals.shape
    check(lib.lcae_topk_init(vals.data_ptr(), ids.data_ptr(), units, K, stream))


def topk_update(act, vals, ids, id0, stream=None):
    """Merge one batch of activations act float32 [m][units] (CUDA) whose sample s is image id0 + s."""
    m, units = act.shape[0], vals.shape[0]
    check(lib.lcae_topk_update(act.data_ptr(), m, units, vals.shape[1], id0, vals.data_ptr(), ids.data_ptr(), stream))


def lcn(x, y, scratch, window=9, floor=1e-4, stream=None):
    """Local contrast normalisation (lcae_lcn): x, y float32 CUDA [m][H][W][C], scratch >= 2 x.numel()."""
    m, H, W, Cc = x.shape
    assert scratch.numel() >= 2 * x.numel()
    check(lib.lcae_lcn(x.data_ptr(), y.data_ptr(), scratch.data_ptr(), m, H, W, Cc, window, floor, stream))

