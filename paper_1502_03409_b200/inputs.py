"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no encode / pool / decode /
gradient / update).  It only knows the layer *shapes* of the BASELINE.json
configs and how to draw seeded inputs of those shapes:

* images  X : [m][H][W][C] float32, i.i.d. N(0,1) per pixel (the synthetic
  analogue of the paper's whitened patches, "whitened as in
  [coates13]"), standardised per image and channel (SPEC.md:424-432
  standardize_image), then (by default) rounded to bf16-representable float32
  so that the fp32 and bf16 device paths and the fp64 oracle all see identical
  values; ``bf16_round=False`` keeps the raw float32 values (the bf16 path then
  rounds x itself, and the parity tests measure that rounding too).
* params  W : [F][k][n] float32, Gaussian rows normalised to unit length
  ("subject to ||W^(k)||_2 = 1"); alpha = alpha_init; b = 0.
  Each field draws from its own SeedSequence([seed, 0x57, f]) so any subset
  of fields can be regenerated on the host without drawing all of them.

Recipe and seeds are restated in DESIGN.md ("Input recipe").
"""
from __future__ import annotations

import dataclasses
from typing import Iterable, Optional

import numpy as np


@dataclasses.dataclass(frozen=True)
class LayerShape:
    """One locally-connected RICA layer (SPEC.md:160-172 FieldGeometry/UntiedLayer)."""
    name: str
    img_h: int
    img_w: int
    img_c: int
    rf_h: int
    rf_w: int
    stride: int
    filters: int          # k per field ("output size 4x4x24" = 384 for the paper layer)
    pool_group: int       # g; g = 1 is the paper's un-pooled sparsity term
    batch: int            # m
    lam: float = 0.1      # PAPER.md:93 "lambda ... set to 0.1 at the first two layers"
    eps: float = 1e-6     # SPEC.md:138 smoothing of sqrt((alpha W x)^2)
    lr: float = 1e-3      # SPEC.md:141 default learning rate
    momentum: float = 0.0
    alpha_init: float = 1.0
    alpha_min: float = 1e-8   # SPEC.md:124 alpha clamp

    # ---- derived geometry (integer bookkeeping only) ----
    @property
    def grid_r(self) -> int:
        return (self.img_h - self.rf_h) // self.stride + 1

    @property
    def grid_c(self) -> int:
        return (self.img_w - self.rf_w) // self.stride + 1

    @property
    def fields(self) -> int:
        return self.grid_r * self.grid_c

    @property
    def n(self) -> int:
        return self.rf_h * self.rf_w * self.img_c

    def replace(self, **kw) -> "LayerShape":
        return dataclasses.replace(self, **kw)


# BASELINE.json "configs" (SURVEY.md §8 shape table; R8: config 3 stride 2).
# lr = 1e-3 / m (R19): the objective sums over the batch (R6), so SPEC.md:141's lr = 1e-3 is the
# per-sample step; with it c2 / c3 diverge within 50 steps (alpha blows up), with 1e-3 / m they descend.
CONFIGS = {
    "c1": LayerShape("c1", 32, 32, 1, 8, 8, 4, 16, 2, 8, lr=1e-3 / 8),
    "c2": LayerShape("c2", 96, 96, 3, 16, 16, 8, 64, 4, 128, lr=1e-3 / 128),
    "c3": LayerShape("c3", 200, 200, 3, 18, 18, 2, 128, 1, 256, lr=1e-3 / 256),
}

# SURVEY.md §8(d)/(f) points beyond BASELINE.json's configs (bench.py --config):
# c15b: the paper's parameter count ("15 billion parameters") as one c3-shaped layer, 347 x 348
#   fields of 18 x 18 x 3 -> 128 filters (15.02 B weights), batch 256, on ONE GPU;
# c3p: the paper-exact layer 1 (16 x 16 x 3 receptive fields, stride 4 -> 4 x 4 x 24 = 384 filters;
#   PAPER.md:111 mini-batch 192) on 300 x 300 x 3 images: 72 x 72 = 5184 fields, 1.53 B weights.
EXTRA_CONFIGS = {
    "c15b": LayerShape("c15b", 710, 712, 3, 18, 18, 2, 128, 1, 256, lr=1e-3 / 256),
    "c3p": LayerShape("c3p", 300, 300, 3, 16, 16, 4, 384, 1, 192, lr=1e-3 / 192),
    # the paper's layer 2 alone (R26): 69 x 69 fields of 16 x 16 x 24 (n = 6144) -> 384, 11.26 B weights
    "paper2": LayerShape("paper2", 288, 288, 24, 16, 16, 4, 384, 1, 192, lam=0.1, lr=1e-3 / 192),
    # the paper's dense layer 3 alone: one field of 62 x 62 x 24 = 92,256 inputs -> 4096 units
    "paper3dense": LayerShape("paper3dense", 62, 62, 24, 62, 62, 1, 4096, 1, 192, lam=0.01, lr=1e-3 / 192),
}


def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16-representable float32 (RN-even)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def make_images(shape: LayerShape, seed: int = 1, index: int = 0,
                batch: Optional[int] = None, bf16_round: bool = True) -> np.ndarray:
    """Seeded whitened-like image batch, NHWC float32 [m][H][W][C] (bf16-representable unless bf16_round=False)."""
    m = shape.batch if batch is None else batch
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x1A, index]))
    x = rng.standard_normal((m, shape.img_h, shape.img_w, shape.img_c))
    mu = x.mean(axis=(1, 2), keepdims=True)
    sd = x.std(axis=(1, 2), keepdims=True)
    x = (x - mu) / np.maximum(sd, 1e-12)
    x = x.astype(np.float32)
    return round_to_bf16(x) if bf16_round else x


def make_field_weights(shape: LayerShape, fields: Iterable[int], seed: int = 0) -> np.ndarray:
    """Unit-row Gaussian W for the listed global field indices: float32 [len][k][n]."""
    fields = list(fields)
    out = np.empty((len(fields), shape.filters, shape.n), dtype=np.float32)
    for i, f in enumerate(fields):
        rng = np.random.default_rng(np.random.SeedSequence([seed, 0x57, int(f)]))
        w = rng.standard_normal((shape.filters, shape.n))
        w /= np.sqrt((w * w).sum(axis=1, keepdims=True))
        out[i] = w.astype(np.float32)
    return out


def make_params(shape: LayerShape, seed: int = 0, fields: Optional[Iterable[int]] = None):
    """(W [F][k][n] f32, alpha [F] f32, b [F][n] f32) for all (or the listed) fields."""
    fl = list(range(shape.fields)) if fields is None else list(fields)
    W = make_field_weights(shape, fl, seed)
    alpha = np.full((len(fl),), shape.alpha_init, dtype=np.float32)
    b = np.zeros((len(fl), shape.n), dtype=np.float32)
    return W, alpha, b


def field_rc(shape: LayerShape, f: int):
    """Row-major field index -> (grid row, grid col)."""
    return divmod(int(f), shape.grid_c)


def stratified_fields(shape: LayerShape, count: int, seed: int = 7) -> list:
    """A deterministic spread of field indices: the four corners, the centre, then seeded picks."""
    F = shape.fields
    base = [0, shape.grid_c - 1, F - shape.grid_c, F - 1, (shape.grid_r // 2) * shape.grid_c + shape.grid_c // 2]
    rng = np.random.default_rng(seed)
    extra = list(rng.choice(F, size=min(F, max(0, count)), replace=False))
    out = []
    for f in base + extra:
        if int(f) not in out:
            out.append(int(f))
        if len(out) >= count:
            break
    return sorted(out)
