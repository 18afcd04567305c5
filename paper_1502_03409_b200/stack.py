"""Three-layer stack with LCN between layers, greedy layer-wise training.

PAPER.md:93-95 (§3.1): three untied (locally connected) RICA layers, "local contrast normalization (LCN) is
applied prior to continuing onto the next layer"; PAPER.md:111 trains the layers greedily, one after the
other. Each layer is an `lcae.Layer` (the fused sm_100a step kernel); the input of layer l is the pooled code
of layer l-1 (lcae_encode) passed through lcae_lcn. The top layer is "dense" by geometry: one field whose
receptive field covers the whole map ("1x1 grid equals dense encoding").

Argument marshalling only: every step runs in the library's kernels.
"""
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import torch

from . import lcae
from .inputs import LayerShape, make_params

HOST_PARAMS_MAX = 4e9   # larger layers are initialised on the device (lcae_create's counter-based generator)


@dataclass
class StackConfig:
    shapes: List[LayerShape]
    lcn_window: int = 3
    lcn_floor: float = 1e-4
    # per layer: its output arranged as blocks of (bh, bw, k/g / (bh bw)) pixels ("output size
    # 4x4x24"), or None (k/g channels at the field's grid position)
    out_block: List[Optional[Tuple[int, int]]] = field(default_factory=list)
    # per layer: the centre crop (h, w) of the previous layer's (LCN'd) map this layer reads, or None
    in_crop: List[Optional[Tuple[int, int]]] = field(default_factory=list)

    def block(self, l):
        return self.out_block[l] if l < len(self.out_block) else None

    def crop(self, l):
        return self.in_crop[l] if l < len(self.in_crop) else None


def desk_stack(batch: int = 16) -> StackConfig:
    """A desk-scale 3-layer geometry chain: 32x32x1 -> 7x7x16 -> 3x3x16 -> 1x1x16 (dense top layer)."""
    l1 = LayerShape("stack1", 32, 32, 1, 8, 8, 4, 16, 1, batch)
    l2 = LayerShape("stack2", l1.grid_r, l1.grid_c, l1.filters // l1.pool_group, 3, 3, 2, 16, 1, batch)
    l3 = LayerShape("stack3", l2.grid_r, l2.grid_c, l2.filters // l2.pool_group, l2.grid_r, l2.grid_c, 1, 16, 1,
                    batch)
    return StackConfig([l1, l2, l3])


def paper_stack(batch: int = 192, image: int = 300, lcn_window: int = 9) -> StackConfig:
    """The paper's network, read as DESIGN.md R26:
    layer 1: 16 x 16 x 3 receptive fields, stride 4, 384 = 4 x 4 x 24 outputs per field (72 x 72 fields on a 300 x 300
    image, 1.53 B weights); its code is arranged as a 288 x 288 x 24 block map; LCN;
    layer 2: 16 spatially contiguous 4 x 4 x 24 blocks (a 16 x 16 x 24 window, n = 6144), stride 4, 384 = 4 x 4 x 24
    outputs (69 x 69 fields, 11.2 B weights); block map 276 x 276 x 24; LCN;
    layer 3: dense (one field) over 62 x 62 x 24 = 92,256 inputs -- the centre of the layer-2 map -- to 4096 units
    (377,972,833 parameters). lambda 0.1 / 0.1 / 0.01; mini-batch 192."""
    l1 = LayerShape("paper1", image, image, 3, 16, 16, 4, 384, 1, batch, lam=0.1, lr=1e-3 / batch)
    m1 = (l1.grid_r * 4, l1.grid_c * 4, 24)
    l2 = LayerShape("paper2", m1[0], m1[1], 24, 16, 16, 4, 384, 1, batch, lam=0.1, lr=1e-3 / batch)
    c3 = min(62, l2.grid_r * 4)
    l3 = LayerShape("paper3", c3, c3, 24, c3, c3, 1, 4096, 1, batch, lam=0.01, lr=1e-3 / batch)
    return StackConfig([l1, l2, l3], lcn_window=lcn_window, lcn_floor=1e-4, out_block=[(4, 4), (4, 4), None],
                       in_crop=[None, None, (c3, c3)])


def out_map_shape(cfg: StackConfig, l):
    s = cfg.shapes[l]
    bl = cfg.block(l)
    ch = s.filters // s.pool_group
    if bl is None:
        return (s.grid_r, s.grid_c, ch)
    return (s.grid_r * bl[0], s.grid_c * bl[1], ch // (bl[0] * bl[1]))


def check_chain(cfg: StackConfig):
    for l, (a, b) in enumerate(zip(cfg.shapes, cfg.shapes[1:])):
        h, w, c = out_map_shape(cfg, l)
        cr = cfg.crop(l + 1)
        if cr is not None:
            if cr[0] > h or cr[1] > w:
                raise ValueError(f"layer {b.name}: crop {cr} larger than the previous map {(h, w)}")
            h, w = cr
        if (b.img_h, b.img_w, b.img_c) != (h, w, c):
            raise ValueError(f"layer {b.name} input {(b.img_h, b.img_w, b.img_c)} does not match the previous "
                             f"layer's output {(h, w, c)}")
        if b.batch != a.batch:
            raise ValueError("all layers of a stack share the mini-batch size")


class Stack:
    def __init__(self, cfg: StackConfig, precision=lcae.BF16, seed=0, stream=None, host_params=True):
        check_chain(cfg)
        self.cfg = cfg
        self.stream = stream
        self.layers = []
        for i, s in enumerate(cfg.shapes):
            L = lcae.Layer(lcae.make_config(s, precision=precision, stream=stream, seed=seed + i))
            if host_params and s.fields * s.filters * s.n <= HOST_PARAMS_MAX:   # else: the library's device init
                W, a, b = make_params(s, seed=seed + i)
                L.set_params(W, a, b)
            self.layers.append(L)

    def close(self):
        for L in self.layers:
            L.close()
        self.layers = []

    def _code(self, l, x):
        """Pooled code of layer l for input x (device NHWC f32), [m][gr][gc][k/g]."""
        s = self.cfg.shapes[l]
        p = torch.empty((s.batch, s.grid_r, s.grid_c, s.filters // s.pool_group), dtype=torch.float32,
                        device=x.device)
        self.layers[l].encode(x, p, want_loss=False)
        return p

    def _lcn(self, p):
        y = torch.empty_like(p)
        scratch = torch.empty(2 * p.numel(), dtype=torch.float32, device=p.device)
        lcae.lcn(p, y, scratch, self.cfg.lcn_window, self.cfg.lcn_floor, self.stream)
        return y

    def to_map(self, l, p):
        """Layer l's code [m][gr][gc][k/g] as its output map (blocks laid out spatially)."""
        bl = self.cfg.block(l)
        if bl is None:
            return p
        m, gr, gc, ch = p.shape
        c = ch // (bl[0] * bl[1])
        return p.reshape(m, gr, gc, bl[0], bl[1], c).permute(0, 1, 3, 2, 4, 5).reshape(m, gr * bl[0], gc * bl[1],
                                                                                       c).contiguous()

    def next_input(self, l, y):
        """The (LCN'd) map y of layer l as layer l+1 reads it (centre crop, if any)."""
        cr = self.cfg.crop(l + 1)
        if cr is None:
            return y
        h, w = y.shape[1], y.shape[2]
        y0, x0 = (h - cr[0]) // 2, (w - cr[1]) // 2
        return y[:, y0:y0 + cr[0], x0:x0 + cr[1], :].contiguous()

    def input_of(self, l, x):
        """The input of layer l: the images for l = 0, else LCN(output map of layer l-1 of the input of l-1)."""
        for i in range(l):
            x = self.next_input(i, self._lcn(self.to_map(i, self._code(i, x))))
        return x

    def forward(self, x):
        """Top-layer code of a batch (the 'activation values' of PAPER.md:156)."""
        return self.to_map(len(self.layers) - 1,
                           self._code(len(self.layers) - 1, self.input_of(len(self.layers) - 1, x)))

    def train_greedy(self, batches, steps_per_layer: int):
        """Greedy layer-wise training: layer l trains on LCN'd codes of the trained layers below.
        Returns the per-layer losses of the last step."""
        losses = []
        for l, L in enumerate(self.layers):
            J = None
            for t in range(steps_per_layer):
                x = batches[t % len(batches)]
                J = L.step(self.input_of(l, x), None)
            losses.append(J)
        return losses
