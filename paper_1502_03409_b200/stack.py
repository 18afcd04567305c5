"""Three-layer stack with LCN between layers, greedy layer-wise training.

PAPER.md:93-95 (§3.1): three untied (locally connected) RICA layers, "local contrast normalization (LCN) is
applied prior to continuing onto the next layer"; PAPER.md:111 trains the layers greedily, one after the
other. Each layer is an `lcae.Layer` (the fused sm_100a step kernel); the input of layer l is the pooled code
of layer l-1 (lcae_encode) passed through lcae_lcn. The top layer is "dense" by geometry: one field whose
receptive field covers the whole map ("1x1 grid equals dense encoding").

Argument marshalling only: every step runs in the library's kernels.
"""
from dataclasses import dataclass
from typing import List

import torch

from . import lcae
from .inputs import LayerShape, make_params


@dataclass
class StackConfig:
    shapes: List[LayerShape]
    lcn_window: int = 3
    lcn_floor: float = 1e-4


def desk_stack(batch: int = 16) -> StackConfig:
    """A desk-scale 3-layer geometry chain: 32x32x1 -> 7x7x16 -> 3x3x16 -> 1x1x16 (dense top layer)."""
    l1 = LayerShape("stack1", 32, 32, 1, 8, 8, 4, 16, 1, batch)
    l2 = LayerShape("stack2", l1.grid_r, l1.grid_c, l1.filters // l1.pool_group, 3, 3, 2, 16, 1, batch)
    l3 = LayerShape("stack3", l2.grid_r, l2.grid_c, l2.filters // l2.pool_group, l2.grid_r, l2.grid_c, 1, 16, 1,
                    batch)
    return StackConfig([l1, l2, l3])


def check_chain(cfg: StackConfig):
    for a, b in zip(cfg.shapes, cfg.shapes[1:]):
        if (b.img_h, b.img_w, b.img_c) != (a.grid_r, a.grid_c, a.filters // a.pool_group):
            raise ValueError(f"layer {b.name} input {(b.img_h, b.img_w, b.img_c)} does not match the previous "
                             f"layer's output {(a.grid_r, a.grid_c, a.filters // a.pool_group)}")
        if b.batch != a.batch:
            raise ValueError("all layers of a stack share the mini-batch size")


class Stack:
    def __init__(self, cfg: StackConfig, precision=lcae.BF16, seed=0, stream=None):
        check_chain(cfg)
        self.cfg = cfg
        self.stream = stream
        self.layers = []
        for i, s in enumerate(cfg.shapes):
            L = lcae.Layer(lcae.make_config(s, precision=precision, stream=stream))
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

    def input_of(self, l, x):
        """The input of layer l: the images for l = 0, else LCN(code of layer l-1 of the input of l-1)."""
        for i in range(l):
            x = self._lcn(self._code(i, x))
        return x

    def forward(self, x):
        """Top-layer code of a batch (the 'activation values' of PAPER.md:156)."""
        return self._code(len(self.layers) - 1, self.input_of(len(self.layers) - 1, x))

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
