"""Model parallelism over receptive fields.

"The training algorithm is model parallel ... distributing the model across the GPUs";
"Communication within the algorithm occurs when a layer's input (or output) field spans multiple GPUs"
(PAPER.md:117); "Global communication is minimized by using untied local receptive fields, and allowing
receptive fields to be trained independently".

The field grid is cut into contiguous rectangular tiles, one per rank, in row-major rank order (SPEC.md:347-355
partition_fields).  Every rank owns the untied weights of its fields (no weight or gradient collective ever
exists) and a rectangle of image pixels.  One step on a rank:

  1. input halo exchange: the rank's fields need pixels  need = [R0*s, (R1-1)*s + rf_h) x [C0*s, ...),
     a superset of its owned pixels; the missing strips are received from the owners (P2P sends/recvs);
  2. lcae_step on the extended region (the C ABI: a layer whose image is the region, field ids offset);
  3. input-gradient return: the dX of pixels owned by a neighbour is sent back and overlap-added by the owner
     (lcae_region_add on the GPU);
  4. (optional) loss all-reduce (sum).

On GPUs this whole step runs INSIDE the library (include/lcae.h world_size > 1, csrc/mp.cu: NCCL send / recv of
bf16 halos overlapping the interior fields, fp32 dX returns, loss all-reduce); bench.py uses that path and
tests/test_abi_cpu.py checks that the library's tiling (lcae_geometry own_px / own_fields) equals plan() below.
This module is the host-side statement of the same plan, and HaloExchange is the same exchange written over
torch.distributed point-to-point ops: tests/test_parallel_cpu.py drives it over gloo (world_size 2 and 4, CPU)
with the oracle as the per-rank engine. Byte counts of every exchange are recorded and checked against the
static prediction, which the library's exchange buffers also match (tests/test_gpu_mp.py).
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Dict, List, Optional, Tuple

Region = Tuple[int, int, int, int]   # y0, y1, x0, x1 (half-open)


def factor(world: int) -> Tuple[int, int]:
    """tiles_r x tiles_c == world, as square as possible with tiles_r >= tiles_c (1x1, 2x1, 2x2, 4x2, ...)."""
    best = (world, 1)
    for tc in range(1, world + 1):
        if world % tc == 0:
            tr = world // tc
            if tr >= tc and (tr - tc) < (best[0] - best[1]):
                best = (tr, tc)
    return best


def split(n: int, parts: int) -> List[Tuple[int, int]]:
    """Balanced contiguous split of range(n) into `parts` pieces (the first n % parts get one more)."""
    if parts > n:
        raise ValueError(f"cannot split {n} field rows/cols over {parts} tiles (SPEC.md:351)")
    base, extra = divmod(n, parts)
    out, a = [], 0
    for p in range(parts):
        b = a + base + (1 if p < extra else 0)
        out.append((a, b))
        a = b
    return out


def intersect(a: Region, b: Region) -> Optional[Region]:
    y0, y1 = max(a[0], b[0]), min(a[1], b[1])
    x0, x1 = max(a[2], b[2]), min(a[3], b[3])
    return (y0, y1, x0, x1) if (y0 < y1 and x0 < x1) else None


@dataclasses.dataclass(frozen=True)
class Tile:
    rank: int
    tr: int
    tc: int
    fields_r: Tuple[int, int]   # [R0, R1) field rows
    fields_c: Tuple[int, int]   # [C0, C1) field cols
    need: Region                # pixels read by this tile's fields
    own: Region                 # pixels this rank owns (input and gradient)

    @property
    def grid(self) -> Tuple[int, int]:
        return self.fields_r[1] - self.fields_r[0], self.fields_c[1] - self.fields_c[0]

    @property
    def need_hw(self) -> Tuple[int, int]:
        return self.need[1] - self.need[0], self.need[3] - self.need[2]

    @property
    def own_hw(self) -> Tuple[int, int]:
        return self.own[1] - self.own[0], self.own[3] - self.own[2]


def plan(shape, world: int) -> List[Tile]:
    """Contiguous 2D tiling of the field grid over `world` ranks (row-major rank order)."""
    tr_n, tc_n = factor(world)
    rows, cols = split(shape.grid_r, tr_n), split(shape.grid_c, tc_n)
    s = shape.stride
    tiles = []
    for rank in range(world):
        tr, tc = divmod(rank, tc_n)
        (R0, R1), (C0, C1) = rows[tr], cols[tc]
        need = (R0 * s, (R1 - 1) * s + shape.rf_h, C0 * s, (C1 - 1) * s + shape.rf_w)
        own = (R0 * s, shape.img_h if tr == tr_n - 1 else R1 * s, C0 * s, shape.img_w if tc == tc_n - 1 else C1 * s)
        tiles.append(Tile(rank, tr, tc, (R0, R1), (C0, C1), need, own))
    return tiles


def predicted_bytes(shape, tiles: List[Tile], elem_bytes: int = 4) -> Dict[str, int]:
    """Static prediction of every exchange: sum over ordered pairs (src != dst) of the
    region sizes x batch x channels x element size."""
    halo = ret = 0
    per_px = shape.batch * shape.img_c * elem_bytes
    for a in tiles:
        for b in tiles:
            if a.rank == b.rank:
                continue
            r = intersect(b.need, a.own)   # a sends input pixels to b
            if r:
                halo += (r[1] - r[0]) * (r[3] - r[2]) * per_px
            r = intersect(a.need, b.own)   # a returns dX of b's pixels to b
            if r:
                ret += (r[1] - r[0]) * (r[3] - r[2]) * per_px
    return {"halo_in": halo, "dx_return": ret}


def _view(t, region: Region, base: Region):
    """Slice of an NHWC tensor `t` covering `base`, restricted to `region` (global pixel coordinates)."""
    return t[:, region[0] - base[0]:region[1] - base[0], region[2] - base[2]:region[3] - base[2], :]


class HaloExchange:
    """Input-halo gather and dX return for one rank, over torch.distributed P2P (NCCL or gloo)."""

    def __init__(self, tiles: List[Tile], rank: int, dist=None):
        if dist is None:
            import torch.distributed as dist
        self.dist = dist
        self.tiles = tiles
        self.me = tiles[rank]
        self.peers = [t for t in tiles if t.rank != rank]
        self.bytes_sent = {"halo_in": 0, "dx_return": 0}
        self.messages = 0

    def _exchange(self, sends, recvs, kind):
        import torch
        ops = []
        for peer, buf in sends:
            ops.append(self.dist.P2POp(self.dist.isend, buf, peer))
            self.bytes_sent[kind] += buf.numel() * buf.element_size()
            self.messages += 1
        for peer, buf in recvs:
            ops.append(self.dist.P2POp(self.dist.irecv, buf, peer))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        return torch

    def gather_input(self, x_own, x_ext):
        """x_own: NHWC over me.own; fills x_ext (NHWC over me.need) with own pixels and the received halo."""
        me = self.me
        mine = intersect(me.need, me.own)
        if mine:
            _view(x_ext, mine, me.need).copy_(_view(x_own, mine, me.own))
        sends, recvs, places = [], [], []
        for p in self.peers:
            r = intersect(p.need, me.own)
            if r:
                sends.append((p.rank, _view(x_own, r, me.own).contiguous()))
            r = intersect(me.need, p.own)
            if r:
                buf = x_ext.new_empty((x_ext.shape[0], r[1] - r[0], r[3] - r[2], x_ext.shape[3]))
                recvs.append((p.rank, buf))
                places.append((r, buf))
        self._exchange(sends, recvs, "halo_in")
        for r, buf in places:
            _view(x_ext, r, me.need).copy_(buf)
        return x_ext

    def return_dx(self, dx_ext, dx_own, add_region: Callable):
        """dx_ext: NHWC over me.need (partial sums of my fields); dx_own receives the full gradient of my
        pixels: my own contribution plus the neighbours' returned partials, added with add_region(dst, src,
        y0, x0) (lcae_region_add on the GPU)."""
        me = self.me
        dx_own.zero_()
        mine = intersect(me.need, me.own)
        if mine:
            add_region(dx_own, _view(dx_ext, mine, me.need).contiguous(), mine[0] - me.own[0], mine[2] - me.own[2])
        sends, recvs, places = [], [], []
        for p in self.peers:
            r = intersect(me.need, p.own)
            if r:
                sends.append((p.rank, _view(dx_ext, r, me.need).contiguous()))
            r = intersect(p.need, me.own)
            if r:
                buf = dx_own.new_empty((dx_own.shape[0], r[1] - r[0], r[3] - r[2], dx_own.shape[3]))
                recvs.append((p.rank, buf))
                places.append((r, buf))
        self._exchange(sends, recvs, "dx_return")
        for r, buf in places:
            add_region(dx_own, buf, r[0] - me.own[0], r[2] - me.own[2])
        return dx_own


def tile_shape(shape, tile: Tile):
    """The LayerShape of the rank-local layer: its image is the tile's `need` region."""
    h, w = tile.need_hw
    return shape.replace(name=f"{shape.name}-r{tile.rank}", img_h=h, img_w=w)
