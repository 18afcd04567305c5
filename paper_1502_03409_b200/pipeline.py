"""Pipelined layer-wise training (PAPER.md:111 and Fig. 3).

Two instances of layer L run "simultaneously": a trainer that keeps training on the data blocks, and a
forwarder that propagates data to layer L+1 with a snapshot of the trainer's parameters, re-synchronised every
`sync_period_blocks` trainer blocks ("periodically synchronized with the layer L instance that continued
training"). Layer L+1 starts once layer L has trained `warmup_blocks` blocks and its objective has stabilised,
and replays the data from block 0 (Fig. 3). A deterministic sequential scheduler interleaves the tasks (one
block per active trainer per tick, bottom layer first), so a run is reproducible bit for bit.

The scheduler is host logic over an engine with the layer operations; `LcaeEngine` runs them on the GPU
through the C ABI (lcae_step / lcae_encode / lcae_lcn / parameter copies between layer instances), one call
after the other on one stream. `StreamEngine` runs them SIMULTANEOUSLY ("two instances of the
layer L are run simultaneously"): every layer instance (trainer or forwarder) owns a CUDA stream, a tick
enqueues every active layer's work without waiting (forwarder chains on the forwarders' streams, trainer steps
on the trainers' streams, ordered only by their data dependencies through CUDA events), and the host reads the
losses once per tick -- except when a start decision needs the current objective. The decisions, and therefore
every parameter bit, are those of the sequential schedule (tests/test_gpu_pipeline.py).
"""
from dataclasses import dataclass, field
from typing import List, Optional


@dataclass
class PipelineConfig:
    warmup_blocks: int = 1000          # PAPER.md:111 "an initial set of data blocks (in our case, 1000)"
    sync_period_blocks: int = 5
    stabilization_window: int = 50
    stabilization_rel_tol: float = 0.01
    epochs_per_layer: int = 1          # SPEC.md:327 open question: a fixed epoch count per layer

    def __post_init__(self):
        if self.warmup_blocks < 1 or self.sync_period_blocks < 1 or self.stabilization_window < 2:
            raise ValueError("warmup_blocks >= 1, sync_period_blocks >= 1, stabilization_window >= 2")


def stabilized(history, window, rel_tol):
    """two-window relative-mean test."""
    if len(history) < 2 * window:
        return False
    last = sum(history[-window:]) / window
    prev = sum(history[-2 * window:-window]) / window
    return abs(last - prev) / max(abs(prev), 1e-12) < rel_tol


@dataclass
class LogRecord:
    layer: int
    block: int
    objective: float
    snapshot_versions: tuple      # versions of the upstream forwarder snapshots used for this block's input
    staleness: int                # max over upstream boundaries of (trainer blocks done - snapshot source block)


@dataclass
class TrainLog:
    records: List[LogRecord] = field(default_factory=list)

    def lines(self):
        return [f"{r.layer}\t{r.block}\t{r.objective!r}\t{','.join(map(str, r.snapshot_versions))}\t{r.staleness}"
                for r in self.records]


@dataclass
class _Boundary:          # the forwarder of layer l (feeds layer l + 1)
    handle: object
    version: int = 0
    source_block: int = 0


def run_pipeline(engine, shapes, blocks, cfg: PipelineConfig, seed=0):
    """Train len(shapes) layers on `blocks` (a list of input batches) with the Fig. 3 pipeline.
    Returns (trainer handles, TrainLog)."""
    n = len(shapes)
    total = cfg.epochs_per_layer * len(blocks)
    if cfg.warmup_blocks > total and n > 1:
        pass   # degenerate pipeline: layer l+1 starts only after layer l finished
    trainers = [engine.make_layer(s, seed + i) for i, s in enumerate(shapes)]
    fwd: List[Optional[_Boundary]] = [None] * n
    done = [0] * n            # blocks trained per layer
    hist = [[] for _ in range(n)]
    active = [True] + [False] * (n - 1)
    log = TrainLog()

    def sync(l):
        b = fwd[l]
        if b is None:
            b = fwd[l] = _Boundary(engine.make_layer(shapes[l], seed + l))
        engine.copy_params(trainers[l], b.handle)      # immutable snapshot: the forwarder never trains
        b.version += 1
        b.source_block = done[l]

    def input_of(l, x):
        if getattr(engine, "concurrent", False):
            return engine.chain(l, [fwd[i].handle for i in range(l)], x, trainers[l])
        for i in range(l):
            x = engine.lcn(engine.encode(fwd[i].handle, x))
        return x

    concurrent = getattr(engine, "concurrent", False)
    if concurrent:
        engine.begin()   # inputs created on other streams are complete before the layer streams read them
    pending = []   # (layer, record, lazy loss) of this tick, resolved in order

    def resolve(upto_layer=None):
        keep = []
        for l_, rec, h in pending:
            if upto_layer is None or l_ == upto_layer:
                rec.objective = engine.loss(h)
                hist[l_].append(rec.objective)
            else:
                keep.append((l_, rec, h))
        pending[:] = keep

    while any(active[l] and done[l] < total for l in range(n)):
        for l in range(n):                              # one block per active trainer, bottom layer first
            if not active[l] or done[l] >= total:
                continue
            x = input_of(l, blocks[done[l] % len(blocks)])
            versions = tuple(fwd[i].version for i in range(l))
            stale = max([done[i] - fwd[i].source_block for i in range(l)], default=0)
            rec = LogRecord(l, done[l], None, versions, stale)
            log.records.append(rec)
            if concurrent:   # enqueue only; the objective is read at the end of the tick (or when needed)
                pending.append((l, rec, engine.step_async(trainers[l], x)))
            else:
                rec.objective = engine.step(trainers[l], x)
                hist[l].append(rec.objective)
            done[l] += 1
            if l + 1 < n:
                started = active[l + 1]
                finished = done[l] >= total
                if not started and done[l] >= cfg.warmup_blocks:
                    resolve(l)   # the start test needs this block's objective
                ready = done[l] >= cfg.warmup_blocks and stabilized(hist[l], cfg.stabilization_window,
                                                                   cfg.stabilization_rel_tol)
                if not started and (ready or finished):
                    sync(l)
                    active[l + 1] = True
                elif started and (done[l] - fwd[l].source_block >= cfg.sync_period_blocks or finished):
                    sync(l)
        resolve()
    return trainers, log


class LcaeEngine:
    """Layer operations on the GPU through the C ABI (bf16 tcgen05 path by default)."""

    def __init__(self, precision=None, lcn_window=3, lcn_floor=1e-4, stream=None):
        from . import lcae
        self.lcae = lcae
        self.precision = lcae.BF16 if precision is None else precision
        self.window, self.floor, self.stream = lcn_window, lcn_floor, stream
        self.layers = []

    def make_layer(self, shape, seed):
        from .inputs import make_params
        L = self.lcae.Layer(self.lcae.make_config(shape, precision=self.precision, stream=self.stream))
        W, a, b = make_params(shape, seed=seed)
        L.set_params(W, a, b)
        L.shape = shape
        self.layers.append(L)
        return L

    def step(self, L, x):
        return L.step(x, None)

    def encode(self, L, x):
        import torch
        s = L.shape
        p = torch.empty((s.batch, s.grid_r, s.grid_c, s.filters // s.pool_group), dtype=torch.float32,
                        device=x.device)
        L.encode(x, p, want_loss=False)
        return p

    def lcn(self, p):
        import torch
        y = torch.empty_like(p)
        self.lcae.lcn(p, y, torch.empty(2 * p.numel(), dtype=torch.float32, device=p.device), self.window,
                      self.floor, self.stream)
        return y

    def copy_params(self, src, dst):
        import torch
        s = src.shape
        W = torch.empty((s.fields, s.filters, s.n), dtype=torch.float32, device="cuda")
        a = torch.empty((s.fields,), dtype=torch.float32, device="cuda")
        b = torch.empty((s.fields, s.n), dtype=torch.float32, device="cuda")
        src.get_params(W, a, b)
        dst.set_params(W, a, b)

    def close(self):
        for L in self.layers:
            L.close()
        self.layers = []


class StreamEngine(LcaeEngine):
    """Concurrent execution of the Fig. 3 pipeline: one CUDA stream per layer instance, dependencies through
    events only ("run simultaneously"). Trainer l's step, forwarder l's encode for layer l+1 and
    the other layers' work of the same tick overlap on the GPU."""
    concurrent = True

    def __init__(self, precision=None, lcn_window=3, lcn_floor=1e-4):
        super().__init__(precision, lcn_window, lcn_floor)
        self.bufs = {}

    def make_layer(self, shape, seed):
        import torch
        from .inputs import make_params
        st = torch.cuda.Stream()
        L = self.lcae.Layer(self.lcae.make_config(shape, precision=self.precision, stream=st.cuda_stream))
        W, a, b = make_params(shape, seed=seed)
        L.set_params(W, a, b)
        L.shape, L.stream, L.done = shape, st, None
        self.layers.append(L)
        return L

    def _buf(self, key, shape):
        import torch
        if key not in self.bufs:
            self.bufs[key] = torch.empty(shape, dtype=torch.float32, device="cuda")
        return self.bufs[key]

    def begin(self):
        import torch
        torch.cuda.synchronize()

    def chain(self, l, fwds, x, consumer):
        """Layer l's input: x through forwarders 0..l-1 (encode + LCN on each forwarder's stream), into buffers
        owned by layer l; returns (tensor, event). The chain starts after layer l's previous step (its buffers
        are free again)."""
        import torch
        ev = None
        for i, F in enumerate(fwds):
            s = F.shape
            st = F.stream
            if i == 0 and consumer.done is not None:
                st.wait_event(consumer.done)
            if ev is not None:
                st.wait_event(ev)
            code = self._buf((l, i, "p"), (s.batch, s.grid_r, s.grid_c, s.filters // s.pool_group))
            y = self._buf((l, i, "y"), code.shape)
            scratch = self._buf((l, i, "s"), (2 * code.numel(),))
            with torch.cuda.stream(st):
                F.encode(x, code, want_loss=False)
                self.lcae.lcn(code, y, scratch, self.window, self.floor, st.cuda_stream)
            ev = st.record_event()
            x = y
        return (x, ev)

    def step_async(self, L, xe):
        x, ev = xe if isinstance(xe, tuple) else (xe, None)
        if ev is not None:
            L.stream.wait_event(ev)
        L.step(x, None, want_loss=False)
        L.done = L.stream.record_event()
        return L

    def loss(self, L):
        jr, js = L.last_loss()   # synchronises this layer's stream only
        return jr + js

    def copy_params(self, src, dst):
        # the snapshot is taken after the trainer's enqueued steps (get_params runs on, and waits for, the
        # trainer's stream) and lands before the forwarder's next encode (set_params waits for its stream)
        super().copy_params(src, dst)
