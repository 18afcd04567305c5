"""Pipelined layer-wise training over the C ABI: the degenerate pipeline reproduces
plain layer-wise training bit for bit, and the staleness bound holds."""
import numpy as np
import pytest

from paper_1502_03409_b200.inputs import make_images
from paper_1502_03409_b200.stack import desk_stack

pytestmark = pytest.mark.gpu


def _params(L):
    s = L.shape
    W = np.zeros((s.fields, s.filters, s.n), np.float32)
    a = np.zeros(s.fields, np.float32)
    b = np.zeros((s.fields, s.n), np.float32)
    L.get_params(W, a, b)
    return W, a, b


def test_degenerate_pipeline_bitwise_equals_layerwise_gpu():
    import torch
    from paper_1502_03409_b200.pipeline import LcaeEngine, PipelineConfig, run_pipeline
    shapes = desk_stack(batch=16).shapes
    blocks = [torch.from_numpy(make_images(shapes[0], seed=200 + i)).cuda() for i in range(3)]
    pc = PipelineConfig(warmup_blocks=10 ** 6, sync_period_blocks=2, stabilization_window=2, epochs_per_layer=2)
    eng = LcaeEngine()
    ref = LcaeEngine()
    try:
        trainers, log = run_pipeline(eng, shapes, blocks, pc)
        # reference: plain greedy layer-wise loops, each layer fed by a snapshot of the finished layer below
        r = [ref.make_layer(s, i) for i, s in enumerate(shapes)]
        snaps = []
        for l in range(len(shapes)):
            for t in range(6):
                x = blocks[t % 3]
                for i in range(l):
                    x = ref.lcn(ref.encode(snaps[i], x))
                ref.step(r[l], x)
            if l + 1 < len(shapes):
                snap = ref.make_layer(shapes[l], 99)
                ref.copy_params(r[l], snap)
                snaps.append(snap)
        for a, b in zip(trainers, r):
            for u, v in zip(_params(a), _params(b)):
                assert np.array_equal(u, v)
        assert [rec.layer for rec in log.records] == [0] * 6 + [1] * 6 + [2] * 6
    finally:
        eng.close()
        ref.close()


def test_pipelined_run_staleness_gpu():
    import torch
    from paper_1502_03409_b200.pipeline import LcaeEngine, PipelineConfig, run_pipeline
    shapes = desk_stack(batch=16).shapes
    blocks = [torch.from_numpy(make_images(shapes[0], seed=300 + i)).cuda() for i in range(5)]
    pc = PipelineConfig(warmup_blocks=4, sync_period_blocks=3, stabilization_window=2, stabilization_rel_tol=10.0,
                        epochs_per_layer=4)
    eng = LcaeEngine()
    try:
        _, log = run_pipeline(eng, shapes, blocks, pc)
    finally:
        eng.close()
    for l in (1, 2):
        recs = [r for r in log.records if r.layer == l]
        assert recs and [r.block for r in recs] == list(range(len(recs)))
        assert all(r.staleness <= pc.sync_period_blocks for r in recs)
        assert all(np.isfinite(r.objective) for r in recs)


def test_concurrent_streams_equal_sequential_schedule():
    """StreamEngine (one CUDA stream per layer instance, trainer and forwarder running simultaneously,
    PAPER.md:111) makes the same decisions and the same parameter bits as the one-stream schedule."""
    import time

    import torch
    from paper_1502_03409_b200.pipeline import LcaeEngine, PipelineConfig, StreamEngine, run_pipeline
    shapes = desk_stack(batch=16).shapes
    blocks = [torch.from_numpy(make_images(shapes[0], seed=400 + i)).cuda() for i in range(5)]
    pc = PipelineConfig(warmup_blocks=4, sync_period_blocks=3, stabilization_window=2, stabilization_rel_tol=10.0,
                        epochs_per_layer=6)
    out = {}
    for name, cls in (("sequential", LcaeEngine), ("streams", StreamEngine)):
        eng = cls()
        try:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            trainers, log = run_pipeline(eng, shapes, blocks, pc)
            torch.cuda.synchronize()
            out[name] = ([_params(L) for L in trainers], log, time.perf_counter() - t0)
        finally:
            eng.close()
    (pa, la, ta), (pb, lb, tb) = out["sequential"], out["streams"]
    for x, y in zip(pa, pb):
        for u, v in zip(x, y):
            assert np.array_equal(u, v)
    assert la.lines() == lb.lines()
    assert any(r.layer == 2 for r in lb.records)
    print(f"pipeline wall time: one stream {ta * 1e3:.1f} ms, concurrent streams {tb * 1e3:.1f} ms "
          f"({len(lb.records)} layer-blocks)")
