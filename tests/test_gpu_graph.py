"""CUDA-graph replay of the training step (launch-bound small configs): a step captured once and replayed must
equal eager steps bit for bit on the parameters (the step counter that seeds degenerate-row re-initialisation
lives on the device, so replays stay exact)."""
import numpy as np
import pytest

from paper_1502_03409_b200.inputs import CONFIGS, make_images, make_params

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_graph_replay_equals_eager_steps(name):
    import torch
    from paper_1502_03409_b200 import lcae
    shape = CONFIGS[name]
    W, a, b = make_params(shape, seed=0)
    x = torch.from_numpy(make_images(shape, seed=1)).cuda()
    s = torch.cuda.Stream()
    outs = []
    for mode in ("eager", "graph"):
        with torch.cuda.stream(s):
            L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16, stream=s.cuda_stream))
            try:
                L.set_params(W, a, b)
                torch.cuda.synchronize()
                if mode == "eager":
                    for _ in range(3):
                        L.step(x, None, want_loss=False)
                else:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=s):
                        L.step(x, None, want_loss=False)
                    torch.cuda.synchronize()
                    # capture does not execute: three replays are three steps
                    for _ in range(3):
                        g.replay()
                torch.cuda.synchronize()
                Wn, an, bn = np.zeros_like(W), np.zeros_like(a), np.zeros_like(b)
                L.get_params(Wn, an, bn)
                outs.append((Wn, an, bn, L.counters()[0]))
            finally:
                L.close()
    (W1, a1, b1, s1), (W2, a2, b2, s2) = outs
    assert np.array_equal(W1, W2) and np.array_equal(a1, a2) and np.array_equal(b1, b2)
    assert s1 == s2 == 3
