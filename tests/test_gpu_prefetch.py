"""lcae_prefetch_input: a step fed from a prefetched host batch equals the step fed from the device copy of the
same batch bit for bit (the overlap only moves the copy to another stream)."""
import numpy as np
import pytest

from paper_1502_03409_b200.inputs import CONFIGS, make_images, make_params

pytestmark = pytest.mark.gpu


def test_prefetched_steps_equal_device_input_steps():
    import torch
    from paper_1502_03409_b200 import lcae
    shape = CONFIGS["c2"]
    W, a, b = make_params(shape, seed=0)
    xs = [make_images(shape, seed=1, index=i) for i in range(3)]
    res = []
    for mode in ("device", "prefetch"):
        L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16))
        try:
            L.set_params(W, a, b)
            losses = []
            if mode == "device":
                for x in xs:
                    losses.append(L.step(torch.from_numpy(x).cuda(), None))
            else:
                hosts = [torch.from_numpy(x).pin_memory() for x in xs]
                L.prefetch_input(hosts[0])
                for i, h in enumerate(hosts):
                    L.step(h, None, want_loss=False)
                    if i + 1 < len(hosts):
                        L.prefetch_input(hosts[i + 1])
                    jr, js = L.last_loss()
                    losses.append(jr + js)
            Wn, an, bn = np.zeros_like(W), np.zeros_like(a), np.zeros_like(b)
            L.get_params(Wn, an, bn)
            res.append((losses, Wn, an, bn))
        finally:
            L.close()
    (l1, W1, a1, b1), (l2, W2, a2, b2) = res
    assert l1 == l2
    assert np.array_equal(W1, W2) and np.array_equal(a1, a2) and np.array_equal(b1, b2)
