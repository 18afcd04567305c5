"""Dev probe: loss trajectory of repeated bf16 steps (divergence check) for configs at a given lr scale.
usage: python tools/c2probe.py LRSCALE cfg [cfg...]   (lr = LRSCALE / batch; 0 keeps the config's lr)"""
import math
import sys

import torch

sys.path.insert(0, '.')
from paper_1502_03409_b200 import lcae  # noqa: E402
from paper_1502_03409_b200.inputs import CONFIGS, make_images, make_params  # noqa: E402

scale = float(sys.argv[1])
for name in sys.argv[2:]:
    shape = CONFIGS[name]
    if scale:
        shape = shape.replace(lr=scale / shape.batch)
    L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16))
    W, a, b = make_params(shape, seed=0)
    L.set_params(W, a, b)
    pool = [torch.from_numpy(make_images(shape, seed=1, index=i)).cuda() for i in range(4)]
    for t in range(301):
        try:
            J = L.step(pool[t % 4], None, want_loss=True)
        except lcae.LcaeError as e:
            print(name, shape.lr, t, "ERROR", e, flush=True)
            break
        if t % 50 == 0:
            print(name, shape.lr, t, J, L.counters(), flush=True)
    L.close()
