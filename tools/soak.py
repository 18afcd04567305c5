"""Dev tool: a long training run on synthetic data (stability of the lazy sigma projection and the loss over many
steps): prints J every `every` steps and the min / max row norm of the returned W at the end.
usage: python tools/soak.py [config] [steps] [every]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_03409_b200 import lcae  # noqa: E402
from paper_1502_03409_b200.inputs import CONFIGS, EXTRA_CONFIGS, make_images  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
every = int(sys.argv[3]) if len(sys.argv) > 3 else 100
shape = {**CONFIGS, **EXTRA_CONFIGS}[name]
L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16, seed=3))
pool = [torch.from_numpy(make_images(shape, seed=40 + i, bf16_round=False)).cuda() for i in range(8)]
t0 = time.perf_counter()
for t in range(steps):
    want = (t % every == 0) or t == steps - 1
    J = L.step(pool[t % len(pool)], None, want_loss=want)
    if want:
        print(f"{name} step {t:6d}  J {J:.6e}  ({time.perf_counter() - t0:.1f} s)", flush=True)
L.sync()
f = min(4, shape.fields)
W = np.zeros((f, shape.filters, shape.n), np.float32)
a = np.zeros(f, np.float32)
b = np.zeros((f, shape.n), np.float32)
L.get_field_params(0, f, W, a, b)
nrm = np.linalg.norm(W.astype(np.float64), axis=-1)
print(f"{name}: {steps} steps, row norms of fields 0..{f - 1} in [{nrm.min():.9f}, {nrm.max():.9f}], "
      f"alpha {a.min():.4g}..{a.max():.4g}, reinit {L.counters()[1]}")
L.close()
