"""Dev tool: run `steps` bf16 training steps of a config (default c3) -- the short command profiled under ncu.
usage: python tools/prof_once.py [c3|c2|c1|c3p|c15b] [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1502_03409_b200 import lcae  # noqa: E402
from paper_1502_03409_b200.inputs import CONFIGS, EXTRA_CONFIGS, make_images, make_params  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
shape = {**CONFIGS, **EXTRA_CONFIGS}[cfg_name]
L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16))
W, a, b = make_params(shape, seed=0)
L.set_params(W, a, b)
x = torch.from_numpy(make_images(shape, seed=1)).cuda()
for _ in range(steps):
    L.step(x, None, want_loss=False)
torch.cuda.synchronize()
print("ok", cfg_name, steps)
