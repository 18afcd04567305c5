"""Dev: exercise every entry point once on small shapes (step / forward / encode / prefetch / top-K / LCN /
region_add) -- the program run under compute-sanitizer memcheck."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_03409_b200 import lcae  # noqa: E402
from paper_1502_03409_b200.inputs import CONFIGS, LayerShape, make_images, make_params  # noqa: E402

# every step-kernel variant: lean (keep_grads 0), full (keep_grads 1 / momentum), generic (forward / encode);
# one and two CTAs per cluster; one field per CTA and (LCAE_DEV_MAX_CLUSTERS) several fields per CTA
CASES = [(CONFIGS["c1"], lcae.BF16, 1, 0.0, None), (CONFIGS["c1"], lcae.BF16, 0, 0.0, "2"),
         (LayerShape("cl2", 20, 20, 3, 8, 8, 4, 32, 2, 200), lcae.BF16, 1, 0.0, None),
         (LayerShape("cl2", 20, 20, 3, 8, 8, 4, 32, 2, 200), lcae.BF16, 0, 0.9, "2"),
         (LayerShape("c3tiny", 22, 22, 3, 18, 18, 2, 128, 1, 256), lcae.BF16, 0, 0.0, None),
         (LayerShape("c3tiny", 22, 22, 3, 18, 18, 2, 128, 1, 256), lcae.BF16, 1, 0.0, "2"),
         (CONFIGS["c1"], lcae.FP32, 1, 0.0, None)]
if len(sys.argv) > 1:
    CASES = CASES[:int(sys.argv[1])]
for shape, prec, keep, mu, cap in CASES:
    if cap:
        os.environ["LCAE_DEV_MAX_CLUSTERS"] = cap
    else:
        os.environ.pop("LCAE_DEV_MAX_CLUSTERS", None)
    shape = shape.replace(momentum=mu)
    print(shape.name, "bf16" if prec else "fp32", "keep" if keep else "lean", "mu", mu, "cap", cap, flush=True)
    L = lcae.Layer(lcae.make_config(shape, precision=prec, keep_grads=bool(keep)))
    W, a, b = make_params(shape, seed=0)
    L.set_params(W, a, b)
    x = torch.from_numpy(make_images(shape, seed=1)).cuda()
    xh = x.cpu().pin_memory()
    pooled = torch.empty((shape.batch, L.grid_r, L.grid_c, shape.filters // shape.pool_group), device="cuda")
    L.forward(x, pooled)
    L.encode(x, pooled)
    L.prefetch_input(xh)
    dx = torch.empty_like(x)
    L.step(xh, dx)
    L.step(x, None)
    units = pooled[0].numel()
    vals = torch.empty((units, 5), device="cuda")
    ids = torch.empty((units, 5), dtype=torch.int32, device="cuda")
    lcae.topk_init(vals, ids)
    lcae.topk_update(pooled.reshape(shape.batch, units), vals, ids, 0)
    if L.grid_r >= 3:
        y = torch.empty_like(pooled)
        lcae.lcn(pooled, y, torch.empty(2 * pooled.numel(), device="cuda"), 3, 1e-4)
    torch.cuda.synchronize()
    L.close()
print("sanitize run ok")
