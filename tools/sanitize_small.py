"""Sanitizer substitute (compute-sanitizer is closed on this pool): exercise every entry point and
kernel variant on small shapes with
  * LCAE_LIB=liblcae_checked.so  -- mbarrier watchdogs (a stuck phase traps with its barrier instead of hanging)
                                    and device bounds checks on every global write / TMA coordinate;
  * LCAE_DEV_POISON=1            -- every allocation starts as 0xFF bytes (NaN): a read before write (initcheck)
                                    poisons the results, which are compared with the fp64 oracle;
  * LCAE_DEV_CANARY=1            -- every allocation has a 4 KB 0xA5 tail, verified after each case (memcheck
                                    for out-of-bounds writes);
and repeats each training step to check that the parameters are bitwise reproducible (a shared-memory or barrier
race shows up as run-to-run differences; racecheck / synccheck substitute).
usage: LCAE_LIB=... LCAE_DEV_POISON=1 LCAE_DEV_CANARY=1 python tools/sanitize_small.py [n_cases]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import lcae_oracle as O  # noqa: E402
from paper_1502_03409_b200 import lcae  # noqa: E402
from paper_1502_03409_b200.inputs import CONFIGS, LayerShape, make_images, make_params  # noqa: E402

lcae.lib.lcae_dev_check_canaries.restype = C.c_int
lcae.lib.lcae_dev_check_canaries.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]

# every step-kernel variant: lean (keep_grads 0), full (keep_grads 1 / momentum), generic (forward / encode);
# one and two CTAs per cluster; one field per CTA and (LCAE_DEV_MAX_CLUSTERS) several fields per CTA; fp32; the
# general bf16 path's GEMM epilogues
CASES = [(CONFIGS["c1"], lcae.BF16, 1, 0.0, None), (CONFIGS["c1"], lcae.BF16, 0, 0.0, "2"),
         (LayerShape("cl2", 20, 20, 3, 8, 8, 4, 32, 2, 200), lcae.BF16, 1, 0.0, None),
         (LayerShape("cl2", 20, 20, 3, 8, 8, 4, 32, 2, 200), lcae.BF16, 0, 0.9, "2"),
         (LayerShape("c3tiny", 22, 22, 3, 18, 18, 2, 128, 1, 256), lcae.BF16, 0, 0.0, None),
         (LayerShape("c3tiny", 26, 26, 3, 18, 18, 2, 128, 1, 256), lcae.BF16, 1, 0.0, "2"),
         (LayerShape("ragged", 21, 25, 2, 5, 7, 2, 24, 4, 37), lcae.BF16, 1, 0.0, "3"),
         (CONFIGS["c1"], lcae.FP32, 1, 0.0, None),
         # the general bf16 path (k > 128): lean SGD epilogue, and SGDF with momentum
         (LayerShape("wide", 21, 25, 2, 5, 7, 2, 200, 4, 37), lcae.BF16, 0, 0.0, None),
         (LayerShape("c3p-small", 24, 24, 3, 16, 16, 4, 384, 1, 192), lcae.BF16, 1, 0.9, None)]
if len(sys.argv) > 1:
    CASES = CASES[:int(sys.argv[1])]


def canaries(L):
    bad, n = C.c_int64(), C.c_int64()
    lcae.check(lcae.lib.lcae_dev_check_canaries(L.h, C.byref(bad), C.byref(n)))
    return bad.value, n.value


def geo(s):
    return dict(img_h=s.img_h, img_w=s.img_w, img_c=s.img_c, rf_h=s.rf_h, rf_w=s.rf_w, stride=s.stride,
                pool_group=s.pool_group, lam=s.lam, eps=s.eps)


def params_after(shape, prec, keep, X, W, a, b, steps):
    L = lcae.Layer(lcae.make_config(shape, precision=prec, keep_grads=bool(keep)))
    L.set_params(W, a, b)
    for _ in range(steps):
        L.step(X, None)
    W1, a1, b1 = np.zeros_like(W), np.zeros_like(a), np.zeros_like(b)
    L.get_params(W1, a1, b1)
    L.close()
    return W1, a1, b1


for shape, prec, keep, mu, cap in CASES:
    if cap:
        os.environ["LCAE_DEV_MAX_CLUSTERS"] = cap
    else:
        os.environ.pop("LCAE_DEV_MAX_CLUSTERS", None)
    shape = shape.replace(momentum=mu)
    print(shape.name, "bf16" if prec else "fp32", "keep" if keep else "lean", "mu", mu, "cap", cap, flush=True)
    L = lcae.Layer(lcae.make_config(shape, precision=prec, keep_grads=bool(keep)))
    W, a, b = make_params(shape, seed=0)
    b = (0.05 * np.random.default_rng(3).standard_normal(b.shape)).astype(np.float32)
    L.set_params(W, a, b)
    Xh = make_images(shape, seed=1, bf16_round=False)
    x = torch.from_numpy(Xh).cuda()
    xh = x.cpu().pin_memory()
    pooled = torch.empty((shape.batch, L.grid_r, L.grid_c, shape.filters // shape.pool_group), device="cuda")
    J0 = L.forward(x, pooled)
    p_fwd = pooled.cpu().numpy()
    L.encode(x, pooled)
    L.prefetch_input(xh)
    dx = torch.empty_like(x)
    J = L.step(xh, dx)
    tol = 2e-2 if prec == lcae.BF16 else 1e-5
    o = O.step(W.astype(np.float64), a.astype(np.float64), b.astype(np.float64), Xh.astype(np.float64), geo(shape),
               lr=shape.lr, momentum=mu)
    err = {"J": abs(J - o["J"]) / abs(o["J"]), "J_fwd": abs(J0 - o["J"]) / abs(o["J"]),
           "p": np.abs(p_fwd - o["p"]).max() / np.abs(o["p"]).max(),
           "dX": np.abs(dx.cpu().numpy() - o["dX"]).max() / np.abs(o["dX"]).max()}
    if keep:
        dW = np.zeros_like(W)
        L.get_grads(dW, None, None)
        err["dW"] = np.abs(dW - o["dW"]).max() / np.abs(o["dW"]).max()
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
    bad, n = canaries(L)
    L.close()
    assert bad == 0, f"{bad} of {n} allocations written past their end"
    assert all(np.isfinite(v) and v <= tol for v in err.values()), err
    # repeatability: the same three steps from the same state give bitwise identical parameters
    r1 = params_after(shape, prec, keep, x, W, a, b, 3)
    r2 = params_after(shape, prec, keep, x, W, a, b, 3)
    assert all(np.array_equal(u, v) for u, v in zip(r1, r2)), "parameters not reproducible"
    print("  ok", {k: f"{v:.1e}" for k, v in err.items()}, f"canaries {n} intact", flush=True)
print("sanitize run ok")
