"""Benchmark of one training step of the locally-connected RICA autoencoder layer (BASELINE.json metric:
images/sec per LC-autoencoder training step, TFLOP/s vs B200 peak).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c2|c1] [--impl ours|reference]

A step = one pass of the whole hot path (input staging, encode, L2 pooling +
sparsity, decode + residual, loss reduction, backprop into the code, weight gradient, input gradient with
overlap-add, fused projected-SGD update) over one batch of synthetic whitened images, through the C ABI.
N = 1: the whole layer on one GPU.  N > 1 (torchrun): the field grid is tiled over ranks inside the library
(include/lcae.h world_size > 1, csrc/mp.cu): every rank runs its tile, the input halo (bf16) and the dX
return travel by NCCL send/recv on the layer's comm stream while the interior fields compute, the loss is
all-reduced; value = images/s of the whole job (model parallel: every
rank sees every image), time = max over ranks.

--impl reference: the fp64 CPU oracle (oracle/), as it stands, timed on this host on a bounded sample of
the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_1502_03409_b200.inputs import (CONFIGS, EXTRA_CONFIGS, LayerShape, make_images, make_params,  # noqa: E402
                                          stratified_fields)

METRIC = "images/sec per LC-autoencoder training step"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sus=d["bf16_tflops_sustained"], src="measured")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


def alg_bytes(shape):
    """SURVEY.md §8(d) algorithmic bytes per step: fp32 W master read + write (and the velocity's with
    momentum), alpha / b read + write, the bf16 input and the fp32 dX output."""
    w = shape.fields * shape.filters * shape.n
    x = shape.batch * shape.img_h * shape.img_w * shape.img_c
    return 8.0 * w * (2 if shape.momentum > 0 else 1) + 8.0 * shape.fields * (shape.n + 1) + 2.0 * x + 4.0 * x


def uses_gt(shape):
    """Shapes beyond the fused kernel (k > 128, m > 256, n > 4096) run on the general tcgen05 GEMM path."""
    return shape.filters > 128 or shape.batch > 256 or -(-shape.n // 64) * 64 > 4096


def gt_executed_flops(shape):
    """FLOPs of the general path's five GEMMs per field with their tile padding (gt_path.cu: 128-row M tiles,
    BN in {64, 128, 192, 256} columns, 64-deep K steps)."""
    up = lambda v, t: -(-v // t) * t
    bn = lambda N: 64 if N <= 64 else 128 if N <= 128 else 192 if N <= 192 else 256
    g = lambda M, N, K: 2.0 * up(M, 128) * up(N, bn(N)) * up(K, 64)
    k, n, m = shape.filters, shape.n, shape.batch
    return (g(k, m, n) + g(n, m, k) + g(k, m, n) + 2 * g(k, n, m) + g(n, m, k)) * shape.fields


def executed_flops(shape):
    """FLOPs the tcgen05 MMAs of the fused step kernel execute: filters padded to KP = 128, patch
    rows to 64-row tiles, samples to 128 per CTA, plus the exact -I tiles of the residual and dX products."""
    if uses_gt(shape):
        return gt_executed_flops(shape)
    KP, NT, MC = 128, 64, 128
    T = -(-shape.n // NT)
    CB = -(-shape.batch // MC)
    per_cta = (2 * MC * KP * T * NT                       # pass 0: U^T = X^T W~^T
               + 2 * MC * NT * (KP + NT) * T                # pass 1: R^T - X^T = H'^T W~_j + X_j^T (-I)
               + 2 * MC * KP * NT * T                       # pass 1: G^T += delta_j^T W~_j^T
               + 2 * MC * NT * (KP + NT) * T                # pass 2: dx^T = D'^T W~_j + delta_j^T (-I)
               + 2 * KP * NT * 2 * MC * T)                  # pass 2: dW_j = H' delta_j^T + D' X_j^T
    return float(per_cta) * CB * shape.fields


def model_flops(shape):
    """12 k n m F: encode, decode, backprop-to-code, two weight-gradient products, input gradient."""
    return 12.0 * shape.filters * shape.n * shape.batch * shape.fields


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    def __init__(self, index=0, period=0.05):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self.index = period, index
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)
        return self

    def _run(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, nm in names.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


_X64 = {}


def cpu_oracle_rate(shape, budget_s=12.0, seed=0):
    """Time the fp64 oracle (as it stands) on a bounded field sample; return images/s extrapolated to the
    whole layer (every field costs the same work) plus a description. The sample grows geometrically but never
    past the time budget's estimate, so one call takes about budget_s."""
    from oracle import lcae_oracle as O
    geo = dict(img_h=shape.img_h, img_w=shape.img_w, img_c=shape.img_c, rf_h=shape.rf_h, rf_w=shape.rf_w,
               stride=shape.stride, pool_group=shape.pool_group, lam=shape.lam, eps=shape.eps)
    if shape.name not in _X64:
        _X64[shape.name] = make_images(shape, seed=1).astype(np.float64)
    X = _X64[shape.name]
    done, t_used = 0, 0.0
    order = stratified_fields(shape, shape.fields, seed=seed)
    while t_used < budget_s and done < shape.fields:
        nb = max(1, done or 4)
        if done:   # stay within the budget: at most the fields the remaining time affords
            nb = min(nb, max(1, int((budget_s - t_used) / (t_used / done))))
        nb = min(nb, shape.fields - done)
        fl = order[done:done + nb]
        W, a, b = make_params(shape, seed=0, fields=fl)
        t0 = time.perf_counter()
        O.step(W.astype(np.float64), a.astype(np.float64), b.astype(np.float64), X, geo, lr=shape.lr, fields=fl)
        t_used += time.perf_counter() - t0
        done += nb
    t_step = t_used * shape.fields / done
    try:
        threads = len(os.sched_getaffinity(0))
    except Exception:
        threads = os.cpu_count()
    return shape.batch / t_step, done, t_used, threads


def _oracle_init(shape):
    """Pool initializer: every worker builds the oracle's fp64 image batch once, before any timed task."""
    _X64[shape.name] = make_images(shape, seed=1).astype(np.float64)


def _oracle_ready(_):
    time.sleep(0.5)   # spreads one task per worker: all initializers have run when these return
    return os.getpid()


def _oracle_worker(task):
    """One field-parallel oracle process (BLAS threads = 1, set through the environment before numpy loads): time
    O.step on its share of the fields. Returns (fields, seconds)."""
    shape, fl = task
    from oracle import lcae_oracle as O
    if shape.name not in _X64:
        _X64[shape.name] = make_images(shape, seed=1).astype(np.float64)
    geo = dict(img_h=shape.img_h, img_w=shape.img_w, img_c=shape.img_c, rf_h=shape.rf_h, rf_w=shape.rf_w,
               stride=shape.stride, pool_group=shape.pool_group, lam=shape.lam, eps=shape.eps)
    W, a, b = make_params(shape, seed=0, fields=fl)
    t0 = time.perf_counter()
    O.step(W.astype(np.float64), a.astype(np.float64), b.astype(np.float64), _X64[shape.name], geo, lr=shape.lr,
           fields=fl)
    return len(fl), time.perf_counter() - t0


def _blas_info():
    try:
        from threadpoolctl import threadpool_info
        return ", ".join(f"{d.get('internal_api')} {d.get('version')}" for d in threadpool_info()
                         if d.get("user_api") == "blas") or None
    except Exception:
        return None


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


class OraclePool:
    """BASELINE.md §4's CPU baseline: the fp64 oracle, one process per host core (BLAS threads = 1), fields split
    across the processes (fields are independent; each costs the same work), plus its single-core time."""

    def __init__(self, shape):
        import multiprocessing as mp
        try:
            self.cores = len(os.sched_getaffinity(0))
        except Exception:
            self.cores = os.cpu_count() or 1
        self.procs = max(1, min(self.cores, 64))   # one oracle image batch (fp64) per process
        self.shape = shape
        env = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
        for k in env:
            os.environ[k] = "1"
        self.pool = mp.get_context("spawn").Pool(self.procs, initializer=_oracle_init, initargs=(shape,))
        for k, v in env.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        self.order = stratified_fields(shape, shape.fields, seed=0)
        self.pool.map(_oracle_ready, range(self.procs), chunksize=1)   # start-up + image generation
        self.pool.map(_oracle_worker, [(shape, self.order[:1])] * self.procs, chunksize=1)   # warm
        n1, t1 = self.pool.apply(_oracle_worker, ((shape, self.order[:4]),))
        self.t_field = t1 / n1   # single-core seconds per field (BLAS threads = 1)

    def sample(self, budget_s):
        """Run a field-parallel sample sized to about budget_s of wall time; returns (images/s of the whole layer,
        fields done, wall seconds)."""
        per = max(1, int(budget_s / self.t_field))
        n = min(self.shape.fields, per * self.procs)
        fl = self.order[:n]
        chunks = [(self.shape, fl[i::self.procs]) for i in range(self.procs) if fl[i::self.procs]]
        t0 = time.perf_counter()
        res = self.pool.map(_oracle_worker, chunks, chunksize=1)
        wall = time.perf_counter() - t0
        done = sum(r[0] for r in res)
        return self.shape.batch * done / (wall * self.shape.fields), done, wall

    def describe(self, done, wall):
        return {"cores": self.procs, "kind": "oracle", "single_core_value": self.shape.batch / (self.t_field * self.shape.fields),
                "cpu_model": _cpu_model(), "blas": _blas_info(), "host_cores": self.cores,
                "sample": f"{done} of {self.shape.fields} fields (stratified) on {self.procs} processes x 1 BLAS thread, "
                          f"{wall:.1f} s wall, extrapolated linearly to the full layer; single_core_value: the same "
                          f"oracle on one core"}

    def close(self):
        self.pool.terminate()


def run_reference(args, shape):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps = []
    # each step is a bounded field-parallel sample of the workload; the whole --steps/--warmup run stays near 150 s
    per = min(args.ref_budget, max(1.0, 150.0 / (args.steps + args.warmup / 4)))
    op = OraclePool(shape)
    try:
        for _ in range(args.warmup):
            op.sample(per / 4)
        for _ in range(args.steps):
            steps.append(op.sample(per))
    finally:
        op.close()
    v = statistics.median(s[0] for s in steps)
    frac = statistics.median(s[1] for s in steps) / shape.fields
    desc = op.describe(steps[0][1], steps[0][2])
    # a "step" of this arm is one bounded sample (a fraction `sample_fraction` of the layer's fields): ms_per_step is
    # its measured time, so steps x ms_per_step is the arm's wall time; value = m x fraction / sample time = the
    # images/s of the whole layer at the oracle's per-field cost (every field costs the same)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "images/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * shape.batch * frac / v,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": shape.name, "image": [shape.img_h, shape.img_w, shape.img_c],
                       "rf": shape.rf_h, "stride": shape.stride, "filters": shape.filters,
                       "pool_group": shape.pool_group, "batch": shape.batch, "fields": shape.fields,
                       "sample_fraction": frac},
            "cpu_baseline": {"value": v, "unit": "images/s", **desc},
            "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


INFER_METRIC = "images/sec forward_dataset (encode + L2 pooling + streaming top-5 stimuli)"


def run_infer(args, shape):
    """the inference path (lcae_encode + lcae_topk_update) on the same layer. Images
    shard across ranks with no exchange (each rank streams its own batches): weak scaling."""
    import torch
    from paper_1502_03409_b200 import lcae
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    pk = peaks()
    K = 5
    with torch.cuda.stream(stream):
        L = lcae.Layer(lcae.make_config(shape, precision=lcae.BF16, stream=stream.cuda_stream))
        W, a, b = make_params(shape, seed=0)
        L.set_params(W, a, b)
        del W
        units = L.grid_r * L.grid_c * (shape.filters // shape.pool_group)
        pool = [torch.from_numpy(make_images(shape, seed=1 + rank, index=i)).cuda() for i in range(4)]
        pooled = torch.empty((shape.batch, units), dtype=torch.float32, device="cuda")
        vals = torch.empty((units, K), dtype=torch.float32, device="cuda")
        ids = torch.empty((units, K), dtype=torch.int32, device="cuda")
        lcae.topk_init(vals, ids, stream.cuda_stream)

        def step(i):
            L.encode(pool[i % len(pool)], pooled, want_loss=False)
            lcae.topk_update(pooled, vals, ids, i * shape.batch, stream.cuda_stream)
        for i in range(args.warmup):
            step(i)
        torch.cuda.synchronize()
        launches = L.last_launch_count() + 1
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        L.profile(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            e0.record(stream)
            for i in range(args.steps):
                step(args.warmup + i)
            e1.record(stream)
            torch.cuda.synchronize()
        L.profile(False)
        ms = e0.elapsed_time(e1)
        kern_ms, kern_n = L.profile_read()
        if dist:
            t = torch.tensor([ms, kern_ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms, kern_ms = t.tolist()
        # end to end: host batches (pinned) in, the top-K state's first unit read back each step
        hosts = [pool[i].cpu().pin_memory() for i in range(2)]
        probe = torch.empty((1, K), dtype=torch.float32).pin_memory()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n_e2e = max(3, min(args.steps, 10))
        L.prefetch_input(hosts[0])
        for i in range(n_e2e):
            L.encode(hosts[i % 2], pooled, want_loss=False)
            if i + 1 < n_e2e:
                L.prefetch_input(hosts[(i + 1) % 2])   # the next batch's H2D overlaps this encode
            lcae.topk_update(pooled, vals, ids, (1000 + i) * shape.batch, stream.cuda_stream)
            probe.copy_(vals[:1], non_blocking=True)
            stream.synchronize()
        dt = (time.perf_counter() - t0) / n_e2e
    if rank != 0:
        return
    ms_step = ms / args.steps
    kern_avg = kern_ms / max(1, kern_n)
    flops = 2.0 * shape.filters * shape.n * shape.batch * shape.fields   # encode U = W X
    enc_bytes = 2.0 * shape.fields * 128 * shape.n + 6.0 * shape.batch * shape.img_h * shape.img_w * shape.img_c \
        + 4.0 * shape.batch * units
    achieved = flops / (kern_avg * 1e-3) / 1e12
    achieved_gbs = enc_bytes / (kern_avg * 1e-3) / 1e9
    hbm_bound = enc_bytes / (pk["hbm"] * 1e9) > flops / (pk["bf16_sus"] * 1e12)
    line = {
        "metric": INFER_METRIC, "value": world * shape.batch / (ms_step * 1e-3), "unit": "images/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": shape.name + "-infer", "image": [shape.img_h, shape.img_w, shape.img_c],
                   "rf": shape.rf_h, "stride": shape.stride, "filters": shape.filters,
                   "pool_group": shape.pool_group, "batch": shape.batch, "fields": shape.fields, "topk": K,
                   "units": units, "parallelism": f"dp{world}" if world > 1 else "single"},
        "roofline": ({"bound": "hbm", "achieved": achieved_gbs, "peak": pk["hbm"], "unit": "GB/s",
                      "frac": achieved_gbs / pk["hbm"], "traffic": None, "kernel": "lcae::tc::step_kernel (encode)",
                      "kernel_ms": kern_avg, "peak_source": f"{pk['src']} hbm_gbs"} if hbm_bound else
                     {"bound": "tensor", "achieved": achieved, "peak": pk["bf16_sus"], "unit": "TFLOP/s",
                      "frac": achieved / pk["bf16_sus"], "traffic": None,
                      "kernel": "lcae::tc::step_kernel (encode)", "kernel_ms": kern_avg,
                      "peak_source": f"{pk['src']} bf16_tflops_sustained", "hbm_frac": achieved_gbs / pk["hbm"]}),
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
        "e2e": {"value": world * shape.batch / dt, "unit": "images/s",
                "h2d_bytes_per_step": hosts[0].numel() * 4, "d2h_bytes_per_step": K * 4, "ms_per_step": dt * 1e3},
    }
    print(json.dumps(line), flush=True)


# SURVEY.md §8(d) c5 "15 B point": the paper's parameter count ("15 billion parameters") as one
# c3-shaped layer, 347 x 348 fields of 18 x 18 x 3 -> 128 filters (15.02 B weights), batch 256, on ONE GPU
# (fp32 master + bf16 shadow ~ 6 B/param = 90 GB of the 180 GB HBM). Weights are initialised on the device.
EXTRA = dict(EXTRA_CONFIGS)   # c15b, c3p (inputs.py); k = 384 (c3p) runs on the general tcgen05 GEMM path in bf16


FP32_ALU_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4 TFLOP/s of FFMA at the 1965 MHz maximum SM clock


def largest_fit_shape(base, free_bytes, frac=0.88):
    """SURVEY.md §8(d) c5 'largest fit': the square field grid of the base field shape whose layer state fills
    `frac` of the free HBM (cudaMemGetInfo): per field the fp32 master W~ (k x n_al), the bf16 shadow (128 x
    n_al), b, the db partials of the two CTAs and the row scales; plus the image buffers."""
    n_al = (base.n + 7) // 8 * 8
    per_field = (4 * base.filters * n_al + 2 * 128 * n_al + 4 * base.n * 3 + 4 * 2 * 128 * 4 + 4 * base.filters * 3
                 + 128)   # W~, shadow, b + 2 db partials, row-sum partials, sigma + rowsq, loss / alpha partials
    g = int(((frac * free_bytes) / per_field) ** 0.5)
    while g > 1:
        img = (g - 1) * base.stride + base.rf_h
        img_bytes = base.batch * img * img * base.img_c * (4 * 4 + 2)   # x stage, dX (HWCN + NHWC), pf, bf16 image
        if g * g * per_field + img_bytes <= frac * free_bytes:
            break
        g -= 1
    img = (g - 1) * base.stride + base.rf_h
    return base.replace(name=f"c5fit-{g}x{g}", img_h=img, img_w=img)
DEVICE_INIT_PARAMS = 4e9   # above this many weights the host never materialises W (lcae_create seeds them)


def run_ours(args, shape):
    import torch
    from paper_1502_03409_b200 import lcae
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    stream = torch.cuda.Stream()
    pk = peaks()
    nid = None
    if world > 1:
        # model parallel inside the library (include/lcae.h world_size > 1): rank 0 creates the NCCL id, the
        # process group (plumbing) broadcasts it; halos, dX returns and the loss all-reduce are the library's
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [lcae.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    with torch.cuda.stream(stream):
        if True:
            cfg = lcae.make_config(shape, precision=args.prec, stream=stream.cuda_stream, world_size=world,
                                   rank=rank, nccl_id=nid)
            L = lcae.Layer(cfg)
            if world > 1:
                R0, R1, C0, C1 = L.own_fields
                mine = [r * shape.grid_c + c for r in range(R0, R1) for c in range(C0, C1)]
                y0, y1, x0, x1 = L.own_px
            else:
                mine, (y0, y1, x0, x1) = None, (0, shape.img_h, 0, shape.img_w)
            if L.F * shape.filters * shape.n < DEVICE_INIT_PARAMS:
                W, a, b = make_params(shape, seed=0, fields=mine)
                L.set_params(W, a, b)
                del W
            pool = [torch.from_numpy(np.ascontiguousarray(
                make_images(shape, seed=1, index=i)[:, y0:y1, x0:x1, :])).cuda() for i in range(4)]
            step = lambda i: L.step(pool[i % len(pool)], None, want_loss=False)  # noqa: E731
            if args.graph:   # one CUDA graph per pool entry (launch-bound small configs)
                torch.cuda.synchronize()
                graphs = []
                for xi in pool:
                    gph = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(gph, stream=stream):
                        L.step(xi, None, want_loss=False)
                    graphs.append(gph)
                eager_step = step
                step = lambda i: graphs[i % len(graphs)].replay()  # noqa: E731
        torch.cuda.synchronize()
        for i in range(args.warmup):
            step(i)
        torch.cuda.synchronize()
        launches_per_step = L.last_launch_count()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        L.profile(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            e0.record(stream)
            for i in range(args.steps):
                step(i)
            e1.record(stream)
            torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        L.profile(False)
        ms = e0.elapsed_time(e1)
        kern_ms, kern_n = L.profile_read()
        prof_steps = args.steps   # model parallel: two step-kernel launches per step (interior, boundary)
        if world == 1 and args.graph:   # graph replays carry no profile events: time the kernel on eager steps
            L.profile(True)
            for i in range(10):
                eager_step(i)
            torch.cuda.synchronize()
            L.profile(False)
            kern_ms, kern_n = L.profile_read()
            prof_steps = 10
        if dist:
            t = torch.tensor([ms, kern_ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms, kern_ms = t.tolist()
        ms_step = ms / args.steps
        # ---- end to end through the C ABI with host buffers (pinned), loss read back every step
        e2e = None
        if True:
            hosts = [p.cpu().pin_memory() for p in pool[:2]]
            h2d = hosts[0].numel() * 4
            # warm-up through the same path (the first lcae_prefetch_input allocates its buffer, stream, events)
            L.prefetch_input(hosts[0])
            for i in range(3):
                L.step(hosts[i % 2], None, want_loss=False)
                L.prefetch_input(hosts[(i + 1) % 2])
                L.last_loss()
            L.step(hosts[1], None, want_loss=True)   # consumes the last prefetch
            torch.cuda.synchronize()
            # every step: its batch's H2D copy (started during the previous step by lcae_prefetch_input, on the
            # layer's copy stream) + the step + the loss read back (lcae_last_loss synchronises)
            t0 = time.perf_counter()
            n_e2e = max(3, min(args.steps, 20))
            L.prefetch_input(hosts[0])
            for i in range(n_e2e):
                L.step(hosts[i % 2], None, want_loss=False)
                if i + 1 < n_e2e:
                    L.prefetch_input(hosts[(i + 1) % 2])
                jr, js = L.last_loss()
                if not np.isfinite(jr + js):
                    raise RuntimeError("non-finite loss in the e2e loop")
            dt = (time.perf_counter() - t0) / n_e2e
            if dist:   # the slowest rank bounds the job
                t = torch.tensor([dt], device="cuda", dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt = t.item()
                t = torch.tensor([float(h2d)], device="cuda", dtype=torch.float64)
                dist.all_reduce(t)   # every rank copies its owned pixels: the job's bytes
                h2d = int(t.item())
            e2e = {"value": shape.batch / dt, "unit": "images/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": 16, "ms_per_step": dt * 1e3, "h2d_overlap": "lcae_prefetch_input"}
    if rank != 0:
        return
    flops = model_flops(shape)
    value = shape.batch / (ms_step * 1e-3)
    if args.scaling == "weak":   # the layer grows with N: report base-layer-equivalent images/s (value x F / F_base)
        value *= shape.fields / args.base_fields
    kern_avg = kern_ms / max(1, prof_steps)   # step-kernel time per step (all its launches)
    if kern_avg <= 0:   # the fp32 path records no step-kernel events: the whole step bounds it
        kern_avg = ms_step
    per_kernel_flops = flops / world
    achieved = per_kernel_flops / (kern_avg * 1e-3) / 1e12
    achieved_gbs = alg_bytes(shape) / world / (kern_avg * 1e-3) / 1e9
    hbm_bound = alg_bytes(shape) / (pk["hbm"] * 1e9) > flops / (pk["bf16_sus"] * 1e12)
    # the denominator follows the clocks seen in the timed region: the burst peak when the SM clock held its
    # maximum (the kernel ran at full clock), the sustained (power-capped) peak otherwise
    ck = clk.summary()
    burst = bool(ck.get("sm_mhz") and ck.get("sm_max_mhz") and ck["sm_mhz"] >= 0.95 * ck["sm_max_mhz"])
    tc_peak = pk["bf16"] if burst else pk["bf16_sus"]
    tc_src = (f"{pk['src']} bf16_tflops (burst: SM clock median {ck.get('sm_mhz')} of max {ck.get('sm_max_mhz')} MHz "
              f"in the timed region)" if burst else
              f"{pk['src']} bf16_tflops_sustained (SM clock median {ck.get('sm_mhz')} MHz below max)")
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            key = shape.name if shape.momentum == 0 else f"{shape.name}_mom{shape.momentum:g}"
            traffic = json.load(fh).get(key, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16" if args.prec else "f32", "data": "synthetic",
        "config": {"workload": shape.name, "image": [shape.img_h, shape.img_w, shape.img_c], "rf": shape.rf_h,
                   "stride": shape.stride, "filters": shape.filters, "pool_group": shape.pool_group,
                   "batch": shape.batch, "fields": shape.fields, "params": shape.fields * shape.filters * shape.n,
                   "momentum": shape.momentum, "cuda_graph": bool(args.graph),
                   "parallelism": f"mp{world}" if world > 1 else "single",
                   "l2": "working set > L2 (fp32 W master 4 B/param streamed every step)"},
        "tflops": flops / (ms_step * 1e-3) / 1e12,
        "roofline": ({"bound": "hbm", "achieved": achieved_gbs, "peak": pk["hbm"], "unit": "GB/s",
                      "frac": achieved_gbs / pk["hbm"], "traffic": traffic,
                      "kernel": "lcae::tc::step_kernel", "kernel_ms": kern_avg,
                      "peak_source": f"{pk['src']} hbm_gbs", "tensor_frac": achieved / pk["bf16_sus"]}
                     if hbm_bound else
                     {"bound": "tensor", "achieved": achieved, "peak": tc_peak, "unit": "TFLOP/s",
                      "frac": achieved / tc_peak, "traffic": traffic,
                      "kernel": ("lcae::gt::bgemm (the five tcgen05 GEMMs of the general path, summed)"
                                 if uses_gt(shape) else "lcae::tc::step_kernel"),
                      "kernel_ms": kern_avg, "peak_source": tc_src,
                      "frac_of_sustained": achieved / pk["bf16_sus"], "frac_of_burst": achieved / pk["bf16"],
                      "model_flops_per_step": flops, "executed_flops_per_step": executed_flops(shape),
                      "executed_tflops": executed_flops(shape) / world / (kern_avg * 1e-3) / 1e12,
                      "hbm_frac": achieved_gbs / pk["hbm"]}),
        "gpu_launches": launches_per_step * args.steps,
        "clocks": ck,
        "e2e": e2e,
    }
    if not args.prec:   # the FFMA path: bound by fp32 ALU throughput (no tensor cores, several kernels per step)
        alu_peak = FP32_ALU_TFLOPS * (ck["sm_mhz"] / ck["sm_max_mhz"] if ck.get("sm_mhz") and ck.get("sm_max_mhz") else 1)
        ach = flops / world / (ms_step * 1e-3) / 1e12
        line["roofline"] = {"bound": "alu", "achieved": ach, "peak": alu_peak, "unit": "TFLOP/s",
                            "frac": ach / alu_peak, "traffic": None, "kernel": "fp32 path (all kernels of the step)",
                            "kernel_ms": ms_step,
                            "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 FLOP/FFMA x SM clock "
                                           "(median of the timed region); DESIGN.md §6"}
    if not args.no_cpu_baseline and world == 1:
        op = OraclePool(shape)
        try:
            v, done, wall = op.sample(args.ref_budget)
        finally:
            op.close()
        line["cpu_baseline"] = {"value": v, "unit": "images/s", **op.describe(done, wall)}
    print(json.dumps(line), flush=True)


PAPER_METRIC = "images/sec per greedy training step of the paper's 3-layer network (one step of every layer)"


def run_paper_stack(args):
    """SURVEY.md §8(f) item 1 at the paper's geometry (R26): 300 x 300 x 3 images ->
    72 x 72 fields x 384 (1.53 B weights) -> LCN -> 69 x 69 fields x 384 over 16 x 16 x 24 windows (11.26 B) -> LCN ->
    dense 92,256 -> 4096 (0.38 B); 13.17 B parameters, mini-batch 192. k = 384 / 4096 exceed the fused bf16
    kernel's TMEM budget (R24): in bf16 every layer runs on the general tcgen05 GEMM path (gt_path.cu), with
    --precision fp32 on the FFMA path. One 'step' = one greedy training step of each
    layer on the same batch (layer l's input produced by the trained layers below, as in layer-wise training);
    the input chains (encode + LCN of the layers below) are timed separately."""
    import torch
    from paper_1502_03409_b200 import lcae
    from paper_1502_03409_b200.stack import Stack, paper_stack
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    cfg = paper_stack(batch=args.batch or 192)
    st = Stack(cfg, precision=lcae.BF16 if args.prec else lcae.FP32, seed=0, host_params=False)
    pool = [torch.from_numpy(make_images(cfg.shapes[0], seed=1, index=i)).cuda() for i in range(2)]
    n = len(cfg.shapes)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for i in range(max(1, args.warmup // 3)):
        for l in range(n):
            st.layers[l].step(st.input_of(l, pool[i % 2]), None, want_loss=False)
    torch.cuda.synchronize()
    t_layer, t_chain = [0.0] * n, [0.0] * n
    with ClockSampler(0) as clk:
        for i in range(args.steps):
            for l in range(n):
                e0, e1, e2 = ev(), ev(), ev()
                e0.record()
                inp = st.input_of(l, pool[i % 2])
                e1.record()
                st.layers[l].step(inp, None, want_loss=False)
                e2.record()
                torch.cuda.synchronize()
                t_chain[l] += e0.elapsed_time(e1) / args.steps
                t_layer[l] += e1.elapsed_time(e2) / args.steps
    J = [st.layers[l].last_loss() for l in range(n)]
    st.close()
    ms = sum(t_layer)
    flops = [12.0 * s.filters * s.n * s.batch * s.fields for s in cfg.shapes]
    ck = clk.summary()
    alu_peak = FP32_ALU_TFLOPS * (ck["sm_mhz"] / ck["sm_max_mhz"] if ck.get("sm_mhz") and ck.get("sm_max_mhz") else 1)
    ach = sum(flops) / (ms * 1e-3) / 1e12
    if args.prec:   # bf16: tensor-bound; the whole three-layer step time against the bf16 peak the clocks select
        pk = peaks()
        burst = bool(ck.get("sm_mhz") and ck.get("sm_max_mhz") and ck["sm_mhz"] >= 0.95 * ck["sm_max_mhz"])
        roof = {"bound": "tensor", "achieved": ach, "peak": pk["bf16"] if burst else pk["bf16_sus"],
                "unit": "TFLOP/s", "frac": ach / (pk["bf16"] if burst else pk["bf16_sus"]), "traffic": None,
                "kernel": "general tcgen05 path (all kernels of the three layer steps)", "kernel_ms": ms,
                "peak_source": f"{pk['src']} {'bf16_tflops (burst)' if burst else 'bf16_tflops_sustained'}"}
    else:
        roof = {"bound": "alu", "achieved": ach, "peak": alu_peak, "unit": "TFLOP/s", "frac": ach / alu_peak,
                "traffic": None, "kernel": "fp32 path (all kernels of the three layer steps)",
                "kernel_ms": ms, "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 FLOP x SM clock"}
    line = {"metric": PAPER_METRIC, "value": cfg.shapes[0].batch / (ms * 1e-3), "unit": "images/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16" if args.prec else "f32", "data": "synthetic",
            "config": {"workload": "paper3 (PAPER.md:95 three-layer network, DESIGN.md R26)",
                       "layers": [{"name": s.name, "input": [s.img_h, s.img_w, s.img_c], "rf": s.rf_h,
                                   "stride": s.stride, "fields": s.fields, "n": s.n, "k": s.filters,
                                   "params": s.fields * (s.filters * s.n + s.n + 1), "step_ms": t_layer[i],
                                   "input_chain_ms": t_chain[i], "tflops": flops[i] / (t_layer[i] * 1e-3) / 1e12,
                                   "J": J[i][0] + J[i][1]} for i, s in enumerate(cfg.shapes)],
                       "params": sum(s.fields * (s.filters * s.n + s.n + 1) for s in cfg.shapes),
                       "batch": cfg.shapes[0].batch, "lcn_window": cfg.lcn_window},
            "tflops": ach,
            "roofline": roof,
            "clocks": ck}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS) + sorted(EXTRA) + ["c5fit", "paper3"])
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"],
                    help="bf16: the tcgen05 paths (default; the fused kernel, or the general GEMM path for k > 128, e.g. "
                         "c3p); fp32: the FFMA path")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-budget", type=float, default=12.0, help="seconds of oracle work per sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--momentum", type=float, default=0.0, help="SGD momentum (SURVEY.md §8(f) item 3: 0.9)")
    ap.add_argument("--batch", type=int, default=0, help="override the config's mini-batch (PAPER.md:111: 192)")
    ap.add_argument("--graph", action="store_true", help="replay each step from a captured CUDA graph (1 GPU)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's layer on N GPUs (default); weak: the field grid grows with N "
                         "(SURVEY.md §8(d) c5: grid_r x grid_c fields per GPU, global grid scaled by the tiles); "
                         "value = base-layer-equivalent images/s")
    ap.add_argument("--mode", default="train", choices=["train", "infer"],
                    help="train: the training step (default); infer: encode + top-K stimuli (§8(f) item 4)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    args.prec = 0 if args.precision == "fp32" else 1
    if args.config == "paper3":
        shape = CONFIGS["c3"]   # placeholder: run_paper_stack builds the three layers itself
    elif args.config == "c5fit":   # largest single-GPU layer of the c3 field shape (sized from cudaMemGetInfo)
        import torch
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        free, _ = torch.cuda.mem_get_info()
        shape = largest_fit_shape(CONFIGS["c3"], free)
    else:
        shape = CONFIGS[args.config] if args.config in CONFIGS else EXTRA[args.config]
    if args.momentum:
        shape = shape.replace(momentum=args.momentum)
    if args.batch:
        shape = shape.replace(name=f"{shape.name}-m{args.batch}", batch=args.batch, lr=1e-3 / args.batch)
    args.base_fields = shape.fields
    if args.scaling == "weak":
        from paper_1502_03409_b200.parallel import factor
        tr, tc = factor(int(os.environ.get("WORLD_SIZE", "1")))
        gr, gc = shape.grid_r * tr, shape.grid_c * tc
        shape = shape.replace(name=f"{shape.name}-weak", img_h=(gr - 1) * shape.stride + shape.rf_h,
                              img_w=(gc - 1) * shape.stride + shape.rf_w)
    if args.config == "paper3":
        run_paper_stack(args)
    elif args.impl == "reference":
        run_reference(args, shape)
    elif args.mode == "infer":
        run_infer(args, shape)
    else:
        run_ours(args, shape)


if __name__ == "__main__":
    main()
