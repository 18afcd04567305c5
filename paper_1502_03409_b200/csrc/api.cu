// api.cu — the extern "C" boundary of liblcae.so (declared and documented in include/lcae.h).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace lcae {
static thread_local std::string g_err = "no error";
void set_error(const std::string &msg) { g_err = msg; }

static lcae_status config_error(const std::string &m) {
  set_error(m);
  return LCAE_ERR_CONFIG;
}

static Geo make_geo(const lcae_config *c, int H, int W);

// Geometry validation (R7) and derived sizes.
static lcae_status validate(const lcae_config *c, Geo *out) {
  if (!c) { set_error("NULL config"); return LCAE_ERR_ARG; }
  if (c->img_h <= 0 || c->img_w <= 0 || c->img_c <= 0 || c->rf_h <= 0 || c->rf_w <= 0 || c->stride <= 0 ||
      c->filters <= 0 || c->pool_group <= 0 || c->batch <= 0)
    return config_error("all sizes must be positive");
  if (c->rf_h > c->img_h || c->rf_w > c->img_w) return config_error("receptive field larger than image");
  int ry = (c->img_h - c->rf_h) % c->stride, rx = (c->img_w - c->rf_w) % c->stride;
  if (ry || rx) {
    char buf[160];
    snprintf(buf, sizeof buf, "non-divisible extent: residue rows=%d cols=%d for stride %d", ry, rx, c->stride);
    return config_error(buf);
  }
  if (c->filters % c->pool_group) return config_error("pool_group must divide filters");
  if (32 % c->pool_group) return config_error("pool_group must divide 32");
  if (c->precision != LCAE_FP32 && c->precision != LCAE_BF16) return config_error("unknown precision");
  if (!(c->eps >= 0.f) || !(c->lr >= 0.f) || !(c->momentum >= 0.f && c->momentum < 1.f) || !(c->alpha_min > 0.f))
    return config_error("eps/lr must be >= 0, momentum in [0,1), alpha_min > 0");
  if (c->world_size < 0) return config_error("world_size must be >= 1");
  Geo g = make_geo(c, c->img_h, c->img_w);
  if ((int64_t)g.H * g.W * g.C * g.m >= (1ll << 31)) return config_error("image x batch too large (>= 2^31 elements)");
  if (out) *out = g;
  return LCAE_OK;
}

// This rank's geometry: the whole layer (world_size <= 1), else the rectangle its tile's fields read (mp.cu).
static lcae_status local_geo(const lcae_config *c, const Geo &gg, MpTile *t, Geo *out) {
  if (c->world_size <= 1) {
    t->R0 = 0; t->R1 = gg.gr; t->C0 = 0; t->C1 = gg.gc;
    t->need[0] = t->own[0] = 0; t->need[1] = t->own[1] = gg.H;
    t->need[2] = t->own[2] = 0; t->need[3] = t->own[3] = gg.W;
    *out = gg;
    return LCAE_OK;
  }
  lcae_status s = mp_tile(c, gg, c->rank, t);
  if (s) return s;
  *out = make_geo(c, t->need[1] - t->need[0], t->need[3] - t->need[2]);
  return LCAE_OK;
}

static Geo make_geo(const lcae_config *c, int H, int W) {
  Geo g{};
  g.H = H; g.W = W; g.C = c->img_c; g.rf_h = c->rf_h; g.rf_w = c->rf_w; g.s = c->stride;
  g.k = c->filters; g.g = c->pool_group; g.m = c->batch;
  g.gr = (g.H - g.rf_h) / g.s + 1;
  g.gc = (g.W - g.rf_w) / g.s + 1;
  g.F = g.gr * g.gc;
  g.n = g.rf_h * g.rf_w * g.C;
  g.RW = g.rf_w * g.C;
  g.SY = (int64_t)g.W * g.C * g.m;
  g.SRC_R = (int64_t)g.s * g.SY;
  g.SRC_C = (int64_t)g.s * g.C * g.m;
  return g;
}

static bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Copy `bytes` between any combination of host/device pointers on the layer stream.
static lcae_status copy_any(lcae_layer *L, void *dst, const void *src, size_t bytes) {
  LCAE_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, L->st));
  return LCAE_OK;
}

// Elements of the caller's input / dx: the layer image, or this rank's owned pixels (model parallel).
static size_t input_elems(lcae_layer *L) {
  const Geo &g = L->geo;
  return L->mpst ? mp_input_elems(L) : (size_t)g.m * g.H * g.W * g.C;
}

// Make x device-resident (staging host data) and convert to the path's internal HWCN layout.
static lcae_status stage_input(lcae_layer *L, const float *x) {
  size_t bytes = input_elems(L) * 4;
  const float *xd = x;
  if (L->pf_host && L->pf_host == (const void *)x) {   // prefetched by lcae_prefetch_input
    LCAE_CK(cudaStreamWaitEvent(L->st, L->pf_done, 0));
    xd = L->x_pf;
    L->pf_host = nullptr;
  } else if (!is_device_ptr(x)) {
    lcae_status s = copy_any(L, L->x_stage, x, bytes);
    if (s) return s;
    xd = L->x_stage;
  }
  lcae_status s = L->mpst ? mp_stage(L, xd)
                 : (L->cfg.precision == LCAE_FP32) ? launch_nhwc_to_hwcn_f32(L, xd, L->xt32)
                                                   : launch_nhwc_to_hwcn_bf16(L, xd, L->xt16);
  if (s) return s;
  if (L->x_consumed) LCAE_CK(cudaEventRecord(L->x_consumed, L->st));   // x_pf may be refilled after this
  return LCAE_OK;
}

// Report (and clear) the sticky device error flags; the stream must be synchronised with flags_host filled.
static lcae_status flag_status(lcae_layer *L) {
  const int f0 = L->flags_host[0], f1 = L->flags_host[1];
  if (!(f0 | f1)) return LCAE_OK;
  LCAE_CK(cudaMemsetAsync(L->flags_dev, 0, 2 * sizeof(int), L->st));
  L->flags_host[0] = L->flags_host[1] = 0;
  if (f0) {
    set_error("non-finite input value (SPEC.md:95): the flagged step and every later step until this report were "
              "skipped; parameters unchanged by them");
    return LCAE_ERR_DATA;
  }
  set_error("non-finite loss (SPEC.md:95): the parameters of that step were updated (non-finite); every later "
            "step until this report was skipped");
  return LCAE_ERR_NUMERIC;
}

static lcae_status sync_flags(lcae_layer *L) {
  LCAE_CK(cudaMemcpyAsync(L->flags_host, L->flags_dev, 2 * sizeof(int), cudaMemcpyDeviceToHost, L->st));
  LCAE_CK(cudaStreamSynchronize(L->st));
  return flag_status(L);
}

static lcae_status read_loss(lcae_layer *L, double *loss) {
  LCAE_CK(cudaMemcpyAsync(L->loss_host, L->loss_dev, 2 * sizeof(double), cudaMemcpyDeviceToHost, L->st));
  LCAE_CK(cudaMemcpyAsync(L->flags_host, L->flags_dev, 2 * sizeof(int), cudaMemcpyDeviceToHost, L->st));
  LCAE_CK(cudaStreamSynchronize(L->st));
  double J = L->loss_host[0] + L->loss_host[1];
  if (loss) *loss = J;
  lcae_status s = flag_status(L);
  if (s) return s;
  if (!std::isfinite(J)) {   // a forward pass (no update): reported directly, nothing is flagged
    set_error("non-finite loss");
    return LCAE_ERR_NUMERIC;
  }
  return LCAE_OK;
}

}  // namespace lcae

using namespace lcae;

extern "C" {

void lcae_config_default(lcae_config *c) {
  if (!c) return;
  memset(c, 0, sizeof *c);
  c->lambda_ = 0.1f;
  c->eps = 1e-6f;
  c->lr = 1e-3f;
  c->momentum = 0.f;
  c->alpha_init = 1.f;
  c->alpha_min = 1e-8f;
  c->pool_group = 1;
  c->precision = LCAE_BF16;
  c->world_size = 1;
}

const char *lcae_last_error(void) { return g_err.c_str(); }
const char *lcae_version(void) { return "lcae 0.1.0 sm_100a"; }

lcae_status lcae_geometry(const lcae_config *cfg, int32_t *grid_r, int32_t *grid_c, int64_t *n_params,
                          int32_t own_px[4], int32_t own_fields[4]) {
  Geo gg, g;
  MpTile t;
  lcae_status s = validate(cfg, &gg);
  if (s) return s;
  if ((s = local_geo(cfg, gg, &t, &g))) return s;
  if (grid_r) *grid_r = g.gr;
  if (grid_c) *grid_c = g.gc;
  if (n_params) *n_params = (int64_t)g.F * ((int64_t)g.k * g.n + g.n + 1);
  if (own_px) for (int i = 0; i < 4; ++i) own_px[i] = t.own[i];
  if (own_fields) { own_fields[0] = t.R0; own_fields[1] = t.R1; own_fields[2] = t.C0; own_fields[3] = t.C1; }
  return LCAE_OK;
}

lcae_status lcae_destroy(lcae_layer *L) {
  if (!L) return LCAE_OK;
  if (L->st) cudaStreamSynchronize(L->st);
  cudaDeviceSynchronize();
  mp_free(L);
  f32_free(L);
  tc_free(L);
  gt_free(L);
  for (void *p : {(void *)L->W, (void *)L->sigma, (void *)L->alpha, (void *)L->b, (void *)L->vW, (void *)L->va,
                  (void *)L->vb, (void *)L->Wb, (void *)L->x_stage, (void *)L->xt32, (void *)L->xt16,
                  (void *)L->dxt, (void *)L->dx_nhwc, (void *)L->pooled, (void *)L->gW, (void *)L->galpha,
                  (void *)L->gb, (void *)L->loss_part, (void *)L->loss_dev, (void *)L->reinit_dev, (void *)L->step_dev,
                  (void *)L->rowsq, (void *)L->flags_dev})
    if (p) cudaFree(p);
  if (L->loss_host) cudaFreeHost(L->loss_host);
  if (L->flags_host) cudaFreeHost(L->flags_host);
  if (L->x_pf) cudaFree(L->x_pf);
  if (L->copy_st) cudaStreamDestroy(L->copy_st);
  if (L->pf_done) cudaEventDestroy(L->pf_done);
  if (L->x_consumed) cudaEventDestroy(L->x_consumed);
  if (L->prof_ev) {
    for (int i = 0; i < 2 * 4096; ++i) cudaEventDestroy(L->prof_ev[i]);
    delete[] L->prof_ev;
  }
  delete L;
  return LCAE_OK;
}

lcae_status lcae_create(const lcae_config *cfg, lcae_layer **out) {
  if (!out) { set_error("NULL out"); return LCAE_ERR_ARG; }
  *out = nullptr;
  Geo gg, g;
  MpTile tile;
  lcae_status s = validate(cfg, &gg);
  if (s) return s;
  if ((s = local_geo(cfg, gg, &tile, &g))) return s;
  lcae_layer *L = new lcae_layer();
  L->cfg = *cfg;
  L->poison = getenv("LCAE_DEV_POISON") ? atoi(getenv("LCAE_DEV_POISON")) : 0;
  L->canary = getenv("LCAE_DEV_CANARY") ? atoi(getenv("LCAE_DEV_CANARY")) : 0;
  if (L->cfg.world_size > 1) {   // the tile's global field offsets key the counter-based init / reinit
    L->cfg.field_row0 = tile.R0;
    L->cfg.field_col0 = tile.C0;
    L->cfg.global_grid_c = gg.gc;
  }
  if (L->cfg.global_grid_c <= 0) L->cfg.global_grid_c = g.gc;
  L->geo = g;
  L->st = (cudaStream_t)cfg->stream;
#define FAIL(x)                         \
  do {                                  \
    lcae_status s_ = (x);               \
    if (s_) { lcae_destroy(L); return s_; } \
  } while (0)
#define CKF(call)                                                                 \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      set_error(std::string(#call) + ": " + cudaGetErrorString(e_));              \
      lcae_destroy(L);                                                            \
      return LCAE_ERR_CUDA;                                                       \
    }                                                                             \
  } while (0)
  CKF(cudaGetDevice(&L->device));
  CKF(cudaDeviceGetAttribute(&L->sm_count, cudaDevAttrMultiProcessorCount, L->device));
  const size_t F = g.F, k = g.k, n = g.n, m = g.m, img = (size_t)g.H * g.W * g.C;
  L->n_al = (int)((n + 7) / 8 * 8);
  // bf16 shapes beyond the fused kernel (k > 128, n > 4096, m > 256) take the general tcgen05 GEMM path (gt_path.cu);
  // LCAE_DEV_FORCE_GT=1 selects it for any shape (test hook: the oracle checks it at small sizes)
  const char *force_gt = getenv("LCAE_DEV_FORCE_GT");
  const bool use_gt = cfg->precision == LCAE_BF16 && (tc_unsupported(g) || (force_gt && atoi(force_gt)));
  // fp32 master row pitch: n (fp32 path), 16-byte rows (fused kernel), 128-byte rows (general path: its SGD epilogue
  // reads 32-column runs)
  L->wp = cfg->precision == LCAE_FP32 ? (int)n : use_gt ? (int)((n + 31) / 32 * 32) : L->n_al;
  const size_t wp = L->wp;
  CKF(dmalloc(L, &L->W, F * k * wp * 4));
  CKF(cudaMemsetAsync(L->W, 0, F * k * wp * 4, L->st));
  CKF(dmalloc(L, &L->sigma, F * k * 4));
  CKF(dmalloc(L, &L->alpha, F * 4));
  CKF(dmalloc(L, &L->b, F * n * 4));
  if (cfg->momentum > 0.f) {
    CKF(dmalloc(L, &L->vW, F * k * wp * 4));
    CKF(dmalloc(L, &L->va, F * 4));
    CKF(dmalloc(L, &L->vb, F * n * 4));
    CKF(cudaMemsetAsync(L->vW, 0, F * k * wp * 4, L->st));
    CKF(cudaMemsetAsync(L->va, 0, F * 4, L->st));
    CKF(cudaMemsetAsync(L->vb, 0, F * n * 4, L->st));
  }
  L->mp = cfg->precision == LCAE_FP32 ? g.m : (g.m + 7) / 8 * 8;
  const size_t mp = L->mp;
  CKF(dmalloc(L, &L->x_stage, m * img * 4));   // >= the owned pixels of a model-parallel rank
  CKF(dmalloc(L, &L->dxt, mp * img * 4));
  CKF(dmalloc(L, &L->dx_nhwc, m * img * 4));
  // the pooled-code buffer (m F k/g floats, 128 KB per c3 field) is allocated on the first forward / encode that
  // asks for it: a training-only layer leaves that HBM to its weights (the largest-fit point)
  CKF(dmalloc(L, &L->loss_part, F * 2 * sizeof(double)));
  CKF(dmalloc(L, &L->loss_dev, 2 * sizeof(double)));
  CKF(cudaMemsetAsync(L->loss_dev, 0, 2 * sizeof(double), L->st));
  CKF(dmalloc(L, &L->reinit_dev, sizeof(int)));
  CKF(cudaMemsetAsync(L->reinit_dev, 0, sizeof(int), L->st));
  CKF(dmalloc(L, &L->step_dev, sizeof(int64_t)));
  CKF(cudaMemsetAsync(L->step_dev, 0, sizeof(int64_t), L->st));
  CKF(cudaMallocHost(&L->loss_host, 2 * sizeof(double)));
  CKF(dmalloc(L, &L->flags_dev, 2 * sizeof(int)));
  CKF(cudaMemsetAsync(L->flags_dev, 0, 2 * sizeof(int), L->st));
  CKF(cudaMallocHost(&L->flags_host, 2 * sizeof(int)));
  L->flags_host[0] = L->flags_host[1] = 0;
  if (cfg->keep_grads) {
    CKF(dmalloc(L, &L->gW, F * k * wp * 4));
    CKF(cudaMemsetAsync(L->gW, 0, F * k * wp * 4, L->st));
    CKF(dmalloc(L, &L->galpha, F * 4));
    CKF(dmalloc(L, &L->gb, F * n * 4));
  }
  if (cfg->precision == LCAE_FP32) {
    CKF(dmalloc(L, &L->xt32, m * img * 4));
    FAIL(f32_alloc(L));
  } else {
    CKF(dmalloc(L, &L->xt16, mp * img * 2));
    CKF(cudaMemset(L->xt16, 0, mp * img * 2));   // padded batch columns stay zero
    CKF(dmalloc(L, &L->rowsq, F * k * 4));
    if (use_gt) {
      FAIL(gt_alloc(L));
    } else {
      FAIL(tc_alloc(L));
    }
  }
  // model parallel: world_size > 1; or one rank with an NCCL id (the whole layer as a single tile: exercises the
  // communicator, the interior / boundary launches and the loss all-reduce on one GPU)
  if (cfg->world_size > 1 || cfg->nccl_id) FAIL(mp_init(L, gg));
  FAIL(launch_init_params(L));
  FAIL(launch_refresh_shadow(L));
  CKF(cudaStreamSynchronize(L->st));
  *out = L;
  return LCAE_OK;
#undef FAIL
#undef CKF
}

lcae_status lcae_set_params(lcae_layer *L, const float *W, const float *alpha, const float *b) {
  if (!L) { set_error("NULL handle"); return LCAE_ERR_ARG; }
  const Geo &g = L->geo;
  lcae_status s;
  if (W) {
    LCAE_CK(cudaMemcpy2DAsync(L->W, (size_t)L->wp * 4, W, (size_t)g.n * 4, (size_t)g.n * 4, (size_t)g.F * g.k,
                              cudaMemcpyDefault, L->st));
    // W is taken as given: sigma = 1 (W~ = W)
    if ((s = launch_fill(L, L->sigma, (int64_t)g.F * g.k, 1.f))) return s;
    if ((s = launch_refresh_shadow(L))) return s;
  }
  if (alpha && (s = copy_any(L, L->alpha, alpha, (size_t)g.F * 4))) return s;
  if (b && (s = copy_any(L, L->b, b, (size_t)g.F * g.n * 4))) return s;
  LCAE_CK(cudaMemsetAsync(L->flags_dev, 0, 2 * sizeof(int), L->st));   // fresh parameters: flags cleared
  LCAE_CK(cudaStreamSynchronize(L->st));
  return LCAE_OK;
}

lcae_status lcae_get_params(lcae_layer *L, float *W, float *alpha, float *b) {
  if (!L) { set_error("NULL handle"); return LCAE_ERR_ARG; }
  const Geo &g = L->geo;
  lcae_status s;
  if (W) {
    size_t bytes = (size_t)g.F * g.k * g.n * 4;
    if (is_device_ptr(W)) {
      if ((s = launch_get_W(L, W))) return s;
    } else {
      float *tmp = nullptr;
      LCAE_CK(cudaMallocAsync(&tmp, bytes, L->st));
      if ((s = launch_get_W(L, tmp))) return s;
      LCAE_CK(cudaMemcpyAsync(W, tmp, bytes, cudaMemcpyDeviceToHost, L->st));
      LCAE_CK(cudaFreeAsync(tmp, L->st));
    }
  }
  if (alpha && (s = copy_any(L, alpha, L->alpha, (size_t)g.F * 4))) return s;
  if (b && (s = copy_any(L, b, L->b, (size_t)g.F * g.n * 4))) return s;
  LCAE_CK(cudaStreamSynchronize(L->st));
  return LCAE_OK;
}

lcae_status lcae_get_field_params(lcae_layer *L, int64_t f0, int64_t count, float *W, float *alpha, float *b) {
  if (!L) { set_error("NULL handle"); return LCAE_ERR_ARG; }
  const Geo &g = L->geo;
  if (f0 < 0 || count < 0 || f0 + count > g.F) { set_error("lcae_get_field_params: field range outside the layer"); return LCAE_ERR_ARG; }
  if (!count) return LCAE_OK;
  lcae_status s;
  if (W) {   // sigma (.) W~ of the range, through a device staging buffer
    const size_t bytes = (size_t)count * g.k * g.n * 4;
    float *tmp = nullptr;
    LCAE_CK(cudaMallocAsync(&tmp, bytes, L->st));
    if ((s = launch_get_W_range(L, tmp, f0, count))) return s;
    LCAE_CK(cudaMemcpyAsync(W, tmp, bytes, cudaMemcpyDefault, L->st));
    LCAE_CK(cudaFreeAsync(tmp, L->st));
  }
  if (alpha && (s = copy_any(L, alpha, L->alpha + f0, (size_t)count * 4))) return s;
  if (b && (s = copy_any(L, b, L->b + f0 * g.n, (size_t)count * g.n * 4))) return s;
  LCAE_CK(cudaStreamSynchronize(L->st));
  return LCAE_OK;
}

lcae_status lcae_get_grads(lcae_layer *L, float *dW, float *dalpha, float *db) {
  if (!L) { set_error("NULL handle"); return LCAE_ERR_ARG; }
  if (!L->cfg.keep_grads) return config_error("lcae_get_grads needs keep_grads = 1");
  const Geo &g = L->geo;
  lcae_status s;
  if (dW)
    LCAE_CK(cudaMemcpy2DAsync(dW, (size_t)g.n * 4, L->gW, (size_t)L->wp * 4, (size_t)g.n * 4, (size_t)g.F * g.k,
                              cudaMemcpyDefault, L->st));
  if (dalpha && (s = copy_any(L, dalpha, L->galpha, (size_t)g.F * 4))) return s;
  if (db && (s = copy_any(L, db, L->gb, (size_t)g.F * g.n * 4))) return s;
  LCAE_CK(cudaStreamSynchronize(L->st));
  return LCAE_OK;
}

static lcae_status run(lcae_layer *L, const float *x, bool update, float *dx, float *pooled, double *loss,
                       bool encode_only = false) {
  if (!L) { set_error("NULL handle"); return LCAE_ERR_ARG; }
  if (!x) { set_error("NULL input"); return LCAE_ERR_ARG; }
  L->launches = 0;
  const Geo &g = L->geo;
  lcae_status s;
  if (L->mpst && mp_external(L)) {
    set_error("model-parallel test-mode layer (nccl_id == NULL): drive it with lcae_mp_phase");
    return LCAE_ERR_ARG;
  }
  if (pooled && !L->pooled) LCAE_CK(dmalloc(L, &L->pooled, (size_t)g.m * g.F * (g.k / g.g) * 4));
  if ((s = stage_input(L, x))) return s;
  if (L->mpst) {   // model parallel (mp.cu): halo exchange, interior / boundary fields, dX return, loss all-reduce
    if (encode_only) { set_error("lcae_encode is not available on a model-parallel layer"); return LCAE_ERR_ARG; }
    for (int ph = 0; ph < 3; ++ph)
      if ((s = mp_phase(L, ph, update, pooled != nullptr))) return s;
  } else {
    s = (L->cfg.precision == LCAE_FP32) ? f32_step(L, update, pooled != nullptr)
        : L->gt                          ? gt_step(L, update, pooled != nullptr, encode_only)
                                         : tc_step(L, update, pooled != nullptr, encode_only);
    if (s) return s;
    if ((s = launch_loss_reduce(L, update))) return s;
    if (update && (s = launch_hwcn_to_nhwc_f32(L, L->dxt, L->dx_nhwc))) return s;
  }
  if (update) {
    if (dx && (s = copy_any(L, dx, L->dx_nhwc, input_elems(L) * 4))) return s;
    L->steps++;
  }
  if (pooled && (s = copy_any(L, pooled, L->pooled, (size_t)g.m * g.F * (g.k / g.g) * 4))) return s;
  if (loss || (dx && !is_device_ptr(dx)) || (pooled && !is_device_ptr(pooled))) {
    if (loss) return read_loss(L, loss);
    return sync_flags(L);
  }
  return LCAE_OK;
}

lcae_status lcae_forward(lcae_layer *L, const float *x, float *pooled, double *loss) {
  return run(L, x, false, nullptr, pooled, loss);
}

lcae_status lcae_prefetch_input(lcae_layer *L, const float *x_host) {
  if (!L || !x_host) { set_error("NULL argument"); return LCAE_ERR_ARG; }
  if (is_device_ptr(x_host)) return LCAE_OK;   // nothing to copy
  const size_t bytes = input_elems(L) * 4;
  if (!L->x_pf) {   // first use: the buffer, a copy stream and two events
    LCAE_CK(dmalloc(L, &L->x_pf, bytes));
    LCAE_CK(cudaStreamCreateWithFlags(&L->copy_st, cudaStreamNonBlocking));
    LCAE_CK(cudaEventCreateWithFlags(&L->pf_done, cudaEventDisableTiming));
    LCAE_CK(cudaEventCreateWithFlags(&L->x_consumed, cudaEventDisableTiming));
    LCAE_CK(cudaEventRecord(L->x_consumed, L->st));
  }
  // the previous prefetched batch must have been converted before x_pf is overwritten
  LCAE_CK(cudaStreamWaitEvent(L->copy_st, L->x_consumed, 0));
  LCAE_CK(cudaMemcpyAsync(L->x_pf, x_host, bytes, cudaMemcpyHostToDevice, L->copy_st));
  LCAE_CK(cudaEventRecord(L->pf_done, L->copy_st));
  L->pf_host = x_host;
  return LCAE_OK;
}

lcae_status lcae_encode(lcae_layer *L, const float *x, float *pooled, double *j_sparse) {
  if (!pooled) { set_error("lcae_encode: pooled output required"); return LCAE_ERR_ARG; }
  lcae_status st = run(L, x, false, nullptr, pooled, nullptr, true);
  if (st || !j_sparse) return st;
  return lcae_last_loss(L, nullptr, j_sparse);   // the sparsity term (the fp32 path also forms J_rec)
}

lcae_status lcae_step(lcae_layer *L, const float *x, float *dx, double *loss) {
  return run(L, x, true, dx, nullptr, loss);
}

lcae_status lcae_last_loss(lcae_layer *L, double *j_rec, double *j_sparse) {
  if (!L) { set_error("NULL handle"); return LCAE_ERR_ARG; }
  LCAE_CK(cudaMemcpyAsync(L->loss_host, L->loss_dev, 2 * sizeof(double), cudaMemcpyDeviceToHost, L->st));
  LCAE_CK(cudaStreamSynchronize(L->st));
  if (j_rec) *j_rec = L->loss_host[0];
  if (j_sparse) *j_sparse = L->loss_host[1];
  return LCAE_OK;
}

lcae_status lcae_mp_phase(lcae_layer *L, int32_t phase, int32_t update, const float *x, float *dx, float *pooled,
                          double *loss) {
  if (!L || !L->mpst || !mp_external(L)) {
    set_error("lcae_mp_phase: needs a model-parallel layer in test mode (world_size > 1, nccl_id == NULL)");
    return LCAE_ERR_ARG;
  }
  if (phase < 0 || phase > 2) { set_error("lcae_mp_phase: phase must be 0, 1 or 2"); return LCAE_ERR_ARG; }
  lcae_status s;
  if (phase == 0) {
    if (!x) { set_error("NULL input"); return LCAE_ERR_ARG; }
    L->launches = 0;
    if ((s = stage_input(L, x))) return s;
  }
  if (pooled && !L->pooled) LCAE_CK(dmalloc(L, &L->pooled, (size_t)L->geo.m * L->geo.F * (L->geo.k / L->geo.g) * 4));
  if ((s = mp_phase(L, phase, update != 0, pooled != nullptr))) return s;
  if (phase == 2) {
    if (update) {
      if (dx && (s = copy_any(L, dx, L->dx_nhwc, input_elems(L) * 4))) return s;
      L->steps++;
    }
    if (pooled && (s = copy_any(L, pooled, L->pooled, (size_t)L->geo.m * L->geo.F * (L->geo.k / L->geo.g) * 4)))
      return s;
    if (loss) return read_loss(L, loss);
    return sync_flags(L);
  }
  return LCAE_OK;
}

lcae_status lcae_mp_buffer(lcae_layer *L, int32_t which, int32_t peer, void **ptr, int64_t *bytes) {
  if (!L || !L->mpst || which < 0 || which > 3) { set_error("lcae_mp_buffer: bad handle or buffer id"); return LCAE_ERR_ARG; }
  return mp_buffer(L, which, peer, ptr, bytes);
}

lcae_status lcae_mp_fields(lcae_layer *L, int32_t *n_interior, int32_t *n_boundary) {
  if (!L) { set_error("NULL handle"); return LCAE_ERR_ARG; }
  int a = 0, b = L->geo.F;
  if (L->mpst) mp_counts(L, &a, &b);
  if (n_interior) *n_interior = a;
  if (n_boundary) *n_boundary = b;
  return LCAE_OK;
}

lcae_status lcae_sync(lcae_layer *L) {
  if (!L) { set_error("NULL handle"); return LCAE_ERR_ARG; }
  return sync_flags(L);
}

lcae_status lcae_field_losses(lcae_layer *L, double *out) {
  if (!L || !out) { set_error("NULL argument"); return LCAE_ERR_ARG; }
  const Geo &g = L->geo;
  const bool tcp = L->tc != nullptr;   // the fused kernel keeps one partial per CTA of a cluster
  const int per = tcp ? tc_loss_count(L) / g.F : 1;   // partials per field (CTAs of a cluster)
  double *part = tcp ? tc_loss_part(L) : L->loss_part;
  double *h = nullptr;
  const size_t bytes = (size_t)g.F * per * 2 * sizeof(double);
  LCAE_CK(cudaMallocHost(&h, bytes));
  cudaError_t e = cudaMemcpyAsync(h, part, bytes, cudaMemcpyDeviceToHost, L->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(L->st);
  if (e != cudaSuccess) {
    cudaFreeHost(h);
    set_error(std::string("lcae_field_losses: ") + cudaGetErrorString(e));
    return LCAE_ERR_CUDA;
  }
  std::vector<double> tmp((size_t)g.F * 2);
  for (int f = 0; f < g.F; ++f)
    for (int q = 0; q < 2; ++q) {
      double a = 0.0;
      for (int c = 0; c < per; ++c) a += h[((size_t)f * per + c) * 2 + q];
      tmp[(size_t)f * 2 + q] = a;
    }
  cudaFreeHost(h);
  if (is_device_ptr(out)) LCAE_CK(cudaMemcpy(out, tmp.data(), tmp.size() * sizeof(double), cudaMemcpyHostToDevice));
  else memcpy(out, tmp.data(), tmp.size() * sizeof(double));
  return LCAE_OK;
}

lcae_status lcae_dx_device(lcae_layer *L, float **dx_dev) {
  if (!L || !dx_dev) { set_error("NULL argument"); return LCAE_ERR_ARG; }
  *dx_dev = L->dx_nhwc;
  return LCAE_OK;
}

lcae_status lcae_counters(lcae_layer *L, int64_t *steps, int64_t *reinit_rows) {
  if (!L) { set_error("NULL handle"); return LCAE_ERR_ARG; }
  int r = 0;
  int64_t st = 0;
  LCAE_CK(cudaMemcpyAsync(&r, L->reinit_dev, sizeof(int), cudaMemcpyDeviceToHost, L->st));
  LCAE_CK(cudaMemcpyAsync(&st, L->step_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, L->st));
  LCAE_CK(cudaStreamSynchronize(L->st));
  if (steps) *steps = st;
  if (reinit_rows) *reinit_rows = r;
  return LCAE_OK;
}

int32_t lcae_last_launch_count(lcae_layer *L) { return L ? L->launches : 0; }

lcae_status lcae_profile(lcae_layer *L, int32_t enable) {
  if (!L) { set_error("NULL handle"); return LCAE_ERR_ARG; }
  if (enable && !L->prof_ev) {
    L->prof_ev = new cudaEvent_t[2 * 4096];
    for (int i = 0; i < 2 * 4096; ++i) LCAE_CK(cudaEventCreate(&L->prof_ev[i]));
  }
  L->prof_on = enable ? 1 : 0;
  return LCAE_OK;
}

lcae_status lcae_profile_read(lcae_layer *L, double *main_kernel_ms, int32_t *launches) {
  if (!L) { set_error("NULL handle"); return LCAE_ERR_ARG; }
  double tot = 0.0;
  if (L->prof_n) LCAE_CK(cudaEventSynchronize(L->prof_ev[2 * L->prof_n - 1]));
  for (int i = 0; i < L->prof_n; ++i) {
    float ms = 0.f;
    LCAE_CK(cudaEventElapsedTime(&ms, L->prof_ev[2 * i], L->prof_ev[2 * i + 1]));
    tot += ms;
  }
  if (main_kernel_ms) *main_kernel_ms = tot;
  if (launches) *launches = L->prof_n;
  L->prof_n = 0;
  return LCAE_OK;
}

}  // extern "C"

// ---- dev hook (sanitizer substitute): count allocations whose 4 KB canary tail was overwritten (LCAE_DEV_CANARY)
extern "C" lcae_status lcae_dev_check_canaries(lcae_layer *L, int64_t *bad_allocs, int64_t *checked) {
  if (!L) { set_error("NULL handle"); return LCAE_ERR_ARG; }
  LCAE_CK(cudaDeviceSynchronize());
  std::vector<unsigned char> tail(CANARY_BYTES);
  int64_t bad = 0;
  for (auto &a : L->allocs) {
    LCAE_CK(cudaMemcpy(tail.data(), reinterpret_cast<char *>(a.first) + a.second, CANARY_BYTES, cudaMemcpyDeviceToHost));
    for (unsigned char c : tail)
      if (c != 0xA5) { ++bad; break; }
  }
  if (bad_allocs) *bad_allocs = bad;
  if (checked) *checked = (int64_t)L->allocs.size();
  return LCAE_OK;
}
