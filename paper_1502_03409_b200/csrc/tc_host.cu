// tc_host.cu — finalize kernel (alpha/b update, row scales, degenerate rows) and host launch code of the bf16
// tcgen05 step (kernel in tc_kernel.cuh).
#include <cfloat>
#include "tc_kernel.cuh"
#include "tma_host.cuh"

#include <vector>

namespace lcae {
namespace tc {

// alpha / b update from the cluster partials, new row scales sigma' = 1/||W~'_row||, degenerate rows.

__global__ void __launch_bounds__(128) finalize_kernel(Geo g, int CB, int n_al, const float *da_part,
                                                       const float *db_part, const float *rowsq_part, float *alpha,
                                                       float *bvec, float *sigma, float *W, __nv_bfloat16 *Wb,
                                                       float *va, float *vb, float lr, float mu, float amin,
                                                       float *galpha, float *gb, uint64_t seed, const int64_t *step_dev,
                                                       int row0, int col0, int ggc, int *reinit, float *vW, int wp,
                                                       const int *flags) {
  __shared__ double sh[32];
  __shared__ int bad[KP];
  __shared__ int nbad;
  if (flags[0] | flags[1]) return;   // the step kernel skipped this step (include/lcae.h "Errors")
  const int f = blockIdx.x, n = g.n, k = g.k;
  if (threadIdx.x == 0) {
    float da = 0.f;
    for (int c = 0; c < CB; ++c) da += da_part[(int64_t)f * CB + c];
    float ua = -lr * da;
    if (va) { ua = fmaf(mu, va[f], ua); va[f] = ua; }
    alpha[f] = fmaxf(alpha[f] + ua, amin);
    if (galpha) galpha[f] = da;
    nbad = 0;
  }
  const bool vec4 = (n & 3) == 0 &&
                    (((uintptr_t)db_part | (uintptr_t)bvec | (uintptr_t)vb | (uintptr_t)gb) & 15) == 0;
  if (vec4) {   // same arithmetic as the scalar loop below, four b entries per thread-iteration (16-byte accesses)
    const int n4 = n >> 2;
    for (int q = threadIdx.x; q < n4; q += blockDim.x) {
      float4 db = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int c = 0; c < CB; ++c) {
        const float4 p = reinterpret_cast<const float4 *>(db_part + ((int64_t)f * CB + c) * n)[q];
        db.x += p.x; db.y += p.y; db.z += p.z; db.w += p.w;
      }
      float4 ub = make_float4(-lr * db.x, -lr * db.y, -lr * db.z, -lr * db.w);
      const int64_t o4 = (int64_t)f * n4 + q;
      if (vb) {
        const float4 v = reinterpret_cast<const float4 *>(vb)[o4];
        ub = make_float4(fmaf(mu, v.x, ub.x), fmaf(mu, v.y, ub.y), fmaf(mu, v.z, ub.z), fmaf(mu, v.w, ub.w));
        reinterpret_cast<float4 *>(vb)[o4] = ub;
      }
      float4 bo = reinterpret_cast<const float4 *>(bvec)[o4];
      bo.x += ub.x; bo.y += ub.y; bo.z += ub.z; bo.w += ub.w;
      reinterpret_cast<float4 *>(bvec)[o4] = bo;
      if (gb) reinterpret_cast<float4 *>(gb)[o4] = db;
    }
  }
  for (int nn = vec4 ? n : threadIdx.x; nn < n; nn += blockDim.x) {
    float db = 0.f;
    for (int c = 0; c < CB; ++c) db += db_part[((int64_t)f * CB + c) * n + nn];
    float ub = -lr * db;
    const int64_t o = (int64_t)f * n + nn;
    if (vb) { ub = fmaf(mu, vb[o], ub); vb[o] = ub; }
    bvec[o] += ub;
    if (gb) gb[o] = db;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < k; r += blockDim.x) {
    float rs = 0.f;
    for (int c = 0; c < 2 * CB; ++c) rs += rowsq_part[((int64_t)f * 2 * CB + c) * KP + r];   // [F][CB][2 halves][KP]
    if (!(rs >= FLT_MIN)) {   // R13 in fp32: squared row norm below the smallest normal float
      int slot = atomicAdd(&nbad, 1);
      bad[slot] = r;
    } else {
      sigma[(int64_t)f * k + r] = rsqrtf(rs);
    }
  }
  __syncthreads();
  for (int ib = 0; ib < nbad; ++ib) {   // rare path: deterministic counter-based re-initialisation
    const int r = bad[ib];
    const int fr = f / g.gc, fc = f - fr * g.gc;
    const uint64_t gf = (uint64_t)((row0 + fr) * ggc + col0 + fc);
    const uint64_t key = splitmix64(seed ^ ((uint64_t)*step_dev << 40) ^ (gf << 20) ^ (uint64_t)r);
    double a2 = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      double u = (double)(splitmix64(key + (uint64_t)t) >> 40) / 16777216.0 - 0.5;
      a2 += u * u;
    }
    double tot = block_sum_f64(a2, sh);
    __shared__ float s_inv;
    if (threadIdx.x == 0) { s_inv = (float)(1.0 / sqrt(tot)); atomicAdd(reinit, 1); sigma[(int64_t)f * k + r] = 1.f; }
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      double u = (double)(splitmix64(key + (uint64_t)t) >> 40) / 16777216.0 - 0.5;
      float w = (float)u * s_inv;
      W[((int64_t)f * k + r) * n_al + t] = w;   // W~ rows use the same 16-byte pitch as the shadow
      Wb[((int64_t)f * KP + r) * n_al + t] = __float2bfloat16_rn(w);
      if (vW) vW[((int64_t)f * k + r) * wp + t] = 0.f;   // a fresh row starts at rest (no stale velocity)
    }
    __syncthreads();
  }
}

}  // namespace tc

struct TcScratch {
  int CB = 1, T = 0, grid = 0, trace_on = 0;
  unsigned long long *trace = nullptr;
  size_t smem = 0;
  double *loss_part = nullptr;
  float *da_part = nullptr, *db_part = nullptr, *rowsq_part = nullptr, *dbscr = nullptr;
  uint8_t *dscr = nullptr;
  CUtensorMap tmW;
  CUtensorMap tmX[tc::NXMAP];
  CUtensorMap tmD[tc::NDMAP];
  uint32_t *xpieces = nullptr, *dxpieces = nullptr;
};

// Pieces of the patch rows [r0, r0 + rows) of a field window: runs of consecutive image rows (one per receptive-field
// row) split into power-of-two boxes of at most 2^maxlg rows. Word: offset in the window, first row relative
// to r0, log2 height (tc::piece_word). Returns false if more than cap pieces are needed.
static bool window_pieces(const Geo &g, int r0, int rows, int maxlg, int cap, uint32_t *out) {
  int np = 0, r = 0;
  while (r < rows) {
    const int nn = r0 + r, ry = nn / g.RW;
    const int run = std::min(rows - r, (ry + 1) * g.RW - nn);
    int off = ry * g.W * g.C + (nn - ry * g.RW), left = run;
    while (left > 0) {
      int lg = maxlg;
      while ((1 << lg) > left) --lg;
      if (np >= cap) return false;
      out[np++] = tc::piece_word((uint32_t)off, (uint32_t)r, (uint32_t)lg);
      off += 1 << lg;
      r += 1 << lg;
      left -= 1 << lg;
    }
  }
  return true;
}

const char *tc_unsupported(const Geo &g) {
  if (g.k > tc::KP) return "filters per field must be <= 128";
  if (g.m > 2 * tc::MC) return "batch must be <= 256";
  if (cdiv(g.n, tc::NT) * tc::NT > tc::MAX_NPAD) return "rf_h*rf_w*C must be <= 4096";
  if ((int64_t)(g.rf_h - 1) * g.W * g.C + g.RW > (1 << 20)) return "field window spans > 2^20 pixel-features";
  return nullptr;
}

lcae_status tc_alloc(lcae_layer *L) {
  const Geo &g = L->geo;
  if (const char *why = tc_unsupported(g)) { set_error(std::string("bf16 fused kernel: ") + why); return LCAE_ERR_CONFIG; }
  const int T = cdiv(g.n, tc::NT);
  TcScratch *s = new TcScratch();
  L->tc = s;
  s->CB = cdiv(g.m, tc::MC);
  s->T = T;
  s->smem = sizeof(tc::Smem) + 1024;
  int ncl = std::max(1, std::min(g.F, L->sm_count / s->CB));
  // test hook: LCAE_DEV_MAX_CLUSTERS caps the persistent grid so that small layers run several fields per CTA
  // (the cross-field barrier phases and buffer reuse of the production kernel, checked against the oracle)
  if (const char *e = getenv("LCAE_DEV_MAX_CLUSTERS")) ncl = std::max(1, std::min(ncl, atoi(e)));
  s->grid = ncl * s->CB;
  LCAE_CK(dmalloc(L, &s->loss_part, (size_t)g.F * s->CB * 2 * sizeof(double)));
  LCAE_CK(dmalloc(L, &s->da_part, (size_t)g.F * s->CB * 4));
  LCAE_CK(dmalloc(L, &s->db_part, (size_t)g.F * s->CB * g.n * 4));
  LCAE_CK(dmalloc(L, &s->rowsq_part, (size_t)g.F * s->CB * 2 * tc::KP * 4));
  LCAE_CK(dmalloc(L, &s->dbscr, (size_t)s->grid * 4 * tc::MAX_NPAD * 4));   // per-CTA db partials (L2)
  LCAE_CK(dmalloc(L, &s->dscr, (size_t)s->grid * T * 16384));   // per-CTA pass-1 delta tiles (L2-resident)
  LCAE_CK(dmalloc(L, &s->trace, (64 + 256) * sizeof(unsigned long long)));
  LCAE_CK(cudaMemset(s->trace, 0, (64 + 256) * sizeof(unsigned long long)));
  // Wb is [F][KP][n_al] (pad rows zero) for the bf16 path
  cudaFree(L->Wb);
  LCAE_CK(dmalloc(L, &L->Wb, (size_t)g.F * tc::KP * L->n_al * 2));
  LCAE_CK(cudaMemset(L->Wb, 0, (size_t)g.F * tc::KP * L->n_al * 2));
  if (!make_tmap_2d_bf16(&s->tmW, L->Wb, (uint64_t)g.F * tc::KP, (uint64_t)L->n_al, (uint64_t)L->n_al, tc::KP)) {
    set_error("cuTensorMapEncodeTiled failed for W");
    return LCAE_ERR_CUDA;
  }
  // X gather: the HWCN bf16 image as [H*W*C rows][mp samples]; one map per power-of-two box height
  const uint64_t prow = (uint64_t)g.H * g.W * g.C;
  for (int i = 0; i < tc::NXMAP; ++i)
    if (!make_tmap_2d_bf16(&s->tmX[i], L->xt16, prow, (uint64_t)L->mp, (uint64_t)L->mp, 1u << i)) {
      set_error("cuTensorMapEncodeTiled failed for X");
      return LCAE_ERR_CUDA;
    }
  // per-tile pieces: runs of consecutive image rows (one per receptive-field row) split into 2^i-row boxes
  std::vector<uint32_t> pcs((size_t)T * tc::XPMAX, 0xFFFFFFFFu);
  for (int j = 0; j < T; ++j)
    if (!window_pieces(g, j * tc::NT, std::min(tc::NT, g.n - j * tc::NT), 6, tc::XPMAX, &pcs[(size_t)j * tc::XPMAX])) {
      set_error("bf16 path: too many X pieces per tile (rf_w*C too small)");
      return LCAE_ERR_CONFIG;
    }
  // dX reduce pieces per 16-column chunk of every tile (box heights <= 16)
  std::vector<uint32_t> dpc((size_t)T * 4 * tc::DXPMAX, 0xFFFFFFFFu);
  for (int j = 0; j < T; ++j)
    for (int q = 0; q < 4; ++q) {
      const int r0 = j * tc::NT + 16 * q, rows = std::min(16, g.n - r0);
      if (rows > 0 && !window_pieces(g, r0, rows, 4, tc::DXPMAX, &dpc[((size_t)j * 4 + q) * tc::DXPMAX])) {
        set_error("bf16 path: too many dX pieces per 16-row chunk");
        return LCAE_ERR_CONFIG;
      }
    }
  LCAE_CK(dmalloc(L, &s->dxpieces, dpc.size() * 4));
  LCAE_CK(cudaMemcpy(s->dxpieces, dpc.data(), dpc.size() * 4, cudaMemcpyHostToDevice));
  for (int i = 0; i < tc::NDMAP; ++i)
    if (!make_tmap_2d_f32(&s->tmD[i], L->dxt, prow, (uint64_t)L->mp, (uint64_t)L->mp, 1u << i, 32)) {
      set_error("cuTensorMapEncodeTiled failed for dX");
      return LCAE_ERR_CUDA;
    }
  LCAE_CK(dmalloc(L, &s->xpieces, pcs.size() * 4));
  LCAE_CK(cudaMemcpy(s->xpieces, pcs.data(), pcs.size() * 4, cudaMemcpyHostToDevice));
  return LCAE_OK;
}

void tc_free(lcae_layer *L) {
  if (!L->tc) return;
  TcScratch *s = L->tc;
  for (void *p : {(void *)s->loss_part, (void *)s->da_part, (void *)s->db_part, (void *)s->rowsq_part, (void *)s->trace, (void *)s->xpieces, (void *)s->dxpieces, (void *)s->dbscr, (void *)s->dscr})
    if (p) cudaFree(p);
  delete s;
  L->tc = nullptr;
}

lcae_status tc_step(lcae_layer *L, bool update, bool want_pooled, bool encode_only, const int *flist, int nfl,
                    bool first, bool last, int reserve_clusters) {
  const Geo &g = L->geo;
  TcScratch *s = L->tc;
  tc::Params P;
  P.tmW = s->tmW;
  for (int i = 0; i < tc::NXMAP; ++i) P.tmX[i] = s->tmX[i];
  P.xpieces = s->xpieces;
  for (int i = 0; i < tc::NDMAP; ++i) P.tmD[i] = s->tmD[i];
  P.dxpieces = s->dxpieces;
  P.g = g;
  P.T = s->T;
  P.mp = L->mp;
  P.CB = s->CB;
  P.n_al = L->n_al;
  P.wp = L->wp;
  P.mode = update ? 1 : (encode_only ? 2 : 0);
  P.dbg = getenv("LCAE_DEBUG_FLAGS") ? atoi(getenv("LCAE_DEBUG_FLAGS")) : 0;
  P.want_pooled = want_pooled ? 1 : 0;
  P.keep_grads = L->cfg.keep_grads;
  P.lam = L->cfg.lambda_;
  P.eps = L->cfg.eps;
  P.lr = L->cfg.lr;
  P.mu = L->cfg.momentum;
  P.xt = L->xt16;
  P.dxt = L->dxt;
  P.W = L->W;
  P.sigma = L->sigma;
  P.alpha = L->alpha;
  P.b = L->b;
  P.Wb = L->Wb;
  P.vW = L->vW;
  P.pooled = L->pooled;
  P.loss_part = s->loss_part;
  P.da_part = s->da_part;
  P.db_part = s->db_part;
  P.rowsq_part = s->rowsq_part;
  P.dbscr = s->dbscr;
  P.dscr = s->dscr;
  P.gW = L->gW;
  P.flags = L->flags_dev;
  P.flist = flist;
  P.nfl = nfl;
  P.trace = s->trace_on ? s->trace : nullptr;
  if (update && first) LCAE_CK(cudaMemsetAsync(L->dxt, 0, (size_t)g.H * g.W * g.C * L->mp * 4, L->st));
  if (flist && nfl == 0) return update && last ? tc_finalize(L) : LCAE_OK;
  cudaLaunchConfig_t cfg = {};
  // a model-parallel interior launch leaves `reserve_clusters` SM pairs free for the NCCL halo kernels
  const int ncl_all = s->grid / s->CB;
  const int ncl_use = std::max(1, std::min(ncl_all - reserve_clusters, flist ? nfl : g.F));
  cfg.gridDim = dim3(ncl_use * s->CB);
  cfg.blockDim = dim3(tc::NTHREADS);
  cfg.dynamicSmemBytes = s->smem;
  cfg.stream = L->st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = s->CB;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void (*kern)(tc::Params) = nullptr;
  // variant: training step lean (plain SGD, no kept gradients, no debug flags), full, or traced (full + wait
  // trace); forward / encode run the generic variant
  const int fl = !update ? 6 : s->trace_on ? 3 : ((L->vW || L->cfg.keep_grads || P.dbg) ? 2 : 0);
#define LCAE_PICK(GPV)                                                                                   \
  if (g.g == GPV) {                                                                                      \
    if (fl == 0) kern = s->CB == 1 ? tc::step_kernel<GPV, 1, 0> : tc::step_kernel<GPV, 2, 0>;             \
    else if (fl == 2) kern = s->CB == 1 ? tc::step_kernel<GPV, 1, 2> : tc::step_kernel<GPV, 2, 2>;        \
    else if (fl == 3) kern = s->CB == 1 ? tc::step_kernel<GPV, 1, 3> : tc::step_kernel<GPV, 2, 3>;        \
    else kern = s->CB == 1 ? tc::step_kernel<GPV, 1, 6> : tc::step_kernel<GPV, 2, 6>;                     \
  }
  LCAE_PICK(1) LCAE_PICK(2) LCAE_PICK(4) LCAE_PICK(8) LCAE_PICK(16) LCAE_PICK(32)
#undef LCAE_PICK
  if (!kern) { set_error("unsupported pool group"); return LCAE_ERR_CONFIG; }
  LCAE_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem));
  const bool prof = L->prof_on && L->prof_n < 4096;
  if (prof) LCAE_CK(cudaEventRecord(L->prof_ev[2 * L->prof_n], L->st));
  LCAE_CK(cudaLaunchKernelEx(&cfg, kern, P));
  LCAE_CK_LAUNCH(L);
  if (prof) LCAE_CK(cudaEventRecord(L->prof_ev[2 * L->prof_n++ + 1], L->st));
  if (update && last) return tc_finalize(L);
  return LCAE_OK;
}

lcae_status tc_finalize(lcae_layer *L) {
  const Geo &g = L->geo;
  TcScratch *s = L->tc;
  {
    tc::finalize_kernel<<<g.F, 128, 0, L->st>>>(
        g, s->CB, L->n_al, s->da_part, s->db_part, s->rowsq_part, L->alpha, L->b, L->sigma, L->W, L->Wb, L->va,
        L->vb, L->cfg.lr, L->cfg.momentum, L->cfg.alpha_min, L->cfg.keep_grads ? L->galpha : nullptr,
        L->cfg.keep_grads ? L->gb : nullptr, L->cfg.seed, L->step_dev, L->cfg.field_row0, L->cfg.field_col0,
        L->cfg.global_grid_c, L->reinit_dev, L->vW, L->wp, L->flags_dev);
    LCAE_CK_LAUNCH(L);
  }
  return LCAE_OK;
}

double *tc_loss_part(lcae_layer *L) { return L->tc ? L->tc->loss_part : nullptr; }
int tc_loss_count(lcae_layer *L) { return L->tc ? L->geo.F * L->tc->CB : 0; }

}  // namespace lcae

// ---- dev hook: per-role barrier-wait cycle trace of the fused step kernel (summed over CTAs)
extern "C" lcae_status lcae_dev_trace(lcae_layer *L, int enable, unsigned long long *out32) {
  using namespace lcae;
  if (!L || !L->tc) { set_error("lcae_dev_trace: bf16 layer required"); return LCAE_ERR_ARG; }
  if (out32) {
    LCAE_CK(cudaStreamSynchronize(L->st));
    LCAE_CK(cudaMemcpy(out32, L->tc->trace, (64 + 256) * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    LCAE_CK(cudaMemset(L->tc->trace, 0, (64 + 256) * sizeof(unsigned long long)));
  }
  L->tc->trace_on = enable ? 1 : 0;
  return LCAE_OK;
}
