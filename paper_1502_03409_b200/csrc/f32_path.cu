// f32_path.cu — the fp32 SIMT step (FFMA only, no TF32), used for the 1e-5 parity path.
//
// Per chunk of Fc fields the step runs as batched SIMT GEMMs with small epilogue kernels; every
// per-field intermediate lives in chunk scratch (bounded memory).  Notation: PAPER.md:88 / DESIGN.md R1-R11.
//   U  = W X_f                  (k x m)    encode            h = alpha U
//   s  = sqrt(eps + sum_G h^2)  p = s      pooling/sparsity  J_s = lambda sum s
//   R  = W^T h                  (n x m)    decode            e = R + b - X_f, J_r = sum e^2, delta = 2e
//   G  = W delta                (k x m)                      D = G + lambda h/s, dalpha = sum D.U
//   dW = h delta^T + alpha D X_f^T                           db = sum_i delta
//   dXp = alpha W^T D - delta   (n x m)    -> overlap-add (deterministic pixel gather) into dX
//   projected SGD update of the chunk's fields.
#include "common.cuh"

namespace lcae {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;

// Operand accessors: value at (batch b, row i, col j).
struct Strided {
  const float *p;
  int64_t bs, rs, cs;
  __device__ float operator()(int b, int i, int j) const { return p[b * bs + i * rs + j * cs]; }
};
// Patch X_f as an (n x m) matrix read straight from the HWCN image: rows n = (ry, rx, c), cols = samples.
struct Patch {
  const float *xt;
  int f0, gc, RW, m;
  int64_t SRC_R, SRC_C, SY;
  __device__ float operator()(int b, int row, int col) const {
    int f = f0 + b, r = f / gc, c = f - r * gc;
    int ry = row / RW;
    return xt[r * SRC_R + c * SRC_C + ry * SY + (int64_t)(row - ry * RW) * m + col];
  }
};
// Transposed patch (m x n).
struct PatchT {
  Patch P;
  __device__ float operator()(int b, int i, int j) const { return P(b, j, i); }
};

// C[b] = scale_b * A[b] B[b] + beta * C0[b]   (M x N, inner K); 256 threads, 64x64 tile, 4x4 per thread.
template <class OpA, class OpB, bool ROWS_A_CONTIG, bool ROWS_B_CONTIG>
__global__ void __launch_bounds__(256) sgemm_batched(int M, int N, int K, OpA A, OpB B, float *C, int64_t cbs,
                                                     int64_t crs, int64_t ccs, const float *scale, float beta,
                                                     const float *C0, int64_t c0bs, int64_t c0rs, int64_t c0cs) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int b = blockIdx.z, m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int e = tid + 256 * q;
      int row, kk;
      if (ROWS_A_CONTIG) { row = e & 63; kk = e >> 6; } else { row = e >> 4; kk = e & 15; }
      As[kk][row] = (m0 + row < M && k0 + kk < K) ? A(b, m0 + row, k0 + kk) : 0.f;
      int col, kb;
      if (ROWS_B_CONTIG) { kb = e & 15; col = e >> 4; } else { kb = e >> 6; col = e & 63; }
      Bs[kb][col] = (n0 + col < N && k0 + kb < K) ? B(b, k0 + kb, n0 + col) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], bb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { a[u] = As[kk][ty * 4 + u]; bb[u] = Bs[kk][tx * 4 + u]; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(a[u], bb[v], acc[u][v]);
    }
    __syncthreads();
  }
  const float sc = scale ? scale[b] : 1.f;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    int i = m0 + ty * 4 + u;
    if (i >= M) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      int j = n0 + tx * 4 + v;
      if (j >= N) continue;
      float o = sc * acc[u][v];
      if (C0) o = fmaf(beta, C0[b * c0bs + i * c0rs + j * c0cs], o);
      C[b * cbs + i * crs + j * ccs] = o;
    }
  }
}

// The same contract on 128 x 128 tiles, 8 x 8 accumulators per thread (two 4 x 4 quadrants 64 rows / columns
// apart, read with 16-byte shared loads), K in steps of 8 with the next step's operands loaded into registers
// while the current one computes. Used when M, N >= 128 (the paper-exact layers, k = 384 / 4096).
constexpr int BM = 128, BN = 128, BK = 8;
template <class OpA, class OpB, bool ROWS_A_CONTIG, bool ROWS_B_CONTIG>
__global__ void __launch_bounds__(256) sgemm_big(int M, int N, int K, OpA A, OpB B, float *C, int64_t cbs,
                                                 int64_t crs, int64_t ccs, const float *scale, float beta,
                                                 const float *C0, int64_t c0bs, int64_t c0rs, int64_t c0cs) {
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];
  const int b = blockIdx.z, m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  float acc[8][8] = {};
  float ra[4], rb[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + 256 * q;
      int row, kk;
      if (ROWS_A_CONTIG) { row = e & 127; kk = e >> 7; } else { row = e >> 3; kk = e & 7; }
      ra[q] = (m0 + row < M && k0 + kk < K) ? A(b, m0 + row, k0 + kk) : 0.f;
      int col, kb;
      if (ROWS_B_CONTIG) { kb = e & 7; col = e >> 3; } else { kb = e >> 7; col = e & 127; }
      rb[q] = (n0 + col < N && k0 + kb < K) ? B(b, k0 + kb, n0 + col) : 0.f;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + 256 * q;
      int row, kk;
      if (ROWS_A_CONTIG) { row = e & 127; kk = e >> 7; } else { row = e >> 3; kk = e & 7; }
      As[kk][row] = ra[q];
      int col, kb;
      if (ROWS_B_CONTIG) { kb = e & 7; col = e >> 3; } else { kb = e >> 7; col = e & 127; }
      Bs[kb][col] = rb[q];
    }
  };
  load(0);
  for (int k0 = 0; k0 < K; k0 += BK) {
    store();
    __syncthreads();
    if (k0 + BK < K) load(k0 + BK);   // next step's operands in flight during this step's FFMAs
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4 *>(&As[kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4 *>(&As[kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[kk][64 + tx * 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[u][v] = fmaf(av[u], bv[v], acc[u][v]);
    }
    __syncthreads();
  }
  const float sc = scale ? scale[b] : 1.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int i = m0 + (u < 4 ? ty * 4 + u : 64 + ty * 4 + u - 4);
    if (i >= M) continue;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int j = n0 + (v < 4 ? tx * 4 + v : 64 + tx * 4 + v - 4);
      if (j >= N) continue;
      float o = sc * acc[u][v];
      if (C0) o = fmaf(beta, C0[b * c0bs + i * c0rs + j * c0cs], o);
      C[b * cbs + i * crs + j * ccs] = o;
    }
  }
}

template <bool RA, bool RB, class OpA, class OpB>
lcae_status gemm(lcae_layer *L, int batch, int M, int N, int K, OpA A, OpB B, float *C, int64_t cbs, int64_t crs,
                 int64_t ccs, const float *scale = nullptr, float beta = 0.f, const float *C0 = nullptr,
                 int64_t c0bs = 0, int64_t c0rs = 0, int64_t c0cs = 0) {
  if (M >= BM && N >= BN) {
    dim3 grid(cdiv(N, BN), cdiv(M, BM), batch);
    sgemm_big<OpA, OpB, RA, RB><<<grid, 256, 0, L->st>>>(M, N, K, A, B, C, cbs, crs, ccs, scale, beta, C0, c0bs,
                                                        c0rs, c0cs);
    LCAE_CK_LAUNCH(L);
    return LCAE_OK;
  }
  dim3 grid(cdiv(N, TN), cdiv(M, TM), batch);
  sgemm_batched<OpA, OpB, RA, RB><<<grid, 256, 0, L->st>>>(M, N, K, A, B, C, cbs, crs, ccs, scale, beta, C0, c0bs,
                                                          c0rs, c0cs);
  LCAE_CK_LAUNCH(L);
  return LCAE_OK;
}

// Pooling + sparsity epilogue: h = alpha U; s_G = sqrt(eps + sum_G h^2); p = s; Q = lambda h / s.
__global__ void __launch_bounds__(256) pool_f32(Geo g, int f0, const float *U, const float *alpha, float lam,
                                                float eps, float *H, float *Q, float *pooled, double *loss_part) {
  __shared__ double sh[32];
  const int b = blockIdx.x, f = f0 + b;
  const int k = g.k, m = g.m, gs = g.g, ng = k / gs;
  const float a = alpha[f];
  const float *Ub = U + (int64_t)b * k * m;
  double acc = 0.0;
  for (int t = threadIdx.x; t < ng * m; t += blockDim.x) {
    int G = t / m, i = t - G * m;
    float ss = 0.f;
    for (int q = 0; q < gs; ++q) {
      float h = a * Ub[(G * gs + q) * m + i];
      ss = fmaf(h, h, ss);
    }
    float s = sqrtf(eps + ss);
    acc += (double)s;
    if (pooled) {
      int r = f / g.gc, c = f - r * g.gc;
      pooled[(((int64_t)i * g.gr + r) * g.gc + c) * ng + G] = s;
    }
    float inv = s > 0.f ? lam / s : 0.f;
    for (int q = 0; q < gs; ++q) {
      int j = G * gs + q;
      float h = a * Ub[j * m + i];
      H[(int64_t)b * k * m + j * m + i] = h;
      Q[(int64_t)b * k * m + j * m + i] = h * inv;
    }
  }
  double t = block_sum_f64(acc, sh);
  if (threadIdx.x == 0) loss_part[2 * f + 1] = (double)lam * t;
}

// Residual epilogue: e = R + b - X_f; J_r = sum e^2; delta = 2e (in place); db = sum_i delta.
__global__ void __launch_bounds__(256) resid_f32(Geo g, int f0, float *R, const float *bvec, Patch X,
                                                 double *loss_part, float *db) {
  __shared__ double sh[32];
  const int b = blockIdx.x, f = f0 + b, n = g.n, m = g.m;
  float *Rb = R + (int64_t)b * n * m;
  const float *bf = bvec + (int64_t)f * n;
  double acc = 0.0;
  for (int t = threadIdx.x; t < n * m; t += blockDim.x) {
    int row = t / m, i = t - row * m;
    float e = Rb[t] + bf[row] - X(b, row, i);
    acc += (double)e * (double)e;
    Rb[t] = 2.f * e;
  }
  double tot = block_sum_f64(acc, sh);
  if (threadIdx.x == 0) loss_part[2 * f] = tot;
  __syncthreads();
  for (int row = threadIdx.x; row < n; row += blockDim.x) {
    float s = 0.f;
    for (int i = 0; i < m; ++i) s += Rb[row * m + i];
    db[(int64_t)b * n + row] = s;
  }
}

// D = G + Q (in place in G); dalpha = sum D (.) U.
__global__ void __launch_bounds__(256) dcode_f32(Geo g, float *Gm, const float *Q, const float *U, float *da) {
  __shared__ double sh[32];
  const int b = blockIdx.x, km = g.k * g.m;
  float *Gb = Gm + (int64_t)b * km;
  const float *Qb = Q + (int64_t)b * km, *Ub = U + (int64_t)b * km;
  double acc = 0.0;
  for (int t = threadIdx.x; t < km; t += blockDim.x) {
    float d = Gb[t] + Qb[t];
    Gb[t] = d;
    acc += (double)d * (double)Ub[t];
  }
  double tot = block_sum_f64(acc, sh);
  if (threadIdx.x == 0) da[b] = (float)tot;
}

// Projected SGD on W rows (fp32 mode keeps W normalised, sigma == 1):
// v = mu v - lr dW; W' = W + v; W' /= ||W'|| (degenerate rows re-initialised).
__global__ void __launch_bounds__(256) update_w_f32(Geo g, int f0, float *W, const float *dW, float *vW, float lr,
                                                    float mu, uint64_t seed, const int64_t *step_dev, int row0, int col0,
                                                    int ggc, int *reinit, const int *flags) {
  __shared__ double sh[32];
  __shared__ float s_scale;
  if (flags[0] | flags[1]) return;   // flagged error: parameters frozen (include/lcae.h "Errors")
  const int b = blockIdx.x, j = blockIdx.y, f = f0 + b, n = g.n;
  float *w = W + ((int64_t)f * g.k + j) * n;
  const float *d = dW + ((int64_t)b * g.k + j) * n;
  float *v = vW ? vW + ((int64_t)f * g.k + j) * n : nullptr;
  double acc = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    float upd = -lr * d[t];
    if (v) { upd = fmaf(mu, v[t], upd); v[t] = upd; }
    float wn = w[t] + upd;
    w[t] = wn;
    acc += (double)wn * wn;
  }
  double tot = block_sum_f64(acc, sh);
  if (threadIdx.x == 0) s_scale = tot < 1e-60 ? -1.f : (float)(1.0 / sqrt(tot));
  __syncthreads();
  float sc = s_scale;
  if (sc < 0.f) {   // degenerate row: deterministic counter-based re-initialisation
    int r = f / g.gc, c = f - r * g.gc;
    uint64_t gf = (uint64_t)((row0 + r) * ggc + col0 + c);
    uint64_t key = splitmix64(seed ^ ((uint64_t)*step_dev << 40) ^ (gf << 20) ^ (uint64_t)j);
    double a2 = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      double u = (double)(splitmix64(key + (uint64_t)t) >> 40) / 16777216.0 - 0.5;
      w[t] = (float)u;
      if (v) v[t] = 0.f;   // a fresh row starts at rest (no stale velocity)
      a2 += u * u;
    }
    double tt = block_sum_f64(a2, sh);
    if (threadIdx.x == 0) { s_scale = (float)(1.0 / sqrt(tt)); atomicAdd(reinit, 1); }
    __syncthreads();
    sc = s_scale;
  }
  for (int t = threadIdx.x; t < n; t += blockDim.x) w[t] *= sc;
}

__global__ void copy_grads_f32(Geo g, int f0, int Fc, const float *dW, const float *da, const float *db, float *gW,
                               float *ga, float *gb) {
  int64_t kn = (int64_t)g.k * g.n, tot = (int64_t)Fc * kn;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    gW[(int64_t)f0 * kn + t] = dW[t];
    if (t < (int64_t)Fc * g.n) gb[(int64_t)f0 * g.n + t] = db[t];
    if (t < Fc) ga[f0 + t] = da[t];
  }
}

}  // namespace

// Overlap-add by owner gather (deterministic): dxt[y][x][c][i] += sum over fields f in [f0, f0+Fc) covering
// (y, x) of dXp[f - f0][n(y,x,c,f)][i], fields visited in row-major order.
// Only the band of image rows the chunk's fields cover is visited (fields are chunked in row-major order).
__global__ void col2im_f32(Geo g, int f0, int Fc, const float *dXp, float *dxt) {
  const int y0 = (f0 / g.gc) * g.s, y1 = min(g.H, ((f0 + Fc - 1) / g.gc) * g.s + g.rf_h);
  const int64_t base = (int64_t)y0 * g.W * g.C * g.m, total = (int64_t)(y1 - y0) * g.W * g.C * g.m;
  for (int64_t tt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; tt < total; tt += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = base + tt;
    int i = (int)(t % g.m);
    int64_t pix = t / g.m;
    int ch = (int)(pix % g.C);
    int64_t yx = pix / g.C;
    int x = (int)(yx % g.W), y = (int)(yx / g.W);
    int r_lo = y - g.rf_h + 1 <= 0 ? 0 : (y - g.rf_h + g.s) / g.s;
    int r_hi = min(y / g.s, g.gr - 1);
    int c_lo = x - g.rf_w + 1 <= 0 ? 0 : (x - g.rf_w + g.s) / g.s;
    int c_hi = min(x / g.s, g.gc - 1);
    float acc = 0.f;
    bool any = false;
    for (int r = r_lo; r <= r_hi; ++r) {
      for (int c = c_lo; c <= c_hi; ++c) {
        int f = r * g.gc + c;
        if (f < f0 || f >= f0 + Fc) continue;
        int nrow = ((y - r * g.s) * g.rf_w + (x - c * g.s)) * g.C + ch;
        acc += dXp[((int64_t)(f - f0) * g.n + nrow) * g.m + i];
        any = true;
      }
    }
    if (any) dxt[t] += acc;
  }
}

__global__ void update_ab_f32(Geo g, int f0, int Fc, float *alpha, float *bvec, const float *da, const float *db,
                              float *va, float *vb, float lr, float mu, float amin, const int *flags) {
  if (flags[0] | flags[1]) return;
  int64_t tot = (int64_t)Fc * g.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    int b = (int)(t / g.n), row = (int)(t - (int64_t)b * g.n), f = f0 + b;
    float upd = -lr * db[t];
    if (vb) { upd = fmaf(mu, vb[(int64_t)f * g.n + row], upd); vb[(int64_t)f * g.n + row] = upd; }
    bvec[(int64_t)f * g.n + row] += upd;
    if (row == 0) {
      float ua = -lr * da[b];
      if (va) { ua = fmaf(mu, va[f], ua); va[f] = ua; }
      alpha[f] = fmaxf(alpha[f] + ua, amin);
    }
  }
}

lcae_status f32_alloc(lcae_layer *L) {
  const Geo &g = L->geo;
  // chunk so that the per-chunk scratch stays below ~768 MiB
  int64_t per_field = 4ll * g.k * g.m + 2ll * g.n * g.m + (int64_t)g.k * g.n + g.n + 1;
  int64_t cap = (768ll << 20) / (4 * per_field);
  int Fc = (int)std::max<int64_t>(1, std::min<int64_t>(cap, g.F));
  F32Scratch &s = L->f32;
  s.Fc = Fc;
  size_t km = (size_t)Fc * g.k * g.m, nm = (size_t)Fc * g.n * g.m;
  LCAE_CK(dmalloc(L, &s.U, km * 4));
  LCAE_CK(dmalloc(L, &s.H, km * 4));
  LCAE_CK(dmalloc(L, &s.Q, km * 4));
  LCAE_CK(dmalloc(L, &s.G, km * 4));
  LCAE_CK(dmalloc(L, &s.R, nm * 4));
  LCAE_CK(dmalloc(L, &s.dXp, nm * 4));
  LCAE_CK(dmalloc(L, &s.dW, (size_t)Fc * g.k * g.n * 4));
  LCAE_CK(dmalloc(L, &s.da, (size_t)Fc * 4));
  LCAE_CK(dmalloc(L, &s.db, (size_t)Fc * g.n * 4));
  return LCAE_OK;
}

void f32_free(lcae_layer *L) {
  F32Scratch &s = L->f32;
  for (float *p : {s.U, s.H, s.Q, s.G, s.R, s.dXp, s.dW, s.da, s.db}) cudaFree(p);
  s = F32Scratch{};
}

lcae_status f32_step(lcae_layer *L, bool update, bool want_pooled) {
  const Geo &g = L->geo;
  F32Scratch &s = L->f32;
  const int k = g.k, n = g.n, m = g.m;
  const int64_t km = (int64_t)k * m, nm = (int64_t)n * m, kn = (int64_t)k * n;
  lcae_status st;
#define TRY(x) do { if ((st = (x)) != LCAE_OK) return st; } while (0)
  LCAE_CK(cudaMemsetAsync(L->dxt, 0, (size_t)g.H * g.W * g.C * L->mp * 4, L->st));
  for (int f0 = 0; f0 < g.F; f0 += s.Fc) {
    const int Fc = std::min(s.Fc, g.F - f0);
    Patch X{L->xt32, f0, g.gc, g.RW, m, g.SRC_R, g.SRC_C, g.SY};
    Strided Wk{L->W + (int64_t)f0 * kn, kn, n, 1};        // W (k x n)
    Strided Wt{L->W + (int64_t)f0 * kn, kn, 1, n};        // W^T (n x k)
    // encode U = W X_f
    TRY((gemm<false, false>(L, Fc, k, m, n, Wk, X, s.U, km, m, 1)));
    pool_f32<<<Fc, 256, 0, L->st>>>(g, f0, s.U, L->alpha, L->cfg.lambda_, L->cfg.eps, s.H, s.Q,
                                    want_pooled ? L->pooled : nullptr, L->loss_part);
    LCAE_CK_LAUNCH(L);
    // decode R = W^T h
    TRY((gemm<true, false>(L, Fc, n, m, k, Wt, Strided{s.H, km, m, 1}, s.R, nm, m, 1)));
    resid_f32<<<Fc, 256, 0, L->st>>>(g, f0, s.R, L->b, X, L->loss_part, s.db);
    LCAE_CK_LAUNCH(L);
    if (!update) continue;
    // backprop into the code: G = W delta; D = G + lambda h/s; dalpha
    TRY((gemm<false, false>(L, Fc, k, m, n, Wk, Strided{s.R, nm, m, 1}, s.G, km, m, 1)));
    dcode_f32<<<Fc, 256, 0, L->st>>>(g, s.G, s.Q, s.U, s.da);
    LCAE_CK_LAUNCH(L);
    // weight gradient dW = h delta^T + alpha D X_f^T
    TRY((gemm<false, true>(L, Fc, k, n, m, Strided{s.H, km, m, 1}, Strided{s.R, nm, 1, m}, s.dW, kn, n, 1)));
    TRY((gemm<false, true>(L, Fc, k, n, m, Strided{s.G, km, m, 1}, PatchT{X}, s.dW, kn, n, 1, L->alpha + f0, 1.f,
                            s.dW, kn, n, 1)));
    // input gradient dXp = alpha W^T D - delta, overlap-added into dX
    TRY((gemm<true, false>(L, Fc, n, m, k, Wt, Strided{s.G, km, m, 1}, s.dXp, nm, m, 1, L->alpha + f0, -1.f, s.R,
                          nm, m, 1)));
    col2im_f32<<<L->sm_count * 8, 256, 0, L->st>>>(g, f0, Fc, s.dXp, L->dxt);
    LCAE_CK_LAUNCH(L);
    if (L->cfg.keep_grads) {
      copy_grads_f32<<<1024, 256, 0, L->st>>>(g, f0, Fc, s.dW, s.da, s.db, L->gW, L->galpha, L->gb);
      LCAE_CK_LAUNCH(L);
    }
    // projected SGD update of this chunk's fields
    update_w_f32<<<dim3(Fc, k), 256, 0, L->st>>>(g, f0, L->W, s.dW, L->vW, L->cfg.lr, L->cfg.momentum, L->cfg.seed,
                                                 L->step_dev, L->cfg.field_row0, L->cfg.field_col0,
                                                 L->cfg.global_grid_c, L->reinit_dev, L->flags_dev);
    LCAE_CK_LAUNCH(L);
    update_ab_f32<<<256, 256, 0, L->st>>>(g, f0, Fc, L->alpha, L->b, s.da, s.db, L->va, L->vb, L->cfg.lr,
                                          L->cfg.momentum, L->cfg.alpha_min, L->flags_dev);
    LCAE_CK_LAUNCH(L);
  }
#undef TRY
  return LCAE_OK;
}

}  // namespace lcae
