// aux.cu — layout conversion, loss reduction, parameter init/readback and the halo overlap-add kernel.
// All HBM-bound; grid-stride loops sized to a multiple of the SM count.
#include "common.cuh"

namespace lcae {
namespace {

// NHWC [m][P] -> HWCN [P][m] (P = H*W*C): 32x32 tiled transpose through shared memory.
// Any non-finite input element sets flag[0] ("non-finite ... error"; include/lcae.h LCAE_ERR_DATA).
template <typename T>
__global__ void nhwc_to_hwcn(const float *__restrict__ x, T *__restrict__ xt, int m, int mp, int64_t P, int *flag) {
  __shared__ float tile[32][33];
  const int64_t p0 = (int64_t)blockIdx.x * 32;
  const int i0 = blockIdx.y * 32;
  bool bad = false;
  for (int r = threadIdx.y; r < 32; r += 8) {
    int i = i0 + r;
    int64_t p = p0 + threadIdx.x;
    const float v = (i < m && p < P) ? x[(int64_t)i * P + p] : 0.f;
    bad |= !isfinite(v);
    tile[r][threadIdx.x] = v;
  }
  if (bad) flag[0] = 1;
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    int64_t p = p0 + r;
    int i = i0 + threadIdx.x;
    if (i < m && p < P) {
      float v = tile[threadIdx.x][r];
      if constexpr (sizeof(T) == 2) xt[p * mp + i] = __float2bfloat16_rn(v);
      else xt[p * mp + i] = v;
    }
  }
}

// Vectorised 64 x 64 variants (16-byte global accesses on both sides; used when P % 4 == 0):
// NHWC f32 [m][P] -> HWCN bf16 [P][mp] (sample rows in [m, mp) written as zeros).
__global__ void __launch_bounds__(256) nhwc_to_hwcn_bf16_v(const float *__restrict__ x, __nv_bfloat16 *__restrict__ xt,
                                                           int m, int mp, int64_t P, int *flag) {
  __shared__ float tile[64][65];   // [sample][pixel-feature]
  const int64_t p0 = (int64_t)blockIdx.x * 64;
  const int i0 = blockIdx.y * 64, t = threadIdx.x;
  bool bad = false;
  for (int r = t / 16; r < 64; r += 16) {   // 16 lanes x float4 = 64 pixel-features of one sample
    const int i = i0 + r, c4 = t % 16;
    const int64_t p = p0 + 4 * c4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < m && p < P) v = __ldg(reinterpret_cast<const float4 *>(x + (int64_t)i * P + p));
    bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
    tile[r][4 * c4] = v.x;
    tile[r][4 * c4 + 1] = v.y;
    tile[r][4 * c4 + 2] = v.z;
    tile[r][4 * c4 + 3] = v.w;
  }
  if (bad) flag[0] = 1;   // benign race: every writer stores the same value
  __syncthreads();
  for (int q = t / 8; q < 64; q += 32) {   // 8 lanes x 8 bf16 = 64 samples of one pixel-feature
    const int g8 = t % 8, i = i0 + 8 * g8;
    const int64_t p = p0 + q;
    if (p >= P || i >= mp) continue;
    uint4 o;
    uint32_t *w = reinterpret_cast<uint32_t *>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float a = i + 2 * e < m ? tile[8 * g8 + 2 * e][q] : 0.f;
      const float b = i + 2 * e + 1 < m ? tile[8 * g8 + 2 * e + 1][q] : 0.f;
      __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
      w[e] = *reinterpret_cast<uint32_t *>(&h);
    }
    *reinterpret_cast<uint4 *>(xt + p * mp + i) = o;
  }
}

// HWCN f32 [P][mp] -> NHWC f32 [m][P]
__global__ void __launch_bounds__(256) hwcn_to_nhwc_v(const float *__restrict__ xt, float *__restrict__ x, int m, int mp,
                                                      int64_t P) {
  __shared__ float tile[64][65];   // [pixel-feature][sample]
  const int64_t p0 = (int64_t)blockIdx.x * 64;
  const int i0 = blockIdx.y * 64, t = threadIdx.x;
  for (int r = t / 16; r < 64; r += 16) {   // 16 lanes x float4 = 64 samples of one pixel-feature
    const int64_t p = p0 + r;
    const int c4 = t % 16, i = i0 + 4 * c4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p < P && i < mp) v = __ldg(reinterpret_cast<const float4 *>(xt + p * mp + i));
    tile[r][4 * c4] = v.x;
    tile[r][4 * c4 + 1] = v.y;
    tile[r][4 * c4 + 2] = v.z;
    tile[r][4 * c4 + 3] = v.w;
  }
  __syncthreads();
  for (int q = t / 16; q < 64; q += 16) {   // 16 lanes x float4 = 64 pixel-features of one sample
    const int i = i0 + q, c4 = t % 16;
    const int64_t p = p0 + 4 * c4;
    if (i >= m || p >= P) continue;
    *reinterpret_cast<float4 *>(x + (int64_t)i * P + p) =
        make_float4(tile[4 * c4][q], tile[4 * c4 + 1][q], tile[4 * c4 + 2][q], tile[4 * c4 + 3][q]);
  }
}

__global__ void hwcn_to_nhwc(const float *__restrict__ xt, float *__restrict__ x, int m, int mp, int64_t P) {
  __shared__ float tile[32][33];
  const int64_t p0 = (int64_t)blockIdx.x * 32;
  const int i0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    int64_t p = p0 + r;
    int i = i0 + threadIdx.x;
    tile[r][threadIdx.x] = (i < m && p < P) ? xt[p * mp + i] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    int i = i0 + r;
    int64_t p = p0 + threadIdx.x;
    if (i < m && p < P) x[(int64_t)i * P + p] = tile[threadIdx.x][r];
  }
}

// Fixed-order fp64 reduction of the per-field loss partials [F][2] -> loss[2]. A step skipped because an error
// flag was set (flags[0] by this step's staging, or either flag earlier; flags[1] is only set here) does not
// count; a non-finite loss sets flags[1].
__global__ void __launch_bounds__(1024) loss_reduce(const double *part, int F, double *out, int64_t *step_dev,
                                                    int update, int *flags) {
  __shared__ double sh[32];
  double a = 0.0, b = 0.0;
  const double2 *p2 = reinterpret_cast<const double2 *>(part);   // [F] pairs, 16-byte aligned (cudaMalloc)
#pragma unroll 4
  for (int f = threadIdx.x; f < F; f += blockDim.x) { const double2 v = p2[f]; a += v.x; b += v.y; }
  double ta = block_sum_f64(a, sh);
  __syncthreads();
  double tb = block_sum_f64(b, sh);
  if (threadIdx.x == 0) {
    out[0] = ta;
    out[1] = tb;
    if (!(flags[0] | flags[1])) {
      if (!isfinite(ta + tb)) flags[1] = 1;
      if (update) ++*step_dev;   // after this step's finalize (stream order), before the next step's
    }
  }
}

// Default init: counter-based uniform rows (unit length), alpha = alpha_init, b = 0, sigma = 1. Keyed by the GLOBAL
// field id (row0 + r) * ggc + col0 + c, so a model-parallel tile starts from the untiled layer's weights.
__global__ void __launch_bounds__(256) init_rows(Geo g, int wp, float *W, float *sigma, uint64_t seed, int row0,
                                                 int col0, int ggc) {
  __shared__ double sh[32];
  __shared__ float s_sc;
  const int f = blockIdx.x, j = blockIdx.y;
  float *w = W + ((int64_t)f * g.k + j) * wp;
  const int fr = f / g.gc, fc = f - fr * g.gc;
  const uint64_t gf = (uint64_t)((row0 + fr) * ggc + col0 + fc);
  uint64_t key = splitmix64(seed ^ 0x5EEDull ^ (gf << 20) ^ (uint64_t)j);
  double acc = 0.0;
  for (int t = threadIdx.x; t < g.n; t += blockDim.x) {
    float u = (float)((double)(splitmix64(key + t) >> 40) / 16777216.0 - 0.5);
    w[t] = u;
    acc += (double)u * u;
  }
  double tot = block_sum_f64(acc, sh);
  if (threadIdx.x == 0) s_sc = (float)(1.0 / sqrt(tot));
  __syncthreads();
  for (int t = threadIdx.x; t < g.n; t += blockDim.x) w[t] *= s_sc;
  if (threadIdx.x == 0) sigma[(int64_t)f * g.k + j] = 1.f;
}

__global__ void fill_f32(float *p, int64_t n, float v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) p[t] = v;
}

// W_out[f][j][t] = sigma[f][j] * W~[f][j][t] for fields [f0, f0 + nf) (W, sigma already offset to f0)
__global__ void get_w(Geo g, int wp, const float *W, const float *sigma, float *out, int64_t nf) {
  const int64_t tot = nf * g.k * g.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / g.n;
    out[t] = W[row * wp + (t - row * g.n)] * sigma[row];
  }
}

// bf16 shadow [F][kp][n_al] of W~ (pad rows and columns zero).
__global__ void shadow_w(Geo g, int kp, int n_al, int wp, const float *W, __nv_bfloat16 *Wb) {
  const int64_t tot = (int64_t)g.F * kp * n_al;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = t / n_al;
    int col = (int)(t - row * n_al);
    int f = (int)(row / kp), r = (int)(row - (int64_t)f * kp);
    Wb[t] = __float2bfloat16_rn(col < g.n && r < g.k ? W[((int64_t)f * g.k + r) * wp + col] : 0.f);
  }
}

__global__ void region_add(float *dst, int dst_h, int dst_w, const float *src, int m, int rows, int cols, int C,
                           int y0, int x0) {
  const int64_t per = (int64_t)rows * cols * C, tot = per * m;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / per, r = t - i * per;
    int c = (int)(r % C);
    int64_t yx = r / C;
    int x = (int)(yx % cols), y = (int)(yx / cols);
    dst[((i * dst_h + y0 + y) * dst_w + x0 + x) * C + c] += src[t];
  }
}

}  // namespace

lcae_status launch_nhwc_to_hwcn_f32(lcae_layer *L, const float *x, float *xt) {
  const Geo &g = L->geo;
  int64_t P = (int64_t)g.H * g.W * g.C;
  dim3 grid((unsigned)cdiv((int)P, 32), cdiv(g.m, 32));
  nhwc_to_hwcn<float><<<grid, dim3(32, 8), 0, L->st>>>(x, xt, g.m, L->mp, P, L->flags_dev);
  LCAE_CK_LAUNCH(L);
  return LCAE_OK;
}

lcae_status launch_nhwc_to_hwcn_bf16(lcae_layer *L, const float *x, __nv_bfloat16 *xt) {
  const Geo &g = L->geo;
  int64_t P = (int64_t)g.H * g.W * g.C;
  if (P % 4 == 0 && L->mp % 8 == 0 && ((uintptr_t)x & 15) == 0) {
    dim3 gv((unsigned)((P + 63) / 64), (unsigned)cdiv(g.m, 64));
    nhwc_to_hwcn_bf16_v<<<gv, 256, 0, L->st>>>(x, xt, g.m, L->mp, P, L->flags_dev);
    LCAE_CK_LAUNCH(L);
    return LCAE_OK;
  }
  dim3 grid((unsigned)cdiv((int)P, 32), cdiv(g.m, 32));
  nhwc_to_hwcn<__nv_bfloat16><<<grid, dim3(32, 8), 0, L->st>>>(x, xt, g.m, L->mp, P, L->flags_dev);
  LCAE_CK_LAUNCH(L);
  return LCAE_OK;
}

lcae_status launch_hwcn_to_nhwc_f32(lcae_layer *L, const float *xt, float *x) {
  const Geo &g = L->geo;
  int64_t P = (int64_t)g.H * g.W * g.C;
  if (P % 4 == 0 && L->mp % 4 == 0 && ((uintptr_t)x & 15) == 0) {
    dim3 gv((unsigned)((P + 63) / 64), (unsigned)cdiv(g.m, 64));
    hwcn_to_nhwc_v<<<gv, 256, 0, L->st>>>(xt, x, g.m, L->mp, P);
    LCAE_CK_LAUNCH(L);
    return LCAE_OK;
  }
  dim3 grid((unsigned)cdiv((int)P, 32), cdiv(g.m, 32));
  hwcn_to_nhwc<<<grid, dim3(32, 8), 0, L->st>>>(xt, x, g.m, L->mp, P);
  LCAE_CK_LAUNCH(L);
  return LCAE_OK;
}

lcae_status launch_loss_reduce(lcae_layer *L, bool update) {
  const bool tcp = L->tc != nullptr;
  loss_reduce<<<1, 1024, 0, L->st>>>(tcp ? tc_loss_part(L) : L->loss_part, tcp ? tc_loss_count(L) : L->geo.F,
                                     L->loss_dev, L->step_dev, update ? 1 : 0, L->flags_dev);
  LCAE_CK_LAUNCH(L);
  return LCAE_OK;
}

lcae_status launch_init_params(lcae_layer *L) {
  const Geo &g = L->geo;
  init_rows<<<dim3(g.F, g.k), 256, 0, L->st>>>(g, L->wp, L->W, L->sigma, L->cfg.seed, L->cfg.field_row0,
                                                L->cfg.field_col0, L->cfg.global_grid_c);
  LCAE_CK_LAUNCH(L);
  fill_f32<<<L->sm_count, 256, 0, L->st>>>(L->alpha, g.F, L->cfg.alpha_init);
  LCAE_CK_LAUNCH(L);
  LCAE_CK(cudaMemsetAsync(L->b, 0, (size_t)g.F * g.n * 4, L->st));
  return LCAE_OK;
}

lcae_status launch_fill(lcae_layer *L, float *p, int64_t n, float v) {
  fill_f32<<<L->sm_count, 256, 0, L->st>>>(p, n, v);
  LCAE_CK_LAUNCH(L);
  return LCAE_OK;
}

lcae_status launch_get_W(lcae_layer *L, float *Wout) {
  get_w<<<L->sm_count * 8, 256, 0, L->st>>>(L->geo, L->wp, L->W, L->sigma, Wout, L->geo.F);
  LCAE_CK_LAUNCH(L);
  return LCAE_OK;
}

lcae_status launch_get_W_range(lcae_layer *L, float *Wout, int64_t f0, int64_t nf) {
  const Geo &g = L->geo;
  get_w<<<L->sm_count * 8, 256, 0, L->st>>>(g, L->wp, L->W + f0 * g.k * L->wp, L->sigma + f0 * g.k, Wout, nf);
  LCAE_CK_LAUNCH(L);
  return LCAE_OK;
}

lcae_status launch_refresh_shadow(lcae_layer *L) {
  if (!L->Wb) return LCAE_OK;
  shadow_w<<<L->sm_count * 8, 256, 0, L->st>>>(L->geo, L->tc ? 128 : L->geo.k, L->n_al, L->wp, L->W, L->Wb);
  LCAE_CK_LAUNCH(L);
  return LCAE_OK;
}

}  // namespace lcae

extern "C" lcae_status lcae_region_add(void *stream, float *dst, int32_t dst_h, int32_t dst_w, const float *src,
                                       int32_t m, int32_t rows, int32_t cols, int32_t C, int32_t y0, int32_t x0) {
  if (!dst || !src) { lcae::set_error("lcae_region_add: NULL pointer"); return LCAE_ERR_ARG; }
  if (m <= 0 || rows <= 0 || cols <= 0 || C <= 0 || y0 < 0 || x0 < 0 || y0 + rows > dst_h || x0 + cols > dst_w) {
    lcae::set_error("lcae_region_add: region outside destination");
    return LCAE_ERR_ARG;
  }
  lcae::region_add<<<148 * 4, 256, 0, (cudaStream_t)stream>>>(dst, dst_h, dst_w, src, m, rows, cols, C, y0, x0);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { lcae::set_error(cudaGetErrorString(e)); return LCAE_ERR_CUDA; }
  return LCAE_OK;
}
