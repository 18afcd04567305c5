// gt_path.cu — the general bf16 tensor-core path: layers the fused step kernel cannot hold (k > 128 filters, n > 4096,
// m > 256; the paper's own layer 1, c3', has k = 384: PAPER.md:95) run the step as five batched tcgen05 GEMMs with
// small epilogue kernels between them. Same step, same notation as f32_path.cu (PAPER.md:88 / DESIGN.md R1-R11), same
// operand rounding as the fused kernel (bf16 x, W, h, delta, alpha D; fp32 accumulation, fp32 master W):
//   U  = W X_f                      (k x m)   GEMM 1          h = alpha U, s_G, p, J_s    (gt_pool)
//   R  = W^T h                      (n x m)   GEMM 2          delta = 2(R + b - x), J_r, db (gt_resid)
//   G  = W delta                    (k x m)   GEMM 3          D = G + lambda h / s, dalpha (gt_dcode)
//   dW = h delta^T + (alpha D) X^T  (k x n)   GEMM 4 (two K segments into one accumulator)
//   dXp = W^T (alpha D) - delta     (n x m)   GEMM 5 (epilogue subtracts delta) -> overlap-add into dX (col2im_f32)
//   projected SGD (gt_update_w: fp32 master + bf16 shadow; update_ab_f32).
// The GEMM kernel `bgemm` is persistent (one CTA per SM): warp 0 issues TMA loads of 128 x 64 A and BN x 64 B tiles
// (SW128, 4-stage ring, zero-filled ragged tails), warp 1 issues tcgen05.mma into one of two TMEM accumulators, warps
// 2-5 drain the other accumulator (tcgen05.ld) to global memory while the next tile's MMAs run.
#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.cuh"

#include <algorithm>

namespace lcae {
namespace gt {

constexpr int BM = 128, BK = 64, ST = 4;

struct GemmArgs {
  CUtensorMap tmA[2], tmB[2];
  int bA[2], bB[2];   // batch-coordinate offset of each operand map (W maps: the chunk's first field)
  int nseg, M, N, K, batch;
  float *C;
  int64_t cbs, crs;   // C[b][i][j] at C + b cbs + i crs + j (cbs, crs multiples of 4)
  const float *C0;    // optional addend: C = acc + beta C0 (same layout as C)
  float beta;
};

// C[b] (M x N, fp32) = sum over segments of A_s[b] (M x K) B_s[b] (K x N); A K-major ([M][K] in global) or
// MN-major ([K][M]); B K-major ([N][K]) or MN-major ([K][N]). Canonical SW128 layouts as in tc_kernel.cuh
// (descriptor conventions pinned by tests/test_gpu_selftest.py).
template <bool AMN, bool BMN, int BN>
__global__ void __launch_bounds__(192, 1) bgemm(const __grid_constant__ GemmArgs P) {
  constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE = A_BYTES + B_BYTES;
  constexpr uint32_t TCOLS = 2 * BN <= 256 ? 256 : 512;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[ST], empty[ST], tfull[2], tempty[2];
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = cdiv(P.M, BM), nt = cdiv(P.N, BN), per = mt * nt;
  const int ntiles = P.batch * per, ksteps = cdiv(P.K, BK);
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { ptx::mbar_init(&tfull[s], 1); ptx::mbar_init(&tempty[s], 4); }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<TCOLS>(&tbase_s);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = tbase_s;
  if (warp == 0) {
    if (lane == 0) {   // TMA producer
      for (int s = 0; s < P.nseg; ++s) { ptx::tma_prefetch(&P.tmA[s]); ptx::tma_prefetch(&P.tmB[s]); }
      uint32_t it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int b = tile / per, r = tile - b * per, m0 = (r / nt) * BM, n0 = (r % nt) * BN;
        for (int sg = 0; sg < P.nseg; ++sg)
          for (int ks = 0; ks < ksteps; ++ks, ++it) {
            const uint32_t s = it % ST, ph = (it / ST) & 1;
            ptx::mbar_wait(&empty[s], ph ^ 1);
            uint8_t *sa = smem + s * STAGE, *sb = sa + A_BYTES;
            ptx::mbar_arrive_expect_tx(&full[s], STAGE);
            const int k0 = ks * BK, ba = P.bA[sg] + b, bb = P.bB[sg] + b;
            if (AMN) {
              ptx::tma_load_3d(sa, &P.tmA[sg], &full[s], m0, k0, ba);
              ptx::tma_load_3d(sa + BK * 128, &P.tmA[sg], &full[s], m0 + 64, k0, ba);
            } else {
              ptx::tma_load_3d(sa, &P.tmA[sg], &full[s], k0, m0, ba);
            }
            if (BMN) {
#pragma unroll
              for (int q = 0; q < BN / 64; ++q) ptx::tma_load_3d(sb + q * BK * 128, &P.tmB[sg], &full[s], n0 + 64 * q, k0, bb);
            } else {
              ptx::tma_load_3d(sb, &P.tmB[sg], &full[s], k0, n0, bb);
            }
          }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // MMA issuer
      constexpr uint32_t idesc = ptx::idesc_bf16(BM, BN, AMN, BMN);
      uint32_t it = 0, tc = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tc) {
        const uint32_t buf = tc & 1;
        ptx::mbar_wait(&tempty[buf], ((tc >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d = tbase + buf * BN;
        uint32_t acc = 0;
        for (int sg = 0; sg < P.nseg; ++sg)
          for (int ks = 0; ks < ksteps; ++ks, ++it) {
            const uint32_t s = it % ST, ph = (it / ST) & 1;
            ptx::mbar_wait(&full[s], ph);
            ptx::tc_fence_after();
            const uint32_t sa = ptx::smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t ad = AMN ? ptx::sdesc_sw128(sa + kk * 2048, BK * 128, 1024) : ptx::sdesc_sw128(sa + kk * 32, 16, 1024);
              const uint64_t bd = BMN ? ptx::sdesc_sw128(sb + kk * 2048, BK * 128, 1024) : ptx::sdesc_sw128(sb + kk * 32, 16, 1024);
              ptx::umma_bf16(d, ad, bd, idesc, acc);
              acc = 1;
            }
            ptx::umma_commit(&empty[s]);   // the stage is free once these MMAs have read it
          }
        ptx::umma_commit(&tfull[buf]);
      }
    }
  } else {   // epilogue: warp w drains TMEM lanes [32 (w % 4), +32) = rows of the tile
    const int q = warp & 3;
    uint32_t tc = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tc) {
      const int b = tile / per, r = tile - b * per, m0 = (r / nt) * BM, n0 = (r % nt) * BN;
      const uint32_t buf = tc & 1;
      ptx::mbar_wait(&tfull[buf], (tc >> 1) & 1);
      ptx::tc_fence_after();
      const int i = m0 + 32 * q + lane;
      float *crow = P.C + b * P.cbs + (int64_t)i * P.crs;
      const float *c0row = P.C0 ? P.C0 + b * P.cbs + (int64_t)i * P.crs : nullptr;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        if (n0 + c >= P.N) break;   // warp-uniform
        float v[16];
        ptx::tmem_ld16(tbase + ((uint32_t)(32 * q) << 16) + buf * BN + c, v);
        ptx::tmem_ld_wait();
        if (i < P.M) {
          const int j0 = n0 + c;
          if (j0 + 16 <= P.N) {
#pragma unroll
            for (int t = 0; t < 16; t += 4) {
              float4 o = make_float4(v[t], v[t + 1], v[t + 2], v[t + 3]);
              if (c0row) {
                const float4 a = *reinterpret_cast<const float4 *>(c0row + j0 + t);
                o.x = fmaf(P.beta, a.x, o.x); o.y = fmaf(P.beta, a.y, o.y);
                o.z = fmaf(P.beta, a.z, o.z); o.w = fmaf(P.beta, a.w, o.w);
              }
              *reinterpret_cast<float4 *>(crow + j0 + t) = o;
            }
          } else {
#pragma unroll
            for (int t = 0; t < 16; ++t)
              if (j0 + t < P.N) crow[j0 + t] = c0row ? fmaf(P.beta, c0row[j0 + t], v[t]) : v[t];
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TCOLS>(tbase);
  }
}

template <bool AMN, bool BMN, int BN>
lcae_status launch_bn(lcae_layer *L, const GemmArgs &a) {
  constexpr int smem = ST * (BM * BK * 2 + BN * BK * 2) + 1024;
  static bool attr = false;
  if (!attr) {
    LCAE_CK(cudaFuncSetAttribute(bgemm<AMN, BMN, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const int tiles = a.batch * cdiv(a.M, BM) * cdiv(a.N, BN);
  const bool prof = L->prof_on && L->prof_n < 4096;   // lcae_profile: events around every GEMM launch
  if (prof) LCAE_CK(cudaEventRecord(L->prof_ev[2 * L->prof_n], L->st));
  bgemm<AMN, BMN, BN><<<std::min(tiles, L->sm_count), 192, smem, L->st>>>(a);
  LCAE_CK_LAUNCH(L);
  if (prof) LCAE_CK(cudaEventRecord(L->prof_ev[2 * L->prof_n++ + 1], L->st));
  return LCAE_OK;
}

inline int pick_bn(int N) { return N <= 64 ? 64 : N <= 128 ? 128 : N <= 192 ? 192 : 256; }

template <bool AMN, bool BMN>
lcae_status gemm(lcae_layer *L, const GemmArgs &a) {
  switch (pick_bn(a.N)) {
    case 64: return launch_bn<AMN, BMN, 64>(L, a);
    case 128: return launch_bn<AMN, BMN, 128>(L, a);
    case 192: return launch_bn<AMN, BMN, 192>(L, a);
    default: return launch_bn<AMN, BMN, 256>(L, a);
  }
}

// ---------------------------------------------------------------- epilogue kernels (one block per field)

// X_f (n x m) gathered from the HWCN bf16 image into [Fc][n][mp] (16-byte runs; rows of one receptive-field row are
// consecutive pixel-features).
__global__ void __launch_bounds__(256) gt_gather(Geo g, int f0, int mp, const __nv_bfloat16 *xt16, __nv_bfloat16 *Xp) {
  const int b = blockIdx.x, f = f0 + b, r = f / g.gc, c = f - r * g.gc;
  const int q8 = mp / 8;
  const int64_t rowstride = (int64_t)g.W * g.C;   // pixel-features per image row
  const int64_t base = ((int64_t)r * g.s * rowstride + (int64_t)c * g.s * g.C) * mp;
  const uint4 *src = reinterpret_cast<const uint4 *>(xt16);
  uint4 *dst = reinterpret_cast<uint4 *>(Xp + (int64_t)b * g.n * mp);
  for (int t = threadIdx.x; t < g.n * q8; t += blockDim.x) {
    const int row = t / q8, qq = t - row * q8, ry = row / g.RW;
    const int64_t off = base + ((int64_t)ry * rowstride + (row - ry * g.RW)) * mp;
    dst[t] = src[off / 8 + qq];
  }
}

// h = alpha U (bf16 copy for the GEMMs), s_G = sqrt(eps + sum_G h^2) -> p, J_s = lambda sum s, Q = lambda h / s.
__global__ void __launch_bounds__(256) gt_pool(Geo g, int f0, int mp, const float *U, const float *alpha, float lam,
                                               float eps, __nv_bfloat16 *H16, float *Q, float *pooled,
                                               double *loss_part, int enc) {
  __shared__ double sh[32];
  const int b = blockIdx.x, f = f0 + b;
  const int k = g.k, m = g.m, gs = g.g, ng = k / gs;
  const float a = alpha[f];
  const int64_t kb = (int64_t)b * k * mp;
  double acc = 0.0;
  for (int t = threadIdx.x; t < ng * m; t += blockDim.x) {
    const int G = t / m, i = t - G * m;
    float ss = 0.f;
    for (int q = 0; q < gs; ++q) {
      const float h = a * U[kb + (int64_t)(G * gs + q) * mp + i];
      ss = fmaf(h, h, ss);
    }
    const float s = sqrtf(eps + ss);
    acc += (double)s;
    if (pooled) {
      const int r = f / g.gc, c = f - r * g.gc;
      pooled[(((int64_t)i * g.gr + r) * g.gc + c) * ng + G] = s;
    }
    const float inv = s > 0.f ? lam / s : 0.f;
    for (int q = 0; q < gs; ++q) {
      const int64_t o = kb + (int64_t)(G * gs + q) * mp + i;
      const float h = a * U[o];
      H16[o] = __float2bfloat16_rn(h);
      if (Q) Q[o] = h * inv;
    }
  }
  const double tot = block_sum_f64(acc, sh);
  if (threadIdx.x == 0) {
    loss_part[2 * f + 1] = (double)lam * tot;
    if (enc) loss_part[2 * f] = 0.0;
  }
}

// e = R + b - x (x: the bf16 image value the GEMMs use); J_r = sum e^2; delta = 2e (fp32 in place, bf16 copy);
// db = sum_i delta. One warp per patch row.
__global__ void __launch_bounds__(256) gt_resid(Geo g, int f0, int mp, float *R, const float *bvec,
                                                const __nv_bfloat16 *Xp, __nv_bfloat16 *d16, double *loss_part,
                                                float *db) {
  __shared__ double sh[32];
  const int b = blockIdx.x, f = f0 + b, n = g.n, m = g.m;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t nb = (int64_t)b * n * mp;
  double acc = 0.0;
  for (int row = wid; row < n; row += nw) {
    const float bb = bvec[(int64_t)f * n + row];
    float dsum = 0.f;
    for (int i = lane; i < m; i += 32) {
      const int64_t o = nb + (int64_t)row * mp + i;
      const float e = R[o] + bb - __bfloat162float(Xp[o]);
      acc += (double)e * (double)e;
      const float dl = 2.f * e;
      R[o] = dl;
      d16[o] = __float2bfloat16_rn(dl);
      dsum += dl;
    }
    dsum = warp_sum(dsum);
    if (lane == 0) db[(int64_t)b * n + row] = dsum;
  }
  const double tot = block_sum_f64(acc, sh);
  if (threadIdx.x == 0) loss_part[2 * f] = tot;
}

// D = G + Q; dalpha = sum D (.) U; D16 = bf16(alpha D) (the operand of dW's second term and of dX).
__global__ void __launch_bounds__(256) gt_dcode(Geo g, int f0, int mp, const float *G, const float *Q, const float *U,
                                                const float *alpha, __nv_bfloat16 *D16, float *da) {
  __shared__ double sh[32];
  const int b = blockIdx.x, m = g.m;
  const float a = alpha[f0 + b];
  const int64_t kb = (int64_t)b * g.k * mp;
  double acc = 0.0;
  for (int t = threadIdx.x; t < g.k * m; t += blockDim.x) {
    const int row = t / m, i = t - row * m;
    const int64_t o = kb + (int64_t)row * mp + i;
    const float d = G[o] + Q[o];
    acc += (double)d * (double)U[o];
    D16[o] = __float2bfloat16_rn(a * d);
  }
  const double tot = block_sum_f64(acc, sh);
  if (threadIdx.x == 0) da[b] = (float)tot;
}

// Projected SGD on W rows (W kept unit-norm, sigma == 1, as in the fp32 path): v = mu v - lr dW; W' = W + v;
// W' /= ||W'|| (degenerate rows re-initialised from the counter-based generator); the bf16 shadow row
// is rewritten from W'. dW rows have pitch n_al.
__global__ void __launch_bounds__(256) gt_update_w(Geo g, int f0, int wp, int n_al, float *W, __nv_bfloat16 *Wb,
                                                   const float *dW, float *vW, float *gW, float lr, float mu,
                                                   uint64_t seed, const int64_t *step_dev, int row0, int col0, int ggc,
                                                   int *reinit, const int *flags) {
  __shared__ double sh[32];
  __shared__ float s_scale;
  const int b = blockIdx.x, j = blockIdx.y, f = f0 + b, n = g.n;
  const float *d = dW + ((int64_t)b * g.k + j) * n_al;
  const int64_t wo = ((int64_t)f * g.k + j) * wp;
  if (gW)
    for (int t = threadIdx.x; t < n; t += blockDim.x) gW[wo + t] = d[t];
  if (flags[0] | flags[1]) return;   // flagged error: parameters frozen (include/lcae.h "Errors")
  float *w = W + wo;
  float *v = vW ? vW + wo : nullptr;
  double acc = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    float upd = -lr * d[t];
    if (v) { upd = fmaf(mu, v[t], upd); v[t] = upd; }
    const float wn = w[t] + upd;
    w[t] = wn;
    acc += (double)wn * wn;
  }
  const double tot = block_sum_f64(acc, sh);
  if (threadIdx.x == 0) s_scale = tot < 1e-60 ? -1.f : (float)(1.0 / sqrt(tot));
  __syncthreads();
  float sc = s_scale;
  if (sc < 0.f) {
    const int r = f / g.gc, c = f - r * g.gc;
    const uint64_t gf = (uint64_t)((row0 + r) * ggc + col0 + c);
    const uint64_t key = splitmix64(seed ^ ((uint64_t)*step_dev << 40) ^ (gf << 20) ^ (uint64_t)j);
    double a2 = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const double u = (double)(splitmix64(key + (uint64_t)t) >> 40) / 16777216.0 - 0.5;
      w[t] = (float)u;
      if (v) v[t] = 0.f;
      a2 += u * u;
    }
    const double tt = block_sum_f64(a2, sh);
    if (threadIdx.x == 0) { s_scale = (float)(1.0 / sqrt(tt)); atomicAdd(reinit, 1); }
    __syncthreads();
    sc = s_scale;
  }
  __nv_bfloat16 *wb = Wb + ((int64_t)f * g.k + j) * n_al;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const float x = w[t] * sc;
    w[t] = x;
    wb[t] = __float2bfloat16_rn(x);
  }
}

__global__ void gt_copy_ab(int f0, int Fc, int n, const float *da, const float *db, float *ga, float *gb) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)Fc * n; t += (int64_t)gridDim.x * blockDim.x) {
    gb[(int64_t)f0 * n + t] = db[t];
    if (t < Fc) ga[f0 + t] = da[t];
  }
}

}  // namespace gt

struct GtScratch {
  int Fc = 0;
  __nv_bfloat16 *Xp = nullptr, *H16 = nullptr, *d16 = nullptr, *D16 = nullptr;   // [Fc][n|k][mp]
  float *U = nullptr, *Q = nullptr, *G = nullptr;                               // [Fc][k][mp]
  float *R = nullptr, *dXp = nullptr;                                           // [Fc][n][mp] (R: r, then delta)
  float *dW = nullptr;                                                          // [Fc][k][n_al]
  float *da = nullptr, *db = nullptr;                                           // [Fc], [Fc][n]
  gt::GemmArgs ga[5];
};

lcae_status gt_alloc(lcae_layer *L) {
  const Geo &g = L->geo;
  const int64_t k = g.k, n = g.n, mp = L->mp, na = L->n_al;
  if (L->mp % 8 || L->n_al % 8) { set_error("gt path: pitches must be multiples of 8"); return LCAE_ERR_CONFIG; }
  const int64_t per_field = n * mp * (2 + 4 + 2 + 4) + k * mp * (4 + 2 + 4 + 4 + 2) + k * na * 4 + n * 4 + 4;
  GtScratch *s = new GtScratch();
  L->gt = s;
  s->Fc = (int)std::max<int64_t>(1, std::min<int64_t>(g.F, (2ll << 30) / per_field));
  const int64_t Fc = s->Fc;
  LCAE_CK(dmalloc(L, &s->Xp, Fc * n * mp * 2));
  LCAE_CK(dmalloc(L, &s->H16, Fc * k * mp * 2));
  LCAE_CK(dmalloc(L, &s->d16, Fc * n * mp * 2));
  LCAE_CK(dmalloc(L, &s->D16, Fc * k * mp * 2));
  LCAE_CK(dmalloc(L, &s->U, Fc * k * mp * 4));
  LCAE_CK(dmalloc(L, &s->Q, Fc * k * mp * 4));
  LCAE_CK(dmalloc(L, &s->G, Fc * k * mp * 4));
  LCAE_CK(dmalloc(L, &s->R, Fc * n * mp * 4));
  LCAE_CK(dmalloc(L, &s->dXp, Fc * n * mp * 4));
  LCAE_CK(cudaMemset(s->dXp, 0, Fc * n * mp * 4));   // padded sample columns are never written: keep them zero
  LCAE_CK(dmalloc(L, &s->dW, Fc * k * na * 4));
  LCAE_CK(dmalloc(L, &s->da, Fc * 4));
  LCAE_CK(dmalloc(L, &s->db, Fc * n * 4));
  // bf16 shadow of W, [F][k][n_al] (pad columns zero)
  cudaFree(L->Wb);
  L->Wb = nullptr;
  LCAE_CK(dmalloc(L, &L->Wb, (size_t)g.F * k * na * 2));
  LCAE_CK(cudaMemset(L->Wb, 0, (size_t)g.F * k * na * 2));
  // operand maps: [batch][rows][cols] with the sample (or n) extent the true size, so ragged tails load as zeros
  const int bnm = gt::pick_bn(g.m), bnn = gt::pick_bn(g.n);
  CUtensorMap mWk, mWmn, mXmn, mXk, mHmn, mHk, mdmn, mdk, mDk, mDmn;
  bool ok = make_tmap_3d_bf16(&mWk, L->Wb, g.F, k, n, na, k * na, gt::BM) &&
            make_tmap_3d_bf16(&mWmn, L->Wb, g.F, k, n, na, k * na, gt::BK) &&
            make_tmap_3d_bf16(&mXmn, s->Xp, Fc, n, g.m, mp, n * mp, gt::BK) &&
            make_tmap_3d_bf16(&mXk, s->Xp, Fc, n, g.m, mp, n * mp, bnn) &&
            make_tmap_3d_bf16(&mHmn, s->H16, Fc, k, g.m, mp, k * mp, gt::BK) &&
            make_tmap_3d_bf16(&mHk, s->H16, Fc, k, g.m, mp, k * mp, gt::BM) &&
            make_tmap_3d_bf16(&mdmn, s->d16, Fc, n, g.m, mp, n * mp, gt::BK) &&
            make_tmap_3d_bf16(&mdk, s->d16, Fc, n, g.m, mp, n * mp, bnn) &&
            make_tmap_3d_bf16(&mDk, s->D16, Fc, k, g.m, mp, k * mp, gt::BM) &&
            make_tmap_3d_bf16(&mDmn, s->D16, Fc, k, g.m, mp, k * mp, gt::BK);
  if (!ok) { set_error("gt path: cuTensorMapEncodeTiled failed"); return LCAE_ERR_CUDA; }
  (void)bnm;
  auto args = [&](const CUtensorMap &A, const CUtensorMap &B, int M, int N, int K, float *C, int64_t cbs, int64_t crs) {
    gt::GemmArgs a{};
    a.tmA[0] = A; a.tmB[0] = B; a.nseg = 1; a.M = M; a.N = N; a.K = K; a.C = C; a.cbs = cbs; a.crs = crs;
    return a;
  };
  s->ga[0] = args(mWk, mXmn, g.k, g.m, g.n, s->U, k * mp, mp);       // U = W X_f
  s->ga[1] = args(mWmn, mHmn, g.n, g.m, g.k, s->R, n * mp, mp);      // R = W^T h
  s->ga[2] = args(mWk, mdmn, g.k, g.m, g.n, s->G, k * mp, mp);       // G = W delta
  s->ga[3] = args(mHk, mdk, g.k, g.n, g.m, s->dW, k * na, na);       // dW = h delta^T + (alpha D) X_f^T
  s->ga[3].tmA[1] = mDk; s->ga[3].tmB[1] = mXk; s->ga[3].nseg = 2;
  s->ga[4] = args(mWmn, mDmn, g.n, g.m, g.k, s->dXp, n * mp, mp);    // dXp = W^T (alpha D) - delta
  s->ga[4].C0 = s->R; s->ga[4].beta = -1.f;
  return LCAE_OK;
}

void gt_free(lcae_layer *L) {
  GtScratch *s = L->gt;
  if (!s) return;
  for (void *p : {(void *)s->Xp, (void *)s->H16, (void *)s->d16, (void *)s->D16, (void *)s->U, (void *)s->Q,
                  (void *)s->G, (void *)s->R, (void *)s->dXp, (void *)s->dW, (void *)s->da, (void *)s->db})
    cudaFree(p);
  delete s;
  L->gt = nullptr;
}

lcae_status gt_step(lcae_layer *L, bool update, bool want_pooled, bool encode_only) {
  const Geo &g = L->geo;
  GtScratch &s = *L->gt;
  const int mp = L->mp;
  lcae_status st;
#define TRY(x) do { if ((st = (x)) != LCAE_OK) return st; } while (0)
  if (update) LCAE_CK(cudaMemsetAsync(L->dxt, 0, (size_t)g.H * g.W * g.C * mp * 4, L->st));
  Geo gp = g;
  gp.m = mp;   // col2im over the padded sample pitch of dXp / dxt
  for (int f0 = 0; f0 < g.F; f0 += s.Fc) {
    const int Fc = std::min(s.Fc, g.F - f0);
    for (auto &a : s.ga) a.batch = Fc;
    s.ga[0].bA[0] = s.ga[1].bA[0] = s.ga[2].bA[0] = s.ga[4].bA[0] = f0;   // W maps span all fields
    gt::gt_gather<<<Fc, 256, 0, L->st>>>(g, f0, mp, L->xt16, s.Xp);
    LCAE_CK_LAUNCH(L);
    TRY((gt::gemm<false, true>(L, s.ga[0])));
    gt::gt_pool<<<Fc, 256, 0, L->st>>>(g, f0, mp, s.U, L->alpha, L->cfg.lambda_, L->cfg.eps, s.H16,
                                       update ? s.Q : nullptr, want_pooled ? L->pooled : nullptr, L->loss_part,
                                       encode_only ? 1 : 0);
    LCAE_CK_LAUNCH(L);
    if (encode_only) continue;
    TRY((gt::gemm<true, true>(L, s.ga[1])));
    gt::gt_resid<<<Fc, 256, 0, L->st>>>(g, f0, mp, s.R, L->b, s.Xp, s.d16, L->loss_part, s.db);
    LCAE_CK_LAUNCH(L);
    if (!update) continue;
    TRY((gt::gemm<false, true>(L, s.ga[2])));
    gt::gt_dcode<<<Fc, 256, 0, L->st>>>(g, f0, mp, s.G, s.Q, s.U, L->alpha, s.D16, s.da);
    LCAE_CK_LAUNCH(L);
    TRY((gt::gemm<false, false>(L, s.ga[3])));
    TRY((gt::gemm<true, true>(L, s.ga[4])));
    col2im_f32<<<L->sm_count * 8, 256, 0, L->st>>>(gp, f0, Fc, s.dXp, L->dxt);
    LCAE_CK_LAUNCH(L);
    if (L->cfg.keep_grads) {
      gt::gt_copy_ab<<<256, 256, 0, L->st>>>(f0, Fc, g.n, s.da, s.db, L->galpha, L->gb);
      LCAE_CK_LAUNCH(L);
    }
    gt::gt_update_w<<<dim3(Fc, g.k), 256, 0, L->st>>>(g, f0, L->wp, L->n_al, L->W, L->Wb, s.dW, L->vW,
                                                      L->cfg.keep_grads ? L->gW : nullptr, L->cfg.lr, L->cfg.momentum,
                                                      L->cfg.seed, L->step_dev, L->cfg.field_row0, L->cfg.field_col0,
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
