// tc_path.cu — the bf16 tcgen05 training step of the locally-connected RICA layer (sm_100a).
//
// One persistent kernel does the whole per-field chain of PAPER.md:88:
// a cluster of CB CTAs (CB = ceil(m/128): each CTA owns a 128-sample slice of the batch) walks the fields;
// for field f every CTA streams the bf16 W~_f tiles (TMA, 128B swizzle) and its X_f patch rows (cp.async
// gather from the batch-innermost HWCN image) through a 2-stage smem ring in three passes over n-tiles of 64:
//
//   pass 0  U^T   = X^T W~^T                   (M = samples, N = k, K = n)       TMEM [0,128)
//           E0: u = sigma.U~, h = alpha u, s_G = sqrt(eps + sum_G h^2), J_s, p; H' = bf16(sigma.h) -> smem
//   pass 1  R^T_j = H'^T W~_j                  (M = samples, N = 64, K = k)      TMEM [128,256) x2
//           E1: e = R + b - x, J_r, delta = 2e -> smem (bf16), db partial (butterfly column sums)
//           G^T  += delta_j^T W~_j^T           (M = samples, N = k, K = 64)      TMEM [256,384)
//           E1b: D = sigma.G~ + lambda h/s, dalpha, D' = bf16(sigma alpha D) -> smem
//   pass 2  R^T_j, dX^T_j = D'^T W~_j          (recompute delta; dx = dX - delta -> red.global into dX)
//           dW_j = H' delta_j^T + D' X_j^T     (M = k, N = 64, K = 2 x samples)  TMEM x2 buffers
//           E2: sum the batch slices of dW_j over the cluster (DSMEM), projected-SGD of W~ (fp32 master +
//               bf16 shadow), row sums of squares for the new row scale sigma.
//
// W = sigma (.) W~ with a per-row scale sigma ("lazy projection"): the unit-norm projection of
// PAPER.md:89 is applied by the finalize kernel as sigma' = 1/||W~'_row||, so the update never re-reads W.
#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.cuh"

namespace lcae {

namespace tc {
constexpr int KP = 128;        // filters padded to one TMEM lane block
constexpr int NT = 64;         // n-tile
constexpr int MC = 128;        // samples per CTA
constexpr int NS = 2;          // smem pipeline stages
constexpr int NTHREADS = 192;  // warp 0 producer, warp 1 MMA, warps 2-5 epilogue
constexpr int MAX_NPAD = 2048;

struct Params {
  CUtensorMap tmW;   // W~ bf16 [F*KP][n_al], box (64, 128)
  Geo g;
  int T, mp, CB, n_al, mode, want_pooled, keep_grads;
  float lam, eps, lr, mu;
  const __nv_bfloat16 *xt;
  float *dxt;
  float *W;
  const float *sigma, *alpha, *b;
  __nv_bfloat16 *Wb;
  float *vW, *pooled;
  double *loss_part;   // [F][CB][2]
  float *da_part;      // [F][CB]
  float *db_part;      // [F][CB][n]
  float *rowsq_part;   // [F][CB][KP]
  float *gW;
};

struct __align__(1024) Smem {
  uint8_t W[NS][16384];
  uint8_t X[NS][16384];
  uint8_t H[32768];
  uint8_t D[32768];
  uint8_t Dl[2][16384];
  float recv[2][32][128];
  int off[MAX_NPAD];
  float sig[KP];
  float dbw[2][4][64];
  double redd[4][2];
  float redf[4];
  uint64_t full[NS], empty[NS];
  uint64_t u_full, h_ready, g_full, d_ready, tmem_free;
  uint64_t r_full[2], r_empty[2], dl_full[2], dl_empty[2];
  uint64_t p2_rdx[2], p2_dw[2], p2_empty[2];
  uint64_t recv_full[2], peer_free[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ float bf(const uint8_t *base, uint32_t off) {
  return __bfloat162float(*reinterpret_cast<const __nv_bfloat16 *>(base + off));
}

// store 8 consecutive bf16 (cols c0..c0+7 of row `row`) into a [rows][64] SW128 block
__device__ __forceinline__ void st8(uint8_t *blk, int row, int c0, const float *v) {
  uint4 q;
  q.x = ptx::pack_bf16x2(v[0], v[1]);
  q.y = ptx::pack_bf16x2(v[2], v[3]);
  q.z = ptx::pack_bf16x2(v[4], v[5]);
  q.w = ptx::pack_bf16x2(v[6], v[7]);
  *reinterpret_cast<uint4 *>(blk + ptx::sw128_off(row, c0)) = q;
}

template <int GP, int CBT>
__global__ void __launch_bounds__(NTHREADS, 1) step_kernel(const __grid_constant__ Params P) {
  extern __shared__ uint8_t smem_raw[];
  Smem &S = *reinterpret_cast<Smem *>((((uintptr_t)smem_raw) + 1023) & ~(uintptr_t)1023);
  const Geo &g = P.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int CB = CBT;
  const uint32_t crank = CB > 1 ? ptx::cluster_ctarank() : 0;
  const int cid = blockIdx.x / CB, ncl = gridDim.x / CB;
  const int s0 = (int)crank * MC;   // first sample of this CTA
  const int T = P.T, n = g.n, k = g.k, m = g.m, mp = P.mp;
  const bool step = P.mode == 1;

  // ---- one-time setup
  for (int t = threadIdx.x; t < T * NT; t += NTHREADS) {
    int ry = t / g.RW, rem = t - ry * g.RW;
    S.off[t] = t < n ? ry * g.W * g.C + rem : -1;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) { ptx::mbar_init(&S.full[i], 33); ptx::mbar_init(&S.empty[i], 1); }
    ptx::mbar_init(&S.u_full, 1);
    ptx::mbar_init(&S.h_ready, 4);
    ptx::mbar_init(&S.g_full, 1);
    ptx::mbar_init(&S.d_ready, 4);
    ptx::mbar_init(&S.tmem_free, 4);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&S.r_full[i], 1);
      ptx::mbar_init(&S.r_empty[i], 4);
      ptx::mbar_init(&S.dl_full[i], 4);
      ptx::mbar_init(&S.dl_empty[i], 1);
      ptx::mbar_init(&S.p2_rdx[i], 1);
      ptx::mbar_init(&S.p2_dw[i], 1);
      ptx::mbar_init(&S.p2_empty[i], 4);
      ptx::mbar_init(&S.recv_full[i], 4);
      ptx::mbar_init(&S.peer_free[i], 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(&S.tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  if (CB > 1) ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tb = S.tmem_base;

  if (warp == 0) {
    // =================================================================== producer
    if (lane == 0) ptx::tma_prefetch(&P.tmW);
    uint32_t q = 0;
    const int npass = step ? 3 : 2;
    for (int f = cid; f < g.F; f += ncl) {
      const int fr = f / g.gc, fc = f - fr * g.gc;
      const int64_t pixbase = ((int64_t)fr * g.s * g.W + (int64_t)fc * g.s) * g.C;
      for (int pass = 0; pass < npass; ++pass) {
        for (int j = 0; j < T; ++j, ++q) {
          const int s = q % NS;
          ptx::mbar_wait(&S.empty[s], ((q / NS) & 1) ^ 1);
          if (lane == 0) {
            ptx::mbar_arrive_expect_tx(&S.full[s], 16384);
            ptx::tma_load_2d(S.W[s], &P.tmW, &S.full[s], j * NT, f * KP);
          }
          const uint32_t xs = ptx::smem_u32(S.X[s]);
#pragma unroll 4
          for (int t = 0; t < 32; ++t) {
            const int id = lane + 32 * t, row = id >> 4, qq = id & 15;
            const int nn = j * NT + row;
            const bool valid = nn < n && (s0 + qq * 8) < mp;
            const __nv_bfloat16 *src = valid ? P.xt + (pixbase + S.off[nn]) * mp + s0 + qq * 8 : P.xt;
            const uint32_t dst = xs + (qq >> 3) * 8192 + row * 128 + (((qq & 7) ^ (row & 7)) << 4);
            ptx::cp_async_16(dst, src, valid ? 16u : 0u);
          }
          ptx::cp_async_mbar_arrive_noinc(&S.full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // =================================================================== MMA issuer
    if (lane == 0) {
      const uint32_t id_enc = ptx::idesc_bf16(128, KP, true, false);
      const uint32_t id_dec = ptx::idesc_bf16(128, NT, false, true);
      const uint32_t id_g = ptx::idesc_bf16(128, KP, false, false);
      const uint32_t id_dw1 = ptx::idesc_bf16(128, NT, true, true);
      const uint32_t id_dw2 = ptx::idesc_bf16(128, NT, true, false);
      const uint32_t sH = ptx::smem_u32(S.H), sD = ptx::smem_u32(S.D);
      uint32_t q = 0, nf = 0, ur = 0, ud = 0, u2 = 0;
      auto wst = [&](uint32_t qq) { return ptx::smem_u32(S.W[qq % NS]); };
      auto xst = [&](uint32_t qq) { return ptx::smem_u32(S.X[qq % NS]); };
      auto wait_full = [&](uint32_t qq) {
        ptx::mbar_wait(&S.full[qq % NS], (qq / NS) & 1);
        ptx::tc_fence_after();
        ptx::fence_proxy_async_smem();
      };
      // R^T_j (or the dX^T_j with D') = A^T W~_j: A = H' or D' (K-major [128][128]), W~_j MN-major
      auto mma_aw = [&](uint32_t dcol, uint32_t a_base, uint32_t w_base) {
        for (int kk = 0; kk < KP / 16; ++kk) {
          uint64_t ad = ptx::sdesc_sw128(a_base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
          uint64_t bd = ptx::sdesc_sw128(w_base + kk * 2048, 16384, 1024);
          ptx::umma_bf16(tb + dcol, ad, bd, id_dec, kk > 0);
        }
      };
      for (int f = cid; f < g.F; f += ncl, ++nf) {
        ptx::mbar_wait(&S.tmem_free, (nf & 1) ^ 1);
        ptx::tc_fence_after();
        // ---- pass 0: U^T = X^T W~^T
        for (int j = 0; j < T; ++j, ++q) {
          wait_full(q);
          for (int kk = 0; kk < NT / 16; ++kk) {
            uint64_t ad = ptx::sdesc_sw128(xst(q) + kk * 2048, 8192, 1024);
            uint64_t bd = ptx::sdesc_sw128(wst(q) + kk * 32, 16, 1024);
            ptx::umma_bf16(tb + 0, ad, bd, id_enc, (j | kk) != 0);
          }
          ptx::umma_commit(&S.empty[q % NS]);
        }
        ptx::umma_commit(&S.u_full);
        // ---- pass 1: R_j, then G += delta_{j} W~_j^T one tile behind
        ptx::mbar_wait(&S.h_ready, nf & 1);
        ptx::tc_fence_after();
        ptx::fence_proxy_async_smem();
        const uint32_t q1 = q;
        auto issue_G = [&](int j) {
          const uint32_t qj = q1 + j, db_ = ud & 1;
          ptx::mbar_wait(&S.dl_full[db_], (ud >> 1) & 1);
          ptx::tc_fence_after();
          ptx::fence_proxy_async_smem();
          const uint32_t dl = ptx::smem_u32(S.Dl[db_]);
          for (int kk = 0; kk < NT / 16; ++kk) {
            uint64_t ad = ptx::sdesc_sw128(dl + kk * 32, 16, 1024);
            uint64_t bd = ptx::sdesc_sw128(wst(qj) + kk * 32, 16, 1024);
            ptx::umma_bf16(tb + 256, ad, bd, id_g, (j | kk) != 0);
          }
          ptx::umma_commit(&S.dl_empty[db_]);
          ptx::umma_commit(&S.empty[qj % NS]);
          ++ud;
        };
        for (int j = 0; j < T; ++j, ++q) {
          wait_full(q);
          const uint32_t rb = ur & 1;
          ptx::mbar_wait(&S.r_empty[rb], ((ur >> 1) & 1) ^ 1);
          ptx::tc_fence_after();
          mma_aw(128 + 64 * rb, sH, wst(q));
          ptx::umma_commit(&S.r_full[rb]);
          if (step) {
            if (j > 0) issue_G(j - 1);
          } else {   // forward: release the stage once the epilogue is done with tile j
            ptx::mbar_wait(&S.r_empty[rb], (ur >> 1) & 1);
            ptx::mbar_arrive(&S.empty[q % NS]);
          }
          ++ur;
        }
        if (!step) continue;
        issue_G(T - 1);
        ptx::umma_commit(&S.g_full);
        // ---- pass 2: R_j, dX_j, then dW_j one tile behind
        ptx::mbar_wait(&S.d_ready, nf & 1);
        ptx::tc_fence_after();
        ptx::fence_proxy_async_smem();
        const uint32_t q2 = q, u2_0 = u2;
        auto issue_dW = [&](int j) {
          const uint32_t qj = q2 + j, pb = (u2_0 + j) & 1, db_ = ud & 1;
          ptx::mbar_wait(&S.dl_full[db_], (ud >> 1) & 1);
          ptx::tc_fence_after();
          ptx::fence_proxy_async_smem();
          const uint32_t dl = ptx::smem_u32(S.Dl[db_]), dcol = 192 * pb + 128;
          for (int kk = 0; kk < MC / 16; ++kk) {   // H' delta_j^T  (K = samples)
            uint64_t ad = ptx::sdesc_sw128(sH + kk * 2048, 16384, 1024);
            uint64_t bd = ptx::sdesc_sw128(dl + kk * 2048, 16384, 1024);
            ptx::umma_bf16(tb + dcol, ad, bd, id_dw1, kk > 0);
          }
          for (int kk = 0; kk < MC / 16; ++kk) {   // + D' X_j^T
            uint64_t ad = ptx::sdesc_sw128(sD + kk * 2048, 16384, 1024);
            uint64_t bd = ptx::sdesc_sw128(xst(qj) + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
            ptx::umma_bf16(tb + dcol, ad, bd, id_dw2, 1);
          }
          ptx::umma_commit(&S.p2_dw[pb]);
          ptx::umma_commit(&S.dl_empty[db_]);
          ptx::umma_commit(&S.empty[qj % NS]);
          ++ud;
        };
        for (int j = 0; j < T; ++j, ++q, ++u2) {
          wait_full(q);
          const uint32_t pb = u2 & 1;
          ptx::mbar_wait(&S.p2_empty[pb], ((u2 >> 1) & 1) ^ 1);
          ptx::tc_fence_after();
          mma_aw(192 * pb, sH, wst(q));        // R^T_j
          mma_aw(192 * pb + 64, sD, wst(q));   // dX^T_j (alpha folded into D')
          ptx::umma_commit(&S.p2_rdx[pb]);
          if (j > 0) issue_dW(j - 1);
        }
        issue_dW(T - 1);
      }
    }
    __syncwarp();
  } else {
    // =================================================================== epilogue (4 warps)
    const int qd = warp & 3;              // TMEM lane quarter
    const int ew = warp - 2;              // epilogue warp index 0..3
    const int etid = threadIdx.x - 64;    // 0..127
    const int row = qd * 32 + lane;       // TMEM lane: sample (U, R, G, dX) or filter row (dW)
    const uint32_t tl = tb + ((uint32_t)(qd * 32) << 16);
    const int gi = s0 + row;              // global sample index
    const bool svalid = gi < m;
    const int ng = k / GP;
    uint32_t q = 0, nf = 0, ur = 0, ud = 0, u2 = 0;
    for (int f = cid; f < g.F; f += ncl, ++nf) {
      const int fr = f / g.gc, fc = f - fr * g.gc;
      const int64_t pixbase = ((int64_t)fr * g.s * g.W + (int64_t)fc * g.s) * g.C;
      ptx::named_bar_sync(1, 128);
      S.sig[etid] = etid < k ? P.sigma[(int64_t)f * k + etid] : 1.f;
      ptx::named_bar_sync(1, 128);
      const float a = P.alpha[f];
      const float *bf_ = P.b + (int64_t)f * n;
      double jr = 0.0, js = 0.0;
      float dap = 0.f, rsq = 0.f;
      // ------------------------------------------------ E0: pooling / sparsity, H'
      ptx::mbar_wait(&S.u_full, nf & 1);
      ptx::tc_fence_after();
      for (int cc = 0; cc < KP / 32; ++cc) {
        float u[32];
        ptx::tmem_ld16(tl + cc * 32, u);
        ptx::tmem_ld16(tl + cc * 32 + 16, u + 16);
        ptx::tmem_ld_wait();
        float hq[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) u[t] *= S.sig[cc * 32 + t];
#pragma unroll
        for (int G0 = 0; G0 < 32; G0 += GP) {
          float ss = 0.f;
#pragma unroll
          for (int t = 0; t < GP; ++t) { float h = a * u[G0 + t]; ss = fmaf(h, h, ss); }
          const int G = (cc * 32 + G0) / GP;
          if (G < ng && svalid) {
            float sG = sqrtf(P.eps + ss);
            js += (double)sG;
            if (P.want_pooled) P.pooled[(((int64_t)gi * g.gr + fr) * g.gc + fc) * ng + G] = sG;
          }
        }
#pragma unroll
        for (int t = 0; t < 32; ++t) hq[t] = svalid ? S.sig[cc * 32 + t] * a * u[t] : 0.f;
        uint8_t *blk = S.H + (cc >> 1) * 16384;
#pragma unroll
        for (int t = 0; t < 32; t += 8) st8(blk, row, (cc & 1) * 32 + t, hq + t);
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&S.h_ready);
      q += T;   // pass-0 tiles
      // ------------------------------------------------ E1: residual, delta, db (pass 1)
      for (int j = 0; j < T; ++j, ++ur) {
        const uint32_t rb = ur & 1;
        ptx::mbar_wait(&S.r_full[rb], (ur >> 1) & 1);
        ptx::tc_fence_after();
        float rv[64];
#pragma unroll
        for (int c = 0; c < 64; c += 16) ptx::tmem_ld16(tl + 128 + 64 * rb + c, rv + c);
        ptx::tmem_ld_wait();
        const uint8_t *xs = S.X[(q + j) % NS] + (row >> 6) * 8192;
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          const int nn = j * NT + c;
          const float bv = nn < n ? __ldg(bf_ + nn) : 0.f;
          float e = rv[c] + bv - bf(xs, ptx::sw128_off(c, row & 63));
          e = svalid ? e : 0.f;
          jr += (double)(e * e);
          rv[c] = 2.f * e;
        }
        if (step) {
          const uint32_t db_ = ud & 1;
          ptx::mbar_wait(&S.dl_empty[db_], ((ud >> 1) & 1) ^ 1);
#pragma unroll
          for (int c = 0; c < 64; c += 8) st8(S.Dl[db_], row, c, rv + c);
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&S.dl_full[db_]);
          ++ud;
          // db partial: column sums over this warp's 32 samples (butterfly transpose-reduce)
#pragma unroll
          for (int o = 16, w = 32; o >= 1; o >>= 1, w >>= 1) {
            const bool up = lane & o;
#pragma unroll
            for (int t = 0; t < w; ++t) {
              float send = up ? rv[t] : rv[t + w];
              float keep = up ? rv[t + w] : rv[t];
              rv[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
          S.dbw[j & 1][ew][2 * lane] = rv[0];
          S.dbw[j & 1][ew][2 * lane + 1] = rv[1];
          ptx::named_bar_sync(1, 128);
          if (ew == 0) {
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int col = 2 * lane + h2, nn = j * NT + col;
              float sdb = S.dbw[j & 1][0][col] + S.dbw[j & 1][1][col] + S.dbw[j & 1][2][col] + S.dbw[j & 1][3][col];
              if (nn < n) P.db_part[((int64_t)f * CB + crank) * n + nn] = sdb;
            }
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&S.r_empty[rb]);
      }
      q += T;
      if (step) {
        // ---------------------------------------------- E1b: D = sigma.G~ + lambda h/s, dalpha, D'
        ptx::mbar_wait(&S.g_full, nf & 1);
        ptx::tc_fence_after();
        for (int cc = 0; cc < KP / 32; ++cc) {
          float u[32], gg[32];
          ptx::tmem_ld16(tl + cc * 32, u);
          ptx::tmem_ld16(tl + cc * 32 + 16, u + 16);
          ptx::tmem_ld16(tl + 256 + cc * 32, gg);
          ptx::tmem_ld16(tl + 256 + cc * 32 + 16, gg + 16);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 32; ++t) u[t] *= S.sig[cc * 32 + t];
#pragma unroll
          for (int G0 = 0; G0 < 32; G0 += GP) {
            float ss = 0.f;
#pragma unroll
            for (int t = 0; t < GP; ++t) { float h = a * u[G0 + t]; ss = fmaf(h, h, ss); }
            const float sG = sqrtf(P.eps + ss);
            const float inv = sG > 0.f ? P.lam / sG : 0.f;
#pragma unroll
            for (int t = 0; t < GP; ++t) {
              const int col = cc * 32 + G0 + t;
              float Dv = fmaf(S.sig[col], gg[G0 + t], a * u[G0 + t] * inv);
              Dv = (svalid && col < k) ? Dv : 0.f;
              dap = fmaf(Dv, u[G0 + t], dap);
              gg[G0 + t] = S.sig[col] * a * Dv;   // D'
            }
          }
          uint8_t *blk = S.D + (cc >> 1) * 16384;
#pragma unroll
          for (int t = 0; t < 32; t += 8) st8(blk, row, (cc & 1) * 32 + t, gg + t);
        }
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&S.d_ready);
        // ---------------------------------------------- E2: dX, dW, fused projected SGD (pass 2)
        const int own0 = CB > 1 ? 32 * (int)crank : 0;
        const float sg_r = S.sig[row];
        const float inv_sg = 1.f / sg_r;
        for (int j = 0; j < T; ++j, ++u2) {
          const uint32_t pb = u2 & 1, base = 192 * pb;
          ptx::mbar_wait(&S.p2_rdx[pb], (u2 >> 1) & 1);
          ptx::tc_fence_after();
          float rv[64];
  #pragma unroll
        for (int c = 0; c < 64; c += 16) ptx::tmem_ld16(tl + base + c, rv + c);
          ptx::tmem_ld_wait();
          const uint8_t *xs = S.X[(q + j) % NS] + (row >> 6) * 8192;
#pragma unroll
          for (int c = 0; c < 64; ++c) {
            const int nn = j * NT + c;
            const float bv = nn < n ? __ldg(bf_ + nn) : 0.f;
            float e = rv[c] + bv - bf(xs, ptx::sw128_off(c, row & 63));
            rv[c] = svalid ? 2.f * e : 0.f;
          }
          {
            const uint32_t db_ = ud & 1;
            ptx::mbar_wait(&S.dl_empty[db_], ((ud >> 1) & 1) ^ 1);
#pragma unroll
            for (int c = 0; c < 64; c += 8) st8(S.Dl[db_], row, c, rv + c);
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&S.dl_full[db_]);
            ++ud;
          }
          // dx = alpha W^T D - delta, overlap-added into the image gradient
          {
            float dv[64];
    #pragma unroll
        for (int c = 0; c < 64; c += 16) ptx::tmem_ld16(tl + base + 64 + c, dv + c);
            ptx::tmem_ld_wait();
            if (svalid) {
#pragma unroll
              for (int c = 0; c < 64; ++c) {
                const int nn = j * NT + c;
                if (nn < n) atomicAdd(P.dxt + (pixbase + S.off[nn]) * mp + gi, dv[c] - rv[c]);
              }
            }
          }
          // dW_j: lanes are filter rows; sum the batch slices over the cluster, then projected SGD
          ptx::mbar_wait(&S.p2_dw[pb], (u2 >> 1) & 1);
          ptx::tc_fence_after();
          float dw[64];
  #pragma unroll
        for (int c = 0; c < 64; c += 16) ptx::tmem_ld16(tl + base + 128 + c, dw + c);
          ptx::tmem_ld_wait();
          if (CB > 1) {
            // own columns [32*crank, +32) of this tile: move them to dw[0..31], send the rest to the peer
            if (crank) {
#pragma unroll
              for (int t = 0; t < 32; ++t) { float tmp = dw[t]; dw[t] = dw[t + 32]; dw[t + 32] = tmp; }
            }
            const uint32_t peer = crank ^ 1u;
            ptx::mbar_wait_cluster(&S.peer_free[pb], ((u2 >> 1) & 1) ^ 1);
            const uint32_t rbase = ptx::mapa(ptx::smem_u32(&S.recv[pb][0][row]), peer);
#pragma unroll
            for (int t = 0; t < 32; ++t) ptx::st_cluster_f32(rbase + t * 128 * 4, dw[32 + t]);
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(&S.recv_full[pb]), peer));
            ptx::mbar_wait_cluster(&S.recv_full[pb], (u2 >> 1) & 1);
#pragma unroll
            for (int t = 0; t < 32; ++t) dw[t] += S.recv[pb][t][row];
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(&S.peer_free[pb]), peer));
          }
          if (row < k) {
            const int64_t wrow = ((int64_t)f * k + row) * n;
            const int64_t brow = ((int64_t)f * KP + row) * P.n_al;
#pragma unroll
            for (int t = 0; t < (CB > 1 ? 32 : 64); ++t) {
              const int nn = j * NT + own0 + t;
              if (nn < n) {
                const float d = dw[t] * inv_sg;   // accumulator holds sigma_r * dJ/dW
                float upd = -P.lr * d;
                if (P.vW) { upd = fmaf(P.mu, P.vW[wrow + nn], upd); P.vW[wrow + nn] = upd; }
                const float wn = fmaf(sg_r, P.W[wrow + nn], upd);
                P.W[wrow + nn] = wn;
                P.Wb[brow + nn] = __float2bfloat16_rn(wn);
                rsq = fmaf(wn, wn, rsq);
                if (P.keep_grads) P.gW[wrow + nn] = d;
              }
            }
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&S.p2_empty[pb]);
        }
        q += T;
        P.rowsq_part[((int64_t)f * CB + crank) * KP + row] = rsq;
      }
      // ------------------------------------------------ per-field partial sums (fixed order)
      jr = warp_sum(jr);
      js = warp_sum(js);
      dap = warp_sum(dap);
      if (lane == 0) { S.redd[ew][0] = jr; S.redd[ew][1] = js; S.redf[ew] = dap; }
      ptx::named_bar_sync(1, 128);
      if (etid == 0) {
        double a0 = 0.0, a1 = 0.0;
        float a2 = 0.f;
        for (int w = 0; w < 4; ++w) { a0 += S.redd[w][0]; a1 += S.redd[w][1]; a2 += S.redf[w]; }
        P.loss_part[((int64_t)f * CB + crank) * 2 + 0] = a0;
        P.loss_part[((int64_t)f * CB + crank) * 2 + 1] = (double)P.lam * a1;
        P.da_part[(int64_t)f * CB + crank] = a2;
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&S.tmem_free);
    }
  }
  // ---- teardown
  ptx::tc_fence_before();
  __syncthreads();
  if (CB > 1) ptx::cluster_sync();
  if (warp == 1) ptx::tmem_dealloc<512>(tb);
}

// alpha / b update from the cluster partials, new row scales sigma' = 1/||W~'_row|| (unit-norm projection,
// PAPER.md:89), degenerate rows re-initialised, kept gradients for tests.
__global__ void __launch_bounds__(128) finalize_kernel(Geo g, int CB, int n_al, const float *da_part,
                                                       const float *db_part, const float *rowsq_part, float *alpha,
                                                       float *bvec, float *sigma, float *W, __nv_bfloat16 *Wb,
                                                       float *va, float *vb, float lr, float mu, float amin,
                                                       float *galpha, float *gb, uint64_t seed, int64_t step,
                                                       int row0, int col0, int ggc, int *reinit) {
  __shared__ double sh[32];
  __shared__ int bad[KP];
  __shared__ int nbad;
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
  for (int nn = threadIdx.x; nn < n; nn += blockDim.x) {
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
    for (int c = 0; c < CB; ++c) rs += rowsq_part[((int64_t)f * CB + c) * KP + r];
    if (!(rs > 0.f)) {
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
    const uint64_t key = splitmix64(seed ^ ((uint64_t)step << 40) ^ (gf << 20) ^ (uint64_t)r);
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
      W[((int64_t)f * k + r) * n + t] = w;
      Wb[((int64_t)f * KP + r) * n_al + t] = __float2bfloat16_rn(w);
    }
    __syncthreads();
  }
}

}  // namespace tc

struct TcScratch {
  int CB = 1, T = 0, grid = 0;
  size_t smem = 0;
  double *loss_part = nullptr;
  float *da_part = nullptr, *db_part = nullptr, *rowsq_part = nullptr;
  CUtensorMap tmW;
};

lcae_status tc_alloc(lcae_layer *L) {
  const Geo &g = L->geo;
  if (g.k > tc::KP) { set_error("bf16 path: filters per field must be <= 128"); return LCAE_ERR_CONFIG; }
  if (g.m > 2 * tc::MC) { set_error("bf16 path: batch must be <= 256"); return LCAE_ERR_CONFIG; }
  const int T = cdiv(g.n, tc::NT);
  if (T * tc::NT > tc::MAX_NPAD) { set_error("bf16 path: rf_h*rf_w*C must be <= 2048"); return LCAE_ERR_CONFIG; }
  TcScratch *s = new TcScratch();
  L->tc = s;
  s->CB = cdiv(g.m, tc::MC);
  s->T = T;
  s->smem = sizeof(tc::Smem) + 1024;
  const int ncl = std::max(1, std::min(g.F, L->sm_count / s->CB));
  s->grid = ncl * s->CB;
  LCAE_CK(cudaMalloc(&s->loss_part, (size_t)g.F * s->CB * 2 * sizeof(double)));
  LCAE_CK(cudaMalloc(&s->da_part, (size_t)g.F * s->CB * 4));
  LCAE_CK(cudaMalloc(&s->db_part, (size_t)g.F * s->CB * g.n * 4));
  LCAE_CK(cudaMalloc(&s->rowsq_part, (size_t)g.F * s->CB * tc::KP * 4));
  // Wb is [F][KP][n_al] (pad rows zero) for the bf16 path
  cudaFree(L->Wb);
  LCAE_CK(cudaMalloc(&L->Wb, (size_t)g.F * tc::KP * L->n_al * 2));
  LCAE_CK(cudaMemset(L->Wb, 0, (size_t)g.F * tc::KP * L->n_al * 2));
  if (!make_tmap_2d_bf16(&s->tmW, L->Wb, (uint64_t)g.F * tc::KP, (uint64_t)L->n_al, (uint64_t)L->n_al, tc::KP)) {
    set_error("cuTensorMapEncodeTiled failed for W");
    return LCAE_ERR_CUDA;
  }
  return LCAE_OK;
}

void tc_free(lcae_layer *L) {
  if (!L->tc) return;
  TcScratch *s = L->tc;
  for (void *p : {(void *)s->loss_part, (void *)s->da_part, (void *)s->db_part, (void *)s->rowsq_part})
    if (p) cudaFree(p);
  delete s;
  L->tc = nullptr;
}

lcae_status tc_step(lcae_layer *L, bool update, bool want_pooled) {
  const Geo &g = L->geo;
  TcScratch *s = L->tc;
  tc::Params P;
  P.tmW = s->tmW;
  P.g = g;
  P.T = s->T;
  P.mp = L->mp;
  P.CB = s->CB;
  P.n_al = L->n_al;
  P.mode = update ? 1 : 0;
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
  P.gW = L->gW;
  if (update) LCAE_CK(cudaMemsetAsync(L->dxt, 0, (size_t)g.H * g.W * g.C * L->mp * 4, L->st));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(s->grid);
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
#define LCAE_PICK(GPV)                                                        \
  if (g.g == GPV) kern = s->CB == 1 ? tc::step_kernel<GPV, 1> : tc::step_kernel<GPV, 2>;
  LCAE_PICK(1) LCAE_PICK(2) LCAE_PICK(4) LCAE_PICK(8) LCAE_PICK(16) LCAE_PICK(32)
#undef LCAE_PICK
  if (!kern) { set_error("unsupported pool group"); return LCAE_ERR_CONFIG; }
  LCAE_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem));
  const bool prof = L->prof_on && L->prof_n < 4096;
  if (prof) LCAE_CK(cudaEventRecord(L->prof_ev[2 * L->prof_n], L->st));
  LCAE_CK(cudaLaunchKernelEx(&cfg, kern, P));
  LCAE_CK_LAUNCH(L);
  if (prof) LCAE_CK(cudaEventRecord(L->prof_ev[2 * L->prof_n++ + 1], L->st));
  if (update) {
    tc::finalize_kernel<<<g.F, 128, 0, L->st>>>(
        g, s->CB, L->n_al, s->da_part, s->db_part, s->rowsq_part, L->alpha, L->b, L->sigma, L->W, L->Wb, L->va,
        L->vb, L->cfg.lr, L->cfg.momentum, L->cfg.alpha_min, L->cfg.keep_grads ? L->galpha : nullptr,
        L->cfg.keep_grads ? L->gb : nullptr, L->cfg.seed, L->steps, L->cfg.field_row0, L->cfg.field_col0,
        L->cfg.global_grid_c, L->reinit_dev);
    LCAE_CK_LAUNCH(L);
  }
  return LCAE_OK;
}

double *tc_loss_part(lcae_layer *L) { return L->tc ? L->tc->loss_part : nullptr; }
int tc_loss_count(lcae_layer *L) { return L->tc ? L->geo.F * L->tc->CB : 0; }

}  // namespace lcae
