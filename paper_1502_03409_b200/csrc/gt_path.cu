// gt_path.cu — the general bf16 tensor-core path: layers the fused step kernel cannot hold (k > 128 filters, n > 4096,
// m > 256; the paper's own layer 1, c3', has k = 384: PAPER.md:95) run the step as five batched tcgen05 GEMMs with
// their epilogues doing the element-wise work. Same step, same notation as f32_path.cu (PAPER.md:88 / DESIGN.md
// R1-R11), same operand rounding and the same lazy projection as the fused kernel (bf16 x, W~, sigma h, delta,
// sigma alpha D; fp32 accumulation; fp32 master W~ with per-row scale sigma, W = sigma (.) W~):
//   U  = sigma (.) W~ X_f           (k x m)   GEMM 1, epilogue: h = alpha U, sigma h (bf16), s_G, p, J_s partials
//   R  = W~^T (sigma h)             (n x m)   GEMM 2, epilogue: delta = 2(R + b - x) (bf16), J_r, db partials
//   G  = sigma (.) W~ delta         (k x m)   GEMM 3, epilogue: D = G + lambda h / s, sigma alpha D (bf16), dalpha
//   dXp^T = (sigma alpha D)^T W~ - delta^T (m x n) GEMM 5, epilogue subtracts delta and TMA-reduce-adds into dX
//   sigma dW = (sigma h) delta^T + (sigma alpha D) X^T (k x n) GEMM 4 (two K segments into one accumulator),
//            epilogue: W~' = W~ - (lr / sigma^2) acc (master + bf16 shadow, TMA stores), ||W~'||^2 row partials;
//   gt_finalize: sigma' = 1 / ||W~'||, degenerate rows; update_ab_f32: alpha, b.
// Only U and the bf16 operands are written between the GEMMs (fixed-order partial sums, reduced per field by
// gt_parts / gt_finalize: deterministic).
#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.cuh"

#include <algorithm>
#include <cfloat>

namespace lcae {
namespace gt {

constexpr int BM = 128, BK = 64;
// operand ring depth and shared memory: + per epilogue warp 16 KB of staging (SGD: 24 KB, a 4-slot W~ ring)
constexpr int stages(int BN, bool sgd) { return sgd ? 2 : BN >= 192 ? 3 : 4; }
constexpr int warp_stage_bytes(bool sgd) { return sgd ? 24576 : 16384; }
constexpr int smem_bytes(int BN, bool sgd) {
  return stages(BN, sgd) * (BM * BK * 2 + BN * BK * 2) + 4 * warp_stage_bytes(sgd) + 1024;
}

// Epilogue modes: the per-element work between the GEMMs runs on the accumulator tile while it is in registers.
// POOLP: POOL + the pooled code p; SGD / SGDF: the projected SGD of W~ on the dW accumulator (lean / with momentum or
// kept gradients).
// DXRED: the transposed input-gradient GEMM (rows = samples, columns = patch rows): subtract delta and reduce-add into
// the image gradient by TMA (boxes of consecutive pixel-feature rows).
enum { EPI_PLAIN = 0, EPI_POOL = 1, EPI_RESID = 2, EPI_DCODE = 3, EPI_POOLP = 5, EPI_SGD = 6, EPI_SGDF = 7, EPI_DXRED = 8 };

struct GemmArgs {
  CUtensorMap tmA[2], tmB[2];
  int bA[2], bB[2];   // batch-coordinate offset of each operand map (W maps: the chunk's first field)
  int nseg, M, N, K, batch, bn;   // bn: N tile width (choose_bn)
  CUtensorMap tmC, tmO;   // store maps of C (fp32, box 32 x 32) and O16 (bf16, box 64 x 32), 128B swizzle
  float *C;           // fp32 output (PLAIN, POOL: U)
  int64_t cbs, crs;   // C[b][i][j] at C + b cbs + i crs + j (cbs, crs multiples of 8); every per-element side
                      // buffer below (bf16 or fp32) has this layout
  // epilogue operands
  int f0, g, gr, gc;  // chunk's first field; pooling group; field grid
  float lam, eps;
  const float *alpha, *bvec, *U;         // alpha [F], b [F][n] (RESID), U (DCODE)
  const __nv_bfloat16 *I16;              // x (RESID)
  __nv_bfloat16 *O16;                    // h (POOL), delta (RESID), alpha D (DCODE)
  float *pooled;                         // p [m][gr][gc][k/g] (POOL, nullable)
  double *part;                          // per (b, M tile, N tile, warp) partial: sum s, sum e^2, sum D.U
  float *dbp;                            // db (RESID) / ||W~'||^2 (SGD) row partials [b][N tiles][M]
  int sb;                                // batch-coordinate offset of the stores (SGD: the chunk's first field)
  // row scales and SGD operands: W = sigma (.) W~ (the bf16 shadow holds W~); the dW accumulator holds sigma dJ/dW
  const float *sigma;                    // [F][k]
  const float *W;                        // W~ master [F][k][wp] (SGD side input)
  float *vW, *gW;                        // velocity, kept gradient (SGDF; nullable)
  int64_t wp;
  float lr, mu;
  const int *flags;                      // sticky error flags: set -> no parameter writes
  // DXRED: the image gradient [H W C rows][mp samples] fp32 as TMA reduce targets with box heights 1, 2, .., 32;
  // patch row j of field f is pixel-feature row base(f) + ry W C + (j - ry RW), ry = j / RW
  CUtensorMap tmR[6];
  int RW, s, Cc;
  int64_t WC;
};

// C[b] (M x N, fp32) = sum over segments of A_s[b] (M x K) B_s[b] (K x N); A K-major ([M][K] in global) or
// MN-major ([K][M]); B K-major ([N][K]) or MN-major ([K][N]). Canonical SW128 layouts as in tc_kernel.cuh
// (descriptor conventions pinned by tests/test_gpu_selftest.py).
template <bool AMN, bool BMN, int BN, int EPI>
__global__ void __launch_bounds__(192, 1) bgemm(const __grid_constant__ GemmArgs P) {
  constexpr bool POOLING = EPI == EPI_POOL || EPI == EPI_POOLP;
  constexpr bool SGD = EPI == EPI_SGD || EPI == EPI_SGDF;
  constexpr int ST = stages(BN, SGD);
  constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE = A_BYTES + B_BYTES;
  constexpr uint32_t TCOLS = 2 * BN <= 256 ? 256 : 512;
  constexpr uint32_t WST = warp_stage_bytes(SGD), OFF16 = SGD ? 16384 : 8192;   // per-warp staging, bf16 boxes
  constexpr bool st32 = EPI == EPI_PLAIN || POOLING || SGD;   // fp32 output (C / W~ master)
  constexpr bool st16 = POOLING || EPI == EPI_RESID || EPI == EPI_DCODE || SGD;   // bf16 output (O16 / shadow)
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[ST], empty[ST], tfull[2], tempty[2];
  constexpr bool RING = SGD || EPI == EPI_DXRED;
  __shared__ uint64_t ringb[RING ? 16 : 1];   // per epilogue warp, 4 ring slots (SGD: W~ boxes, DXRED: delta boxes)
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = cdiv(P.M, BM), nt = cdiv(P.N, BN), per = mt * nt;
  const int ntiles = P.batch * per, ksteps = cdiv(P.K, BK);
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { ptx::mbar_init(&tfull[s], 1); ptx::mbar_init(&tempty[s], 4); }
    if (RING)
      for (int s = 0; s < 16; ++s) ptx::mbar_init(&ringb[s], 1);
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
  } else {
    // Epilogue: warp w drains TMEM lanes [32 (w % 4), +32) = rows of the tile, 32 columns at a time; results go
    // through this warp's 128B-swizzled staging boxes (two fp32 32 x 32, two bf16 32 x 64: double-buffered) and
    // leave by TMA tensor stores (ragged rows / columns clipped by the tensor bounds).
    const int q = warp & 3, ew = warp - 2, sw = lane & 7;
    // [0, 8K): fp32 boxes (SGD: [0, 16K) the W~ ring, read and rewritten in place), then two bf16 boxes
    uint8_t *stg = smem + ST * STAGE + ew * WST;
    // SGD: the W~ master box (32 rows x 32 columns) of chunk `nc` is TMA-loaded into ring slot nc % 4, two chunks
    // ahead; the slot was last read by the store group of chunk nc - 4 (or nc - 2 when issued mid-tile)
    // DXRED: the delta box (32 patch rows x 32 samples, bf16) of chunk nc goes to slot nc % 4 of [8K, 16K)
    auto ring_load = [&](uint32_t nc, int jj, int row0_, int bb) {
      if constexpr (SGD) {
        uint64_t *bar = &ringb[ew * 4 + (nc & 3)];
        ptx::mbar_arrive_expect_tx(bar, 4096);
        ptx::tma_load_3d(stg + (nc & 3) * 4096, &P.tmC, bar, jj, row0_, bb);
      } else if constexpr (EPI == EPI_DXRED) {
        uint64_t *bar = &ringb[ew * 4 + (nc & 3)];
        ptx::mbar_arrive_expect_tx(bar, 2048);
        ptx::tma_load_3d(stg + 8192 + (nc & 3) * 2048, &P.tmO, bar, row0_, jj, bb);   // (samples, patch rows)
      }
    };
    uint32_t tc = 0, nchunk = 0, nbox = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tc) {
      const int b = tile / per, r = tile - b * per, mi = r / nt, ni = r % nt, m0 = mi * BM, n0 = ni * BN;
      const uint32_t buf = tc & 1;
      const int row0 = m0 + 32 * q, i = row0 + lane, f = P.f0 + b;
      const bool rv = i < P.M;
      // this row's offset in the side inputs (rows past M read row M - 1 and are masked; the sample pitch is a
      // multiple of 32, so a 32-column chunk never leaves its row)
      const int64_t ro = b * P.cbs + (int64_t)(rv ? i : P.M - 1) * P.crs;
      const float a = (POOLING || EPI == EPI_DCODE) ? P.alpha[f] : 0.f;
      const float brow = (EPI == EPI_RESID && rv) ? P.bvec[(int64_t)f * P.M + i] : 0.f;
      const float sgr = (POOLING || EPI == EPI_DCODE || SGD) && rv ? P.sigma[(int64_t)f * P.M + i] : 1.f;
      const int64_t wrow = ((int64_t)f * P.M + (rv ? i : P.M - 1)) * P.wp;   // W~ master row (SGD)
      const bool frozen = SGD && (P.flags[0] | P.flags[1]);
      double part = 0.0;
      float dbs = 0.f;
      // per-element side input (x / delta in bf16, U or W~ in fp32), loaded one 32-column chunk ahead in registers:
      // the first chunk's loads are in flight while the accumulator is still being computed
      constexpr bool has_in = EPI == EPI_RESID || EPI == EPI_DCODE;
      uint32_t raw[has_in ? 32 : 1];
      auto load_in = [&](int jj) {
        if constexpr (EPI == EPI_RESID) {
          const uint4 *src = reinterpret_cast<const uint4 *>(P.I16 + ro + jj);
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const uint4 u = src[h];
            raw[4 * h] = u.x; raw[4 * h + 1] = u.y; raw[4 * h + 2] = u.z; raw[4 * h + 3] = u.w;
          }
        } else if constexpr (has_in) {
          const float4 *src = reinterpret_cast<const float4 *>(P.U + ro + jj);
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            const float4 u = src[h];
            raw[4 * h] = __float_as_uint(u.x); raw[4 * h + 1] = __float_as_uint(u.y);
            raw[4 * h + 2] = __float_as_uint(u.z); raw[4 * h + 3] = __float_as_uint(u.w);
          }
        }
      };
      if constexpr (has_in) load_in(n0);
      if constexpr (RING) {
        ptx::fence_proxy_async_smem();   // this warp's earlier reads of the slots precede the TMA writes
        __syncwarp();
        if (lane == 0) {
          if (SGD) ptx::bulk_wait_read1();
          ring_load(nchunk, n0, row0, P.sb + b);
          if (32 < BN && n0 + 32 < P.N) ring_load(nchunk + 1, n0 + 32, row0, P.sb + b);
        }
      }
      ptx::mbar_wait(&tfull[buf], (tc >> 1) & 1);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < BN; c += 32, ++nchunk) {
        if (n0 + c >= P.N) break;   // warp-uniform
        const int j0 = n0 + c;
        float in[32];
        if constexpr (EPI == EPI_RESID) {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            in[2 * t] = __uint_as_float(raw[t] << 16);
            in[2 * t + 1] = __uint_as_float(raw[t] & 0xFFFF0000u);
          }
        } else if constexpr (has_in) {
#pragma unroll
          for (int t = 0; t < 32; ++t) in[t] = __uint_as_float(raw[t]);
        }
        if constexpr (has_in)
          if (c + 32 < BN && j0 + 32 < P.N) load_in(j0 + 32);
        if constexpr (EPI == EPI_DXRED) {
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && c + 64 < BN && j0 + 64 < P.N) ring_load(nchunk + 2, j0 + 64, row0, b);
          ptx::mbar_wait(&ringb[ew * 4 + (nchunk & 3)], (nchunk >> 2) & 1);
          const __nv_bfloat16 *slot = reinterpret_cast<const __nv_bfloat16 *>(stg + 8192 + (nchunk & 3) * 2048);
#pragma unroll
          for (int t = 0; t < 32; ++t) in[t] = __bfloat162float(slot[t * 32 + lane]);   // delta[j0 + t][i]
        }
        if constexpr (SGD) {
          if (lane == 0) {
            ptx::bulk_wait_read1();   // chunk nchunk - 2's store has read slot (nchunk + 2) % 4
            if (c + 64 < BN && j0 + 64 < P.N) ring_load(nchunk + 2, j0 + 64, row0, P.sb + b);
          }
          ptx::mbar_wait(&ringb[ew * 4 + (nchunk & 3)], (nchunk >> 2) & 1);
          const float *slot = reinterpret_cast<const float *>(stg + (nchunk & 3) * 4096);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 w4 = *reinterpret_cast<const float4 *>(slot + lane * 32 + 4 * (u ^ sw));
            in[4 * u] = w4.x; in[4 * u + 1] = w4.y; in[4 * u + 2] = w4.z; in[4 * u + 3] = w4.w;
          }
        }
        float v[32];
        ptx::tmem_ld16(tbase + ((uint32_t)(32 * q) << 16) + buf * BN + c, v);
        ptx::tmem_ld16(tbase + ((uint32_t)(32 * q) << 16) + buf * BN + c + 16, v + 16);
        ptx::tmem_ld_wait();
        uint32_t okm = 0;   // valid columns of this row
#pragma unroll
        for (int t = 0; t < 32; ++t) okm |= (rv && j0 + t < P.N) ? 1u << t : 0u;
        float o[32];        // fp32 result (C) or the value rounded to the bf16 side output
        if constexpr (EPI == EPI_PLAIN) {
#pragma unroll
          for (int t = 0; t < 32; ++t) o[t] = v[t];
        } else if constexpr (EPI == EPI_DXRED) {
          // this thread: sample i; columns: patch rows j0 .. j0 + 31 (delta from the ring box, zero past the edges)
#pragma unroll
          for (int t = 0; t < 32; ++t) o[t] = v[t] - in[t];   // dXp^T = (sigma alpha D)^T W~ - delta^T
        } else if constexpr (SGD) {
          // the accumulator holds sigma dJ/dW. Lean: rownorm(sigma W~ - lr dJ/dW) = rownorm(W~ - (lr / sigma^2) acc),
          // so W~ is updated without the sigma scale and sigma' = 1 / ||W~'|| (gt_finalize); with momentum the
          // velocity lives in W's scale and W~' = sigma W~ + v (as the fused kernel)
          const float isg = 1.f / sgr, cr = -P.lr * isg;
          float rs = 0.f;
          float vo[32];
          if constexpr (EPI == EPI_SGDF) {
            if (P.vW) {
#pragma unroll
              for (int t = 0; t < 32; t += 4) {
                const float4 q4 = *reinterpret_cast<const float4 *>(P.vW + wrow + j0 + t);
                vo[t] = q4.x; vo[t + 1] = q4.y; vo[t + 2] = q4.z; vo[t + 3] = q4.w;
              }
            }
          }
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const float acc = (okm >> t & 1) ? v[t] : 0.f;
            if constexpr (EPI == EPI_SGD) {
              o[t] = fmaf(cr * isg, acc, in[t]);
            } else {
              float upd = cr * acc;
              if (P.vW) { upd = fmaf(P.mu, vo[t], upd); vo[t] = upd; }
              o[t] = fmaf(sgr, in[t], upd);
              v[t] = acc * isg;   // dJ/dW (kept gradient)
            }
            rs = fmaf(o[t], o[t], rs);
          }
          dbs += rs;
          if constexpr (EPI == EPI_SGDF) {
            if (rv && !frozen) {
#pragma unroll
              for (int t = 0; t < 32; t += 4) {
                if (P.vW) *reinterpret_cast<float4 *>(P.vW + wrow + j0 + t) = make_float4(vo[t], vo[t + 1], vo[t + 2], vo[t + 3]);
                if (P.gW) *reinterpret_cast<float4 *>(P.gW + wrow + j0 + t) = make_float4(v[t], v[t + 1], v[t + 2], v[t + 3]);
              }
            }
          }
        } else if constexpr (EPI == EPI_RESID) {
          float jr = 0.f;
#pragma unroll
          for (int t = 0; t < 32; ++t) {   // e = r + b - x; delta = 2e
            const float e = (okm >> t & 1) ? v[t] + brow - in[t] : 0.f;
            jr = fmaf(e, e, jr);
            o[t] = 2.f * e;
            dbs += o[t];
          }
          part += (double)jr;
        } else {   // POOL (h = alpha U) or DCODE (D = G + lambda h / s, output alpha D): group sums over g rows
          float ss[32];
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            v[t] *= sgr;   // U = sigma (.) (W~ X) or G = sigma (.) (W~ delta)
            const float h = (okm >> t & 1) ? a * (POOLING ? v[t] : in[t]) : 0.f;
            ss[t] = h * h;
          }
          for (int w = 1; w < P.g; w <<= 1)
#pragma unroll
            for (int t = 0; t < 32; ++t) ss[t] += __shfl_xor_sync(0xffffffffu, ss[t], w);
          const bool lead = (lane & (P.g - 1)) == 0;
          float acc = 0.f;
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            if constexpr (POOLING) {
              const float sg = sqrtf(P.eps + ss[t]);
              o[t] = sgr * a * v[t];   // sigma h: the decode W^T h = W~^T (sigma h), dW's first term sigma h delta^T
              if (lead && (okm >> t & 1)) {
                acc += sg;
                if constexpr (EPI == EPI_POOLP)
                  P.pooled[(((int64_t)(j0 + t) * P.gr + f / P.gc) * P.gc + f % P.gc) * (P.M / P.g) + i / P.g] = sg;
              }
            } else {
              // lambda / s_G (as the fused kernel: s_G = 0 only with h = 0, where the product below is 0; R12)
              const float inv = P.lam * rsqrtf(fmaxf(P.eps + ss[t], 1.17549435e-38f));
              const float D = (okm >> t & 1) ? fmaf(a * in[t], inv, v[t]) : 0.f;
              acc = fmaf(D, in[t], acc);   // dalpha = sum D (.) U
              o[t] = sgr * a * D;   // sigma alpha D (as sigma h above)
            }
          }
          part += (double)acc;
        }
        // staging: the chunk's buffers were last read by the store group of chunk nchunk - 2
        if (lane == 0) ptx::bulk_wait_read1();
        __syncwarp();
        if constexpr (st32) {
          float *sb32 = reinterpret_cast<float *>(stg + (SGD ? (nchunk & 3) : (nchunk & 1)) * 4096);
          const float *src = POOLING ? v : o;   // POOL keeps U (fp32) for GEMM 3's epilogue
#pragma unroll
          for (int u = 0; u < 8; ++u)
            *reinterpret_cast<float4 *>(sb32 + lane * 32 + 4 * (u ^ sw)) =
                make_float4(src[4 * u], src[4 * u + 1], src[4 * u + 2], src[4 * u + 3]);
        }
        if constexpr (EPI == EPI_DXRED) {   // [32 patch rows][32 samples]: lane = sample, conflict-free rows
          float *sbr = reinterpret_cast<float *>(stg + (nchunk & 1) * 4096);
#pragma unroll
          for (int t = 0; t < 32; ++t) sbr[t * 32 + lane] = o[t];
        }
        const int hb = (c >> 5) & 1;   // 32-column half of the 64-column bf16 box
        const bool box_done = hb == 1 || n0 + c + 32 >= P.N;
        if constexpr (st16) {
          uint8_t *sb16 = stg + OFF16 + (nbox & 1) * 4096;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<uint4 *>(sb16 + lane * 128 + 16 * ((4 * hb + u) ^ sw)) =
                make_uint4(ptx::pack_bf16x2(o[8 * u], o[8 * u + 1]), ptx::pack_bf16x2(o[8 * u + 2], o[8 * u + 3]),
                           ptx::pack_bf16x2(o[8 * u + 4], o[8 * u + 5]), ptx::pack_bf16x2(o[8 * u + 6], o[8 * u + 7]));
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (!frozen) {
            if constexpr (st32)
              ptx::tma_store_3d(&P.tmC, stg + (SGD ? (nchunk & 3) : (nchunk & 1)) * 4096, j0, row0, P.sb + b);
            if constexpr (st16)
              if (box_done) ptx::tma_store_3d(&P.tmO, stg + OFF16 + (nbox & 1) * 4096, j0 - 32 * hb, row0, P.sb + b);
          }
          if constexpr (EPI == EPI_DXRED) {
            if (!frozen) {
              // the chunk's patch rows split into runs of consecutive pixel-feature rows, each into power-of-two boxes
              const int fr = f / P.gc, fc = f - fr * P.gc;
              const int64_t base = (int64_t)fr * P.s * P.WC + (int64_t)fc * P.s * P.Cc;
              const int jend = min(j0 + 32, P.N);
              for (int ja = j0; ja < jend;) {
                const int ry = ja / P.RW, run_end = min(jend, (ry + 1) * P.RW);
                int h = run_end - ja;
                while (h > 0) {
                  const int lg = min(5, 31 - __clz(h));
                  ptx::tma_red_add_2d(&P.tmR[lg], stg + (nchunk & 1) * 4096 + (ja - j0) * 128, m0 + 32 * q,
                                      (int)(base + (int64_t)ry * P.WC + (ja - ry * P.RW)));
                  ja += 1 << lg;
                  h -= 1 << lg;
                }
              }
            }
          }
          ptx::bulk_commit();   // one group per chunk (possibly empty)
        }
        if (st16 && box_done) ++nbox;
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
      if constexpr (EPI != EPI_PLAIN && EPI != EPI_DXRED && !SGD) {   // fixed-order partials (gt_parts sums them)
        part = warp_sum(part);
        if (lane == 0) P.part[((int64_t)(b * mt + mi) * nt + ni) * 4 + q] = part;
      }
      if ((EPI == EPI_RESID || SGD) && rv) P.dbp[((int64_t)b * nt + ni) * P.M + i] = dbs;
    }
    if (lane == 0) ptx::bulk_wait0();   // this warp's stores have completed
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TCOLS>(tbase);
  }
}

template <bool AMN, bool BMN, int BN, int EPI>
lcae_status launch_bn(lcae_layer *L, const GemmArgs &a) {
  constexpr int smem = smem_bytes(BN, EPI == EPI_SGD || EPI == EPI_SGDF);
  static bool attr = false;
  if (!attr) {
    LCAE_CK(cudaFuncSetAttribute(bgemm<AMN, BMN, BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const int tiles = a.batch * cdiv(a.M, BM) * cdiv(a.N, BN);
  const bool prof = L->prof_on && L->prof_n < 4096;   // lcae_profile: events around every GEMM launch
  if (prof) LCAE_CK(cudaEventRecord(L->prof_ev[2 * L->prof_n], L->st));
  bgemm<AMN, BMN, BN, EPI><<<std::min(tiles, L->sm_count), 192, smem, L->st>>>(a);
  LCAE_CK_LAUNCH(L);
  if (prof) LCAE_CK(cudaEventRecord(L->prof_ev[2 * L->prof_n++ + 1], L->st));
  return LCAE_OK;
}

inline int pick_bn(int N) { return N <= 64 ? 64 : N <= 128 ? 128 : N <= 192 ? 192 : 256; }

// N tile width: the narrowest of {64, 128, 192, 256} covering N, narrowed further for single-field layers whose
// tiles would not fill the SMs (the paper's dense layer: one field, 32 M tiles) -- only with an MN-major B, whose boxes are 64
// columns wide whatever BN is (K-major B maps are built for the chosen BN). Fixed per layer (the epilogue partial
// sums are laid out by N tile).
inline int choose_bn(int M, int N, int batch, bool bmn, int sms, int F) {
  int bn = pick_bn(N);
  if (bmn && F <= 2)   // single-field (dense) layers only: a tiled (model-parallel) layer keeps the untiled N tiling
    while (bn > 64 && (int64_t)batch * cdiv(M, BM) * cdiv(N, bn) < sms) bn = bn == 256 ? 192 : bn - 64;
  return bn;
}

template <bool AMN, bool BMN, int EPI>
lcae_status gemm(lcae_layer *L, const GemmArgs &a) {
  switch (a.bn) {
    case 64: return launch_bn<AMN, BMN, 64, EPI>(L, a);
    case 128: return launch_bn<AMN, BMN, 128, EPI>(L, a);
    case 192: return launch_bn<AMN, BMN, 192, EPI>(L, a);
    default: return launch_bn<AMN, BMN, 256, EPI>(L, a);
  }
}

// ---------------------------------------------------------------- epilogue kernels (one block per field)

// X_f (n x m) gathered from the HWCN bf16 image into [Fc][n][mp] (16-byte runs; rows of one receptive-field row are
// consecutive pixel-features).
__global__ void __launch_bounds__(256) gt_gather(Geo g, int f0, int mp, int mq, const __nv_bfloat16 *xt16,
                                                 __nv_bfloat16 *Xp) {
  const int b = blockIdx.x, f = f0 + b, r = f / g.gc, c = f - r * g.gc;
  const int q8 = mq / 8, p8 = mp / 8;   // 16-byte runs per row: destination (pitch mq), source (pitch mp)
  const int64_t rowstride = (int64_t)g.W * g.C;   // pixel-features per image row
  const int64_t base = ((int64_t)r * g.s * rowstride + (int64_t)c * g.s * g.C) * mp;
  const uint4 *src = reinterpret_cast<const uint4 *>(xt16);
  uint4 *dst = reinterpret_cast<uint4 *>(Xp + (int64_t)b * g.n * mq);
  for (int t = blockIdx.y * blockDim.x + threadIdx.x; t < g.n * q8; t += gridDim.y * blockDim.x) {
    const int row = t / q8, qq = t - row * q8, ry = row / g.RW;
    const int64_t off = base + ((int64_t)ry * rowstride + (row - ry * g.RW)) * mp;
    dst[t] = qq < p8 ? src[off / 8 + qq] : make_uint4(0, 0, 0, 0);
  }
}

// Per-field sums of the epilogue partials in a fixed order (deterministic): J_s = lambda sum s (GEMM 1), J_r (GEMM 2),
// dalpha (GEMM 3), db = sum over N tiles of the per-row partials (GEMM 2).
__global__ void __launch_bounds__(256) gt_parts(int f0, int n, float lam, const double *P1, int n1, const double *P2,
                                                int n2, const double *P3, int n3, const float *dbp, int nt2,
                                                double *loss_part, float *da, float *db, int enc) {
  const int b = blockIdx.x, f = f0 + b;
  if (threadIdx.x == 0 && blockIdx.y == 0) {
    double s1 = 0.0;
    for (int e = 0; e < n1; ++e) s1 += P1[(int64_t)b * n1 + e];
    loss_part[2 * f + 1] = (double)lam * s1;
    if (P2) {
      double s2 = 0.0;
      for (int e = 0; e < n2; ++e) s2 += P2[(int64_t)b * n2 + e];
      loss_part[2 * f] = s2;
    } else if (enc) {
      loss_part[2 * f] = 0.0;
    }
    if (P3) {
      double s3 = 0.0;
      for (int e = 0; e < n3; ++e) s3 += P3[(int64_t)b * n3 + e];
      da[b] = (float)s3;
    }
  }
  if (P2)
    for (int row = blockIdx.y * blockDim.x + threadIdx.x; row < n; row += gridDim.y * blockDim.x) {
      float acc = 0.f;
      for (int t = 0; t < nt2; ++t) acc += dbp[((int64_t)b * nt2 + t) * n + row];
      db[(int64_t)b * n + row] = acc;
    }
}

// New row scales sigma' = 1 / ||W~'_row|| from the SGD epilogue's row partials (fixed order; PAPER.md:89 unit-norm
// projection), degenerate rows re-initialised from the counter-based generator (as the fused path).
__global__ void __launch_bounds__(128) gt_finalize(Geo g, int f0, int nt4, const float *rsqp, float *sigma, float *W,
                                                   __nv_bfloat16 *Wb, int64_t wp, int n_al, float *vW, uint64_t seed,
                                                   const int64_t *step_dev, int row0, int col0, int ggc, int *reinit,
                                                   const int *flags) {
  __shared__ double sh[32];
  __shared__ int bad[128];
  __shared__ int nbad;
  __shared__ float s_inv;
  if (flags[0] | flags[1]) return;   // flagged step: parameters frozen (include/lcae.h "Errors")
  const int b = blockIdx.x, f = f0 + b, k = g.k, n = g.n;
  if (threadIdx.x == 0) nbad = 0;
  __syncthreads();
  for (int r = blockIdx.y * blockDim.x + threadIdx.x; r < k; r += gridDim.y * blockDim.x) {
    float rs = 0.f;
    for (int t = 0; t < nt4; ++t) rs += rsqp[((int64_t)b * nt4 + t) * k + r];
    if (!(rs >= FLT_MIN)) {   // R13: squared row norm below the smallest normal float
      const int slot = atomicAdd(&nbad, 1);
      if (slot < 128) bad[slot] = r;
    } else {
      sigma[(int64_t)f * k + r] = rsqrtf(rs);
    }
  }
  __syncthreads();
  const int nb = min(nbad, 128);
  for (int ib = 0; ib < nb; ++ib) {   // rare path
    const int r = bad[ib];
    const int fr = f / g.gc, fc = f - fr * g.gc;
    const uint64_t gf = (uint64_t)((row0 + fr) * ggc + col0 + fc);
    const uint64_t key = splitmix64(seed ^ ((uint64_t)*step_dev << 40) ^ (gf << 20) ^ (uint64_t)r);
    double a2 = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const double u = (double)(splitmix64(key + (uint64_t)t) >> 40) / 16777216.0 - 0.5;
      a2 += u * u;
    }
    const double tot = block_sum_f64(a2, sh);
    if (threadIdx.x == 0) { s_inv = (float)(1.0 / sqrt(tot)); atomicAdd(reinit, 1); sigma[(int64_t)f * k + r] = 1.f; }
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const double u = (double)(splitmix64(key + (uint64_t)t) >> 40) / 16777216.0 - 0.5;
      const float w = (float)u * s_inv;
      W[((int64_t)f * k + r) * wp + t] = w;
      Wb[((int64_t)f * k + r) * n_al + t] = __float2bfloat16_rn(w);
      if (vW) vW[((int64_t)f * k + r) * wp + t] = 0.f;   // a fresh row starts at rest
    }
    __syncthreads();
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
  int Fc = 0, mq = 0;   // fields per chunk; sample pitch of the per-field buffers (multiple of 32)
  __nv_bfloat16 *Xp = nullptr, *H16 = nullptr, *d16 = nullptr, *D16 = nullptr;   // [Fc][n|k][mp]
  float *U = nullptr;                                                           // [Fc][k][mp]
  float *da = nullptr, *db = nullptr;                                           // [Fc], [Fc][n]
  double *part[3] = {nullptr, nullptr, nullptr};                                // epilogue partials of GEMMs 1-3
  int npart[3] = {0, 0, 0};                                                     // per field
  float *dbp = nullptr;                                                         // [Fc][N tiles][n]
  float *rsqp = nullptr;                                                        // [Fc][N tiles][k]
  int nt2 = 0, nt4 = 0;
  gt::GemmArgs ga[5];
};

lcae_status gt_alloc(lcae_layer *L) {
  const Geo &g = L->geo;
  // the general path's per-field buffers use a sample pitch mq that is a multiple of 32 (one 32-column epilogue
  // chunk never leaves its row); the image and dX keep L->mp
  const int64_t k = g.k, n = g.n, mp = (g.m + 31) / 32 * 32, na = L->n_al;
  if (L->mp % 8 || L->n_al % 8) { set_error("gt path: pitches must be multiples of 8"); return LCAE_ERR_CONFIG; }
  const int bnm = gt::pick_bn(g.m), bnn = gt::pick_bn(g.n);
  const int mtk = cdiv(g.k, gt::BM), mtn = cdiv(g.n, gt::BM), ntm = cdiv(g.m, 64);   // ntm: the most N tiles
  const int64_t per_field = n * mp * (2 + 2) + k * mp * (2 + 4 + 2) + k * 4 * (cdiv(g.n, bnn) + 1) + n * 4 * (1 + ntm) + 4 +
                            8 * 4 * (2 * mtk + mtn) * ntm;
  GtScratch *s = new GtScratch();
  L->gt = s;
  s->Fc = (int)std::max<int64_t>(1, std::min<int64_t>(g.F, (2ll << 30) / per_field));
  if (const char *e = getenv("LCAE_DEV_GT_FC")) s->Fc = std::max(1, std::min(s->Fc, atoi(e)));   // dev: chunk size
  s->mq = (int)mp;
  const int64_t Fc = s->Fc;
  LCAE_CK(dmalloc(L, &s->Xp, Fc * n * mp * 2));
  LCAE_CK(dmalloc(L, &s->H16, Fc * k * mp * 2));
  LCAE_CK(dmalloc(L, &s->d16, Fc * n * mp * 2));
  LCAE_CK(dmalloc(L, &s->D16, Fc * k * mp * 2));
  LCAE_CK(dmalloc(L, &s->U, Fc * k * mp * 4));
  LCAE_CK(dmalloc(L, &s->da, Fc * 4));
  LCAE_CK(dmalloc(L, &s->db, Fc * n * 4));
  // N tile widths of the five GEMMs (fixed per layer: the epilogue partials are laid out by N tile)
  const int bn1 = gt::choose_bn(g.k, g.m, (int)Fc, true, L->sm_count, g.F),
            bn2 = gt::choose_bn(g.n, g.m, (int)Fc, true, L->sm_count, g.F);
  s->npart[0] = mtk * cdiv(g.m, bn1) * 4;   // GEMM 1 (U, pooling)
  s->npart[1] = mtn * cdiv(g.m, bn2) * 4;   // GEMM 2 (residual)
  s->npart[2] = mtk * cdiv(g.m, bn1) * 4;   // GEMM 3 (D, dalpha)
  for (int i = 0; i < 3; ++i) LCAE_CK(dmalloc(L, &s->part[i], Fc * s->npart[i] * sizeof(double)));
  s->nt2 = cdiv(g.m, bn2);
  LCAE_CK(dmalloc(L, &s->dbp, Fc * s->nt2 * n * 4));
  s->nt4 = cdiv(g.n, bnn);
  LCAE_CK(dmalloc(L, &s->rsqp, Fc * s->nt4 * k * 4));
  // bf16 shadow of W, [F][k][n_al] (pad columns zero)
  cudaFree(L->Wb);
  L->Wb = nullptr;
  LCAE_CK(dmalloc(L, &L->Wb, (size_t)g.F * k * na * 2));
  LCAE_CK(cudaMemset(L->Wb, 0, (size_t)g.F * k * na * 2));
  // operand maps: [batch][rows][cols] with the sample (or n) extent the true size, so ragged tails load as zeros
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
  // epilogue store maps (box 32 rows; fp32 32 columns, bf16 64 columns)
  CUtensorMap sU, sH, sd, sD, sdW, sWb;
  ok = ok && make_tmap_3d_f32(&sU, s->U, Fc, k, g.m, mp, k * mp, 32) &&
       make_tmap_3d_bf16(&sH, s->H16, Fc, k, g.m, mp, k * mp, 32) &&
       make_tmap_3d_bf16(&sd, s->d16, Fc, n, g.m, mp, n * mp, 32) &&
       make_tmap_3d_bf16(&sD, s->D16, Fc, k, g.m, mp, k * mp, 32) &&
       make_tmap_3d_f32(&sdW, L->W, g.F, k, n, L->wp, k * L->wp, 32) &&      // SGD: W~ master
       make_tmap_3d_bf16(&sWb, L->Wb, g.F, k, n, na, k * na, 32);            // SGD: bf16 shadow
  if (!ok) { set_error("gt path: cuTensorMapEncodeTiled failed"); return LCAE_ERR_CUDA; }
  auto args = [&](const CUtensorMap &A, const CUtensorMap &B, int M, int N, int K, float *C, int64_t cbs, int64_t crs) {
    gt::GemmArgs a{};
    a.tmA[0] = A; a.tmB[0] = B; a.nseg = 1; a.M = M; a.N = N; a.K = K; a.C = C; a.cbs = cbs; a.crs = crs;
    a.g = g.g; a.gr = g.gr; a.gc = g.gc; a.lam = L->cfg.lambda_; a.eps = L->cfg.eps;
    a.alpha = L->alpha; a.bvec = L->b; a.sigma = L->sigma; a.flags = L->flags_dev;
    a.lr = L->cfg.lr; a.mu = L->cfg.momentum;
    return a;
  };
  // 1: U = W X_f; epilogue h = alpha U -> bf16, pooling, p, sum s
  s->ga[0] = args(mWk, mXmn, g.k, g.m, g.n, s->U, k * mp, mp);
  s->ga[0].O16 = s->H16; s->ga[0].part = s->part[0]; s->ga[0].tmC = sU; s->ga[0].tmO = sH;
  // 2: r = W^T h; epilogue e = r + b - x, delta = 2e -> bf16, sum e^2, db partials
  s->ga[1] = args(mWmn, mHmn, g.n, g.m, g.k, nullptr, n * mp, mp);
  s->ga[1].I16 = s->Xp; s->ga[1].O16 = s->d16; s->ga[1].part = s->part[1]; s->ga[1].dbp = s->dbp; s->ga[1].tmO = sd;
  // 3: G = W delta; epilogue D = G + lambda h / s, alpha D -> bf16, sum D.U
  s->ga[2] = args(mWk, mdmn, g.k, g.m, g.n, nullptr, k * mp, mp);
  s->ga[2].U = s->U; s->ga[2].O16 = s->D16; s->ga[2].part = s->part[2]; s->ga[2].tmO = sD;
  // 4: sigma dW = (sigma h) delta^T + (sigma alpha D) X_f^T (two K segments into one accumulator); epilogue: projected
  //    SGD of W~ (master + shadow), ||W~'||^2 row partials
  s->ga[3] = args(mHk, mdk, g.k, g.n, g.m, nullptr, 0, 0);
  s->ga[3].tmA[1] = mDk; s->ga[3].tmB[1] = mXk; s->ga[3].nseg = 2; s->ga[3].tmC = sdW; s->ga[3].tmO = sWb;
  s->ga[3].W = L->W; s->ga[3].wp = L->wp; s->ga[3].dbp = s->rsqp; s->ga[3].vW = L->vW;
  s->ga[3].gW = L->cfg.keep_grads ? L->gW : nullptr;
  // 5: dXp^T = (sigma alpha D)^T W~ - delta^T (rows = samples, columns = patch rows), reduce-added into dX by TMA
  s->ga[4] = args(mDmn, mWmn, g.m, g.n, g.k, nullptr, 0, 0);
  if (!make_tmap_3d_bf16_32x32(&s->ga[4].tmO, s->d16, Fc, n, g.m, mp, n * mp)) {
    set_error("gt path: cuTensorMapEncodeTiled failed (delta)");
    return LCAE_ERR_CUDA;
  }
  s->ga[4].RW = g.RW; s->ga[4].s = g.s; s->ga[4].Cc = g.C; s->ga[4].WC = (int64_t)g.W * g.C;
  for (int lg = 0; lg < 6; ++lg)
    if (!make_tmap_2d_f32(&s->ga[4].tmR[lg], L->dxt, (uint64_t)g.H * g.W * g.C, (uint64_t)g.m, (uint64_t)L->mp,
                          1u << lg, 32)) {
      set_error("gt path: cuTensorMapEncodeTiled failed (dX)");
      return LCAE_ERR_CUDA;
    }
  s->ga[0].bn = s->ga[2].bn = bn1;
  s->ga[1].bn = bn2;
  s->ga[4].bn = gt::choose_bn(g.m, g.n, (int)Fc, true, L->sm_count, g.F);
  s->ga[3].bn = bnn;   // K-major B: its maps are built for this width
  (void)bnm;
  return LCAE_OK;
}

void gt_free(lcae_layer *L) {
  GtScratch *s = L->gt;
  if (!s) return;
  for (void *p : {(void *)s->Xp, (void *)s->H16, (void *)s->d16, (void *)s->D16, (void *)s->U,
                  (void *)s->rsqp, (void *)s->da, (void *)s->db, (void *)s->part[0], (void *)s->part[1],
                  (void *)s->part[2], (void *)s->dbp})
    cudaFree(p);
  delete s;
  L->gt = nullptr;
}

lcae_status gt_step(lcae_layer *L, bool update, bool want_pooled, bool encode_only) {
  using namespace gt;
  const Geo &g = L->geo;
  GtScratch &s = *L->gt;
  const int mp = L->mp;
  lcae_status st;
#define TRY(x) do { if ((st = (x)) != LCAE_OK) return st; } while (0)
  if (update) LCAE_CK(cudaMemsetAsync(L->dxt, 0, (size_t)g.H * g.W * g.C * mp * 4, L->st));
  s.ga[0].pooled = want_pooled ? L->pooled : nullptr;
  for (int f0 = 0; f0 < g.F; f0 += s.Fc) {
    const int Fc = std::min(s.Fc, g.F - f0);
    for (auto &a : s.ga) { a.batch = Fc; a.f0 = f0; }
    s.ga[0].bA[0] = s.ga[1].bA[0] = s.ga[2].bA[0] = s.ga[4].bB[0] = f0;   // W maps span all fields
    const int ysplit = std::max(1, std::min(64, 4 * L->sm_count / Fc));   // blocks per field (few-field layers)
    gt_gather<<<dim3(Fc, ysplit), 256, 0, L->st>>>(g, f0, mp, s.mq, L->xt16, s.Xp);
    LCAE_CK_LAUNCH(L);
    TRY(want_pooled ? (gemm<false, true, EPI_POOLP>(L, s.ga[0])) : (gemm<false, true, EPI_POOL>(L, s.ga[0])));
    if (!encode_only) TRY((gemm<true, true, EPI_RESID>(L, s.ga[1])));
    if (update) TRY((gemm<false, true, EPI_DCODE>(L, s.ga[2])));
    gt_parts<<<dim3(Fc, ysplit), 256, 0, L->st>>>(f0, g.n, L->cfg.lambda_, s.part[0], s.npart[0],
                                    encode_only ? nullptr : s.part[1], s.npart[1], update ? s.part[2] : nullptr,
                                    s.npart[2], s.dbp, s.nt2, L->loss_part, s.da, s.db, encode_only ? 1 : 0);
    LCAE_CK_LAUNCH(L);
    if (!update) continue;
    TRY((gemm<true, true, EPI_DXRED>(L, s.ga[4])));   // dX first: it reads the pre-update shadow
    s.ga[3].sb = f0;
    s.ga[4].sb = 0;
    if (L->vW || L->cfg.keep_grads) TRY((gemm<false, false, EPI_SGDF>(L, s.ga[3])));
    else TRY((gemm<false, false, EPI_SGD>(L, s.ga[3])));
    if (L->cfg.keep_grads) {
      gt_copy_ab<<<256, 256, 0, L->st>>>(f0, Fc, g.n, s.da, s.db, L->galpha, L->gb);
      LCAE_CK_LAUNCH(L);
    }
    gt_finalize<<<dim3(Fc, cdiv(g.k, 128)), 128, 0, L->st>>>(g, f0, s.nt4, s.rsqp, L->sigma, L->W, L->Wb, L->wp, L->n_al, L->vW,
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
