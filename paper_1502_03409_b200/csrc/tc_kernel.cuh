// tc_kernel.cuh — the fused bf16 tcgen05 training-step kernel of the locally-connected RICA layer (sm_100a).
//
// One persistent kernel does the whole per-field chain of PAPER.md:88: a cluster of
// CB CTAs (CB = ceil(m/128); CTA c owns samples [128c, 128c+128)) walks the fields; for field f every CTA
// streams bf16 W~_f tiles (TMA, 128B swizzle, 4-stage ring) and its X_f patch rows (cp.async gather from the
// batch-innermost HWCN image) in three passes over n-tiles of 64:
//
//   pass 0  U^T   = X^T W~^T                   (M = samples, N = k, K = n)      TMEM [384,512)
//           E0: u = sigma.U~, h = alpha u, s_G = sqrt(eps + sum_G h^2), J_s, p; H' = bf16(sigma.h) -> smem
//   pass 1  R^T_j - X_j^T = H'^T W~_j + X_j^T (-I)   (M = samples, N = 64)       TMEM [0,256) (4 buffers)
//           E1: e = (R - x) + b, J_r, delta = 2e -> smem (bf16) and its image to a per-CTA global scratch,
//               db partial (butterfly column sums)
//           G^T  += delta_j^T W~_j^T  (lag 1)  (M = samples, N = k, K = 64)     TMEM [256,384)
//           E1b: D = sigma.G~ + lambda h/s, dalpha, D' = bf16(sigma alpha D) -> smem
//   pass 2  delta_j reloaded (bulk copy, L2), dx^T_j = D'^T W~_j + delta_j^T (-I) -> red.global.v4 into dX
//           dW_j = H' delta_j^T + D' X_j^T     (M = k, N = 64, K = 2 x samples) TMEM 3 x [dX|dW] in [0,384)
//           E2: sum the batch slices of dW_j over the cluster (DSMEM), projected-SGD of W~ (fp32 master +
//               bf16 shadow, 16-byte vectors), row sums of squares for the new row scale sigma.
//
// The "- x" of the residual is accumulated by the tensor core (X_j^T times a constant -I tile; exact in
// bf16/fp32), so the epilogue never touches x.
// W = sigma (.) W~ with a per-row scale sigma ("lazy projection"): the unit-norm projection of
// PAPER.md:89 is applied by the finalize kernel as sigma' = 1/||W~'_row||, so the update never re-reads W.
//
// U lives outside the pass-2 columns, so the next field's pass 0 overlaps this field's last pass-2 epilogue tiles.
// Warp roles: 0 = W TMA producer, 1 = MMA issuer (warp-uniform, elected lane issues), 2-9 = epilogue (TMEM lane
// quarter = warp % 4, column half = (warp - 2) / 4), 10 = X TMA producer. X tiles of pass 0 borrow the D', delta,
// pass-2 X and H' buffers (all idle during pass 0) as an 8-slot ring, those of pass 1 the D' buffer, those of
// pass 2 a dedicated 2-slot ring.
#pragma once
#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"

namespace lcae {
namespace tc {

constexpr int KP = 128;        // filters padded to one TMEM lane block
constexpr int NT = 64;         // n-tile
constexpr int MC = 128;        // samples per CTA
constexpr int NW = 4;          // W ring stages (pass 1 holds W~_j from R_j until G_j: 4 stages give the
                               // ~2 us L2 -> smem TMA latency a tile of slack)
constexpr int NX = 2;          // pass-2 X ring stages
constexpr int NP0 = 8;         // pass-0 X ring slots (D'[0..1], delta[0..1], pass-2 X ring [0..1], H'[0..1])
constexpr int NRB = 4;         // pass-1 R buffers
constexpr int NB2 = 3;         // pass-2 TMEM buffers [dX | dW] (128 columns each)
constexpr int GLAG = 1;        // G_j issued after R_{j+GLAG}
constexpr int NEPI = 8;        // epilogue warps
constexpr int XWARP = 2 + NEPI;
constexpr int NTHREADS = 32 * (XWARP + 1);
constexpr int MAX_NPAD = 4096;   // n = rf_h rf_w C <= 4096 (b_f fits the 16 KB of staging slices)

// TMA piece words (host table): window offset (20 bits) | first row in the tile / chunk (7 bits) << 20 |
// log2 box height (3 bits) << 27; 0xFFFFFFFF ends a list (row 127 never occurs)
__host__ __device__ constexpr uint32_t piece_word(uint32_t off, uint32_t row, uint32_t lg) {
  return off | (row << 20) | (lg << 27);
}
__host__ __device__ inline uint32_t piece_off(uint32_t w) { return w & 0xFFFFFu; }
__host__ __device__ inline uint32_t piece_row(uint32_t w) { return (w >> 20) & 0x7Fu; }
__host__ __device__ inline uint32_t piece_lg(uint32_t w) { return (w >> 27) & 0x7u; }

constexpr int NXMAP = 7;       // X tensor maps with box heights 1, 2, 4, ..., 64 rows
constexpr int XPMAX = 64;      // max TMA pieces per 64-row X tile
constexpr int NDMAP = 5;       // dX reduce tensor maps with box heights 1, 2, 4, 8, 16 rows (x 32 samples)
constexpr int DXPMAX = 16;     // max TMA pieces per 16-column dX chunk

struct Params {
  CUtensorMap tmW;   // W~ bf16 [F*KP][n_al], box (64, 128)
  CUtensorMap tmX[NXMAP];   // X HWCN bf16 viewed as [H*W*C rows][mp], box (64 samples, 2^i rows)
  const uint32_t *xpieces;  // [T][XPMAX] piece words (piece_word); 0xFFFFFFFF ends
  CUtensorMap tmD[NDMAP];   // dX HWCN f32 viewed as [H*W*C rows][mp], box (32 samples, 2^i rows), no swizzle
  const uint32_t *dxpieces; // [T][4][DXPMAX]: the pieces of 16-column chunk q of tile j, same encoding
  const int *flist;         // nullable: the launch walks fields flist[0..nfl) (model-parallel interior / boundary
  int nfl;                  // split); NULL: fields 0..F-1
  Geo g;
  int T, mp, CB, n_al, wp, mode, want_pooled, keep_grads;
  int dbg;   // dev-only (LCAE_DEBUG_FLAGS): bit 0 skips the dX reductions, bit 1 the W~/shadow stores,
             // bit 2 all epilogue arithmetic (hand-offs kept; for pipeline-ceiling measurements only)
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
  float *rowsq_part;   // [F][CB][2][KP]
  float *dbscr;        // [grid][4][MAX_NPAD]: per-lane-quarter db partials of the current field
  uint8_t *dscr;       // [grid][T][16 KB]: pass-1 delta tiles (their swizzled smem image), reloaded in pass 2
  float *gW;
  const int *flags;   // sticky error flags (non-finite input / loss): a training step does nothing while set
  unsigned long long *trace;   // nullable: per-role wait cycles summed over CTAs
};

struct __align__(1024) Smem {
  uint8_t Wr[NW][16384];
  uint8_t Xr[NX][16384];
  uint8_t H[32768];
  uint8_t D[32768];          // pass 0: X slots 0,1; pass 1: X ring
  uint8_t Dl[2][16384];      // pass 0: X slots 2,3
  uint8_t negI[2048];        // -I_16 (16 x 16 bf16, SW128 rows): the -x / -delta MMAs run as 4 N = 16 blocks
  uint32_t recv[2][128][8];  // peer's dW partial for this CTA's owned 16-column chunks, [half][row][16 bf16] (R25)
  float stg[NEPI][32][16];   // per-warp 2 KB staging: the own dW chunk's transpose (16-byte chunks swizzled), then
                             // the dX rounds ([16 patch rows][32 samples], the TMA reduce-add source); during
                             // E0 / E1 of a training step the first 4 KB hold b_f (all warps), in forward / encode
                             // the pooled-output staging
  float sig[KP];
  float isig[KP];            // 1 / sig
  double redd[NEPI][2];
  float redf[NEPI];
  uint64_t wfull[NW], wempty[NW], xfull[NX], xempty[NX], p0full[NP0], p0empty[NP0], p1full[4], p1empty[4];
  uint64_t p0_ok, u_full, h_ready, g_full, d_ready, d_stored;
  uint64_t uf[4], ue[4];     // encode-only mode: 4 U buffers in TMEM (full / free)
  uint64_t r_full[NRB], r_empty[NRB], dl_full[2], dl_empty[2];
  uint64_t p2_full[NB2], p2_empty[NB2], d2full[2], d2empty[2];
  uint64_t recv_full[NEPI], peer_free[NEPI];   // per epilogue warp: the dW exchange couples warp w of the two
                                               // CTAs only (not all 16 warps of the pair)
  uint32_t tmem_base;
  unsigned long long tr[64];   // optional wait-cycle / section trace (lcae_dev_trace); [48+w]/[56+w]: per epilogue warp
};


static_assert(offsetof(Smem, stg) % 16 == 0, "float4 reads of b_f");
static_assert(sizeof(Smem::stg) >= MAX_NPAD * sizeof(float), "b_f fits the staging slices");

// pass 1's X ring: the D' buffer (2 slots) and, in a training step, the pass-2 X ring too (idle from the end of
// pass 0 to the start of pass 2): 4 slots, so the X tiles arrive ahead of the R MMAs despite ~2 us of L2 -> smem
// TMA latency (measured with the traced variant's timeline)
__device__ __forceinline__ uint8_t *p1slot(Smem &S, uint32_t i) { return i < 2 ? S.D + i * 16384 : S.Xr[i - 2]; }

// pass 0 borrows every operand buffer the previous field's pass 2 is done with (all free at p0_ok)
__device__ __forceinline__ uint8_t *p0slot(Smem &S, int i) {
  return i < 2 ? S.D + i * 16384 : i < 4 ? S.Dl[i - 2] : i < 6 ? S.Xr[i - 4] : S.H + (i - 6) * 16384;
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

__device__ __forceinline__ void red_v4(float *p, float a, float b, float c, float d) {
  // no "memory" clobber: the reductions need no ordering against the kernel's other memory operations, and a
  // clobber would pin every following shared-memory load behind them
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d));
}

// e = (R - x) + b over this warp's 32 columns of a tile for this thread's sample; rv <- delta = 2e (masked);
// returns sum delta^2 = 4 sum e^2. b2 holds 2 b (the training step keeps 2 b_f in shared memory, b2_ready) or b:
// delta = fma(2, R - x, 2b) rounds exactly as 2 ((R - x) + b) (scaling by 2 is exact), one FFMA per element.
__device__ __forceinline__ float residual32(float (&rv)[32], int c0, int n, const float *b2, bool svalid, bool b16,
                                            bool b2_ready) {
  float jr = 0.f;
  const float4 *b4 = reinterpret_cast<const float4 *>(b2 + c0);   // c0 % 32 == 0: 16-byte aligned broadcasts
  const float bs = b2_ready ? 1.f : 2.f;
  if (svalid && c0 + 32 <= n && b16) {   // full run (all but the ragged last tile): no masking
    float ja[4] = {0.f, 0.f, 0.f, 0.f};   // four accumulators: a chain of 8 FFMAs instead of 32
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 bv = b4[q];
      const float bb[4] = {bv.x * bs, bv.y * bs, bv.z * bs, bv.w * bs};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float d = fmaf(2.f, rv[4 * q + t], bb[t]);
        ja[t] = fmaf(d, d, ja[t]);
        rv[4 * q + t] = d;
      }
    }
    return (ja[0] + ja[1]) + (ja[2] + ja[3]);
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const int nn = c0 + c;
    float d = fmaf(2.f, rv[c], nn < n ? b2[nn] * bs : 0.f);
    d = (svalid && nn < n) ? d : 0.f;
    jr = fmaf(d, d, jr);
    rv[c] = d;
  }
  return jr;
}

// FL bit 0: wait / section tracing compiled in (lcae_dev_trace); bit 1: the full epilogue (momentum velocity,
// kept gradients, debug flags); bit 2: generic mode (forward / encode). The lean variant (FL = 0) is the common
// training step.
template <int GP, int CBT, int FL>
__global__ void __launch_bounds__(NTHREADS, 1) step_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the SW128 tiles by pointer arithmetic on the shared array (keeps the shared
  // address space visible to the compiler: LDS/STS, not generic LD/ST)
  const uint32_t pad = (1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u;
  Smem &S = *reinterpret_cast<Smem *>(smem_raw + pad);
  const Geo &g = P.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int CB = CBT;
  const uint32_t crank = CB > 1 ? ptx::cluster_ctarank() : 0;
  const int cid = blockIdx.x / CB, ncl = gridDim.x / CB;
  const int s0 = (int)crank * MC;   // first sample of this CTA
  const int T = P.T, n = g.n, k = g.k, m = g.m;
  // FL bit 2: generic variant (forward / encode / step chosen at run time, pooled output); otherwise the
  // kernel is the training step and the forward-only paths are compiled out
  constexpr bool TR = (FL & 1) != 0, FULL = (FL & 2) != 0, GEN = (FL & 4) != 0;
  const bool step = GEN ? P.mode == 1 : true;
  const bool enc = GEN && P.mode == 2;   // encode-only inference (pass 0 + pooling)
  const bool want_pooled = GEN && P.want_pooled;
  // a flagged error (this step's input had a non-finite value, or an earlier loss was non-finite) freezes the
  // parameters: every CTA reads the same flags (written by earlier kernels), so all return together
  if (step && (P.flags[0] | P.flags[1])) return;
  const int nfl = P.flist ? P.nfl : P.g.F;
  auto fid = [&](int i) {
    const int f_ = P.flist ? __ldg(P.flist + i) : i;
    LCAE_DCHECK(f_ >= 0 && f_ < P.g.F);
    return f_;
  };
  const uint32_t np1 = step ? 4u : 2u;   // pass-1 X ring slots (p1slot)
  const int64_t prow = (int64_t)P.g.H * P.g.W * P.g.C;   // pixel-feature rows of the HWCN image (checked build)
  (void)prow;
  // trace: lane 0 of the producers / MMA warp and of epilogue warp 2 record their barrier-wait cycles
  const bool trec = TR && P.trace != nullptr && lane == 0 && (warp <= 2 || warp == XWARP);
  const long long t_start = clock64();
// the MMA issuer polls (LCAE_MMA_WAIT_POLL) or suspends (default) on its barriers
#ifdef LCAE_MMA_WAIT_POLL
#define MMA_WAIT(...) ptx::mbar_wait_poll(__VA_ARGS__)
#else
#define MMA_WAIT(...) ptx::mbar_wait(__VA_ARGS__)
#endif
#define TWAIT(IDX, ...)                                                                          \
  do {                                                                                           \
    if (trec) {                                                                                  \
      const long long t0_ = clock64();                                                           \
      __VA_ARGS__;                                                                               \
      atomicAdd(&S.tr[IDX], (unsigned long long)(clock64() - t0_));                              \
    } else {                                                                                     \
      __VA_ARGS__;                                                                               \
    }                                                                                            \
  } while (0)

  // timeline (traced variant only): clock64 of pipeline events of CTA 0's third field, into P.trace[64 + id]
#define TLOG(ID, NF)                                                                             \
  do {                                                                                           \
    if (TR && P.trace && blockIdx.x == 0 && (NF) == 2 && lane == 0 && P.T <= 16)                \
      P.trace[64 + (ID)] = (unsigned long long)clock64();                                        \
  } while (0)
  // ---- one-time setup
  if (threadIdx.x < 64) S.tr[threadIdx.x] = 0ull;
  long long tmark = 0;
#define TMARK(IDX)                                                                               \
  do {                                                                                           \
    if (trec) {                                                                                  \
      const long long t_ = clock64();                                                            \
      if ((IDX) >= 0) atomicAdd(&S.tr[(IDX) < 0 ? 0 : (IDX)], (unsigned long long)(t_ - tmark)); \
      tmark = t_;                                                                                \
    }                                                                                            \
  } while (0)
  {  // X slots start zeroed: rows past n of the last tile are never written (their products are masked,
     // but must stay finite)
    uint4 *z = reinterpret_cast<uint4 *>(S.Xr[0]);
    for (int t = threadIdx.x; t < (int)(sizeof(S.Xr) + sizeof(S.H) + sizeof(S.D) + sizeof(S.Dl)) / 16; t += NTHREADS)
      z[t] = make_uint4(0, 0, 0, 0);
  }
  for (int t = threadIdx.x; t < 16 * 64; t += NTHREADS) {   // rows 0..15 of a SW128 K-major tile; K 0..15 used
    const int r = t >> 6, c = t & 63;
    *reinterpret_cast<__nv_bfloat16 *>(S.negI + ptx::sw128_off(r, c)) = __float2bfloat16_rn(r == c ? -1.f : 0.f);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < NW; ++i) { ptx::mbar_init(&S.wfull[i], 1); ptx::mbar_init(&S.wempty[i], 1); }
    for (int i = 0; i < NX; ++i) { ptx::mbar_init(&S.xfull[i], 1); ptx::mbar_init(&S.xempty[i], 1); }
    for (int i = 0; i < NP0; ++i) { ptx::mbar_init(&S.p0full[i], 1); ptx::mbar_init(&S.p0empty[i], 1); }
    for (int i = 0; i < 4; ++i) { ptx::mbar_init(&S.p1full[i], 1); ptx::mbar_init(&S.p1empty[i], 1); }
    ptx::mbar_init(&S.p0_ok, 1);
    for (int i = 0; i < NB2; ++i) { ptx::mbar_init(&S.p2_full[i], 1); ptx::mbar_init(&S.p2_empty[i], NEPI); }
    ptx::mbar_init(&S.u_full, 1);
    for (int i = 0; i < 4; ++i) { ptx::mbar_init(&S.uf[i], 1); ptx::mbar_init(&S.ue[i], NEPI); }
    ptx::mbar_init(&S.h_ready, NEPI);
    ptx::mbar_init(&S.g_full, 1);
    ptx::mbar_init(&S.d_ready, NEPI);
    ptx::mbar_init(&S.d_stored, 1);
    for (int i = 0; i < NRB; ++i) { ptx::mbar_init(&S.r_full[i], 1); ptx::mbar_init(&S.r_empty[i], NEPI); }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&S.dl_full[i], NEPI);
      ptx::mbar_init(&S.dl_empty[i], 2);   // G MMA commit + delta store-out (warp 0 lane 1)
      ptx::mbar_init(&S.d2full[i], 1);
      ptx::mbar_init(&S.d2empty[i], 1);
    }
    for (int i = 0; i < NEPI; ++i) {
      ptx::mbar_init(&S.recv_full[i], 1);   // armed per tile with expect_tx; completed by the peer's st.async bytes
      ptx::mbar_init(&S.peer_free[i], 1);   // the peer's warp i has read its receive slice
    }
    ptx::fence_mbar_init();
  }
  ptx::fence_proxy_async_smem();   // -I tile is read by the tensor core
  if (warp == 1) ptx::tmem_alloc<512>(&S.tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  if (CB > 1) ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tb = S.tmem_base;

  if (warp == 0) {
    // =================================================================== W producer (TMA)
    if (lane == 0) {
      ptx::tma_prefetch(&P.tmW);
      const uint64_t pol = ptx::policy_evict_first();   // W is streamed once per pass: keep X / dX in L2
      uint32_t q = 0;
      const int npass = step ? 3 : (enc ? 1 : 2);
      for (int fi = cid; fi < nfl; fi += ncl) {
        const int f = fid(fi);
        for (int pass = 0; pass < npass; ++pass)
          for (int j = 0; j < T; ++j, ++q) {
            const int s = q % NW;
            TWAIT(27, ptx::mbar_wait(&S.wempty[s], ((q / NW) & 1) ^ 1));
            ptx::mbar_arrive_expect_tx(&S.wfull[s], 16384);
            if (pass == npass - 1)   // last read of W~_f this step: evict first; earlier passes keep it in L2
              ptx::tma_load_2d_hint(S.Wr[s], &P.tmW, &S.wfull[s], j * NT, f * KP, pol);
            else
              ptx::tma_load_2d(S.Wr[s], &P.tmW, &S.wfull[s], j * NT, f * KP);
          }
      }
    } else if (lane == 1 && step) {
      // =================================================================== delta store-out (bulk S2G)
      // every pass-1 delta tile goes to this CTA's global scratch as its swizzled smem image; pass 2 reloads it
      uint32_t ud = 0, nf = 0;
      for (int fi = cid; fi < nfl; fi += ncl, ++nf) {
        uint8_t *dst = P.dscr + (size_t)blockIdx.x * T * 16384;
        for (int j = 0; j < T; ++j, ++ud) {
          const uint32_t db_ = ud & 1;
          ptx::mbar_wait(&S.dl_full[db_], (ud >> 1) & 1);
          ptx::bulk_s2g(dst + (size_t)j * 16384, S.Dl[db_], 16384);
          ptx::bulk_commit();
          ptx::bulk_wait_read0();   // smem read done: the epilogue may refill the slot
          ptx::mbar_arrive(&S.dl_empty[db_]);
        }
        ptx::bulk_wait0();                 // all of the field's delta images written
        ptx::fence_proxy_async_global();
        ptx::mbar_arrive(&S.d_stored);
      }
    }
    __syncwarp();
  } else if (warp == XWARP) {
    // =================================================================== X producer (cp.async gather)
    uint32_t q0 = 0, q1 = 0, qx = 0, nf = 0, qd2 = 0;
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < NXMAP; ++i) ptx::tma_prefetch(&P.tmX[i]);
    }
    for (int fi = cid; fi < nfl; fi += ncl, ++nf) {
      const int f = fid(fi);
      const int fr = f / g.gc, fc = f - fr * g.gc;
      const int pixbase = (fr * g.s * g.W + fc * g.s) * g.C;
      // X_j = runs of consecutive image rows (one per receptive-field row): a few TMA boxes per 64-sample half;
      // the 128B swizzle follows the absolute smem address, so boxes may land at any row of the tile.
      // the whole warp reads a tile's piece table at once (one load latency, not one per piece), one tile ahead
      // of its TMA issue, and every lane issues the boxes of its own pieces
      static_assert(XPMAX == 64, "two piece words per lane");
      auto piece_x = [&](int j, uint32_t &a0, uint32_t &a1) {
        const uint32_t *pc = P.xpieces + j * XPMAX;
        a0 = __ldg(pc + lane);
        a1 = __ldg(pc + 32 + lane);
      };
      auto load_tile = [&](uint8_t *dst_tile, uint64_t *bar, int j, uint32_t w0, uint32_t w1) {
        if (lane == 0) ptx::mbar_arrive_expect_tx(bar, (uint32_t)min(NT, n - j * NT) * 128u * 2u);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint32_t w = e ? w1 : w0;
          if (w != 0xFFFFFFFFu) {
            const int offp = (int)piece_off(w), dr = (int)piece_row(w), lg = (int)piece_lg(w);
            LCAE_DCHECK(lg < NXMAP && dr + (1 << lg) <= NT && pixbase + offp + (1 << lg) <= prow);
#pragma unroll
            for (int h = 0; h < 2; ++h)
              ptx::tma_load_2d(dst_tile + h * 8192 + dr * 128, &P.tmX[lg], bar, s0 + 64 * h, pixbase + offp);
          }
        }
        __syncwarp();
      };
      // pass 0 ring borrows the D'/delta/X/H' buffers: wait until the previous field is done with them
      if (step) TWAIT(28, ptx::mbar_wait(&S.p0_ok, (nf & 1) ^ 1));
      uint32_t xa0, xa1, xb0 = 0, xb1 = 0;
      piece_x(0, xa0, xa1);
      for (int j = 0; j < T; ++j, ++q0) {
        const int s = q0 % NP0;
        if (j + 1 < T) piece_x(j + 1, xb0, xb1);
        TWAIT(29, ptx::mbar_wait(&S.p0empty[s], ((q0 / NP0) & 1) ^ 1));
        load_tile(p0slot(S, s), &S.p0full[s], j, xa0, xa1);
        xa0 = xb0; xa1 = xb1;
      }
      if (enc) continue;   // encode-only: the pass-0 ring's own barriers order the next field's loads
      // pass 1 ring lives in the D' buffer once the encode MMAs are done
      TWAIT(30, ptx::mbar_wait(&S.u_full, nf & 1));
      piece_x(0, xa0, xa1);
      for (int j = 0; j < T; ++j, ++q1) {
        const uint32_t s = q1 % np1;
        if (j + 1 < T) piece_x(j + 1, xb0, xb1);
        TWAIT(30, ptx::mbar_wait(&S.p1empty[s], ((q1 / np1) & 1) ^ 1));
        load_tile(p1slot(S, s), &S.p1full[s], j, xa0, xa1);
        xa0 = xb0; xa1 = xb1;
      }
      if (!step) {   // forward: the next field's pass 0 reuses D'; wait until both slots were consumed
        for (uint32_t qq = q1 - std::min<uint32_t>(q1, np1); qq < q1; ++qq)
          ptx::mbar_wait(&S.p1empty[qq % np1], (qq / np1) & 1);
        continue;
      }
      // pass 2: delta_j (the pass-1 images, once all are stored and the G MMAs are done with the ring) and X_j
      TWAIT(28, ptx::mbar_wait(&S.d_stored, nf & 1));
      TWAIT(28, ptx::mbar_wait(&S.g_full, nf & 1));
      ptx::fence_proxy_async_global();
      const uint8_t *dsrc = P.dscr + (size_t)blockIdx.x * T * 16384;
      // a reloaded delta tile is dead once its MMAs completed (d2empty): its scratch lines are discarded from
      // L2 so they are never written back to HBM (the next field's store-out rewrites them much later)
      auto discard_tile = [&](int jj) {
#pragma unroll
        for (int l4 = 0; l4 < 4; ++l4) ptx::discard_l2(dsrc + (size_t)jj * 16384 + (size_t)(l4 * 32 + lane) * 128);
        ptx::fence_proxy_async_global();   // ordered before the (async-proxy) bulk stores that rewrite the lines
      };
      piece_x(0, xa0, xa1);
      for (int j = 0; j < T; ++j, ++qx, ++qd2) {
        const int sd = qd2 & 1;
        if (j + 1 < T) piece_x(j + 1, xb0, xb1);
        TWAIT(31, ptx::mbar_wait(&S.d2empty[sd], ((qd2 >> 1) & 1) ^ 1));
        if (j >= 2) discard_tile(j - 2);
        if (lane == 0) {
          ptx::mbar_arrive_expect_tx(&S.d2full[sd], 16384);
          ptx::bulk_g2s(S.Dl[sd], dsrc + (size_t)j * 16384, 16384, &S.d2full[sd]);
        }
        __syncwarp();
        const int s = qx % NX;
        TWAIT(31, ptx::mbar_wait(&S.xempty[s], ((qx / NX) & 1) ^ 1));
        load_tile(S.Xr[s], &S.xfull[s], j, xa0, xa1);
        xa0 = xb0; xa1 = xb1;
      }
      for (int j = std::max(0, T - 2); j < T; ++j) {   // the field's last two reloads: wait for their MMAs
        const uint32_t qq = qd2 - T + j;
        ptx::mbar_wait(&S.d2empty[qq & 1], (qq >> 1) & 1);
        discard_tile(j);
      }
    }
  } else if (warp == 1) {
    // =================================================================== MMA issuer
    // The warp walks the schedule (waits are warp-wide); one elected lane issues each GROUP of MMAs and its
    // commits. Descriptors are built once per operand tile and advanced by adding the byte offset >> 4 to the
    // start-address field (smem addresses < 2^18, so the 14-bit field never carries): a handful of instructions
    // per MMA. (The MMA warp shares an SM sub-partition with two epilogue warps: its instruction count is
    // their issue time.)
    {
      const uint32_t id_enc = ptx::idesc_bf16(128, KP, true, false);
      const uint32_t id_dec = ptx::idesc_bf16(128, NT, false, true);
      const uint32_t id_nx = ptx::idesc_bf16(128, 16, true, false);   // X^T (-I_16), per 16-column block
      const uint32_t id_g = ptx::idesc_bf16(128, KP, false, false);
      const uint32_t id_dw1 = ptx::idesc_bf16(128, NT, true, true);
      const uint32_t id_dw2 = ptx::idesc_bf16(128, NT, true, false);
      const uint32_t id_nd = ptx::idesc_bf16(128, 16, false, false);   // delta^T (-I_16), per 16-column block
      const uint32_t sH = ptx::smem_u32(S.H), sD = ptx::smem_u32(S.D), sNI = ptx::smem_u32(S.negI);
      // fixed-buffer descriptors
      const uint64_t dH_k = ptx::sdesc_sw128(sH, 16, 1024);       // H' K-major (A of the decode)
      const uint64_t dD_k = ptx::sdesc_sw128(sD, 16, 1024);       // D' K-major (A of dx)
      const uint64_t dH_mn = ptx::sdesc_sw128(sH, 16384, 1024);   // H' as [filters x samples] (A of dW)
      const uint64_t dD_mn = ptx::sdesc_sw128(sD, 16384, 1024);   // D' likewise
      const uint64_t dNI = ptx::sdesc_sw128(sNI, 16, 1024);       // -I (K-major B)
      auto adv = [](uint64_t d, uint32_t bytes) { return d + (uint64_t)(bytes >> 4); };
      uint32_t qw = 0, q0 = 0, q1 = 0, qx = 0, nf = 0, ur = 0, ud = 0, u2 = 0, qd2 = 0;
      auto wst = [&](uint32_t qq) { return ptx::smem_u32(S.Wr[qq % NW]); };
      auto wait_w = [&](uint32_t qq) {
        TWAIT(0, MMA_WAIT(&S.wfull[qq % NW], (qq / NW) & 1));
        ptx::tc_fence_after();
      };
      // D = A^T W~_j: A = H' or D' (K-major [128][128]), W~_j MN-major (elected lane only)
      auto mma_aw = [&](uint32_t dcol, uint64_t a_desc, uint32_t w_base) {
        const uint64_t bd = ptx::sdesc_sw128(w_base, 16384, 1024);
#pragma unroll
        for (int kk = 0; kk < KP / 16; ++kk)
          ptx::umma_bf16(tb + dcol, adv(a_desc, (kk >> 2) * 16384 + (kk & 3) * 32), adv(bd, kk * 2048), id_dec, kk > 0);
      };
      // D += X_j^T (-I): subtracts the patch values exactly (X_j MN-major A, -I K-major B): columns 16kk..+16 of D
      // take K rows 16kk..+16 of X_j^T times -I_16 (elected lane only)
      auto mma_negx = [&](uint32_t dcol, uint32_t x_base) {
        const uint64_t ad = ptx::sdesc_sw128(x_base, 8192, 1024);
#pragma unroll
        for (int kk = 0; kk < NT / 16; ++kk) ptx::umma_bf16(tb + dcol + 16 * kk, adv(ad, kk * 2048), dNI, id_nx, 1);
      };
      for (int fi = cid; fi < nfl; fi += ncl, ++nf) {
        // ---- pass 0: U^T = X^T W~^T (encode-only: into one of 4 U buffers, so that the next fields' encodes
        // overlap this field's pooling epilogue)
        const uint32_t ucol = enc ? 128 * (nf & 3) : 384;
        if (enc) {
          TWAIT(2, MMA_WAIT(&S.ue[nf & 3], ((nf >> 2) & 1) ^ 1));
          ptx::tc_fence_after();
        }
        for (int j = 0; j < T; ++j, ++qw, ++q0) {
          wait_w(qw);
          TWAIT(1, MMA_WAIT(&S.p0full[q0 % NP0], (q0 / NP0) & 1));
          ptx::tc_fence_after();   // (TMA-written operands: no proxy fence needed on this side)
          if (ptx::elect_one()) {
            const uint64_t ad = ptx::sdesc_sw128(ptx::smem_u32(p0slot(S, q0 % NP0)), 8192, 1024);
            const uint64_t bd = ptx::sdesc_sw128(wst(qw), 16, 1024);
#pragma unroll
            for (int kk = 0; kk < NT / 16; ++kk)
              ptx::umma_bf16(tb + ucol, adv(ad, kk * 2048), adv(bd, kk * 32), id_enc, (j | kk) != 0);
            ptx::umma_commit(&S.wempty[qw % NW]);
            ptx::umma_commit(&S.p0empty[q0 % NP0]);
            if (j == T - 1) ptx::umma_commit(enc ? &S.uf[nf & 3] : &S.u_full);
          }
          __syncwarp();
        }
        if (enc) continue;
        // ---- pass 1: R_j - X_j, then G += delta_{j-GLAG} W~_{j-GLAG}^T
        TWAIT(3, MMA_WAIT(&S.h_ready, nf & 1));
        ptx::tc_fence_after();   // H' was fenced to the async proxy by its writers before their arrivals
        const uint32_t qw1 = qw;
        auto issue_G = [&](int j) {
          const uint32_t qj = qw1 + j, db_ = ud & 1;
          TWAIT(5, MMA_WAIT(&S.dl_full[db_], (ud >> 1) & 1));
          ptx::tc_fence_after();   // delta_j: fenced by its writers
          if (ptx::elect_one()) {
            const uint64_t ad = ptx::sdesc_sw128(ptx::smem_u32(S.Dl[db_]), 16, 1024);
            const uint64_t bd = ptx::sdesc_sw128(wst(qj), 16, 1024);
#pragma unroll
            for (int kk = 0; kk < NT / 16; ++kk)
              ptx::umma_bf16(tb + 256, adv(ad, kk * 32), adv(bd, kk * 32), id_g, (j | kk) != 0);
            ptx::umma_commit(&S.dl_empty[db_]);
            ptx::umma_commit(&S.wempty[qj % NW]);
            if (j == T - 1) ptx::umma_commit(&S.g_full);
          }
          __syncwarp();
          TLOG(16 + j, nf);
          ++ud;
        };
        for (int j = 0; j < T; ++j, ++qw, ++ur, ++q1) {
          wait_w(qw);
          TLOG(80 + j, nf);
          const uint32_t rb = ur % NRB, s1 = q1 % np1;
          TWAIT(4, MMA_WAIT(&S.r_empty[rb], ((ur / NRB) & 1) ^ 1));
          TWAIT(44, MMA_WAIT(&S.p1full[s1], (q1 / np1) & 1));
          TLOG(64 + j, nf);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            mma_aw(64 * rb, dH_k, wst(qw));
            mma_negx(64 * rb, ptx::smem_u32(p1slot(S, s1)));
            ptx::umma_commit(&S.r_full[rb]);
            ptx::umma_commit(&S.p1empty[s1]);
            if (!step) ptx::umma_commit(&S.wempty[qw % NW]);
          }
          __syncwarp();
          TLOG(0 + j, nf);
          if (step && j >= GLAG) issue_G(j - GLAG);
        }
        if (!step) continue;
        for (int j = std::max(0, T - GLAG); j < T; ++j) issue_G(j);
        // ---- pass 2 (TMEM: NB2 buffers [dX | dW] in [0,384)): delta_j is the pass-1 tile reloaded from global
        //   dx^T_j = D'^T W~_j + delta_j^T (-I)   (alpha folded into D')
        //   dW_j   = H' delta_j^T + D' X_j^T
        TWAIT(6, MMA_WAIT(&S.d_ready, nf & 1));
        ptx::tc_fence_after();   // D': fenced by its writers
        for (int j = 0; j < T; ++j, ++qw, ++u2, ++qx, ++qd2) {
          const uint32_t pb = u2 % NB2, xsl = qx % NX, sd = qd2 & 1;
          const uint32_t dcol = 128 * pb;
          wait_w(qw);
          TLOG(176 + j, nf);
          TWAIT(8, MMA_WAIT(&S.d2full[sd], (qd2 >> 1) & 1));
          TLOG(160 + j, nf);
          TWAIT(7, MMA_WAIT(&S.p2_empty[pb], ((u2 / NB2) & 1) ^ 1));
          TLOG(192 + j, nf);
          ptx::tc_fence_after();
          const uint32_t dl = ptx::smem_u32(S.Dl[sd]);
          if (ptx::elect_one()) {
            mma_aw(dcol, dD_k, wst(qw));   // D'^T W~_j
            const uint64_t dlk = ptx::sdesc_sw128(dl, 16, 1024);
#pragma unroll
            for (int kk = 0; kk < NT / 16; ++kk)   // + delta_j^T (-I): 16-column blocks
              ptx::umma_bf16(tb + dcol + 16 * kk, adv(dlk, kk * 32), dNI, id_nd, 1);
            ptx::umma_commit(&S.wempty[qw % NW]);
            const uint64_t dlmn = ptx::sdesc_sw128(dl, 16384, 1024);
#pragma unroll
            for (int kk = 0; kk < MC / 16; ++kk)   // H' delta_j^T  (K = samples)
              ptx::umma_bf16(tb + dcol + 64, adv(dH_mn, kk * 2048), adv(dlmn, kk * 2048), id_dw1, kk > 0);
          }
          __syncwarp();
          TWAIT(9, MMA_WAIT(&S.xfull[xsl], (qx / NX) & 1));
          TLOG(144 + j, nf);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            const uint64_t xd = ptx::sdesc_sw128(ptx::smem_u32(S.Xr[xsl]), 16, 1024);
#pragma unroll
            for (int kk = 0; kk < MC / 16; ++kk)   // + D' X_j^T
              ptx::umma_bf16(tb + dcol + 64, adv(dD_mn, kk * 2048), adv(xd, (kk >> 2) * 8192 + (kk & 3) * 32), id_dw2, 1);
            ptx::umma_commit(&S.p2_full[pb]);
            ptx::umma_commit(&S.d2empty[sd]);
            ptx::umma_commit(&S.xempty[xsl]);
            if (j == T - 1) ptx::umma_commit(&S.p0_ok);   // D', delta and the X ring are free for the next field
          }
          __syncwarp();
          TLOG(96 + j, nf);
        }
      }
    }
    __syncwarp();
  } else {
    // =================================================================== epilogue (warps 2..9)
    const int qd = warp & 3;              // TMEM lane quarter
    const int ew = warp - 2;              // epilogue warp index 0..7
    const int half = ew >> 2;             // column half of every 64-column tile (and of the 128 filters)
    const int etid = threadIdx.x - 64;    // 0..255
    const int row = qd * 32 + lane;       // TMEM lane: sample (U, R, G, dX) or filter row (dW)
    const uint32_t tl = tb + ((uint32_t)(qd * 32) << 16);
    const int gi = s0 + row;              // global sample index
    const bool svalid = gi < m;
    const int ng = k / GP;
    const int hc = 32 * half;             // first column of this warp within a tile
    uint32_t nf = 0, ur = 0, ud = 0, u2 = 0;
    // cluster-peer addresses of the dW exchange, mapped once (mapa is an MIO round trip)
    const uint32_t peer_recv = CB > 1 ? ptx::mapa(ptx::smem_u32(&S.recv[half][row][0]), crank ^ 1u) : 0u;
    const uint32_t peer_recv_full = CB > 1 ? ptx::mapa(ptx::smem_u32(&S.recv_full[ew]), crank ^ 1u) : 0u;
    const uint32_t peer_free_bar = CB > 1 ? ptx::mapa(ptx::smem_u32(&S.peer_free[ew]), crank ^ 1u) : 0u;
    float *const bsm = &S.stg[0][0][0];   // b_f during E0 / E1 of a training step
    for (int fi = cid; fi < nfl; fi += ncl, ++nf) {
      const int f = fid(fi);
      const int fr = f / g.gc, fc = f - fr * g.gc;
      const int64_t pixbase = ((int64_t)fr * g.s * g.W + (int64_t)fc * g.s) * g.C;
      ptx::bulk_wait_read0();   // the previous field's last dX rounds have been read out of the staging slices
      ptx::named_bar_sync(1, 32 * NEPI);
      if (etid < KP) {
        const float sg = etid < k ? P.sigma[(int64_t)f * k + etid] : 1.f;
        S.sig[etid] = sg;
        S.isig[etid] = 1.f / sg;
      }
      if (!GEN)   // 2 b_f (see residual32)
        for (int t = etid; t < n; t += 32 * NEPI) bsm[t] = 2.f * P.b[(int64_t)f * n + t];
      ptx::named_bar_sync(1, 32 * NEPI);
      const float a = P.alpha[f];
      // forward / encode stage the pooled output in the slices: b_f is read from global there (not the hot path)
      const float *bf_ = GEN ? P.b + (int64_t)f * n : bsm;
      const bool b16 = !GEN || ((((int64_t)f * n) & 3) == 0);
      double jr = 0.0, js = 0.0;
      float dap = 0.f, rsq4[4] = {0.f, 0.f, 0.f, 0.f};   // rsq4[i]: row 8i + lane/4 of this warp
      TMARK(-1);
      // ------------------------------------------------ E0: pooling / sparsity, H' (filters [64 half, +64))
      const uint32_t ucol = enc ? 128 * (nf & 3) : 384;
      if (enc) TWAIT(11, ptx::mbar_wait(&S.uf[nf & 3], (nf >> 2) & 1));
      else TWAIT(11, ptx::mbar_wait(&S.u_full, nf & 1));
      ptx::tc_fence_after();
#pragma unroll 1
      for (int cc = 2 * half; cc < 2 * half + 2; ++cc) {
        float u[32];
        ptx::tmem_ld16(tl + ucol + cc * 32, u);
        ptx::tmem_ld16(tl + ucol + cc * 32 + 16, u + 16);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int t = 0; t < 32; ++t) u[t] *= S.sig[cc * 32 + t];
        constexpr int NGC = 32 / GP;   // pooling groups per 32-filter chunk
        float pv[NGC];
        float jsc = 0.f;   // this chunk's sum of s_G (fp32 over <= 32 terms, then into the fp64 total)
#pragma unroll
        for (int G0 = 0; G0 < 32; G0 += GP) {
          float ss = 0.f;
#pragma unroll
          for (int t = 0; t < GP; ++t) { float h = a * u[G0 + t]; ss = fmaf(h, h, ss); }
          const int G = (cc * 32 + G0) / GP;
          const float v = P.eps + ss;
          const float sG = v * rsqrtf(fmaxf(v, 1.17549435e-38f));   // sqrt(eps + sum_G h^2); 0 at v = 0
          pv[G0 / GP] = sG;
          if (G < ng) jsc += sG;
        }
        if (svalid) js += (double)jsc;
        if (want_pooled) {   // p [m][gr][gc][ng] (forward / encode only: recv + stg are idle then)
          const int G0c = cc * NGC;   // first group of the chunk
          if constexpr (NGC >= 4) {
            // coalesced: the warp's 32 samples x GH groups are transposed through its 2 KB staging slice so
            // that each store instruction writes whole 16-byte runs of consecutive groups of a few samples
            constexpr int GH = NGC < 16 ? NGC : 16, NC4 = GH / 4;
            float *pst = &S.stg[ew][0][0];
#pragma unroll
            for (int hh = 0; hh < NGC / GH; ++hh) {
#pragma unroll
              for (int c4 = 0; c4 < NC4; ++c4)
                *reinterpret_cast<float4 *>(pst + lane * GH + 4 * (c4 ^ (lane % NC4))) =
                    make_float4(pv[hh * GH + 4 * c4], pv[hh * GH + 4 * c4 + 1], pv[hh * GH + 4 * c4 + 2],
                                pv[hh * GH + 4 * c4 + 3]);
              __syncwarp();
#pragma unroll
              for (int e = lane; e < 32 * NC4; e += 32) {
                const int r = e / NC4, c4 = e % NC4, gs = s0 + qd * 32 + r;
                const float4 q = *reinterpret_cast<const float4 *>(pst + r * GH + 4 * (c4 ^ (r % NC4)));
                const int g0 = G0c + hh * GH + 4 * c4;
                float *dst = P.pooled + (((int64_t)gs * g.gr + fr) * g.gc + fc) * ng + g0;
                if (gs < m) {
                  if ((ng & 3) == 0) {   // 16-byte aligned rows
                    if (g0 < ng) *reinterpret_cast<float4 *>(dst) = q;
                  } else {
                    const float qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                    for (int e2 = 0; e2 < 4; ++e2)
                      if (g0 + e2 < ng) dst[e2] = qq[e2];
                  }
                }
              }
              __syncwarp();
            }
          } else {
#pragma unroll
            for (int q = 0; q < NGC; ++q)
              if (G0c + q < ng && svalid) P.pooled[(((int64_t)gi * g.gr + fr) * g.gc + fc) * ng + G0c + q] = pv[q];
          }
        }
#pragma unroll
        for (int t = 0; t < 32; ++t) u[t] = svalid ? S.sig[cc * 32 + t] * a * u[t] : 0.f;
        uint8_t *blk = S.H + (cc >> 1) * 16384;
        if (!enc) {   // encode-only: H is a pass-0 X slot of the next field
#pragma unroll
          for (int t = 0; t < 32; t += 8) st8(blk, row, (cc & 1) * 32 + t, u + t);
        }
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (enc) {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&S.ue[nf & 3]);   // U buffer read: the MMA may encode into it again
      } else if (lane == 0) {
        ptx::mbar_arrive(&S.h_ready);
      }
      TMARK(32);
      // ------------------------------------------------ E1: residual, delta, db (pass 1)
#pragma unroll 1
      for (int j = 0; j < (enc ? 0 : T); ++j, ++ur) {
        const uint32_t rb = ur % NRB;
        if (j == 0) TWAIT(43, ptx::mbar_wait(&S.r_full[rb], (ur / NRB) & 1));
        else {
          const long long tw0 = TR ? clock64() : 0;
          TWAIT(12, ptx::mbar_wait(&S.r_full[rb], (ur / NRB) & 1));
          if (ew == 0) TLOG(32 + j, nf);
          if (TR && P.trace && lane == 0) atomicAdd(&S.tr[56 + ew], (unsigned long long)(clock64() - tw0));
        }
        ptx::tc_fence_after();
        float rv[32];
        ptx::tmem_ld16(tl + 64 * rb + hc, rv);
        ptx::tmem_ld16(tl + 64 * rb + hc + 16, rv + 16);
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&S.r_empty[rb]);
        jr += 0.25 * (double)residual32(rv, j * NT + hc, n, bf_, svalid, b16, !GEN);   // sum e^2 (x 1/4 exact)
        if (step) {
          const uint32_t db_ = ud & 1;
          TWAIT(14, ptx::mbar_wait(&S.dl_empty[db_], ((ud >> 1) & 1) ^ 1));
#pragma unroll
#pragma unroll
          for (int c = 0; c < 32; c += 8) st8(S.Dl[db_], row, hc + c, rv + c);
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&S.dl_full[db_]);
          if (ew == 0) TLOG(48 + j, nf);
          if (j >= 4 && j < 10) TLOG(208 + (j - 4) * 8 + ew, nf);   // every warp's delta_j, tiles 4..9
          ++ud;
          // db partial: column sums over this warp's 32 samples (butterfly transpose-reduce: lane l <- column l;
          // measured faster than a transpose through the staging slice, whose loads wait behind the stores)
#pragma unroll
          for (int o = 16, w = 16; o >= 1; o >>= 1, w >>= 1) {
            const bool up = lane & o;
#pragma unroll
            for (int t = 0; t < w; ++t) {
              float send = up ? rv[t] : rv[t + w];
              float keep = up ? rv[t + w] : rv[t];
              rv[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
          const float dsum = rv[0];
          // this lane quarter's partial; the four quarters are summed once per field (no per-tile barrier)
          LCAE_DCHECK(j * NT + hc + lane < MAX_NPAD);
          P.dbscr[((size_t)blockIdx.x * 4 + qd) * MAX_NPAD + j * NT + hc + lane] = dsum;
        }
      }
      if (step) {
        TMARK(33);
        // ---------------------------------------------- E1b: D = sigma.G~ + lambda h/s, dalpha, D'
        TWAIT(16, ptx::mbar_wait(&S.g_full, nf & 1));
        ptx::tc_fence_after();
#pragma unroll 1
        for (int cc = 2 * half; cc < 2 * half + 2; ++cc) {
          float u[32], gg[32];
          ptx::tmem_ld16(tl + 384 + cc * 32, u);
          ptx::tmem_ld16(tl + 384 + cc * 32 + 16, u + 16);
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
            const float v = P.eps + ss;
            const float inv = P.lam * rsqrtf(fmaxf(v, 1.17549435e-38f));   // lambda / s_G (v = 0 only with h = 0: R12)
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
        TMARK(34);
        // ---------------------------------------------- E2: dX, dW, fused projected SGD (pass 2)
        const uint64_t pol_ef = ptx::policy_evict_first();   // W~ master / shadow streams
        constexpr int NC = CB > 1 ? 16 : 32, NCH = NC / 16;
        const int oc = CB > 1 ? 16 * (int)crank : 0;
        const int rr = lane >> 2, cq = lane & 3;
        const int64_t wrow0 = (int64_t)f * k + qd * 32 + rr;   // W~ master row of i = 0
        // per-field invariants of this thread's E2 work, hoisted out of the tile loop
        const bool do_red = !FULL || !(P.dbg & 1), do_sgd = !FULL || !(P.dbg & 2);
        const bool sgd_ld = !FULL || !(P.dbg & 4), sgd_st = !FULL || !(P.dbg & 8);   // dev experiments
        const bool has_v = FULL && P.vW != nullptr, keep = FULL && P.keep_grads != 0;
        const float *wrp[4];
        float sgr[4], isgr[4];
        bool rok[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = qd * 32 + 8 * i + rr;
          rok[i] = r < k;
          wrp[i] = P.W + (wrow0 + 8 * i) * P.wp + hc + oc + 4 * cq;
          sgr[i] = S.sig[r];
          isgr[i] = S.isig[r];
        }
        // dX piece words of the warp's two 16-column rounds, loaded one tile ahead (an L2 round trip: the 227 KB
        // shared-memory carve-out leaves L1 too small to keep the table resident)
        auto piece_words = [&](int jj, uint32_t &a0, uint32_t &a1) {
          const uint32_t *dxp = P.dxpieces + ((size_t)jj * 4 + 2 * half) * DXPMAX;
          a0 = lane < DXPMAX ? __ldg(dxp + lane) : 0xFFFFFFFFu;
          a1 = lane < DXPMAX ? __ldg(dxp + DXPMAX + lane) : 0xFFFFFFFFu;
        };
        uint32_t pwn0, pwn1;
        piece_words(0, pwn0, pwn1);
        for (int j = 0; j < T; ++j, ++u2) {
          const uint32_t pb = u2 % NB2, base = 128 * pb;
          {
            const long long tw0 = TR ? clock64() : 0;
            TWAIT(18, ptx::mbar_wait(&S.p2_full[pb], (u2 / NB2) & 1));
            if (ew == 0) TLOG(112 + j, nf);
            if (TR && P.trace && lane == 0) atomicAdd(&S.tr[48 + ew], (unsigned long long)(clock64() - tw0));
          }
          ptx::tc_fence_after();
          TMARK(35);
          const int swr = (lane >> 1) & 3;                     // swizzle of this lane's row (row = lane)
          float *stg = &S.stg[ew][0][0];                       // [32 rows][16] fp32, 16-byte chunks swizzled
          const uint32_t *rcv = &S.recv[half][qd * 32][0];     // [32 rows][16 bf16], written by the peer
          // dx = alpha W^T D - delta (both halves accumulated in TMEM) is overlap-added into the image gradient by the
          // TMA unit: each 16-column round is staged in this warp's slice as [16 patch rows][32 samples] (one
          // conflict-free 128-byte row per column) and reduce-added (cp.reduce.async.bulk.tensor .add.f32) in boxes
          // of consecutive image rows from the host piece table (lanes 0..15 issue one piece each).
          const uint32_t pw0 = pwn0, pw1 = pwn1;
          if (j + 1 < T) piece_words(j + 1, pwn0, pwn1);
          float xv[32];
          auto dx_round = [&](auto RI, uint32_t pw) {
            constexpr int r = decltype(RI)::value;
            ptx::bulk_wait_read0();   // this lane's earlier reduce boxes have read the staging slice
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 16; ++c) stg[c * 32 + lane] = xv[16 * r + c];
            ptx::fence_proxy_async_smem();
            __syncwarp();
            LCAE_DCHECK(pw == 0xFFFFFFFFu || (piece_lg(pw) < (uint32_t)NDMAP && piece_row(pw) + (1u << piece_lg(pw)) <= 16u &&
                                             pixbase + piece_off(pw) + (1u << piece_lg(pw)) <= prow));
            if (pw != 0xFFFFFFFFu && do_red)
              ptx::tma_red_add_2d(&P.tmD[piece_lg(pw)], stg + piece_row(pw) * 32, s0 + qd * 32,
                                  (int)pixbase + (int)piece_off(pw));
            ptx::bulk_commit();
          };
          // dW_j (lanes = filter rows, this warp's 32 columns). CTA c owns the 16-column chunk [16c, 16c+16) of
          // each half; the batch slices of that chunk are summed over the cluster (DSMEM), then the projected SGD
          // runs in a coalesced layout: the own chunk is transposed through this warp's 2 KB staging slice and
          // the peer's is read from the receive slice, so that lane l updates rows 8i + l/4, columns 4(l%4)..+3.
          float4 wv[4 * NCH];   // owned W~ runs, coalesced layout (issued before the dW read)
#pragma unroll
          for (int h = 0; h < NCH; ++h) {
            const int cc0 = j * NT + hc + oc + 16 * h + 4 * cq;
#pragma unroll
            for (int i = 0; i < 4; ++i)
              wv[4 * h + i] = (rok[i] && cc0 < P.wp && sgd_ld) ? ptx::ld_f4_ef(wrp[i] + j * NT + 16 * h, pol_ef)
                                                     : make_float4(0, 0, 0, 0);
          }
          float4 vvp[FULL ? 4 * NCH : 1];   // momentum velocity runs, issued with the W~ runs (full variant)
          if constexpr (FULL) {
#pragma unroll
            for (int h = 0; h < NCH; ++h) {
              const int cc0 = j * NT + hc + oc + 16 * h + 4 * cq;
#pragma unroll
              for (int i = 0; i < 4; ++i)
                vvp[4 * h + i] = (has_v && rok[i] && cc0 < P.wp)
                                     ? ptx::ld_f4_ef(P.vW + (wrp[i] - P.W) + j * NT + 16 * h, pol_ef)
                                     : make_float4(0, 0, 0, 0);
            }
          }
          float4 dq[4 * NCH];   // summed dW chunk(s), coalesced layout
          ptx::bulk_wait_read0();   // the previous tile's last dX round has been read out of the staging slice
          __syncwarp();
          if constexpr (CB > 1) {
            // the dW half the peer owns goes out first and the own half is staged, so that the exchange is in
            // flight while this warp stages and issues the dX reductions
            {
              float dw[32];   // dw[0..15] = the owned chunk, dw[16..31] = the peer's chunk
              ptx::tmem_ld16(tl + base + 64 + hc + 16 * crank, dw);
              ptx::tmem_ld16(tl + base + 64 + hc + 16 * (1 - crank), dw + 16);
              ptx::tmem_ld_wait();
              // arm this warp's receive phase: 32 rows x 16 bf16 arrive from the peer's warp ew via st.async
              if (lane == 0) ptx::mbar_arrive_expect_tx(&S.recv_full[ew], 32 * 16 * 2);
              TWAIT(22, ptx::mbar_wait(&S.peer_free[ew], (u2 & 1) ^ 1));
              // the peer's half crosses DSMEM in bf16 (RN-even; R25): 32 bytes per row
#pragma unroll
              for (int t = 0; t < 2; ++t)
                ptx::st_async_u4(peer_recv + 16 * t,
                                 make_uint4(ptx::pack_bf16x2(dw[16 + 8 * t], dw[17 + 8 * t]),
                                            ptx::pack_bf16x2(dw[18 + 8 * t], dw[19 + 8 * t]),
                                            ptx::pack_bf16x2(dw[20 + 8 * t], dw[21 + 8 * t]),
                                            ptx::pack_bf16x2(dw[22 + 8 * t], dw[23 + 8 * t])),
                                 peer_recv_full);
#pragma unroll
              for (int t = 0; t < 4; ++t)
                *reinterpret_cast<float4 *>(stg + lane * 16 + 4 * (t ^ swr)) =
                    make_float4(dw[4 * t], dw[4 * t + 1], dw[4 * t + 2], dw[4 * t + 3]);
            }
            TMARK(40);
            ptx::tmem_ld16(tl + base + hc, xv);
            ptx::tmem_ld16(tl + base + hc + 16, xv + 16);
            ptx::tmem_ld_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&S.p2_empty[pb]);   // TMEM buffer pb fully read by this warp
            if (ew == 0) TLOG(128 + j, nf);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int r = 8 * i + rr, o = r * 16 + 4 * (cq ^ ((r >> 1) & 3));
              dq[i] = *reinterpret_cast<const float4 *>(stg + o);
            }
            dx_round(std::integral_constant<int, 0>{}, pw0);   // first dX round while the peer's chunk arrives
            TMARK(36);
            TMARK(41);
            // + the peer's batch slice, read straight from the receive slice in the same layout
            TWAIT(22, ptx::mbar_wait(&S.recv_full[ew], u2 & 1));
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int r = 8 * i + rr;
              const uint2 v = *reinterpret_cast<const uint2 *>(rcv + r * 8 + 2 * cq);   // 4 bf16 of columns 4cq..
              dq[i].x += __uint_as_float(v.x << 16);
              dq[i].y += __uint_as_float(v.x & 0xFFFF0000u);
              dq[i].z += __uint_as_float(v.y << 16);
              dq[i].w += __uint_as_float(v.y & 0xFFFF0000u);
            }
            __syncwarp();
            if (lane == 0)   // receive slice read: the peer may send the next tile (reads only; relaxed suffices)
              ptx::mbar_arrive_remote_relaxed(peer_free_bar);
          } else {
            ptx::tmem_ld16(tl + base + hc, xv);
            ptx::tmem_ld16(tl + base + hc + 16, xv + 16);
            float dw[32];
            ptx::tmem_ld16(tl + base + 64 + hc, dw);
            ptx::tmem_ld16(tl + base + 64 + hc + 16, dw + 16);
            ptx::tmem_ld_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&S.p2_empty[pb]);   // TMEM buffer pb fully read by this warp
            TMARK(40);
            TMARK(41);
#pragma unroll
            for (int h = 0; h < NCH; ++h) {
#pragma unroll
              for (int t = 0; t < 4; ++t)
                *reinterpret_cast<float4 *>(stg + lane * 16 + 4 * (t ^ swr)) =
                    make_float4(dw[16 * h + 4 * t], dw[16 * h + 4 * t + 1], dw[16 * h + 4 * t + 2],
                                dw[16 * h + 4 * t + 3]);
              __syncwarp();
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int r = 8 * i + rr, o = r * 16 + 4 * (cq ^ ((r >> 1) & 3));
                dq[4 * h + i] = *reinterpret_cast<const float4 *>(stg + o);
              }
              __syncwarp();
            }
            dx_round(std::integral_constant<int, 0>{}, pw0);
            TMARK(36);
          }
          TMARK(42);
          if (do_sgd) {
            const bool fullc = (j + 1) * NT <= n;   // no column of this tile past n
            const float nlr = -P.lr;
#pragma unroll
            for (int h = 0; h < NCH; ++h) {
              const int cc0 = j * NT + hc + oc + 16 * h + 4 * cq;
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                if (!rok[i] || cc0 >= P.wp) continue;
                float *wp_ = const_cast<float *>(wrp[i]) + j * NT + 16 * h;   // = W~ + row * wp + cc0
                LCAE_DCHECK(wp_ >= P.W && wp_ + 4 <= P.W + (int64_t)g.F * k * P.wp && cc0 + 4 <= P.wp);
                LCAE_DCHECK(((int64_t)f * KP + qd * 32 + 8 * i + rr) * P.n_al + cc0 + 4 <= (int64_t)g.F * KP * P.n_al ||
                            cc0 >= P.n_al);
                const float d0[4] = {dq[4 * h + i].x, dq[4 * h + i].y, dq[4 * h + i].z, dq[4 * h + i].w};
                const float wo4[4] = {wv[4 * h + i].x, wv[4 * h + i].y, wv[4 * h + i].z, wv[4 * h + i].w};
                float d[4], wn[4], vo[4] = {0.f, 0.f, 0.f, 0.f};
                if constexpr (FULL) {
                  const float4 vv = vvp[4 * h + i];
                  vo[0] = vv.x; vo[1] = vv.y; vo[2] = vv.z; vo[3] = vv.w;
                }
                // the accumulator holds sigma_r dJ/dW: dJ/dW = acc / sigma_r; W~' = sigma_r W~ - lr dJ/dW
                const float cr = nlr * isgr[i];
                // plain SGD (lean): rownorm(sigma W~ - lr acc / sigma) = rownorm(W~ - (lr / sigma^2) acc) for
                // sigma > 0, so W~ is updated without the sigma scale (one FFMA per element) and sigma' = 1 / ||W~'||
                // follows in the finalize kernel as before; with momentum the velocity lives in W's scale
                const float cr2 = cr * isgr[i];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float acc = (fullc || cc0 + e < n) ? d0[e] : 0.f;
                  d[e] = acc;
                  if constexpr (FULL) {
                    float upd = cr * acc;
                    if (has_v) { upd = fmaf(P.mu, vo[e], upd); vo[e] = upd; }
                    wn[e] = fmaf(sgr[i], wo4[e], upd);
                  } else {
                    wn[e] = fmaf(cr2, acc, wo4[e]);
                  }
                  rsq4[i] = fmaf(wn[e], wn[e], rsq4[i]);
                }
                wv[4 * h + i] = make_float4(wn[0], wn[1], wn[2], wn[3]);   // stored after the second dX round
                if (has_v) *reinterpret_cast<float4 *>(P.vW + (wp_ - P.W)) = make_float4(vo[0], vo[1], vo[2], vo[3]);
                if (keep) {
                  const float is = isgr[i];
                  *reinterpret_cast<float4 *>(P.gW + (wp_ - P.W)) = make_float4(d[0] * is, d[1] * is, d[2] * is, d[3] * is);
                }
              }
            }
          }
          dx_round(std::integral_constant<int, 1>{}, pw1);   // second dX round (its staging read overlaps the next tile)
          // the W~' runs (fp32 master, bf16 shadow) leave after the dX round: its shared-memory proxy fence then
          // does not wait behind these global stores, which drain while the next tile starts
          if (do_sgd && sgd_st) {
#pragma unroll
            for (int h = 0; h < NCH; ++h) {
              const int cc0 = j * NT + hc + oc + 16 * h + 4 * cq;
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                if (!rok[i] || cc0 >= P.wp) continue;
                const int r = qd * 32 + 8 * i + rr;
                const float4 w4 = wv[4 * h + i];
                ptx::st_f4_ef(const_cast<float *>(wrp[i]) + j * NT + 16 * h, w4, pol_ef);
                if (cc0 < P.n_al)
                  ptx::st_u2_ef(P.Wb + ((int64_t)f * KP + r) * P.n_al + cc0,
                                make_uint2(ptx::pack_bf16x2(w4.x, w4.y), ptx::pack_bf16x2(w4.z, w4.w)), pol_ef);
              }
            }
          }
          TMARK(37);
        }
      }
      TMARK(step ? 38 : 33);
      // ------------------------------------------------ per-field partial sums (fixed order)
      jr = warp_sum(jr);
      js = warp_sum(js);
      dap = warp_sum(dap);
      if (lane == 0) { S.redd[ew][0] = jr; S.redd[ew][1] = js; S.redf[ew] = dap; }
      ptx::named_bar_sync(1, 32 * NEPI);
      if (step) {   // db of this CTA's samples: the four lane quarters' partials (fixed order)
        const float *d = P.dbscr + (size_t)blockIdx.x * 4 * MAX_NPAD;
        for (int t = etid; t < n; t += 32 * NEPI)
          P.db_part[((int64_t)f * CB + crank) * n + t] = ((d[t] + d[MAX_NPAD + t]) + d[2 * MAX_NPAD + t]) + d[3 * MAX_NPAD + t];
      }
      LCAE_DCHECK(f < g.F && (int)crank < CB);
      if (etid == 0) {
        double a0 = 0.0, a1 = 0.0;
        float a2 = 0.f;
        for (int w = 0; w < NEPI; ++w) { a0 += S.redd[w][0]; a1 += S.redd[w][1]; a2 += S.redf[w]; }
        P.loss_part[((int64_t)f * CB + crank) * 2 + 0] = a0;
        P.loss_part[((int64_t)f * CB + crank) * 2 + 1] = (double)P.lam * a1;
        P.da_part[(int64_t)f * CB + crank] = a2;
      }
      if (step) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {   // the 4 lanes of a row run hold its partial sums
          float v = rsq4[i];
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          if ((lane & 3) == 0) P.rowsq_part[(((int64_t)f * CB + crank) * 2 + half) * KP + qd * 32 + 8 * i + (lane >> 2)] = v;
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
    }
  }
  // ---- teardown
  if (step && warp >= 2 && warp < XWARP) ptx::bulk_wait0();   // every dX reduce box complete before exit
  if (trec) atomicAdd(&S.tr[warp == 1 ? 10 : warp == 0 ? 25 : warp == XWARP ? 24 : 26],
                      (unsigned long long)(clock64() - t_start));
  ptx::tc_fence_before();
  __syncthreads();
  if (P.trace && threadIdx.x < 64) atomicAdd(&P.trace[threadIdx.x], S.tr[threadIdx.x]);
#undef TWAIT
#undef TMARK
#undef TLOG
#undef MMA_WAIT
  if (CB > 1) ptx::cluster_sync();
  if (warp == 1) ptx::tmem_dealloc<512>(tb);
}

}  // namespace tc
}  // namespace lcae
