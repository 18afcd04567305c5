// common.cuh — shared device helpers and the layer's internal state (liblcae.so, sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>
#include <utility>
#include <vector>

#include "../../include/lcae.h"

namespace lcae {

void set_error(const std::string &msg);

#define LCAE_CK(call)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      ::lcae::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                 \
      return LCAE_ERR_CUDA;                                                                  \
    }                                                                                        \
  } while (0)

#define LCAE_CK_LAUNCH(L)                                                                    \
  do {                                                                                       \
    cudaError_t e_ = cudaGetLastError();                                                     \
    if (e_ != cudaSuccess) {                                                                 \
      ::lcae::set_error(std::string("kernel launch: ") + cudaGetErrorString(e_));            \
      return LCAE_ERR_CUDA;                                                                  \
    }                                                                                        \
    (L)->launches++;                                                                         \
  } while (0)

// Geometry derived from lcae_config (integer bookkeeping only).
struct Geo {
  int H, W, C, rf_h, rf_w, s, k, g, m;
  int gr, gc, F, n, RW;   // RW = rf_w*C (contiguous (rx, c) run of one receptive-field row)
  int64_t SY;             // HWCN element stride between image rows: W*C*m
  int64_t SRC_R, SRC_C;   // HWCN element offset of field (r,c): r*s*W*C*m, c*s*C*m
};

// Chunk scratch of the fp32 SIMT path.
struct F32Scratch {
  int Fc = 0;
  float *U = nullptr, *H = nullptr, *Q = nullptr, *G = nullptr;   // [Fc][k][m]
  float *R = nullptr;                                           // [Fc][n][m] (r, then delta)
  float *dXp = nullptr;                                         // [Fc][n][m]
  float *dW = nullptr;                                          // [Fc][k][n]
  float *da = nullptr;                                          // [Fc]
  float *db = nullptr;                                          // [Fc][n]
};

struct TcScratch;   // bf16 tensor-core path: the fused step kernel (tc_host.cu)
struct GtScratch;   // bf16 tensor-core path for shapes beyond the fused kernel (gt_path.cu)
struct MpState;     // model-parallel tile state (mp.cu)

// One rank's tile of a model-parallel layer (mp.cu): field rows [R0, R1) x cols [C0, C1) of the global grid;
// need / own = pixel rectangles (y0, y1, x0, x1) read by its fields / owned (input and input gradient).
struct MpTile {
  int tr_n = 1, tc_n = 1, R0 = 0, R1 = 0, C0 = 0, C1 = 0;
  int need[4] = {0, 0, 0, 0}, own[4] = {0, 0, 0, 0};
};

}  // namespace lcae

struct lcae_layer {
  lcae_config cfg;
  lcae::Geo geo;
  cudaStream_t st = nullptr;
  int device = 0;
  int sm_count = 148;
  // parameters (device). W holds W~ with per-row scale sigma: W = sigma (.) W~ (sigma == 1 in fp32 mode)
  float *W = nullptr, *sigma = nullptr, *alpha = nullptr, *b = nullptr;
  float *vW = nullptr, *va = nullptr, *vb = nullptr;   // momentum velocity (momentum > 0)
  __nv_bfloat16 *Wb = nullptr;                         // bf16 shadow [F][k][n_al] (bf16 mode)
  int n_al = 0;                                        // n rounded up to 8 (16-byte rows)
  int mp = 0;                                          // batch stride of the internal HWCN buffers
  int wp = 0;                                          // row pitch (floats) of W~, vW, gW
  // inputs / outputs
  float *x_stage = nullptr;      // NHWC f32 staging for host inputs
  // input prefetch (lcae_prefetch_input): host batch copied on its own stream into x_pf, overlapping a step
  float *x_pf = nullptr;
  const void *pf_host = nullptr;   // host pointer whose copy is in flight / landed in x_pf
  cudaStream_t copy_st = nullptr;
  cudaEvent_t pf_done = nullptr, x_consumed = nullptr;
  float *xt32 = nullptr;         // HWCN f32 (fp32 mode)
  __nv_bfloat16 *xt16 = nullptr; // HWCN bf16 (bf16 mode)
  float *dxt = nullptr;          // HWCN f32 dX accumulator
  float *dx_nhwc = nullptr;      // NHWC f32 dX
  float *pooled = nullptr;       // [m][gr][gc][k/g]
  // gradients kept for tests
  float *gW = nullptr, *galpha = nullptr, *gb = nullptr;
  // loss: per-field partials [F][2] fp64 (rec, sparse) and the reduced pair
  double *loss_part = nullptr, *loss_dev = nullptr, *loss_host = nullptr;
  int *reinit_dev = nullptr;   // degenerate rows re-initialised (device counter)
  int64_t *step_dev = nullptr;   // steps taken (device counter: CUDA-graph replays stay exact)
  // sticky error flags (device): [0] non-finite input seen by the staging kernel, [1] non-finite loss. While
  // either is set every parameter-updating kernel returns without writing; lcae_sync / a loss read reports and
  // clears them (include/lcae.h "Errors").
  int *flags_dev = nullptr, *flags_host = nullptr;
  float *rowsq = nullptr;      // [F][k] row sums of squares of the updated W~ (bf16 mode)
  int64_t steps = 0;
  int launches = 0;
  lcae::F32Scratch f32;
  lcae::TcScratch *tc = nullptr;
  lcae::GtScratch *gt = nullptr;   // bf16 layers the fused kernel cannot hold (k > 128, n > 4096, m > 256)
  lcae::MpState *mpst = nullptr;   // model-parallel state (world_size > 1)
  // dev checks (sanitizer substitute, include/lcae.h is unaffected): LCAE_DEV_POISON=1 fills every allocation
  // with 0xFF bytes (NaN) so that a read before write shows up in the results; LCAE_DEV_CANARY=1 pads every
  // allocation with a 4 KB 0xA5 tail that lcae_dev_check_canaries verifies (out-of-bounds writes)
  int poison = 0, canary = 0;
  std::vector<std::pair<void *, size_t>> allocs;
  // profiling (lcae_profile): events around the dominant kernel
  int prof_on = 0, prof_n = 0;
  cudaEvent_t *prof_ev = nullptr;   // [2 * 4096]
};

namespace lcae {

constexpr size_t CANARY_BYTES = 4096;

// Device-side bounds checks of the checked build (LCAE_CHECKED; no code in the production build).
#ifdef LCAE_CHECKED
#define LCAE_DCHECK(cond)                                                                                  \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("lcae check failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, blockIdx.x, threadIdx.x, \
             #cond);                                                                                       \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define LCAE_DCHECK(cond) do { } while (0)
#endif

// Every device allocation of a layer goes through here (dev poison / canary modes above).
template <typename T>
inline cudaError_t dmalloc(lcae_layer *L, T **p, size_t bytes) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void **>(p), bytes + (L->canary ? CANARY_BYTES : 0));
  if (e != cudaSuccess) return e;
  if (L->poison && (e = cudaMemset(*p, 0xFF, bytes)) != cudaSuccess) return e;
  if (L->canary) {
    if ((e = cudaMemset(reinterpret_cast<char *>(*p) + bytes, 0xA5, CANARY_BYTES)) != cudaSuccess) return e;
    L->allocs.emplace_back(*p, bytes);
  }
  return cudaSuccess;
}

__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }

// SplitMix64 finaliser (same counter-based generator as oracle.reinit_row; implemented separately).
__host__ __device__ inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
__device__ inline T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide fp64 sum in a fixed order (deterministic). blockDim.x multiple of 32, <= 1024.
__device__ inline double block_sum_f64(double v, double *sh /*[32]*/) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;   // valid in thread 0
}

// ---- host-side entry points implemented in the .cu files ----
lcae_status f32_alloc(lcae_layer *L);
void f32_free(lcae_layer *L);
lcae_status f32_step(lcae_layer *L, bool update, bool want_pooled);

lcae_status tc_alloc(lcae_layer *L);
void tc_free(lcae_layer *L);
// flist/nfl: the fields of this launch (NULL: all); first: zero the dX accumulator; last: run the finalize kernel;
// reserve_clusters: SM pairs left free (model-parallel interior launch overlapping the NCCL halo exchange)
lcae_status tc_step(lcae_layer *L, bool update, bool want_pooled, bool encode_only = false, const int *flist = nullptr,
                    int nfl = 0, bool first = true, bool last = true, int reserve_clusters = 0);
lcae_status tc_finalize(lcae_layer *L);
// the fused kernel's limits (NULL = holds): a bf16 layer beyond them runs on the general tcgen05 GEMM path
const char *tc_unsupported(const Geo &g);

lcae_status gt_alloc(lcae_layer *L);
void gt_free(lcae_layer *L);
lcae_status gt_step(lcae_layer *L, bool update, bool want_pooled, bool encode_only);

// shared by the fp32 and the general bf16 paths (f32_path.cu)
__global__ void col2im_f32(Geo g, int f0, int Fc, const float *dXp, float *dxt);
__global__ void update_ab_f32(Geo g, int f0, int Fc, float *alpha, float *bvec, const float *da, const float *db,
                              float *va, float *vb, float lr, float mu, float amin, const int *flags);

// model parallelism (mp.cu)
lcae_status mp_tile(const lcae_config *c, const Geo &global, int rank, MpTile *t);
lcae_status mp_init(lcae_layer *L, const Geo &global);
void mp_free(lcae_layer *L);
size_t mp_input_elems(lcae_layer *L);
lcae_status mp_stage(lcae_layer *L, const float *x_dev);
lcae_status mp_phase(lcae_layer *L, int phase, bool update, bool want_pooled);
bool mp_external(lcae_layer *L);
lcae_status mp_buffer(lcae_layer *L, int which, int peer, void **ptr, int64_t *bytes);
void mp_counts(lcae_layer *L, int *n_int, int *n_bnd);
const MpTile &mp_tile_of(lcae_layer *L);
double *tc_loss_part(lcae_layer *L);
int tc_loss_count(lcae_layer *L);

// aux kernels (aux.cu)
lcae_status launch_nhwc_to_hwcn_f32(lcae_layer *L, const float *x, float *xt);
lcae_status launch_nhwc_to_hwcn_bf16(lcae_layer *L, const float *x, __nv_bfloat16 *xt);
lcae_status launch_hwcn_to_nhwc_f32(lcae_layer *L, const float *xt, float *x);
lcae_status launch_loss_reduce(lcae_layer *L, bool update);
lcae_status launch_init_params(lcae_layer *L);
lcae_status launch_fill(lcae_layer *L, float *p, int64_t n, float v);
lcae_status launch_get_W(lcae_layer *L, float *Wout);   // sigma (.) W~ -> dense [F][k][n]
lcae_status launch_get_W_range(lcae_layer *L, float *Wout, int64_t f0, int64_t nf);
lcae_status launch_refresh_shadow(lcae_layer *L);       // W~ -> bf16 shadow

}  // namespace lcae
