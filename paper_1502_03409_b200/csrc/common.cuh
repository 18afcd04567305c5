// common.cuh — shared device helpers and the layer's internal state (liblcae.so, sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>

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

struct TcScratch;   // bf16 tensor-core path (tc_path.cu)

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
  // profiling (lcae_profile): events around the dominant kernel
  int prof_on = 0, prof_n = 0;
  cudaEvent_t *prof_ev = nullptr;   // [2 * 4096]
};

namespace lcae {

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
lcae_status tc_step(lcae_layer *L, bool update, bool want_pooled, bool encode_only = false);
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
lcae_status launch_refresh_shadow(lcae_layer *L);       // W~ -> bf16 shadow

}  // namespace lcae
