// topk.cu — streaming top-K stimuli per unit.
// One thread per unit keeps its K best (value, image id) pairs in registers while it walks the batch; the
// order is value descending, ties by lower image id. HBM-bound: the batch's activations are
// read once, coalesced across units (act is [m][units]).
#include <climits>

#include "common.cuh"

namespace lcae {
namespace {

constexpr int KMAX = 32;

__device__ __forceinline__ bool better(float a, int ia, float b, int ib) { return a > b || (a == b && ia < ib); }

__global__ void topk_init_kernel(float *vals, int32_t *ids, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    vals[i] = -INFINITY;
    ids[i] = INT_MAX;
  }
}

// KT: the state length as a compile-time constant (the common K = 1..8, 16, 32: insertion and register arrays sized
// exactly), or KMAX with the runtime K masking the rest
template <int KT>
__global__ void __launch_bounds__(128) topk_update_kernel(const float *__restrict__ act, int64_t m, int64_t units,
                                                          int K_, int64_t id0, float *vals, int32_t *ids) {
  const int K = KT < KMAX ? KT : K_;
  constexpr int KMAX = KT;
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= units) return;
  float v[KMAX];
  int id[KMAX];
#pragma unroll
  for (int t = 0; t < KMAX; ++t) {
    v[t] = t < K ? vals[u * K + t] : -INFINITY;
    id[t] = t < K ? ids[u * K + t] : INT_MAX;
  }
  // the K-th entry, kept in registers (static indexing only: the arrays stay in registers)
  auto kth = [&](float &vl, int &il) {
#pragma unroll
    for (int t = 0; t < KMAX; ++t)
      if (t == K - 1) { vl = v[t]; il = id[t]; }
  };
  float vl;
  int il;
  kth(vl, il);
  // samples in chunks of 8: the chunk's loads are issued together (HBM latency overlapped), then merged
  for (int64_t s0 = 0; s0 < m; s0 += 8) {
    float cvs[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) cvs[q] = s0 + q < m ? __ldg(act + (s0 + q) * units + u) : -INFINITY;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
    float cv = cvs[q];
    int ci = (int)(id0 + s0 + q);
    if (s0 + q >= m || !better(cv, ci, vl, il)) continue;
    // insertion by exchange from the top: the incoming pair moves down past every better-ranked entry
#pragma unroll
    for (int t = 0; t < KMAX; ++t) {
      if (t < K && better(cv, ci, v[t], id[t])) {
        const float tv = v[t];
        const int ti = id[t];
        v[t] = cv;
        id[t] = ci;
        cv = tv;
        ci = ti;
      }
    }
    kth(vl, il);
    }
  }
#pragma unroll
  for (int t = 0; t < KMAX; ++t)
    if (t < K) {
      vals[u * K + t] = v[t];
      ids[u * K + t] = id[t];
    }
}

}  // namespace
}  // namespace lcae

using namespace lcae;

extern "C" lcae_status lcae_topk_init(float *vals, int32_t *ids, int64_t units, int32_t K, void *stream) {
  if (!vals || !ids || units < 0 || K < 1 || K > KMAX) { set_error("lcae_topk_init: bad arguments (1 <= K <= 32)"); return LCAE_ERR_ARG; }
  const int64_t n = units * K;
  if (n == 0) return LCAE_OK;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  topk_init_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(vals, ids, n);
  LCAE_CK(cudaGetLastError());
  return LCAE_OK;
}

extern "C" lcae_status lcae_topk_update(const float *act, int64_t m, int64_t units, int32_t K, int64_t id0,
                                        float *vals, int32_t *ids, void *stream) {
  if (!act || !vals || !ids || m < 0 || units < 0 || K < 1 || K > KMAX || id0 < 0 || id0 + m > INT_MAX) {
    set_error("lcae_topk_update: bad arguments (1 <= K <= 32, image ids < 2^31)");
    return LCAE_ERR_ARG;
  }
  if (m == 0 || units == 0) return LCAE_OK;
  const unsigned blocks = (unsigned)((units + 127) / 128);
  cudaStream_t st = (cudaStream_t)stream;
  switch (K) {
#define LCAE_TOPK(KV) \
  case KV: topk_update_kernel<KV><<<blocks, 128, 0, st>>>(act, m, units, K, id0, vals, ids); break;
    LCAE_TOPK(1) LCAE_TOPK(2) LCAE_TOPK(3) LCAE_TOPK(4) LCAE_TOPK(5) LCAE_TOPK(6) LCAE_TOPK(7) LCAE_TOPK(8)
    LCAE_TOPK(16)
#undef LCAE_TOPK
    default: topk_update_kernel<KMAX><<<blocks, 128, 0, st>>>(act, m, units, K, id0, vals, ids); break;
  }
  LCAE_CK(cudaGetLastError());
  return LCAE_OK;
}
