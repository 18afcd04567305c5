// lcn.cu — local contrast normalisation between stacked layers (formula
// per SPEC.md:215-223 / DESIGN.md R15): v = x - mean_w(x), y = v / max(floor, sqrt(mean_w(v^2))), uniform
// w x w window per channel, zero padding with count-correct divisors. Separable box sums, four HBM-bound
// passes over [m][H][W][C] (C innermost: every pass is coalesced across channels).
#include "common.cuh"

namespace lcae {
namespace {

// t = horizontal window sum of a (or of a^2 when SQ)
template <bool SQ>
__global__ void lcn_hsum(const float *__restrict__ a, float *__restrict__ t, int64_t n, int W, int C, int r) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % C);
    const int x = (int)((e / C) % W);
    const int64_t row = e - (int64_t)x * C - c;   // element (.., .., 0, 0) of this row
    const int x0 = max(0, x - r), x1 = min(W - 1, x + r);
    float s = 0.f;
    for (int xx = x0; xx <= x1; ++xx) {
      const float v = __ldg(a + row + (int64_t)xx * C + c);
      s += SQ ? v * v : v;
    }
    t[e] = s;
  }
}

// vertical window sum of t, divided by the in-bounds count: the local mean. FIRST: v = x - mean -> out;
// else: y = v / max(floor, sqrt(mean)) -> out (v passed as x).
template <bool FIRST>
__global__ void lcn_vsum(const float *__restrict__ t, const float *__restrict__ x, float *__restrict__ out,
                         int64_t n, int H, int W, int C, int r, float floor_) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t wc = (int64_t)W * C;
    const int y = (int)((e / wc) % H);
    const int xcol = (int)((e / C) % W);
    const int64_t colbase = e - (int64_t)y * wc;   // same (x, c) in row 0 of this image
    const int y0 = max(0, y - r), y1 = min(H - 1, y + r);
    const int x0 = max(0, xcol - r), x1 = min(W - 1, xcol + r);
    float s = 0.f;
    for (int yy = y0; yy <= y1; ++yy) s += __ldg(t + colbase + (int64_t)yy * wc);
    const float mean = s / (float)((y1 - y0 + 1) * (x1 - x0 + 1));
    if (FIRST) out[e] = x[e] - mean;
    else out[e] = x[e] / fmaxf(floor_, sqrtf(mean));
  }
}

}  // namespace
}  // namespace lcae

using namespace lcae;

extern "C" lcae_status lcae_lcn(const float *x, float *y, float *scratch, int32_t m, int32_t H, int32_t W, int32_t C,
                                int32_t window, float floor_, void *stream) {
  if (!x || !y || !scratch || m < 0 || H < 1 || W < 1 || C < 1 || window < 1 || (window & 1) == 0 || window > H ||
      window > W || !(floor_ > 0.f)) {
    set_error("lcae_lcn: bad arguments (odd window <= map size, floor > 0)");
    return LCAE_ERR_CONFIG;
  }
  const int64_t n = (int64_t)m * H * W * C;
  if (n == 0) return LCAE_OK;
  float *t = scratch, *v = scratch + n;
  const int r = window / 2;
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = 256, blocks = (int)std::min<int64_t>((n + threads - 1) / threads, 148 * 32);
  lcn_hsum<false><<<blocks, threads, 0, st>>>(x, t, n, W, C, r);
  lcn_vsum<true><<<blocks, threads, 0, st>>>(t, x, v, n, H, W, C, r, floor_);
  lcn_hsum<true><<<blocks, threads, 0, st>>>(v, t, n, W, C, r);
  lcn_vsum<false><<<blocks, threads, 0, st>>>(t, v, y, n, H, W, C, r, floor_);
  LCAE_CK(cudaGetLastError());
  return LCAE_OK;
}
