// dev_mma_rate.cu — microbenchmark of back-to-back tcgen05.mma issue (kind::f16, M = 128, SS operands) for the
// shapes the step kernel uses; reports cycles per MMA instruction. Dev hook only (lcae_dev_mma_rate).
#include "common.cuh"
#include "ptx.cuh"

namespace lcae {
namespace {

__global__ void __launch_bounds__(128) mma_rate_kernel(int N, int a_mn, int b_mn, int iters, int commit_every,
                                                       unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *sA = smem;            // 32 KB: 128 x 128 bf16 (either majorness)
  uint8_t *sB = smem + 32768;    // 32 KB: up to 256 x 64 / 64 x 256
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3c003c00u;
  ptx::fence_proxy_async_smem();
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc<256>(&tbase_s);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tb = tbase_s;
  if (commit_every < 0 && threadIdx.x < 32) {
    // warp-uniform issue loop: all lanes compute the (uniform) descriptors, one elected lane issues
    const uint32_t idesc = ptx::idesc_bf16(128, N, a_mn, b_mn);
    const uint32_t a0 = ptx::smem_u32(sA), b0 = ptx::smem_u32(sB);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad = a_mn ? ptx::sdesc_sw128(a0 + kk * 2048, 8192, 1024) : ptx::sdesc_sw128(a0 + kk * 32, 16, 1024);
        uint64_t bd = b_mn ? ptx::sdesc_sw128(b0 + kk * 2048, 16384, 1024) : ptx::sdesc_sw128(b0 + kk * 32, 16, 1024);
        if (ptx::elect_one()) ptx::umma_bf16(tb, ad, bd, idesc, (it | kk) != 0);
        __syncwarp();
      }
    }
    if (ptx::elect_one()) ptx::umma_commit(&bar);
    __syncwarp();
    ptx::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  } else if (commit_every >= 0 && threadIdx.x == 0) {
    const uint32_t idesc = ptx::idesc_bf16(128, N, a_mn, b_mn);
    const uint32_t a0 = ptx::smem_u32(sA), b0 = ptx::smem_u32(sB);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad = a_mn ? ptx::sdesc_sw128(a0 + kk * 2048, 8192, 1024) : ptx::sdesc_sw128(a0 + kk * 32, 16, 1024);
        uint64_t bd = b_mn ? ptx::sdesc_sw128(b0 + kk * 2048, 16384, 1024) : ptx::sdesc_sw128(b0 + kk * 32, 16, 1024);
        ptx::umma_bf16(tb, ad, bd, idesc, (it | kk) != 0);
      }
      if (commit_every && (it % commit_every) == commit_every - 1) {
        ptx::umma_commit(&bar);
        ptx::mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    ptx::umma_commit(&bar);
    ptx::mbar_wait(&bar, ph);
    long long t1 = clock64();
    out[0] = (unsigned long long)(t1 - t0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc<256>(tb);
}

}  // namespace
}  // namespace lcae

using namespace lcae;

extern "C" lcae_status lcae_dev_mma_rate(int N, int a_mn, int b_mn, int iters, int commit_every,
                                         double *cycles_per_mma) {
  unsigned long long *d = nullptr, h = 0;
  LCAE_CK(cudaMalloc(&d, 8));
  int smem = 65536 + 1024;
  LCAE_CK(cudaFuncSetAttribute(mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  mma_rate_kernel<<<1, 128, smem>>>(N, a_mn, b_mn, iters, commit_every, d);
  LCAE_CK(cudaGetLastError());
  LCAE_CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
  cudaFree(d);
  *cycles_per_mma = (double)h / (4.0 * iters);
  return LCAE_OK;
}
