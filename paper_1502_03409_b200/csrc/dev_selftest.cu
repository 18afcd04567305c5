// dev_selftest.cu — hardware self-tests of the PTX layer (descriptor encodings, TMA swizzle) and a
// global-reduction throughput probe. Exported as lcae_dev_* test hooks; not part of the training path.
#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.cuh"

namespace lcae {
namespace {

// D (128 x N, fp32) = A (128 x K) * B (K x N); A, B row-major bf16 in global; laid out in smem as the
// requested majorness (SW128 canonical layouts), one CTA of 128 threads.
__global__ void __launch_bounds__(128) umma_selftest_kernel(int a_mn, int b_mn, int N, int K, int variant,
                                                            const __nv_bfloat16 *A, const __nv_bfloat16 *B,
                                                            float *D) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *sA = smem;                       // 128*K*2 bytes
  uint8_t *sB = smem + 128 * K * 2;         // K*N*2 bytes
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  // ---- fill A
  for (int e = tid; e < 128 * K; e += 128) {
    int mrow = e / K, kk = e % K;
    uint32_t off;
    if (!a_mn) off = (kk / 64) * (128 * 128) + ptx::sw128_off(mrow, kk % 64);           // [M][64K] blocks
    else off = (mrow / 64) * (K * 128) + ptx::sw128_off(kk, mrow % 64);                 // [K][64M] blocks
    *reinterpret_cast<__nv_bfloat16 *>(sA + off) = A[e];
  }
  // ---- fill B (K x N)
  for (int e = tid; e < K * N; e += 128) {
    int kk = e / N, ncol = e % N;
    uint32_t off;
    if (!b_mn) off = (kk / 64) * (N * 128) + ptx::sw128_off(ncol, kk % 64);             // [N][64K] blocks
    else off = (ncol / 64) * (K * 128) + ptx::sw128_off(kk, ncol % 64);                 // [K][64N] blocks
    *reinterpret_cast<__nv_bfloat16 *>(sB + off) = B[e];
  }
  ptx::fence_proxy_async_smem();
  if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (tid < 32) ptx::tmem_alloc<256>(&tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = ptx::idesc_bf16(128, N, a_mn, b_mn);
    for (int k0 = 0; k0 < K; k0 += 16) {
      uint64_t ad, bd;
      uint32_t lbo_a = a_mn ? K * 128 : 16, sbo_a = 1024;
      uint32_t lbo_b = b_mn ? K * 128 : 16, sbo_b = 1024;
      if (variant == 1) {   // swapped interpretation for MN-major operands
        if (a_mn) { uint32_t t = lbo_a; lbo_a = sbo_a; sbo_a = t; }
        if (b_mn) { uint32_t t = lbo_b; lbo_b = sbo_b; sbo_b = t; }
      }
      uint32_t a_addr = ptx::smem_u32(sA) + (a_mn ? k0 * 128 : (k0 / 64) * (128 * 128) + (k0 % 64) * 2);
      uint32_t b_addr = ptx::smem_u32(sB) + (b_mn ? k0 * 128 : (k0 / 64) * (N * 128) + (k0 % 64) * 2);
      ad = ptx::sdesc_sw128(a_addr, lbo_a, sbo_a);
      bd = ptx::sdesc_sw128(b_addr, lbo_b, sbo_b);
      ptx::umma_bf16(tbase, ad, bd, idesc, k0 > 0);
    }
    ptx::umma_commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  const int warp = tid >> 5, lane = tid & 31;
  for (int c = 0; c < N; c += 8) {
    float v[8];
    ptx::tmem_ld8(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
    ptx::tmem_ld_wait();
    for (int q = 0; q < 8; ++q) D[(warp * 32 + lane) * N + c + q] = v[q];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (tid < 32) ptx::tmem_dealloc<256>(tbase);
}

__global__ void tma_selftest_kernel(const __grid_constant__ CUtensorMap tmap, int box_rows, int r0, int c0,
                                    uint8_t *dump) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  const int bytes = box_rows * 128;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bar, bytes);
    ptx::tma_load_2d(smem, &tmap, &bar, c0, r0);
  }
  ptx::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) dump[i] = smem[i];
}

// TMA box landing at an arbitrary 128-byte row offset inside a 1024-byte swizzle atom (the X gather of the
// step kernel places runs of patch rows this way): dump the whole 16-row region.
__global__ void tma_offset_selftest_kernel(const __grid_constant__ CUtensorMap tmap, int box_rows, int r0, int c0,
                                           int dst_row, uint8_t *dump) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 64 * 128; i += blockDim.x) smem[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  ptx::fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bar, box_rows * 128);
    ptx::tma_load_2d(smem + dst_row * 128, &tmap, &bar, c0, r0);
  }
  ptx::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 64 * 128; i += blockDim.x) dump[i] = smem[i];
}

// Throughput probe: every thread issues `reps` fp32 reductions (mode 0: red.global.add.f32 coalesced,
// mode 1: red.global.add.v4.f32, mode 2: plain ld+add+st) over a buffer of n floats.
__global__ void red_probe_kernel(float *buf, int64_t n, int reps, int mode) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    if (mode == 1) {
      int64_t idx = ((tid + r * 977 * 32) % (n / 4)) * 4;
      float *p = buf + idx;
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f),
                   "f"(1.f)
                   : "memory");
    } else {
      int64_t idx = (tid + r * 977 * 32) % n;
      if (mode == 0) atomicAdd(buf + idx, 1.f);
      else buf[idx] += 1.f;
    }
  }
  (void)nthreads;
}

}  // namespace
}  // namespace lcae

using namespace lcae;

extern "C" lcae_status lcae_dev_umma_selftest(int a_mn, int b_mn, int N, int K, int variant, const void *A,
                                              const void *B, float *D) {
  if (N % 16 || N < 16 || N > 256 || K % 64 || K > 128) { set_error("selftest: bad shape"); return LCAE_ERR_ARG; }
  int Npad = (N + 63) / 64 * 64;
  int smem = 128 * K * 2 + K * Npad * 2 + 1024;
  LCAE_CK(cudaFuncSetAttribute(umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  umma_selftest_kernel<<<1, 128, smem>>>(a_mn, b_mn, N, K, variant, (const __nv_bfloat16 *)A,
                                         (const __nv_bfloat16 *)B, D);
  LCAE_CK(cudaGetLastError());
  LCAE_CK(cudaDeviceSynchronize());
  return LCAE_OK;
}

extern "C" lcae_status lcae_dev_tma_selftest(const void *src, int rows, int cols, int box_rows, int r0, int c0,
                                             uint8_t *dump) {
  CUtensorMap m;
  if (!make_tmap_2d_bf16(&m, src, rows, cols, cols, box_rows)) { set_error("tensor map encode failed"); return LCAE_ERR_CUDA; }
  int smem = box_rows * 128 + 1024;
  LCAE_CK(cudaFuncSetAttribute(tma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  tma_selftest_kernel<<<1, 128, smem>>>(m, box_rows, r0, c0, dump);
  LCAE_CK(cudaGetLastError());
  LCAE_CK(cudaDeviceSynchronize());
  return LCAE_OK;
}

extern "C" lcae_status lcae_dev_red_probe(float *buf, int64_t n, int reps, int mode, int blocks, float *ms) {
  cudaEvent_t e0, e1;
  LCAE_CK(cudaEventCreate(&e0));
  LCAE_CK(cudaEventCreate(&e1));
  red_probe_kernel<<<blocks, 256>>>(buf, n, 1, mode);   // warm-up
  LCAE_CK(cudaEventRecord(e0));
  red_probe_kernel<<<blocks, 256>>>(buf, n, reps, mode);
  LCAE_CK(cudaEventRecord(e1));
  LCAE_CK(cudaEventSynchronize(e1));
  LCAE_CK(cudaEventElapsedTime(ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return LCAE_OK;
}

extern "C" lcae_status lcae_dev_tma_offset_selftest(const void *src, int rows, int cols, int box_rows, int r0, int c0,
                                                    int dst_row, uint8_t *dump) {
  CUtensorMap m;
  if (!make_tmap_2d_bf16(&m, src, rows, cols, cols, box_rows)) { set_error("tensor map encode failed"); return LCAE_ERR_CUDA; }
  int smem = 64 * 128 + 1024;
  LCAE_CK(cudaFuncSetAttribute(tma_offset_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  tma_offset_selftest_kernel<<<1, 128, smem>>>(m, box_rows, r0, c0, dst_row, dump);
  LCAE_CK(cudaGetLastError());
  LCAE_CK(cudaDeviceSynchronize());
  return LCAE_OK;
}

// ---- dev hook: the thread <- (lane, column) map of tcgen05.ld.16x256b.x2 (out: [4 warps][2 halves][32][8])
namespace lcae {
__global__ void __launch_bounds__(128) tmem_shape_kernel(uint32_t *out) {
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) ptx::tmem_alloc<32>(&tbase_s);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tb = tbase_s, tl = tb + ((uint32_t)(warp * 32) << 16);
  uint32_t r[16];
  for (int c = 0; c < 16; ++c) r[c] = ((uint32_t)(warp * 32 + lane) << 8) | (uint32_t)c;
  ptx::tmem_st16(tl, r);
  ptx::tmem_st_wait();
  __syncwarp();
  for (int h = 0; h < 2; ++h) {
    float v[8];
    ptx::tmem_ld_16x256b_x2(tl + ((uint32_t)(16 * h) << 16), v);
    ptx::tmem_ld_wait();
    for (int i = 0; i < 8; ++i) out[((warp * 2 + h) * 32 + lane) * 8 + i] = __float_as_uint(v[i]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<32>(tb);
}
}  // namespace lcae

extern "C" lcae_status lcae_dev_tmem_shape_selftest(uint32_t *host_out) {
  uint32_t *d = nullptr;
  LCAE_CK(cudaMalloc(&d, 4 * 2 * 32 * 8 * 4));
  tmem_shape_kernel<<<1, 128>>>(d);
  LCAE_CK(cudaGetLastError());
  LCAE_CK(cudaMemcpy(host_out, d, 4 * 2 * 32 * 8 * 4, cudaMemcpyDeviceToHost));
  cudaFree(d);
  return LCAE_OK;
}

