// selftest.cu — hardware self-tests for the tcgen05 / TMEM / TMA building blocks
// the attention kernels are made of.  Exported as mt_selftest_* test hooks (not
// part of the attention API): each runs one 128-row MMA configuration on one CTA
// so a descriptor or layout mistake shows up as a wrong small matrix, not as a
// wrong attention output.
//
// Variants (M = 128 always; D fp32 [128][N] row-major):
//   0: A K-major  [128][128], B K-major  [64][128]  -> D = A B^T        (S = Q K^T)
//   1: A K-major  [128][64],  B MN-major [64][128]  -> D = A B          (O += P V)
//   2: A MN-major [128k][128m], B MN-major [128k][64n] -> D = A^T B      (dQ^T = K^T dS^T)
//   3: A in TMEM  [128][64],  B MN-major [64][128]  -> D = A B          (P kept in TMEM)
//   4: as 0, but A/B staged by TMA from [256][2][128] tensors: A = X[128:256,1,:],
//      B = Y[64:128,0,:]
#include "sm100.cuh"
#include "tmap.cuh"
#include "../../include/mtsa.h"

using namespace mt;

namespace {

// Row-major global [rows][cols] bf16 -> SWIZZLE_128B smem tile stored as
// column chunks of 64 elements: chunk c at c*rows*128 bytes.
__device__ void stage_sw128(uint8_t* smem, const __nv_bfloat16* g, int rows, int cols) {
  const int pieces = rows * (cols / 8);
  for (int p = threadIdx.x; p < pieces; p += blockDim.x) {
    int r = p / (cols / 8), c16 = p % (cols / 8);
    int chunk = c16 / 8, c16i = c16 % 8;
    uint4 v = *reinterpret_cast<const uint4*>(g + (size_t)r * cols + c16 * 8);
    *reinterpret_cast<uint4*>(smem + chunk * rows * 128 + sw128(r, c16i)) = v;
  }
}

__global__ void __launch_bounds__(128, 1)
    selftest_mma_kernel(int variant, const __nv_bfloat16* A, const __nv_bfloat16* B, float* D,
                        const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                // 32 KB
  uint8_t* sB = smem + 32768;        // 32 KB
  __shared__ uint64_t bar_mma, bar_tma;
  __shared__ uint32_t tmem_base_s;

  const int warp = warp_id();
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar_mma), 1);
    mbar_init(smem_u32(&bar_tma), 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tmem_base_s), 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  int N = 64, K = 128;
  bool a_mn = false, b_mn = false;
  if (variant == 0 || variant == 4) { N = 64; K = 128; }
  if (variant == 1 || variant == 3) { N = 128; K = 64; b_mn = true; }
  if (variant == 2) { N = 64; K = 128; a_mn = true; b_mn = true; }

  if (variant == 4) {
    if (threadIdx.x == 0) {
      const uint32_t bar = smem_u32(&bar_tma);
      mbar_expect_tx(bar, 128 * 128 * 2 + 64 * 128 * 2);
      // A: rows 128..255 of head 1, two 64-row boxes x two 64-col chunks.
      for (int ch = 0; ch < 2; ++ch)
        for (int rb = 0; rb < 2; ++rb)
          tma_load_3d(smem_u32(sA + ch * 128 * 128 + rb * 64 * 128), &tmA, bar, ch * 64, 1,
                      128 + rb * 64);
      for (int ch = 0; ch < 2; ++ch)
        tma_load_3d(smem_u32(sB + ch * 64 * 128), &tmB, bar, ch * 64, 0, 64);
    }
    mbar_wait(smem_u32(&bar_tma), 0);
  } else {
    if (variant == 0) { stage_sw128(sA, A, 128, 128); stage_sw128(sB, B, 64, 128); }
    if (variant == 1) { stage_sw128(sA, A, 128, 64);  stage_sw128(sB, B, 64, 128); }
    if (variant == 2) { stage_sw128(sA, A, 128, 128); stage_sw128(sB, B, 128, 64); }
    if (variant == 3) {
      stage_sw128(sB, B, 64, 128);
      // A row m -> TMEM lane m, columns 128..159 (bf16 pairs).
      uint32_t r[32];
      const int m = threadIdx.x;
      for (int c = 0; c < 32; ++c) {
        float lo = __bfloat162float(A[m * 64 + 2 * c]);
        float hi = __bfloat162float(A[m * 64 + 2 * c + 1]);
        r[c] = pack_bf16x2(lo, hi);
      }
      tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + 128, r);
      tmem_st_wait();
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_bf16(128, N, a_mn, b_mn);
    for (int k0 = 0; k0 < K; k0 += 16) {
      uint64_t ad, bd;
      // A
      if (!a_mn) ad = make_sdesc(smem_u32(sA) + (k0 / 64) * 128 * 128 + (k0 % 64) * 2, 16, 1024);
      else       ad = make_sdesc(smem_u32(sA) + k0 * 128, K * 128, 1024);
      // B
      if (!b_mn) bd = make_sdesc(smem_u32(sB) + (k0 / 64) * N * 128 + (k0 % 64) * 2, 16, 1024);
      else       bd = make_sdesc(smem_u32(sB) + k0 * 128, K * 128, 1024);
      if (variant == 3)
        mma_ts(tmem, tmem + 128 + k0 / 2, bd, idesc, k0 > 0);
      else
        mma_ss(tmem, ad, bd, idesc, k0 > 0);
    }
    mma_commit(smem_u32(&bar_mma));
  }
  mbar_wait(smem_u32(&bar_mma), 0);
  tc_fence_after();

  const int row = warp * 32 + lane_id();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) D[row * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

}  // namespace

extern "C" mt_status mt_selftest_mma(int variant, const void* A, const void* B, float* D,
                                     cudaStream_t stream) {
  CUtensorMap tmA{}, tmB{};
  if (variant == 4) {
    if (make_tmap_bf16_3d(&tmA, A, 128, 2, 256, 64, 1, 64) != 0) return MT_ECUDA;
    if (make_tmap_bf16_3d(&tmB, B, 128, 2, 256, 64, 1, 64) != 0) return MT_ECUDA;
  }
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(selftest_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  selftest_mma_kernel<<<1, 128, smem, stream>>>(variant, (const __nv_bfloat16*)A,
                                                (const __nv_bfloat16*)B, D, tmA, tmB);
  return cudaGetLastError() == cudaSuccess ? MT_OK : MT_ECUDA;
}
