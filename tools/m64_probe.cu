// m64_probe.cu — where does a cta_group::1 M = 64 tcgen05.mma put its 64 result rows in
// TMEM, and does the D address's lane field move them?  A[r][0] = r + 1, B[n][0] = 1, all
// other K entries 0, so D[r][n] = r + 1; each case zeroes TMEM, issues one MMA (N = 32,
// K = 16) and dumps lanes 0..127 x column 0.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2510_18830_b200/csrc \
//        tools/m64_probe.cu -o /tmp/m64_probe && /tmp/m64_probe
#include <cstdio>
#include <cuda_bf16.h>
#include "sm100.cuh"
using namespace mt;

__device__ uint32_t sw128(int row, int k) {  // byte offset of bf16 (row, k) in a SW128 K-major tile
  const int chunk = (k * 2) / 16;
  return (uint32_t)((row / 8) * 1024 + (row % 8) * 128 + ((chunk ^ (row % 8)) * 16) + (k * 2) % 16);
}

__global__ void __launch_bounds__(128, 1) probe(int M, int dlane, int arow, int ncols_probe, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *a = sm, *b = sm + 16384;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 24576 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  __syncthreads();
  if (threadIdx.x < 128) {
    const int r = threadIdx.x;
    *reinterpret_cast<__nv_bfloat16*>(a + sw128(r, 0)) = __float2bfloat16((float)(r + 1));
    if (r < 64) *reinterpret_cast<__nv_bfloat16*>(b + sw128(r, 0)) = __float2bfloat16(1.f);
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
  if (warp_id() == 0) tmem_alloc(smem_u32(&tbase), 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const int w = warp_id();
  {
    uint32_t z[32];
    for (int c = 0; c < 32; ++c) z[c] = 0;
    const uint32_t lb = (uint32_t)(w * 32) << 16;
    tmem_st32(tmem + lb, z);
    tmem_st32(tmem + lb + 32, z);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) {
    if (elect_one()) {
      const uint64_t ad = make_sdesc(smem_u32(a) + arow * 128, 16, 1024);
      const uint64_t bd = make_sdesc(smem_u32(b), 16, 1024);
      mma_ss(tmem + ((uint32_t)dlane << 16), ad, bd, make_idesc_bf16(M, 32, false, false), 0);
      mma_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
  }
  __syncthreads();
  tc_fence_after();
  {
    uint32_t v[32];
    tmem_ld32(tmem + ((uint32_t)(w * 32) << 16), v);
    tmem_ld_wait();
    const int lane = w * 32 + (threadIdx.x & 31);
    for (int c = 0; c < ncols_probe; ++c) out[lane * ncols_probe + c] = __uint_as_float(v[c]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc(tmem, 128);
}

int main() {
  float* d;
  const int nc = 32;
  cudaMalloc(&d, 128 * nc * sizeof(float));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  struct Case { int M, dlane, arow; } cases[] = {{128, 0, 0}, {64, 0, 0}, {64, 0, 64}, {64, 64, 0},
                                                  {64, 32, 0}, {64, 16, 0}, {64, 96, 0}};
  for (auto c : cases) {
    cudaMemset(d, 0xff, 128 * nc * sizeof(float));
    probe<<<1, 128, 40 * 1024>>>(c.M, c.dlane, c.arow, nc, d);
    cudaError_t e = cudaDeviceSynchronize();
    printf("M=%d dlane=%d arow=%d: %s\n", c.M, c.dlane, c.arow, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    float h[128 * nc];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    // per lane: value in column 0, and how many of the 32 columns equal it
    for (int l = 0; l < 128; ++l) {
      int same = 0;
      for (int cc = 0; cc < nc; ++cc) same += h[l * nc + cc] == h[l * nc];
      printf("%s%3d:%g/%d", l % 8 ? " " : "\n  ", l, h[l * nc], same);
    }
    printf("\n");
  }
  return 0;
}
