// issue_bench.cu — how long the issuing thread spends in tcgen05.mma issue (not execution):
// clock64 around the issue of n MMAs behind a long-running MMA batch, then around the wait.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2510_18830_b200/csrc \
//        tools/issue_bench.cu -o /tmp/issue_bench && /tmp/issue_bench
#include <cstdio>
#include "sm100.cuh"
using namespace mt;

__global__ void __launch_bounds__(128, 1) bench(int n, int pre, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
  if (warp_id() == 0) tmem_alloc(smem_u32(&tbase), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp_id() == 0 && elect_one()) {
    const uint64_t a = make_sdesc(smem_u32(sm), 16, 1024), b = make_sdesc(smem_u32(sm + 32768), 16, 1024);
    const uint32_t big = make_idesc_bf16(128, 256, false, false), small = make_idesc_bf16(128, 64, false, false);
    for (int i = 0; i < pre; ++i) mma_ss(tmem, a, b, big, 1);  // keep the pipe busy (128 clk each)
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) mma_ss(tmem + 256, sdesc_add(a, (i & 3) * 32), sdesc_add(b, (i & 3) * 32), small, i > 0);
    const long long t1 = clock64();
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    const long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t1;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp_id() == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 2 * sizeof(long long));
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int pre : {0, 4, 32})
    for (int n : {1, 4, 8, 16, 32, 64}) {
      bench<<<1, 128, 80 * 1024>>>(n, pre, d);
      long long h[2];
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("pre %2d  n %2d  issue %6lld clk (%5.1f / MMA)  drain %6lld clk\n", pre, n, h[0], (double)h[0] / n, h[1]);
    }
  return 0;
}
