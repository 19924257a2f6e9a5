// tmem_bench.cu — tcgen05.ld (TMEM -> registers) throughput on one SM and on all 148:
// W warps (W/4 per lane quarter) each load 32 lanes x 32 columns (4 KB) per iteration.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2510_18830_b200/csrc \
//        tools/tmem_bench.cu -o tools/tmem_bench.bin
#include <cstdio>
#include "sm100.cuh"
using namespace mt;

__global__ void __launch_bounds__(512, 1) bench(int reps, int ncols_per_ld, long long* out, float* sink) {
  __shared__ uint32_t tbase;
  if (warp_id() == 0) tmem_alloc(smem_u32(&tbase), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const int w = warp_id(), quad = w & 3, grp = w >> 2;
  const uint32_t lb = (uint32_t)(quad * 32) << 16;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint32_t v[32];
    const uint32_t col = (uint32_t)((grp * 64 + (r & 3) * 32 + 128 * (r & 1)) & 511) & ~31u;
    tmem_ld32(tmem + lb + col, v);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += __uint_as_float(v[i]);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp_id() == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  float* s;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaMalloc(&s, 148 * 512 * sizeof(float));
  for (int threads : {128, 256, 512}) {
    for (int grid : {1, 148}) {
      const int reps = 4096;
      bench<<<grid, threads>>>(reps, 32, d, s);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
      long long h[148];
      cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      const double bytes = (double)reps * (threads / 32) * 4096.0;
      printf("warps %2d grid %3d: %8.1f clk per round of %d x 4 KB loads -> %6.1f B/clk/SM\n", threads / 32,
             grid, mx / reps, threads / 32, bytes / mx);
    }
  }
  return 0;
}
