// mma_bench.cu — issue-rate / throughput of the backward kernel's tcgen05 MMA
// shapes on one SM (operands: whatever is in shared memory; timing only).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2510_18830_b200/csrc \
//        tools/mma_bench.cu -o /tmp/mma_bench && /tmp/mma_bench
#include <cstdio>
#include "sm100.cuh"
using namespace mt;

__global__ void __launch_bounds__(128, 1) bench(int variant, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // layout as attn_bwd: k 32K, v 32K, q 16K, dO 16K, pd 32K
  uint8_t *k = sm, *v = sm + 32768, *q = sm + 65536, *dO = sm + 81920, *pd = sm + 98304;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
  if (warp_id() == 0) tmem_alloc(smem_u32(&tbase), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp_id() == 0) {
    const bool leader = elect_one();
    const uint32_t id_s = make_idesc_bf16(128, 64, false, false);
    const uint32_t id_kv = make_idesc_bf16(128, 128, false, true);
    const uint32_t id_q = make_idesc_bf16(128, 64, true, true);
    const uint64_t dK = make_sdesc(smem_u32(k), 16, 1024), dV = make_sdesc(smem_u32(v), 16, 1024);
    const uint64_t dKmn = make_sdesc(smem_u32(k), 16384, 1024);
    const uint64_t dq = make_sdesc(smem_u32(q), 16, 1024), ddo = make_sdesc(smem_u32(dO), 16, 1024);
    const uint64_t dqm = make_sdesc(smem_u32(q), 8192, 1024), dom = make_sdesc(smem_u32(dO), 8192, 1024);
    const uint64_t dpt = make_sdesc(smem_u32(pd), 16, 1024), dst = make_sdesc(smem_u32(pd + 16384), 16, 1024);
    const uint64_t dstm = make_sdesc(smem_u32(pd + 16384), 8192, 1024);
    const long long t0 = clock64();
    if (leader) {
      for (int r = 0; r < reps; ++r) {
        if (variant == 0 || variant == 3) {
#pragma unroll
          for (int kk = 0; kk < 128; kk += 16) {
            const uint32_t ko = (kk >> 6) * 16384 + (kk & 63) * 2, qo = (kk >> 6) * 8192 + (kk & 63) * 2;
            mma_ss(tmem + 256, sdesc_add(dK, ko), sdesc_add(dq, qo), id_s, kk > 0);
            mma_ss(tmem + 320, sdesc_add(dV, ko), sdesc_add(ddo, qo), id_s, kk > 0);
          }
        }
        if (variant == 1 || variant == 3) {
#pragma unroll
          for (int kq = 0; kq < 64; kq += 16) {
            mma_ss(tmem + 128, sdesc_add(dpt, kq * 2), sdesc_add(dom, kq * 128), id_kv, 1);
            mma_ss(tmem + 0, sdesc_add(dst, kq * 2), sdesc_add(dqm, kq * 128), id_kv, 1);
          }
        }
        if (variant == 2 || variant == 3) {
#pragma unroll
          for (int kk = 0; kk < 128; kk += 16)
            mma_ss(tmem + 384, sdesc_add(dKmn, kk * 128), sdesc_add(dstm, kk * 128), id_q, kk > 0);
        }
        if (variant == 5 || variant == 6) {  // dV + dK with A = P^T / dS^T from TMEM (.ts), N = 128
#pragma unroll
          for (int kq = 0; kq < 64; kq += 16) {
            mma_ts(tmem + 128, tmem + 256 + kq / 2, sdesc_add(dom, kq * 128), id_kv, 1);
            mma_ts(tmem + 0, tmem + 288 + kq / 2, sdesc_add(dqm, kq * 128), id_kv, 1);
          }
        }
        if (variant == 6) {  // + S^T, dP^T, dQ^T: the backward's per-chunk sequence
#pragma unroll
          for (int kk = 0; kk < 128; kk += 16) {
            const uint32_t ko = (kk >> 6) * 16384 + (kk & 63) * 2, qo = (kk >> 6) * 8192 + (kk & 63) * 2;
            mma_ss(tmem + 320, sdesc_add(dK, ko), sdesc_add(dq, qo), id_s, kk > 0);
            mma_ss(tmem + 384, sdesc_add(dV, ko), sdesc_add(ddo, qo), id_s, kk > 0);
          }
#pragma unroll
          for (int kk = 0; kk < 128; kk += 16)
            mma_ss(tmem + 448, sdesc_add(dKmn, kk * 128), sdesc_add(dstm, kk * 128), id_q, kk > 0);
        }
        if (variant == 7) {  // issue rate: 32 tiny MMAs (M128 N8)
#pragma unroll
          for (int kk = 0; kk < 32; ++kk)
            mma_ss(tmem + 256, sdesc_add(dK, (kk & 3) * 32), sdesc_add(dq, (kk & 3) * 32),
                   make_idesc_bf16(128, 8, false, false), kk > 0);
        }
        if (variant == 8) {  // S^T with A = K from TMEM (.ts), N = 64
#pragma unroll
          for (int kk = 0; kk < 128; kk += 16)
            mma_ts(tmem + 256, tmem + 448 + kk / 2, sdesc_add(dq, (kk >> 6) * 8192 + (kk & 63) * 2), id_s, kk > 0);
        }
        if (variant == 9) {  // S^T + dP^T at M = 64 (one live 64-key slot), N = 64
#pragma unroll
          for (int kk = 0; kk < 128; kk += 16) {
            const uint32_t ko = (kk >> 6) * 16384 + (kk & 63) * 2, qo = (kk >> 6) * 8192 + (kk & 63) * 2;
            mma_ss(tmem + 256, sdesc_add(dK, ko), sdesc_add(dq, qo), make_idesc_bf16(64, 64, false, false), kk > 0);
            mma_ss(tmem + 320, sdesc_add(dV, ko), sdesc_add(ddo, qo), make_idesc_bf16(64, 64, false, false), kk > 0);
          }
        }
        if (variant == 4) {  // S^T only, K-major B but N=128 (two query blocks)
#pragma unroll
          for (int kk = 0; kk < 128; kk += 16) {
            const uint32_t ko = (kk >> 6) * 16384 + (kk & 63) * 2;
            mma_ss(tmem + 256, sdesc_add(dK, ko), sdesc_add(dV, ko), make_idesc_bf16(128, 128, false, false), kk > 0);
          }
        }
      }
      mma_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    const long long t1 = clock64();
    if (leader) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp_id() == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const char* names[] = {"S^T+dP^T (16x M128N64 KK)", "dV+dK (8x M128N128 K/MN)", "dQ^T (8x M128N64 MN/MN)",
                         "all per chunk (32 MMAs)", "S^T-like N128 KK (8x)", "dV+dK .ts (8x M128N128)",
                         "chunk: SS S/dP/dQ + ts dV/dK", "issue: 32x M128N8", "S^T .ts A=K (8x N64)",
                         "S^T+dP^T M64 (16x M64N64 KK)"};
  const double ideal[] = {16 * 32, 8 * 64, 8 * 32, 16 * 32 + 8 * 64 + 8 * 32, 8 * 64, 8 * 64,
                          24 * 32 + 8 * 64, 32 * 4, 8 * 32, 16 * 32};
  for (int grid : {1, 148}) {
    for (int v = 0; v < 10; ++v) {
      const int reps = 2000;
      bench<<<grid, 128, 140 * 1024>>>(v, reps, d);
      long long h[148];
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
      cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("grid %3d  %-28s %8.1f clk/iter  (floor %4.0f)  x%.2f\n", grid, names[v], mx / reps, ideal[v], mx / reps / ideal[v]);
    }
  }
  return 0;
}
