// gather4_check.cu — does TMA tile::gather4 place 4 gathered rows in the same
// SWIZZLE_128B layout as our manual sw128() staging, for 512-B aligned
// destinations inside a 1024-B pattern?  Byte compare on one CTA.
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2510_18830_b200/csrc \
//        tools/gather4_check.cu -o /tmp/g4 -lcuda && /tmp/g4
#include <cstdio>
#include <vector>
#include <cudaTypedefs.h>
#include "sm100.cuh"
using namespace mt;

__global__ void k(const __grid_constant__ CUtensorMap tm, const int* rows, const uint16_t* g,
                  int ncols_total, int col0, int* bad) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* a = sm_raw;            // gather4 result   [128 rows][128 B]
  uint8_t* b = sm_raw + 16384;    // manual result
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(smem_u32(&bar), 16384);
    for (int r = 0; r < 128; r += 4)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(a + r * 128)), "l"(&tm),
          "r"(col0), "r"(rows[r]), "r"(rows[r + 1]), "r"(rows[r + 2]), "r"(rows[r + 3]),
          "r"(smem_u32(&bar))
          : "memory");
  }
  for (int p = threadIdx.x; p < 128 * 8; p += blockDim.x) {
    const int r = p >> 3, c16 = p & 7;
    const uint4 v = *reinterpret_cast<const uint4*>(g + (size_t)rows[r] * ncols_total + col0 + c16 * 8);
    *reinterpret_cast<uint4*>(b + sw128(r, c16)) = v;
  }
  mbar_wait(smem_u32(&bar), 0);
  __syncthreads();
  int nb = 0;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) nb += a[i] != b[i];
  atomicAdd(bad, nb);
}

int main() {
  const int T = 4096, C = 2 * 128;  // tokens x (Hkv=2 x d=128)
  std::vector<uint16_t> h((size_t)T * C);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i * 2654435761u >> 7);
  std::vector<int> rows(128);
  for (int r = 0; r < 128; ++r) rows[r] = (r * 977 + 13) % T;
  uint16_t* dg; int *dr, *dbad;
  cudaMalloc(&dg, h.size() * 2); cudaMalloc(&dr, 128 * 4); cudaMalloc(&dbad, 4);
  cudaMemcpy(dg, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, rows.data(), 128 * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  int fails = 0;
  for (int col0 : {0, 64, 128, 192}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)T};
    cuuint64_t strides[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dg, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    cudaMemset(dbad, 0, 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    k<<<1, 256, 40000>>>(tm, dr, dg, C, col0, dbad);
    cudaError_t e = cudaDeviceSynchronize();
    int bad = -1;
    cudaMemcpy(&bad, dbad, 4, cudaMemcpyDeviceToHost);
    printf("col0=%d err=%s mismatched bytes=%d\n", col0, cudaGetErrorString(e), bad);
    fails += bad != 0 || e != cudaSuccess;
  }
  printf(fails ? "GATHER4 LAYOUT MISMATCH\n" : "gather4 layout == sw128 staging\n");
  return fails != 0;
}
