// xattn_score.cu — XAttention antidiagonal block scores (PAPER.md P:826,
// reading R25), hand-written for sm_100a: the strided score contraction on tcgen05 with
// the row softmax and the 8 x 8 block sums fused behind it, so the n x n score matrix is
// never written.
//
// Per q head h (kv head h / grp), stride st = 16, n = S / 16 stride rows:
//   A[i][j] = Qr[i] . Kr[j] / (st sqrt d)   (Qr, Kr: 2048-wide reshaped rows, xattn.cu)
//   Bs[I][J] = sum_{i in I, j in J} softmax_{j <= i}(A[i][.])_j      (I, J: 8 stride rows)
// Tiles: 128 stride rows (16 query blocks) x 256 stride columns (M = 128, N = 256: the
// 2048-deep contraction moves (128 + 256) x 2048 x 2 bytes per tile, so wider tiles cut
// the operand traffic per flop), K = 2048 streamed by TMA in 64-wide chunks (SW128) through
// a 4-stage ring; the accumulator is double-buffered in TMEM (2 x 256 columns).  A CTA
// walks one row tile's column tiles in order, as 128-column halves C = 0 .. R, and its 4
// epilogue warps (thread = stride row = TMEM lane) keep the running max / sum of their row
// (online softmax, log2 domain) and write
//   P[r][J] = sum_{j in J} 2^(A log2e - m_C)   and   Mt[r][C] = m_C
// (m_C: the running max after tile C) to a per-CTA scratch.  After the diagonal tile the
// same warps combine their row tile:
//   Bs[I][J] = sum_{r in I} P[r][J] 2^(Mt[r][J/16] - m_r) / l_r
// Work items (head, row tile) are dealt in descending row-tile order, snake-wise over the
// persistent CTAs (the work of a row tile is proportional to R + 1).  Default: clusters of
// two CTAs take row tiles 2j + 1 and 2j and share every B tile (each loads one 128-row
// half and multicasts it; a stage is refilled once both CTAs' MMAs released it), which
// halves the B traffic (MT_XATTN_PAIR=0: one CTA per row tile).
// Warp roles: 0 TMA, 1 MMA (one elected lane), 2-5 epilogue.
#include <cuda_bf16.h>

#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace mt {
namespace xs {

constexpr int kStages = 4;
constexpr int kChunk = 64;            // K elements per stage
constexpr int kKChunks = 2048 / kChunk;
constexpr int kN = 256;               // stride columns per MMA tile (two 128-column halves)
constexpr uint32_t kTileA = 128 * kChunk * 2;  // 16 KB per stage
constexpr uint32_t kTileB = kN * kChunk * 2;   // 32 KB per stage
constexpr int kThreads = 192;

struct Smem {
  uint8_t a[kStages][kTileA];
  uint8_t b[kStages][kTileB];
  uint64_t full[kStages], empty[kStages];
  uint64_t tfull[2], tempty[2];
  float fm[128], fl[128];  // final row max (log2) / sum of the item
  uint32_t tmem_base;
};

struct Params {
  int64_t n;        // stride rows (= stride columns) per head
  int nrt;          // row tiles = ceil(n / 128)
  int nI;           // query blocks = S / 128
  int hb;           // q heads in this launch
  int h0;           // first q head of the launch (global)
  int grp;          // q heads per kv head
  float scale_log2; // log2(e) / (st sqrt d)
  int ldp;          // P row stride: 16 nrt (16-byte aligned rows)
  float* P;         // per CTA: [128][ldp]
  float* Mt;        // per CTA: [128][nrt]
  float* tri;       // [Hq][nI (nI + 1) / 2] block scores, row I at I (I + 1) / 2
  int64_t T;        // nI (nI + 1) / 2
};

// item k of this CTA: the snake-dealt k-th item; items sorted by descending row tile.
// kPair: CTAs come in clusters of two that take row tiles 2j + 1 and 2j of one head (both
// walk column tiles 0 .. j) and share each 256-row B tile, every CTA loading one half and
// multicasting it to both (a row tile past the end computes masked rows only).
template <bool kPair>
__device__ __forceinline__ bool item_of(const Params& p, int k, int& hh, int& R) {
  const int G = kPair ? (int)gridDim.x / 2 : (int)gridDim.x;
  const int me = kPair ? (int)blockIdx.x / 2 : (int)blockIdx.x;
  const int i = k * G + ((k & 1) ? G - 1 - me : me);
  const int nu = kPair ? (p.nrt + 1) / 2 : p.nrt;
  if (i >= p.hb * nu) return false;
  hh = i % p.hb;
  if (kPair)
    R = 2 * (nu - 1 - i / p.hb) + 1 - (int)(blockIdx.x & 1);
  else
    R = p.nrt - 1 - i / p.hb;
  return true;
}

__device__ __forceinline__ void tma_load_3d_mc(uint32_t dst, const void* tmap, uint32_t bar, int c0,
                                               int c1, int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <bool kPair>
__global__ void __launch_bounds__(kThreads, 1)
    xattn_score_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap tma,
                       const __grid_constant__ CUtensorMap tmb) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // SW128 operand tiles need 1024-byte alignment: the launch reserves 1 KB of slack
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(smem_u32(&sm.full[s]), 1);
      mbar_init(smem_u32(&sm.empty[s]), kPair ? 2 : 1);  // kPair: both CTAs' MMAs read the stage
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&sm.tfull[b]), 1);
      mbar_init(smem_u32(&sm.tempty[b]), 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(smem_u32(&sm.tmem_base), 2 * kN);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tma);
    tma_prefetch_desc(&tmb);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kPair) cluster_sync_all();  // the peer's barriers are initialised
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int crank = kPair ? (int)(blockIdx.x & 1) : 0;

  if (warp == 0) {
    // ---- TMA producer
    uint32_t it = 0;
    int hh, R;
    for (int k = 0; item_of<kPair>(p, k, hh, R); ++k) {
      const int kvh = (p.h0 + hh) / p.grp;
      const int rmax = kPair ? (R | 1) : R;  // the pair walks the odd row tile's columns
      for (int C2 = 0; 2 * C2 <= rmax; ++C2)
        for (int kc = 0; kc < kKChunks; ++kc, ++it) {
          const uint32_t s = it % kStages;
          mbar_wait(smem_u32(&sm.empty[s]), ((it / kStages) & 1) ^ 1);
          if (lane == 0) {
            const uint32_t bar = smem_u32(&sm.full[s]);
            mbar_expect_tx(bar, kTileA + kTileB);
            tma_load_3d(smem_u32(sm.a[s]), &tma, bar, kc * kChunk, R * 128, hh);
            if constexpr (kPair)  // this CTA's half of B, to both CTAs of the pair
              tma_load_3d_mc(smem_u32(sm.b[s]) + crank * (kTileB / 2), &tmb, bar, kc * kChunk,
                             C2 * kN + crank * (kN / 2), kvh, (uint16_t)3);
            else
              tma_load_3d(smem_u32(sm.b[s]), &tmb, bar, kc * kChunk, C2 * kN, kvh);
          }
          __syncwarp();
        }
    }
  } else if (warp == 1) {
    // ---- MMA issuer
    const bool leader = elect_one();
    constexpr uint32_t idesc = make_idesc_bf16(128, kN, false, false);
    uint32_t it = 0, tile = 0;
    int hh, R;
    for (int k = 0; item_of<kPair>(p, k, hh, R); ++k) {
      const int rmax = kPair ? (R | 1) : R;
      for (int C2 = 0; 2 * C2 <= rmax; ++C2, ++tile) {
        const uint32_t b = tile & 1;
        mbar_wait(smem_u32(&sm.tempty[b]), ((tile >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + kN * b;
        for (int kc = 0; kc < kKChunks; ++kc, ++it) {
          const uint32_t s = it % kStages;
          mbar_wait(smem_u32(&sm.full[s]), (it / kStages) & 1);
          tc_fence_after();
          if (leader) {
            const uint64_t da = make_sdesc(smem_u32(sm.a[s]), 16, 1024);
            const uint64_t db = make_sdesc(smem_u32(sm.b[s]), 16, 1024);
#pragma unroll
            for (int kk = 0; kk < kChunk; kk += 16)
              mma_ss(d, sdesc_add(da, kk * 2), sdesc_add(db, kk * 2), idesc, (kc | kk) ? 1u : 0u);
            if constexpr (kPair)
              mma_commit_mc(smem_u32(&sm.empty[s]), (uint16_t)3);  // frees the stage in both CTAs
            else
              mma_commit(smem_u32(&sm.empty[s]));
          }
          __syncwarp();
        }
        if (leader) mma_commit(smem_u32(&sm.tfull[b]));
        __syncwarp();
      }
    }
  } else {
    // ---- epilogue: thread = stride row of the tile = TMEM lane 32 (warp % 4) + lane
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int et = threadIdx.x - 64;  // 0..127 over the 4 epilogue warps
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    float* P = p.P + (size_t)blockIdx.x * 128 * p.ldp;
    float* Mt = p.Mt + (size_t)blockIdx.x * 128 * p.nrt;
    uint32_t tile = 0;
    int hh, R;
    for (int k = 0; item_of<kPair>(p, k, hh, R); ++k) {
      const int64_t grow = (int64_t)R * 128 + r;  // this thread's stride row
      const int rmax = kPair ? (R | 1) : R;
      float m = -INFINITY, l = 0.f;
      for (int C2 = 0; 2 * C2 <= rmax; ++C2, ++tile) {
        const uint32_t b = tile & 1;
        mbar_wait(smem_u32(&sm.tfull[b]), (tile >> 1) & 1);
        tc_fence_after();
        for (int half = 0; half < 2; ++half) {  // 128-column halves C = 2 C2 + half
          const int C = 2 * C2 + half;
          if (C > R) break;  // beyond the diagonal tile: nothing valid
          uint32_t v[4][32];
#pragma unroll
          for (int g = 0; g < 4; ++g)
            tmem_ld32(tmem + lane_base + kN * b + 128 * half + 32 * g, v[g]);
          tmem_ld_wait();
          // valid columns: j <= i (causal, the diagonal tile) and j < n
          const int64_t c0 = (int64_t)C * 128;
          int lim = (int)min((int64_t)127, min(grow, p.n - 1) - c0);  // last valid column
          if (grow >= p.n) lim = -1;
          float tmax = -INFINITY;
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (32 * g + c <= lim) tmax = fmaxf(tmax, __uint_as_float(v[g][c]) * p.scale_log2);
          const float mn = fmaxf(m, tmax);
          float part[16];
          float s = 0.f;
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              float acc = 0.f;
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const int col = 32 * g + 8 * jj + c;
                const float e = col <= lim ? exp2f(__uint_as_float(v[g][8 * jj + c]) * p.scale_log2 - mn) : 0.f;
                acc += e;
              }
              part[4 * g + jj] = acc;
              s += acc;
            }
          l = (m == -INFINITY ? 0.f : l * exp2f(m - mn)) + s;
          m = mn;
          if (grow < p.n) {
            float4* dst = reinterpret_cast<float4*>(P + (size_t)r * p.ldp + 16 * C);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              dst[u] = make_float4(part[4 * u], part[4 * u + 1], part[4 * u + 2], part[4 * u + 3]);
            Mt[(size_t)r * p.nrt + C] = mn;
          }
        }
        tc_fence_before();
        mbar_arrive(smem_u32(&sm.tempty[b]));  // the accumulator may be overwritten
      }
      // ---- combine the row tile: Bs[I][J] for its 16 query blocks, J <= I
      sm.fm[r] = m;
      sm.fl[r] = l;
      named_bar_sync(1, 128);  // P / Mt rows of every thread of the tile written
      float* tri = p.tri + (size_t)(p.h0 + hh) * p.T;
      for (int ib = 0; ib < 16; ++ib) {
        const int I = R * 16 + ib;
        if (I >= p.nI) break;
        float* out = tri + (size_t)I * (I + 1) / 2;
        for (int J = et; J <= I; J += 128) {
          float acc = 0.f;
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) {
            const int row = 8 * ib + rr;
            const float lr = sm.fl[row];
            if (lr > 0.f)
              acc += P[(size_t)row * p.ldp + J] * exp2f(Mt[(size_t)row * p.nrt + J / 16] - sm.fm[row]) / lr;
          }
          out[J] = acc;
        }
      }
      named_bar_sync(1, 128);  // scratch free for the next item
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kPair) cluster_sync_all();  // no multicast or remote arrive is still in flight
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 2 * kN);
}

}  // namespace xs

size_t xattn_score_scratch_bytes(int64_t n, int nI, int num_sms) {
  const int nrt = (int)((n + 127) / 128);
  (void)nI;
  return (size_t)num_sms * 128 * ((size_t)16 * nrt + nrt) * 4;
}

// Block scores of q heads [h0, h0 + hb) into tri (layout above).  qr: [hb][n][2048] bf16
// (reversed stride rows of those heads), kr: [Hkv][n][2048] bf16, scratch: see above.
mt_status xattn_scores_tc(const void* qr, const void* kr, int64_t n, int nI, int hb, int h0,
                          int Hkv, int grp, float scale_log2, float* tri, int64_t T,
                          void* scratch, int num_sms, cudaStream_t st) {
  using namespace xs;
  Params p{};
  p.n = n;
  p.nrt = (int)((n + 127) / 128);
  p.nI = nI;
  p.hb = hb;
  p.h0 = h0;
  p.grp = grp;
  p.scale_log2 = scale_log2;
  p.ldp = 16 * p.nrt;
  p.P = static_cast<float*>(scratch);
  p.Mt = p.P + (size_t)num_sms * 128 * p.ldp;
  p.tri = tri;
  p.T = T;
  // MT_XATTN_PAIR=0: one CTA per row tile, each loading its whole B tile (A/B switch)
  static const bool pair = !getenv("MT_XATTN_PAIR") || atoi(getenv("MT_XATTN_PAIR"));
  CUtensorMap ta, tb;
  if (make_tmap_bf16_3d(&ta, qr, 2048, (uint64_t)n, (uint64_t)hb, kChunk, 128, 1) ||
      make_tmap_bf16_3d(&tb, kr, 2048, (uint64_t)n, (uint64_t)Hkv, kChunk, pair ? kN / 2 : kN, 1))
    return fail(MT_ECUDA, "cuTensorMapEncodeTiled (xattn scores) failed");
  const size_t smem = sizeof(Smem) + 1024;
  if (p.ldp < 0) return fail(MT_ESHAPE, "xattn scores: bad shape");
  if (pair) {
    if (cudaFuncSetAttribute(xattn_score_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return fail(MT_ECUDA, "cudaFuncSetAttribute(xattn_score_kernel) failed");
    const int units = hb * ((p.nrt + 1) / 2);
    int pairs = num_sms / 2;
    if (units < pairs) pairs = units;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, xattn_score_kernel<true>, p, ta, tb) != cudaSuccess)
      return fail(MT_ECUDA, "cudaLaunchKernelEx(xattn_score_kernel, cluster 2) failed");
    return check_launch("xattn_score_kernel");
  }
  if (cudaFuncSetAttribute(xattn_score_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return fail(MT_ECUDA, "cudaFuncSetAttribute(xattn_score_kernel) failed");
  const int items = hb * p.nrt;
  const int grid = items < num_sms ? items : num_sms;
  xattn_score_kernel<false><<<grid, kThreads, smem, st>>>(p, ta, tb);
  return check_launch("xattn_score_kernel");
}

}  // namespace mt
