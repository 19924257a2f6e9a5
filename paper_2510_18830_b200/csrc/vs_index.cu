// vs_index.cu — Alg. 1 "Dynamic Sparse Training Head" index on the GPU
// (PAPER.md P:213-232), in the VS-IDX v1 arithmetic of DESIGN.md §2.1
// so that it is bit-identical to the CPU oracle and independent of the number
// of ranks the keys are striped over:
//   stage1  I1-I2  t = fold_c fma(q, k, acc) (exact bf16 products, one RN per
//                  add), causal mask, row max (order-free)
//   stage2  I3-I4  e = exp2s(RN(RN(t - M) * C_d)) with a specified polynomial
//                  (no MUFU ex2, no FMA contraction); E = sum floor(e 2^31) (uint64)
//   stage3  I5-I6  w = floor(RN(e / l) 2^32); V_m = sum_i w; P_kb = sum_{m in kb} V_m;
//                  sort keys (score desc, index asc) packed into uint64
//   select  I7-I8  one radix sort of every head's keys (head id in the top key
//                  bits, so each head's keys come out contiguous and in (score
//                  desc, index asc) order), exact integer top-p, forced members,
//                  ascending compaction -> i_v, i_s
// The window scoring is deliberately on CUDA cores in fp32: the tensor cores'
// accumulation order is unspecified, which would break bit-exactness
// ("what differs from the paper").
#include <cub/cub.cuh>
#include <cstdlib>

#include "common.cuh"
#include "f32x2.cuh"
#include "plan.cuh"
#include "rope.cuh"
#include "vsidx.cuh"

namespace mt {

int device_num_sms();

namespace vsi {

constexpr int kThreads = 256;   // keys per CTA in stages 1-3
constexpr int kScoreBits = 39;  // V_m, P_kb <= 64 * 2^32 * (1 + 2^-9) < 2^39

// Sort-key layout: key = (h << (kScoreBits + ib)) | ((2^39 - 1 - score) << ib) | index,
// ib = bits of the largest index; hb = head bits, 0 when they do not fit in 64 bits
// (then each head is sorted on its own).
struct KeyLayout {
  int ib, hb;
};
__host__ __device__ inline int bits_for(int64_t n) {  // bits of the values 0..n-1, >= 1
  int b = 1;
  while ((1LL << b) < n) ++b;
  return b;
}
inline KeyLayout key_layout(int64_t n, int Hq) {
  // MT_VS_SORT_PER_HEAD=1 forces the per-head sorts (the equality test of both paths)
  static const bool per_head = getenv("MT_VS_SORT_PER_HEAD") && atoi(getenv("MT_VS_SORT_PER_HEAD"));
  const int ib = bits_for(n), hb = bits_for(Hq);
  return {ib, !per_head && kScoreBits + ib + hb <= 64 ? hb : 0};
}

__constant__ uint32_t kExp2CoefBits[8] = {0x3F800000u, 0x3F317218u, 0x3E75FDF0u, 0x3D635847u,
                                          0x3C1D955Bu, 0x3AAEC3FFu, 0x39218489u, 0x377FE5FEu};
constexpr uint32_t kCdBits = 0x3E0293EEu;  // RN(log2(e) / sqrt(128))

struct Geo {
  int64_t S;      // global
  int64_t S_loc;  // local keys
  int Hq, Hkv, W, r;
  int layout, zc;  // sequence layout of the ranks (plan.cuh)
};

__device__ __forceinline__ int64_t global_col(const Geo& g, int64_t m_loc) {
  return (int64_t)layout_l2g(g.layout, g.W, g.zc, g.r, (int)(m_loc >> 6)) * 64 + (m_loc & 63);
}

// I3: specified 2^y (y <= 0), every operation one IEEE RN op.
__device__ __forceinline__ float exp2s(float y) {
  if (!(y >= -125.0f)) return 0.0f;
  const float j = rintf(y);
  const float f = __fsub_rn(y, j);
  float p = __uint_as_float(kExp2CoefBits[7]);
#pragma unroll
  for (int c = 6; c >= 0; --c) p = __fadd_rn(__fmul_rn(p, f), __uint_as_float(kExp2CoefBits[c]));
  const int ji = (int)j;
  return __fmul_rn(p, __int_as_float((ji + 127) << 23));
}

__device__ __forceinline__ void atomic_max_f32(float* a, float v) {
  if (v >= 0.f)
    atomicMax(reinterpret_cast<int*>(a), __float_as_int(v));
  else
    atomicMin(reinterpret_cast<unsigned*>(a), __float_as_uint(v));
}

__device__ __forceinline__ uint64_t shfl_down_u64(uint64_t v, int o) {
  uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  lo = __shfl_down_sync(0xffffffffu, lo, o);
  hi = __shfl_down_sync(0xffffffffu, hi, o);
  return ((uint64_t)hi << 32) | lo;
}

// ---------------------------------------------------------------- stage 1
// t[h][i][m] (fp32) and row max M[h][i].  Thread = key m.  Each accumulator still
// folds c = 0..127 in order (I1); the loops only tile it: 32 window rows per pass
// (32 accumulators) x 32 k values per block in registers, ~80 registers, so three
// CTAs (24 warps) share an SM to hide the shared-memory broadcast latency
// (kMinBlocks = 3: 80 registers; 2: 128 registers, no spill; MT_VS_S1_MINB picks).
//
// kRope (f3 upstream fusion, mt_rope_vs_index): k holds PRE-RoPE rows; each thread
// rotates its key row once (rope.cuh, the arithmetic of mt_rope, so the bf16 values are
// the same bits) into dynamic shared memory, the fold reads it from there, and the first
// CTA of the kv group (q head h % grp == 0, z == 0) writes the rotated row to k_out.
constexpr int kRows = 32, kKB = 32;
constexpr size_t kRopeSmem = (size_t)16 * kThreads * 16;  // 128 bf16 per key row
template <int kMinBlocks, bool kRope>
__global__ void __launch_bounds__(kThreads, kMinBlocks) stage1_scores(Geo g, const __nv_bfloat16* qwin,
                                                             const __nv_bfloat16* k, float* t,
                                                             float* M,
                                                             const __grid_constant__ RopeArgs ra,
                                                             __nv_bfloat16* k_out) {
  // window queries as row pairs: qs2[i / 2][c][i % 2], so one 16-byte load gives rows (i, i + 1)
  // at columns c and c + 1 for two packed f32x2 FMAs (FFMA2: per lane the same IEEE fma)
  __shared__ __align__(16) float qs2[32][128][2];
  __shared__ float wmax[kThreads / 32][64];
  extern __shared__ __align__(16) uint4 krot[];  // kRope: [16][kThreads] rotated rows
  const int h = blockIdx.y;
  const int grp = g.Hq / g.Hkv;
  // window rows [rlo, rhi) of this CTA: gridDim.z splits the 64 rows at short lengths
  const int rlo = blockIdx.z * (64 / gridDim.z), rhi = rlo + 64 / gridDim.z;
  for (int e = threadIdx.x + rlo * 128; e < rhi * 128; e += kThreads) {
    const int i = e >> 7, c = e & 127;
    qs2[i >> 1][c][i & 1] = __bfloat162float(qwin[((size_t)i * g.Hq + h) * 128 + c]);
  }
  __syncthreads();
  const int64_t m = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const bool in = m < g.S_loc;
  const uint4* src = reinterpret_cast<const uint4*>(k + ((size_t)(in ? m : 0) * g.Hkv + h / grp) * 128);
  const int64_t mg = in ? global_col(g, m) : INT64_MAX;
  if constexpr (kRope) {
    uint4* dst = reinterpret_cast<uint4*>(k_out + ((size_t)(in ? m : 0) * g.Hkv + h / grp) * 128);
    const bool wr = in && h % grp == 0 && blockIdx.z == 0;
#pragma unroll 1
    for (int v = 0; v < 8; ++v) {  // pairs (c, c + 64), c = 8v .. 8v + 7
      uint4 lo = in ? src[v] : make_uint4(0u, 0u, 0u, 0u);
      uint4 hi = in ? src[v + 8] : make_uint4(0u, 0u, 0u, 0u);
      __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(&lo);
      __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&hi);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 a = __bfloat1622float2(l2[e]), b = __bfloat1622float2(h2[e]);
        float s0, c0, s1, c1, y[4];
        rope_sincos(mg, ra.theta[8 * v + 2 * e], &s0, &c0);
        rope_sincos(mg, ra.theta[8 * v + 2 * e + 1], &s1, &c1);
        rope_rotate(a.x, b.x, s0, c0, ra.mscale, &y[0], &y[2]);
        rope_rotate(a.y, b.y, s1, c1, ra.mscale, &y[1], &y[3]);
        l2[e] = __floats2bfloat162_rn(y[0], y[1]);
        h2[e] = __floats2bfloat162_rn(y[2], y[3]);
      }
      krot[v * kThreads + threadIdx.x] = lo;
      krot[(v + 8) * kThreads + threadIdx.x] = hi;
      if (wr) {
        dst[v] = lo;
        dst[v + 8] = hi;
      }
    }
  }
  const int64_t n0 = g.S - 64;
  float* th = t + (size_t)h * 64 * g.S_loc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 1
  for (int i0 = rlo; i0 < rhi; i0 += kRows) {
    float2 acc2[kRows / 2];  // rows (i0 + 2 rp, i0 + 2 rp + 1)
#pragma unroll
    for (int rp = 0; rp < kRows / 2; ++rp) acc2[rp] = make_float2(0.f, 0.f);
#pragma unroll 1
    for (int cb = 0; cb < 128; cb += kKB) {
      float kf[kKB];
#pragma unroll
      for (int v = 0; v < kKB / 8; ++v) {
        uint4 u;
        if constexpr (kRope)
          u = krot[(cb / 8 + v) * kThreads + threadIdx.x];  // own row: no barrier needed
        else
          u = in ? src[cb / 8 + v] : make_uint4(0u, 0u, 0u, 0u);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          kf[v * 8 + 2 * j] = __uint_as_float(w[j] << 16);
          kf[v * 8 + 2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
        }
      }
#pragma unroll
      for (int c = 0; c < kKB; c += 2) {
        const float2 k0 = make_float2(kf[c], kf[c]), k1 = make_float2(kf[c + 1], kf[c + 1]);
#pragma unroll
        for (int rp = 0; rp < kRows / 2; ++rp) {
          const float4 qv = *reinterpret_cast<const float4*>(&qs2[(i0 >> 1) + rp][cb + c][0]);
          acc2[rp] = ffma2(make_float2(qv.x, qv.y), k0, acc2[rp]);  // I1's fold, column c
          acc2[rp] = ffma2(make_float2(qv.z, qv.w), k1, acc2[rp]);  // then column c + 1
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int i = i0 + r;
      const bool causal = mg <= n0 + i;
      const float tv = causal ? ((r & 1) ? acc2[r >> 1].y : acc2[r >> 1].x) : -INFINITY;
      if (in) th[(size_t)i * g.S_loc + m] = tv;
      float mx = tv;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_down_sync(0xffffffffu, mx, o));
      if (lane == 0) wmax[warp][i] = mx;
    }
  }
  __syncthreads();
  if (threadIdx.x >= rlo && threadIdx.x < rhi) {
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) mx = fmaxf(mx, wmax[w][threadIdx.x]);
    if (mx > -INFINITY) atomic_max_f32(&M[h * 64 + threadIdx.x], mx);
  }
}

inline mt_status stage1_launch(dim3 grid, const Geo& g, const __nv_bfloat16* qwin,
                               const __nv_bfloat16* k, float* t, float* M, cudaStream_t st,
                               const RopeArgs* rope = nullptr, __nv_bfloat16* k_out = nullptr) {
  static const int minb = getenv("MT_VS_S1_MINB") ? atoi(getenv("MT_VS_S1_MINB")) : 3;
  const RopeArgs none{};
  if (rope) {
    if (cudaFuncSetAttribute(stage1_scores<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kRopeSmem) != cudaSuccess)
      return fail(MT_ECUDA, "cudaFuncSetAttribute(stage1 rope) failed");
    stage1_scores<2, true><<<grid, kThreads, kRopeSmem, st>>>(g, qwin, k, t, M, *rope, k_out);
  } else if (minb == 2) {
    stage1_scores<2, false><<<grid, kThreads, 0, st>>>(g, qwin, k, t, M, none, nullptr);
  } else {
    stage1_scores<3, false><<<grid, kThreads, 0, st>>>(g, qwin, k, t, M, none, nullptr);
  }
  return MT_OK;
}

// f3: the window queries' RoPE (positions pos0 + i) while staging them: qwin[i][h][:] =
// RoPE(q[row0 + i][h][:]), the arithmetic of mt_rope (rope.cuh)
__global__ void rope_window_kernel(const __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ qwin,
                                   int64_t row0, int64_t pos0, int Hq,
                                   const __grid_constant__ RopeArgs ra) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;  // (i, h, pair c)
  if (t >= 64 * Hq * 64) return;
  const int c = t & 63, ih = t >> 6, hh = ih % Hq, i = ih / Hq;
  const __nv_bfloat16* src = q + ((size_t)(row0 + i) * Hq + hh) * 128;
  __nv_bfloat16* dst = qwin + ((size_t)i * Hq + hh) * 128;
  float s, co, yl, yh;
  rope_sincos(pos0 + i, ra.theta[c], &s, &co);
  rope_rotate(__bfloat162float(src[c]), __bfloat162float(src[c + 64]), s, co, ra.mscale, &yl, &yh);
  dst[c] = __float2bfloat16_rn(yl);
  dst[c + 64] = __float2bfloat16_rn(yh);
}

// ---------------------------------------------------------------- stage 2
// e = exp2s(...) overwrites t; E[h][i] += sum floor(e 2^31).
__global__ void __launch_bounds__(kThreads) stage2_exp(Geo g, float* t, const float* M,
                                                       unsigned long long* E) {
  __shared__ uint64_t wsum[kThreads / 32][64];
  const int h = blockIdx.y;
  const int64_t m = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const bool in = m < g.S_loc;
  const float Cd = __uint_as_float(kCdBits);
  float* th = t + (size_t)h * 64 * g.S_loc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rlo = blockIdx.z * (64 / gridDim.z), rhi = rlo + 64 / gridDim.z;
#pragma unroll 4
  for (int i = rlo; i < rhi; ++i) {
    uint64_t fx = 0;
    if (in) {
      const float tv = th[(size_t)i * g.S_loc + m];
      float e = 0.f;
      if (tv > -INFINITY) {
        const float y = __fmul_rn(__fsub_rn(tv, M[h * 64 + i]), Cd);
        e = exp2s(y);
      }
      th[(size_t)i * g.S_loc + m] = e;
      fx = __float2ull_rz(__fmul_rn(e, 2147483648.0f));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) fx += shfl_down_u64(fx, o);
    if (lane == 0) wsum[warp][i] = fx;
  }
  __syncthreads();
  if (threadIdx.x >= rlo && threadIdx.x < rhi) {
    uint64_t s = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) s += wsum[w][threadIdx.x];
    if (s) atomicAdd(&E[h * 64 + threadIdx.x], (unsigned long long)s);
  }
}

// ---------------------------------------------------------------- stage 3
// V_m, P_kb, packed sort keys (KeyLayout above).
__global__ void __launch_bounds__(kThreads) stage3_scores(Geo g, const float* t,
                                                          const unsigned long long* E,
                                                          uint64_t* keysV, uint64_t* keysP,
                                                          uint64_t* colV, uint64_t* blkP,
                                                          KeyLayout kv, KeyLayout kp) {
  __shared__ float l_s[64];
  __shared__ uint64_t half[kThreads / 32];
  const int h = blockIdx.y;
  if (threadIdx.x < 64) {
    const float Ef = __ull2float_rn(E[h * 64 + threadIdx.x]);
    l_s[threadIdx.x] = __fmul_rn(Ef, 4.656612873077393e-10f);  // 2^-31
  }
  __syncthreads();
  const int64_t m = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const bool in = m < g.S_loc;
  const float* th = t + (size_t)h * 64 * g.S_loc;
  uint64_t V = 0;
  if (in) {
#pragma unroll 8
    for (int i = 0; i < 64; ++i) {
      const float e = th[(size_t)i * g.S_loc + m];
      if (e > 0.f) {
        const float p = __fdiv_rn(e, l_s[i]);
        V += __float2ull_rz(__fmul_rn(p, 4294967296.0f));
      }
    }
  }
  const uint64_t smax = (1ull << kScoreBits) - 1;
  if (in) {
    const int64_t mg = global_col(g, m);
    const uint64_t hk = kv.hb ? (uint64_t)h << (kScoreBits + kv.ib) : 0ull;
    keysV[(size_t)h * g.S_loc + m] = hk | ((smax - V) << kv.ib) | (uint64_t)mg;
    if (colV) colV[(size_t)h * g.S + mg] = V;
  }
  // block sums over 64 consecutive local keys = one global block
  uint64_t s = V;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += shfl_down_u64(s, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) half[warp] = s;
  __syncthreads();
  if (threadIdx.x < kThreads / 64) {
    const int64_t lb = (int64_t)blockIdx.x * (kThreads / 64) + threadIdx.x;
    if (lb * 64 < g.S_loc) {
      const uint64_t P = half[2 * threadIdx.x] + half[2 * threadIdx.x + 1];
      const int64_t kb = layout_l2g(g.layout, g.W, g.zc, g.r, (int)lb);
      const int64_t nb = g.S / 64;
      const int64_t o = nb - 1 - kb;  // slash offset scored by this block (I6, reading R1)
      const uint64_t hk = kp.hb ? (uint64_t)h << (kScoreBits + kp.ib) : 0ull;
      keysP[(size_t)h * (g.S_loc / 64) + lb] = hk | ((smax - P) << kp.ib) | (uint64_t)o;
      if (blkP) blkP[(size_t)h * nb + o] = P;
    }
  }
}

// ---------------------------------------------------------------- select
// Per (head, list), block-wide (every thread of the CTA calls these):
//   topp_count  exact integer top-p budget k over keys sorted by (score desc, index asc)
//               (I7: smallest k with 2^24 sum_{x<k} score_x >= round(p 2^24) sum score)
//   mark_bits   the first k indices plus the forced index 0 (reading R7) -> bitmap
//   compact     ascending compaction of the bitmap -> index list + count (I8)
// `keys` / `bits` may live in global or shared memory.
__device__ int64_t topp_count(const uint64_t* keys, int64_t n, uint64_t pq, int ib) {
  const uint64_t smax = (1ull << kScoreBits) - 1;
  __shared__ unsigned long long red[32];
  __shared__ unsigned long long tot_s;
  __shared__ long long kmin;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t per = (n + nt - 1) / nt;
  const int64_t b = tid * per, e = min(n, b + per);
  // chunk sums
  unsigned long long cs = 0;
  for (int64_t x = b; x < e; ++x) cs += smax - ((keys[x] >> ib) & smax);
  // inclusive scan of chunk sums (warp + smem)
  const int lane = tid & 31, warp = tid >> 5;
  unsigned long long incl = cs;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) red[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < nt / 32 ? red[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    red[lane] = w;
    if (lane == 31) tot_s = w;
    if (lane == 0) kmin = LLONG_MAX;
  }
  __syncthreads();
  const unsigned long long T = tot_s;
  unsigned long long cum = (warp ? red[warp - 1] : 0ull) + incl - cs;  // exclusive prefix
  int64_t k;
  if (pq >= (1ull << 24)) {
    k = n;  // p = 1: every item (reading R22)
  } else {
    const unsigned long long rhs = pq * T;
    long long found = LLONG_MAX;
    for (int64_t x = b; x < e; ++x) {
      cum += smax - ((keys[x] >> ib) & smax);
      if ((cum << 24) >= rhs) { found = x + 1; break; }
    }
    if (found != LLONG_MAX) atomicMin(&kmin, found);
    __syncthreads();
    k = kmin;
    if (k == LLONG_MAX) k = n;
  }
  __syncthreads();  // red / kmin reusable
  return k;
}

__device__ __forceinline__ void mark_bits(const uint64_t* keys, int64_t k, int ib, uint32_t* bits) {
  const uint64_t imask = (1ull << ib) - 1;
  for (int64_t x = threadIdx.x; x < k; x += blockDim.x) {
    const uint64_t idx = keys[x] & imask;
    atomicOr(&bits[idx >> 5], 1u << (idx & 31));
  }
  if (threadIdx.x == 0) atomicOr(&bits[0], 1u);  // forced: column 0 / offset 0 (reading R7)
}

__device__ void compact(const uint32_t* bits, int64_t words, int32_t* out, int32_t* cnt_out) {
  __shared__ int red[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t per = (words + nt - 1) / nt;
  const int64_t b = tid * per, e = min(words, b + per);
  int cnt = 0;
  for (int64_t w = b; w < e; ++w) cnt += __popc(bits[w]);
  const int lane = tid & 31, warp = tid >> 5;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) red[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nt / 32 ? red[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    red[lane] = w;
  }
  __syncthreads();
  int pos = (warp ? red[warp - 1] : 0) + incl - cnt;
  for (int64_t w = b; w < e; ++w) {
    uint32_t x = bits[w];
    while (x) {
      const int bit = __ffs(x) - 1;
      x &= x - 1;
      out[pos++] = (int32_t)(w * 32 + bit);
    }
  }
  if (tid == nt - 1) *cnt_out = red[31];
}

// One CTA per (head, list): top-p budget over the sorted keys, bitmap marks.
__global__ void __launch_bounds__(1024) topp_mark(const uint64_t* sortedV, const uint64_t* sortedP,
                                                   int64_t nV, int64_t nP, uint64_t pq_v,
                                                   uint64_t pq_s, uint32_t* bitsV,
                                                   uint32_t* bitsP, int ibV, int ibP) {
  const int h = blockIdx.x, which = blockIdx.y;
  const int64_t n = which ? nP : nV;
  const uint64_t* keys = (which ? sortedP : sortedV) + (size_t)h * n;
  uint32_t* bits = (which ? bitsP : bitsV) + (size_t)h * ((n + 31) / 32);
  const int ib = which ? ibP : ibV;
  const int64_t k = topp_count(keys, n, which ? pq_s : pq_v, ib);
  mark_bits(keys, k, ib, bits);
}

// Ascending compaction of a bitmap into an index list.
__global__ void __launch_bounds__(1024) compact_bits(const uint32_t* bitsV, const uint32_t* bitsP,
                                                     int64_t nV, int64_t nP, int32_t* v_cnt,
                                                     int32_t* v_idx, int64_t v_stride,
                                                     int32_t* s_cnt, int32_t* s_off,
                                                     int64_t s_stride) {
  const int h = blockIdx.x, which = blockIdx.y;
  const int64_t n = which ? nP : nV;
  const int64_t words = (n + 31) / 32;
  const uint32_t* bits = (which ? bitsP : bitsV) + (size_t)h * words;
  int32_t* out = which ? s_off + (size_t)h * s_stride : v_idx + (size_t)h * v_stride;
  compact(bits, words, out, (which ? s_cnt : v_cnt) + h);
}

// Short sequences (n <= kSmallSel keys per head and list): the whole select in one launch,
// one CTA per (head, list), keys in registers, no sort.  The top-p set of I7-I8 is the
// k smallest keys (key order = score desc, index asc) with k the smallest count whose
// score mass reaches the budget, i.e. every key <= K* where K* is the smallest key value
// with 2^24 sum_{key <= K*} score >= round(p 2^24) sum score (the mass is a step function
// of the key value, so K* is a key).  K* is found by a radix search, two key bits per
// round (three block-wide sums per round); k >= 1 as in the sorted form.  Replaces the
// device-wide radix sorts (~20 launches), two memsets and two kernels, which dominate
// the index below ~8K tokens.
constexpr int kSmallSel = 8192;
constexpr int kSelThreads = 512;
constexpr int kSelPer = kSmallSel / kSelThreads;  // keys per thread, in registers
__global__ void __launch_bounds__(kSelThreads) select_small(const uint64_t* keysV, const uint64_t* keysP,
                                                      int64_t nV, int64_t nP, uint64_t pq_v,
                                                      uint64_t pq_s, int ibV, int ibP,
                                                      int32_t* v_cnt, int32_t* v_idx,
                                                      int64_t v_stride, int32_t* s_cnt,
                                                      int32_t* s_off, int64_t s_stride) {
  __shared__ uint32_t bits[kSmallSel / 32];
  constexpr int kWarps = kSelThreads / 32;
  __shared__ unsigned long long part[2][kWarps][3];
  const int h = blockIdx.x, which = blockIdx.y;
  const int n = (int)(which ? nP : nV);
  const int ib = which ? ibP : ibV;
  const uint64_t pq = which ? pq_s : pq_v;
  const uint64_t* src = (which ? keysP : keysV) + (size_t)h * n;
  const int nbits = kScoreBits + ib;
  const uint64_t lowmask = nbits >= 64 ? ~0ull : (1ull << nbits) - 1;
  const uint64_t smax = (1ull << kScoreBits) - 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t kr[kSelPer];  // key (head bits dropped); ~0 = no key
#pragma unroll
  for (int u = 0; u < kSelPer; ++u) {
    const int x = u * kSelThreads + tid;
    kr[u] = x < n ? (src[x] & lowmask) : ~0ull;
  }
  const int words = (n + 31) / 32;
  for (int x = tid; x < words; x += kSelThreads) bits[x] = 0u;
  auto score = [&](uint64_t key) { return smax - ((key >> ib) & smax); };
  // block-wide sums of (a, b, c); round r uses part[r & 1] (one barrier per round)
  auto block_sum3 = [&](int r, unsigned long long& a, unsigned long long& b,
                        unsigned long long& c) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (lane == 0) {
      part[r & 1][warp][0] = a;
      part[r & 1][warp][1] = b;
      part[r & 1][warp][2] = c;
    }
    __syncthreads();
    a = b = c = 0ull;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      a += part[r & 1][w][0];
      b += part[r & 1][w][1];
      c += part[r & 1][w][2];
    }
  };
  // total mass and the smallest key (k >= 1)
  unsigned long long tot = 0;
  uint64_t mn = ~0ull;
#pragma unroll
  for (int u = 0; u < kSelPer; ++u)
    if (kr[u] != ~0ull) {
      tot += score(kr[u]);
      mn = min(mn, kr[u]);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = min(mn, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)mn, o));
  {
    unsigned long long dummy = 0;
    block_sum3(0, tot, dummy, dummy);
  }
  __shared__ unsigned long long wmin[kWarps];
  if (lane == 0) wmin[warp] = mn;
  __syncthreads();
  mn = ~0ull;
  for (int w = 0; w < kWarps; ++w) mn = min(mn, (uint64_t)wmin[w]);
  uint64_t thr = ~0ull;  // select every key <= thr
  if (pq < (1ull << 24)) {
    const unsigned long long rhs = pq * tot;
    uint64_t prefix = 0;
    int round = 1;
    for (int b = ((nbits + 1) & ~1) - 2; b >= 0; b -= 2, ++round) {
      const uint64_t ones = (1ull << b) - 1;
      const uint64_t c0 = prefix | ones, c1 = prefix | (1ull << b) | ones,
                     c2 = prefix | (2ull << b) | ones;
      unsigned long long s0 = 0, s1 = 0, s2 = 0;
#pragma unroll
      for (int u = 0; u < kSelPer; ++u) {
        const uint64_t key = kr[u];
        const unsigned long long sc = key != ~0ull ? score(key) : 0ull;
        s0 += key <= c0 ? sc : 0ull;
        s1 += key <= c1 ? sc : 0ull;
        s2 += key <= c2 ? sc : 0ull;
      }
      block_sum3(round, s0, s1, s2);
      const uint64_t d = (s0 << 24) >= rhs ? 0 : (s1 << 24) >= rhs ? 1 : (s2 << 24) >= rhs ? 2 : 3;
      prefix |= d << b;
    }
    thr = max(prefix, mn);
  }
  // marks (plus the forced index 0, reading R7), then ascending compaction
  const uint64_t imask = (1ull << ib) - 1;
#pragma unroll
  for (int u = 0; u < kSelPer; ++u)
    if (kr[u] != ~0ull && kr[u] <= thr) {
      const uint32_t idx = (uint32_t)(kr[u] & imask);
      atomicOr(&bits[idx >> 5], 1u << (idx & 31));
    }
  if (tid == 0) atomicOr(&bits[0], 1u);
  __syncthreads();
  int32_t* out = which ? s_off + (size_t)h * s_stride : v_idx + (size_t)h * v_stride;
  compact(bits, words, out, (which ? s_cnt : v_cnt) + h);
}

// S <= 4096: the same select with the keys SORTED in one CTA (cub::BlockRadixSort over the
// key bits, 512 threads x 8 keys, blocked arrangement), then the budget by a block scan of
// the sorted scores: k = 1 + the first position whose inclusive mass reaches the budget
// (topp_count's rule), and the first k keys marked.  Measured faster than the radix search
// above at 4K (whose rounds rescan every key while most share the leading bits).
constexpr int kSortSel = 4096;
constexpr int kSortItems = kSortSel / kSelThreads;  // 8
__global__ void __launch_bounds__(kSelThreads) select_sorted(const uint64_t* keysV, const uint64_t* keysP,
                                                              int64_t nV, int64_t nP, uint64_t pq_v,
                                                              uint64_t pq_s, int ibV, int ibP,
                                                              int32_t* v_cnt, int32_t* v_idx,
                                                              int64_t v_stride, int32_t* s_cnt,
                                                              int32_t* s_off, int64_t s_stride) {
  using Sort = cub::BlockRadixSort<uint64_t, kSelThreads, kSortItems>;
  using Scan = cub::BlockScan<unsigned long long, kSelThreads>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ uint32_t bits[kSortSel / 32];
  __shared__ int kmin;
  const int h = blockIdx.x, which = blockIdx.y;
  const int n = (int)(which ? nP : nV);
  const int ib = which ? ibP : ibV;
  const uint64_t pq = which ? pq_s : pq_v;
  const uint64_t* src = (which ? keysP : keysV) + (size_t)h * n;
  const int nbits = kScoreBits + ib;  // < 64 for n <= 4096
  const uint64_t lowmask = (1ull << nbits) - 1;
  const uint64_t smax = (1ull << kScoreBits) - 1;
  const int tid = threadIdx.x;
  const int words = (n + 31) / 32;
  for (int x = tid; x < words; x += kSelThreads) bits[x] = 0u;
  if (tid == 0) kmin = n;
  uint64_t key[kSortItems];
#pragma unroll
  for (int u = 0; u < kSortItems; ++u) {  // blocked: thread t holds positions 8t .. 8t + 7
    const int x = tid * kSortItems + u;
    key[u] = x < n ? (src[x] & lowmask) : (1ull << nbits);  // padding sorts last
  }
  Sort(tmp.sort).Sort(key, 0, nbits + 1);
  __syncthreads();
  unsigned long long sc[kSortItems], tsum = 0;
#pragma unroll
  for (int u = 0; u < kSortItems; ++u) {
    const bool pad = key[u] >> nbits;
    sc[u] = pad ? 0ull : smax - ((key[u] >> ib) & smax);
    tsum += sc[u];
  }
  unsigned long long excl, tot;
  Scan(tmp.scan).ExclusiveSum(tsum, excl, tot);
  int k = n;  // p = 1: every item (reading R22)
  if (pq < (1ull << 24)) {
    const unsigned long long rhs = pq * tot;
    unsigned long long cum = excl;
#pragma unroll
    for (int u = 0; u < kSortItems; ++u) {
      cum += sc[u];
      const int pos = tid * kSortItems + u;
      if (pos < n && (cum << 24) >= rhs) {
        atomicMin(&kmin, pos + 1);
        break;
      }
    }
    __syncthreads();
    k = kmin;
  }
  const uint64_t imask = (1ull << ib) - 1;
#pragma unroll
  for (int u = 0; u < kSortItems; ++u)
    if (tid * kSortItems + u < k) {
      const uint32_t idx = (uint32_t)(key[u] & imask);
      atomicOr(&bits[idx >> 5], 1u << (idx & 31));
    }
  if (tid == 0) atomicOr(&bits[0], 1u);  // forced: column 0 / offset 0 (reading R7)
  __syncthreads();
  int32_t* out = which ? s_off + (size_t)h * s_stride : v_idx + (size_t)h * v_stride;
  compact(bits, words, out, (which ? s_cnt : v_cnt) + h);
}

__global__ void fill_f32(float* p, float v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void seg_offsets(int* off, int n_seg, int64_t len) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n_seg) off[i] = (int)(i * len);
}

}  // namespace vsi

// ---------------------------------------------------------------- host side
struct VSIndexWs {
  float* t;                     // [Hq][64][S_loc]
  float* M;                     // [Hq][64]
  unsigned long long* E;        // [Hq][64]
  uint64_t* keysV_loc;          // [Hq][S_loc]
  uint64_t* keysP_loc;          // [Hq][nloc]
  uint64_t* keysV;              // [Hq][S]   (gathered)
  uint64_t* keysP;              // [Hq][nb]
  uint64_t* sortV;              // [Hq][S]
  uint64_t* sortP;              // [Hq][nb]
  uint32_t* bitsV;              // [Hq][S/32]
  uint32_t* bitsP;              // [Hq][ceil(nb/32)]
  int* segP;                    // [Hq+1]
  __nv_bfloat16* qwin;          // [64][Hq][128]
  void* cub_tmp;
  size_t cub_bytes;
  size_t total;
};

static size_t cub_sort_bytes(int Hq, int64_t n) {
  size_t b = 0;
  cub::DeviceSegmentedRadixSort::SortKeys(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                          (int)(Hq * n), Hq, (const int*)nullptr,
                                          (const int*)nullptr, 0, 64);
  return b;
}
// Device-wide radix sorts: all heads at once when the head id fits in the key (a
// segmented sort over Hq segments keeps only ~Hq CTAs busy per pass; per-head sorts
// cost ~10 launches per head, which dominates the index below ~128K tokens).
static size_t cub_sort1_bytes(int64_t n) {
  size_t b = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int)n,
                                 0, 64);
  return b;
}

static VSIndexWs carve_vsidx(void* base, int64_t S, int Hq, int W) {
  VSIndexWs w{};
  const int64_t S_loc = S / W, nb = S / 64, nloc = nb / W;
  uint8_t* p = static_cast<uint8_t*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    void* r = p ? p + off : nullptr;
    off = (off + bytes + 255) & ~size_t(255);
    return r;
  };
  w.t = (float*)take((size_t)Hq * 64 * S_loc * 4);
  w.M = (float*)take((size_t)Hq * 64 * 4);
  w.E = (unsigned long long*)take((size_t)Hq * 64 * 8);
  w.keysV_loc = (uint64_t*)take((size_t)Hq * S_loc * 8);
  w.keysP_loc = (uint64_t*)take((size_t)Hq * nloc * 8);
  w.keysV = (uint64_t*)take((size_t)Hq * S * 8);
  w.keysP = (uint64_t*)take((size_t)Hq * nb * 8);
  w.sortV = (uint64_t*)take((size_t)Hq * S * 8);
  w.sortP = (uint64_t*)take((size_t)Hq * nb * 8);
  w.bitsV = (uint32_t*)take((size_t)Hq * ((S + 31) / 32) * 4);
  w.bitsP = (uint32_t*)take((size_t)Hq * ((nb + 31) / 32) * 4);
  w.segP = (int*)take((size_t)(Hq + 1) * 4);
  w.qwin = (__nv_bfloat16*)take((size_t)64 * Hq * 128 * 2);
  w.cub_bytes = std::max(std::max(cub_sort1_bytes((int64_t)Hq * S), cub_sort1_bytes((int64_t)Hq * nb)),
                         cub_sort_bytes(Hq, nb));
  w.cub_tmp = take(w.cub_bytes);
  w.total = off;
  return w;
}

size_t vsidx_workspace_bytes(int64_t S, int Hq, int W) { return carve_vsidx(nullptr, S, Hq, W).total; }

mt_status vsidx_build(VSCollectives* coll, int64_t S, int Hq, int Hkv, int W, int r, int layout,
                      float p_v, float p_s, const void* q_loc, const void* k_loc, int32_t* v_cnt,
                      int32_t* v_idx, int64_t v_stride, int32_t* s_cnt, int32_t* s_off,
                      int64_t s_stride, uint64_t* dbg_colV, uint64_t* dbg_blkP, void* ws,
                      cudaStream_t st, const RopeArgs* rope, void* q_out, void* k_out) {
  using namespace vsi;
  VSIndexWs w = carve_vsidx(ws, S, Hq, W);
  const int64_t S_loc = S / W, nb = S / 64, nloc = nb / W;
  if (W == 1) layout = 0;
  Geo g{S, S_loc, Hq, Hkv, W, r, layout, layout ? (int)(nb / (2 * W)) : 0};
  // window queries (global rows S-64..S-1): the last global block, which is the last local
  // block of its owner (rank W-1 block-striped, rank 0 zigzag)
  // (f3, rope != NULL: q / k are pre-RoPE; the window is rotated while staged, then q is
  // rotated into q_out and k into k_out by stage 1, as mt_rope would)
  const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(q_loc);
  const int root = coll ? layout_owner(layout, W, g.zc, (int)(nb - 1)) : 0;
  if (r == root) {
    if (rope) {
      rope_window_kernel<<<(64 * Hq * 64 + 255) / 256, 256, 0, st>>>(q, w.qwin, S_loc - 64, S - 64,
                                                                     Hq, *rope);
      MT_TRY(check_launch("vs rope window"));
    } else {
      cudaMemcpyAsync(w.qwin, q + (size_t)(S_loc - 64) * Hq * 128, (size_t)64 * Hq * 128 * 2,
                      cudaMemcpyDeviceToDevice, st);
    }
  }
  if (coll) MT_TRY(coll->bcast_window(w.qwin, (size_t)64 * Hq * 128, root, st));
  if (rope) MT_TRY(rope_launch(*rope, 0, S, W, r, layout, Hq, q_loc, q_out, st));
  fill_f32<<<(Hq * 64 + 255) / 256, 256, 0, st>>>(w.M, -INFINITY, Hq * 64);
  cudaMemsetAsync(w.E, 0, (size_t)Hq * 64 * 8, st);
  const dim3 grid((unsigned)((S_loc + kThreads - 1) / kThreads), Hq);
  // short lengths: split the 64 window rows over 2 CTAs (stages 1-2) to fill the SMs
  const dim3 grid12(grid.x, grid.y, (int64_t)grid.x * grid.y < 2 * device_num_sms() ? 2 : 1);
  MT_TRY(stage1_launch(grid12, g, w.qwin, static_cast<const __nv_bfloat16*>(k_loc), w.t, w.M, st,
                       rope, static_cast<__nv_bfloat16*>(k_out)));
  count_launches(1);  // fill_f32
  MT_TRY(check_launch("vs stage1"));
  if (coll) MT_TRY(coll->allreduce_max(w.M, (size_t)Hq * 64, st));
  stage2_exp<<<grid12, kThreads, 0, st>>>(g, w.t, w.M, w.E);
  MT_TRY(check_launch("vs stage2"));
  if (coll) MT_TRY(coll->allreduce_sum_u64(w.E, (size_t)Hq * 64, st));
  if (dbg_colV) cudaMemsetAsync(dbg_colV, 0, (size_t)Hq * S * 8, st);
  const KeyLayout kv = key_layout(S, Hq), kp = key_layout(nb, Hq);
  stage3_scores<<<grid, kThreads, 0, st>>>(g, w.t, w.E, coll ? w.keysV_loc : w.keysV,
                                           coll ? w.keysP_loc : w.keysP, dbg_colV, dbg_blkP, kv,
                                           kp);
  MT_TRY(check_launch("vs stage3"));
  if (coll) {
    MT_TRY(coll->allgather_keys(w.keysV_loc, w.keysV, Hq, S_loc, st));
    MT_TRY(coll->allgather_keys(w.keysP_loc, w.keysP, Hq, nloc, st));
  }
  const uint64_t pq_v = (uint64_t)llrint((double)p_v * 16777216.0);
  const uint64_t pq_s = (uint64_t)llrint((double)p_s * 16777216.0);
  // MT_VS_SELECT_SMALL=0 forces the radix-sort path (tests compare the two)
  static const bool small_ok = !getenv("MT_VS_SELECT_SMALL") || atoi(getenv("MT_VS_SELECT_SMALL"));
  if (S <= kSmallSel && small_ok) {
    if (S <= kSortSel) {
      select_sorted<<<dim3(Hq, 2), kSelThreads, 0, st>>>(w.keysV, w.keysP, S, nb, pq_v, pq_s,
                                                         kv.ib, kp.ib, v_cnt, v_idx, v_stride,
                                                         s_cnt, s_off, s_stride);
    } else {
      select_small<<<dim3(Hq, 2), kSelThreads, 0, st>>>(w.keysV, w.keysP, S, nb, pq_v, pq_s,
                                                        kv.ib, kp.ib, v_cnt, v_idx, v_stride,
                                                        s_cnt, s_off, s_stride);
    }
    return check_launch("vs select_small");
  }
  size_t tb;
  if (kv.hb) {  // one sort of every head's keys (see cub_sort1_bytes)
    tb = w.cub_bytes;
    if (cub::DeviceRadixSort::SortKeys(w.cub_tmp, tb, w.keysV, w.sortV, (int)(Hq * S), 0,
                                       kScoreBits + kv.ib + kv.hb, st) != cudaSuccess)
      return fail(MT_ECUDA, "radix sort (verticals) failed");
    count_library_calls(1);
  } else {
    for (int h = 0; h < Hq; ++h) {  // per head: a device-wide sort
      tb = w.cub_bytes;
      if (cub::DeviceRadixSort::SortKeys(w.cub_tmp, tb, w.keysV + (size_t)h * S,
                                         w.sortV + (size_t)h * S, (int)S, 0, kScoreBits + kv.ib,
                                         st) != cudaSuccess)
        return fail(MT_ECUDA, "radix sort (verticals) failed");
      count_library_calls(1);
    }
  }
  tb = w.cub_bytes;
  if (kp.hb) {
    if (cub::DeviceRadixSort::SortKeys(w.cub_tmp, tb, w.keysP, w.sortP, (int)(Hq * nb), 0,
                                       kScoreBits + kp.ib + kp.hb, st) != cudaSuccess)
      return fail(MT_ECUDA, "radix sort (slashes) failed");
    count_library_calls(1);
  } else {
    seg_offsets<<<1, 64, 0, st>>>(w.segP, Hq, nb);
    count_launches(1);
    if (cub::DeviceSegmentedRadixSort::SortKeys(w.cub_tmp, tb, w.keysP, w.sortP, (int)(Hq * nb),
                                                Hq, w.segP, w.segP + 1, 0, kScoreBits + kp.ib,
                                                st) != cudaSuccess)
      return fail(MT_ECUDA, "segmented sort (slashes) failed");
    count_library_calls(1);
  }
  cudaMemsetAsync(w.bitsV, 0, (size_t)Hq * ((S + 31) / 32) * 4, st);
  cudaMemsetAsync(w.bitsP, 0, (size_t)Hq * ((nb + 31) / 32) * 4, st);
  topp_mark<<<dim3(Hq, 2), 1024, 0, st>>>(w.sortV, w.sortP, S, nb, pq_v, pq_s, w.bitsV, w.bitsP,
                                          kv.ib, kp.ib);
  MT_TRY(check_launch("vs topp"));
  compact_bits<<<dim3(Hq, 2), 1024, 0, st>>>(w.bitsV, w.bitsP, S, nb, v_cnt, v_idx, v_stride,
                                             s_cnt, s_off, s_stride);
  return check_launch("vs compact");
}

}  // namespace mt

// ---------------------------------------------------------------- C ABI
using namespace mt;

// distributed variant lives with the NCCL communicator (comm.cu)
mt_status mt_build_vs_index_dist(mt_comm* comm, const mt_shape* sh, const mt_vs_params* prm,
                                 const void* q, const void* k, mt_vs_index* out, void* ws,
                                 size_t ws_bytes, mt_stream_t st, const RopeArgs* rope,
                                 void* q_out, void* k_out);

extern "C" size_t mt_build_vs_index_workspace_bytes(const mt_shape* sh, int world) {
  if (!sh || world <= 0) return 0;
  return vsidx_workspace_bytes(sh->seq_len, sh->n_q_heads, world);
}

static mt_status vs_validate(const mt_shape* sh, const mt_vs_params* prm, const void* q,
                             const void* k, void* ws, size_t ws_bytes, int W) {
  MT_TRY(check_shape(sh, W));
  if (!prm) return fail(MT_ESHAPE, "params is NULL");
  if (!(prm->p_v > 0.f && prm->p_v <= 1.f) || !(prm->p_s > 0.f && prm->p_s <= 1.f))
    return fail(MT_ECONFIG, "p_v, p_s must lie in (0, 1] (got %g, %g)", prm->p_v, prm->p_s);
  if (sh->seq_len > (1LL << 22)) return fail(MT_ESHAPE, "seq_len must be <= 2^22 for the index");
  if (!q || !k) return fail(MT_ESHAPE, "NULL q/k");
  const size_t need = vsidx_workspace_bytes(sh->seq_len, sh->n_q_heads, W);
  if (!ws || ws_bytes < need) return fail(MT_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  return check_device();
}

extern "C" mt_status mt_build_vs_index(mt_comm* comm, const mt_shape* sh,
                                       const mt_vs_params* prm, const void* q, const void* k,
                                       mt_vs_index* out, void* ws, size_t ws_bytes,
                                       mt_stream_t st) {
  if (comm)
    return mt_build_vs_index_dist(comm, sh, prm, q, k, out, ws, ws_bytes, st, nullptr, nullptr,
                                  nullptr);
  MT_TRY(vs_validate(sh, prm, q, k, ws, ws_bytes, 1));
  if (!out || !out->v_cnt || !out->v_idx || !out->s_cnt || !out->s_off)
    return fail(MT_ESHAPE, "output index pointers must be non-NULL");
  if (out->v_stride < sh->seq_len || out->s_stride < sh->seq_len / 64)
    return fail(MT_ECAPACITY, "index capacity: need v_stride >= %lld, s_stride >= %lld",
                (long long)sh->seq_len, (long long)(sh->seq_len / 64));
  return vsidx_build(nullptr, sh->seq_len, sh->n_q_heads, sh->n_kv_heads, 1, 0, 0, prm->p_v,
                     prm->p_s, q, k, out->v_cnt, out->v_idx, out->v_stride, out->s_cnt,
                     out->s_off, out->s_stride, nullptr, nullptr, ws, st);
}

extern "C" mt_status mt_rope_vs_index(mt_comm* comm, const mt_shape* sh,
                                      const mt_vs_params* prm, const double* theta, float mscale,
                                      const void* q, const void* k, void* q_out, void* k_out,
                                      mt_vs_index* out, void* ws, size_t ws_bytes,
                                      mt_stream_t st) {
  if (!theta || !q_out || !k_out) return fail(MT_ESHAPE, "NULL theta / q_out / k_out");
  if (k_out == k) return fail(MT_ESHAPE, "k_out must not alias k (stage 1 reads k while writing)");
  RopeArgs ra{};
  for (int i = 0; i < 64; ++i) ra.theta[i] = theta[i];
  ra.mscale = mscale;
  if (comm) return mt_build_vs_index_dist(comm, sh, prm, q, k, out, ws, ws_bytes, st, &ra, q_out, k_out);
  MT_TRY(vs_validate(sh, prm, q, k, ws, ws_bytes, 1));
  if (!out || !out->v_cnt || !out->v_idx || !out->s_cnt || !out->s_off)
    return fail(MT_ESHAPE, "output index pointers must be non-NULL");
  if (out->v_stride < sh->seq_len || out->s_stride < sh->seq_len / 64)
    return fail(MT_ECAPACITY, "index capacity: need v_stride >= %lld, s_stride >= %lld",
                (long long)sh->seq_len, (long long)(sh->seq_len / 64));
  return vsidx_build(nullptr, sh->seq_len, sh->n_q_heads, sh->n_kv_heads, 1, 0, 0, prm->p_v,
                     prm->p_s, q, k, out->v_cnt, out->v_idx, out->v_stride, out->s_cnt,
                     out->s_off, out->s_stride, nullptr, nullptr, ws, st, &ra, q_out, k_out);
}

extern "C" mt_status mt_vs_column_scores(const mt_shape* sh, const void* q, const void* k,
                                         uint64_t* col_scores, uint64_t* slash_scores, void* ws,
                                         size_t ws_bytes, mt_stream_t st) {
  mt_vs_params prm{1.f, 1.f};
  MT_TRY(vs_validate(sh, &prm, q, k, ws, ws_bytes, 1));
  if (!col_scores || !slash_scores) return fail(MT_ESHAPE, "NULL score outputs");
  // Runs stages I1-I6 only; the lists go to scratch inside the workspace tail.
  const int64_t S = sh->seq_len;
  const int Hq = sh->n_q_heads;
  VSIndexWs w = carve_vsidx(ws, S, Hq, 1);
  (void)w;
  using namespace vsi;
  Geo g{S, S, Hq, sh->n_kv_heads, 1, 0, 0, 0};
  cudaMemcpyAsync(w.qwin, static_cast<const __nv_bfloat16*>(q) + (size_t)(S - 64) * Hq * 128,
                  (size_t)64 * Hq * 128 * 2, cudaMemcpyDeviceToDevice, st);
  fill_f32<<<(Hq * 64 + 255) / 256, 256, 0, st>>>(w.M, -INFINITY, Hq * 64);
  cudaMemsetAsync(w.E, 0, (size_t)Hq * 64 * 8, st);
  const dim3 grid((unsigned)((S + kThreads - 1) / kThreads), Hq);
  MT_TRY(stage1_launch(grid, g, w.qwin, static_cast<const __nv_bfloat16*>(k), w.t, w.M, st));
  stage2_exp<<<grid, kThreads, 0, st>>>(g, w.t, w.M, w.E);
  stage3_scores<<<grid, kThreads, 0, st>>>(g, w.t, w.E, w.keysV, w.keysP, col_scores,
                                           slash_scores, key_layout(S, Hq), key_layout(S / 64, Hq));
  count_launches(3);  // fill_f32, stage 1, stage 2 (+ stage 3 in check_launch)
  return check_launch("mt_vs_column_scores");
}
