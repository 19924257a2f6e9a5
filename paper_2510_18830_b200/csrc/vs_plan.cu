// vs_plan.cu — build the kernel-side VSPlan (plan.cuh) from index lists.
//
// One CTA per q head.  (1) slash bitmap of i_s[h]; (2) i_v[h] split by KV
// origin s = owner(floor(m / 64)) (block-striped: floor(m / 64) mod W; plan.cuh
// layouts) with order kept (stable compaction), which is
// the per-origin vertical list of convert_index (Alg. 2, P:845;
// DESIGN.md I10).
#include <cstdlib>

#include "common.cuh"
#include "plan.cuh"

namespace mt {

namespace {

constexpr int kThreads = 1024;

// Exclusive scan of one int per thread over the CTA; returns the total.
__device__ int block_exclusive_scan(int v, int* smem /*[32]*/, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = (lane < (int)(blockDim.x >> 5)) ? smem[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    smem[lane] = w;
  }
  __syncthreads();
  const int base = warp ? smem[warp - 1] : 0;
  total = smem[(blockDim.x >> 5) - 1];
  __syncthreads();
  return base + x - v;
}

__global__ void __launch_bounds__(kThreads) vs_plan_kernel(VSPlan p, const int32_t* v_cnt,
                                                           const int32_t* v_idx,
                                                           int64_t v_stride, uint32_t* s_bits,
                                                           int32_t* vptr, int32_t* vcol) {
  __shared__ int scan_smem[32];
  const int h = blockIdx.x;
  // (1) slash bitmap
  uint32_t* bits = s_bits + (int64_t)h * p.bits_words;
  for (int w = threadIdx.x; w < p.bits_words; w += blockDim.x) bits[w] = 0u;
  __syncthreads();
  // counts are clamped to the row stride and out-of-range entries dropped: a malformed
  // caller index must not write outside this head's rows (check_index: stride >= nb, S)
  const int ns = min(max(p.s_cnt[h], 0), p.s_stride);
  for (int i = threadIdx.x; i < ns; i += blockDim.x) {
    const int o = p.s_off[(int64_t)h * p.s_stride + i];
    if (o >= 0 && o < p.nb) atomicOr(&bits[o >> 5], 1u << (o & 31));
  }
  // (2) stable split of i_v[h] by origin
  const int nv = (int)min((int64_t)max(v_cnt[h], 0), min(v_stride, p.S));
  const int32_t* vin = v_idx + (int64_t)h * v_stride;
  int32_t* vout = vcol + (int64_t)h * p.S;
  int32_t* ptr = vptr + (int64_t)h * (p.W + 1);
  int written = 0;
  for (int s = 0; s < p.W; ++s) {
    if (threadIdx.x == 0) ptr[s] = written;
    for (int base = 0; base < nv; base += blockDim.x) {
      const int i = base + threadIdx.x;
      int m = (i < nv) ? vin[i] : 0;
      const int keep = (i < nv) && m >= 0 && m < p.S && plan_owner(p, m >> 6) == s;
      int total;
      const int pos = block_exclusive_scan(keep, scan_smem, total);
      if (keep) vout[written + pos] = m;
      written += total;
    }
  }
  if (threadIdx.x == 0) ptr[p.W] = written;
}

}  // namespace

// Packed-row capacity per head (forward bar chunks): the origin's columns, at most
// 16384 (MT_PACK_CAP lowers it, so tests reach the gather fallback of heads with more
// columns at small sizes), rounded to whole 128-row chunks.
int packed_cap(int64_t S, int W) {
  static const int64_t cap = getenv("MT_PACK_CAP") ? atoll(getenv("MT_PACK_CAP")) : 16384;
  int64_t c = S / W;
  if (c > cap) c = cap;
  if (c < 0) c = 0;
  return (int)((c + 127) / 128 * 128);
}

size_t vs_plan_bytes(int64_t S, int Hq, int W) {
  const int nb = (int)(S / 64);
  const int words = (nb + 31) / 32;
  size_t b = 0;
  b += (size_t)Hq * words * 4;
  b = (b + 255) & ~size_t(255);
  b += (size_t)Hq * (W + 1) * 4;
  b = (b + 255) & ~size_t(255);
  b += (size_t)Hq * S * 4;
  b = (b + 255) & ~size_t(255);
  b += (size_t)(16 + (int64_t)Hq * nb) * 4;  // scratch
  b = (b + 255) & ~size_t(255);
  b += 2 * (size_t)packed_cap(S, W) * Hq * 128 * 2;  // packed vertical K / V rows
  return (b + 255) & ~size_t(255);
}

// Carve the plan out of `ws` and launch the builder.
mt_status vs_plan_build(VSPlan* out, int64_t S, int Hq, int Hkv, int W, int layout,
                        const int32_t* v_cnt,
                        const int32_t* v_idx, int64_t v_stride, const int32_t* s_cnt,
                        const int32_t* s_off, int s_stride, void* ws, cudaStream_t st) {
  const int nb = (int)(S / 64);
  const int words = (nb + 31) / 32;
  uint8_t* p = static_cast<uint8_t*>(ws);
  uint32_t* bits = reinterpret_cast<uint32_t*>(p);
  size_t off = ((size_t)Hq * words * 4 + 255) & ~size_t(255);
  int32_t* vptr = reinterpret_cast<int32_t*>(p + off);
  off = (off + (size_t)Hq * (W + 1) * 4 + 255) & ~size_t(255);
  int32_t* vcol = reinterpret_cast<int32_t*>(p + off);
  off = (off + (size_t)Hq * S * 4 + 255) & ~size_t(255);
  int32_t* scratch = reinterpret_cast<int32_t*>(p + off);
  off = (off + (size_t)(16 + (int64_t)Hq * nb) * 4 + 255) & ~size_t(255);
  const int pcap = packed_cap(S, W);
  void* kp = p + off;
  void* vp = p + off + (size_t)pcap * Hq * 128 * 2;
  VSPlan pl{};
  pl.S = S;
  pl.Hq = Hq;
  pl.Hkv = Hkv;
  pl.W = W;
  pl.layout = W > 1 ? layout : 0;  // one rank: every layout is the identity
  pl.zc = pl.layout ? nb / (2 * W) : 0;
  pl.nb = nb;
  pl.s_stride = s_stride;
  pl.bits_words = words;
  pl.s_cnt = s_cnt;
  pl.s_off = s_off;
  pl.s_bits = bits;
  pl.vptr = vptr;
  pl.vcol = vcol;
  pl.scratch = scratch;
  pl.kp = kp;
  pl.vp = vp;
  pl.pcap = pcap;
  vs_plan_kernel<<<Hq, kThreads, 0, st>>>(pl, v_cnt, v_idx, v_stride, bits, vptr, vcol);
  MT_TRY(check_launch("vs_plan_kernel"));
  *out = pl;
  return MT_OK;
}

}  // namespace mt
