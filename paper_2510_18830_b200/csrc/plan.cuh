// plan.cuh — device-side view of a vertical-slash index as consumed by the
// sparse attention kernels.
//
// The global index (Alg. 1 output): per q head h, sorted vertical
// token columns i_v[h] and sorted slash block offsets i_s[h] (offset o selects
// key block g - o for query block g).  The kernels never materialise
// sparseformat's per-query-block lists (convert_index P:845); they derive
// them on the fly from:
//   s_off/s_cnt : i_s[h] ascending
//   s_bits      : i_s[h] as a bitmap over [0, nb)      (membership test, I9)
//   vptr/vcol   : i_v[h] grouped by KV origin s = (m/64) mod W, ascending
//                 inside each group (per-origin lists of I10)
#pragma once
#include <cstdint>

#ifndef __CUDACC__
#include <algorithm>
using std::max;
using std::min;
#endif

namespace mt {

struct VSPlan {
  int64_t S;        // global sequence length
  int Hq, Hkv, W;   // heads, world size (ranks of the layout)
  int layout;       // MT_LAYOUT_STRIPED (0) or MT_LAYOUT_ZIGZAG (1), see layout_* below
  int zc;           // zigzag: blocks per chunk (nb / 2W)
  int nb;           // global 64-token blocks = S / 64
  int s_stride;     // row stride of s_off (>= nb)
  int bits_words;   // 32-bit words per head in s_bits
  const int32_t* s_cnt;
  const int32_t* s_off;
  const uint32_t* s_bits;
  const int32_t* vptr;  // [Hq][W + 1]
  const int32_t* vcol;  // [Hq][S] (global column ids, grouped by origin)
  int32_t* scratch;     // [16 + Hq * nb] ints: [0] fwd fix-up count, [1] fwd tile counter,
                        // [2], [3] bwd tile counters, [16..] fix-up list
  // Block-CSR mode (mt_block_sparse_attn_*, W = 1): explicit key-block
  // lists replace the slash lists (s_cnt = 0, no verticals).  nullptr: VS mode.
  const int64_t* bptr;  // [Hq][nb + 1] row pointers into bidx
  const int32_t* bidx;  // key blocks of query block g (ascending, <= g, unique)
  const int64_t* tptr;  // [Hq * npairs + 1] segment offsets (backward only)
  const int32_t* tidx;  // per (head, key pair p): (g << 1 | kb - 2p) ascending
  int npairs;           // ceil(nb / 2)
  // Packed vertical rows for the forward (bar chunks as TMA tile loads): per step,
  // the held chunk's K / V rows of each head's vertical list of that origin, row i of
  // head h at [i][h][128] bf16 (rows up to the next multiple of 128 zero-filled).
  // Heads with more than pcap columns of one origin use the cp.async gather path.
  void* kp;
  void* vp;
  int pcap;             // packed rows per head (multiple of 128; 0 = no packing)
};

// ---- sequence layouts (Fig. 1), at 64-token block granularity
//   striped (the method): global block b on rank b mod W, local block b / W;
//   zigzag  (the "Ours w/ ZigZag" ablation): 2W chunks of zc blocks, rank r holds
//           chunk r then chunk 2W-1-r.
// Both map a rank's local blocks to ascending global blocks.
__host__ __device__ __forceinline__ int layout_l2g(int layout, int W, int zc, int r, int lb) {
  if (layout == 0) return lb * W + r;
  return lb < zc ? r * zc + lb : (2 * W - 1 - r) * zc + (lb - zc);
}
__host__ __device__ __forceinline__ int layout_owner(int layout, int W, int zc, int gb) {
  if (layout == 0) return gb % W;
  const int k = gb / zc;
  return k < W ? k : 2 * W - 1 - k;
}
__host__ __device__ __forceinline__ int layout_g2l(int layout, int W, int zc, int gb) {
  if (layout == 0) return gb / W;
  const int k = gb / zc;
  return k < W ? gb - k * zc : zc + gb - k * zc;
}
// local blocks of rank r whose global block is <= g
__host__ __device__ __forceinline__ int layout_count_le(int layout, int W, int zc, int r, int g) {
  if (layout == 0) return g < r ? 0 : (g - r) / W + 1;
  const int a = min(max(g - r * zc + 1, 0), zc);
  const int b = min(max(g - (2 * W - 1 - r) * zc + 1, 0), zc);
  return a + b;
}
__device__ __forceinline__ bool plan_has_slash(const VSPlan& p, int h, int o) {
  return (p.s_bits[(int64_t)h * p.bits_words + (o >> 5)] >> (o & 31)) & 1u;
}

__host__ __device__ __forceinline__ int plan_l2g(const VSPlan& p, int r, int lb) {
  return layout_l2g(p.layout, p.W, p.zc, r, lb);
}
__host__ __device__ __forceinline__ int plan_owner(const VSPlan& p, int gb) {
  return layout_owner(p.layout, p.W, p.zc, gb);
}
__host__ __device__ __forceinline__ int plan_g2l(const VSPlan& p, int gb) {
  return layout_g2l(p.layout, p.W, p.zc, gb);
}
__host__ __device__ __forceinline__ int plan_count_le(const VSPlan& p, int r, int g) {
  return layout_count_le(p.layout, p.W, p.zc, r, g);
}
// the same with the layout fixed at compile time (the kernels' producers are instantiated
// per layout: the striped walk then compiles to round 1's lattice arithmetic)
template <int L>
__device__ __forceinline__ int l2g_(const VSPlan& p, int r, int lb) { return layout_l2g(L, p.W, p.zc, r, lb); }
template <int L>
__device__ __forceinline__ int g2l_(const VSPlan& p, int gb) { return layout_g2l(L, p.W, p.zc, gb); }
template <int L>
__device__ __forceinline__ int count_le_(const VSPlan& p, int r, int g) {
  return layout_count_le(L, p.W, p.zc, r, g);
}

}  // namespace mt
