// block_csr.cu — sparse attention over an explicit block-sparse index (per query
// block, a list of 64-token key blocks), the "I_block" form of the paper's kernel
// interface (block_bar_sparse_attention_forward(Q, K, V, I_block, I_bar), P:878,
// with I_bar empty) and the format an XAttention block index feeds (SURVEY §8(f)
// f2).  Same tcgen05 kernels as the VS path; only the chunk streams differ:
//   forward : query block g walks its row of bidx (diagonal first);
//   backward: key-major tile (h, key pair p) walks the transposed list of query
//             blocks that attend 2p or 2p + 1, built here (count, scan, fill,
//             segmented sort of (g << 1 | slot)).
#include <cub/cub.cuh>

#include "common.cuh"
#include "plan.cuh"
#include "../../include/mtsa.h"

namespace mt {

mt_status check_shape(const mt_shape* sh, int W);
mt_status check_device();
int device_num_sms();
size_t vs_plan_bytes(int64_t S, int Hq, int W);
mt_status attn_fwd_step(const VSPlan& plan, int r, int s, int nloc, const void* q,
                        const void* k, const void* v, void* o, float* o_acc, float* lse,
                        int first, int last, int num_sms, cudaStream_t st);
mt_status attn_bwd_step(const VSPlan& plan, int r, int s, int nloc, const void* q,
                        const void* k, const void* v, const void* dO, const float* lse,
                        const float* D, float* dq, float* dk, float* dv, int num_sms,
                        cudaStream_t st);
mt_status attn_bwd_preprocess(const void* o, const void* dO, float* D, int64_t S_loc, int Hq,
                              cudaStream_t st, float* zq = nullptr, float* zk = nullptr,
                              float* zv = nullptr, int Hkv = 0);
mt_status f32_to_bf16(const float* x, void* y, int64_t n, cudaStream_t st);
mt_status f32_to_bf16_x3(const float* x0, void* y0, int64_t n0, const float* x1, void* y1,
                         int64_t n1, const float* x2, void* y2, int64_t n2, cudaStream_t st);

namespace {

// Per (head, key pair) counts of (query block, slot) entries.
__global__ void pair_count_kernel(const int64_t* __restrict__ bptr, const int32_t* __restrict__ bidx,
                                  int nb, int npairs, int64_t* __restrict__ cnt) {
  const int g = blockIdx.x, h = blockIdx.y;
  const int64_t b = bptr[(int64_t)h * (nb + 1) + g], e = bptr[(int64_t)h * (nb + 1) + g + 1];
  for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[(int64_t)h * npairs + (bidx[i] >> 1)]), 1ull);
}

__global__ void pair_fill_kernel(const int64_t* __restrict__ bptr, const int32_t* __restrict__ bidx,
                                 int nb, int npairs, const int64_t* __restrict__ off,
                                 unsigned long long* __restrict__ pos, int32_t* __restrict__ out) {
  const int g = blockIdx.x, h = blockIdx.y;
  const int64_t b = bptr[(int64_t)h * (nb + 1) + g], e = bptr[(int64_t)h * (nb + 1) + g + 1];
  for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
    const int kb = bidx[i];
    const int64_t seg = (int64_t)h * npairs + (kb >> 1);
    out[off[seg] + (int64_t)atomicAdd(&pos[seg], 1ull)] = (g << 1) | (kb & 1);
  }
}

struct CsrWs {
  void* vsplan;    // zero slash bitmap / vertical pointers + scratch (VS-mode layout)
  int64_t* cnt;    // [Hq * npairs + 1]
  int64_t* off;    // [Hq * npairs + 1]
  unsigned long long* pos;
  int32_t* tunsorted;
  int32_t* tsorted;
  void* cub_tmp;
  size_t cub_bytes;
  size_t total;
};

size_t sort_tmp_bytes(int64_t n, int64_t nseg) {
  size_t b = 0;
  cub::DeviceSegmentedSort::SortKeys((void*)nullptr, b, (const int32_t*)nullptr, (int32_t*)nullptr,
                                     n, nseg, (const int64_t*)nullptr, (const int64_t*)nullptr);
  return b;
}

size_t scan_tmp_bytes(int64_t n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum((void*)nullptr, b, (const int64_t*)nullptr, (int64_t*)nullptr, n);
  return b;
}

CsrWs carve(void* base, const mt_shape* sh, int64_t n_blk, bool bwd) {
  const int64_t S = sh->seq_len, nb = S / 64;
  const int Hq = sh->n_q_heads;
  const int64_t npairs = (nb + 1) / 2, nseg = (int64_t)Hq * npairs;
  uint8_t* p = static_cast<uint8_t*>(base);
  size_t o = 0;
  auto take = [&](size_t b) {
    void* r = p ? p + o : nullptr;
    o = (o + b + 255) & ~size_t(255);
    return r;
  };
  CsrWs w{};
  w.vsplan = take(vs_plan_bytes(S, Hq, 1));
  if (bwd) {
    w.cnt = (int64_t*)take((size_t)(nseg + 1) * 8);
    w.off = (int64_t*)take((size_t)(nseg + 1) * 8);
    w.pos = (unsigned long long*)take((size_t)nseg * 8);
    w.tunsorted = (int32_t*)take((size_t)(n_blk > 0 ? n_blk : 1) * 4);
    w.tsorted = (int32_t*)take((size_t)(n_blk > 0 ? n_blk : 1) * 4);
    const size_t a = sort_tmp_bytes(n_blk, nseg), b = scan_tmp_bytes(nseg + 1);
    w.cub_bytes = a > b ? a : b;
    w.cub_tmp = take(w.cub_bytes);
  }
  w.total = o;
  return w;
}

// The VS-mode plan with every list empty (vertical pointers and slash bitmap zero),
// plus the block-CSR pointers.
mt_status csr_plan(VSPlan* out, const mt_shape* sh, const int64_t* bptr, const int32_t* bidx,
                   void* ws, cudaStream_t st) {
  const int64_t S = sh->seq_len;
  const int Hq = sh->n_q_heads;
  const int nb = (int)(S / 64), words = (nb + 31) / 32;
  uint8_t* p = static_cast<uint8_t*>(ws);
  size_t off = ((size_t)Hq * words * 4 + 255) & ~size_t(255);
  int32_t* vptr = reinterpret_cast<int32_t*>(p + off);
  off = (off + (size_t)Hq * 2 * 4 + 255) & ~size_t(255);
  int32_t* vcol = reinterpret_cast<int32_t*>(p + off);
  off = (off + (size_t)Hq * S * 4 + 255) & ~size_t(255);
  VSPlan pl{};
  pl.S = S;
  pl.Hq = Hq;
  pl.Hkv = sh->n_kv_heads;
  pl.W = 1;
  pl.nb = nb;
  pl.s_stride = nb;
  pl.bits_words = words;
  pl.s_cnt = nullptr;
  pl.s_off = nullptr;
  pl.s_bits = reinterpret_cast<uint32_t*>(p);
  pl.vptr = vptr;
  pl.vcol = vcol;
  pl.scratch = reinterpret_cast<int32_t*>(p + off);
  pl.bptr = bptr;
  pl.bidx = bidx;
  pl.npairs = (nb + 1) / 2;
  if (cudaMemsetAsync(p, 0, (size_t)Hq * words * 4, st) != cudaSuccess ||
      cudaMemsetAsync(vptr, 0, (size_t)Hq * 2 * 4, st) != cudaSuccess)
    return fail(MT_ECUDA, "block-csr plan memset failed");
  *out = pl;
  return MT_OK;
}

mt_status check_csr(const mt_shape* sh, const int64_t* bptr, const int32_t* bidx, int64_t n_blk) {
  MT_TRY(check_shape(sh, 1));
  if (!bptr || (n_blk > 0 && !bidx)) return fail(MT_ESHAPE, "block index pointers must be non-NULL");
  if (n_blk < 0 || n_blk > (int64_t)1 << 31) return fail(MT_ESHAPE, "n_blk out of range");
  return MT_OK;
}

}  // namespace
}  // namespace mt

using namespace mt;

extern "C" size_t mt_block_sparse_attn_fwd_workspace_bytes(const mt_shape* sh) {
  if (!sh || sh->seq_len < 64) return 0;
  return carve(nullptr, sh, 0, false).total;
}

extern "C" mt_status mt_block_sparse_attn_fwd(const mt_shape* sh, const void* q, const void* k,
                                              const void* v, const int64_t* blk_ptr,
                                              const int32_t* blk_idx, int64_t n_blk, void* o,
                                              float* lse, void* ws, size_t ws_bytes,
                                              mt_stream_t stream) {
  MT_TRY(check_csr(sh, blk_ptr, blk_idx, n_blk));
  if (!q || !k || !v || !o || !lse) return fail(MT_ESHAPE, "NULL tensor");
  CsrWs w = carve(ws, sh, n_blk, false);
  if (!ws || ws_bytes < w.total) return fail(MT_EWORKSPACE, "workspace %zu < %zu", ws_bytes, w.total);
  MT_TRY(check_device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  VSPlan pl;
  MT_TRY(csr_plan(&pl, sh, blk_ptr, blk_idx, w.vsplan, st));
  return attn_fwd_step(pl, 0, 0, (int)(sh->seq_len / 64), q, k, v, o, nullptr, lse, 1, 1,
                       device_num_sms(), st);
}

extern "C" size_t mt_block_sparse_attn_bwd_workspace_bytes(const mt_shape* sh, int64_t n_blk) {
  if (!sh || sh->seq_len < 64 || n_blk < 0) return 0;
  const int64_t S = sh->seq_len;
  const size_t acc = (((size_t)S * sh->n_q_heads * 128 * 4 + 255) & ~size_t(255)) +
                     2 * (((size_t)S * sh->n_kv_heads * 128 * 4 + 255) & ~size_t(255)) +
                     (((size_t)sh->n_q_heads * S * 4 + 255) & ~size_t(255));
  return carve(nullptr, sh, n_blk, true).total + acc;
}

extern "C" mt_status mt_block_sparse_attn_bwd(const mt_shape* sh, const void* q, const void* k,
                                              const void* v, const void* o, const float* lse,
                                              const void* dO, const int64_t* blk_ptr,
                                              const int32_t* blk_idx, int64_t n_blk, void* dq,
                                              void* dk, void* dv, void* ws, size_t ws_bytes,
                                              mt_stream_t stream) {
  MT_TRY(check_csr(sh, blk_ptr, blk_idx, n_blk));
  if (!q || !k || !v || !o || !lse || !dO || !dq || !dk || !dv) return fail(MT_ESHAPE, "NULL tensor");
  const size_t need = mt_block_sparse_attn_bwd_workspace_bytes(sh, n_blk);
  if (!ws || ws_bytes < need) return fail(MT_EWORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  MT_TRY(check_device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t S = sh->seq_len, nb = S / 64;
  const int Hq = sh->n_q_heads, Hkv = sh->n_kv_heads;
  CsrWs w = carve(ws, sh, n_blk, true);
  uint8_t* accb = static_cast<uint8_t*>(ws) + w.total;
  auto a256 = [](size_t x) { return (x + 255) & ~size_t(255); };
  float* dq32 = reinterpret_cast<float*>(accb);
  float* dk32 = reinterpret_cast<float*>(accb + a256((size_t)S * Hq * 128 * 4));
  float* dv32 = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(dk32) + a256((size_t)S * Hkv * 128 * 4));
  float* D = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(dv32) + a256((size_t)S * Hkv * 128 * 4));

  VSPlan pl;
  MT_TRY(csr_plan(&pl, sh, blk_ptr, blk_idx, w.vsplan, st));
  // transposed pair lists
  const int64_t npairs = (nb + 1) / 2, nseg = (int64_t)Hq * npairs;
  cudaMemsetAsync(w.cnt, 0, (size_t)(nseg + 1) * 8, st);
  cudaMemsetAsync(w.pos, 0, (size_t)nseg * 8, st);
  const dim3 grid((unsigned)nb, Hq);
  pair_count_kernel<<<grid, 64, 0, st>>>(blk_ptr, blk_idx, (int)nb, (int)npairs, w.cnt);
  MT_TRY(check_launch("pair_count_kernel"));
  size_t tb = w.cub_bytes;
  if (cub::DeviceScan::ExclusiveSum(w.cub_tmp, tb, w.cnt, w.off, nseg + 1, st) != cudaSuccess)
    return fail(MT_ECUDA, "pair scan failed");
  pair_fill_kernel<<<grid, 64, 0, st>>>(blk_ptr, blk_idx, (int)nb, (int)npairs, w.off, w.pos,
                                        w.tunsorted);
  MT_TRY(check_launch("pair_fill_kernel"));
  if (n_blk > 0) {
    tb = w.cub_bytes;
    if (cub::DeviceSegmentedSort::SortKeys(w.cub_tmp, tb, w.tunsorted, w.tsorted, n_blk, nseg,
                                           w.off, w.off + 1, st) != cudaSuccess)
      return fail(MT_ECUDA, "pair sort failed");
  }
  pl.tptr = w.off;
  pl.tidx = w.tsorted;

  MT_TRY(attn_bwd_preprocess(o, dO, D, S, Hq, st, dq32, dk32, dv32, Hkv));  // + zeroed accumulators
  MT_TRY(attn_bwd_step(pl, 0, 0, (int)nb, q, k, v, dO, lse, D, dq32, dk32, dv32,
                       device_num_sms(), st));
  return f32_to_bf16_x3(dq32, dq, S * Hq * 128, dk32, dk, S * Hkv * 128, dv32, dv, S * Hkv * 128,
                        st);
}
