// vs_format.cu — explicit per-query-block key lists of a vertical-slash index
// (the sparseformat step; SURVEY §8 a6 and §8(b)'s optional
// CSR).  The attention kernels never need these lists (they derive them on the
// fly from the VSPlan); this export makes a6 testable on its own and serves
// callers that want the block-sparse format.
//
// For q head h and query block g (reading I9):
//   B_g = sort_asc{ g - o : o in i_s[h], o <= g }                       (key blocks)
//   C_g = sort_asc{ m in i_v[h] : m/64 < g, (g - m/64) not in i_s[h] }    (bar columns)
// Two passes: count (|B_g|, |C_g| -> global row pointers by one scan) and fill.
#include "common.cuh"
#include "plan.cuh"

namespace mt {

size_t vs_plan_bytes(int64_t S, int Hq, int W);
mt_status vs_plan_build(VSPlan* out, int64_t S, int Hq, int Hkv, int W, int layout,
                        const int32_t* v_cnt,
                        const int32_t* v_idx, int64_t v_stride, const int32_t* s_cnt,
                        const int32_t* s_off, int s_stride, void* ws, cudaStream_t st);
mt_status check_shape(const mt_shape* sh, int W);
mt_status check_index(const mt_vs_index* idx, const mt_shape* sh);

namespace {

constexpr int kThreads = 256;

// number of entries of the ascending list a[0..n) that are < x
__device__ int lower_count(const int32_t* a, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ int block_sum(int v, int* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  }
  __syncthreads();
  return t;  // valid in thread 0
}

// One CTA per (g, h): |B_g|, |C_g|.  Vertical columns are per origin in the plan;
// with W = 1 the single origin's list is i_v[h] ascending.
__global__ void __launch_bounds__(kThreads) count_kernel(VSPlan pl, int64_t* nblk, int64_t* ncol) {
  __shared__ int red[kThreads / 32];
  const int g = blockIdx.x, h = blockIdx.y;
  const int32_t* offs = pl.s_off + (int64_t)h * pl.s_stride;
  const int32_t* vc = pl.vcol + (int64_t)h * pl.S;
  const int nv = pl.vptr[h * (pl.W + 1) + 1] - pl.vptr[h * (pl.W + 1)];
  const int nprefix = lower_count(vc, nv, g * 64);  // columns in blocks < g
  int c = 0;
  for (int i = threadIdx.x; i < nprefix; i += kThreads) c += !plan_has_slash(pl, h, g - (vc[i] >> 6));
  const int tot = block_sum(c, red);
  if (threadIdx.x == 0) {
    nblk[(int64_t)h * pl.nb + g] = lower_count(offs, pl.s_cnt[h], g + 1);
    ncol[(int64_t)h * pl.nb + g] = tot;
  }
}

// Exclusive scan of [Hq][nb] counts into global row pointers [Hq][nb + 1] (one CTA;
// Hq * nb is at most a few 10^5).
__global__ void __launch_bounds__(1024) scan_kernel(const int64_t* cnt, int64_t* ptr, int Hq,
                                                    int nb, int64_t* total) {
  __shared__ int64_t part[1024];
  const int64_t n = (int64_t)Hq * nb;
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t b = threadIdx.x * per, e = min(n, b + per);
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += cnt[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const int64_t t = part[i];
      part[i] = run;
      run += t;
    }
    *total = run;
  }
  __syncthreads();
  int64_t run = part[threadIdx.x];
  for (int64_t i = b; i < e; ++i) {
    const int h = (int)(i / nb), g = (int)(i % nb);
    ptr[(int64_t)h * (nb + 1) + g] = run;
    run += cnt[i];
    if (g == nb - 1) ptr[(int64_t)h * (nb + 1) + nb] = run;
  }
}

__global__ void __launch_bounds__(kThreads) fill_kernel(VSPlan pl, const int64_t* blk_ptr,
                                                        const int64_t* col_ptr, int32_t* blk_idx,
                                                        int32_t* col_idx) {
  __shared__ int warp_tot[kThreads / 32];
  const int g = blockIdx.x, h = blockIdx.y;
  const int64_t row = (int64_t)h * (pl.nb + 1) + g;
  const int32_t* offs = pl.s_off + (int64_t)h * pl.s_stride;
  // B_g: offsets <= g are offs[0..u) ascending, so g - o is descending: reverse
  const int u = (int)(blk_ptr[row + 1] - blk_ptr[row]);
  for (int i = threadIdx.x; i < u; i += kThreads) blk_idx[blk_ptr[row] + i] = g - offs[u - 1 - i];
  // C_g: order-preserving compaction of the uncovered columns of blocks < g
  const int32_t* vc = pl.vcol + (int64_t)h * pl.S;
  const int nv = pl.vptr[h * (pl.W + 1) + 1] - pl.vptr[h * (pl.W + 1)];
  const int nprefix = lower_count(vc, nv, g * 64);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t out = col_ptr[row];
  for (int base = 0; base < nprefix; base += kThreads) {
    const int i = base + threadIdx.x;
    const int m = i < nprefix ? vc[i] : 0;
    const bool keep = i < nprefix && !plan_has_slash(pl, h, g - (m >> 6));
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    int before = 0, all = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      before += w < warp ? warp_tot[w] : 0;
      all += warp_tot[w];
    }
    if (keep) col_idx[out + before + __popc(bal & ((1u << lane) - 1u))] = m;
    out += all;
    __syncthreads();
  }
}

}  // namespace
}  // namespace mt

using namespace mt;

namespace {
struct FormatWs {
  void* plan;
  int64_t* nblk;
  int64_t* ncol;
  int64_t* totals;
  size_t total;
};
FormatWs carve_format(void* base, const mt_shape* sh) {
  const int64_t S = sh->seq_len, nb = S / 64;
  const int Hq = sh->n_q_heads;
  uint8_t* p = static_cast<uint8_t*>(base);
  size_t off = 0;
  auto take = [&](size_t b) {
    void* r = p ? p + off : nullptr;
    off = (off + b + 255) & ~size_t(255);
    return r;
  };
  FormatWs w{};
  w.plan = take(vs_plan_bytes(S, Hq, 1));
  w.nblk = (int64_t*)take((size_t)Hq * nb * 8);
  w.ncol = (int64_t*)take((size_t)Hq * nb * 8);
  w.totals = (int64_t*)take(16);
  w.total = off;
  return w;
}
}  // namespace

extern "C" size_t mt_vs_format_workspace_bytes(const mt_shape* sh) {
  if (!sh || sh->seq_len < 64) return 0;
  return carve_format(nullptr, sh).total;
}

extern "C" mt_status mt_vs_format_count(const mt_shape* sh, const mt_vs_index* idx,
                                        int64_t* blk_ptr, int64_t* col_ptr, int64_t* n_blk,
                                        int64_t* n_col, void* ws, size_t ws_bytes,
                                        mt_stream_t stream) {
  MT_TRY(check_shape(sh, 1));
  MT_TRY(check_index(idx, sh));
  if (!blk_ptr || !col_ptr || !n_blk || !n_col) return fail(MT_ESHAPE, "NULL output");
  FormatWs w = carve_format(ws, sh);
  if (!ws || ws_bytes < w.total) return fail(MT_EWORKSPACE, "workspace %zu < %zu", ws_bytes, w.total);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t S = sh->seq_len, nb = S / 64;
  const int Hq = sh->n_q_heads;
  VSPlan pl;
  MT_TRY(vs_plan_build(&pl, S, Hq, sh->n_kv_heads, 1, 0, idx->v_cnt, idx->v_idx, idx->v_stride,
                       idx->s_cnt, idx->s_off, (int)idx->s_stride, w.plan, st));
  count_kernel<<<dim3((unsigned)nb, Hq), kThreads, 0, st>>>(pl, w.nblk, w.ncol);
  MT_TRY(check_launch("vs_format count"));
  scan_kernel<<<1, 1024, 0, st>>>(w.nblk, blk_ptr, Hq, (int)nb, w.totals);
  scan_kernel<<<1, 1024, 0, st>>>(w.ncol, col_ptr, Hq, (int)nb, w.totals + 1);
  MT_TRY(check_launch("vs_format scan"));
  int64_t h_tot[2];
  if (cudaMemcpyAsync(h_tot, w.totals, 16, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return fail(MT_ECUDA, "vs_format totals copy failed");
  *n_blk = h_tot[0];
  *n_col = h_tot[1];
  return MT_OK;
}

extern "C" mt_status mt_vs_format_fill(const mt_shape* sh, const mt_vs_index* idx,
                                       const int64_t* blk_ptr, const int64_t* col_ptr,
                                       int32_t* blk_idx, int64_t blk_cap, int32_t* col_idx,
                                       int64_t col_cap, int64_t n_blk, int64_t n_col, void* ws,
                                       size_t ws_bytes, mt_stream_t stream) {
  MT_TRY(check_shape(sh, 1));
  MT_TRY(check_index(idx, sh));
  if (!blk_ptr || !col_ptr || (n_blk > 0 && !blk_idx) || (n_col > 0 && !col_idx))
    return fail(MT_ESHAPE, "NULL output");
  if (blk_cap < n_blk || col_cap < n_col)
    return fail(MT_ECAPACITY, "capacity %lld/%lld < required %lld/%lld", (long long)blk_cap,
                (long long)col_cap, (long long)n_blk, (long long)n_col);
  FormatWs w = carve_format(ws, sh);
  if (!ws || ws_bytes < w.total) return fail(MT_EWORKSPACE, "workspace %zu < %zu", ws_bytes, w.total);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t S = sh->seq_len, nb = S / 64;
  const int Hq = sh->n_q_heads;
  VSPlan pl;
  MT_TRY(vs_plan_build(&pl, S, Hq, sh->n_kv_heads, 1, 0, idx->v_cnt, idx->v_idx, idx->v_stride,
                       idx->s_cnt, idx->s_off, (int)idx->s_stride, w.plan, st));
  fill_kernel<<<dim3((unsigned)nb, Hq), kThreads, 0, st>>>(pl, blk_ptr, col_ptr, blk_idx, col_idx);
  return check_launch("vs_format fill");
}
