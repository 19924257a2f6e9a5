// xattn.cu — XAttention antidiagonal block index (PAPER.md P:826,
// P:347 "Ours w/ XAttn Idx."; reading R25 in DESIGN.md, oracle/xattn.py).
//
// Per q head h (kv head h / (Hq/Hkv)), block B = 128, stride st = 16, n = S / st:
//   1. Qr[i] = (q[i st + st-1], ..., q[i st]), Kr[j] = (k[j st], ..., k[j st + st-1])
//      (2048-wide rows; reshape kernels), so A = Qr Kr^T / (st sqrt d) sums each
//      st x st sub-block's antidiagonal;
//   2.-3. row softmax over j <= i, then the 8 x 8 block sums Bs[I][J], J <= I (lower
//      triangle, fp32).  Default: one hand-written tcgen05 kernel does 1.-3. without
//      materialising A (xattn_score.cu).  MT_XATTN_CUBLAS=1: round 1's path, A by a cuBLAS
//      bf16 GEMM in row chunks of R (columns bounded causally), then one CTA per 128-block
//      row for the online max/sum and the block sums;
//   4. all heads at once: stable segmented sort of each row descending (ties keep the
//      smaller J first), one warp per row keeps J while the sum before it is
//      < tau * row total; the diagonal is always kept (bitmap [Hq][nI][nI/32]);
//   5. 64-token CSR: count, scan, fill (query blocks 2I, 2I+1; key blocks 2J, 2J+1,
//      the diagonal's causal half).
#include <cstdlib>
#include <mutex>
#include <cublas_v2.h>

#include <cub/cub.cuh>

#include "common.cuh"
#include "../../include/mtsa.h"

namespace mt {

mt_status check_shape(const mt_shape* sh, int W);
mt_status check_device();
int device_num_sms();
size_t xattn_score_scratch_bytes(int64_t n, int nI, int num_sms);
mt_status xattn_scores_tc(const void* qr, const void* kr, int64_t n, int nI, int hb, int h0,
                          int Hkv, int grp, float scale_log2, float* tri, int64_t T,
                          void* scratch, int num_sms, cudaStream_t st);

namespace {

constexpr int kSt = 16, kB = 128, kR = kB / kSt;  // 8 stride rows per block
constexpr int kD = 128, kWide = kSt * kD;         // 2048
constexpr size_t kGemmWs = size_t(32) << 20;      // cuBLAS workspace slice

// dst[i][s * 128 + c] = src[(i st + (rev ? st-1-s : s)) * H + h][c], 16 B per thread
__global__ void reshape_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                               int64_t n, int H, int h, int rev) {
  const int64_t total = n * (kWide / 8);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / (kWide / 8);
    const int r = (int)(t % (kWide / 8));
    const int s = r / (kD / 8), c8 = r % (kD / 8);
    const int64_t tok = i * kSt + (rev ? kSt - 1 - s : s);
    reinterpret_cast<uint4*>(dst)[t] =
        reinterpret_cast<const uint4*>(src + (tok * H + h) * kD)[c8];
  }
}

__device__ __forceinline__ void merge_ml(float& m, float& l, float m2, float l2) {
  const float mm = fmaxf(m, m2);
  if (mm == -INFINITY) return;
  l = l * exp2f(m - mm) + l2 * exp2f(m2 - mm);
  m = mm;
}

// C: rows [i0, i0 + rows) of the strided scores (natural-log units), row stride ldc.
// One CTA per 128-block row I in the chunk; Bs row I: tri + I (I + 1) / 2.
__global__ void __launch_bounds__(256) softmax_blocksum_kernel(const float* __restrict__ C,
                                                               int64_t ldc, int64_t i0,
                                                               float* __restrict__ tri) {
  __shared__ float red_m[8], red_l[8];
  __shared__ float row_m[kR], row_l[kR];
  const int64_t I = i0 / kR + blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr float kLog2e = 1.4426950408889634f;
  for (int r = 0; r < kR; ++r) {
    const int64_t i = I * kR + r;  // stride row
    const float* row = C + (i - i0) * ldc;
    float m = -INFINITY, l = 0.f;
    for (int64_t j = threadIdx.x; j <= i; j += blockDim.x) {
      const float x = row[j] * kLog2e;
      if (x > m) {
        l = l * exp2f(m - x) + 1.f;
        m = x;
      } else {
        l += exp2f(x - m);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), l2 = __shfl_xor_sync(0xffffffffu, l, o);
      merge_ml(m, l, m2, l2);
    }
    if (lane == 0) {
      red_m[warp] = m;
      red_l[warp] = l;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float mm = red_m[0], ll = red_l[0];
      for (int w = 1; w < 8; ++w) merge_ml(mm, ll, red_m[w], red_l[w]);
      row_m[r] = mm;
      row_l[r] = ll;
    }
    __syncthreads();
  }
  float* out = tri + I * (I + 1) / 2;
  for (int64_t J = threadIdx.x; J <= I; J += blockDim.x) {
    float acc = 0.f;
    for (int r = 0; r < kR; ++r) {
      const int64_t i = I * kR + r;
      const float* row = C + (i - i0) * ldc + J * kR;
      const float m = row_m[r], inv = 1.f / row_l[r];
      float s = 0.f;
#pragma unroll
      for (int c = 0; c < kR; ++c)
        if (J * kR + c <= i) s += exp2f(row[c] * kLog2e - m);
      acc += s * inv;
    }
    out[J] = acc;
  }
}

// segment offsets over all heads: seg (h, I) = [h T + I (I+1)/2, + I + 1); values = J
__global__ void seg_init_kernel(int64_t nI, int Hq, int64_t* __restrict__ off, int32_t* __restrict__ jv) {
  const int64_t T = nI * (nI + 1) / 2;
  const int64_t nseg = (int64_t)Hq * nI;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s <= nseg;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = s / nI, I = s % nI;
    off[s] = s == nseg ? (int64_t)Hq * T : h * T + I * (I + 1) / 2;
  }
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)Hq * T;
       e += (int64_t)gridDim.x * blockDim.x) {
    // J of entry e: e % T = I (I+1)/2 + J
    const int64_t x = e % T;
    int64_t I = (int64_t)((sqrt(8.0 * (double)x + 1.0) - 1.0) / 2.0);
    while (I * (I + 1) / 2 > x) --I;
    while ((I + 1) * (I + 2) / 2 <= x) ++I;
    jv[e] = (int32_t)(x - I * (I + 1) / 2);
  }
}

// One warp per segment (h, I): keep the shortest descending prefix reaching tau * total.
__global__ void select_kernel(const float* __restrict__ keys, const int32_t* __restrict__ jv,
                              const float* __restrict__ tri_unsorted, int64_t nI, int Hq,
                              float tau, uint32_t* __restrict__ bits) {
  const int lane = threadIdx.x & 31;
  const int64_t seg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (seg >= (int64_t)Hq * nI) return;
  const int64_t h = seg / nI, I = seg % nI;
  const int64_t T = nI * (nI + 1) / 2;
  const int64_t b = h * T + I * (I + 1) / 2, n = I + 1;
  const int64_t words = (nI + 31) / 32;
  uint32_t* row = bits + seg * words;
  // total in the row's natural (J ascending) order
  float tot = 0.f;
  for (int64_t x = lane; x < n; x += 32) tot += tri_unsorted[b + x];
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  const float lim = tau * tot;
  float acc = 0.f;  // sum of the entries before this batch
  for (int64_t base = 0; base < n; base += 32) {
    const int64_t x = base + lane;
    const float v = x < n ? keys[b + x] : 0.f;
    float inc = v;  // inclusive prefix within the batch
    for (int o = 1; o < 32; o <<= 1) {
      const float y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const float before = acc + inc - v;
    const bool keep = x < n && before < lim;
    if (keep) {
      const int J = jv[b + x];
      atomicOr(&row[J >> 5], 1u << (J & 31));
    }
    acc += __shfl_sync(0xffffffffu, inc, 31);
    if (!__any_sync(0xffffffffu, keep)) break;
  }
  if (lane == 0) atomicOr(&row[I >> 5], 1u << (I & 31));  // the diagonal
}

// 64-token rows: count for (h, g) = 2 (popcount of row I without the diagonal) + (g odd ? 2 : 1)
__global__ void count64_kernel(const uint32_t* __restrict__ bits, int64_t nI, int Hq, int64_t* __restrict__ cnt) {
  const int64_t nb = 2 * nI, words = (nI + 31) / 32;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)Hq * nb;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = t / nb, g = t % nb, I = g / 2;
    const uint32_t* row = bits + (h * nI + I) * words;
    int pc = 0;
    for (int64_t w = 0; w < words; ++w) pc += __popc(row[w]);
    cnt[t] = 2 * (pc - 1) + ((g & 1) ? 2 : 1);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[(int64_t)Hq * nb] = 0;
}

// flat exclusive scan [Hq nb + 1] -> [Hq][nb + 1] row pointers (global offsets)
__global__ void ptr_layout_kernel(const int64_t* __restrict__ flat, int64_t nb, int Hq, int64_t* __restrict__ ptr) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)Hq * (nb + 1);
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = t / (nb + 1), g = t % (nb + 1);
    ptr[t] = flat[h * nb + g];  // g == nb reads the next head's start (or the total)
  }
}

// one warp per (h, g): ascending key blocks of the row
__global__ void fill64_kernel(const uint32_t* __restrict__ bits, int64_t nI, int Hq,
                              const int64_t* __restrict__ ptr, int32_t* __restrict__ idx) {
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nb = 2 * nI, words = (nI + 31) / 32;
  if (t >= (int64_t)Hq * nb) return;
  const int64_t h = t / nb, g = t % nb, I = g / 2;
  const uint32_t* row = bits + (h * nI + I) * words;
  int64_t out = ptr[h * (nb + 1) + g];
  for (int64_t w0 = 0; w0 < words; w0 += 32) {
    const int64_t w = w0 + lane;
    const uint32_t x = w < words ? row[w] : 0u;
    int c = 0;  // entries this lane writes
    for (uint32_t y = x; y; y &= y - 1) {
      const int J = (int)(w * 32 + __ffs(y) - 1);
      c += J < I ? 2 : ((g & 1) ? 2 : 1);
    }
    int pre = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += y;
    }
    int64_t pos = out + pre - c;
    for (uint32_t y = x; y; y &= y - 1) {
      const int J = (int)(w * 32 + __ffs(y) - 1);
      idx[pos++] = 2 * J;
      if (J < I || (g & 1)) idx[pos++] = 2 * J + 1;
    }
    out += __shfl_sync(0xffffffffu, pre, 31);
  }
}

struct XWs {
  __nv_bfloat16 *qr, *kr;
  float* C;
  float *tri, *keys;
  int32_t *jv, *jv_sorted;
  int64_t* off;
  uint32_t* bits;
  int64_t *cnt, *scan;
  void* cub_tmp;
  size_t cub_bytes;
  void* gemm_ws;   // cuBLAS workspace (cublasSetWorkspace): no allocation inside the GEMM
  int64_t R;  // stride rows per GEMM chunk
  // hand-written path (xattn_score.cu): q heads reshaped hb at a time, every kv head's K
  __nv_bfloat16 *qrb, *krall;
  void* xsc;  // per-CTA P / Mt scratch
  int hb;
  size_t total;
};

// q heads per fused-score launch: enough (head, row tile) items for ~8 per SM
inline int xattn_hb(int64_t n, int Hq) {
  const int nrt = (int)((n + 127) / 128);
  int hb = (8 * 148 + nrt - 1) / nrt;
  return hb < 1 ? 1 : (hb > Hq ? Hq : hb);
}
// MT_XATTN_CUBLAS=1: round 1's cuBLAS GEMM + softmax pass (A/B)
inline bool xattn_use_cublas() {
  static const bool v = getenv("MT_XATTN_CUBLAS") && atoi(getenv("MT_XATTN_CUBLAS"));
  return v;
}

XWs carve(void* base, const mt_shape* sh) {
  const int64_t S = sh->seq_len, n = S / kSt, nI = S / kB, nb = S / 64;
  const int Hq = sh->n_q_heads;
  const int64_t T = nI * (nI + 1) / 2;
  uint8_t* p = static_cast<uint8_t*>(base);
  size_t o = 0;
  auto take = [&](size_t b) {
    void* r = p ? p + o : nullptr;
    o = (o + b + 255) & ~size_t(255);
    return r;
  };
  XWs w{};
  int64_t R = ((int64_t)1 << 28) / n;  // chunk of <= 2^28 fp32 scores
  R = R < kR ? kR : (R / kR) * kR;
  if (R > n) R = n;
  w.R = R;
  w.qr = (__nv_bfloat16*)take((size_t)n * kWide * 2);
  w.kr = (__nv_bfloat16*)take((size_t)n * kWide * 2);
  w.C = (float*)take((size_t)R * n * 4);
  w.tri = (float*)take((size_t)Hq * T * 4);
  w.keys = (float*)take((size_t)Hq * T * 4);
  w.jv = (int32_t*)take((size_t)Hq * T * 4);
  w.jv_sorted = (int32_t*)take((size_t)Hq * T * 4);
  w.off = (int64_t*)take((size_t)(Hq * nI + 1) * 8);
  w.bits = (uint32_t*)take((size_t)Hq * nI * ((nI + 31) / 32) * 4);
  w.cnt = (int64_t*)take((size_t)(Hq * nb + 1) * 8);
  w.scan = (int64_t*)take((size_t)(Hq * nb + 1) * 8);
  size_t a = 0, b = 0;
  cub::DeviceSegmentedSort::StableSortPairsDescending((void*)nullptr, a, (const float*)nullptr,
                                                      (float*)nullptr, (const int32_t*)nullptr,
                                                      (int32_t*)nullptr, Hq * T, Hq * nI,
                                                      (const int64_t*)nullptr, (const int64_t*)nullptr);
  cub::DeviceScan::ExclusiveSum((void*)nullptr, b, (const int64_t*)nullptr, (int64_t*)nullptr,
                                Hq * nb + 1);
  w.cub_bytes = a > b ? a : b;
  w.cub_tmp = take(w.cub_bytes);
  w.gemm_ws = take(kGemmWs);
  w.hb = xattn_hb(n, Hq);
  w.qrb = (__nv_bfloat16*)take((size_t)w.hb * n * kWide * 2);
  w.krall = (__nv_bfloat16*)take((size_t)sh->n_kv_heads * n * kWide * 2);
  w.xsc = take(xattn_score_scratch_bytes(n, (int)nI, 148));
  w.total = o;
  return w;
}

mt_status check_x(const mt_shape* sh, const mt_xattn_params* prm) {
  MT_TRY(check_shape(sh, 1));
  if (!prm) return fail(MT_ESHAPE, "params NULL");
  if (prm->block != kB || prm->stride != kSt)
    return fail(MT_EUNSUPPORTED, "xattn: block %d / stride %d (supported: 128 / 16)", prm->block,
                prm->stride);
  if (!(prm->threshold >= 0.f && prm->threshold <= 1.f)) return fail(MT_ESHAPE, "threshold not in [0, 1]");
  if (sh->seq_len % kB) return fail(MT_EWINDOW, "xattn: seq_len must be a multiple of 128");
  {  // the segmented sort counts items in int: Hq * nI (nI + 1) / 2 must fit
    const int64_t nI = sh->seq_len / kB;
    if ((int64_t)sh->n_q_heads * (nI * (nI + 1) / 2) > (int64_t)INT32_MAX)
      return fail(MT_ESHAPE, "xattn: Hq x causal block pairs exceeds INT_MAX (seq_len %lld, Hq %d)",
                  (long long)sh->seq_len, sh->n_q_heads);
  }
  return MT_OK;
}

// one cuBLAS handle per device (a handle is bound to the device current at creation),
// created under a lock so concurrent host threads do not race on the cache
cublasHandle_t handle() {
  constexpr int kMaxDev = 64;
  static cublasHandle_t h[kMaxDev] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!h[dev] && cublasCreate(&h[dev]) != CUBLAS_STATUS_SUCCESS) h[dev] = nullptr;
  return h[dev];
}

}  // namespace
}  // namespace mt

using namespace mt;

extern "C" size_t mt_xattn_index_workspace_bytes(const mt_shape* sh) {
  if (!sh || sh->seq_len < kB || sh->seq_len % kB || sh->n_q_heads <= 0) return 0;
  return carve(nullptr, sh).total;
}

extern "C" mt_status mt_xattn_index_count(const mt_shape* sh, const mt_xattn_params* prm,
                                          const void* q, const void* k, int64_t* blk_ptr,
                                          int64_t* n_blk, float* block_scores, void* ws,
                                          size_t ws_bytes, mt_stream_t stream) {
  MT_TRY(check_x(sh, prm));
  if (!q || !k || !blk_ptr || !n_blk) return fail(MT_ESHAPE, "NULL argument");
  XWs w = carve(ws, sh);
  if (!ws || ws_bytes < w.total) return fail(MT_EWORKSPACE, "workspace %zu < %zu", ws_bytes, w.total);
  MT_TRY(check_device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t S = sh->seq_len, n = S / kSt, nI = S / kB, nb = S / 64;
  const int Hq = sh->n_q_heads, Hkv = sh->n_kv_heads, grp = Hq / Hkv;
  const int64_t T = nI * (nI + 1) / 2;
  cublasHandle_t hb = nullptr;
  if (xattn_use_cublas()) {
    hb = handle();
    if (!hb) return fail(MT_ECUDA, "cublasCreate failed");
    if (cublasSetStream(hb, st) != CUBLAS_STATUS_SUCCESS ||
        cublasSetWorkspace(hb, w.gemm_ws, kGemmWs) != CUBLAS_STATUS_SUCCESS)
      return fail(MT_ECUDA, "cublasSetStream/SetWorkspace failed");
  }
  const float alpha = 1.f / (kSt * sqrtf((float)kD)), beta = 0.f;
  const int rgrid = 148 * 8;
  if (!xattn_use_cublas()) {
    // hand-written tcgen05 scores with the softmax / block sums fused (xattn_score.cu)
    const int sms = device_num_sms() < 148 ? device_num_sms() : 148;
    for (int g = 0; g < Hkv; ++g) {
      reshape_kernel<<<rgrid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(k),
                                           w.krall + (size_t)g * n * kWide, n, Hkv, g, 0);
      MT_TRY(check_launch("xattn reshape k"));
    }
    for (int h0 = 0; h0 < Hq; h0 += w.hb) {
      const int hb = Hq - h0 < w.hb ? Hq - h0 : w.hb;
      for (int hh = 0; hh < hb; ++hh) {
        reshape_kernel<<<rgrid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(q),
                                             w.qrb + (size_t)hh * n * kWide, n, Hq, h0 + hh, 1);
        MT_TRY(check_launch("xattn reshape q"));
      }
      MT_TRY(xattn_scores_tc(w.qrb, w.krall, n, (int)nI, hb, h0, Hkv, grp,
                             alpha * 1.4426950408889634f, w.tri, T, w.xsc, sms, st));
    }
  }
  for (int h = 0; h < Hq && xattn_use_cublas(); ++h) {
    if (h % grp == 0) {
      reshape_kernel<<<rgrid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(k), w.kr, n, Hkv,
                                           h / grp, 0);
      MT_TRY(check_launch("xattn reshape k"));
    }
    reshape_kernel<<<rgrid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(q), w.qr, n, Hq, h, 1);
    MT_TRY(check_launch("xattn reshape q"));
    for (int64_t i0 = 0; i0 < n; i0 += w.R) {
      const int64_t rows = i0 + w.R <= n ? w.R : n - i0;
      const int64_t cols = i0 + rows;  // causal bound
      // row-major C[rows][cols] = Qr[i0:] Kr[:cols]^T  <=>  col-major C^T = Kr^T' Qr
      if (cublasGemmEx(hb, CUBLAS_OP_T, CUBLAS_OP_N, (int)cols, (int)rows, kWide, &alpha, w.kr,
                       CUDA_R_16BF, kWide, w.qr + i0 * kWide, CUDA_R_16BF, kWide, &beta, w.C,
                       CUDA_R_32F, (int)cols, CUBLAS_COMPUTE_32F,
                       CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
        return fail(MT_ECUDA, "cublasGemmEx failed");
      softmax_blocksum_kernel<<<(unsigned)(rows / kR), 256, 0, st>>>(w.C, cols, i0,
                                                                     w.tri + (int64_t)h * T);
      MT_TRY(check_launch("xattn softmax_blocksum"));
    }
  }
  if (block_scores)
    cudaMemcpyAsync(block_scores, w.tri, (size_t)Hq * T * 4, cudaMemcpyDeviceToDevice, st);
  seg_init_kernel<<<rgrid, 256, 0, st>>>(nI, Hq, w.off, w.jv);
  MT_TRY(check_launch("xattn seg_init"));
  size_t tb = w.cub_bytes;
  if (cub::DeviceSegmentedSort::StableSortPairsDescending(w.cub_tmp, tb, w.tri, w.keys, w.jv,
                                                          w.jv_sorted, Hq * T, Hq * nI, w.off,
                                                          w.off + 1, st) != cudaSuccess)
    return fail(MT_ECUDA, "xattn segmented sort failed");
  cudaMemsetAsync(w.bits, 0, (size_t)Hq * nI * ((nI + 31) / 32) * 4, st);
  const int64_t warps = (int64_t)Hq * nI;
  select_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(
      w.keys, w.jv_sorted, w.tri, nI, Hq, prm->threshold, w.bits);
  MT_TRY(check_launch("xattn select"));
  count64_kernel<<<rgrid, 256, 0, st>>>(w.bits, nI, Hq, w.cnt);
  tb = w.cub_bytes;
  if (cub::DeviceScan::ExclusiveSum(w.cub_tmp, tb, w.cnt, w.scan, Hq * nb + 1, st) != cudaSuccess)
    return fail(MT_ECUDA, "xattn scan failed");
  ptr_layout_kernel<<<rgrid, 256, 0, st>>>(w.scan, nb, Hq, blk_ptr);
  MT_TRY(check_launch("xattn ptr"));
  if (cudaMemcpyAsync(n_blk, w.scan + (int64_t)Hq * nb, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return fail(MT_ECUDA, "xattn total copy failed");
  return MT_OK;
}

extern "C" mt_status mt_xattn_index_fill(const mt_shape* sh, const mt_xattn_params* prm,
                                         const int64_t* blk_ptr, int32_t* blk_idx, int64_t cap,
                                         int64_t n_blk, void* ws, size_t ws_bytes,
                                         mt_stream_t stream) {
  MT_TRY(check_x(sh, prm));
  if (!blk_ptr || (n_blk > 0 && !blk_idx)) return fail(MT_ESHAPE, "NULL argument");
  if (cap < n_blk) return fail(MT_ECAPACITY, "capacity %lld < %lld", (long long)cap, (long long)n_blk);
  XWs w = carve(ws, sh);
  if (!ws || ws_bytes < w.total) return fail(MT_EWORKSPACE, "workspace %zu < %zu", ws_bytes, w.total);
  const int64_t nI = sh->seq_len / kB;
  const int Hq = sh->n_q_heads;
  const int64_t warps = (int64_t)Hq * 2 * nI;
  fill64_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      w.bits, nI, Hq, blk_ptr, blk_idx);
  return check_launch("xattn fill");
}
