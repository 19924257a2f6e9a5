// api_attn.cu — C-ABI entry points for the sparse attention forward/backward
// (include/mtsa.h).  Validation is synchronous; compute is enqueued on the
// caller's stream.
#include <mutex>

#include <cstdlib>

#include "common.cuh"
#include "plan.cuh"

namespace mt {

size_t vs_plan_bytes(int64_t S, int Hq, int W);
mt_status vs_plan_build(VSPlan* out, int64_t S, int Hq, int Hkv, int W, int layout,
                        const int32_t* v_cnt,
                        const int32_t* v_idx, int64_t v_stride, const int32_t* s_cnt,
                        const int32_t* s_off, int s_stride, void* ws, cudaStream_t st);
mt_status attn_fwd_step(const VSPlan& plan, int r, int s, int nloc, const void* q,
                        const void* k, const void* v, void* o, float* o_acc, float* lse,
                        int first, int last, int num_sms, cudaStream_t st);

// SM count of the CURRENT device, cached per device (a process may drive several GPUs
// from several threads: the cache is per device and its fill is serialised).
int device_num_sms() {
  constexpr int kMaxDev = 64;
  static int n[kMaxDev] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev) {
    int x = 0;
    cudaDeviceGetAttribute(&x, cudaDevAttrMultiProcessorCount, dev);
    return x > 0 ? x : 148;
  }
  std::lock_guard<std::mutex> lk(mu);
  if (n[dev] == 0) {
    cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
    if (n[dev] <= 0) n[dev] = 148;
  }
  return n[dev];
}

mt_status check_device() {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(MT_ECUDA, "no CUDA device");
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0)
    return fail(MT_EUNSUPPORTED, "device is sm_%d%d; this library is built for sm_100a", major,
                minor);
  return MT_OK;
}

mt_status check_shape(const mt_shape* sh, int W) {
  if (!sh) return fail(MT_ESHAPE, "shape is NULL");
  if (sh->head_dim != 128) return fail(MT_EUNSUPPORTED, "head_dim must be 128 (got %d)", sh->head_dim);
  if (sh->block != 64) return fail(MT_EUNSUPPORTED, "block must be 64 (got %d)", sh->block);
  if (sh->last_q != 0 && sh->last_q != 64)
    return fail(MT_EUNSUPPORTED, "last_q must be 64 (got %d; reading R2)", sh->last_q);
  if (sh->n_q_heads <= 0 || sh->n_kv_heads <= 0 || sh->n_q_heads % sh->n_kv_heads)
    return fail(MT_ESHAPE, "bad head counts Hq=%d Hkv=%d", sh->n_q_heads, sh->n_kv_heads);
  if (sh->seq_len < 64 || sh->seq_len % 64)
    return fail(MT_EWINDOW, "seq_len %lld must be a positive multiple of 64",
                (long long)sh->seq_len);
  if (W <= 0) return fail(MT_ESHAPE, "world must be >= 1");
  if (sh->seq_len % (64LL * W))
    return fail(MT_ELAYOUT, "seq_len %lld is not a multiple of 64 * world (%d)",
                (long long)sh->seq_len, W);
  if (sh->seq_len / 64 > (1LL << 24)) return fail(MT_ESHAPE, "seq_len too large");
  if (sh->layout != MT_LAYOUT_STRIPED && sh->layout != MT_LAYOUT_ZIGZAG)
    return fail(MT_ESHAPE, "unknown layout %d", sh->layout);
  if (sh->layout == MT_LAYOUT_ZIGZAG && W > 1 && sh->seq_len % (128LL * W))
    return fail(MT_ELAYOUT, "zigzag: seq_len %lld is not a multiple of 128 * world (%d)",
                (long long)sh->seq_len, W);
  return MT_OK;
}

// Row strides must hold a full list (v_stride >= S, s_stride >= S/64): the plan builder
// reads up to min(count, stride) entries per head and drops out-of-range entries, so a
// malformed caller index cannot make it write outside its own head's plan rows.
mt_status check_index(const mt_vs_index* idx, const mt_shape* sh) {
  if (!idx || !idx->v_cnt || !idx->v_idx || !idx->s_cnt || !idx->s_off)
    return fail(MT_ESHAPE, "index pointers must be non-NULL");
  if (idx->v_stride < 1 || idx->s_stride < 1 || idx->s_stride > (1LL << 30))
    return fail(MT_ESHAPE, "bad index strides");
  if (sh && (idx->v_stride < sh->seq_len || idx->s_stride < sh->seq_len / 64))
    return fail(MT_ESHAPE, "index strides (%lld, %lld) below (seq_len, seq_len/64) = (%lld, %lld)",
                (long long)idx->v_stride, (long long)idx->s_stride, (long long)sh->seq_len,
                (long long)(sh->seq_len / 64));
  return MT_OK;
}

}  // namespace mt

using namespace mt;

extern "C" size_t mt_sparse_attn_fwd_workspace_bytes(const mt_shape* sh, int world) {
  if (!sh || world <= 0) return 0;
  return vs_plan_bytes(sh->seq_len, sh->n_q_heads, world);
}

extern "C" mt_status mt_attn_fwd_step(const mt_shape* sh, int world, int rank, int origin,
                                      int first, int last, const void* q_loc,
                                      const void* k_chunk, const void* v_chunk,
                                      const mt_vs_index* idx, void* o, float* o_acc, float* lse,
                                      void* ws, size_t ws_bytes, mt_stream_t stream) {
  MT_TRY(check_shape(sh, world));
  MT_TRY(check_index(idx, sh));
  if (rank < 0 || rank >= world || origin < 0 || origin >= world)
    return fail(MT_ESHAPE, "rank/origin out of range");
  if (!q_loc || !k_chunk || !v_chunk || !lse) return fail(MT_ESHAPE, "NULL tensor");
  if (last && !o) return fail(MT_ESHAPE, "o must be non-NULL when last");
  if (!(first && last) && !o_acc) return fail(MT_ESHAPE, "o_acc must be non-NULL");
  const size_t need = mt_sparse_attn_fwd_workspace_bytes(sh, world);
  if (!ws || ws_bytes < need)
    return fail(MT_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  MT_TRY(check_device());
  VSPlan plan;
  MT_TRY(vs_plan_build(&plan, sh->seq_len, sh->n_q_heads, sh->n_kv_heads, world, sh->layout,
                       idx->v_cnt,
                       idx->v_idx, idx->v_stride, idx->s_cnt, idx->s_off, (int)idx->s_stride, ws,
                       stream));
  const int nloc = (int)(sh->seq_len / 64 / world);
  return attn_fwd_step(plan, rank, origin, nloc, q_loc, k_chunk, v_chunk, o, o_acc, lse, first,
                       last, device_num_sms(), stream);
}

extern "C" mt_status mt_sparse_attn_fwd(const mt_shape* sh, const void* q, const void* k,
                                        const void* v, const mt_vs_index* idx, void* o,
                                        float* lse, void* ws, size_t ws_bytes,
                                        mt_stream_t stream) {
  return mt_attn_fwd_step(sh, 1, 0, 0, 1, 1, q, k, v, idx, o, nullptr, lse, ws, ws_bytes, stream);
}

// ------------------------------------------------------------------ backward
namespace mt {
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

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct BwdWs {
  void* plan;
  float* D;
  float* dq;
  float* dk;
  float* dv;
  size_t total;
};

static BwdWs carve_bwd(void* base, const mt_shape* sh) {
  const int64_t S = sh->seq_len;
  const int Hq = sh->n_q_heads, Hkv = sh->n_kv_heads;
  uint8_t* p = static_cast<uint8_t*>(base);
  size_t off = 0;
  auto take = [&](size_t b) {
    void* r = p ? p + off : nullptr;
    off = align256(off + b);
    return r;
  };
  BwdWs w{};
  w.plan = take(vs_plan_bytes(S, Hq, 1));
  w.D = (float*)take((size_t)Hq * S * 4);
  w.dq = (float*)take((size_t)S * Hq * 128 * 4);
  w.dk = (float*)take((size_t)S * Hkv * 128 * 4);
  w.dv = (float*)take((size_t)S * Hkv * 128 * 4);
  w.total = off;
  return w;
}
}  // namespace mt

extern "C" size_t mt_sparse_attn_bwd_workspace_bytes(const mt_shape* sh) {
  if (!sh) return 0;
  return carve_bwd(nullptr, sh).total;
}

extern "C" size_t mt_attn_step_workspace_bytes(const mt_shape* sh, int world) {
  if (!sh || world <= 0) return 0;
  return vs_plan_bytes(sh->seq_len, sh->n_q_heads, world);
}

extern "C" mt_status mt_sparse_attn_bwd(const mt_shape* sh, const void* q, const void* k,
                                        const void* v, const void* o, const float* lse,
                                        const void* dO, const mt_vs_index* idx, void* dq,
                                        void* dk, void* dv, void* ws, size_t ws_bytes,
                                        mt_stream_t stream) {
  MT_TRY(check_shape(sh, 1));
  MT_TRY(check_index(idx, sh));
  if (!q || !k || !v || !o || !lse || !dO || !dq || !dk || !dv)
    return fail(MT_ESHAPE, "NULL tensor");
  BwdWs w = carve_bwd(ws, sh);
  if (!ws || ws_bytes < w.total)
    return fail(MT_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, w.total);
  MT_TRY(check_device());
  const int64_t S = sh->seq_len;
  const int Hq = sh->n_q_heads, Hkv = sh->n_kv_heads;
  VSPlan plan;
  MT_TRY(vs_plan_build(&plan, S, Hq, Hkv, 1, 0, idx->v_cnt, idx->v_idx, idx->v_stride, idx->s_cnt,
                       idx->s_off, (int)idx->s_stride, w.plan, stream));
  // D, and the fp32 dQ / dK / dV accumulators zeroed in the same pass
  static const bool memset_acc = getenv("MT_BWD_MEMSET") && atoi(getenv("MT_BWD_MEMSET"));
  if (memset_acc) {  // A/B: round 1's separate memset of the accumulators
    MT_TRY(attn_bwd_preprocess(o, dO, w.D, S, Hq, stream));
    cudaMemsetAsync(w.dq, 0, (size_t)((const char*)(w.dv + S * Hkv * 128) - (const char*)w.dq),
                    stream);
  } else {
    MT_TRY(attn_bwd_preprocess(o, dO, w.D, S, Hq, stream, w.dq, w.dk, w.dv, Hkv));
  }
  MT_TRY(attn_bwd_step(plan, 0, 0, (int)(S / 64), q, k, v, dO, lse, w.D, w.dq, w.dk, w.dv,
                       device_num_sms(), stream));
  return f32_to_bf16_x3(w.dq, dq, S * Hq * 128, w.dk, dk, S * Hkv * 128, w.dv, dv, S * Hkv * 128,
                        stream);
}

extern "C" mt_status mt_attn_bwd_preprocess(const mt_shape* sh, int world, const void* o_loc,
                                            const void* dO_loc, float* D_loc,
                                            mt_stream_t stream) {
  MT_TRY(check_shape(sh, world));
  if (!o_loc || !dO_loc || !D_loc) return fail(MT_ESHAPE, "NULL tensor");
  return attn_bwd_preprocess(o_loc, dO_loc, D_loc, sh->seq_len / world, sh->n_q_heads, stream);
}

extern "C" mt_status mt_attn_bwd_step(const mt_shape* sh, int world, int rank, int origin,
                                      const void* q_loc, const void* k_chunk,
                                      const void* v_chunk, const void* dO_loc,
                                      const float* lse_loc, const float* D_loc,
                                      const mt_vs_index* idx, float* dq_acc, float* dk_acc,
                                      float* dv_acc, void* ws, size_t ws_bytes,
                                      mt_stream_t stream) {
  MT_TRY(check_shape(sh, world));
  MT_TRY(check_index(idx, sh));
  if (rank < 0 || rank >= world || origin < 0 || origin >= world)
    return fail(MT_ESHAPE, "rank/origin out of range");
  if (!q_loc || !k_chunk || !v_chunk || !dO_loc || !lse_loc || !D_loc || !dq_acc || !dk_acc ||
      !dv_acc)
    return fail(MT_ESHAPE, "NULL tensor");
  const size_t need = mt_attn_step_workspace_bytes(sh, world);
  if (!ws || ws_bytes < need) return fail(MT_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  MT_TRY(check_device());
  VSPlan plan;
  MT_TRY(vs_plan_build(&plan, sh->seq_len, sh->n_q_heads, sh->n_kv_heads, world, sh->layout,
                       idx->v_cnt,
                       idx->v_idx, idx->v_stride, idx->s_cnt, idx->s_off, (int)idx->s_stride, ws,
                       stream));
  return attn_bwd_step(plan, rank, origin, (int)(sh->seq_len / 64 / world), q_loc, k_chunk,
                       v_chunk, dO_loc, lse_loc, D_loc, dq_acc, dk_acc, dv_acc,
                       device_num_sms(), stream);
}
