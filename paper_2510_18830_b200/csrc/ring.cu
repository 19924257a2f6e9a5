// ring.cu — balanced (block-striped) sparse ring attention over NCCL, flat and
// hierarchical (Alg. 2).
//
// Every rank keeps its striped Q/O and the KV chunks circulate.  The
// schedule (which origin each rank holds at each step) is computed on the host
// by literally passing chunk ids through the flat ring (send r+1 / recv r-1,
// reading R13) or the two-level ring (outer r +- G posted at the start of each
// outer step with the chunk held then, inner node_base + (l +- 1) mod G;
// readings R14-R16), exactly as the CPU oracle's ring.schedule does.
//
// Forward: per step, the KV exchange for the next step runs on comm streams
// while the sparse forward kernel (attn_fwd_step) merges the held chunk into the
// fp32 running (O, LSE) (merge_out_and_lse); the last step writes bf16 O.
// Backward (Table 4 rows P:712-716; reading R17 variant "return to owner"):
// per step the held chunk's dK/dV partial is computed into a zeroed fp32
// buffer and sent straight to the chunk's owner, which adds it into its own
// accumulators; dQ stays local.  All transfers overlap the next step's compute.
#include <vector>

#include "comm.cuh"
#include <cudaTypedefs.h>
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
mt_status check_shape(const mt_shape* sh, int W);
mt_status check_index(const mt_vs_index* idx, const mt_shape* sh);
mt_status check_device();
int device_num_sms();

// held[t][x]: origin of the KV chunk rank x holds at step t.
std::vector<std::vector<int>> ring_schedule(int W, int G) {
  const int nout = W / G;
  std::vector<int> held(W);
  for (int x = 0; x < W; ++x) held[x] = x;
  std::vector<std::vector<int>> steps;
  for (int i = 0; i < nout; ++i) {
    std::vector<int> outer(W, -1);
    if (i < nout - 1)
      for (int x = 0; x < W; ++x) outer[(x + G) % W] = held[x];
    for (int j = 0; j < G; ++j) {
      steps.push_back(held);
      if (j < G - 1) {
        std::vector<int> nxt(W, -1);
        for (int x = 0; x < W; ++x) {
          const int n = x / G, l = x % G;
          nxt[n * G + (l + 1) % G] = held[x];
        }
        held = nxt;
      }
    }
    if (i < nout - 1) held = outer;
  }
  return steps;
}

namespace {

__global__ void add_f32_kernel(float* __restrict__ y, const float* __restrict__ x, int64_t n) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    float4 a = *reinterpret_cast<float4*>(y + i);
    const float4 b = *reinterpret_cast<const float4*>(x + i);
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    *reinterpret_cast<float4*>(y + i) = a;
  } else {
    for (int64_t j = i; j < n; ++j) y[j] += x[j];
  }
}

mt_status add_f32(float* y, const float* x, int64_t n, cudaStream_t st) {
  const int64_t per = 256 * 4;
  add_f32_kernel<<<(unsigned)((n + per - 1) / per), 256, 0, st>>>(y, x, n);
  return check_launch("add_f32");
}

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

struct RingWs {
  void* plan;
  uint8_t* kv[4];   // each: K then V, [S_loc][Hkv][128] bf16 x 2
  float* o_acc;     // fwd: [S_loc][Hq][128]
  float* D;         // bwd: [Hq][S_loc]
  float* dq;        // bwd: [S_loc][Hq][128]
  float* dkv_acc;   // bwd: own chunk dK, dV fp32 [2][S_loc][Hkv][128]
  float* part[2];   // bwd: partial dK/dV of the held chunk
  float* recv[2];   // bwd: incoming partials of the own chunk
  size_t total;
};

RingWs carve_ring(void* base, const mt_shape* sh, int W, bool bwd) {
  const int64_t S_loc = sh->seq_len / W;
  const int Hq = sh->n_q_heads, Hkv = sh->n_kv_heads;
  const size_t kvb = (size_t)S_loc * Hkv * 128 * 2 * 2;
  const size_t dkvb = (size_t)S_loc * Hkv * 128 * 4 * 2;
  uint8_t* p = static_cast<uint8_t*>(base);
  size_t off = 0;
  auto take = [&](size_t b) {
    void* r = p ? p + off : nullptr;
    off = al(off + b);
    return r;
  };
  RingWs w{};
  w.plan = take(vs_plan_bytes(sh->seq_len, Hq, W));
  for (int i = 0; i < 4; ++i) w.kv[i] = (uint8_t*)take(kvb);
  if (!bwd) {
    w.o_acc = (float*)take((size_t)S_loc * Hq * 128 * 4);
  } else {
    w.D = (float*)take((size_t)Hq * S_loc * 4);
    w.dq = (float*)take((size_t)S_loc * Hq * 128 * 4);
    w.dkv_acc = (float*)take(dkvb);
    for (int i = 0; i < 2; ++i) w.part[i] = (float*)take(dkvb);
    for (int i = 0; i < 2; ++i) w.recv[i] = (float*)take(dkvb);
  }
  w.total = off;
  return w;
}


}  // namespace
}  // namespace mt

using namespace mt;

extern "C" size_t mt_ring_attn_workspace_bytes(const mt_shape* sh, int world, int backward) {
  if (!sh || world <= 0) return 0;
  return carve_ring(nullptr, sh, world, backward != 0).total;
}

namespace mt {
namespace {
#ifdef MT_HAVE_NCCL
// SMs for the ring's attention launches: all but the ones kept free for NCCL.
int ring_sms(const mt_comm* c, bool bwd) {
  const int n = device_num_sms() - (c->world > 1 ? (bwd ? c->reserve_sms_bwd : c->reserve_sms) : 0);
  return n > 0 ? n : 1;
}

// KV rotation shared by the forward and backward rings.  Buffers: the caller's
// chunk, two inner buffers (alternating receive targets of the node ring) and
// two outer buffers (alternating receive targets of the outer ring).  The chunk
// held at the start of an outer step is only read (outer send + compute) until
// that outer step ends (reading R16).
struct KVRing {
  mt_comm* c;
  int W, G, r;
  size_t half;  // elements of K (= of V) per chunk
  uint8_t* ib[2];
  uint8_t* ob[2];
  const __nv_bfloat16* curK;
  const __nv_bfloat16* curV;
  int inner_sel = 0, outer_sel = 0;
  int pass = 0;  // profiling: 0 forward, 1 backward
  cudaEvent_t ev_c, ev_i, ev_o;
  bool inner_pending = false, outer_pending = false;

  KVRing(mt_comm* cm, int64_t S_loc, int Hkv, const void* k, const void* v, uint8_t* const* bufs)
      : c(cm), W(cm->world), G(cm->inner), r(cm->rank) {
    half = (size_t)S_loc * Hkv * 128;
    ib[0] = bufs[0]; ib[1] = bufs[1]; ob[0] = bufs[2]; ob[1] = bufs[3];
    curK = (const __nv_bfloat16*)k;
    curV = (const __nv_bfloat16*)v;
    cudaEventCreateWithFlags(&ev_c, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_i, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_o, cudaEventDisableTiming);
  }
  ~KVRing() {
    cudaEventDestroy(ev_c);
    cudaEventDestroy(ev_i);
    cudaEventDestroy(ev_o);
  }
  mt_status xchg(ncclComm_t nc, cudaStream_t cs, const __nv_bfloat16* k, const __nv_bfloat16* v,
                 int to, __nv_bfloat16* dst, int from) {
    ncclGroupStart();
    ncclSend(k, half, ncclBfloat16, to, nc, cs);
    ncclSend(v, half, ncclBfloat16, to, nc, cs);
    ncclRecv(dst, half, ncclBfloat16, from, nc, cs);
    ncclRecv(dst + half, half, ncclBfloat16, from, nc, cs);
    MT_TRY(nccl_check(ncclGroupEnd(), "ring exchange"));
    emu_inbound(c, from, 2 * half * sizeof(__nv_bfloat16), cs);
    return MT_OK;
  }
  // Post the transfers of step t (before its compute).  `ready` = the stream
  // whose prior work must finish before receive targets are overwritten.
  mt_status post(int t, cudaStream_t compute) {
    const int nout = W / G, i = t / G, j = t % G;
    const int n = r / G, l = r % G;
    cudaEventRecord(ev_c, compute);
    if (j == 0 && i < nout - 1) {  // outer: send the chunk held now (start of outer step)
      cudaStreamWaitEvent(c->comm_stream2, ev_c, 0);
      __nv_bfloat16* dst = (__nv_bfloat16*)ob[outer_sel];
      prof_mark(c, pass, t, RingProfile::kOuterB, c->comm_stream2);
      MT_TRY(xchg(c->nccl2, c->comm_stream2, curK, curV, (r + G) % W, dst, (r - G + W) % W));
      prof_mark(c, pass, t, RingProfile::kOuterE, c->comm_stream2);
      cudaEventRecord(ev_o, c->comm_stream2);
      outer_pending = true;
    }
    if (j < G - 1) {
      cudaStreamWaitEvent(c->comm_stream, ev_c, 0);
      __nv_bfloat16* dst = (__nv_bfloat16*)ib[inner_sel];
      prof_mark(c, pass, t, RingProfile::kInnerB, c->comm_stream);
      MT_TRY(xchg(c->nccl, c->comm_stream, curK, curV, n * G + (l + 1) % G, dst,
                  n * G + (l + G - 1) % G));
      prof_mark(c, pass, t, RingProfile::kInnerE, c->comm_stream);
      cudaEventRecord(ev_i, c->comm_stream);
      inner_pending = true;
    }
    return MT_OK;
  }
  // After the compute of step t: make the next held chunk current.
  void advance(int t, cudaStream_t compute) {
    const int j = t % G;
    if (j < G - 1 && inner_pending) {
      cudaStreamWaitEvent(compute, ev_i, 0);
      curK = (const __nv_bfloat16*)ib[inner_sel];
      curV = curK + half;
      inner_sel ^= 1;
      inner_pending = false;
    } else if (j == G - 1 && outer_pending) {
      cudaStreamWaitEvent(compute, ev_o, 0);
      curK = (const __nv_bfloat16*)ob[outer_sel];
      curV = curK + half;
      outer_sel ^= 1;
      outer_pending = false;
    }
  }
};
#endif
}  // namespace
}  // namespace mt

#ifdef MT_HAVE_NCCL
namespace mt {
CeStreamValueFn ce_wait_fn();
CeStreamValueFn ce_write_fn();
namespace {
// Flat forward ring over the copy engines (mt_comm_register_workspace).  Counters (uint32,
// monotone since registration; waits compare the signed difference, so they wrap safely):
//   ready  (my flag word 0, written by rank r-1): KV transfers received;
//   done   (my flag word 16, written by rank r+1): compute steps rank r+1 has finished.
// In call e (calls since registration) at step t:
//   send (t < W-1): comm stream waits ready >= e(W-1) + t (the chunk I hold arrived; t >= 1),
//                   and done >= eW + t (rank r+1 finished its steps < t, so its receive slot
//                   t % 2 -- last read at step t-1 or in an earlier call -- is free);
//                   copies K and V into rank r+1's slot t % 2 (cudaMemcpyAsync: copy engines,
//                   no SM), then writes rank r+1's ready = e(W-1) + t + 1;
//   compute:        waits ready >= e(W-1) + t (t >= 1), runs step t on slot (t-1) % 2, then
//                   writes rank r-1's done = eW + t + 1.
mt_status ring_fwd_ce(mt_comm* c, const std::vector<std::vector<int>>& sched, const VSPlan& plan,
                      int r, int nloc, int64_t S_loc, int Hkv, const void* q_loc, const void* k_loc,
                      const void* v_loc, void* o_loc, float* o_acc, float* lse_loc,
                      uint8_t* const* kv, uint8_t* ws, cudaStream_t stream) {
  auto wait = ce_wait_fn();
  auto write = ce_write_fn();
  if (!wait || !write) return fail(MT_EUNSUPPORTED, "stream memory operations unavailable");
  const int W = c->world;
  const uint32_t e = c->ce_calls++;
  const size_t half = (size_t)S_loc * Hkv * 128 * sizeof(__nv_bfloat16);
  uint32_t* my_flags = reinterpret_cast<uint32_t*>(ws + c->ce_bytes - 256);
  uint32_t* next_ready = reinterpret_cast<uint32_t*>(c->ce_next_ws + c->ce_next_bytes - 256);
  uint32_t* prev_done = reinterpret_cast<uint32_t*>(c->ce_prev_ws + c->ce_prev_bytes - 256) + 16;
  const CUdeviceptr d_ready = reinterpret_cast<CUdeviceptr>(my_flags);
  const CUdeviceptr d_done = reinterpret_cast<CUdeviceptr>(my_flags + 16);
  const uint32_t rbase = e * (uint32_t)(W - 1), cbase = e * (uint32_t)W;
  cudaStream_t cs = c->comm_stream;
  // the caller's chunk is complete once the compute stream reaches this point
  cudaEventRecord(c->ev_ready, stream);
  cudaStreamWaitEvent(cs, c->ev_ready, 0);
  const __nv_bfloat16* curK = static_cast<const __nv_bfloat16*>(k_loc);
  const __nv_bfloat16* curV = static_cast<const __nv_bfloat16*>(v_loc);
  cudaEvent_t ev_sent;  // the send of step t read the chunk compute step t reads
  cudaEventCreateWithFlags(&ev_sent, cudaEventDisableTiming);
  for (int t = 0; t < W; ++t) {
    if (t >= 1) {
      curK = reinterpret_cast<const __nv_bfloat16*>(kv[(t - 1) & 1]);
      curV = curK + half / sizeof(__nv_bfloat16);
    }
    if (t < W - 1) {  // ---- send the chunk held at step t to rank r+1's slot t % 2
      if (t >= 1 && wait(cs, d_ready, rbase + (uint32_t)t, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        return fail(MT_ECUDA, "cuStreamWaitValue32 (ready)");
      if (wait(cs, d_done, cbase + (uint32_t)t, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        return fail(MT_ECUDA, "cuStreamWaitValue32 (done)");
      uint8_t* dst = c->ce_next_ws + (kv[t & 1] - ws);
      prof_mark(c, 0, t, RingProfile::kInnerB, cs);
      if (cudaMemcpyAsync(dst, curK, half, cudaMemcpyDeviceToDevice, cs) != cudaSuccess ||
          cudaMemcpyAsync(dst + half, curV, half, cudaMemcpyDeviceToDevice, cs) != cudaSuccess)
        return fail(MT_ECUDA, "ring copy to the next rank failed");
      prof_mark(c, 0, t, RingProfile::kInnerE, cs);
      if (write(cs, reinterpret_cast<CUdeviceptr>(next_ready), rbase + (uint32_t)t + 1u,
                CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
        return fail(MT_ECUDA, "cuStreamWriteValue32 (ready)");
      cudaEventRecord(ev_sent, cs);
    }
    // ---- compute step t
    if (t >= 1 && wait(stream, d_ready, rbase + (uint32_t)t, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return fail(MT_ECUDA, "cuStreamWaitValue32 (compute)");
    prof_mark(c, 0, t, RingProfile::kCompB, stream);
    MT_TRY(attn_fwd_step(plan, r, sched[t][r], nloc, q_loc, curK, curV, o_loc, o_acc, lse_loc,
                         t == 0, t == W - 1, device_num_sms(), stream));
    prof_mark(c, 0, t, RingProfile::kCompE, stream);
    // my slot (t-1) % 2 is free once compute step t and its forwarding copy are done
    if (t < W - 1) cudaStreamWaitEvent(stream, ev_sent, 0);
    if (write(stream, reinterpret_cast<CUdeviceptr>(prev_done), cbase + (uint32_t)t + 1u,
              CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
      return fail(MT_ECUDA, "cuStreamWriteValue32 (done)");
  }
  cudaEventDestroy(ev_sent);
  // the comm stream's last copy read the chunk of step W-2; later calls reuse the buffers
  cudaEventRecord(c->ev_done, cs);
  cudaStreamWaitEvent(stream, c->ev_done, 0);
  return check_launch("mt_ring_attn_fwd (copy engines)");
}
}  // namespace
}  // namespace mt
#endif

extern "C" mt_status mt_ring_attn_fwd(mt_comm* comm, const mt_shape* sh, const void* q_loc,
                                      const void* k_loc, const void* v_loc,
                                      const mt_vs_index* idx, void* o_loc, float* lse_loc,
                                      void* ws, size_t ws_bytes, mt_stream_t stream) {
#ifdef MT_HAVE_NCCL
  if (!comm) return fail(MT_ESHAPE, "comm is NULL");
  const int W = comm->world, r = comm->rank;
  MT_TRY(check_shape(sh, W));
  MT_TRY(check_index(idx, sh));
  if (!q_loc || !k_loc || !v_loc || !o_loc || !lse_loc) return fail(MT_ESHAPE, "NULL tensor");
  RingWs w = carve_ring(ws, sh, W, false);
  if (!ws || ws_bytes < w.total) return fail(MT_EWORKSPACE, "workspace %zu < %zu", ws_bytes, w.total);
  MT_TRY(check_device());
  const int64_t S_loc = sh->seq_len / W;
  const int nloc = (int)(S_loc / 64);
  VSPlan plan;
  MT_TRY(vs_plan_build(&plan, sh->seq_len, sh->n_q_heads, sh->n_kv_heads, W, sh->layout,
                       idx->v_cnt,
                       idx->v_idx, idx->v_stride, idx->s_cnt, idx->s_off, (int)idx->s_stride,
                       w.plan, stream));
  const auto sched = ring_schedule(W, comm->inner);
  if (comm->prof) comm->prof->steps[0] = 0;
  if (comm->ce_ok && ws == comm->ce_ws && ws_bytes == comm->ce_bytes && comm->inner == W &&
      comm->emu_gbps <= 0.0)
    return ring_fwd_ce(comm, sched, plan, r, nloc, S_loc, sh->n_kv_heads, q_loc, k_loc, v_loc,
                       o_loc, w.o_acc, lse_loc, w.kv, static_cast<uint8_t*>(ws), stream);
  KVRing ring(comm, S_loc, sh->n_kv_heads, k_loc, v_loc, w.kv);
  for (int t = 0; t < W; ++t) {
    MT_TRY(ring.post(t, stream));
    prof_mark(comm, 0, t, RingProfile::kCompB, stream);
    MT_TRY(attn_fwd_step(plan, r, sched[t][r], nloc, q_loc, ring.curK, ring.curV, o_loc, w.o_acc,
                         lse_loc, t == 0, t == W - 1, ring_sms(comm, false), stream));
    prof_mark(comm, 0, t, RingProfile::kCompE, stream);
    ring.advance(t, stream);
  }
  return check_launch("mt_ring_attn_fwd");
#else
  (void)comm; (void)sh; (void)q_loc; (void)k_loc; (void)v_loc; (void)idx; (void)o_loc;
  (void)lse_loc; (void)ws; (void)ws_bytes; (void)stream;
  return fail(MT_EUNSUPPORTED, "built without NCCL");
#endif
}

extern "C" mt_status mt_ring_attn_bwd(mt_comm* comm, const mt_shape* sh, const void* q_loc,
                                      const void* k_loc, const void* v_loc, const void* o_loc,
                                      const float* lse_loc, const void* dO_loc,
                                      const mt_vs_index* idx, void* dq_loc, void* dk_loc,
                                      void* dv_loc, void* ws, size_t ws_bytes,
                                      mt_stream_t stream) {
#ifdef MT_HAVE_NCCL
  if (!comm) return fail(MT_ESHAPE, "comm is NULL");
  const int W = comm->world, r = comm->rank;
  MT_TRY(check_shape(sh, W));
  MT_TRY(check_index(idx, sh));
  if (!q_loc || !k_loc || !v_loc || !o_loc || !lse_loc || !dO_loc || !dq_loc || !dk_loc || !dv_loc)
    return fail(MT_ESHAPE, "NULL tensor");
  RingWs w = carve_ring(ws, sh, W, true);
  if (!ws || ws_bytes < w.total) return fail(MT_EWORKSPACE, "workspace %zu < %zu", ws_bytes, w.total);
  MT_TRY(check_device());
  const int64_t S_loc = sh->seq_len / W;
  const int nloc = (int)(S_loc / 64);
  const int Hq = sh->n_q_heads, Hkv = sh->n_kv_heads;
  const int64_t nkv = S_loc * Hkv * 128;  // floats of dK (= of dV)
  VSPlan plan;
  MT_TRY(vs_plan_build(&plan, sh->seq_len, Hq, Hkv, W, sh->layout, idx->v_cnt, idx->v_idx, idx->v_stride,
                       idx->s_cnt, idx->s_off, (int)idx->s_stride, w.plan, stream));
  MT_TRY(attn_bwd_preprocess(o_loc, dO_loc, w.D, S_loc, Hq, stream));
  cudaMemsetAsync(w.dq, 0, (size_t)S_loc * Hq * 128 * 4, stream);
  cudaMemsetAsync(w.dkv_acc, 0, (size_t)nkv * 2 * 4, stream);
  const auto sched = ring_schedule(W, comm->inner);
  KVRing ring(comm, S_loc, Hkv, k_loc, v_loc, w.kv);
  ring.pass = 1;
  if (comm->prof) comm->prof->steps[1] = 0;
  cudaEvent_t ev_done, ev_p[2];
  cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming);
  for (int i = 0; i < 2; ++i) cudaEventCreateWithFlags(&ev_p[i], cudaEventDisableTiming);
  bool p_pending[2] = {false, false}, r_pending[2] = {false, false};
  mt_status st = MT_OK;
  for (int t = 0; t < W && st == MT_OK; ++t) {
    const int s = sched[t][r];
    int holder = -1;  // rank holding MY chunk at step t
    for (int x = 0; x < W; ++x)
      if (sched[t][x] == r) holder = x;
    const int b = t & 1;
    // buffers of step t-2 may be reused only after their transfer finished
    if (p_pending[b] || r_pending[b]) {
      cudaStreamWaitEvent(stream, ev_p[b], 0);
      if (r_pending[b]) MT_TRY(add_f32(w.dkv_acc, w.recv[b], 2 * nkv, stream));
      p_pending[b] = r_pending[b] = false;
    }
    MT_TRY(ring.post(t, stream));
    float* dk = w.dkv_acc;
    if (s != r) {
      cudaMemsetAsync(w.part[b], 0, (size_t)nkv * 2 * 4, stream);
      dk = w.part[b];
    }
    prof_mark(comm, 1, t, RingProfile::kCompB, stream);
    MT_TRY(attn_bwd_step(plan, r, s, nloc, q_loc, ring.curK, ring.curV, dO_loc, lse_loc, w.D,
                         w.dq, dk, dk + nkv, ring_sms(comm, true), stream));
    prof_mark(comm, 1, t, RingProfile::kCompE, stream);
    // partial of the held chunk -> its owner; my own chunk's partial <- its holder
    if (s != r || holder != r) {
      cudaEventRecord(ev_done, stream);
      cudaStreamWaitEvent(comm->comm_stream3, ev_done, 0);
      prof_mark(comm, 1, t, RingProfile::kDkvB, comm->comm_stream3);
      ncclGroupStart();
      if (s != r) ncclSend(w.part[b], 2 * nkv, ncclFloat32, s, comm->nccl3, comm->comm_stream3);
      if (holder != r)
        ncclRecv(w.recv[b], 2 * nkv, ncclFloat32, holder, comm->nccl3, comm->comm_stream3);
      if (ncclGroupEnd() != ncclSuccess) st = fail(MT_ENCCL, "dKV partial exchange failed");
      if (holder != r) emu_inbound(comm, holder, (size_t)nkv * 2 * 4, comm->comm_stream3);
      prof_mark(comm, 1, t, RingProfile::kDkvE, comm->comm_stream3);
      cudaEventRecord(ev_p[b], comm->comm_stream3);
      p_pending[b] = (s != r);
      r_pending[b] = (holder != r);
      if (!p_pending[b] && !r_pending[b]) p_pending[b] = true;  // keep the event wait
    }
    ring.advance(t, stream);
  }
  for (int b = 0; b < 2 && st == MT_OK; ++b)
    if (p_pending[b] || r_pending[b]) {
      cudaStreamWaitEvent(stream, ev_p[b], 0);
      if (r_pending[b]) st = add_f32(w.dkv_acc, w.recv[b], 2 * nkv, stream);
    }
  cudaEventDestroy(ev_done);
  for (int i = 0; i < 2; ++i) cudaEventDestroy(ev_p[i]);
  MT_TRY(st);
  return f32_to_bf16_x3(w.dq, dq_loc, S_loc * Hq * 128, w.dkv_acc, dk_loc, nkv,
                        w.dkv_acc + nkv, dv_loc, nkv, stream);
#else
  (void)comm; (void)sh; (void)q_loc; (void)k_loc; (void)v_loc; (void)o_loc; (void)lse_loc;
  (void)dO_loc; (void)idx; (void)dq_loc; (void)dk_loc; (void)dv_loc; (void)ws; (void)ws_bytes;
  (void)stream;
  return fail(MT_EUNSUPPORTED, "built without NCCL");
#endif
}

extern "C" mt_status mt_ring_schedule(int world, int inner, int32_t* out) {
  if (!out || world < 1) return fail(MT_ESHAPE, "bad arguments");
  if (inner <= 0) inner = world;
  if (world % inner) return fail(MT_ESHAPE, "inner must divide world");
  const auto s = ring_schedule(world, inner);
  for (int t = 0; t < world; ++t)
    for (int x = 0; x < world; ++x) out[t * world + x] = s[t][x];
  return MT_OK;
}
