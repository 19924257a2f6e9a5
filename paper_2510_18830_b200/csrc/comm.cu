// comm.cu — mt_comm lifecycle and the distributed (context-parallel) index build.
//
// The distributed Alg. 1 index under block-striped keys: the window
// queries live on rank W-1 (its last local block is global block nb-1), every
// rank scores its own keys, and the exact reductions of VS-IDX v1 are completed
// with NCCL collectives whose results do not depend on reduction order:
// broadcast (window Q), all-reduce MAX (fp32 row maxima), all-reduce SUM
// (uint64 fixed-point row sums), all-gather (packed sort keys).  Every rank then
// runs the same sort/top-p and obtains the same global lists, bit-identical to
// the single-GPU result.
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <vector>

#include "comm.cuh"
#include "vsidx.cuh"
#include <cuda_bf16.h>

namespace mt {

#ifdef MT_HAVE_NCCL
struct NcclCollectives final : VSCollectives {
  mt_comm* c;
  explicit NcclCollectives(mt_comm* cm) : c(cm) {}
  mt_status bcast_window(__nv_bfloat16* qwin, size_t n, int root, cudaStream_t st) override {
    return nccl_check(ncclBroadcast(qwin, qwin, n * 2, ncclUint8, root, c->nccl, st),
                      "ncclBroadcast(window)");
  }
  mt_status allreduce_max(float* M, size_t n, cudaStream_t st) override {
    return nccl_check(ncclAllReduce(M, M, n, ncclFloat32, ncclMax, c->nccl, st),
                      "ncclAllReduce(max)");
  }
  mt_status allreduce_sum_u64(unsigned long long* E, size_t n, cudaStream_t st) override {
    return nccl_check(ncclAllReduce(E, E, n, ncclUint64, ncclSum, c->nccl, st),
                      "ncclAllReduce(sum)");
  }
  mt_status allgather_keys(const uint64_t* loc, uint64_t* glob, int Hq, int64_t n_loc,
                           cudaStream_t st) override {
    MT_TRY(nccl_check(ncclGroupStart(), "ncclGroupStart"));
    for (int h = 0; h < Hq; ++h)
      MT_TRY(nccl_check(ncclAllGather(loc + (size_t)h * n_loc, glob + (size_t)h * n_loc * c->world,
                                      (size_t)n_loc, ncclUint64, c->nccl, st),
                        "ncclAllGather(keys)"));
    return nccl_check(ncclGroupEnd(), "ncclGroupEnd");
  }
};
#endif

}  // namespace mt

using namespace mt;

extern "C" mt_status mt_comm_unique_id(uint8_t id[128]) {
#ifdef MT_HAVE_NCCL
  if (!id) return fail(MT_ESHAPE, "id is NULL");
  ncclUniqueId u;
  MT_TRY(nccl_check(ncclGetUniqueId(&u), "ncclGetUniqueId"));
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  memcpy(id, &u, 128);
  return MT_OK;
#else
  (void)id;
  return fail(MT_EUNSUPPORTED, "built without NCCL");
#endif
}

extern "C" mt_status mt_comm_create(const uint8_t id[128], int world, int rank, int inner,
                                    mt_comm** out) {
#ifdef MT_HAVE_NCCL
  if (!id || !out) return fail(MT_ESHAPE, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(MT_ESHAPE, "bad world/rank");
  if (inner <= 0) inner = world;
  if (world % inner) return fail(MT_ESHAPE, "inner ring size %d must divide world %d", inner, world);
  MT_TRY(check_device());
  mt_comm* c = new mt_comm();
  c->world = world;
  c->rank = rank;
  c->inner = inner;
  if (const char* e = getenv("MT_EMU_INTER_GBPS")) c->emu_gbps = atof(e);
  c->emu_node = getenv("MT_EMU_NODE") ? atoi(getenv("MT_EMU_NODE")) : inner;
  if (c->emu_node <= 0) c->emu_node = world;
  if (const char* e = getenv("MT_RING_RESERVE_SMS")) c->reserve_sms = atoi(e);
  if (const char* e = getenv("MT_RING_RESERVE_SMS_BWD")) c->reserve_sms_bwd = atoi(e);
  if (c->reserve_sms < 0 || c->reserve_sms > 32) c->reserve_sms = 0;
  if (c->reserve_sms_bwd < 0 || c->reserve_sms_bwd > 32) c->reserve_sms_bwd = 0;
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  const int cap = c->reserve_sms > c->reserve_sms_bwd ? c->reserve_sms : c->reserve_sms_bwd;
  if (cap > 0) {
    cfg.minCTAs = 1;
    cfg.maxCTAs = cap;
  }
  ncclResult_t r = ncclCommInitRankConfig(&c->nccl, world, u, rank, &cfg);
  if (r != ncclSuccess) {
    delete c;
    return fail(MT_ENCCL, "ncclCommInitRankConfig: %s", ncclGetErrorString(r));
  }
  if (ncclCommSplit(c->nccl, 0, rank, &c->nccl2, &cfg) != ncclSuccess ||
      ncclCommSplit(c->nccl, 0, rank, &c->nccl3, &cfg) != ncclSuccess) {
    ncclCommDestroy(c->nccl);
    delete c;
    return fail(MT_ENCCL, "ncclCommSplit failed");
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi);
  cudaStreamCreateWithPriority(&c->comm_stream2, cudaStreamNonBlocking, hi);
  cudaStreamCreateWithPriority(&c->comm_stream3, cudaStreamNonBlocking, hi);
  cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming);
  *out = c;
  return MT_OK;
#else
  (void)id; (void)world; (void)rank; (void)inner; (void)out;
  return fail(MT_EUNSUPPORTED, "built without NCCL");
#endif
}

namespace {
void sleep_host(void* p) {
  const double ms = *static_cast<double*>(p);
  delete static_cast<double*>(p);
  std::this_thread::sleep_for(std::chrono::microseconds((long long)(ms * 1e3)));
}
}  // namespace

void mt::emu_inbound(mt_comm* c, int from, size_t bytes, cudaStream_t st) {
  if (!c || c->emu_gbps <= 0.0 || from / c->emu_node == c->rank / c->emu_node) return;
  cudaLaunchHostFunc(st, sleep_host, new double(bytes / (c->emu_gbps * 1e9) * 1e3));
}

static void prof_free(mt_comm* c) {
  if (!c->prof) return;
  for (auto& p : c->prof->ev)
    for (auto& st : p)
      for (auto& e : st)
        if (e) cudaEventDestroy(e);
  delete c->prof;
  c->prof = nullptr;
}

extern "C" mt_status mt_comm_profile(mt_comm* c, int enable) {
  if (!c) return mt::fail(MT_ESHAPE, "comm is NULL");
  if (!enable) {
    prof_free(c);
    return MT_OK;
  }
  if (c->prof) return MT_OK;
  c->prof = new RingProfile();
  for (auto& p : c->prof->ev)
    for (auto& st : p)
      for (auto& e : st)
        if (cudaEventCreate(&e) != cudaSuccess) {
          prof_free(c);
          return mt::fail(MT_ECUDA, "cudaEventCreate(profile) failed");
        }
  return MT_OK;
}

extern "C" mt_status mt_comm_step_times(mt_comm* c, int backward, int max_steps, float* out,
                                        int* n_steps) {
  if (!c || !out || !n_steps || max_steps < 0) return mt::fail(MT_ESHAPE, "NULL argument");
  if (!c->prof) return mt::fail(MT_ECONFIG, "profiling not enabled (mt_comm_profile)");
  const int pass = backward ? 1 : 0;
  const int n = c->prof->steps[pass] < max_steps ? c->prof->steps[pass] : max_steps;
  for (int t = 0; t < n; ++t)
    for (int k = 0; k < 4; ++k) {
      const int b = 2 * k, e = 2 * k + 1;
      float ms = -1.f;
      if (c->prof->rec[pass][t][b] && c->prof->rec[pass][t][e]) {
        if (cudaEventSynchronize(c->prof->ev[pass][t][e]) != cudaSuccess ||
            cudaEventElapsedTime(&ms, c->prof->ev[pass][t][b], c->prof->ev[pass][t][e]) != cudaSuccess)
          return mt::fail(MT_ECUDA, "profile event query failed");
      }
      out[t * 4 + k] = ms;
    }
  for (auto& st : c->prof->rec[pass])
    for (auto& r : st) r = false;
  *n_steps = n;
  return MT_OK;
}

extern "C" mt_status mt_comm_check(mt_comm* c) {
  if (!c) return mt::fail(MT_ESHAPE, "comm is NULL");
#ifdef MT_HAVE_NCCL
  for (ncclComm_t nc : {c->nccl, c->nccl2, c->nccl3}) {
    if (!nc) continue;
    ncclResult_t ar = ncclSuccess;
    if (ncclCommGetAsyncError(nc, &ar) != ncclSuccess || ar != ncclSuccess)
      return mt::fail(MT_ENCCL, "NCCL asynchronous error: %s", ncclGetErrorString(ar));
  }
#endif
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return mt::fail(MT_ECUDA, "CUDA error: %s", cudaGetErrorString(e));
  return MT_OK;
}

extern "C" mt_status mt_comm_destroy(mt_comm* c) {
  if (!c) return MT_OK;
  prof_free(c);
#ifdef MT_HAVE_NCCL
  mt::ce_release(c);
  if (c->nccl3) ncclCommDestroy(c->nccl3);
  if (c->nccl2) ncclCommDestroy(c->nccl2);
  if (c->nccl) ncclCommDestroy(c->nccl);
#endif
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->comm_stream2) cudaStreamDestroy(c->comm_stream2);
  if (c->comm_stream3) cudaStreamDestroy(c->comm_stream3);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  delete c;
  return MT_OK;
}

mt_status mt_build_vs_index_dist(mt_comm* comm, const mt_shape* sh, const mt_vs_params* prm,
                                 const void* q, const void* k, mt_vs_index* out, void* ws,
                                 size_t ws_bytes, mt_stream_t st, const mt::RopeArgs* rope,
                                 void* q_out, void* k_out) {
#ifdef MT_HAVE_NCCL
  const int W = comm->world;
  MT_TRY(check_shape(sh, W));
  if (!prm) return fail(MT_ESHAPE, "params is NULL");
  if (!(prm->p_v > 0.f && prm->p_v <= 1.f) || !(prm->p_s > 0.f && prm->p_s <= 1.f))
    return fail(MT_ECONFIG, "p_v, p_s must lie in (0, 1] (got %g, %g)", prm->p_v, prm->p_s);
  if (sh->seq_len > (1LL << 22)) return fail(MT_ESHAPE, "seq_len must be <= 2^22 for the index");
  if (!q || !k || !out || !out->v_cnt || !out->v_idx || !out->s_cnt || !out->s_off)
    return fail(MT_ESHAPE, "NULL argument");
  if (out->v_stride < sh->seq_len || out->s_stride < sh->seq_len / 64)
    return fail(MT_ECAPACITY, "index capacity too small");
  const size_t need = vsidx_workspace_bytes(sh->seq_len, sh->n_q_heads, W);
  if (!ws || ws_bytes < need) return fail(MT_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  NcclCollectives coll(comm);
  return vsidx_build(&coll, sh->seq_len, sh->n_q_heads, sh->n_kv_heads, W, comm->rank, sh->layout,
                     prm->p_v,
                     prm->p_s, q, k, out->v_cnt, out->v_idx, out->v_stride, out->s_cnt,
                     out->s_off, out->s_stride, nullptr, nullptr, ws, st, rope, q_out, k_out);
#else
  (void)comm; (void)sh; (void)prm; (void)q; (void)k; (void)out; (void)ws; (void)ws_bytes; (void)st;
  (void)rope; (void)q_out; (void)k_out;
  return fail(MT_EUNSUPPORTED, "built without NCCL");
#endif
}

// ------------------------------------------------------------------ copy-engine ring
#ifdef MT_HAVE_NCCL
#include <cudaTypedefs.h>

namespace mt {
namespace {
struct CeHandle {
  cudaIpcMemHandle_t h;
  uint64_t off;    // workspace offset inside its allocation
  uint64_t bytes;  // registered workspace bytes
  int32_t dev;
  int32_t pad;
};

PFN_cuMemGetAddressRange_v3020 get_range() {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &p, 3020, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  });
  return fn;
}

}  // namespace

void ce_release(mt_comm* c) {
  if (c->ce_next_map) cudaIpcCloseMemHandle(c->ce_next_map);
  if (c->ce_prev_map && c->ce_prev_map != c->ce_next_map) cudaIpcCloseMemHandle(c->ce_prev_map);
  c->ce_next_map = c->ce_prev_map = nullptr;
  c->ce_next_ws = c->ce_prev_ws = nullptr;
  c->ce_ws = nullptr;
  c->ce_ok = false;
}

CeStreamValueFn ce_wait_fn() {
  static CeStreamValueFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<CeStreamValueFn>(p);
  });
  return fn;
}

CeStreamValueFn ce_write_fn() {
  static CeStreamValueFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<CeStreamValueFn>(p);
  });
  return fn;
}
}  // namespace mt
#endif

extern "C" size_t mt_ring_flags_bytes(void) { return 256; }

extern "C" mt_status mt_comm_register_workspace(mt_comm* c, void* ws, size_t ws_bytes,
                                                mt_stream_t stream) {
#ifdef MT_HAVE_NCCL
  if (!c || !ws) return fail(MT_ESHAPE, "NULL argument");
  if (ws_bytes < 4096) return fail(MT_EWORKSPACE, "workspace too small to register");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  mt::ce_release(c);
  const int W = c->world, r = c->rank;
  if (W < 2) return MT_OK;
  // my handle, gathered from every rank over NCCL (the exchange uses the first W * 96
  // bytes of the workspace as scratch; the flag words at its end are zeroed first)
  CeHandle mine{};
  bool ok = true;
  CUdeviceptr base = 0;
  size_t size = 0;
  auto range = mt::get_range();
  if (!range || range(&base, &size, reinterpret_cast<CUdeviceptr>(ws)) != CUDA_SUCCESS ||
      cudaIpcGetMemHandle(&mine.h, reinterpret_cast<void*>(base)) != cudaSuccess)
    ok = false;
  cudaGetLastError();
  mine.off = ok ? (uint64_t)(reinterpret_cast<uintptr_t>(ws) - (uintptr_t)base) : 0;
  mine.bytes = ok ? ws_bytes : 0;  // 0: this rank cannot share (everyone falls back)
  cudaGetDevice(&mine.dev);
  uint8_t* scratch = static_cast<uint8_t*>(ws);
  const size_t hb = sizeof(CeHandle);
  if (cudaMemsetAsync(static_cast<uint8_t*>(ws) + ws_bytes - 256, 0, 256, st) != cudaSuccess ||
      cudaMemcpyAsync(scratch + (size_t)W * hb, &mine, hb, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return fail(MT_ECUDA, "register: staging failed");
  MT_TRY(nccl_check(ncclAllGather(scratch + (size_t)W * hb, scratch, hb, ncclUint8, c->nccl, st),
                    "register all-gather"));
  std::vector<CeHandle> all(W);
  if (cudaMemcpyAsync(all.data(), scratch, (size_t)W * hb, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return fail(MT_ECUDA, "register: handle copy failed");
  for (int i = 0; i < W; ++i) ok = ok && all[i].bytes > 0;
  const int nx = (r + 1) % W, pv = (r - 1 + W) % W;
  if (ok) {
    int can = 0;
    cudaDeviceCanAccessPeer(&can, mine.dev, all[nx].dev);
    ok = can != 0;
    cudaDeviceCanAccessPeer(&can, mine.dev, all[pv].dev);
    ok = ok && can != 0;
  }
  if (ok) {
    if (cudaIpcOpenMemHandle(&c->ce_next_map, all[nx].h, cudaIpcMemLazyEnablePeerAccess) !=
        cudaSuccess) {
      c->ce_next_map = nullptr;
      ok = false;
    }
  }
  if (ok) {
    if (pv == nx) {
      c->ce_prev_map = c->ce_next_map;
    } else if (cudaIpcOpenMemHandle(&c->ce_prev_map, all[pv].h, cudaIpcMemLazyEnablePeerAccess) !=
               cudaSuccess) {
      c->ce_prev_map = nullptr;
      ok = false;
    }
  }
  cudaGetLastError();
  // every rank must agree: an all-reduce(min) of the local verdicts; it also orders every
  // rank's flag zeroing before any rank's first remote flag write
  int32_t* flag = reinterpret_cast<int32_t*>(scratch);
  const int32_t okv = ok ? 1 : 0;
  if (cudaMemcpyAsync(flag, &okv, 4, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return fail(MT_ECUDA, "register: verdict copy failed");
  MT_TRY(nccl_check(ncclAllReduce(flag, flag, 1, ncclInt32, ncclMin, c->nccl, st), "register verdict"));
  int32_t all_ok = 0;
  if (cudaMemcpyAsync(&all_ok, flag, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return fail(MT_ECUDA, "register: verdict readback failed");
  if (!all_ok) {
    mt::ce_release(c);
    return MT_OK;  // the ring keeps its NCCL transport
  }
  c->ce_ws = ws;
  c->ce_bytes = ws_bytes;
  c->ce_next_ws = static_cast<uint8_t*>(c->ce_next_map) + all[nx].off;
  c->ce_next_bytes = all[nx].bytes;
  c->ce_prev_ws = static_cast<uint8_t*>(c->ce_prev_map) + all[pv].off;
  c->ce_prev_bytes = all[pv].bytes;
  c->ce_calls = 0;
  c->ce_ok = true;
  return MT_OK;
#else
  (void)c; (void)ws; (void)ws_bytes; (void)stream;
  return fail(MT_EUNSUPPORTED, "built without NCCL");
#endif
}

extern "C" int mt_comm_copy_engine(mt_comm* c) { return (c && c->ce_ok) ? 1 : 0; }
