// comm.cuh — the mt_comm object: one NCCL communicator over a context-parallel
// group plus the streams/events the ring uses to overlap P2P with compute.
#pragma once
#include "common.cuh"

#ifdef MT_HAVE_NCCL
#include <nccl.h>
#endif

// Optional per-step timeline of the ring calls (mt_comm_profile): CUDA events on
// the compute stream around each step's kernels and on the comm streams around
// each transfer.  [pass 0 fwd / 1 bwd][step][event]
struct RingProfile {
  static constexpr int kMaxSteps = 64, kEv = 8;
  enum { kCompB, kCompE, kInnerB, kInnerE, kOuterB, kOuterE, kDkvB, kDkvE };
  cudaEvent_t ev[2][kMaxSteps][kEv] = {};
  bool rec[2][kMaxSteps][kEv] = {};
  int steps[2] = {0, 0};
};

struct mt_comm {
#ifdef MT_HAVE_NCCL
  ncclComm_t nccl = nullptr;   // inner (node) ring KV exchange, index collectives
  ncclComm_t nccl2 = nullptr;  // outer ring KV exchange (hierarchical)
  ncclComm_t nccl3 = nullptr;  // backward dK/dV partials to their owners
#endif
  int world = 1, rank = 0, inner = 1;
  cudaStream_t comm_stream = nullptr;   // inner ring P2P
  cudaStream_t comm_stream2 = nullptr;  // outer ring P2P
  cudaStream_t comm_stream3 = nullptr;  // dK/dV partial P2P
  cudaEvent_t ev_ready = nullptr;      // compute -> comm ordering
  cudaEvent_t ev_done = nullptr;       // comm -> compute ordering
  RingProfile* prof = nullptr;         // non-null while profiling is enabled
  // Slow inter-node link emulation (env MT_EMU_INTER_GBPS, MT_EMU_NODE):
  // ring receives from a rank of another emulated node are held back by
  // bytes / emu_gbps on their comm stream (a host function: no SM is taken).
  double emu_gbps = 0.0;  // 0 = off
  int emu_node = 0;       // ranks per emulated node
  // SMs left free by the ring's forward / backward attention launches so the NCCL
  // kernels (capped at max(reserve_sms, reserve_sms_bwd) CTAs when either is set)
  // find an SM: the persistent attention kernels hold one CTA per SM for a whole
  // step, and a transfer that cannot start until the step ends delays the next
  // step (env MT_RING_RESERVE_SMS / MT_RING_RESERVE_SMS_BWD; 0 = off).
  int reserve_sms = 0;
  int reserve_sms_bwd = 0;
  // Copy-engine KV ring (flat forward; mt_comm_register_workspace).  The ring neighbours'
  // registered workspaces are mapped through CUDA IPC; a step's KV chunk is written into
  // the next rank's receive slot by cudaMemcpyAsync on comm_stream (copy engines over
  // NVLink: no SM, so the transfer overlaps the persistent attention kernel), ordered by
  // stream memory operations on monotone 32-bit counters in the workspaces' flag words.
  void* ce_ws = nullptr;          // my registered workspace
  size_t ce_bytes = 0;
  void* ce_next_map = nullptr;    // IPC mapping of rank r+1's allocation (base)
  uint8_t* ce_next_ws = nullptr;  // rank r+1's registered workspace, in this address space
  size_t ce_next_bytes = 0;
  void* ce_prev_map = nullptr;    // same for rank r-1
  uint8_t* ce_prev_ws = nullptr;
  size_t ce_prev_bytes = 0;
  uint32_t ce_calls = 0;          // forward ring calls since registration (identical on all ranks)
  bool ce_ok = false;
};

#include <cuda.h>
namespace mt {
// cuStreamWaitValue32 / cuStreamWriteValue32 (driver API, fetched by entry point)
typedef CUresult (*CeStreamValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
// Release the copy-engine ring's IPC mappings (mt_comm_register_workspace).
void ce_release(mt_comm* c);
// Emulated wire time of `bytes` arriving at rank c->rank from rank `from` (no-op
// unless emulation is on and the two ranks sit on different emulated nodes).
void emu_inbound(mt_comm* c, int from, size_t bytes, cudaStream_t st);
// Record profiling event e of (pass, step) on stream st (no-op when not profiling).
inline void prof_mark(mt_comm* c, int pass, int step, int e, cudaStream_t st) {
  if (!c || !c->prof || step >= RingProfile::kMaxSteps) return;
  cudaEventRecord(c->prof->ev[pass][step][e], st);
  c->prof->rec[pass][step][e] = true;
  if (step + 1 > c->prof->steps[pass]) c->prof->steps[pass] = step + 1;
}
}  // namespace mt

namespace mt {
#ifdef MT_HAVE_NCCL
inline mt_status nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) return fail(MT_ENCCL, "%s: %s", what, ncclGetErrorString(r));
  return MT_OK;
}
#endif
}  // namespace mt
