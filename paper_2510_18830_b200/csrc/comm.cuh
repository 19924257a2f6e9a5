// comm.cuh — the mt_comm object: one NCCL communicator over a context-parallel
// group plus the streams/events the ring uses to overlap P2P with compute.
#pragma once
#include "common.cuh"

#ifdef MT_HAVE_NCCL
#include <nccl.h>
#endif

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
};

namespace mt {
#ifdef MT_HAVE_NCCL
inline mt_status nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) return fail(MT_ENCCL, "%s: %s", what, ncclGetErrorString(r));
  return MT_OK;
}
#endif
}  // namespace mt
