// vsidx.cuh — internal interface of the index builder (vs_index.cu) shared with
// the distributed driver (comm.cu).
#pragma once
#include <cuda_bf16.h>
#include "common.cuh"
#include "rope.cuh"

namespace mt {

// Collectives that complete the order-free reductions of VS-IDX v1 across the
// ranks of a layout (NULL = single GPU).
struct VSCollectives {
  virtual mt_status bcast_window(__nv_bfloat16* qwin, size_t n, int root, cudaStream_t st) = 0;
  virtual mt_status allreduce_max(float* M, size_t n, cudaStream_t st) = 0;
  virtual mt_status allreduce_sum_u64(unsigned long long* E, size_t n, cudaStream_t st) = 0;
  virtual mt_status allgather_keys(const uint64_t* loc, uint64_t* glob, int Hq, int64_t n_loc,
                                   cudaStream_t st) = 0;
  virtual ~VSCollectives() = default;
};

// rope != NULL (f3 fusion): q_loc / k_loc are pre-RoPE, q_out / k_out receive the rotated
// tensors (k_out must not alias k_loc; q_out may alias q_loc)
mt_status vsidx_build(VSCollectives* coll, int64_t S, int Hq, int Hkv, int W, int r, int layout,
                      float p_v, float p_s, const void* q_loc, const void* k_loc, int32_t* v_cnt,
                      int32_t* v_idx, int64_t v_stride, int32_t* s_cnt, int32_t* s_off,
                      int64_t s_stride, uint64_t* dbg_colV, uint64_t* dbg_blkP, void* ws,
                      cudaStream_t st, const RopeArgs* rope = nullptr, void* q_out = nullptr,
                      void* k_out = nullptr);
mt_status rope_launch(const RopeArgs& ra, int inverse, int64_t seq_len, int world, int rank,
                      int layout, int n_heads, const void* x_in, void* x_out, cudaStream_t st);
size_t vsidx_workspace_bytes(int64_t S, int Hq, int W);
mt_status check_shape(const mt_shape* sh, int W);
mt_status check_device();

}  // namespace mt
