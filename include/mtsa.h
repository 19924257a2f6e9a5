/* mtsa.h — C ABI of the B200-native MTraining hot path (arXiv 2510.18830).
 *
 * What this library computes (citations are PAPER.md lines, "P:n", of
 * /root/reference/PAPER.md at the time of writing):
 *   - the vertical-slash (VS) sparse index of Alg. 1: window
 *     attention of the last 64 queries, online top-p budgets for
 *     vertical columns and 64x64-pooled slash offsets (P:228-229,
 *     P:249), sparseformat;
 *   - block-sparse attention forward/backward over that index (Eq. 1
 *     P:111, Eq. 12), with the merge of partial (O, LSE) across ring
 *     steps (merge_out_and_lse);
 *   - the balanced (64-token block-striped) sparse ring, flat and
 *     hierarchical (Alg. 2), over NCCL send/recv.
 *
 * Conventions shared by every entry point:
 *   - All tensor pointers are CUDA DEVICE pointers owned by the caller, unless a
 *     parameter says "host".  The library never allocates device memory: calls
 *     that need scratch take a caller workspace sized by the matching
 *     *_workspace_bytes() function.
 *   - All compute calls are asynchronous on the caller's stream.  Argument
 *     validation happens synchronously before any launch; a validation failure
 *     launches nothing.  Asynchronous CUDA failures surface as MT_ECUDA on the
 *     next call that checks (or via cudaStreamSynchronize by the caller).
 *   - Layouts (token-major, bf16 = IEEE bfloat16):
 *       Q, O, dO, dQ : [S_loc][Hq][d]      K, V, dK, dV : [S_loc][Hkv][d]
 *       LSE          : float32 [Hq][S_loc], natural log.
 *     S_loc = S / W is the rank-local (block-striped) length; W = 1 on one GPU.
 *   - Supported: d = 128, block = last_q = 64, Hq % Hkv == 0, S % (64 W) == 0.
 *   - No exceptions, abort() or exit() cross this boundary; functions return
 *     mt_status, and mt_last_error() gives a thread-local message.
 */
#ifndef MTSA_H_
#define MTSA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* mt_stream_t; /* == cudaStream_t */

typedef enum {
  MT_OK = 0,
  MT_ESHAPE = 1,       /* null pointer / bad dimension */
  MT_EWINDOW = 2,      /* S < 64 or S % 64 != 0 (window = last 64 queries) */
  MT_ECONFIG = 3,      /* p_v or p_s outside (0, 1] */
  MT_ELAYOUT = 4,      /* S not divisible for the layout (64 W striped, 128 W zigzag) */
  MT_ECAPACITY = 5,    /* an output buffer is too small */
  MT_EWORKSPACE = 6,   /* workspace too small */
  MT_EUNSUPPORTED = 7, /* d != 128, block != 64, non-sm_100 device */
  MT_ECUDA = 8,        /* CUDA runtime / launch error */
  MT_ENCCL = 9         /* NCCL error */
} mt_status;

/* Thread-local description of the last non-MT_OK status returned on this thread. */
const char* mt_last_error(void);

/* Process-wide counters (for benchmarks; thread-safe, monotone):
 *   mt_launch_count       kernels this library has enqueued (its own sm_100a kernels);
 *   mt_library_call_count CUB radix-sort calls it has enqueued (each launches several
 *                         CUB kernels compiled into this library).                   */
unsigned long long mt_launch_count(void);
unsigned long long mt_library_call_count(void);

/* Sequence-to-rank layouts of the ring (Fig. 1), at 64-token
 * block granularity; a rank's local blocks are always in ascending global order.
 *   MT_LAYOUT_STRIPED  the method: global block b -> rank b mod W, local
 *                      block b / W.  Needs S % (64 W) == 0.
 *   MT_LAYOUT_ZIGZAG   the "Ours w/ ZigZag" ablation: the sequence
 *                      is cut into 2W equal chunks, rank r holds chunk r then chunk
 *                      2W-1-r.  Needs S % (128 W) == 0.
 * With world == 1 both are the identity. */
enum { MT_LAYOUT_STRIPED = 0, MT_LAYOUT_ZIGZAG = 1 };

/* Problem shape.  seq_len is the GLOBAL sequence length S.  A zero-initialised
 * `layout` is the block-striped layout. */
typedef struct {
  int64_t seq_len;
  int32_t n_q_heads;  /* Hq */
  int32_t n_kv_heads; /* Hkv; q head h uses kv head h / (Hq / Hkv) */
  int32_t head_dim;   /* d, must be 128 */
  int32_t block;      /* B = stripe = slash block, must be 64 */
  int32_t last_q;     /* window rows of Alg. 1 (`last_q`, never given: reading R2), must be
                         64 = one block; 0 means 64 */
  int32_t layout;     /* MT_LAYOUT_STRIPED or MT_LAYOUT_ZIGZAG (multi-rank calls) */
} mt_shape;

/* Online top-p targets of Alg. 1 ("p_v, p_s", read as reals in (0, 1]). */
typedef struct {
  float p_v;
  float p_s;
} mt_vs_params;

/* Vertical-slash index (Alg. 1 output, P:225 i_v and P:229 i_s), caller-owned
 * DEVICE arrays.  For q head h:
 *   v_idx[h * v_stride + 0 .. v_cnt[h])  vertical token columns, ascending,
 *                                        global positions in [0, S)
 *   s_off[h * s_stride + 0 .. s_cnt[h])  slash offsets in 64-token block units
 *                                        (offset o: key block = query block - o,
 *                                        P:249), ascending, in [0, S/64)
 * Offset 0 (the diagonal) must be present for every head: it guarantees every
 * query attends at least itself (reading R7).  mt_build_vs_index
 * produces it; callers may also supply their own lists (v_stride >= S,
 * s_stride >= S/64 when written by mt_build_vs_index). */
typedef struct {
  int32_t* v_cnt; /* [Hq] */
  int32_t* v_idx; /* [Hq][v_stride] */
  int64_t v_stride;
  int32_t* s_cnt; /* [Hq] */
  int32_t* s_off; /* [Hq][s_stride] */
  int64_t s_stride;
} mt_vs_index;

/* Opaque NCCL communicator over the ranks of one context-parallel group
 * (see the ring section below).  NULL means "single GPU". */
typedef struct mt_comm mt_comm;

/* Communicator lifecycle (one process per GPU, P:64 context parallelism).
 * mt_comm_unique_id: rank 0 creates a 128-byte NCCL unique id (host buffer);
 *   the caller distributes it to every rank (e.g. torch.distributed).
 * mt_comm_create: collective over `world` ranks; `inner` = ranks per node of the
 *   hierarchical ring (Alg. 2 w_inner); inner = world (or <= 0) is the
 *   flat ring.  The current CUDA device is used.  Errors: MT_ESHAPE (bad
 *   rank/world, inner not dividing world), MT_ENCCL, MT_EUNSUPPORTED.
 * mt_comm_destroy: releases NCCL resources and the comm stream/events. */
mt_status mt_comm_unique_id(uint8_t id[128]);
mt_status mt_comm_create(const uint8_t id[128], int world, int rank, int inner, mt_comm** out);
mt_status mt_comm_destroy(mt_comm* comm);
/* Surface asynchronous failures: MT_ENCCL if any of the
 * communicator's NCCL comms reports an async error, MT_ECUDA for a sticky or
 * pending CUDA error, else MT_OK.  Non-blocking. */
mt_status mt_comm_check(mt_comm* comm);

/* Ring step profiling (per-step compute vs communication, ring
 * GB/s).  mt_comm_profile(comm, 1) makes later ring calls on `comm` record CUDA
 * events around each step's kernels (compute stream) and each transfer (comm
 * streams); 0 disables and frees them.  Recording adds a few microseconds per
 * step: keep it out of timed regions.
 * mt_comm_step_times: after a profiled mt_ring_attn_fwd (backward = 0) or _bwd
 * (1), waits for its events and writes out[t * 4 + {0,1,2,3}] = milliseconds
 * of step t's {compute, inner-ring KV transfer, outer-ring KV transfer, dK/dV
 * partial transfer} (-1 where the step had none); *n_steps = steps written
 * (<= max_steps).  Errors: MT_ESHAPE, MT_ECONFIG (not profiling), MT_ECUDA. */
mt_status mt_comm_profile(mt_comm* comm, int enable);
mt_status mt_comm_step_times(mt_comm* comm, int backward, int max_steps, float* out,
                             int* n_steps);

/* ------------------------------------------------------------- VS index */
/* Workspace (bytes) for mt_build_vs_index on a `world`-rank layout. */
size_t mt_build_vs_index_workspace_bytes(const mt_shape* shape, int world);

/* Alg. 1 vertical-slash index of every q head, in the VS-IDX v1
 * arithmetic: fp32 window scores of the last 64 queries
 * against all causal keys, softmax in specified fixed point, column
 * sums (token level) and 64x64-pooled block-diagonal sums, exact
 * integer top-p budgets, argtopk with ties to the smaller index,
 * forced column 0 and offset 0.  The window scores are a fold of fused
 * multiply-adds (the bf16 x bf16 product is not rounded on its own, reading R11),
 * so the result is bit-identical to the CPU oracle for EVERY bf16 input
 * (subnormals, products below 2^-149 and huge values included; NaN/Inf inputs
 * give unspecified lists) and independent of `world`.
 *   comm == NULL : single GPU; q [S][Hq][128], k [S][Hkv][128].
 *   comm != NULL : q/k are this rank's block-striped local slices
 *                  [S/W][.][128]; every rank receives the same global lists.
 * out: caller-allocated, v_stride >= S, s_stride >= S/64 (MT_ECAPACITY).
 * Caller-supplied indices (any call taking an mt_vs_index) must hold lists like
 * this function's: strictly ascending, columns in [0, S), offsets in [0, S/64),
 * offset 0 present; strides below (S, S/64) are MT_ESHAPE.  Out-of-range entries
 * are dropped by the plan builder (no out-of-bounds writes), other violations
 * give unspecified attention results.
 * Errors: MT_ESHAPE, MT_EWINDOW (S < 64 or S % 64), MT_ECONFIG (p outside
 * (0, 1]), MT_ELAYOUT, MT_EWORKSPACE, MT_EUNSUPPORTED, MT_ECUDA, MT_ENCCL. */
mt_status mt_build_vs_index(mt_comm* comm, const mt_shape* shape, const mt_vs_params* params,
                            const void* q, const void* k, mt_vs_index* out, void* ws,
                            size_t ws_bytes, mt_stream_t stream);

/* f3 upstream fusion (P:339 RoPE/YaRN, Appendix A): the index of
 * the ROTATED q / k built from PRE-RoPE inputs, with the RoPE pass folded into it.  q, k
 * are pre-RoPE (layout, world and shapes as mt_build_vs_index); on return q_out / k_out
 * hold RoPE(q) / RoPE(k) at the tokens' global positions (theta[64] and mscale as
 * mt_rope_inv_freq; the same bf16 bits as mt_rope) and `out` holds exactly the lists
 * mt_build_vs_index gives for (q_out, k_out).  The window queries are rotated while
 * staged, k is rotated in registers by the index's first stage (each key row read once
 * for both), q by one extra pass.  q_out may alias q; k_out must not alias k (MT_ESHAPE).
 * Same workspace as mt_build_vs_index.  Errors: as mt_build_vs_index. */
mt_status mt_rope_vs_index(mt_comm* comm, const mt_shape* shape, const mt_vs_params* params,
                           const double* theta, float mscale, const void* q, const void* k,
                           void* q_out, void* k_out, mt_vs_index* out, void* ws,
                           size_t ws_bytes, mt_stream_t stream);

/* Test hook (single GPU): the exact intermediate scores of Alg. 1 —
 * col_scores [Hq][S] = sum_v(A_hat) per token column (uint64 fixed point,
 * 2^32 = probability 1) and slash_scores [Hq][S/64] = the 64x64-pooled
 * diagonal score of each block offset.  Same workspace as mt_build_vs_index. */
mt_status mt_vs_column_scores(const mt_shape* shape, const void* q, const void* k,
                              uint64_t* col_scores, uint64_t* slash_scores, void* ws,
                              size_t ws_bytes, mt_stream_t stream);

/* ------------------------------------------------------- sparse attention */
/* Workspace (bytes) needed by mt_sparse_attn_fwd / mt_attn_fwd_step for a
 * layout of `world` ranks (world = 1 on one GPU). */
size_t mt_sparse_attn_fwd_workspace_bytes(const mt_shape* shape, int world);

/* Single-GPU sparse attention forward, Alg. 1 line "y <- sparse(softmax(QK^T /
 * sqrt(d)) V, i_vs)" over the key set of each query n in block g:
 *   K_n = { m : floor(m/64) = g - o for some o in i_s, m <= n }
 *         U { m in i_v : floor(m/64) < g }      (I9)
 * q [S][Hq][128], k/v [S][Hkv][128] bf16 in; o [S][Hq][128] bf16 and
 * lse [Hq][S] float32 (natural log) out.  Errors: MT_ESHAPE, MT_EWINDOW,
 * MT_EUNSUPPORTED, MT_EWORKSPACE, MT_ECUDA. */
mt_status mt_sparse_attn_fwd(const mt_shape* shape, const void* q, const void* k, const void* v,
                             const mt_vs_index* idx, void* o, float* lse, void* ws,
                             size_t ws_bytes, mt_stream_t stream);

/* One ring step of the forward (Alg. 2) for rank `rank` of a
 * `world`-rank block-striped layout, holding the KV chunk of origin `origin`:
 * computes the partial attention of the rank's local queries q_loc over the
 * chunk's keys and merges it into (o_acc, lse) (merge_out_and_lse).
 *   first != 0 : (o_acc, lse) are initialised instead of read;
 *   last  != 0 : the merged result is written as bf16 to o (o_acc not written).
 * q_loc [S/W][Hq][128], k_chunk/v_chunk [S/W][Hkv][128] bf16; o_acc
 * [S/W][Hq][128] float32; lse [Hq][S/W] float32.  `shape->seq_len` is the
 * GLOBAL S.  The ring entry points call this; it is exported so a single GPU
 * can emulate every (rank, step) of a ring (tests). */
mt_status mt_attn_fwd_step(const mt_shape* shape, int world, int rank, int origin, int first,
                           int last, const void* q_loc, const void* k_chunk,
                           const void* v_chunk, const mt_vs_index* idx, void* o, float* o_acc,
                           float* lse, void* ws, size_t ws_bytes, mt_stream_t stream);

/* Workspace (bytes) of mt_sparse_attn_bwd (single GPU). */
size_t mt_sparse_attn_bwd_workspace_bytes(const mt_shape* shape);

/* Single-GPU sparse attention backward with the forward's index held fixed
 * ("superposition of the forward-phase sparsity"): Eq. 1 and
 * Eq. 12 restricted to each query's key set K_n:
 *   P = exp(q k^T / sqrt(d) - LSE), D = rowsum(dO o O), dS = P o (dO v^T - D),
 *   dV = P^T dO, dK = dS^T Q / sqrt(d), dQ = dS K / sqrt(d)
 * (GQA: dK/dV of a kv head sum over its q heads).  o/lse are the forward's
 * outputs; dq [S][Hq][128], dk/dv [S][Hkv][128] bf16 out (fp32 accumulation
 * inside the workspace).  Errors as mt_sparse_attn_fwd. */
mt_status mt_sparse_attn_bwd(const mt_shape* shape, const void* q, const void* k, const void* v,
                             const void* o, const float* lse, const void* dO,
                             const mt_vs_index* idx, void* dq, void* dk, void* dv, void* ws,
                             size_t ws_bytes, mt_stream_t stream);

/* Workspace (bytes) of mt_attn_fwd_step / mt_attn_bwd_step for `world` ranks. */
size_t mt_attn_step_workspace_bytes(const mt_shape* shape, int world);

/* Backward preprocessing for one rank: D_loc[h][n] = dO_n . O_n (float32
 * [Hq][S/W]) — the sum_j dL/dA_ij A_ij term of Eq. 1. */
mt_status mt_attn_bwd_preprocess(const mt_shape* shape, int world, const void* o_loc,
                                 const void* dO_loc, float* D_loc, mt_stream_t stream);

/* One ring step of the backward (Table 4 "attention computation for a chunk"
 * plus "backward for vertical lines") for rank `rank` holding the
 * KV chunk of origin `origin`: reduce-adds the contributions of the rank's
 * local queries into dq_acc [S/W][Hq][128] (float32, local queries) and into
 * dk_acc/dv_acc [S/W][Hkv][128] (float32, the chunk's keys).  Accumulators are
 * caller-initialised.  Exported so one GPU can emulate every (rank, step). */
mt_status mt_attn_bwd_step(const mt_shape* shape, int world, int rank, int origin,
                           const void* q_loc, const void* k_chunk, const void* v_chunk,
                           const void* dO_loc, const float* lse_loc, const float* D_loc,
                           const mt_vs_index* idx, float* dq_acc, float* dk_acc, float* dv_acc,
                           void* ws, size_t ws_bytes, mt_stream_t stream);

/* ------------------------------------------------------------- sparse ring */
/* Workspace (bytes) of mt_ring_attn_fwd (backward = 0) / mt_ring_attn_bwd
 * (backward = 1) on `world` ranks. */
size_t mt_ring_attn_workspace_bytes(const mt_shape* shape, int world, int backward);

/* Balanced sparse ring attention forward (Alg. 2)
 * on the communicator's ranks: rank r holds the block-striped slices
 * q_loc [S/W][Hq][128], k_loc/v_loc [S/W][Hkv][128] (global 64-token block b
 * on rank b mod W at local block b / W).  KV chunks circulate over NCCL
 * send/recv — flat ring (comm inner == world) or hierarchical inner/outer ring —
 * overlapped with the per-step sparse forward; o_loc [S/W][Hq][128] bf16 and
 * lse_loc [Hq][S/W] float32 out.  idx is the GLOBAL index (identical on every
 * rank, e.g. from mt_build_vs_index with the same comm).  Collective: every
 * rank must call it.  Errors: as mt_sparse_attn_fwd, MT_ELAYOUT, MT_ENCCL. */
mt_status mt_ring_attn_fwd(mt_comm* comm, const mt_shape* shape, const void* q_loc,
                           const void* k_loc, const void* v_loc, const mt_vs_index* idx,
                           void* o_loc, float* lse_loc, void* ws, size_t ws_bytes,
                           mt_stream_t stream);

/* Balanced sparse ring attention backward (Table 4): KV circulates as
 * in the forward; at every step the dK/dV partial of the held chunk is sent to
 * the chunk's owner over NCCL (reading R17) while the next step computes; dQ
 * stays local.  Outputs dq_loc [S/W][Hq][128], dk_loc/dv_loc [S/W][Hkv][128]
 * bf16 for the rank's own striped rows.  Collective. */
mt_status mt_ring_attn_bwd(mt_comm* comm, const mt_shape* shape, const void* q_loc,
                           const void* k_loc, const void* v_loc, const void* o_loc,
                           const float* lse_loc, const void* dO_loc, const mt_vs_index* idx,
                           void* dq_loc, void* dk_loc, void* dv_loc, void* ws, size_t ws_bytes,
                           mt_stream_t stream);

/* Copy-engine transport for the flat forward ring.  Collective: every
 * rank of `comm` calls it with the workspace it will pass to mt_ring_attn_fwd / _bwd
 * (ws_bytes >= the ring workspace + mt_ring_flags_bytes(); the last 256 bytes are reserved
 * flag words and must not be touched between ring calls).  The ring neighbours'
 * workspaces are then mapped through CUDA IPC, and the forward ring moves each step's KV
 * chunk with cudaMemcpyAsync into the next rank's receive slot (copy engines over NVLink:
 * no SM, so the transfer overlaps the persistent attention kernel), ordered by stream
 * memory operations (cuStreamWaitValue32 / WriteValue32) on monotone step counters.  Where
 * IPC or peer access is unavailable on any rank, the call succeeds and the ring keeps NCCL
 * send/recv (mt_comm_copy_engine reports which).  Registering again (e.g. after the
 * workspace moved) replaces the mappings; ring calls with another workspace use NCCL.
 * Synchronizes `stream`.  Errors: MT_ESHAPE, MT_EWORKSPACE, MT_ECUDA, MT_ENCCL. */
size_t mt_ring_flags_bytes(void);
mt_status mt_comm_register_workspace(mt_comm* comm, void* ws, size_t ws_bytes, mt_stream_t stream);
int mt_comm_copy_engine(mt_comm* comm);

/* Host-only: the ring schedule — out[t * world + x] = origin of the KV chunk
 * rank x holds at step t, for a ring of `world` ranks with `inner` ranks per
 * node (inner == world: flat).  out must hold world * world ints. */
mt_status mt_ring_schedule(int world, int inner, int32_t* out);

/* ------------------------------------------------------------------ format */
/* The per-query-block key lists of an index — the sparseformat step (PAPER.md
 * P:231-232, reading I9), global layout (world 1).  For q head h and query block g:
 *   B_g = blk_idx[blk_ptr[h*(nb+1)+g] .. blk_ptr[h*(nb+1)+g+1])  key blocks g - o, o in
 *         i_s[h], o <= g, ascending;
 *   C_g = col_idx[col_ptr[...] .. col_ptr[...+1])  columns m in i_v[h] with m/64 < g and
 *         (g - m/64) not in i_s[h] (covered verticals dropped), ascending.
 * blk_ptr / col_ptr: device int64 [Hq][nb + 1], global offsets (head h's rows follow
 * head h-1's).  Two passes: mt_vs_format_count fills the pointers and returns the
 * totals n_blk / n_col to the host (it synchronizes the stream); mt_vs_format_fill
 * writes the lists (blk_idx, col_idx: device int32, capacities >= the totals, else
 * MT_ECAPACITY).  The attention kernels do not need this format (they derive the
 * lists on the fly); it exists for verification and for callers that want CSR.
 * Errors: MT_ESHAPE, MT_EWINDOW, MT_EUNSUPPORTED, MT_EWORKSPACE, MT_ECAPACITY,
 * MT_ECUDA. */
size_t mt_vs_format_workspace_bytes(const mt_shape* shape);
mt_status mt_vs_format_count(const mt_shape* shape, const mt_vs_index* index, int64_t* blk_ptr,
                             int64_t* col_ptr, int64_t* n_blk, int64_t* n_col, void* workspace,
                             size_t ws_bytes, mt_stream_t stream);
mt_status mt_vs_format_fill(const mt_shape* shape, const mt_vs_index* index,
                            const int64_t* blk_ptr, const int64_t* col_ptr, int32_t* blk_idx,
                            int64_t blk_cap, int32_t* col_idx, int64_t col_cap, int64_t n_blk,
                            int64_t n_col, void* workspace, size_t ws_bytes, mt_stream_t stream);

/* ---------------------------------------------------- block-sparse index */
/* Sparse attention over an explicit block index: the paper's kernel interface
 * block_bar_sparse_attention_forward(Q, K, V, I_block, I_bar) with I_bar
 * empty, the form an XAttention block index takes ("w/ XAttn Idx.", P:347, P:826;
 * SURVEY §8(f) f2).  Single GPU (world 1), same shapes and layouts as
 * mt_sparse_attn_fwd/bwd.  The index is the CSR of mt_vs_format: for q head h and
 * query block g the key blocks blk_idx[blk_ptr[h*(nb+1)+g] .. blk_ptr[h*(nb+1)+g+1]),
 * device int64 pointers with global offsets, device int32 entries, n_blk entries
 * in total.  Each row must be strictly ascending with entries <= g (causal); the
 * block g itself is masked causally.  These properties are NOT checked on the
 * device (a violation is undefined behaviour; mt_xattn_index and mt_vs_format
 * produce valid rows).  Query rows with no key block get O = 0, LSE = -inf.
 * The backward builds the transposed (key-pair-major) lists in its workspace
 * (mt_block_sparse_attn_bwd_workspace_bytes(shape, n_blk)); the forward's
 * workspace is mt_block_sparse_attn_fwd_workspace_bytes(shape).
 * Errors: MT_ESHAPE, MT_EWINDOW, MT_EUNSUPPORTED, MT_EWORKSPACE, MT_ECUDA. */
size_t mt_block_sparse_attn_fwd_workspace_bytes(const mt_shape* shape);
mt_status mt_block_sparse_attn_fwd(const mt_shape* shape, const void* q, const void* k,
                                   const void* v, const int64_t* blk_ptr, const int32_t* blk_idx,
                                   int64_t n_blk, void* o, float* lse, void* workspace,
                                   size_t ws_bytes, mt_stream_t stream);
size_t mt_block_sparse_attn_bwd_workspace_bytes(const mt_shape* shape, int64_t n_blk);
mt_status mt_block_sparse_attn_bwd(const mt_shape* shape, const void* q, const void* k,
                                   const void* v, const void* o, const float* lse,
                                   const void* dO, const int64_t* blk_ptr,
                                   const int32_t* blk_idx, int64_t n_blk, void* dq, void* dk,
                                   void* dv, void* workspace, size_t ws_bytes,
                                   mt_stream_t stream);

/* XAttention antidiagonal block index ("w/ XAttn Idx."; block 128,
 * stride 16, threshold 0.9; reading R25 in DESIGN.md).  Per q head, on the stride
 * grid i, j < S/16: A[i][j] = sum_s q[16i+15-s] . k[16j+s] / (16 sqrt d); row
 * softmax over j <= i; block scores Bs[I][J] = sums of 8 x 8 sub-blocks (J <= I);
 * per query block I the shortest descending prefix of Bs[I][.] reaching
 * threshold * row total is kept (ties: smaller J first), plus the diagonal; the
 * kept 128-blocks are written as the 64-token CSR of mt_block_sparse_attn_*
 * (query blocks 2I, 2I+1; key blocks 2J, 2J+1; for J = I the causal half).
 * q [S][Hq][128], k [S][Hkv][128] bf16 device (post-RoPE), world 1, S % 128 == 0.
 * Two calls sharing one workspace: mt_xattn_index_count computes everything,
 * writes blk_ptr (device int64 [Hq][nb + 1], global offsets) and the total n_blk
 * to the HOST (it synchronizes the stream), and optionally copies the block scores
 * to block_scores (device fp32 [Hq][nI (nI + 1) / 2], row I at I (I + 1) / 2,
 * nI = S / 128; may be NULL); mt_xattn_index_fill then writes blk_idx (device
 * int32, capacity >= n_blk) from the selection left in the workspace.
 * The strided score GEMM is a cuBLAS bf16 GEMM (fp32 output) that runs in a 32 MiB
 * slice of the caller's workspace; everything else is this library's kernels.  The
 * process-wide cuBLAS handle (created on first use) holds cuBLAS's own small
 * internal state, the one allocation outside caller workspaces.  Errors: MT_ESHAPE, MT_EWINDOW (S % 128), MT_EUNSUPPORTED
 * (block/stride other than 128/16), MT_EWORKSPACE, MT_ECAPACITY, MT_ECUDA. */
typedef struct {
  int block;       /* 128 */
  int stride;      /* 16 */
  float threshold; /* in [0, 1]; the paper's 0.9 */
} mt_xattn_params;
size_t mt_xattn_index_workspace_bytes(const mt_shape* shape);
mt_status mt_xattn_index_count(const mt_shape* shape, const mt_xattn_params* params,
                               const void* q, const void* k, int64_t* blk_ptr, int64_t* n_blk,
                               float* block_scores, void* workspace, size_t ws_bytes,
                               mt_stream_t stream);
mt_status mt_xattn_index_fill(const mt_shape* shape, const mt_xattn_params* params,
                              const int64_t* blk_ptr, int32_t* blk_idx, int64_t capacity,
                              int64_t n_blk, void* workspace, size_t ws_bytes,
                              mt_stream_t stream);

/* ------------------------------------------------------------------ rope */
/* Rotary position embedding, the step upstream of the index and the attention
 * (SURVEY §8(f) f3).  PAPER.md Appendix A: the half-split pairs
 * (x[i], x[i + 64]) of a 128-wide head vector at global position n rotate by
 * n * theta_i; YaRN with factor 32 (readings: DESIGN.md R-rope).
 * mt_rope_inv_freq (host only): theta[0..63] = base^(-2i/128), YaRN-adjusted
 * (NTK-by-parts, beta_fast 32, beta_slow 1, original context
 * original_max_position) when yarn_factor > 1, and the YaRN scale mscale
 * (0.1 ln(factor) + 1; 1 without YaRN).
 * mt_rope: in place on a token-major bf16 [S/W][n_heads][128] device tensor of
 * rank `rank` in the block-striped layout (global positions as mt_stripe);
 * x <- mscale * R(n) x, or mscale * R(-n) x when inverse (the backward map).
 * Errors: MT_ESHAPE, MT_EWINDOW, MT_ELAYOUT, MT_ECUDA. */
mt_status mt_rope_inv_freq(int head_dim, double base, double yarn_factor,
                           int64_t original_max_position, double* theta, float* mscale);
mt_status mt_rope(int64_t seq_len, int world, int rank, int n_heads, const double* theta,
                  float mscale, int inverse, void* x, mt_stream_t stream);

/* ------------------------------------------------------------------ layout */
/* Block-striped context-parallel layout (SURVEY §8 a1,
 * reading Q12): global 64-token block b lives on rank b mod W as local block
 * floor(b / W), i.e. local row j of rank r <-> global token
 * (floor(j / 64) * W + r) * 64 + j mod 64.  Tensors are token-major with
 * `row_bytes` bytes per token (e.g. Hq * 128 * 2 for bf16 Q); both pointers are
 * device pointers owned by the caller; row_bytes must be a multiple of 16.
 *   mt_stripe:   local[S/W rows]  <- global[S rows]   (rank r's share)
 *   mt_unstripe: global[S rows]   <- local[S/W rows]  (writes only rank r's rows)
 * Errors: MT_ESHAPE (NULL, row_bytes % 16, bad rank/world), MT_EWINDOW,
 * MT_ELAYOUT (S % (64 W)), MT_ECUDA. */
mt_status mt_stripe(int64_t seq_len, int64_t row_bytes, int world, int rank,
                    const void* global, void* local, mt_stream_t stream);
mt_status mt_unstripe(int64_t seq_len, int64_t row_bytes, int world, int rank,
                      const void* local, void* global, mt_stream_t stream);

/* The same copies for either layout (MT_LAYOUT_STRIPED as mt_stripe / mt_unstripe, or
 * MT_LAYOUT_ZIGZAG: local row j of rank r <-> global token of chunk r (j < S/2W) or
 * chunk 2W-1-r; Fig. 1).  Errors as above, plus MT_ESHAPE for an
 * unknown layout and MT_ELAYOUT when zigzag and S % (128 W) != 0. */
mt_status mt_layout_to_local(int layout, int64_t seq_len, int64_t row_bytes, int world,
                             int rank, const void* global, void* local, mt_stream_t stream);
mt_status mt_layout_to_global(int layout, int64_t seq_len, int64_t row_bytes, int world,
                              int rank, const void* local, void* global, mt_stream_t stream);

/* ------------------------------------------------------------------ tests */
/* Hardware self-test hook (not part of the attention API): one 128-row tcgen05
 * MMA configuration on one CTA, see csrc/selftest.cu for the variants.
 * A, B: bf16 device buffers, D: float32 device buffer [128][N]. */
mt_status mt_selftest_mma(int variant, const void* A, const void* B, float* D,
                          mt_stream_t stream);

/* Profiling hook (not part of the attention API): copies the backward kernel's
 * timeline probe — int64 clock64 stamps [8 events][4096 chunk events] of CTA 0 of
 * the most recent launch — to host memory `out` (8 * 4096 int64).  All zeros
 * unless the library was built with -DMT_TIMELINE (MT_NVCC_EXTRA). */
mt_status mt_debug_bwd_timeline(int64_t* out);
/* Same for the forward kernel (CTA 0 of the most recent launch). */
mt_status mt_debug_fwd_timeline(int64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* MTSA_H_ */
