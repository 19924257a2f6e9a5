// attn_fwd.cu — block-sparse vertical-slash attention forward for sm_100a, one
// ring step (Alg. 2 "block_bar_sparse_attention_forward" P:878 then
// "merge_out_and_lse" P:879; with W = 1 the single step is Alg. 1's
// "sparse(softmax(QK^T/sqrt d)V, i_vs)").
//
// Transposed ("key-major") tiles so the 64-granular pattern costs no MMA waste:
//   tile  = one 64-query block g of one q head h (N = 64 of every MMA);
//   chunk = 128 keys that ALL belong to this block's key set: two 64-key slash
//           blocks of B_g (TMA), or up to 128 gathered vertical columns of C_g
//           (cp.async), restricted to the held KV origin (I9/I10);
//   S^T = K Q^T          tcgen05 M=128 (keys) N=64 K=128 (d)      -> TMEM
//   P^T = 2^(S^T c - m_q) in registers (thread = key row, 32 query columns)
//   O^T += V^T P^T       tcgen05 M=128 (d)    N=64 K=128 (keys)   -> TMEM
// The column stabiliser m_q is the exact max of the tile's first chunk (every
// query sees >= 1 key there); later chunks move it (with an O^T / l rescale)
// only if a score exceeds it by 2^64 — a rare slow path.  Row sums l_q are
// per-thread partials reduced once per tile.
//
// Warp roles (384 threads, 1 CTA / SM, persistent; setmaxnreg moves registers
// from warpgroup 0 to the softmax warpgroups):
//   warp 0       producer (chunk stream from the VSPlan, TMA / cp.async)
//   warp 1       MMA issuer (one lane)
//   warp 2       V producer (decoupled from K through a metadata ring)
//   warp 3       idle
//   warps 4..11  two softmax warpgroups; warpgroup g takes the tile's chunks
//                k = g (mod 2); warp w covers TMEM lanes 32*(w%4)..
#include <cstdlib>

#include "common.cuh"
#include "plan.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace mt {

namespace fwd {

#ifndef MT_FWD_KST
#define MT_FWD_KST 2
#endif
#ifndef MT_FWD_VST
#define MT_FWD_VST 3
#endif
constexpr int kKSt = MT_FWD_KST, kVSt = MT_FWD_VST;  // V lives ~2 chunks longer than K (O^T lags S^T)
constexpr int kThreads = 384;  // warpgroup 0: producer, MMA, 2 idle; warpgroups 1-2: softmax
constexpr int kSoftmax = 256;
constexpr uint32_t kTileKV = 128 * 128 * 2;  // 32 KB
constexpr uint32_t kTileQ = 64 * 128 * 2;    // 16 KB
constexpr uint32_t kTileP = 128 * 64 * 2;    // 16 KB
constexpr float kOverflow = 64.f;            // log2 headroom before the stabiliser moves

// kBarP: a bar chunk of 128 consecutive packed rows (TMA), live rows in `mask`
enum : int { kBlk = 0, kBar = 1, kEnd = 2, kDone = 3, kBarP = 4 };

struct alignas(16) ChunkMeta {  // per K slot: what the MMA / softmax need
  int kind;
  int n;           // kBar: live rows
  uint32_t flags;  // kBlk: bit0 rows 64..127 live, bit1 rows 0..63 diagonal, bit2 rows 64..127 diagonal
  int tile;        // kEnd: the tile it closes
  uint32_t mask[4];  // kBarP: live rows (not covered by a selected slash, inside the prefix)
};

struct alignas(16) VMeta {  // per data chunk: what the producers need to stage K/V
  int kind;
  int n;
  int lb0, lb1;    // kBarP: lb0 = first packed row
  int gkv;         // kBarP: the q head (packed rows are per q head)
  int pad[3];
  int rows[128];   // kBar local rows
};

constexpr int kVM = 4;  // V-metadata ring depth
constexpr int kSbitsWords = 1024;  // SMEM copy of a head's slash bitmap: nb <= 32768 (2M tokens)

struct SMeta {
  int kind, n;
  uint32_t flags;
  int tile;
  int seq;  // data chunk index (timeline probe)
  uint32_t mask[4];  // kBarP live rows
};

struct Smem {
  uint8_t k[kKSt][kTileKV];
  uint8_t v[kVSt][kTileKV];
  uint8_t q[kTileQ];
  uint8_t p[2][kTileP];
  ChunkMeta meta[kKSt];
  VMeta vmeta[kVM];
  SMeta smeta[2];
  alignas(16) float red[2][4][32];  // column-max partials (two 32-column halves)
  alignas(16) float lsum[2][4][64]; // per WG, per lane quadrant: row-sum partials
  alignas(16) float m[64];          // column stabiliser (log2 domain), read as float4
  alignas(16) float wa[64];         // rescale factors / epilogue merge weights
  alignas(16) float wb[64];
  int stage_rows[192];
  // bar chunks: K-gather requests from the K producer (warp 0) to the gatherer (warp 3)
  struct alignas(16) GatherReq {
    int rows[128];
    int ks, gkv, pad[2];
  } greq[2];
  uint32_t sbits[kSbitsWords];  // the tile head's slash bitmap (producer warp only)
  int ovf;
  uint64_t kfull[kKSt], kempty[kKSt], vfull[kVSt], vempty[kVSt];
  uint64_t sfull[2], sfree[2], pfull[2], obar[2];
  uint64_t vmfull[kVM], vmfree[kVM];
  uint64_t qfull, qempty, mready;
  uint64_t gqfull[2], gqempty[2];
  uint32_t tmem_base;
};

struct Params {
  VSPlan plan;
  int r, s, t;
  int nloc;
  int n_tiles;
  int first, last;
  float scale_log2;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  __nv_bfloat16* o;
  float* o_acc;
  float* lse;
  int* fix_count;  // tiles flagged for the exact fix-up pass (stabiliser overflow)
  int* fix_list;
  int* tile_counter;  // dynamic tile scheduler (zeroed before the launch)
  int order;          // tile order (MT_FWD_ORDER): 1 head-major (default; L2 reuse of K/V), 0 query-block-major
  int packed;         // bar chunks from the packed rows (plan.kp / vp) by TMA (MT_FWD_PACK, default 1)
};

constexpr uint32_t kColO = 0, kColS = 64;  // TMEM: O^T [0,64), S^T buffers [64,128) [128,192)

__device__ __forceinline__ void tile_coords(const Params& P, int tile, int& h, int& j) {
  const int Hq = P.plan.Hq;
  if (P.order) {  // head-major: resident tiles = consecutive query blocks of one head
    h = tile / P.nloc;
    j = P.nloc - 1 - tile % P.nloc;
  } else {
    j = P.nloc - 1 - tile / Hq;  // late query blocks (most keys) first
    h = tile % Hq;
  }
}

// ------------------------------------------------------------------ producers
// Warp 0 builds the chunk stream and issues K (slot frees after S^T three chunks
// back); warp 2 issues V (slot frees after the O^T two data chunks back).  They
// are decoupled by a 4-entry ring of V metadata, so a late V slot never delays
// the next K.  K slots (and the per-chunk meta the MMA reads) are indexed by
// every chunk including END markers; V slots only by data chunks.
__device__ void producer_k(Smem& sm, const Params& P, const CUtensorMap* tmq,
                           const CUtensorMap* tmk, const CUtensorMap* tmkp) {
  const int lane = lane_id();
  const VSPlan& pl = P.plan;
  const int W = pl.W;
  const int grp = pl.Hq / pl.Hkv;
  uint32_t c = 0, dk = 0;  // chunks (incl. END), data chunks
  uint32_t ng = 0;         // K-gather requests posted to warp 3
  uint32_t qe_phase = 0;
  bool first_tile = true;

  auto kacquire = [&]() {
    mbar_wait(smem_u32(&sm.kempty[c % kKSt]), ((c / kKSt) & 1) ^ 1);
  };
  auto vmacquire = [&]() -> VMeta& {
    mbar_wait(smem_u32(&sm.vmfree[dk % kVM]), ((dk / kVM) & 1) ^ 1);
    return sm.vmeta[dk % kVM];
  };
  auto vmrelease = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&sm.vmfull[dk % kVM]));
    ++dk;
  };

  for (;;) {
    int tile = 0;
    if (lane == 0) tile = atomicAdd(P.tile_counter, 1);
    tile = __shfl_sync(0xffffffffu, tile, 0);
    if (tile >= P.n_tiles) break;
    int h, j;
    tile_coords(P, tile, h, j);
    const int g = j * W + P.r;
    const int gkv = h / grp;
    if (!first_tile) {
      mbar_wait(smem_u32(&sm.qempty), qe_phase);
      qe_phase ^= 1;
    }
    first_tile = false;
    if (lane == 0) {
      const uint32_t bar = smem_u32(&sm.qfull);
      mbar_expect_tx(bar, kTileQ);
      for (int cc = 0; cc < 2; ++cc)
        tma_load_3d(smem_u32(sm.q + cc * 8192), tmq, bar, cc * 64, h, j * 64);
    }
    // ---- slash blocks of residue t, two per chunk
    {
      auto emit_pair = [&](int o0, int o1) {  // o1 < 0: second slot empty
        const int lb0 = (g - o0 - P.s) / W;
        const int lb1 = o1 >= 0 ? (g - o1 - P.s) / W : lb0;
        uint32_t flags = 0;
        if (o1 >= 0) flags |= 1u;
        if (o0 == 0) flags |= 2u;
        if (o1 == 0) flags |= 4u;
        VMeta& vm = vmacquire();
        kacquire();
        if (lane == 0) {
          vm.kind = kBlk;
          vm.lb0 = lb0;
          vm.lb1 = lb1;
          vm.gkv = gkv;
          const uint32_t ks = c % kKSt;
          ChunkMeta& m = sm.meta[ks];
          m.kind = kBlk;
          m.flags = flags;
          const uint32_t kb = smem_u32(&sm.kfull[ks]);
          mbar_expect_tx(kb, kTileKV);
#ifndef MT_TL_FWD_TILE
          MT_TL(0, dk);
#endif
          for (int cc = 0; cc < 2; ++cc)
            for (int x = 0; x < 2; ++x)
              tma_load_3d(smem_u32(sm.k[ks] + cc * 16384 + x * 8192), tmk, kb, cc * 64, gkv,
                          (x ? lb1 : lb0) * 64);
        }
        vmrelease();
        ++c;
      };
      // offsets of residue t (= ring step) with o <= g, ascending, two per chunk.  The
      // list is read 32 offsets per coalesced load and filtered with a ballot: a scalar
      // walk costs one dependent global load per offset, and at W > 1 it skips the
      // (W-1)/W offsets of other steps (measured: 3.2K cycles per chunk at W = 4).
      int pending = -1;
      auto take = [&](int ov) {
        if (pending < 0) {
          pending = ov;
        } else {
          emit_pair(pending, ov);
          pending = -1;
        }
      };
      if (pl.bptr) {
        // block-CSR mode (W = 1): the row's key blocks, last first (offsets ascending,
        // the diagonal first as in VS mode)
        const int64_t rb = pl.bptr[(int64_t)h * (pl.nb + 1) + g];
        const int64_t re = pl.bptr[(int64_t)h * (pl.nb + 1) + g + 1];
        for (int64_t top = re - 1; top >= rb; top -= 32) {
          const int64_t i = top - lane;
          const int o = i >= rb ? g - pl.bidx[i] : 0;
          uint32_t bal = __ballot_sync(0xffffffffu, i >= rb);
          while (bal) {
            const int l = __ffs(bal) - 1;
            bal &= bal - 1;
            take(__shfl_sync(0xffffffffu, o, l));
          }
        }
      }
      const int ns = pl.bptr ? 0 : pl.s_cnt[h];
      const int32_t* offs = pl.s_off + (int64_t)h * pl.s_stride;
      for (int base = 0; base < ns; base += 32) {
        const int o = base + lane < ns ? offs[base + lane] : INT_MAX;
        const bool past = o > g;  // ascending: nothing later matches
        uint32_t bal = __ballot_sync(0xffffffffu, !past && (o % W) == P.t);
        while (bal) {
          const int l = __ffs(bal) - 1;
          bal &= bal - 1;
          take(__shfl_sync(0xffffffffu, o, l));
        }
        if (__any_sync(0xffffffffu, past)) break;
      }
      if (pending >= 0) emit_pair(pending, -1);
    }
    // ---- bars of origin s: block < g, offset not a selected slash; 128 per chunk
    {
      const int32_t* vc = pl.vcol + (int64_t)h * pl.S;
      const int vb = pl.vptr[h * (W + 1) + P.s];
      const int ve = pl.vptr[h * (W + 1) + P.s + 1];
      int nst = 0;
      // the coverage test reads the head's slash bitmap from SMEM (once per tile)
      const bool bits_smem = pl.bits_words <= kSbitsWords;
      if (bits_smem && vb < ve) {
        const uint32_t* gb = pl.s_bits + (int64_t)h * pl.bits_words;
        for (int w = lane; w < pl.bits_words; w += 32) sm.sbits[w] = gb[w];
        __syncwarp();
      }
      auto covered = [&](int o) {
        return bits_smem ? ((sm.sbits[o >> 5] >> (o & 31)) & 1u) != 0u : plan_has_slash(pl, h, o);
      };
      if (P.packed && ve - vb <= pl.pcap) {
        // packed path: the head's columns of origin s are packed rows 0 .. ve-vb-1; the
        // columns of blocks < g are a prefix; chunk = 128 consecutive rows (TMA), rows
        // covered by a selected slash masked out (all-masked chunks are skipped)
        for (int i0 = 0; vb + i0 < ve; i0 += 128) {
          uint32_t msk[4];
          bool past = false;
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const int i = vb + i0 + 32 * w + lane;
            const int m = i < ve ? vc[i] : INT_MAX;
            const bool in = (m >> 6) < g;
            msk[w] = __ballot_sync(0xffffffffu, in && !covered(g - (m >> 6)));
            past |= __ballot_sync(0xffffffffu, in) != 0xffffffffu;
          }
          if (msk[0] | msk[1] | msk[2] | msk[3]) {
            VMeta& vm = vmacquire();
            kacquire();
            if (lane == 0) {
              vm.kind = kBarP;
              vm.lb0 = i0;
              vm.gkv = h;
              const uint32_t ks = c % kKSt;
              ChunkMeta& m = sm.meta[ks];
              m.kind = kBarP;
              m.n = 128;
#pragma unroll
              for (int w = 0; w < 4; ++w) m.mask[w] = msk[w];
              const uint32_t kb = smem_u32(&sm.kfull[ks]);
              mbar_expect_tx(kb, kTileKV);
              for (int cc = 0; cc < 2; ++cc)
                for (int x = 0; x < 2; ++x)
                  tma_load_3d(smem_u32(sm.k[ks] + cc * 16384 + x * 8192), tmkp, kb, cc * 64, h,
                              i0 + 64 * x);
            }
            vmrelease();
            ++c;
          }
          if (past) break;
        }
      } else {
      auto emit = [&](int n) {
        VMeta& vm = vmacquire();
        kacquire();
        const uint32_t ks = c % kKSt;
        for (int x = lane; x < 128; x += 32) vm.rows[x] = sm.stage_rows[x < n ? x : 0];
        if (lane == 0) {
          vm.kind = kBar;
          vm.n = n;
          vm.gkv = gkv;
          sm.meta[ks].kind = kBar;
          sm.meta[ks].n = n;
        }
        __syncwarp();
        {  // hand the K gather to warp 3 (it arrives on kfull[ks] when the rows land)
          const uint32_t gi = ng & 1;
          mbar_wait(smem_u32(&sm.gqempty[gi]), ((ng >> 1) & 1) ^ 1);
          for (int x = lane; x < 128; x += 32) sm.greq[gi].rows[x] = vm.rows[x];
          if (lane == 0) {
            sm.greq[gi].ks = (int)ks;
            sm.greq[gi].gkv = gkv;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&sm.gqfull[gi]));
          ++ng;
        }
        vmrelease();
        ++c;
        const int rem = nst - n;  // shift the remaining staged columns down
        int t0 = 0;
        if (lane < rem) t0 = sm.stage_rows[n + lane];
        __syncwarp();
        if (lane < rem) sm.stage_rows[lane] = t0;
        __syncwarp();
        nst = rem;
      };
      int m_next = vb + lane < ve ? vc[vb + lane] : 0;  // loads run one batch ahead
      for (int base = vb; base < ve; base += 32) {
        const int i = base + lane;
        const int m = m_next;
        if (base + 32 + lane < ve) m_next = vc[base + 32 + lane];
        bool keep = false, more = false;
        int lrow = 0;
        if (i < ve) {
          const int blk = m >> 6;
          if (blk < g) {
            more = true;
            keep = !covered(g - blk);
            lrow = ((blk - P.s) / W) * 64 + (m & 63);
          }
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (keep) sm.stage_rows[nst + __popc(bal & ((1u << lane) - 1u))] = lrow;
        __syncwarp();
        nst += __popc(bal);
        if (nst >= 128) emit(128);
        if (!__any_sync(0xffffffffu, more)) break;
      }
      if (nst > 0) emit(nst);
      }
    }
    // ---- END (K slot + meta only)
    kacquire();
    if (lane == 0) {
      const uint32_t ks = c % kKSt;
      sm.meta[ks].kind = kEnd;
      sm.meta[ks].tile = tile;
      mbar_arrive(smem_u32(&sm.kfull[ks]));
    }
    __syncwarp();
    ++c;
  }
  // ---- DONE: no more tiles for this CTA; stop the K gatherer
  {
    const uint32_t gi = ng & 1;
    mbar_wait(smem_u32(&sm.gqempty[gi]), ((ng >> 1) & 1) ^ 1);
    if (lane == 0) {
      sm.greq[gi].ks = -1;
      mbar_arrive(smem_u32(&sm.gqfull[gi]));
    }
    __syncwarp();
    ++ng;
  }
  kacquire();
  if (lane == 0) {
    const uint32_t ks = c % kKSt;
    sm.meta[ks].kind = kDone;
    mbar_arrive(smem_u32(&sm.kfull[ks]));
  }
  __syncwarp();
  // tell the V producer there is nothing more
  VMeta& vm = vmacquire();
  if (lane == 0) vm.kind = kEnd;
  vmrelease();
}

// Warp 3: K rows of bar chunks, gathered with cp.async into the K stage the K
// producer acquired (so its column scan runs on while the rows are in flight).
__device__ void k_gatherer(Smem& sm, const Params& P) {
  const int lane = lane_id();
  const int Hkv = P.plan.Hkv;
  for (uint32_t n = 0;; ++n) {
    const uint32_t gi = n & 1;
    mbar_wait_idle(smem_u32(&sm.gqfull[gi]), (n >> 1) & 1);
    const int ks = sm.greq[gi].ks, gkv = sm.greq[gi].gkv;
    if (ks < 0) break;
    const uint32_t kbase = smem_u32(sm.k[ks]);
    for (int pidx = lane; pidx < 128 * 16; pidx += 32) {
      const int row = pidx >> 4, c16 = pidx & 15;
      const size_t goff = ((size_t)sm.greq[gi].rows[row] * Hkv + gkv) * 128 + c16 * 8;
      cp_async_16(kbase + (c16 >> 3) * 16384 + sw128(row, c16 & 7), P.k + goff);
    }
    const uint32_t kb = smem_u32(&sm.kfull[ks]);
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(kb) : "memory");
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(kb);
      mbar_arrive(smem_u32(&sm.gqempty[gi]));  // rows read: the request slot is free
    }
  }
}

__device__ void producer_v(Smem& sm, const Params& P, const CUtensorMap* tmv,
                           const CUtensorMap* tmvp) {
  const int lane = lane_id();
  const VSPlan& pl = P.plan;
  for (uint32_t dv = 0;; ++dv) {
    mbar_wait(smem_u32(&sm.vmfull[dv % kVM]), (dv / kVM) & 1);
    const VMeta& vm = sm.vmeta[dv % kVM];
    const int kind = vm.kind;
    if (kind == kEnd) break;
    const uint32_t vs = dv % kVSt;
    mbar_wait(smem_u32(&sm.vempty[vs]), ((dv / kVSt) & 1) ^ 1);
#if !defined(MT_TL_FWD_WG) && !defined(MT_TL_FWD_TILE)
    if (lane == 0) MT_TL(1, dv);
#endif
    const uint32_t vb = smem_u32(&sm.vfull[vs]);
    if (kind == kBlk) {
      if (lane == 0) {
        mbar_expect_tx(vb, kTileKV);
        for (int cc = 0; cc < 2; ++cc)
          for (int x = 0; x < 2; ++x)
            tma_load_3d(smem_u32(sm.v[vs] + cc * 16384 + x * 8192), tmv, vb, cc * 64, vm.gkv,
                        (x ? vm.lb1 : vm.lb0) * 64);
      }
    } else if (kind == kBarP) {
      if (lane == 0) {
        mbar_expect_tx(vb, kTileKV);
        for (int cc = 0; cc < 2; ++cc)
          for (int x = 0; x < 2; ++x)
            tma_load_3d(smem_u32(sm.v[vs] + cc * 16384 + x * 8192), tmvp, vb, cc * 64, vm.gkv,
                        vm.lb0 + 64 * x);
      }
    } else {
      const uint32_t vbase = smem_u32(sm.v[vs]);
      for (int pidx = lane; pidx < 128 * 16; pidx += 32) {
        const int row = pidx >> 4, c16 = pidx & 15;
        const size_t goff = ((size_t)vm.rows[row] * pl.Hkv + vm.gkv) * 128 + c16 * 8;
        cp_async_16(vbase + (c16 >> 3) * 16384 + sw128(row, c16 & 7), P.v + goff);
      }
      asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(vb) : "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(vb);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&sm.vmfree[dv % kVM]));
  }
}

// ------------------------------------------------------------------ MMA issuer
// Chunk k of a tile goes to S^T / P^T buffer k & 1, i.e. to softmax warpgroup
// k & 1: the two warpgroups alternate chunks so one computes while the tensor
// core works for the other.  O^T for a chunk is issued two chunks later (after
// S^T(k + 2)), so a warpgroup's next S^T never waits for its own P^T.  END is
// published to both warpgroups after the tile's last O^T.
__device__ void mma_issuer(Smem& sm, const Params& P, uint32_t tmem) {
  const bool leader = elect_one();
  const uint32_t id_s = make_idesc_bf16(128, 64, false, false);
  const uint32_t id_o = make_idesc_bf16(128, 64, true, true);
  // descriptor bases; each MMA only adds an immediate to the address field
  const uint64_t dq0 = make_sdesc(smem_u32(sm.q), 16, 1024);
  const uint64_t dk0 = make_sdesc(smem_u32(sm.k[0]), 16, 1024);
  const uint64_t dv0 = make_sdesc(smem_u32(sm.v[0]), 16384, 1024);
  const uint64_t dp0 = make_sdesc(smem_u32(sm.p[0]), 8192, 1024);
  uint32_t c = 0, dc = 0, oc = 0, qf_phase = 0;  // chunks, data chunks S-issued, O^T-issued
  uint32_t su0 = 0, su1 = 0, pu0 = 0, pu1 = 0;   // per-buffer use counts (S events, P data)
  bool o_started = false;
  int kind_ring[4];
  uint32_t buf_ring[4];  // S^T / P^T buffer of each pending data chunk (tile-local parity)
  auto wait_sfree = [&](uint32_t b) {
    if (b == 0) { mbar_wait(smem_u32(&sm.sfree[0]), (su0 & 1) ^ 1); ++su0; }
    else        { mbar_wait(smem_u32(&sm.sfree[1]), (su1 & 1) ^ 1); ++su1; }
  };
  // O^T += V^T P^T for the oldest data chunk not yet accumulated (oc)
  auto issue_o = [&]() {
    const uint32_t b = buf_ring[oc & 3], vs = oc % kVSt;
    mbar_wait(smem_u32(&sm.vfull[vs]), (oc / kVSt) & 1);
    if (leader) MT_TL(7, oc);
    if (kind_ring[oc & 3] == kBar) fence_proxy_async_smem();
    if (b == 0) { mbar_wait(smem_u32(&sm.pfull[0]), pu0 & 1); ++pu0; }
    else        { mbar_wait(smem_u32(&sm.pfull[1]), pu1 & 1); ++pu1; }
    tc_fence_after();
    const uint64_t dv = sdesc_add(dv0, vs * kTileKV), dp = sdesc_add(dp0, b * kTileP);
    if (leader) {
#pragma unroll
      for (int kk = 0; kk < 128; kk += 16)
        mma_ss(tmem + kColO, sdesc_add(dv, kk * 128), sdesc_add(dp, kk * 128), id_o,
               (o_started || kk > 0) ? 1u : 0u);
      mma_commit(smem_u32(&sm.obar[b]));
      mma_commit(smem_u32(&sm.vempty[vs]));
      MT_TL(3, oc);
    }
    o_started = true;
    ++oc;
  };
  for (;;) {
    {  // the next chunk tells whether another tile follows
      const uint32_t ks = c % kKSt;
      mbar_wait(smem_u32(&sm.kfull[ks]), (c / kKSt) & 1);
      if (sm.meta[ks].kind == kDone) {
        for (uint32_t b = 0; b < 2; ++b) {
          wait_sfree(b);
          if (leader) {
            sm.smeta[b].kind = kDone;
            mbar_arrive(smem_u32(&sm.sfull[b]));
            mbar_arrive(smem_u32(&sm.sfull[b]));
          }
        }
        break;
      }
    }
    mbar_wait(smem_u32(&sm.qfull), qf_phase);
#ifdef MT_TL_FWD_TILE
    if (leader) MT_TL(6, dc);  // next tile's Q landed
#endif
    qf_phase ^= 1;
    tc_fence_after();
    o_started = false;
    uint32_t k = 0;  // chunk index inside the tile (data chunks)
    for (;;) {
      const uint32_t ks = c % kKSt;
      mbar_wait(smem_u32(&sm.kfull[ks]), (c / kKSt) & 1);
      const int kind = sm.meta[ks].kind;
      const int end_tile = sm.meta[ks].tile;  // read before the slot is released
      if (kind == kBar) fence_proxy_async_smem();
      tc_fence_after();
      ++c;
      if (kind == kEnd) {
#ifdef MT_TL_FWD_TILE
        if (leader) MT_TL(0, dc);  // END seen (dc = next tile's first data chunk)
#endif
        if (leader) {
          mma_commit(smem_u32(&sm.qempty));  // every S^T of the tile issued before
          mbar_arrive(smem_u32(&sm.kempty[ks]));
        }
        while (oc < dc) issue_o();
        for (uint32_t b = 0; b < 2; ++b) {
          wait_sfree(b);
          if (leader) {
            sm.smeta[b].kind = kEnd;
            sm.smeta[b].tile = end_tile;
            mbar_arrive(smem_u32(&sm.sfull[b]));
            mbar_arrive(smem_u32(&sm.sfull[b]));
          }
        }
#ifdef MT_TL_FWD_TILE
        if (leader) MT_TL(1, dc);  // remaining O^T issued, END published
#endif
        break;
      }
#ifndef MT_TL_FWD_TILE
      if (leader) MT_TL(6, dc);
#endif
      const uint32_t b = k & 1;
      wait_sfree(b);
      if (leader) {
        sm.smeta[b].seq = (int)dc;
        sm.smeta[b].kind = kind;
        sm.smeta[b].n = sm.meta[ks].n;
        sm.smeta[b].flags = sm.meta[ks].flags;
#pragma unroll
        for (int w = 0; w < 4; ++w) sm.smeta[b].mask[w] = sm.meta[ks].mask[w];
        mbar_arrive(smem_u32(&sm.sfull[b]));  // 1 of 2: publishes smeta
        const uint64_t dk = sdesc_add(dk0, ks * kTileKV);
        const uint32_t ts = tmem + kColS + 64 * b;
#pragma unroll
        for (int kk = 0; kk < 128; kk += 16)
          mma_ss(ts, sdesc_add(dk, (kk >> 6) * 16384 + (kk & 63) * 2),
                 sdesc_add(dq0, (kk >> 6) * 8192 + (kk & 63) * 2), id_s, kk > 0);
        mma_commit(smem_u32(&sm.sfull[b]));  // 2 of 2: S^T ready
        mma_commit(smem_u32(&sm.kempty[ks]));
        MT_TL(2, dc);
      }
      kind_ring[dc & 3] = kind;
      buf_ring[dc & 3] = b;
      ++dc;
      ++k;
      if (dc - oc > 2) issue_o();  // O^T lags S^T by two data chunks
    }
  }
}

// ------------------------------------------------------------------ softmax + epilogue
// Reduce 32 columns across the 32 lanes of a warp (recursive halving, 31
// shuffles): afterwards lane L holds the reduction of column L.
template <bool kMax>
__device__ __forceinline__ float warp_colreduce(float* x) {
  const int lane = lane_id();
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool upper = lane & w;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float send = upper ? x[i] : x[i + w];
      const float keep = upper ? x[i + w] : x[i];
      const float got = __shfl_xor_sync(0xffffffffu, send, w);
      x[i] = kMax ? fmaxf(keep, got) : keep + got;
    }
  }
  return x[0];
}

__device__ __forceinline__ float4 lds_f4(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Warpgroup `wg` owns S^T / P^T buffer wg and processes the tile's chunks
// k = wg (mod 2), all 64 query columns; warp w covers TMEM lanes 32*(w%4)...
// The stabiliser m_q is the exact column max of the tile's chunk 0 (computed by
// warpgroup 0, handed to warpgroup 1 through the mready mbarrier).  A score
// more than 2^64 above it marks the tile for the exact fix-up pass.
__device__ void softmax_epilogue(Smem& sm, const Params& P, uint32_t tmem) {
  const int w = warp_id();
  const int quad = w & 3, wg = (w - 4) >> 2;
  const int lane = lane_id();
  const int row = quad * 32 + lane;  // key row of S^T (and d row of O^T)
  const uint32_t lb = ((uint32_t)(quad * 32) << 16);
  const int Hq = P.plan.Hq;
  const int64_t S_loc = (int64_t)P.nloc * 64;
  const uint32_t sfull = smem_u32(&sm.sfull[wg]), sfree = smem_u32(&sm.sfree[wg]);
  const uint32_t pfull = smem_u32(&sm.pfull[wg]), obar = smem_u32(&sm.obar[wg]);
  const uint32_t mready = smem_u32(&sm.mready);
  const uint32_t prow = smem_u32(sm.p[wg]) + row * 128;
  uint32_t su = 0, pc = 0, pw = 0, mr_phase = 0;

  for (;;) {
    float l[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) l[i] = 0.f;
    bool m_synced = false;
    bool ovf = false;
    int tile = -1;
    for (;;) {
      mbar_wait(sfull, su & 1);
      ++su;
      const SMeta cm = sm.smeta[wg];
      if (cm.kind == kEnd || cm.kind == kDone) {
        mbar_arrive(sfree);
        tile = cm.kind == kEnd ? cm.tile : -1;
        break;
      }
      if (row == 0) MT_TL(4, cm.seq);
      tc_fence_after();
      uint32_t sr[64];
      tmem_ld32(tmem + lb + kColS + 64 * wg, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
      tmem_ld32(tmem + lb + kColS + 64 * wg + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(sfree);
      const int kk = row & 63;
      bool live, diag;
      if (cm.kind == kBlk) {
        live = row < 64 || (cm.flags & 1u);
        diag = (row < 64) ? (cm.flags & 2u) : (cm.flags & 4u);
      } else if (cm.kind == kBarP) {
        live = (cm.mask[row >> 5] >> (row & 31)) & 1u;
        diag = false;
      } else {
        live = row < cm.n;
        diag = false;
      }
      if (!m_synced) {
        // chunk 0 of the tile: exact column max over the 128 rows (4 warps) = the
        // tile's fixed stabiliser (log2 units)
        float x[64];
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const bool ok = live && (!diag || kk <= i);
          x[i] = ok ? __uint_as_float(sr[i]) * P.scale_log2 : -INFINITY;
        }
        if (wg == 0) {
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float tmp[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) tmp[i] = x[half * 32 + i];
            sm.red[half][quad][lane] = warp_colreduce<true>(tmp);
          }
          named_bar_sync(1, 128);
          if (quad < 2) {
            const int half = quad;
            sm.m[half * 32 + lane] =
                fmaxf(fmaxf(sm.red[half][0][lane], sm.red[half][1][lane]),
                      fmaxf(sm.red[half][2][lane], sm.red[half][3][lane]));
          }
          named_bar_sync(1, 128);
          mbar_arrive(mready);
        } else {
          mbar_wait(mready, mr_phase);
        }
        m_synced = true;
      }
      // P = exp2(S log2e/sqrt d - m): one FFMA + one MUFU per element; overflow of the
      // fixed stabiliser is tracked as the largest exponent (checked once per chunk)
      uint32_t pk[32];
      float emax = -INFINITY;
      const float sc = P.scale_log2;
      if (!live) {
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
      } else if (!diag) {
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
          const float4 m4 = lds_f4(&sm.m[i]);
          const float t0 = fmaf(__uint_as_float(sr[i]), sc, -m4.x);
          const float t1 = fmaf(__uint_as_float(sr[i + 1]), sc, -m4.y);
          const float t2 = fmaf(__uint_as_float(sr[i + 2]), sc, -m4.z);
          const float t3 = fmaf(__uint_as_float(sr[i + 3]), sc, -m4.w);
          emax = fmaxf(emax, fmaxf(fmaxf(t0, t1), fmaxf(t2, t3)));
          const float p0 = ex2(t0), p1 = ex2(t1), p2 = ex2(t2), p3 = ex2(t3);
          l[i] += p0;
          l[i + 1] += p1;
          l[i + 2] += p2;
          l[i + 3] += p3;
          pk[i >> 1] = pack_bf16x2(p0, p1);
          pk[(i >> 1) + 1] = pack_bf16x2(p2, p3);
        }
      } else {  // diagonal block: causal mask inside (query i sees key kk <= i)
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
          const float4 m4 = lds_f4(&sm.m[i]);
          const float ma[4] = {m4.x, m4.y, m4.z, m4.w};
          float p[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float t = kk <= i + u ? fmaf(__uint_as_float(sr[i + u]), sc, -ma[u]) : -INFINITY;
            emax = fmaxf(emax, t);
            p[u] = ex2(t);
            l[i + u] += p[u];
          }
          pk[i >> 1] = pack_bf16x2(p[0], p[1]);
          pk[(i >> 1) + 1] = pack_bf16x2(p[2], p[3]);
        }
      }
      ovf |= emax > kOverflow;
#ifdef MT_TL_FWD_WG
      if (row == 0) MT_TL(1, cm.seq);  // math done, before waiting for the P^T buffer
#endif
      while (pw < pc) {  // the O^T that last read this P^T buffer is complete
        mbar_wait(obar, pw & 1);
        ++pw;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                         prow + (((uint32_t)u ^ (uint32_t)(row & 7)) << 4)),
                     "r"(pk[4 * u]), "r"(pk[4 * u + 1]), "r"(pk[4 * u + 2]), "r"(pk[4 * u + 3])
                     : "memory");
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(pfull);
      if (row == 0) MT_TL(5, cm.seq);
      ++pc;
    }
    if (tile < 0) break;  // DONE
    int h, j;
    tile_coords(P, tile, h, j);
    // keep the once-per-tile mready phase aligned even without data chunks
    if (!m_synced) {
      if (wg == 0) mbar_arrive(mready);
      else mbar_wait(mready, mr_phase);
    }
    mr_phase ^= 1;
    if (ovf) sm.ovf = 1;

    // ---- epilogue (both warpgroups): l_q, O = O^T / l, LSE, merge with the running result
    // Ring steps after the first merge into the running (O, LSE): issue those global
    // loads now so their latency hides behind the O^T wait and the l reductions.
    const int64_t tok0 = (int64_t)j * 64;
    const size_t qstride = (size_t)Hq * 128;
    const size_t obase = (size_t)tok0 * qstride + (size_t)h * 128 + row;  // O[tok][h][d=row]
    const int col0 = wg * 32;
    float oacc_pre[32];
    float lse_pre = -INFINITY;
    if (!P.first) {
#pragma unroll
      for (int i = 0; i < 32; ++i) oacc_pre[i] = P.o_acc[obase + (size_t)(col0 + i) * qstride];
      if (wg == 0 && quad < 2) lse_pre = P.lse[(int64_t)h * S_loc + tok0 + quad * 32 + lane];
    }
    while (pw < pc) {
      mbar_wait(obar, pw & 1);
      ++pw;
    }
    tc_fence_after();
    named_bar_sync(3, kSoftmax);  // every O^T of the tile complete, ovf flags posted
    sm.lsum[wg][quad][lane] = warp_colreduce<false>(&l[0]);
    sm.lsum[wg][quad][32 + lane] = warp_colreduce<false>(&l[32]);
    const bool tile_ovf = sm.ovf != 0;
    named_bar_sync(3, kSoftmax);
    if (wg == 0 && quad < 2) {
      const int q = quad * 32 + lane;
      float lq = 0.f;
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) lq += sm.lsum[a][b][q];
      float* lp = P.lse + (int64_t)h * S_loc + tok0 + q;
      float wa = 0.f, wb = 0.f;
      if (!tile_ovf) {
        float lse_new = -INFINITY, inv_l = 0.f;
        if (lq > 0.f) {
          inv_l = 1.f / lq;
          lse_new = (sm.m[q] + __log2f(lq)) * 0.69314718055994531f;
        }
        const float lse_old = lse_pre;  // -inf on the first step
        const float mx = fmaxf(lse_old, lse_new);
        float out = -INFINITY;
        if (mx > -INFINITY) {
          const float eo = lse_old == -INFINITY ? 0.f : __expf(lse_old - mx);
          const float en = lse_new == -INFINITY ? 0.f : __expf(lse_new - mx);
          out = mx + __logf(eo + en);
          wa = eo / (eo + en);
          wb = en / (eo + en) * inv_l;
        }
        *lp = out;
      }
      sm.wa[q] = wa;
      sm.wb[q] = wb;
      if (q == 0 && tile_ovf) P.fix_list[atomicAdd(P.fix_count, 1)] = tile;
    }
    named_bar_sync(3, kSoftmax);
    if (!tile_ovf) {  // flagged tiles are written by the exact fix-up pass
      uint32_t o[32];
      tmem_ld32(tmem + lb + kColO + col0, o);
      tmem_ld_wait();
#pragma unroll 8
      for (int i = 0; i < 32; ++i) {
        const int q = col0 + i;
        float val = __uint_as_float(o[i]) * sm.wb[q];
        if (!P.first) val += sm.wa[q] * oacc_pre[i];
        if (P.last)
          P.o[obase + (size_t)q * qstride] = __float2bfloat16_rn(val);
        else
          P.o_acc[obase + (size_t)q * qstride] = val;
      }
    }
    tc_fence_before();
    if (threadIdx.x == 128) sm.ovf = 0;
    named_bar_sync(3, kSoftmax);  // m / wa / wb / lsum / ovf are reused by the next tile
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ Params P, const __grid_constant__ CUtensorMap tmq,
                    const __grid_constant__ CUtensorMap tmk,
                    const __grid_constant__ CUtensorMap tmv,
                    const __grid_constant__ CUtensorMap tmkp,
                    const __grid_constant__ CUtensorMap tmvp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // dynamic shared memory starts 1024-aligned (no static __shared__ in this kernel);
  // using it directly keeps LDS/STS (not generic) addressing for every Smem field
  if ((smem_u32(smem_raw) & 1023u) != 0u) __trap();
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int warp = warp_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kKSt; ++s) {
      mbar_init(smem_u32(&sm.kfull[s]), 1);
      mbar_init(smem_u32(&sm.kempty[s]), 1);
    }
    for (int s = 0; s < kVSt; ++s) {
      mbar_init(smem_u32(&sm.vfull[s]), 1);
      mbar_init(smem_u32(&sm.vempty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&sm.sfull[b]), 2);
      mbar_init(smem_u32(&sm.sfree[b]), 128);  // buffer b belongs to softmax warpgroup b
      mbar_init(smem_u32(&sm.pfull[b]), 128);
      mbar_init(smem_u32(&sm.obar[b]), 1);
    }
    mbar_init(smem_u32(&sm.qfull), 1);
    mbar_init(smem_u32(&sm.qempty), 1);
    mbar_init(smem_u32(&sm.mready), 128);
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&sm.gqfull[i]), 1);
      mbar_init(smem_u32(&sm.gqempty[i]), 1);
    }
    for (int i = 0; i < kVM; ++i) {
      mbar_init(smem_u32(&sm.vmfull[i]), 1);
      mbar_init(smem_u32(&sm.vmfree[i]), 1);
    }
    sm.ovf = 0;
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(smem_u32(&sm.tmem_base), 256);
  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tmq);
    tma_prefetch_desc(&tmk);
    tma_prefetch_desc(&tmv);
    if (P.packed) {
      tma_prefetch_desc(&tmkp);
      tma_prefetch_desc(&tmvp);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
    if (warp == 0) {
      producer_k(sm, P, &tmq, &tmk, &tmkp);
    } else if (warp == 2) {
      producer_v(sm, P, &tmv, &tmvp);
    } else if (warp == 1) {
      mma_issuer(sm, P, tmem);  // whole warp: uniform control flow, one elected lane issues
    } else {
      k_gatherer(sm, P);
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;" ::: "memory");
    softmax_epilogue(sm, P, tmem);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 256);
}

// ------------------------------------------------------------------ exact fix-up
// Tiles whose scores exceeded the first-chunk stabiliser by > 2^64 are redone
// here with an exact two-pass softmax on CUDA cores (one warp per query, lane =
// 4 head dims).  Never taken on realistic inputs; it keeps the kernel correct
// on adversarial ones.
template <typename F>
__device__ __forceinline__ void for_each_key(const Params& P, int h, int g, int i, F&& fn) {
  const VSPlan& pl = P.plan;
  const int W = pl.W;
  if (pl.bptr) {  // block-CSR mode (W = 1)
    const int64_t rb = pl.bptr[(int64_t)h * (pl.nb + 1) + g];
    const int64_t re = pl.bptr[(int64_t)h * (pl.nb + 1) + g + 1];
    for (int64_t x = rb; x < re; ++x) {
      const int kb = pl.bidx[x];
      const int lim = (kb == g) ? i : 63;
      for (int kk = 0; kk <= lim; ++kk) fn(kb * 64 + kk);
    }
    return;
  }
  const int ns = pl.s_cnt[h];
  const int32_t* offs = pl.s_off + (int64_t)h * pl.s_stride;
  for (int x = 0; x < ns; ++x) {
    const int o = offs[x];
    if (o > g) break;
    if ((o % W) != P.t) continue;
    const int lb = (g - o - P.s) / W;
    const int lim = (o == 0) ? i : 63;  // diagonal block: causal
    for (int kk = 0; kk <= lim; ++kk) fn(lb * 64 + kk);
  }
  const int32_t* vc = pl.vcol + (int64_t)h * pl.S;
  const int vb = pl.vptr[h * (W + 1) + P.s], ve = pl.vptr[h * (W + 1) + P.s + 1];
  for (int e = vb; e < ve; ++e) {
    const int m = vc[e];
    const int blk = m >> 6;
    if (blk >= g) break;
    if (plan_has_slash(pl, h, g - blk)) continue;
    fn(((blk - P.s) / W) * 64 + (m & 63));
  }
}

__global__ void __launch_bounds__(256) attn_fwd_fixup(const __grid_constant__ Params P,
                                                      const __nv_bfloat16* __restrict__ q) {
  const int n = *P.fix_count;
  const int lane = lane_id(), w = warp_id();
  const VSPlan& pl = P.plan;
  const int grp = pl.Hq / pl.Hkv;
  const int64_t S_loc = (int64_t)P.nloc * 64;
  for (int f = blockIdx.x; f < n; f += gridDim.x) {
    int h, j;
    tile_coords(P, P.fix_list[f], h, j);
    const int g = j * pl.W + P.r, gkv = h / grp;
    for (int i = w; i < 64; i += 8) {
      const int64_t tok = (int64_t)j * 64 + i;
      float qv[4];
      const __nv_bfloat16* qr = q + ((size_t)tok * pl.Hq + h) * 128 + lane * 4;
#pragma unroll
      for (int u = 0; u < 4; ++u) qv[u] = __bfloat162float(qr[u]);
      auto score = [&](int row) {
        const __nv_bfloat16* kr = P.k + ((size_t)row * pl.Hkv + gkv) * 128 + lane * 4;
        float sdot = 0.f;
#pragma unroll
        for (int u = 0; u < 4; ++u) sdot += qv[u] * __bfloat162float(kr[u]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
        return sdot * P.scale_log2;
      };
      float mx = -INFINITY;
      for_each_key(P, h, g, i, [&](int row) { mx = fmaxf(mx, score(row)); });
      float l = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
      for_each_key(P, h, g, i, [&](int row) {
        const float p = exp2f(score(row) - mx);
        l += p;
        const __nv_bfloat16* vr = P.v + ((size_t)row * pl.Hkv + gkv) * 128 + lane * 4;
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] += p * __bfloat162float(vr[u]);
      });
      const float lse_new = l > 0.f ? (mx + log2f(l)) * 0.69314718055994531f : -INFINITY;
      float* lp = P.lse + (int64_t)h * S_loc + tok;
      const float lse_old = P.first ? -INFINITY : *lp;
      const float m2 = fmaxf(lse_old, lse_new);
      float wa = 0.f, wb = 0.f, out = -INFINITY;
      if (m2 > -INFINITY) {
        const float eo = lse_old == -INFINITY ? 0.f : expf(lse_old - m2);
        const float en = lse_new == -INFINITY ? 0.f : expf(lse_new - m2);
        out = m2 + logf(eo + en);
        wa = eo / (eo + en);
        wb = l > 0.f ? en / (eo + en) / l : 0.f;
      }
      const size_t base = ((size_t)tok * pl.Hq + h) * 128 + lane * 4;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float val = acc[u] * wb;
        if (!P.first) val += wa * P.o_acc[base + u];
        if (P.last) P.o[base + u] = __float2bfloat16_rn(val);
        else P.o_acc[base + u] = val;
      }
      __syncwarp();
      if (lane == 0) *lp = out;
    }
  }
}

// Packed vertical rows of origin s (VSPlan.kp / vp): row i of q head h = the held
// chunk's K / V row of the head's i-th column of that origin; rows up to the next
// multiple of 128 zero-filled.  Heads with more than pcap columns are skipped (their
// bar chunks use the gather path).  One thread per 16 B of a row's K or V.
__global__ void pack_bars_kernel(VSPlan pl, int s, const __nv_bfloat16* __restrict__ k,
                                 const __nv_bfloat16* __restrict__ v) {
  const int h = blockIdx.y;
  const int W = pl.W, grp = pl.Hq / pl.Hkv;
  const int vb = pl.vptr[h * (W + 1) + s], ve = pl.vptr[h * (W + 1) + s + 1];
  const int n = ve - vb;
  if (n > pl.pcap) return;
  const int nr = (n + 127) / 128 * 128;
  const int32_t* vc = pl.vcol + (int64_t)h * pl.S + vb;
  uint4* kp = static_cast<uint4*>(pl.kp);
  uint4* vp = static_cast<uint4*>(pl.vp);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nr * 32; t += gridDim.x * blockDim.x) {
    const int i = t >> 5, part = t & 31, c16 = part & 15;
    uint4 val = make_uint4(0u, 0u, 0u, 0u);
    if (i < n) {
      const int m = vc[i];
      const int64_t lrow = (int64_t)(((m >> 6) - s) / W) * 64 + (m & 63);
      const __nv_bfloat16* src = (part < 16 ? k : v) + (lrow * pl.Hkv + h / grp) * 128;
      val = reinterpret_cast<const uint4*>(src)[c16];
    }
    (part < 16 ? kp : vp)[((int64_t)i * pl.Hq + h) * 16 + c16] = val;
  }
}

}  // namespace fwd

size_t fwd_smem_bytes() { return sizeof(fwd::Smem); }  // the dynamic base is 1024-aligned

mt_status attn_fwd_step(const VSPlan& plan, int r, int s, int nloc, const void* q,
                        const void* k, const void* v, void* o, float* o_acc, float* lse,
                        int first, int last, int num_sms, cudaStream_t st) {
  using namespace fwd;
  Params P{};
  P.plan = plan;
  P.r = r;
  P.s = s;
  P.t = ((r - s) % plan.W + plan.W) % plan.W;
  P.nloc = nloc;
  P.n_tiles = plan.Hq * nloc;
  P.first = first;
  P.last = last;
  P.scale_log2 = 1.4426950408889634f / sqrtf(128.f);
  P.k = static_cast<const __nv_bfloat16*>(k);
  P.v = static_cast<const __nv_bfloat16*>(v);
  P.o = static_cast<__nv_bfloat16*>(o);
  P.o_acc = o_acc;
  P.lse = lse;
  P.fix_count = plan.scratch;
  P.tile_counter = plan.scratch + 1;
  static const int ord = getenv("MT_FWD_ORDER") ? atoi(getenv("MT_FWD_ORDER")) : 1;
  P.order = ord;
  P.fix_list = plan.scratch + 16;
  static const int pack = getenv("MT_FWD_PACK") ? atoi(getenv("MT_FWD_PACK")) : 1;
  P.packed = pack && plan.kp && plan.pcap > 0;
  const uint64_t S_loc = (uint64_t)nloc * 64;
  CUtensorMap tmq, tmk, tmv, tmkp, tmvp;
  if (make_tmap_bf16_3d(&tmq, q, 128, plan.Hq, S_loc, 64, 1, 64) ||
      make_tmap_bf16_3d(&tmk, k, 128, plan.Hkv, S_loc, 64, 1, 64) ||
      make_tmap_bf16_3d(&tmv, v, 128, plan.Hkv, S_loc, 64, 1, 64))
    return fail(MT_ECUDA, "cuTensorMapEncodeTiled failed");
  tmkp = tmk;
  tmvp = tmv;
  if (P.packed) {
    if (make_tmap_bf16_3d(&tmkp, plan.kp, 128, plan.Hq, plan.pcap, 64, 1, 64) ||
        make_tmap_bf16_3d(&tmvp, plan.vp, 128, plan.Hq, plan.pcap, 64, 1, 64))
      return fail(MT_ECUDA, "cuTensorMapEncodeTiled (packed) failed");
    pack_bars_kernel<<<dim3(16, plan.Hq), 256, 0, st>>>(plan, s, static_cast<const __nv_bfloat16*>(k),
                                                        static_cast<const __nv_bfloat16*>(v));
    MT_TRY(check_launch("pack_bars_kernel"));
  }
  const size_t smem = fwd_smem_bytes();
  // set on every launch: the attribute applies to the current device only
  if (cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return fail(MT_ECUDA, "cudaFuncSetAttribute(attn_fwd) failed (smem %zu)", smem);
  const int grid = P.n_tiles < num_sms ? P.n_tiles : num_sms;
  cudaMemsetAsync(P.fix_count, 0, 2 * sizeof(int), st);  // fix-up count, tile counter
  if (grid > 0) attn_fwd_kernel<<<grid, kThreads, smem, st>>>(P, tmq, tmk, tmv, tmkp, tmvp);
  MT_TRY(check_launch("attn_fwd_kernel"));
  attn_fwd_fixup<<<num_sms, 256, 0, st>>>(P, static_cast<const __nv_bfloat16*>(q));
  return check_launch("attn_fwd_fixup");
}

}  // namespace mt

extern "C" mt_status mt_debug_fwd_timeline(int64_t* out) {
  if (!out) return mt::fail(MT_ESHAPE, "NULL output");
  if (cudaMemcpyFromSymbol(out, mt::g_mt_tl, sizeof(mt::g_mt_tl)) != cudaSuccess)
    return mt::fail(MT_ECUDA, "cudaMemcpyFromSymbol(timeline) failed");
  return MT_OK;
}
