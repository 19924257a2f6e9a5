// attn_fwd.cu — block-sparse vertical-slash attention forward for sm_100a, one
// ring step (Alg. 2 "block_bar_sparse_attention_forward" P:878 then
// "merge_out_and_lse" P:879; with W = 1 the single step is Alg. 1's
// "sparse(softmax(QK^T/sqrt d)V, i_vs)").
//
// Row-wise tiles over HEAD PAIRS (round 2):
//   tile  = one 64-query block g x two q heads (h0, h1) of one kv group: 128 query
//           rows = the MMA's M (rows 0-63 head h0, 64-127 head h1), which share every
//           K/V tile they load;
//   chunk = 128 keys from the union of the two heads' key sets of the block: two 64-key
//           slash blocks of B_g^(h0) U B_g^(h1) (TMA; per head / slot liveness bits), or
//           128 packed vertical columns of ONE head (TMA; the other head's rows masked);
//   S  = [Q_h0; Q_h1] K^T    tcgen05 M=128 N=128 K=128   SMEM x SMEM  -> TMEM
//   P  = 2^(S c - m_row) in registers (thread = query row = TMEM lane), bf16 -> TMEM
//        over S (A operand of the next MMA)
//   O += P V                 tcgen05 M=128 N=128 K=128   TMEM x SMEM  -> TMEM
// Round 1's transposed tiles (one head, N = 64 queries) read K and V as 32 KB A operands
// per chunk for 64 queries, and P^T through SMEM: 176 KB of SMEM traffic per chunk, and
// its N = 64 MMAs are SMEM-bound (51.6 instead of 32 cycles, profiles/r02_mma_bench.txt).
// Here a chunk moves 64 KB (TMA) + 64 KB (S: Q, K) + 32 KB (O: V) for up to 128 query rows
// at the MMAs' 64-cycle floor.  The price is the union: a key block selected for only one
// of the two heads computes dead rows (per chunk, ~0.66 of the rows are live on the C4
// index: offsets shared by heads of a kv group).
// The row stabiliser m_row is the exact max of the row's live scores in the tile's chunk 0
// (which holds each head's first key block); each thread owns its row, so row max and row
// sum need no cross-thread reduction.  A later score above m_row + 64 (log2 units), or a
// live score in a row with none in chunk 0, sends the tile to the exact two-pass
// attn_fwd_fixup kernel.
//
// Warp roles (384 threads, 1 CTA / SM, persistent; setmaxnreg moves registers
// from warpgroup 0 to the softmax warpgroups):
//   warp 0       producer (chunk stream from the VSPlan, TMA / cp.async)
//   warp 1       MMA issuer (one lane)
//   warp 2       V producer (decoupled from K through a metadata ring)
//   warp 3       K gatherer for bar chunks of heads above the packed-row capacity
//   warps 4..11  two softmax warpgroups; warpgroup b takes the tile's chunks
//                k = b (mod 2); warp w covers TMEM lanes (query rows) 32*(w%4)..
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
constexpr int kKSt = MT_FWD_KST, kVSt = MT_FWD_VST;
#ifndef MT_FWD_POLY
#define MT_FWD_POLY 0  // 1: a quarter of the all-live exponentials by the FMA-pipe cubic (A/B)
#endif
constexpr int kThreads = 384;  // warpgroup 0: producers, MMA, gatherer; warpgroups 1-2: softmax
constexpr int kSoftmax = 256;
constexpr uint32_t kTileKV = 128 * 128 * 2;  // 32 KB
constexpr uint32_t kTileQ2 = 128 * 128 * 2;  // 32 KB: the head pair's 128 query rows
constexpr float kOverflow = 64.f;            // log2 headroom above the stabiliser
constexpr float kUnderflow = -100.f;         // a row whose every live score is this far below
                                             // its stabiliser (log2) goes to the exact fix-up

// kBarP: a bar chunk of 128 consecutive packed rows of one head (TMA), live rows in `mask`
enum : int { kBlk = 0, kBar = 1, kEnd = 2, kDone = 3, kBarP = 4 };

struct alignas(16) ChunkMeta {  // per K slot: what the MMA / softmax need
  int kind;
  int n;           // kBar: live rows
  uint32_t flags;  // kBlk: bit0/1 slot0 live for head 0/1, bit2/3 slot1 live for head 0/1,
                   //       bit4 slot0 diagonal, bit5 slot1 diagonal
                   // kBar / kBarP: bit0 = the head (0/1) whose rows are live
  int tile;        // kEnd: the tile it closes
  uint32_t mask[4];  // kBarP / kBar: live keys (not covered by a selected slash, inside the prefix)
};

struct alignas(16) VMeta {  // per data chunk: what the producers need to stage K/V
  int kind;
  int n;
  int lb0, lb1;    // kBlk: local key blocks; kBarP: lb0 = first packed row
  int gkv;         // kBlk / kBar: kv head; kBarP: the q head (packed rows are per q head)
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
  uint32_t mask[4];
};

struct Smem {
  uint8_t k[kKSt][kTileKV];
  uint8_t v[kVSt][kTileKV];
  uint8_t q[kTileQ2];   // [d-atom c][128 rows: head 0's 64 queries, head 1's][128 B]
  ChunkMeta meta[kKSt];
  VMeta vmeta[kVM];
  SMeta smeta[3];
  alignas(16) float m[128];         // row stabilisers of the tile (log2 domain)
  alignas(16) float lsum[2][128];   // per warpgroup: row sums of its chunks
  alignas(16) float emx[2][128];    // per warpgroup: largest live exponent of the row
  int stage_rows[192];
  // bar chunks: K-gather requests from the K producer (warp 0) to the gatherer (warp 3)
  struct alignas(16) GatherReq {
    int rows[128];
    int ks, gkv, pad[2];
  } greq[2];
  uint32_t sbits[2][kSbitsWords];  // the tile heads' slash bitmaps (producer warp only)
  int ovf[2];  // per tile parity: some row of the tile overflowed its stabiliser
  uint64_t kfull[kKSt], kempty[kKSt], vfull[kVSt], vempty[kVSt];
  uint64_t sfull[3], sfree[3], pfull[3], obar[2];
  uint64_t edone;  // the softmax warps finished a tile's epilogue (obar's phase is theirs)
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
  int* fix_count;  // tiles flagged for the exact fix-up pass
  int stabfix;     // 1: chunk-0 fallback stabiliser + underflow check (MT_FWD_STABFIX=0: off, A/B)
  int dbg;         // profiling knock-outs (MT_FWD_DBG): bit0 skip the softmax math (wrong results)
  int* fix_list;
  int* tile_counter;  // dynamic tile scheduler (zeroed before the launch)
  int order;          // tile order (MT_FWD_ORDER): 1 head-major (default; L2 reuse of K/V), 0 query-block-major
  int packed;         // bar chunks from the packed rows (plan.kp / vp) by TMA (MT_FWD_PACK, default 1)
  int ppg;            // tiles per kv group and query block: ceil((Hq / Hkv) / 2) head pairs,
                      // or Hq / Hkv single heads in block-CSR mode
  int single;         // 1: one head per tile (block-CSR mode), rows 64-127 dead
};

// TMEM: O [0, 128), three S / P buffers at [128 + 128 b, 256 + 128 b): chunk k of a tile
// uses buffer k % 3 and softmax warpgroup k % 2, so S(k + 1), S(k + 2) run on the tensor
// core while warpgroup k % 2 works on chunk k.
constexpr int kNB = 3;
constexpr uint32_t kColO = 0, kColS = 128;

// per-buffer event counters packed in one word (10 bits each: only parities are used)
__device__ __forceinline__ uint32_t cnt_get(uint32_t c, uint32_t b) { return (c >> (10 * b)) & 1023u; }
__device__ __forceinline__ uint32_t cnt_inc(uint32_t c, uint32_t b) {
  return (c & ~(1023u << (10 * b))) | (((cnt_get(c, b) + 1u) & 1023u) << (10 * b));
}
// buffer of softmax warpgroup w's next event when a tile has closed after n chunks
__device__ __forceinline__ uint32_t end_buffer(uint32_t n, uint32_t w) {
  return (n + ((n & 1u) != w ? 1u : 0u)) % kNB;
}
// events a tile of n chunks puts on buffer b: its chunks k = b (mod 3) and END(s)
__device__ __forceinline__ uint32_t tile_events(uint32_t n, uint32_t b) {
  const uint32_t chunks = n > b ? (n - 1u - b) / kNB + 1u : 0u;
  return chunks + (end_buffer(n, 0) == b ? 1u : 0u) + (end_buffer(n, 1) == b ? 1u : 0u);
}

// tile -> (first head h0, second head h1 or -1, local query block j)
__device__ __forceinline__ void tile_coords(const Params& P, int tile, int& h0, int& h1, int& j) {
  const int grp = P.plan.Hq / P.plan.Hkv;
  const int npairs = P.plan.Hkv * P.ppg;
  int pi;
  if (P.order) {  // head-major: resident tiles = consecutive query blocks of one head pair
    pi = tile / P.nloc;
    j = P.nloc - 1 - tile % P.nloc;
  } else {
    j = P.nloc - 1 - tile / npairs;  // late query blocks (most keys) first
    pi = tile % npairs;
  }
  const int gkv = pi / P.ppg;
  if (P.single) {
    h0 = gkv * grp + pi % P.ppg;
    h1 = -1;
    return;
  }
  h0 = gkv * grp + 2 * (pi % P.ppg);
  h1 = h0 + 1 < (gkv + 1) * grp ? h0 + 1 : -1;
}

// ------------------------------------------------------------------ producers
// Warp 0 builds the chunk stream and issues K (slot frees after the S MMA); warp 2
// issues V (slot frees after the O MMA).  They are decoupled by a 4-entry ring of V
// metadata, so a late V slot never delays the next K.  K slots (and the per-chunk meta
// the MMA reads) are indexed by every chunk including END markers; V slots only by
// data chunks.
template <int L>  // sequence layout (plan.cuh), fixed per launch
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
    int h0, h1, j;
    tile_coords(P, tile, h0, h1, j);
    const int g = l2g_<L>(pl, P.r, j);  // global query block (plan.cuh layouts)
    const int gkv = h0 / grp;
    if (!first_tile) {
      mbar_wait(smem_u32(&sm.qempty), qe_phase);
      qe_phase ^= 1;
    }
    first_tile = false;
    if (lane == 0) {  // the pair's queries: rows 0-63 head h0, 64-127 head h1 (h0 again if none)
      const uint32_t bar = smem_u32(&sm.qfull);
      mbar_expect_tx(bar, kTileQ2);
      for (int x = 0; x < 2; ++x)
        for (int cc = 0; cc < 2; ++cc)
          tma_load_3d(smem_u32(sm.q + cc * 16384 + x * 8192), tmq, bar, cc * 64,
                      (x && h1 >= 0) ? h1 : h0, j * 64);
    }
    // the heads' slash bitmaps in SMEM (membership tests of the union walk and of bars)
    const bool bits_smem = !pl.bptr && pl.bits_words <= kSbitsWords;
    if (bits_smem) {
      for (int x = 0; x < 2; ++x) {
        const int hx = x ? h1 : h0;
        if (hx < 0) continue;
        const uint32_t* gb = pl.s_bits + (int64_t)hx * pl.bits_words;
        for (int w = lane; w < pl.bits_words; w += 32) sm.sbits[x][w] = gb[w];
      }
      __syncwarp();
    }
    auto has = [&](int x, int o) {  // offset o selected for head x of the pair
      const int hx = x ? h1 : h0;
      if (hx < 0 || o < 0 || pl.bptr) return false;
      return bits_smem ? ((sm.sbits[x][o >> 5] >> (o & 31)) & 1u) != 0u : plan_has_slash(pl, hx, o);
    };
    // ---- slash blocks of residue t: the union of both heads' offsets o <= g, two per
    // chunk.  Chunk 0 holds each head's FIRST block (the row stabilisers come from it).
    {
      // live0 / live1: per slot, bit x = head x of the pair attends that key block
      auto emit_pair = [&](int o0, int o1, uint32_t live0, uint32_t live1) {  // o1 < 0: slot empty
        const int lb0 = g2l_<L>(pl, g - o0);
        const int lb1 = o1 >= 0 ? g2l_<L>(pl, g - o1) : lb0;
        uint32_t flags = live0 & 3u;
        if (o1 >= 0) flags |= (live1 & 3u) << 2;
        if (o0 == 0) flags |= 16u;
        if (o1 == 0) flags |= 32u;
#ifdef MT_TL_PROD
        if (lane == 0) MT_TL(4, dk);  // producer reached the chunk (before the vmeta / K waits)
#endif
        VMeta& vm = vmacquire();
#ifdef MT_TL_PROD
        if (lane == 0) MT_TL(5, dk);  // vmeta slot acquired
#endif
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
          MT_TL(0, dk);
          for (int cc = 0; cc < 2; ++cc)
            for (int x = 0; x < 2; ++x)
              tma_load_3d(smem_u32(sm.k[ks] + cc * 16384 + x * 8192), tmk, kb, cc * 64, gkv,
                          (x ? lb1 : lb0) * 64);
        }
        vmrelease();
        ++c;
      };
      auto vs_live = [&](int o) { return (has(0, o) ? 1u : 0u) | (has(1, o) ? 2u : 0u); };
      if (pl.bptr) {
        // block-CSR mode (W = 1, one head per tile): the row's key blocks, last first
        // (the diagonal, when present, in chunk 0)
        const int64_t rb = pl.bptr[(int64_t)h0 * (pl.nb + 1) + g];
        const int64_t re = pl.bptr[(int64_t)h0 * (pl.nb + 1) + g + 1];
        int pend = -1;
        for (int64_t top = re - 1; top >= rb; top -= 32) {
          const int64_t i = top - lane;
          const int o = i >= rb ? g - pl.bidx[i] : 0;
          uint32_t bal = __ballot_sync(0xffffffffu, i >= rb);
          while (bal) {
            const int l = __ffs(bal) - 1;
            bal &= bal - 1;
            const int ov = __shfl_sync(0xffffffffu, o, l);
            if (pend < 0) {
              pend = ov;
            } else {
              emit_pair(pend, ov, 1u, 1u);
              pend = -1;
            }
          }
        }
        if (pend >= 0) emit_pair(pend, -1, 1u, 0u);
      }
      // the origin's key blocks <= g, nearest first: point m is local key block
      // npts-1-m, offset o(m) = g - l2g(s, npts-1-m) ascending (block-striped: the lattice
      // o = t + mW); tested 32 at a time against both bitmaps
      const int npts = pl.bptr ? 0 : count_le_<L>(pl, P.s, g);
      auto o_of = [&](int m) {
        if constexpr (L == 0) return P.t + m * W;  // the residue lattice
        else return g - l2g_<L>(pl, P.s, npts - 1 - m);
      };
      int f0 = -1, f1 = -1;  // each head's first offset
      for (int m0 = 0; m0 < npts && (f0 < 0 || (h1 >= 0 && f1 < 0)); m0 += 32) {
        const int o = o_of(m0 + lane);
        const bool in = m0 + lane < npts;
        const uint32_t ba = __ballot_sync(0xffffffffu, in && has(0, o));
        const uint32_t bb = __ballot_sync(0xffffffffu, in && has(1, o));
        if (f0 < 0 && ba) f0 = o_of(m0 + __ffs(ba) - 1);
        if (f1 < 0 && bb) f1 = o_of(m0 + __ffs(bb) - 1);
      }
      int skip0 = -1, skip1 = -1;
      if (f0 >= 0 && f1 >= 0 && f0 != f1) {
        emit_pair(min(f0, f1), max(f0, f1), vs_live(min(f0, f1)), vs_live(max(f0, f1)));
        skip0 = f0;
        skip1 = f1;
      }
      int pending = -1;
      for (int m0 = 0; m0 < npts; m0 += 32) {
        const int o = o_of(m0 + lane);
        const bool in = m0 + lane < npts && o != skip0 && o != skip1;
        uint32_t bal = __ballot_sync(0xffffffffu, in && (has(0, o) || has(1, o)));
        while (bal) {
          const int l = __ffs(bal) - 1;
          bal &= bal - 1;
          const int ov = o_of(m0 + l);
          if (pending < 0) {
            pending = ov;
          } else {
            emit_pair(pending, ov, vs_live(pending), vs_live(ov));
            pending = -1;
          }
        }
      }
      if (pending >= 0) emit_pair(pending, -1, vs_live(pending), 0u);
    }
    // ---- bars of origin s, per head: block < g, offset not a selected slash of that
    // head; 128 per chunk, the other head's rows masked
    for (int x = 0; x < 2; ++x) {
      const int h = x ? h1 : h0;
      if (h < 0) continue;
      const int32_t* vc = pl.vcol + (int64_t)h * pl.S;
      const int vb = pl.vptr[h * (W + 1) + P.s];
      const int ve = pl.vptr[h * (W + 1) + P.s + 1];
      int nst = 0;
      auto covered = [&](int o) { return has(x, o); };
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
              m.flags = (uint32_t)x;
#pragma unroll
              for (int w = 0; w < 4; ++w) m.mask[w] = msk[w];
              const uint32_t kb = smem_u32(&sm.kfull[ks]);
              mbar_expect_tx(kb, kTileKV);
              for (int cc = 0; cc < 2; ++cc)
                for (int xx = 0; xx < 2; ++xx)
                  tma_load_3d(smem_u32(sm.k[ks] + cc * 16384 + xx * 8192), tmkp, kb, cc * 64, h,
                              i0 + 64 * xx);
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
          for (int xx = lane; xx < 128; xx += 32) vm.rows[xx] = sm.stage_rows[xx < n ? xx : 0];
          if (lane == 0) {
            vm.kind = kBar;
            vm.n = n;
            vm.gkv = gkv;
            sm.meta[ks].kind = kBar;
            sm.meta[ks].n = n;
            sm.meta[ks].flags = (uint32_t)x;
          }
          __syncwarp();
          {  // hand the K gather to warp 3 (it arrives on kfull[ks] when the rows land)
            const uint32_t gi = ng & 1;
            mbar_wait(smem_u32(&sm.gqempty[gi]), ((ng >> 1) & 1) ^ 1);
            for (int xx = lane; xx < 128; xx += 32) sm.greq[gi].rows[xx] = vm.rows[xx];
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
              lrow = g2l_<L>(pl, blk) * 64 + (m & 63);
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
// Chunk k of a tile goes to S/P buffer k & 1 (softmax warpgroup k & 1).  O(k) is issued
// after S(k+1) and before S(k+2): S(k+2) overwrites the buffer O(k) reads P(k) from, and
// tcgen05 MMAs execute in issue order.  END is published to both warpgroups after the
// tile's last O, with one commit (obar) they wait on before the epilogue.
__device__ void mma_issuer(Smem& sm, const Params& P, uint32_t tmem) {
  const bool leader = elect_one();
  const uint32_t id_s = make_idesc_bf16(128, 128, false, false);  // S = Q K^T
  const uint32_t id_o = make_idesc_bf16(128, 128, false, true);   // O += P V (V MN-major)
  const uint64_t dq0 = make_sdesc(smem_u32(sm.q), 16, 1024);
  const uint64_t dk0 = make_sdesc(smem_u32(sm.k[0]), 16, 1024);
  const uint64_t dv0 = make_sdesc(smem_u32(sm.v[0]), 16384, 1024);
  uint32_t c = 0, dc = 0, oc = 0, qf_phase = 0;  // K slots, data chunks S-issued, O-issued
  uint32_t nt = 0;                               // tiles closed (obar commits)
  bool o_started = false;
  uint32_t pcnt = 0;  // per buffer: P publications consumed (pfull phases)
  uint32_t ecnt = 0;  // per buffer: events published (sfree phases)
  // smeta[b] may be rewritten once the warpgroup that read the previous event took its copy
  auto wait_sfree = [&](uint32_t b) {
    MT_CRUMB(0, 40 + (int)b);
    const uint32_t n = cnt_get(ecnt, b);
    if (n > 0) mbar_wait(smem_u32(&sm.sfree[b]), (n - 1) & 1);
    ecnt = cnt_inc(ecnt, b);
  };
  int kind_ring[4] = {0, 0, 0, 0};
  uint32_t buf_ring[4] = {0, 0, 0, 0};
  // O += P V for the oldest data chunk not yet accumulated (oc)
  auto issue_o = [&]() {
    const uint32_t b = buf_ring[oc & 3], vs = oc % kVSt;
    MT_CRUMB(0, 20 + (int)b);
    MT_CRUMB(1, (int)oc);
    mbar_wait(smem_u32(&sm.vfull[vs]), (oc / kVSt) & 1);
    MT_CRUMB(0, 30 + (int)b);
    if (leader) MT_TL(7, oc);
    if (kind_ring[oc & 3] == kBar) fence_proxy_async_smem();
    mbar_wait(smem_u32(&sm.pfull[b]), cnt_get(pcnt, b) & 1);
    pcnt = cnt_inc(pcnt, b);
    tc_fence_after();
    const uint64_t dv = sdesc_add(dv0, vs * kTileKV);
    const uint32_t pb = tmem + kColS + 128 * b;  // P: keys 2c, 2c+1 packed in column c
    if (leader) {
#pragma unroll
      for (int kk = 0; kk < 128; kk += 16)
        mma_ts(tmem + kColO, pb + kk / 2, sdesc_add(dv, kk * 128), id_o,
               (o_started || kk > 0) ? 1u : 0u);
      mma_commit(smem_u32(&sm.vempty[vs]));
      MT_TL(3, oc);
    }
    o_started = true;
    ++oc;
  };
  // END / DONE to both softmax warpgroups, each on the buffer its next chunk would use
  auto publish = [&](int kind, int tile, uint32_t n) {
    for (uint32_t w = 0; w < 2; ++w) {
      const uint32_t b = end_buffer(n, w);
      wait_sfree(b);
      if (leader) {
        sm.smeta[b].kind = kind;
        sm.smeta[b].tile = tile;
        sm.smeta[b].n = (int)n;  // lets both warpgroups account every buffer's events
        mbar_arrive(smem_u32(&sm.sfull[b]));
        mbar_arrive(smem_u32(&sm.sfull[b]));
      }
    }
  };
  for (;;) {
    {  // the next chunk tells whether another tile follows
      const uint32_t ks = c % kKSt;
      mbar_wait(smem_u32(&sm.kfull[ks]), (c / kKSt) & 1);
      if (sm.meta[ks].kind == kDone) {
        publish(kDone, -1, 0);
        break;
      }
    }
    MT_CRUMB(0, 10);
    mbar_wait(smem_u32(&sm.qfull), qf_phase);
    MT_CRUMB(0, 11);
    qf_phase ^= 1;
    tc_fence_after();
    o_started = false;
    uint32_t k = 0;  // data chunk index inside the tile
    for (;;) {
      const uint32_t ks = c % kKSt;
      mbar_wait(smem_u32(&sm.kfull[ks]), (c / kKSt) & 1);
      const int kind = sm.meta[ks].kind;
      const int end_tile = sm.meta[ks].tile;  // read before the slot is released
      if (kind == kBar) fence_proxy_async_smem();
      tc_fence_after();
      ++c;
      if (kind == kEnd) {
        if (leader) {
          mma_commit(smem_u32(&sm.qempty));  // every S of the tile issued before
          mbar_arrive(smem_u32(&sm.kempty[ks]));
        }
        while (oc < dc) issue_o();
        // obar is waited on by parity: the previous tile's epilogue must have passed its
        // wait before this tile's commit (a tile without chunks would otherwise complete
        // two phases while a warpgroup still waits for the first)
        if (nt > 0) mbar_wait(smem_u32(&sm.edone), (nt - 1) & 1);
        if (leader) mma_commit(smem_u32(&sm.obar[0]));  // the tile's O complete
        ++nt;
        publish(kEnd, end_tile, k);
        break;
      }
      if (leader) MT_TL(6, dc);
      if (dc - oc >= (uint32_t)kNB) issue_o();  // O(k-3) before S(k) overwrites its P buffer
      const uint32_t b = k % kNB;
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
        const uint32_t ts = tmem + kColS + 128 * b;
#pragma unroll
        for (int kk = 0; kk < 128; kk += 16) {
          const uint32_t off = (kk >> 6) * 16384 + (kk & 63) * 2;
          mma_ss(ts, sdesc_add(dq0, off), sdesc_add(dk, off), id_s, kk > 0);
        }
        mma_commit(smem_u32(&sm.sfull[b]));  // 2 of 2: S ready
        mma_commit(smem_u32(&sm.kempty[ks]));
        MT_TL(2, dc);
      }
      kind_ring[dc & 3] = kind;
      buf_ring[dc & 3] = b;
      ++dc;
      ++k;
    }
  }
}

// ------------------------------------------------------------------ softmax + epilogue
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Live keys (bit c = key 32 cg + c) of this thread's query row in one 32-key group.
__device__ __forceinline__ uint32_t live_bits(const SMeta& cm, int x, int i, int cg) {
  if (cm.kind == kBlk) {
    const int slot = cg >> 1;
    const bool live = (cm.flags >> (2 * slot + x)) & 1u;
    if (!live) return 0u;
    if (!((cm.flags >> (4 + slot)) & 1u)) return ~0u;
    // diagonal block: query i sees keys kk <= i (kk = 32 (cg & 1) + c)
    const int lim = i - 32 * (cg & 1);  // keys c <= lim
    return lim < 0 ? 0u : (lim >= 31 ? ~0u : ((2u << lim) - 1u));
  }
  if ((int)(cm.flags & 1u) != x) return 0u;
  if (cm.kind == kBarP) return cm.mask[cg];
  const int n = cm.n - 32 * cg;  // kBar: the first n keys are live
  return n <= 0 ? 0u : (n >= 32 ? ~0u : ((1u << n) - 1u));
}

// Warpgroup wg owns S/P buffer wg and the tile's chunks k = wg (mod 2); thread = query row
// (TMEM lane) with all 128 keys of a chunk.  m_row: the exact max of the row's live scores
// in chunk 0 (computed by warpgroup 0, handed to warpgroup 1 through the mready mbarrier).
__device__ void softmax_epilogue(Smem& sm, const Params& P, uint32_t tmem) {
  const int w = warp_id();
  const int quad = w & 3, wg = (w - 4) >> 2;
  const int lane = lane_id();
  const int row = quad * 32 + lane;  // query row of the pair tile == TMEM lane
  const int x = row >> 6, qi = row & 63;
  const uint32_t lb = ((uint32_t)(quad * 32) << 16);
  const int Hq = P.plan.Hq;
  const int64_t S_loc = (int64_t)P.nloc * 64;
  const uint32_t mready = smem_u32(&sm.mready);
  const float sc = P.scale_log2;
  // base: events published on each buffer before the current tile (both warpgroups'); the
  // buffer-b event of chunk k is number base[b] + k / 3, END's follows the tile's chunks
  uint32_t base = 0, mr_phase = 0, ntile = 0;

  for (;;) {
    float m = -INFINITY, l = 0.f, tile_emax = -INFINITY;
    bool m_synced = false, ovf = false;
    int tile = -1;
    for (uint32_t k = (uint32_t)wg;; k += 2) {  // this warpgroup's chunks of the tile
      const uint32_t b = k % kNB;
      if (row == 0) MT_CRUMB(3 + wg, 1000000 + (int)k);
      // the k-th chunk index is an END when the tile closed before it: END's event number
      // on b is base[b] + (chunks of the tile on b) = base[b] + k / 3 as well
      mbar_wait(smem_u32(&sm.sfull[b]), (cnt_get(base, b) + k / kNB) & 1);
      const SMeta cm = sm.smeta[b];
      mbar_arrive(smem_u32(&sm.sfree[b]));  // the copy is taken: smeta[b] reusable
      const uint32_t Sb = tmem + lb + kColS + 128 * b;
      const uint32_t pfull = smem_u32(&sm.pfull[b]);
      if (cm.kind == kEnd || cm.kind == kDone) {
        tile = cm.kind == kEnd ? cm.tile : -1;
        const uint32_t n = (uint32_t)cm.n;
#pragma unroll
        for (uint32_t bb = 0; bb < (uint32_t)kNB; ++bb)
          base = (base & ~(1023u << (10 * bb))) | (((cnt_get(base, bb) + tile_events(n, bb)) & 1023u) << (10 * bb));
        break;
      }
#ifndef MT_TL_PROD
      if (row == 0) MT_TL(4, cm.seq);
#endif
      tc_fence_after();
      if (!m_synced) {
        if (wg == 0) {  // chunk 0: exact max of the row's live scores
          float mx = -INFINITY, mx_all = -INFINITY;
#pragma unroll 1
          for (int cg = 0; cg < 4; ++cg) {
            uint32_t sv[32];
            tmem_ld32(Sb + 32 * cg, sv);
            tmem_ld_wait();
            const uint32_t lv = live_bits(cm, x, qi, cg);
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) {
              const float v = __uint_as_float(sv[cc]) * sc;
              mx_all = fmaxf(mx_all, v);
              if ((lv >> cc) & 1u) mx = fmaxf(mx, v);
            }
          }
          // a row with no live key in chunk 0 (ring steps: its head has no slash block of
          // this origin, only bars) takes the chunk's largest score against the same kv
          // head's keys as its scale; the overflow / underflow checks keep it exact
          if (mx == -INFINITY && P.stabfix) mx = mx_all;
          sm.m[row] = mx;
          m = mx;
          mbar_arrive(mready);
        } else {
          mbar_wait(mready, mr_phase);
          m = sm.m[row];
        }
        m_synced = true;
      }
      // P = exp2(S log2e/sqrt d - m): one FFMA + one MUFU per live key; P (bf16, 2 keys
      // per column) over the S columns already read; overflow tracked as the largest
      // exponent
      float emax = -INFINITY;
      bool any_live = false;
#pragma unroll 1
      for (int cg = 0; cg < ((P.dbg & 1) ? 0 : 4); ++cg) {  // MT_FWD_DBG=1: no softmax (timing only)
        uint32_t sv[32], pk[16];
        const uint32_t lv = live_bits(cm, x, qi, cg);
        any_live |= lv != 0u;
        // a 32-key group no row of the warp sees (a head of the pair without this slash
        // block: ~1/3 of the rows on the bench index) needs no TMEM load
        if (!__all_sync(0xffffffffu, lv == 0u || m == -INFINITY)) {
          tmem_ld32(Sb + 32 * cg, sv);
          tmem_ld_wait();
        }
        if (lv == ~0u && m != -INFINITY) {
          // every key live (the common case): FFMA + MUFU + max + add per key
          // packed f32x2 FMA / ADD (FFMA2 / FADD2): the same IEEE results as the scalar pairs
          float2 ls = make_float2(0.f, 0.f);
          const float2 sc2 = make_float2(sc, sc), nm2 = make_float2(-m, -m);
#pragma unroll
          for (int cc = 0; cc < 32; cc += 2) {
            const float2 t = ffma2(make_float2(__uint_as_float(sv[cc]), __uint_as_float(sv[cc + 1])), sc2, nm2);
#if MT_FWD_POLY == 0
            const float p0 = ex2(t.x);
            const float p1 = ex2(t.y);
#else
            const float p0 = ex2(t.x);
            const float p1 = (cc & 2) ? ex2_poly(t.y) : ex2(t.y);
#endif
            emax = fmaxf(emax, fmaxf(t.x, t.y));
            ls = fadd2(ls, make_float2(p0, p1));
            pk[cc >> 1] = pack_bf16x2(p0, p1);
          }
          l += ls.x + ls.y;
        } else if (lv == 0u || m == -INFINITY) {
#pragma unroll
          for (int cc = 0; cc < 16; ++cc) pk[cc] = 0u;
        } else {
#pragma unroll
          for (int cc = 0; cc < 32; cc += 2) {
            const float t0 = fmaf(__uint_as_float(sv[cc]), sc, -m);
            const float t1 = fmaf(__uint_as_float(sv[cc + 1]), sc, -m);
            const bool on0 = (lv >> cc) & 1u, on1 = (lv >> (cc + 1)) & 1u;
            const float p0 = on0 ? ex2(t0) : 0.f;
            const float p1 = on1 ? ex2(t1) : 0.f;
            emax = fmaxf(emax, fmaxf(on0 ? t0 : -INFINITY, on1 ? t1 : -INFINITY));
            l += p0 + p1;
            pk[cc >> 1] = pack_bf16x2(p0, p1);
          }
        }
        tmem_st16(Sb + 16 * cg, pk);
      }
      ovf |= emax > kOverflow || (any_live && m == -INFINITY);
      tile_emax = fmaxf(tile_emax, emax);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(pfull);
#ifndef MT_TL_PROD
      if (row == 0) MT_TL(5, cm.seq);
#endif
    }
    if (tile < 0) break;  // DONE
    int h0, h1, j;
    tile_coords(P, tile, h0, h1, j);
    // keep the once-per-tile mready phase aligned even without data chunks
    if (!m_synced) {
      if (wg == 0) {
        sm.m[row] = -INFINITY;
        mbar_arrive(mready);
      } else {
        mbar_wait(mready, mr_phase);
        m = sm.m[row];
      }
    }
    mr_phase ^= 1;
    if (ovf) sm.ovf[ntile & 1] = 1;

    // ---- epilogue (both warpgroups: d columns [64 wg, 64 wg + 64) of each row)
    const int h = x ? h1 : h0;
    const int64_t tok = (int64_t)j * 64 + qi;
    const size_t obase = ((size_t)tok * Hq + (h < 0 ? 0 : h)) * 128 + 64 * wg;
    float lse_old = -INFINITY;
    if (!P.first && h >= 0) lse_old = P.lse[(int64_t)h * S_loc + tok];
    if (row == 0) MT_CRUMB(3 + wg, 5000000 + (int)ntile);
    mbar_wait(smem_u32(&sm.obar[0]), ntile & 1);  // every O MMA of the tile complete
    if (row == 0) MT_CRUMB(3 + wg, 6000000 + (int)ntile);
    tc_fence_after();
    sm.lsum[wg][row] = l;
    sm.emx[wg][row] = tile_emax;
    named_bar_sync(3, kSoftmax);
    {  // underflow: the row has live keys but all of them sit far below the stabiliser
      const float e = fmaxf(sm.emx[0][row], sm.emx[1][row]);
      if (P.stabfix && e > -INFINITY && e < kUnderflow) sm.ovf[ntile & 1] = 1;
    }
    named_bar_sync(3, kSoftmax);
    if (row == 0) MT_CRUMB(5 + wg, 7000000 + (int)ntile);
    const bool tile_ovf = sm.ovf[ntile & 1] != 0;
    const float lt = sm.lsum[0][row] + sm.lsum[1][row];
    if (!tile_ovf && h >= 0) {  // flagged tiles are written by the exact fix-up pass
      float lse_new = -INFINITY, inv_l = 0.f;
      if (lt > 0.f) {
        inv_l = 1.f / lt;
        lse_new = (m + __log2f(lt)) * 0.69314718055994531f;
      }
      const float mx = fmaxf(lse_old, lse_new);
      float out = -INFINITY, wa = 0.f, wb = 0.f;
      if (mx > -INFINITY) {
        const float eo = lse_old == -INFINITY ? 0.f : __expf(lse_old - mx);
        const float en = lse_new == -INFINITY ? 0.f : __expf(lse_new - mx);
        out = mx + __logf(eo + en);
        wa = eo / (eo + en);
        wb = en / (eo + en) * inv_l;
      }
      if (wg == 0) P.lse[(int64_t)h * S_loc + tok] = out;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        // a row without live keys in this step has no O contribution: the accumulator
        // holds another tile's data (or was never written), so it is not read
        uint32_t o[32];
        tmem_ld32(tmem + lb + kColO + 64 * wg + 32 * hh, o);
        tmem_ld_wait();
        float val[32];
#pragma unroll
        for (int cc = 0; cc < 32; ++cc) val[cc] = lt > 0.f ? __uint_as_float(o[cc]) * wb : 0.f;
        if (!P.first) {
          const float4* src = reinterpret_cast<const float4*>(P.o_acc + obase + 32 * hh);
#pragma unroll
          for (int v4 = 0; v4 < 8; ++v4) {
            const float4 a = src[v4];
            val[4 * v4] += wa * a.x;
            val[4 * v4 + 1] += wa * a.y;
            val[4 * v4 + 2] += wa * a.z;
            val[4 * v4 + 3] += wa * a.w;
          }
        }
        if (P.last) {
          uint4* dst = reinterpret_cast<uint4*>(P.o + obase + 32 * hh);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            dst[u] = make_uint4(pack_bf16x2(val[8 * u], val[8 * u + 1]),
                                pack_bf16x2(val[8 * u + 2], val[8 * u + 3]),
                                pack_bf16x2(val[8 * u + 4], val[8 * u + 5]),
                                pack_bf16x2(val[8 * u + 6], val[8 * u + 7]));
        } else {
          float4* dst = reinterpret_cast<float4*>(P.o_acc + obase + 32 * hh);
#pragma unroll
          for (int v4 = 0; v4 < 8; ++v4)
            dst[v4] = make_float4(val[4 * v4], val[4 * v4 + 1], val[4 * v4 + 2], val[4 * v4 + 3]);
        }
      }
    }
    if (tile_ovf && threadIdx.x == 128) P.fix_list[atomicAdd(P.fix_count, 1)] = tile;
    tc_fence_before();
    named_bar_sync(3, kSoftmax);  // m / lsum are reused by the next tile
    mbar_arrive(smem_u32(&sm.edone));
    if (row == 0) MT_CRUMB(5 + wg, 8000000 + (int)ntile);
    if (row == 32) MT_CRUMB(7, 9000000 + wg * 100000 + (int)ntile);
    if (threadIdx.x == 128) sm.ovf[ntile & 1] = 0;  // next used two tiles later
    ++ntile;
  }
}

// one instantiation per sequence layout (each carries only its own K-producer walk)
template <int L>
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
    for (int b = 0; b < kNB; ++b) {
      mbar_init(smem_u32(&sm.sfull[b]), 2);
      mbar_init(smem_u32(&sm.sfree[b]), 128);  // smeta[b] read by the chunk's warpgroup
      mbar_init(smem_u32(&sm.pfull[b]), 128);  // P of the chunk in buffer b written
    }
    for (int b = 0; b < 2; ++b) mbar_init(smem_u32(&sm.obar[b]), 1);
    mbar_init(smem_u32(&sm.qfull), 1);
    mbar_init(smem_u32(&sm.qempty), 1);
    mbar_init(smem_u32(&sm.mready), 128);
    mbar_init(smem_u32(&sm.edone), kSoftmax);
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&sm.gqfull[i]), 1);
      mbar_init(smem_u32(&sm.gqempty[i]), 1);
    }
    for (int i = 0; i < kVM; ++i) {
      mbar_init(smem_u32(&sm.vmfull[i]), 1);
      mbar_init(smem_u32(&sm.vmfree[i]), 1);
    }
    sm.ovf[0] = sm.ovf[1] = 0;
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(smem_u32(&sm.tmem_base), 512);
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
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;" ::: "memory");
    if (warp == 0) {
      producer_k<L>(sm, P, &tmq, &tmk, &tmkp);
    } else if (warp == 2) {
      producer_v(sm, P, &tmv, &tmvp);
    } else if (warp == 1) {
      mma_issuer(sm, P, tmem);  // whole warp: uniform control flow, one elected lane issues
    } else {
      k_gatherer(sm, P);
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
    softmax_epilogue(sm, P, tmem);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
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
    if (plan_owner(pl, g - o) != P.s) continue;
    const int lb = plan_g2l(pl, g - o);
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
    fn(plan_g2l(pl, blk) * 64 + (m & 63));
  }
}
__global__ void __launch_bounds__(256) attn_fwd_fixup(const __grid_constant__ Params P,
                                                      const __nv_bfloat16* __restrict__ q) {
  const int n = *P.fix_count;
  const int lane = lane_id(), w = warp_id();
  const VSPlan& pl = P.plan;
  const int grp = pl.Hq / pl.Hkv;
  const int64_t S_loc = (int64_t)P.nloc * 64;
  for (int f = blockIdx.x; f < 2 * n; f += gridDim.x) {  // (flagged tile, head of the pair)
    int h0, h1, j;
    tile_coords(P, P.fix_list[f >> 1], h0, h1, j);
    const int h = (f & 1) ? h1 : h0;
    if (h < 0) continue;
    const int g = plan_l2g(pl, P.r, j), gkv = h / grp;
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
      const int64_t lrow = (int64_t)plan_g2l(pl, m >> 6) * 64 + (m & 63);
      const __nv_bfloat16* src = (part < 16 ? k : v) + (lrow * pl.Hkv + h / grp) * 128;
      val = reinterpret_cast<const uint4*>(src)[c16];
    }
    (part < 16 ? kp : vp)[((int64_t)i * pl.Hq + h) * 16 + c16] = val;
  }
}

}  // namespace fwd

static_assert(sizeof(fwd::Smem) <= 232448, "forward SMEM exceeds 227 KB");
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
  const int grp = plan.Hq / plan.Hkv;
  P.single = plan.bptr ? 1 : 0;  // block-CSR rows are per head: one head per tile
  P.ppg = P.single ? grp : (grp + 1) / 2;
  P.n_tiles = plan.Hkv * P.ppg * nloc;
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
  static const int stabfix = getenv("MT_FWD_STABFIX") ? atoi(getenv("MT_FWD_STABFIX")) : 1;
  static const int fdbg = getenv("MT_FWD_DBG") ? atoi(getenv("MT_FWD_DBG")) : 0;
  P.dbg = fdbg;
  P.stabfix = stabfix;
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
  auto kernel = plan.layout ? attn_fwd_kernel<1> : attn_fwd_kernel<0>;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return fail(MT_ECUDA, "cudaFuncSetAttribute(attn_fwd) failed (smem %zu)", smem);
  const int grid = P.n_tiles < num_sms ? P.n_tiles : num_sms;
  cudaMemsetAsync(P.fix_count, 0, 2 * sizeof(int), st);  // fix-up count, tile counter
  if (grid > 0) kernel<<<grid, kThreads, smem, st>>>(P, tmq, tmk, tmv, tmkp, tmvp);
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
