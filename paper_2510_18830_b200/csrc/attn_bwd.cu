// attn_bwd.cu — block-sparse vertical-slash attention backward for sm_100a, one
// ring step.  PAPER.md Eq. 1 and Eq. 12:
//   P = exp(S - LSE), dP = dO V^T, dS = P o (dP - D), D_n = dO_n . O_n,
//   dV = P^T dO, dK = dS^T Q / sqrt(d), dQ = dS K / sqrt(d),
// with the forward's sparsity ("superposition"): the same key sets.
//
// Key-major ("column-parallel") tiles: the 128 key rows of a tile stay in smem
// and their dK/dV accumulate in TMEM over every (q head, query block) chunk
// that attends them; dQ of each chunk is reduce-added to an fp32 accumulator.
//   mode BLOCK: tile = q head h x local key blocks (lb0, lb0+1) of the held
//               chunk; chunks = local query blocks j of head h with
//               g_q - kb = o for a selected slash o (o = t mod W).  The 8 q heads
//               of a kv group add into the same dK/dV rows -> bulk tensor
//               reduce-add.  Tile order: see "L2 locality" below.
//   mode BAR  : tile = q head h x 128 consecutive entries of the origin's
//               vertical list; chunks = every later local query block; a
//               (column, block) pair is live iff the column is not covered by a
//               selected slash of that block (I9).  dK/dV -> atomic scatter-add
//               (the paper's "backward for all vertical lines").
// Per chunk (M = 128 keys, N = 64 queries), in the TMEM region of the softmax
// warpgroup that owns the chunk:
//   S^T = K Q^T, then dP^T = V dO^T         (tcgen05, SMEM x SMEM -> TMEM; separate commits)
//   P^T from S^T while dP^T runs, then dS^T (bf16, dS pre-scaled by 1/sqrt d), both
//     tcgen05.st back over S^T (A operands of dV, dK); dS^T also -> SMEM
//   dQ^T = K^T dS^T                          (TMEM over dP^T, M = d; live 64-key slots only)
//     committed on its own: the warpgroup drains it (bulk reduce-add) while
//   dV += P^T dO, dK += dS^T Q              (A from TMEM, N = 128) run
// Keeping P^T/dS^T in TMEM saves 48 KB of shared-memory traffic per chunk: the
// SMEM x SMEM N = 64 MMAs are shared-memory-bandwidth bound (51 instead of 32
// cycles per MMA, tools/mma_bench.cu), so SMEM bytes are this kernel's currency.
// Warp roles: warp 0 producer (TMA / cp.async), warp 1 MMA issuer, warps 4..11
// two softmax-backward warpgroups (alternate chunks) + dQ drain + epilogue.
//
// L2 locality (BLOCK): the streamed operands (Q, dO: 32 KB, dQ reduce: 32 KB per
// chunk) dominate DRAM traffic.  A query block (h, g_q) is needed by the tiles
// kb = g_q - o, o in i_s[h].  Tiles are numbered head-major with key pairs
// ascending and handed out by an atomic counter, so the ~148 resident tiles are
// consecutive key pairs of one head walking the same offset list at the same
// pace: each query block they touch is reused by ~(2 x 148 x |i_s| / nb) tiles
// while L2-resident (measured: DRAM traffic 1.84 TB -> 0.20 TB per 512K launch,
// L2 hit 19% -> 70%).  (Starting each wave of 148 tiles together behind a grid
// barrier was measured slower and dropped.)
#include <cstdlib>

#include "common.cuh"
#include "plan.cuh"
#define MT_TL_ON (P.dbg >= 0)  // timeline probe: every tile
#include "sm100.cuh"
#include "tmap.cuh"

namespace mt {

namespace bwd {

#ifndef MT_BWD_STAGES
#define MT_BWD_STAGES 4
#endif
// Q / dO / LSE / D stages.  4: each softmax warpgroup's 16 KB buffer stages dQ in two
// halves.  3 (-DMT_BWD_STAGES=3) gives each a 32 KB buffer and ONE bulk reduce-add per
// chunk, but measured slower (296 vs 278 ms at 512K: the loads starve with 3 stages).
constexpr int kStages = MT_BWD_STAGES;
#ifndef MT_BWD_SPLIT_SDP
#define MT_BWD_SPLIT_SDP 1  // S^T committed before dP^T is issued (P^T overlaps the dP^T MMAs)
#endif
// (Issuing dV += P^T dO as soon as P^T was in TMEM, ahead of dS^T, measured 258.6 vs 249.5 ms
// at 512K: the extra MMA group in the in-order tensor pipe delays the other region's S^T.)
constexpr int kThreads = 384;   // warpgroup 0: producer, MMA, 2 idle; warpgroups 1-2: softmax
constexpr uint32_t kTileKV = 128 * 128 * 2;  // 32 KB (128 keys x d)
constexpr uint32_t kTileQ = 64 * 128 * 2;    // 16 KB (64 queries x d)
constexpr uint32_t kTileP = 128 * 64 * 2;    // 16 KB (128 keys x 64 queries)
constexpr uint32_t kTilePD = (kStages <= 3) ? 2 * kTileP : kTileP;  // per-warpgroup buffer

enum : int { kModeBlock = 0, kModeBar = 1 };
enum : int { kChunk = 0, kEnd = 1, kDone = 2 };

// TMEM columns: dK, dV accumulators, then one 128-column region per softmax
// warpgroup b at kColR + 128 b:
//   [0, 64)   S^T (fp32)  -> P^T (bf16 pairs, cols 0-31) + dS^T (bf16 pairs, 32-63)
//   [64, 128) dP^T (fp32) -> dQ^T (fp32, lanes = d)
constexpr uint32_t kColDK = 0, kColDV = 128, kColR = 256;

struct alignas(16) ChunkMeta {
  int kind;
  int h;           // q head
  int j;           // local query block
  uint32_t flags;  // BLOCK: bit0/1 slot0/1 live, bit2/3 slot0/1 diagonal
  int stage;       // smem stage holding the chunk's Q / dO / LSE / D
  int tile;        // kEnd: the tile it closes
  int seq;         // producer event index (timeline probe)
  int mode;        // kModeBlock / kModeBar: the tile kind this chunk belongs to
};

struct Smem {
  uint8_t k[kTileKV];
  uint8_t v[kTileKV];
  uint8_t q[kStages][kTileQ];
  uint8_t dO[kStages][kTileQ];
  // per softmax warpgroup: dS^T (16 KB, the B operand of dQ^T); once the gradient
  // MMAs are done the same 16 KB stages its dQ tile, 32 queries [32][128] fp32 at
  // a time, for the bulk reduce-adds (P^T lives in TMEM)
  uint8_t pd[2][kTilePD];
  alignas(16) float lse[kStages][64];
  alignas(16) float dd[kStages][64];
  ChunkMeta meta[kStages];
  ChunkMeta smeta[2];      // handed to softmax warpgroup 0 / 1
  int cols[128];           // BAR: global column of each key row (-1 = padding)
  int tile_chunks[2];      // chunks each softmax warpgroup saw in the current tile
  uint64_t full[kStages], empty[kStages];
  uint64_t kvfull, kvempty, tfree;
  uint64_t sfull[2], dsfull[2], gdone[2], dqfree[2];  // dqfree: region drained
  uint64_t dqdone[2];  // dQ^T complete (committed before dV / dK: the drain overlaps them)
  uint64_t dpfull[2];  // dP^T landed (MMA commit; S^T lands first, on sfull)
  uint32_t tmem_base;
};

struct Params {
  VSPlan plan;
  int n_block;              // tiles [0, n_block) are BLOCK tiles, the rest BAR tiles (one launch)
  int bar_first;            // 1: BAR tiles are numbered first (longest tiles first)
  int r, s, t;              // rank, origin, step residue
  int nloc;                 // local blocks per rank (queries and keys)
  int n_tiles;              // n_block + upper bound of BAR tiles (per-head lists)
  int n_bar;                // upper bound of BAR tiles
  float scale_log2;         // log2(e)/sqrt(d)
  float inv_sqrt_d;
  const __nv_bfloat16* k;   // held chunk [S_loc][Hkv][128]
  const __nv_bfloat16* v;
  const float* lse;         // [Hq][S_loc] natural log
  const float* dvec;        // [Hq][S_loc] D = rowsum(dO o O)
  float* dq;                // [S_loc][Hq][128] fp32 accumulator (reduce-add)
  float* dk;                // [S_loc][Hkv][128] fp32 accumulator of the held chunk
  float* dv;
  int* tile_counter;        // dynamic tile scheduler (zeroed before the launch)
  int static_tiles;         // 1: round-robin tiles instead (A/B switch, MT_BWD_STATIC=1)
  int bar_parts;            // BAR: query-range parts per column group
  int bar_part_len;         // BAR: query blocks per part
  int dbg;                  // A/B and profiling switches (MT_BWD_DBG): bit0 skip dQ reduce-adds
                            // (timing only), bit2 per-element dQ red.add, bit5 scalar BAR dK/dV
                            // red.add, bit6 no dead-slot softmax skip, bit7 no dQ^T slot skip
  int hpt;                  // BLOCK: q heads per tile (of one kv head; their dK/dV sum stays in
                            // TMEM, so the tile's K/V load and dK/dV epilogue are shared)
};

// ---- tile decoding
struct Tile {
  int mode;    // kModeBlock / kModeBar
  bool ok;
  bool skip;   // BAR: part holds no query block after the tile's first column
  int g;       // kv head
  int h;       // BAR: q head
  int lb0;     // BLOCK: first local key block
  int e0, e1;  // BAR: entry range in vcol (absolute)
  int j_lo, j_hi;  // BAR: local query blocks [j_lo, j_hi) of this part
};

// Tile kinds a launch holds (template M): kOnlyBlock / kOnlyBar launches (large sequences:
// the block pass compiles without any bar-tile branch, as round 1's) or kMixed (one launch
// for both kinds: short sequences, where the tail of one pass overlaps the other).
enum : int { kOnlyBlock = 0, kOnlyBar = 1, kMixed = 2 };
template <int M>
__device__ __forceinline__ bool is_block(int mode) { return M == kOnlyBlock || (M == kMixed && mode == kModeBlock); }
template <int M>
__device__ __forceinline__ bool is_bar(int mode) { return M == kOnlyBar || (M == kMixed && mode == kModeBar); }

// BAR tiles of this launch: sum over q heads of ceil(|origin list| / 128) x parts
template <int M>
__device__ __forceinline__ int bar_tile_count(const Params& P) {
  const VSPlan& pl = P.plan;
  if (M == kOnlyBlock || P.n_bar == 0) return 0;
  int n = 0;
  for (int h = 0; h < pl.Hq; ++h)
    n += (pl.vptr[h * (pl.W + 1) + P.s + 1] - pl.vptr[h * (pl.W + 1) + P.s] + 127) / 128;
  return n * P.bar_parts;
}

// One launch runs both tile kinds (the tail of one overlaps the other): BLOCK tiles
// [0, n_block) and BAR tiles after them, or BAR tiles first when P.bar_first (their
// per-tile work is the longest).  nbar = bar_tile_count(P).
template <int M>
__device__ __forceinline__ Tile decode_tile(const Params& P, int tile, int nbar) {
  Tile T{};
  const VSPlan& pl = P.plan;
  const int W = pl.W;
  const int nblk = M == kOnlyBar ? 0 : P.n_block;
  if (tile < 0 || tile >= nblk + nbar) return T;
  int bt;  // BLOCK tile index, or -1
  if (M == kOnlyBlock) {
    bt = tile;
  } else if (M == kOnlyBar) {
    bt = -1 - tile;
  } else if (P.bar_first) {
    bt = tile >= nbar ? tile - nbar : -1;
    if (bt < 0) bt = -1 - tile;  // BAR tile -(bt + 1)
  } else {
    bt = tile < P.n_block ? tile : -1 - (tile - P.n_block);
  }
  if (bt >= 0) {
    const int npairs = (P.nloc + 1) / 2;
    T.mode = kModeBlock;
    T.ok = true;
    T.h = (bt / npairs) * P.hpt;  // first q head of the tile
    T.g = T.h / (pl.Hq / pl.Hkv);
    T.lb0 = 2 * (bt % npairs);  // early key blocks (most work) first
    return T;
  }
  tile = -1 - bt;
  T.mode = kModeBar;
  // BAR: (head, 128-column group, part of the query range).  Parts of at most
  // bar_part_len query blocks keep tile lengths comparable (a group of early
  // columns otherwise walks every later query block); within a head, the parts
  // nearest the end go first, matching the descending walk.
  int base = 0;
  for (int h = 0; h < pl.Hq; ++h) {
    const int b = pl.vptr[h * (W + 1) + P.s], e = pl.vptr[h * (W + 1) + P.s + 1];
    const int n = (e - b + 127) / 128;
    if (tile < base + n * P.bar_parts) {
      const int t = tile - base;
      const int part = P.bar_parts - 1 - t / n;
      T.ok = true;
      T.h = h;
      T.g = h / (pl.Hq / pl.Hkv);
      T.e0 = b + (t % n) * 128;
      T.e1 = min(e, T.e0 + 128);
      T.j_lo = part * P.bar_part_len;
      T.j_hi = min(P.nloc, T.j_lo + P.bar_part_len);
      // first rank-local query block after the group's first (smallest) column
      const int bfirst = pl.vcol[(int64_t)h * pl.S + T.e0] >> 6;
      const int j0 = plan_count_le(pl, P.r, bfirst);
      T.skip = max(T.j_lo, j0) >= T.j_hi;
      return T;
    }
    base += n * P.bar_parts;
  }
  return T;
}

// ------------------------------------------------------------------ producer
template <int L, int M>  // sequence layout (plan.cuh) and tile kinds, fixed per launch
__device__ void producer(Smem& sm, const Params& P, const CUtensorMap* tmq,
                         const CUtensorMap* tmdo, const CUtensorMap* tmk,
                         const CUtensorMap* tmv) {
  const int lane = lane_id();
  const VSPlan& pl = P.plan;
  const int W = pl.W;
  const int64_t S_loc = (int64_t)P.nloc * 64;
  uint32_t c = 0;  // chunk events (incl. END)
  uint32_t ntile = 0;
  int cur_mode = kModeBlock;
  const int nbar = bar_tile_count<M>(P);
  auto emit = [&](int h, int j, uint32_t flags) {
    const uint32_t stage = c % kStages;
    MT_CRUMB(2, 1000000 + (int)c);
    mbar_wait(smem_u32(&sm.empty[stage]), ((c / kStages) & 1) ^ 1);
    if (lane == 0) MT_TL(0, c);
    if (lane == 0) {
      ChunkMeta& m = sm.meta[stage];
      m.seq = (int)c;
      m.kind = kChunk;
      m.h = h;
      m.j = j;
      m.flags = flags;
      m.mode = cur_mode;
      m.stage = (int)stage;
      const uint32_t bar = smem_u32(&sm.full[stage]);
      mbar_expect_tx(bar, 2 * kTileQ + 512);
      for (int cc = 0; cc < 2; ++cc) {
        tma_load_3d(smem_u32(sm.q[stage] + cc * 8192), tmq, bar, cc * 64, h, j * 64);
        tma_load_3d(smem_u32(sm.dO[stage] + cc * 8192), tmdo, bar, cc * 64, h, j * 64);
      }
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(
              smem_u32(sm.lse[stage])),
          "l"(P.lse + (int64_t)h * S_loc + (int64_t)j * 64), "r"(bar)
          : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(
              smem_u32(sm.dd[stage])),
          "l"(P.dvec + (int64_t)h * S_loc + (int64_t)j * 64), "r"(bar)
          : "memory");
    }
    __syncwarp();
    ++c;
  };

  for (int it = 0;; ++it) {
    int tile = 0;
    if (P.static_tiles) {
      tile = blockIdx.x + it * gridDim.x;
    } else {
      if (lane == 0) tile = atomicAdd(P.tile_counter, 1);
      tile = __shfl_sync(0xffffffffu, tile, 0);
    }
    const Tile T = decode_tile<M>(P, tile, nbar);
    if (!T.ok) break;
    cur_mode = T.mode;
    if (T.skip) continue;
    // ---- K/V tile: wait until every MMA of the previous tile finished and its
    // epilogue (which reads cols[]) is done
    if (ntile > 0) {
      MT_CRUMB(2, 2000000 + (int)ntile);
      mbar_wait(smem_u32(&sm.kvempty), (ntile - 1) & 1);
      MT_CRUMB(2, 3000000 + (int)ntile);
      mbar_wait(smem_u32(&sm.tfree), (ntile - 1) & 1);
    }
    ++ntile;
    const uint32_t kvbar = smem_u32(&sm.kvfull);
    if (is_block<M>(T.mode)) {
      const bool v1 = T.lb0 + 1 < P.nloc;
      if (lane == 0) {
        // a missing second slot re-loads block lb0: every K/V row must be finite
        // because dQ^T = K^T dS^T contracts over all 128 rows (masked rows have dS = 0)
        mbar_expect_tx(kvbar, 2 * kTileKV);
        for (int sl = 0; sl < 2; ++sl)
          for (int cc = 0; cc < 2; ++cc) {
            const uint32_t off = cc * 16384 + sl * 8192;
            const int blk = v1 ? T.lb0 + sl : T.lb0;
            tma_load_3d(smem_u32(sm.k + off), tmk, kvbar, cc * 64, T.g, blk * 64);
            tma_load_3d(smem_u32(sm.v + off), tmv, kvbar, cc * 64, T.g, blk * 64);
          }
      }
      __syncwarp();
    } else {
      const int n = T.e1 - T.e0;
      const int32_t* vc = pl.vcol + (int64_t)T.h * pl.S;
      for (int rr = lane; rr < 128; rr += 32) sm.cols[rr] = rr < n ? vc[T.e0 + rr] : -1;
      __syncwarp();
      const uint32_t kb = smem_u32(sm.k), vb = smem_u32(sm.v);
      const int m0 = sm.cols[0];
      for (int pidx = lane; pidx < 128 * 16; pidx += 32) {
        const int row = pidx >> 4, c16 = pidx & 15;
        int m = sm.cols[row];
        if (m < 0) m = m0;  // padding rows duplicate a live row (masked later)
        const int blk = m >> 6;
        const int64_t lrow = (int64_t)g2l_<L>(pl, blk) * 64 + (m & 63);
        const size_t goff = ((size_t)lrow * pl.Hkv + T.g) * 128 + c16 * 8;
        const uint32_t doff = (c16 >> 3) * 16384 + sw128(row, c16 & 7);
        cp_async_16(kb + doff, P.k + goff);
        cp_async_16(vb + doff, P.v + goff);
      }
      asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(kvbar) : "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(kvbar);
    }

    // ---- chunk stream
    if (is_block<M>(T.mode)) {
      const bool v1 = T.lb0 + 1 < P.nloc;
      const int kb0 = l2g_<L>(pl, P.s, T.lb0);  // global key block of slot 0
      if (pl.tptr) {
        // block-CSR mode (W = 1): the pair's sorted (gq << 1 | slot) entries; a query
        // block attending both slots has two adjacent entries, emitted once (at the
        // second) with both slot flags
        const int64_t seg = (int64_t)T.h * pl.npairs + (T.lb0 >> 1);
        const int64_t eb = pl.tptr[seg], ee = pl.tptr[seg + 1];
        int carry = -1;  // last entry of the previous batch
        for (int64_t base = eb; base < ee; base += 32) {
          const int64_t i = base + lane;
          const bool live = i < ee;
          const int e = live ? pl.tidx[i] : -1;
          const int nx0 = __shfl_down_sync(0xffffffffu, e, 1);
          const int nx = i + 1 < ee ? (lane < 31 ? nx0 : pl.tidx[i + 1]) : -1;
          const int pv0 = __shfl_up_sync(0xffffffffu, e, 1);
          const int pv = lane == 0 ? carry : pv0;
          const int gq = e >> 1;
          uint32_t flags = 0;
          if (live) {
            flags |= (e & 1) ? (gq == kb0 + 1 ? 10u : 2u) : (gq == kb0 ? 5u : 1u);
            if (pv >= 0 && (pv >> 1) == gq)
              flags |= (pv & 1) ? (gq == kb0 + 1 ? 10u : 2u) : (gq == kb0 ? 5u : 1u);
          }
          uint32_t bal = __ballot_sync(0xffffffffu, live && (nx < 0 || (nx >> 1) != gq));
          while (bal) {
            const int l = __ffs(bal) - 1;
            bal &= bal - 1;
            emit(T.h, __shfl_sync(0xffffffffu, gq, l), __shfl_sync(0xffffffffu, flags, l));
          }
          carry = __shfl_sync(0xffffffffu, e, 31);
        }
      } else {
        // local query blocks j >= jfirst (global gq = l2g(r, j) >= kb0; block-striped:
        // the lattice gq = kb0 + t + mW): slot 0 (key block kb0) is live iff gq - kb0 is a
        // selected offset, slot 1 (key block kb1) iff gq - kb1 is.  32 query blocks per
        // ballot from the slash bitmap: a scalar walk of the offset list costs a dependent
        // global load per offset and skips (W-1)/W of them.
        const int kb1 = v1 ? l2g_<L>(pl, P.s, T.lb0 + 1) : -1;
        const int jfirst = count_le_<L>(pl, P.r, kb0 - 1);
        for (int h = T.h; h < T.h + P.hpt; ++h) {  // the tile's q heads one after another
        const uint32_t* bits = pl.s_bits + (int64_t)h * pl.bits_words;
        auto has = [&](int x) { return x >= 0 && ((bits[x >> 5] >> (x & 31)) & 1u) != 0u; };
        if constexpr (L == 0) {
          // block-striped: gq = kb0 + x on the lattice x = t + mW, slot 1 = kb0 + W
          // (measured: the generic walk below costs the striped backward ~9 ms at 512K)
          const int xmax = pl.nb - kb0;  // gq < nb
          for (int m0 = 0; P.t + m0 * W < xmax; m0 += 32) {
            const int x = P.t + (m0 + lane) * W;
            const bool in = x < xmax;
            const bool a = in && has(x);
            const bool b = in && v1 && has(x - W);
            const uint32_t ba = __ballot_sync(0xffffffffu, a), bb = __ballot_sync(0xffffffffu, b);
            uint32_t bal = ba | bb;
            while (bal) {
              const int l = __ffs(bal) - 1;
              bal &= bal - 1;
              const int xs = P.t + (m0 + l) * W;
              uint32_t flags = 0;
              if ((ba >> l) & 1u) flags |= xs == 0 ? 5u : 1u;  // slot 0 live (+ diagonal)
              if ((bb >> l) & 1u) flags |= xs == W ? 10u : 2u;  // slot 1 live (+ diagonal)
              emit(h, (kb0 + xs - P.r) / W, flags);
            }
          }
        } else {
        for (int j0 = jfirst; j0 < P.nloc; j0 += 32) {
          const int j = j0 + lane;
          const bool in = j < P.nloc;
          const int gq = l2g_<L>(pl, P.r, j);
          const bool a = in && has(gq - kb0);
          const bool b = in && v1 && has(gq - kb1);
          const uint32_t ba = __ballot_sync(0xffffffffu, a), bb = __ballot_sync(0xffffffffu, b);
          uint32_t bal = ba | bb;
          while (bal) {
            const int l = __ffs(bal) - 1;
            bal &= bal - 1;
            const int gl = l2g_<L>(pl, P.r, j0 + l);
            uint32_t flags = 0;
            if ((ba >> l) & 1u) flags |= gl == kb0 ? 5u : 1u;  // slot 0 live (+ diagonal)
            if ((bb >> l) & 1u) flags |= gl == kb1 ? 10u : 2u;  // slot 1 live (+ diagonal)
            emit(h, j0 + l, flags);
          }
        }
        }
        }
      }
      (void)v1;
    } else {
      const int bfirst = sm.cols[0] >> 6;
      // first rank-local query block with global block > bfirst
      const int j0 = count_le_<L>(pl, P.r, bfirst);
      // walk this part's query blocks from the last one down: the resident bar tiles
      // of a head start together and share each Q/dO/dQ block while it is in L2
      for (int j = T.j_hi - 1; j >= max(j0, T.j_lo); --j) emit(T.h, j, 0u);
    }
    // ---- END
    {
      const uint32_t stage = c % kStages;
      mbar_wait(smem_u32(&sm.empty[stage]), ((c / kStages) & 1) ^ 1);
      if (lane == 0) {
        sm.meta[stage].kind = kEnd;
        sm.meta[stage].tile = tile;
        mbar_arrive(smem_u32(&sm.full[stage]));
      }
      __syncwarp();
      ++c;
    }
  }
  // ---- DONE, only once the last tile's epilogue is over: both softmax warpgroups
  // have then consumed that tile's END, so sfull never runs two phases ahead of a
  // warpgroup still draining its last chunk (parity aliasing)
  if (ntile > 0) mbar_wait(smem_u32(&sm.tfree), (ntile - 1) & 1);
  const uint32_t stage = c % kStages;
  mbar_wait(smem_u32(&sm.empty[stage]), ((c / kStages) & 1) ^ 1);
  if (lane == 0) {
    sm.meta[stage].kind = kDone;
    mbar_arrive(smem_u32(&sm.full[stage]));
  }
  __syncwarp();
}

// ------------------------------------------------------------------ MMA issuer
// Chunk k of a tile goes to softmax warpgroup k & 1.  Per chunk: S^T, dP^T into
// the shared TMEM pair, then the gradient MMAs of the previous chunk (dV, dK
// accumulate; dQ^T into that warpgroup's buffer).
template <int M>
__device__ void mma_issuer(Smem& sm, const Params& P, uint32_t tmem) {
  const bool leader = elect_one();
  const uint32_t id_s = make_idesc_bf16(128, 64, false, false);   // S^T, dP^T
  const uint32_t id_kv = make_idesc_bf16(128, 128, false, true);  // dV, dK
  const uint32_t id_q = make_idesc_bf16(128, 64, true, true);     // dQ^T
  // descriptor bases; each MMA only adds an immediate to the address field
  const uint64_t dK = make_sdesc(smem_u32(sm.k), 16, 1024);         // K-major K (S^T)
  const uint64_t dV = make_sdesc(smem_u32(sm.v), 16, 1024);         // K-major V (dP^T)
  const uint64_t dKmn = make_sdesc(smem_u32(sm.k), 16384, 1024);    // MN-major K^T (dQ^T)
  const uint64_t dQ0 = make_sdesc(smem_u32(sm.q[0]), 16, 1024);
  const uint64_t dO0 = make_sdesc(smem_u32(sm.dO[0]), 16, 1024);
  const uint64_t dQmn0 = make_sdesc(smem_u32(sm.q[0]), 8192, 1024);
  const uint64_t dOmn0 = make_sdesc(smem_u32(sm.dO[0]), 8192, 1024);
  const uint64_t dDSTmn0 = make_sdesc(smem_u32(sm.pd[0]), 8192, 1024);
  uint32_t c = 0, ntile = 0;
  uint32_t sq0 = 0, sq1 = 0;                    // S^T/dP^T issued into region 0 / 1
  uint32_t ds0 = 0, ds1 = 0;  // per buffer: dsfull waits
  for (;;) {
    {  // the next chunk tells whether another tile follows
      const uint32_t stage = c % kStages;
      mbar_wait(smem_u32(&sm.full[stage]), (c / kStages) & 1);
      if (sm.meta[stage].kind == kDone) {
        for (uint32_t b = 0; b < 2; ++b)
          if (leader) {
            sm.smeta[b].kind = kDone;
            mbar_arrive(smem_u32(&sm.sfull[b]));
            mbar_arrive(smem_u32(&sm.sfull[b]));
          }
        break;
      }
    }
    MT_CRUMB(0, 2);
    mbar_wait(smem_u32(&sm.kvfull), ntile & 1);
    ++ntile;
    {  // BAR tiles: K/V rows arrived by cp.async (generic proxy)
      const ChunkMeta& m0 = sm.meta[c % kStages];  // the tile's first event (waited above)
      if (M == kOnlyBar || (M == kMixed && m0.kind == kChunk && m0.mode == kModeBar))
        fence_proxy_async_smem();
    }
    tc_fence_after();
    // Event-driven issue: S^T/dP^T of chunk k as soon as its Q/dO landed and its
    // warpgroup's TMEM region is drained; the gradient MMAs of chunk g as soon as its
    // P/dS^T is published.  (A fixed S(k), G(k-1), S(k+1) order makes G(k) wait for chunk
    // k+1's load, which holds chunk k's stage ~2x longer: measured.)
    bool acc_started = false, end_seen = false;
    uint32_t k = 0, g = 0;  // tile-local: chunks whose S^T issued / gradients issued
    // per region: stage / producer seq of its pending chunk (scalars: no local memory)
    uint32_t pst0 = 0, pst1 = 0, end_stage = 0;
    uint32_t plv0 = 3, plv1 = 3;  // live 64-key slots (bit 0 / 1) of the pending chunk
    int pseq0 = 0, pseq1 = 0, end_tile = 0;
    auto uni = [](bool x) { return __shfl_sync(0xffffffffu, x ? 1 : 0, 0) != 0; };
    auto try_grads = [&]() {  // dK, dQ^T of chunk g (softmax warpgroup g & 1)
      const uint32_t bg = g & 1;
      uint32_t& ds = bg ? ds1 : ds0;
      if (!uni(mbar_test_wait(smem_u32(&sm.dsfull[bg]), ds & 1))) return false;
      ++ds;
#ifdef MT_TL_ISSUER
      if (leader) MT_TL(6, bg ? pseq1 : pseq0);
#endif
      tc_fence_after();
      const uint32_t st = bg ? pst1 : pst0;
      const uint64_t dqm = sdesc_add(dQmn0, st * kTileQ);
      const uint64_t dom = sdesc_add(dOmn0, st * kTileQ);
      const uint64_t dstm = sdesc_add(dDSTmn0, bg * kTilePD);
      const uint32_t R = tmem + kColR + 128 * bg;
      if (leader) {
        // dQ^T = K^T dS^T first, with its own commit, so the warpgroup drains it while dV / dK
        // run.  It contracts over the tile's 128 keys: a dead 64-key slot (its dS^T rows are
        // zero) is skipped, 4 of the 8 K-steps (0.86 of the 512K bench chunks have exactly one
        // live slot)
        const uint32_t lv = bg ? plv1 : plv0;
        const int k0 = (lv & 1u) ? 0 : 64, k1 = (lv & 2u) ? 128 : 64;
#pragma unroll
        for (int kk = 0; kk < 128; kk += 16)
          if (kk >= k0 && kk < k1)
            mma_ss(R + 64, sdesc_add(dKmn, kk * 128), sdesc_add(dstm, kk * 128), id_q, kk > k0);
        mma_commit(smem_u32(&sm.dqdone[bg]));
#pragma unroll
        for (int kq = 0; kq < 64; kq += 16) {  // A = P^T / dS^T from TMEM (2 bf16 per column)
          const uint32_t acc = (acc_started || kq > 0) ? 1u : 0u;
          mma_ts(tmem + kColDV, R + kq / 2, sdesc_add(dom, kq * 128), id_kv, acc);
          mma_ts(tmem + kColDK, R + 32 + kq / 2, sdesc_add(dqm, kq * 128), id_kv, acc);
        }
        mma_commit(smem_u32(&sm.gdone[bg]));
        mma_commit(smem_u32(&sm.empty[st]));
        MT_TL(3, bg ? pseq1 : pseq0);
      }
      acc_started = true;
      ++g;
      return true;
    };
    auto try_s = [&]() {  // S^T/dP^T of the next chunk, or note the tile's END
      const uint32_t stage = c % kStages;
      if (!uni(mbar_test_wait(smem_u32(&sm.full[stage]), (c / kStages) & 1))) return false;
      if (sm.meta[stage].kind == kEnd) {
        end_seen = true;
        end_stage = stage;
        end_tile = sm.meta[stage].tile;  // read before the stage is released
        ++c;
        return true;
      }
      const uint32_t b = k & 1;
      // region b is free once the chunk it held two chunks ago was drained
      const uint32_t nsq = b ? sq1 : sq0;
      if (nsq > 0 && !uni(mbar_test_wait(smem_u32(&sm.dqfree[b]), (nsq - 1) & 1)))
        return false;
      // ... and its dV / dK MMAs (readers of P^T / dS^T in the region) are complete
      if (nsq > 0 && !uni(mbar_test_wait(smem_u32(&sm.gdone[b]), (nsq - 1) & 1)))
        return false;
#ifdef MT_TL_ISSUER
      if (leader) MT_TL(7, sm.meta[stage].seq);
#endif
      tc_fence_after();
      const uint32_t R = tmem + kColR + 128 * b;
      if (leader) {
        sm.smeta[b] = sm.meta[stage];
        mbar_arrive(smem_u32(&sm.sfull[b]));  // 1 of 2: publishes smeta
        const uint64_t dq = sdesc_add(dQ0, stage * kTileQ), ddo = sdesc_add(dO0, stage * kTileQ);
#pragma unroll
        for (int kk = 0; kk < 128; kk += 16) {
          const uint32_t ko = (kk >> 6) * 16384 + (kk & 63) * 2;
          const uint32_t qo = (kk >> 6) * 8192 + (kk & 63) * 2;
          mma_ss(R, sdesc_add(dK, ko), sdesc_add(dq, qo), id_s, kk > 0);
          if (!MT_BWD_SPLIT_SDP) mma_ss(R + 64, sdesc_add(dV, ko), sdesc_add(ddo, qo), id_s, kk > 0);
        }
        mma_commit(smem_u32(&sm.sfull[b]));  // 2 of 2: S^T ready (P^T starts on it)
        if (MT_BWD_SPLIT_SDP)
#pragma unroll
        for (int kk = 0; kk < 128; kk += 16) {
          const uint32_t ko = (kk >> 6) * 16384 + (kk & 63) * 2;
          const uint32_t qo = (kk >> 6) * 8192 + (kk & 63) * 2;
          mma_ss(R + 64, sdesc_add(dV, ko), sdesc_add(ddo, qo), id_s, kk > 0);
        }
        mma_commit(smem_u32(&sm.dpfull[b]));  // dP^T ready
        MT_TL(2, sm.meta[stage].seq);
      }
      uint32_t lv = (is_block<M>(sm.meta[stage].mode) && !(P.dbg & 128)) ? (sm.meta[stage].flags & 3u) : 3u;
      lv = lv ? lv : 3u;
      if (b) {
        plv1 = lv;
        pst1 = stage;
        pseq1 = sm.meta[stage].seq;
        ++sq1;
      } else {
        plv0 = lv;
        pst0 = stage;
        pseq0 = sm.meta[stage].seq;
        ++sq0;
      }
      ++k;
      ++c;
      return true;
    };
    MT_CRUMB(0, 1);
    for (;;) {
      if (g < k) try_grads();
      if (!end_seen) try_s();
      if (end_seen && g == k) break;
    }
    if (leader) {
      mma_commit(smem_u32(&sm.kvempty));  // K/V smem reusable after all MMAs so far
      mbar_arrive(smem_u32(&sm.empty[end_stage]));
    }
    // every chunk's gradients are issued, so each warpgroup consumed its last sfull
    for (uint32_t b = 0; b < 2; ++b)
      if (leader) {
        sm.smeta[b].kind = kEnd;
        sm.smeta[b].tile = end_tile;
        mbar_arrive(smem_u32(&sm.sfull[b]));
        mbar_arrive(smem_u32(&sm.sfull[b]));
      }
  }
}

// ------------------------------------------------------------------ softmax-backward
__device__ __forceinline__ void red_add_f32(float* addr, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add_f32x4(float* addr, const uint32_t* v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(__uint_as_float(v[0])),
               "f"(__uint_as_float(v[1])), "f"(__uint_as_float(v[2])), "f"(__uint_as_float(v[3]))
               : "memory");
}


__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int M>
__device__ void softmax_bwd(Smem& sm, const Params& P, uint32_t tmem, const CUtensorMap* tmdq,
                            const CUtensorMap* tmdk, const CUtensorMap* tmdv) {
  const int w = warp_id();
  const int quad = w & 3, wg = (w - 4) >> 2;
  const int lane = lane_id();
  const int row = quad * 32 + lane;  // key row of the tile == TMEM lane; d index for dQ^T
  const int slot = row >> 6, kk = row & 63;
  const uint32_t lb = (uint32_t)(quad * 32) << 16;
  const VSPlan& pl = P.plan;
  const uint32_t sfull = smem_u32(&sm.sfull[wg]);
  const uint32_t R = tmem + lb + kColR + 128 * wg;  // this warpgroup's TMEM region (own lanes)
  const uint32_t dsfull = smem_u32(&sm.dsfull[wg]), gdone = smem_u32(&sm.gdone[wg]);
  const uint32_t dqdone = smem_u32(&sm.dqdone[wg]);
  const uint32_t dpfull = smem_u32(&sm.dpfull[wg]);
  const uint32_t dqfree = smem_u32(&sm.dqfree[wg]);
  const uint32_t pdbuf = smem_u32(sm.pd[wg]);
  const uint32_t drow = pdbuf + row * 128;  // dS^T row in SMEM (B of dQ^T)
  const uint32_t wg_bar = 1 + wg;  // named barrier of this warpgroup
  uint32_t su = 0, gw = 0, dpu = 0;  // sfull events, dqdone waits (= chunks), dP^T chunks
  uint32_t ntile = 0;
  const int nbar = bar_tile_count<M>(P);
  bool staging_busy = false;  // a bulk reduce may still be reading this warpgroup's buffer

  auto wait_staging = [&]() {  // warpgroup-uniform
    if (!staging_busy) return;
    if (row == 0) MT_CRUMB(3 + wg, 3000000);
    if (row == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    named_bar_sync(wg_bar, 128);
    staging_busy = false;
  };
  // dQ^T of this warpgroup's chunk (h, j) -> dQ[q][h][d = row].  Runs right after the
  // chunk's P/dS^T is published, so it overlaps the next S^T instead of delaying the
  // gradient MMAs; the reduce's smem read is only waited for before the buffer is
  // rewritten (next P/dS^T or the epilogue).
  auto drain_dq = [&](int h, int j, int seq) {
    if (row == 0) MT_CRUMB(3 + wg, 2000000 + (int)gw);
    mbar_wait(dqdone, gw & 1);  // dQ^T complete (dS^T in SMEM read; dV / dK may still run)
    ++gw;
#if !defined(MT_TL_WARPS) && !defined(MT_TL_ISSUER) && !defined(MT_TL_WGSPLIT)
    if (row == 0) MT_TL(6, seq);
#endif
    tc_fence_after();
    uint32_t r0[32], r1[32];
    tmem_ld32(R + 64, r0);
    tmem_ld32(R + 96, r1);
    tmem_ld_wait();
    tc_fence_before();
    mbar_arrive(dqfree);
    if (P.dbg & 1) return;
    if (P.dbg & 4) {  // A/B: coalesced per-element reduction (thread = d, 64 queries)
      float* dst = P.dq + ((size_t)j * 64 * pl.Hq + h) * 128 + row;
      const size_t qs = (size_t)pl.Hq * 128;
#pragma unroll
      for (int c = 0; c < 32; ++c) red_add_f32(dst + c * qs, __uint_as_float(r0[c]));
#pragma unroll
      for (int c = 0; c < 32; ++c) red_add_f32(dst + (c + 32) * qs, __uint_as_float(r1[c]));
      return;
    }
    if (kTilePD >= 2 * kTileP) {
      // stage dQ[q][d] (fp32, all 64 queries, 32 KB) in this warpgroup's buffer and issue
      // ONE bulk tensor reduce-add; its read is waited for before the buffer is rewritten
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const uint32_t(&rv)[32] = hf ? r1 : r0;
#pragma unroll
        for (int c = 0; c < 32; ++c)
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(pdbuf + (uint32_t)((hf * 32 + c) * 128 + row) * 4),
                       "f"(__uint_as_float(rv[c]))
                       : "memory");
      }
      fence_proxy_async_smem();
      named_bar_sync(wg_bar, 128);
      if (row == 0) {
        asm volatile(
            "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group"
            " [%0, {%1, %2, %3}], [%4];" ::"l"(tmdq),
            "r"(0), "r"(h), "r"(j * 64), "r"(pdbuf)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else {
    // stage dQ[q][d] (fp32) in this warpgroup's 16 KB buffer, 32 queries at a time,
    // each half one bulk tensor reduce-add into the fp32 dQ accumulator
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      if (hf == 1) {  // the first half's reduce must have read the buffer
        if (row == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        named_bar_sync(wg_bar, 128);
      }
      const uint32_t(&rv)[32] = hf ? r1 : r0;
#pragma unroll
      for (int c = 0; c < 32; ++c)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(pdbuf + (uint32_t)(c * 128 + row) * 4),
                     "f"(__uint_as_float(rv[c]))
                     : "memory");
      fence_proxy_async_smem();
      named_bar_sync(wg_bar, 128);
      if (row == 0) {
        asm volatile(
            "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group"
            " [%0, {%1, %2, %3}], [%4];" ::"l"(tmdq),
            "r"(0), "r"(h), "r"(j * 64 + hf * 32), "r"(pdbuf)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    }
#if !defined(MT_TL_WARPS) && !defined(MT_TL_ISSUER) && !defined(MT_TL_WGSPLIT)
    if (row == 0) MT_TL(7, seq);
#endif
    staging_busy = true;
  };

  for (;;) {
    int my_col = -2;  // BAR: this row's column, read at the first chunk
    bool had_chunk = false;
    int tile = -1;
    for (;;) {
      if (row == 0) MT_CRUMB(3 + wg, 1000000 + (int)su);
      mbar_wait(sfull, su & 1);
      ++su;
      const ChunkMeta cm = sm.smeta[wg];
      if (cm.kind == kEnd || cm.kind == kDone) {
        tile = cm.kind == kEnd ? cm.tile : -1;
        break;
      }
      if (is_bar<M>(cm.mode) && my_col == -2) my_col = sm.cols[row];
#ifndef MT_TL_WARPS
      if (row == 0) MT_TL(4, cm.seq);
#endif
      tc_fence_after();
      // which of the 64 queries see this key row
      uint64_t vis;
      if (is_block<M>(cm.mode)) {
        const bool live = (cm.flags >> slot) & 1u;
        const bool diag = (cm.flags >> (2 + slot)) & 1u;
        vis = live ? (diag ? (~0ull << kk) : ~0ull) : 0ull;  // causal: query i >= key kk
      } else {
        bool live = my_col >= 0;
        if (live) {
          const int gq = plan_l2g(pl, P.r, cm.j);
          const int blk = my_col >> 6;
          live = blk < gq && !plan_has_slash(pl, cm.h, gq - blk);
        }
        vis = live ? ~0ull : 0ull;
      }
      // per-query constants of the chunk, scaled in registers as they are used (no barrier):
      // -LSE log2(e) and -D / sqrt(d), the same products as a pre-scaled copy
      const float* nl = sm.lse[cm.stage];
      const float* nd = sm.dd[cm.stage];
      const float2 nlog2e = make_float2(-1.4426950408889634f, -1.4426950408889634f);
      const float2 nisd = make_float2(-P.inv_sqrt_d, -P.inv_sqrt_d);
      // a key row no query of the chunk sees contributes P = dS = 0.  In BLOCK mode a dead
      // 64-key slot is two whole warps (slot = row / 64): they skip the TMEM loads and the
      // exponentials (0.43 of the slot-rows of the 512K bench index) and
      // leave the MUFU / FMA pipes of their SM sub-partitions to the other warpgroup.
      const bool dead = !(P.dbg & 64) && __all_sync(0xffffffffu, vis == 0ull);
      // phase 1: P^T = exp2(S^T log2e/sqrt d - LSE log2e) while the dP^T MMAs still run;
      // P^T (bf16 pairs) over S^T columns 0-31
      float p[64];
      uint32_t pk[32];
      if (dead) {
#pragma unroll
        for (int c = 0; c < 64; ++c) p[c] = 0.f;
      } else {
        uint32_t sv[2][32];
        tmem_ld32(R, sv[0]);
        tmem_ld32(R + 32, sv[1]);
        tmem_ld_wait();
        const float2 sc2 = make_float2(P.scale_log2, P.scale_log2);
        if (vis == ~0ull) {  // every query sees the row (the common case)
#pragma unroll
          for (int q = 0; q < 64; q += 2) {
            const float2 t = ffma2(make_float2(__uint_as_float(sv[q >> 5][q & 31]),
                                               __uint_as_float(sv[q >> 5][(q & 31) + 1])),
                                   sc2, fmul2(*reinterpret_cast<const float2*>(nl + q), nlog2e));
            p[q] = ex2(t.x);
            p[q + 1] = ex2(t.y);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 64; q += 2) {
            const float2 t = ffma2(make_float2(__uint_as_float(sv[q >> 5][q & 31]),
                                               __uint_as_float(sv[q >> 5][(q & 31) + 1])),
                                   sc2, fmul2(*reinterpret_cast<const float2*>(nl + q), nlog2e));
            p[q] = ((vis >> q) & 1ull) ? ex2(t.x) : 0.f;
            p[q + 1] = ((vis >> (q + 1)) & 1ull) ? ex2(t.y) : 0.f;
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) pk[c] = pack_bf16x2(p[2 * c], p[2 * c + 1]);
      tmem_st32(R, pk);
      // phase 2: dS^T = P^T o (dP^T - D) / sqrt d (pre-scaled D) once dP^T has landed
      uint32_t dk[32];
      if (dead) {
#pragma unroll
        for (int c = 0; c < 32; ++c) dk[c] = 0u;
      } else {
        mbar_wait(dpfull, dpu & 1);
        tc_fence_after();
        uint32_t dpv[2][32];
        tmem_ld32(R + 64, dpv[0]);
        tmem_ld32(R + 96, dpv[1]);
        tmem_ld_wait();
        const float2 iv2 = make_float2(P.inv_sqrt_d, P.inv_sqrt_d);
#pragma unroll
        for (int c = 0; c < 32; ++c) {  // packed f32x2 FMA / MUL: the same IEEE results per lane
          const int q = 2 * c;
          const float2 u = ffma2(make_float2(__uint_as_float(dpv[q >> 5][q & 31]),
                                             __uint_as_float(dpv[q >> 5][(q & 31) + 1])),
                                 iv2, fmul2(*reinterpret_cast<const float2*>(nd + q), nisd));
          const float2 d = fmul2(make_float2(p[q], p[q + 1]), u);
          dk[c] = pack_bf16x2(d.x, d.y);
        }
      }
      ++dpu;
      // dS^T over S^T columns 32-63 in this warpgroup's TMEM region (A of dK)
#ifdef MT_TL_WGSPLIT
      if (row == 0) MT_TL(6, cm.seq);  // math done
#endif
      tmem_st32(R + 32, dk);
      wait_staging();  // the previous chunk's dQ reduce has read the buffer
#ifdef MT_TL_WGSPLIT
      if (row == 0) MT_TL(7, cm.seq);  // staging buffer free
#endif
      // dS^T rows of a dead BLOCK slot are not read: dQ^T skips that slot's K-steps
      if (!(dead && is_block<M>(cm.mode) && !(P.dbg & 128)))
#pragma unroll
      for (int c16 = 0; c16 < 8; ++c16) {
        const uint32_t sw = (uint32_t)((c16 ^ (row & 7)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(drow + sw), "r"(dk[4 * c16]),
                     "r"(dk[4 * c16 + 1]), "r"(dk[4 * c16 + 2]), "r"(dk[4 * c16 + 3])
                     : "memory");
      }
      tmem_st_wait();
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(dsfull);
#ifdef MT_TL_WARPS
      if (lane == 0) MT_TL(4 + quad, cm.seq);  // per-warp publish times (quad 0..3)
#else
      if (row == 0) MT_TL(5, cm.seq);
#endif
      drain_dq(cm.h, cm.j, cm.seq);
      had_chunk = true;
    }
    if (tile < 0) break;  // DONE
    const Tile T = decode_tile<M>(P, tile, nbar);
    wait_staging();  // the epilogue stages dK/dV in the same buffer
    if (gw > 0) mbar_wait(gdone, (gw - 1) & 1);  // this warpgroup's last dV / dK MMAs
    tc_fence_after();
    if (row == 0) sm.tile_chunks[wg] = had_chunk ? 1 : 0;
    if (row == 0) MT_CRUMB(3 + wg, 5000000 + (int)ntile);
    named_bar_sync(3, 256);  // both warpgroups: every MMA of the tile complete
    const bool any_chunk = (sm.tile_chunks[0] | sm.tile_chunks[1]) != 0;  // else TMEM is stale

    // ---- dK (warpgroup 0) / dV (warpgroup 1) epilogue: the tile's key rows
    bool live_row;
    int64_t lrow;
    if (is_block<M>(T.mode)) {
      live_row = any_chunk && !(slot == 1 && T.lb0 + 1 >= P.nloc);
      lrow = (int64_t)(T.lb0 + slot) * 64 + kk;
    } else {
      const int m = sm.cols[row];
      live_row = any_chunk && m >= 0;
      lrow = live_row ? (int64_t)plan_g2l(pl, m >> 6) * 64 + (m & 63) : 0;
    }
    const uint32_t col = wg == 0 ? kColDK : kColDV;
    if (is_block<M>(T.mode)) {
      // rows lb0*64 .. +127 are contiguous: stage [128 rows][32 d] fp32 (SW128) in this
      // warpgroup's P/dS buffer, two column groups per round, and bulk reduce-add them
      // (rows past the chunk end are clipped by the tensor map; they hold zeros anyway)
      const CUtensorMap* tm = wg == 0 ? tmdk : tmdv;
#pragma unroll 1
      for (int rd = 0; rd < 4; ++rd) {  // 32 d-columns (16 KB of staging) per round
        uint32_t a[32];
        tmem_ld32(tmem + lb + col + rd * 32, a);
        tmem_ld_wait();
        const uint32_t base = pdbuf + row * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                           base + ((uint32_t)(c ^ (row & 7)) << 4)),
                       "r"(a[4 * c]), "r"(a[4 * c + 1]), "r"(a[4 * c + 2]), "r"(a[4 * c + 3])
                       : "memory");
        fence_proxy_async_smem();
        named_bar_sync(wg_bar, 128);
        if (row == 0 && any_chunk) {
          asm volatile(
              "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group"
              " [%0, {%1, %2, %3}], [%4];" ::"l"(tm),
              "r"(rd * 32), "r"(T.g), "r"(T.lb0 * 64), "r"(pdbuf)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        named_bar_sync(wg_bar, 128);
      }
    } else {
      float* dst = (wg == 0 ? P.dk : P.dv) + ((size_t)lrow * pl.Hkv + T.g) * 128;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t a[32];
        tmem_ld32(tmem + lb + col + c0, a);
        tmem_ld_wait();
        if (!live_row) continue;
        if (P.dbg & 32) {  // A/B: scalar reductions (round 1)
#pragma unroll
          for (int c = 0; c < 32; ++c) red_add_f32(dst + c0 + c, __uint_as_float(a[c]));
        } else {
#pragma unroll
          for (int c = 0; c < 32; c += 4) red_add_f32x4(dst + c0 + c, a + c);
        }
      }
    }
    tc_fence_before();
    if (row == 0) MT_CRUMB(3 + wg, 7000000 + (int)ntile);
    named_bar_sync(3, 256);  // TMEM dK/dV and cols[] free for the next tile
    if (threadIdx.x == 128) mbar_arrive(smem_u32(&sm.tfree));
    ++ntile;
  }
}

// one instantiation per sequence layout: each carries only its own producer walk (the kernel
// with both was 52% larger, and its instruction footprint measurably slowed the striped case)
template <int L, int M>
__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_kernel(const __grid_constant__ Params P, const __grid_constant__ CUtensorMap tmq,
                    const __grid_constant__ CUtensorMap tmdo,
                    const __grid_constant__ CUtensorMap tmk,
                    const __grid_constant__ CUtensorMap tmv,
                    const __grid_constant__ CUtensorMap tmdq,
                    const __grid_constant__ CUtensorMap tmdk,
                    const __grid_constant__ CUtensorMap tmdv) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023u) != 0u) __trap();
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int warp = warp_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(smem_u32(&sm.full[s]), 1);
      mbar_init(smem_u32(&sm.empty[s]), 1);
    }
    mbar_init(smem_u32(&sm.kvfull), 1);
    mbar_init(smem_u32(&sm.kvempty), 1);
    mbar_init(smem_u32(&sm.tfree), 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&sm.sfull[b]), 2);
      mbar_init(smem_u32(&sm.dsfull[b]), 128);
      mbar_init(smem_u32(&sm.gdone[b]), 1);
      mbar_init(smem_u32(&sm.dqdone[b]), 1);
      mbar_init(smem_u32(&sm.dqfree[b]), 128);
      mbar_init(smem_u32(&sm.dpfull[b]), 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(smem_u32(&sm.tmem_base), 512);
  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tmq);
    tma_prefetch_desc(&tmdo);
    tma_prefetch_desc(&tmk);
    tma_prefetch_desc(&tmv);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
    if (warp == 0) {
      producer<L, M>(sm, P, &tmq, &tmdo, &tmk, &tmv);
    } else if (warp == 1) {
      mma_issuer<M>(sm, P, tmem);  // whole warp: uniform control flow, one elected lane issues
    }
#ifdef MT_TIMELINE
    else if (warp == 3 && blockIdx.x == 0) {
      // observer: stamps each stage's "full" completion (load latency = event 1 - event 0)
      for (uint32_t c = 0;; ++c) {
        const uint32_t st = c % kStages;
        mbar_wait(smem_u32(&sm.full[st]), (c / kStages) & 1);
        if (lane_id() == 0) MT_TL(1, c);
        if (sm.meta[st].kind == kDone) break;
      }
    }
#endif
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;" ::: "memory");
    softmax_bwd<M>(sm, P, tmem, &tmdq, &tmdk, &tmdv);
    if (threadIdx.x % 128 == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// D_n = dO_n . O_n (Eq. 1's sum_j dL/dA_ij A_ij), one warp per (token, head) row.
// D = rowsum(dO o O) per (token, q head), one warp per row.  zq / zk / zv (optional):
// fp32 accumulators zeroed on the way, [rows][128] for dQ and [S_loc][Hkv][128] for dK / dV
// (the single-GPU backward: saves the memset pass and its launch)
__global__ void bwd_preprocess_kernel(const __nv_bfloat16* o, const __nv_bfloat16* dO, float* D,
                                      int64_t rows, int Hq, int64_t S_loc, float* zq, float* zk,
                                      float* zv, int Hkv) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= rows) return;
  if (zq) {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    reinterpret_cast<float4*>(zq + w * 128)[lane] = z;
    const int h = (int)(w % Hq);
    if (h < Hkv) {
      const int64_t kr = (w / Hq) * Hkv + h;
      reinterpret_cast<float4*>(zk + kr * 128)[lane] = z;
      reinterpret_cast<float4*>(zv + kr * 128)[lane] = z;
    }
  }
  const uint2 a = reinterpret_cast<const uint2*>(o + w * 128)[lane];
  const uint2 b = reinterpret_cast<const uint2*>(dO + w * 128)[lane];
  const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const float2 x = __bfloat1622float2(a2[u]), y = __bfloat1622float2(b2[u]);
    s += x.x * y.x + x.y * y.y;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) {
    const int64_t tok = w / Hq;
    const int h = (int)(w % Hq);
    D[(int64_t)h * S_loc + tok] = s;
  }
}

struct Cvt3 {  // three fp32 -> bf16 conversions in one launch (dQ, dK, dV)
  const float* x[3];
  __nv_bfloat16* y[3];
  int64_t n[3];
  int64_t b1, b2;  // first block of segment 1 / 2
};

__global__ void f32_to_bf16_kernel(Cvt3 c) {
  const int seg = blockIdx.x < c.b1 ? 0 : (blockIdx.x < c.b2 ? 1 : 2);
  const int64_t blk = (int64_t)blockIdx.x - (seg == 0 ? 0 : (seg == 1 ? c.b1 : c.b2));
  // select by comparisons (a dynamic index into the parameter struct would copy it to local
  // memory in every thread: measured 3x slower)
  const float* x = seg == 0 ? c.x[0] : (seg == 1 ? c.x[1] : c.x[2]);
  __nv_bfloat16* y = seg == 0 ? c.y[0] : (seg == 1 ? c.y[1] : c.y[2]);
  const int64_t n = seg == 0 ? c.n[0] : (seg == 1 ? c.n[1] : c.n[2]);
  const int64_t i = (blk * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    const float4 v = *reinterpret_cast<const float4*>(x + i);
    uint2 o;
    o.x = pack_bf16x2(v.x, v.y);
    o.y = pack_bf16x2(v.z, v.w);
    *reinterpret_cast<uint2*>(y + i) = o;
  } else {
    for (int64_t j = i; j < n; ++j) y[j] = __float2bfloat16_rn(x[j]);
  }
}

}  // namespace bwd

static_assert(sizeof(bwd::Smem) <= 232448, "backward SMEM exceeds 227 KB");
size_t bwd_smem_bytes() { return sizeof(bwd::Smem); }  // the dynamic base is 1024-aligned

mt_status attn_bwd_preprocess(const void* o, const void* dO, float* D, int64_t S_loc, int Hq,
                              cudaStream_t st, float* zq, float* zk, float* zv, int Hkv) {
  const int64_t rows = S_loc * Hq;
  const int threads = 256;
  const int64_t blocks = (rows * 32 + threads - 1) / threads;
  bwd::bwd_preprocess_kernel<<<(unsigned)blocks, threads, 0, st>>>(
      static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dO), D, rows, Hq,
      S_loc, zq, zk, zv, Hkv);
  return check_launch("bwd_preprocess");
}

// y_i = bf16(x_i) for the three (x, y, n) pairs, one launch
mt_status f32_to_bf16_x3(const float* x0, void* y0, int64_t n0, const float* x1, void* y1,
                         int64_t n1, const float* x2, void* y2, int64_t n2, cudaStream_t st) {
  const int64_t threads = 256, per = threads * 4;
  bwd::Cvt3 c{{x0, x1, x2},
              {static_cast<__nv_bfloat16*>(y0), static_cast<__nv_bfloat16*>(y1),
               static_cast<__nv_bfloat16*>(y2)},
              {n0, n1, n2}, 0, 0};
  const int64_t g0 = (n0 + per - 1) / per, g1 = (n1 + per - 1) / per, g2 = (n2 + per - 1) / per;
  c.b1 = g0;
  c.b2 = g0 + g1;
  if (g0 + g1 + g2 > 0)
    bwd::f32_to_bf16_kernel<<<(unsigned)(g0 + g1 + g2), (unsigned)threads, 0, st>>>(c);
  return check_launch("f32_to_bf16");
}

mt_status f32_to_bf16(const float* x, void* y, int64_t n, cudaStream_t st) {
  return f32_to_bf16_x3(x, y, n, nullptr, nullptr, 0, nullptr, nullptr, 0, st);
}

// One ring step of the backward: block part then bar part, accumulating into
// dq (local queries, fp32) and dk/dv (held chunk, fp32).
mt_status attn_bwd_step(const VSPlan& plan, int r, int s, int nloc, const void* q,
                        const void* k, const void* v, const void* dO, const float* lse,
                        const float* D, float* dq, float* dk, float* dv, int num_sms,
                        cudaStream_t st) {
  using namespace bwd;
  Params P{};
  P.plan = plan;
  P.r = r;
  P.s = s;
  P.t = ((r - s) % plan.W + plan.W) % plan.W;
  P.nloc = nloc;
  P.scale_log2 = 1.4426950408889634f / sqrtf(128.f);
  P.inv_sqrt_d = 1.f / sqrtf(128.f);
  P.k = static_cast<const __nv_bfloat16*>(k);
  P.v = static_cast<const __nv_bfloat16*>(v);
  P.lse = lse;
  P.dvec = D;
  P.dq = dq;
  P.dk = dk;
  P.dv = dv;
  P.tile_counter = plan.scratch + 2;
  static const int static_tiles = getenv("MT_BWD_STATIC") ? atoi(getenv("MT_BWD_STATIC")) : 0;
  P.static_tiles = static_tiles;
  static const int dbg = getenv("MT_BWD_DBG") ? atoi(getenv("MT_BWD_DBG")) : 0;
  P.dbg = dbg;
  // q heads per block-pass tile: 4 by default (MT_BWD_HPT overrides), the largest divisor
  // of the GQA group size not above it; block-CSR mode keeps one head per tile.  Measured
  // (profiles/r01_bwd_hpt_ab.json): the K/V load and dK/dV epilogue of a tile are shared by
  // 4 heads' chunk streams; 8 heads lose Q/dO locality in L2.
  static const int hpt_env = getenv("MT_BWD_HPT") ? atoi(getenv("MT_BWD_HPT")) : 4;
  const int grp = plan.Hq / plan.Hkv;
  int hpt = hpt_env < 1 ? 1 : hpt_env;
  while (grp % hpt) --hpt;
  P.hpt = (plan.bptr || plan.tptr) ? 1 : hpt;
  const uint64_t S_loc = (uint64_t)nloc * 64;
  CUtensorMap tmq, tmdo, tmk, tmv, tmdq, tmdk, tmdv;
  if (make_tmap_f32_3d(&tmdq, dq, 128, plan.Hq, S_loc, 128, 1, kTilePD >= 2 * kTileP ? 64 : 32) ||
      make_tmap_f32_3d(&tmdk, dk, 128, plan.Hkv, S_loc, 32, 1, 128, true) ||
      make_tmap_f32_3d(&tmdv, dv, 128, plan.Hkv, S_loc, 32, 1, 128, true) ||
      make_tmap_bf16_3d(&tmq, q, 128, plan.Hq, S_loc, 64, 1, 64) ||
      make_tmap_bf16_3d(&tmdo, dO, 128, plan.Hq, S_loc, 64, 1, 64) ||
      make_tmap_bf16_3d(&tmk, k, 128, plan.Hkv, S_loc, 64, 1, 64) ||
      make_tmap_bf16_3d(&tmv, v, 128, plan.Hkv, S_loc, 64, 1, 64))
    return fail(MT_ECUDA, "cuTensorMapEncodeTiled failed");
  const size_t smem = bwd_smem_bytes();
  // set on every launch: the attribute applies to the current device only (a process may
  // drive several GPUs), and the call is cheap next to the launch
  using KernelFn = void (*)(Params, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap,
                           CUtensorMap, CUtensorMap);
  KernelFn kernels[2][3] = {{attn_bwd_kernel<0, kOnlyBlock>, attn_bwd_kernel<0, kOnlyBar>,
                             attn_bwd_kernel<0, kMixed>},
                            {attn_bwd_kernel<1, kOnlyBlock>, attn_bwd_kernel<1, kOnlyBar>,
                             attn_bwd_kernel<1, kMixed>}};
  KernelFn* kl = kernels[plan.layout ? 1 : 0];
  for (int m = 0; m < 3; ++m)
    if (cudaFuncSetAttribute(kl[m], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return fail(MT_ECUDA, "cudaFuncSetAttribute(attn_bwd) failed");
  // BLOCK (slash) tiles and BAR (vertical) tiles share one dynamic tile counter per launch
  cudaMemsetAsync(P.tile_counter, 0, 2 * sizeof(int), st);
  const int npairs = (nloc + 1) / 2;
  // fewer heads per BLOCK tile when the launch would otherwise hold too few tiles to fill
  // the SMs (short sequences / many ring ranks)
  while (P.hpt > 1 && (plan.Hq / P.hpt) * npairs < 2 * num_sms) {
    int h2 = P.hpt - 1;
    while (grp % h2) --h2;
    P.hpt = h2;
  }
  P.n_block = (plan.Hq / P.hpt) * npairs;
  // bar (vertical) part (none in block-CSR mode): tile count bounded by
  // sum_h ceil(|i_v^(s)(h)| / 128) <= Hq * ceil(S/128); the exact count is read on device.
  // Query blocks per bar-tile part: 1024 (MT_BWD_BAR_PART overrides, so tests reach the
  // multi-part path at sizes the oracle checks in full); ranges of <= 1024 blocks are cut into
  // 4 parts of >= 16 blocks so a few long early-column tiles do not make the tail.
  static const int part_env = getenv("MT_BWD_BAR_PART") ? atoi(getenv("MT_BWD_BAR_PART")) : 0;
  int part_len = part_env > 0 ? part_env : 1024;
  if (part_env <= 0 && nloc <= 1024) part_len = nloc / 4 > 16 ? nloc / 4 : 16;
  P.bar_part_len = nloc < part_len ? (nloc > 0 ? nloc : 1) : part_len;
  P.bar_parts = (nloc + P.bar_part_len - 1) / P.bar_part_len;
  P.n_bar = plan.bptr ? 0 : plan.Hq * (int)((S_loc + 127) / 128) * P.bar_parts;
  P.n_tiles = P.n_block + P.n_bar;
  // Up to 2048 local blocks: ONE launch with the BAR tiles first (the longest first), so the
  // tail of one pass overlaps the other (4K: 0.25 -> 0.095 ms, 128K: 17.8 vs 18.1 ms).  Beyond:
  // a block-only launch, then a bar-only launch; their kernels compile without the other kind's
  // branches (a mixed kernel measured 4% slower on the 512K block pass, and with the bar tiles
  // first 298 vs 279 ms).  Ring steps (W > 1) split from 2048 local blocks on: 512K on 4 GPUs,
  // 74.1 -> 72.1 ms per backward (profiles/r02d_split4/).  MT_BWD_SPLIT=0/1 overrides.
  static const int split_env = getenv("MT_BWD_SPLIT") ? atoi(getenv("MT_BWD_SPLIT")) : -1;
  const bool split = P.n_bar > 0 && (split_env >= 0 ? split_env != 0 : (nloc > 2048 || (plan.W > 1 && nloc >= 2048)));
  if (split) {
    Params Pb = P, Pv = P;
    Pb.n_bar = 0;
    Pb.n_tiles = P.n_block;
    Pv.n_block = 0;
    Pv.n_tiles = P.n_bar;
    Pv.tile_counter = plan.scratch + 3;
    const int gb = Pb.n_tiles < num_sms ? Pb.n_tiles : num_sms;
    if (gb > 0) kl[kOnlyBlock]<<<gb, kThreads, smem, st>>>(Pb, tmq, tmdo, tmk, tmv, tmdq, tmdk, tmdv);
    MT_TRY(check_launch("attn_bwd_kernel(block)"));
    kl[kOnlyBar]<<<num_sms, kThreads, smem, st>>>(Pv, tmq, tmdo, tmk, tmv, tmdq, tmdk, tmdv);
    return check_launch("attn_bwd_kernel(bar)");
  }
  P.bar_first = 1;
  const int grid = P.n_tiles < num_sms ? P.n_tiles : num_sms;
  if (grid > 0) {
    if (P.n_bar > 0)
      kl[kMixed]<<<grid, kThreads, smem, st>>>(P, tmq, tmdo, tmk, tmv, tmdq, tmdk, tmdv);
    else  // block-CSR mode: block tiles only
      kl[kOnlyBlock]<<<grid, kThreads, smem, st>>>(P, tmq, tmdo, tmk, tmv, tmdq, tmdk, tmdv);
  }
  return check_launch("attn_bwd_kernel");
}

}  // namespace mt

extern "C" mt_status mt_debug_bwd_timeline(int64_t* out) {
  if (!out) return mt::fail(MT_ESHAPE, "NULL output");
  if (cudaMemcpyFromSymbol(out, mt::g_mt_tl, sizeof(mt::g_mt_tl)) != cudaSuccess)
    return mt::fail(MT_ECUDA, "cudaMemcpyFromSymbol(timeline) failed");
  return MT_OK;
}
