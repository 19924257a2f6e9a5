// attn_fwd.cu — block-sparse vertical-slash attention forward for sm_100a,
// one ring step (Alg. 2 "block_bar_sparse_attention_forward" P:878
// followed by "merge_out_and_lse" P:879; on one GPU W = 1 and the single step
// is Alg. 1's "sparse(softmax(QK^T/sqrt d)V, i_vs)").
//
// Work unit (tile): 128 query rows = two 64-row slots = local query blocks
// (j0, j0+1) of ONE q head h (global blocks g0 = j0 W + r, g1 = g0 + W).  For the
// held KV chunk of origin s the tile visits, in one merged stream:
//   BLOCK chunks: local key block lb of every slash offset o = t (mod W) that
//                 either slot needs (kb = g - o), TMA-staged, 64 contiguous keys;
//   BAR chunks  : up to 64 gathered vertical columns of origin s that either
//                 slot needs and no selected slash covers (I9), cp.async-staged.
// Per chunk: S = Q K^T (tcgen05, M=128 N=64 K=128, fp32 in TMEM), online
// softmax in registers (one thread per row; per-slot masks, causal diagonal),
// P (bf16) -> smem, O += P V (tcgen05, M=128 N=128 K=64, O in TMEM).
//
// Warp roles (192 threads, 1 CTA/SM, persistent over tiles):
//   warp 0      producer: builds the chunk stream from the VSPlan, TMA/cp.async
//   warp 1      MMA issuer (one elected lane)
//   warps 2..5  softmax + epilogue (row = 32 * (warp % 4) + lane = TMEM lane)
#include "common.cuh"
#include "plan.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace mt {

namespace fwd {

constexpr int kStages = 4;
constexpr int kThreads = 192;
constexpr uint32_t kTileQ = 128 * 128 * 2;   // 32 KB
constexpr uint32_t kTileKV = 64 * 128 * 2;   // 16 KB
constexpr uint32_t kTileP = 128 * 64 * 2;    // 16 KB

enum : int { kBlock = 0, kBar = 1, kEnd = 2 };

struct ChunkMeta {
  int kind;
  int lb;            // local key block (kBlock)
  uint32_t flags;    // bit0/1: slot0/1 uses it; bit2/3: slot0/1 diagonal (kBlock)
  int pad;
  uint64_t mask[2];  // per-slot column masks (kBar)
  int rows[64];      // local key rows (kBar)
};

struct Smem {
  uint8_t q[kTileQ];
  uint8_t k[kStages][kTileKV];
  uint8_t v[kStages][kTileKV];
  uint8_t p[kTileP];
  ChunkMeta meta[kStages];
  ChunkMeta smeta[2];        // copy handed to the softmax per S buffer
  int stage_rows[128];       // producer staging for bar columns
  uint32_t stage_bits[128];
  uint64_t full[kStages], empty[kStages];
  uint64_t sfull[2], sfree[2];
  uint64_t qfull, qempty, pfull, pvdone;
  uint32_t tmem_base;
};

struct Params {
  VSPlan plan;
  int r, s, t;               // rank, origin of the held chunk, ring step (= (r - s) mod W)
  int nloc;                  // local query blocks = S_loc / 64
  int n_tiles;
  int first, last;           // merge mode
  float scale_log2;          // log2(e) / sqrt(d)
  const __nv_bfloat16* k;    // held chunk [S_loc][Hkv][128]
  const __nv_bfloat16* v;
  __nv_bfloat16* o;          // [S_loc][Hq][128]  (written when last)
  float* o_acc;              // [S_loc][Hq][128]  (ring accumulator when !last or !first)
  float* lse;                // [Hq][S_loc]       (running / final LSE, natural log)
};

__device__ __forceinline__ void tile_coords(const Params& P, int tile, int& h, int& j0) {
  const int npairs = (P.nloc + 1) / 2;
  const int pr = npairs - 1 - tile / P.plan.Hq;   // heavy (late) query blocks first
  h = tile % P.plan.Hq;
  j0 = 2 * pr;
}

// ------------------------------------------------------------------ producer
__device__ void producer(Smem& sm, const Params& P, const CUtensorMap* tmq,
                         const CUtensorMap* tmk, const CUtensorMap* tmv) {
  const int lane = lane_id();
  const VSPlan& pl = P.plan;
  const int W = pl.W;
  const int grp = pl.Hq / pl.Hkv;
  int stage = 0;
  uint32_t ephase = 0;  // phase parity of empty[] waits
  uint32_t qe_phase = 0;
  bool first_tile = true;

  auto next_stage = [&]() {
    if (++stage == kStages) { stage = 0; ephase ^= 1; }
  };
  auto acquire = [&]() { mbar_wait(smem_u32(&sm.empty[stage]), ephase ^ 1); };

  for (int tile = blockIdx.x; tile < P.n_tiles; tile += gridDim.x) {
    int h, j0;
    tile_coords(P, tile, h, j0);
    const int j1 = j0 + 1;
    const bool v1 = j1 < P.nloc;
    const int g0 = j0 * W + P.r;
    const int g1 = v1 ? j1 * W + P.r : -1;
    const int gkv = h / grp;

    // ---- Q tile (two 64-row slots x two 64-column chunks)
    if (!first_tile) {
      mbar_wait(smem_u32(&sm.qempty), qe_phase);
      qe_phase ^= 1;
    }
    first_tile = false;
    if (lane == 0) {
      const uint32_t bar = smem_u32(&sm.qfull);
      mbar_expect_tx(bar, v1 ? kTileQ : kTileQ / 2);
      for (int c = 0; c < 2; ++c) {
        tma_load_3d(smem_u32(sm.q + c * 16384), tmq, bar, c * 64, h, j0 * 64);
        if (v1) tma_load_3d(smem_u32(sm.q + c * 16384 + 8192), tmq, bar, c * 64, h, j1 * 64);
      }
    }

    // ---- slash blocks: offsets o = t (mod W); kb = g - o, merged over both slots
    {
      const int ns = pl.s_cnt[h];
      const int32_t* offs = pl.s_off + (int64_t)h * pl.s_stride;
      // walk candidates in ascending kb: slot1 kb = g1 - o, slot0 kb = g0 - o.
      // Both sequences are produced by walking offsets descending.
      int ia = ns - 1, ib = ns - 1;  // ia: slot0 pointer, ib: slot1 pointer
      auto next_valid = [&](int i, int g) {
        while (i >= 0) {
          const int o = offs[i];
          if (o <= g && (o % W) == P.t) break;
          --i;
        }
        return i;
      };
      ia = next_valid(ia, g0);
      ib = v1 ? next_valid(ib, g1) : -1;
      while (ia >= 0 || ib >= 0) {
        const int kba = ia >= 0 ? g0 - offs[ia] : INT32_MAX;
        const int kbb = ib >= 0 ? g1 - offs[ib] : INT32_MAX;
        const int kb = min(kba, kbb);
        uint32_t flags = 0;
        if (kba == kb) { flags |= 1u; if (kb == g0) flags |= 4u; ia = next_valid(ia - 1, g0); }
        if (kbb == kb) { flags |= 2u; if (kb == g1) flags |= 8u; ib = next_valid(ib - 1, g1); }
        const int lb = (kb - P.s) / W;
        acquire();
        if (lane == 0) {
          ChunkMeta& m = sm.meta[stage];
          m.kind = kBlock;
          m.lb = lb;
          m.flags = flags;
          const uint32_t bar = smem_u32(&sm.full[stage]);
          mbar_expect_tx(bar, 2 * kTileKV);
          for (int c = 0; c < 2; ++c) {
            tma_load_3d(smem_u32(sm.k[stage] + c * 8192), tmk, bar, c * 64, gkv, lb * 64);
            tma_load_3d(smem_u32(sm.v[stage] + c * 8192), tmv, bar, c * 64, gkv, lb * 64);
          }
        }
        __syncwarp();
        next_stage();
      }
    }

    // ---- bars: vertical columns of origin s, block < g, offset not a selected slash
    {
      const int32_t* vc = pl.vcol + (int64_t)h * pl.S;
      const int vb = pl.vptr[h * (W + 1) + P.s];
      const int ve = pl.vptr[h * (W + 1) + P.s + 1];
      const int glim = v1 ? g1 : g0;
      int nstaged = 0;  // columns staged in sm.stage_rows (warp-uniform)
      auto emit = [&](int n) {
        // emit the first n (<= 64) staged columns as one BAR chunk
        acquire();
        ChunkMeta& m = sm.meta[stage];
        uint32_t b0 = 0, c0 = 0;
        // lane l covers columns l and l + 32
        const int ca = lane, cb = lane + 32;
        int ra = sm.stage_rows[ca < n ? ca : 0];
        int rb = sm.stage_rows[cb < n ? cb : 0];
        if (ca < n) { b0 = sm.stage_bits[ca]; }
        if (cb < n) { c0 = sm.stage_bits[cb]; }
        m.rows[ca] = ra;
        m.rows[cb] = rb;
        const uint32_t lo0 = __ballot_sync(0xffffffffu, b0 & 1u);
        const uint32_t lo1 = __ballot_sync(0xffffffffu, (b0 >> 1) & 1u);
        const uint32_t hi0 = __ballot_sync(0xffffffffu, c0 & 1u);
        const uint32_t hi1 = __ballot_sync(0xffffffffu, (c0 >> 1) & 1u);
        if (lane == 0) {
          m.kind = kBar;
          m.mask[0] = (uint64_t)lo0 | ((uint64_t)hi0 << 32);
          m.mask[1] = (uint64_t)lo1 | ((uint64_t)hi1 << 32);
        }
        __syncwarp();
        // gather K/V rows: 64 rows x 16 pieces of 16 B each, for K and V
        const uint32_t kbase = smem_u32(sm.k[stage]), vbase = smem_u32(sm.v[stage]);
        for (int pidx = lane; pidx < 64 * 16; pidx += 32) {
          const int row = pidx >> 4, c16 = pidx & 15;
          const int src = m.rows[row];
          const size_t goff = ((size_t)src * pl.Hkv + gkv) * 128 + c16 * 8;
          const uint32_t doff = (c16 >> 3) * 8192 + sw128(row, c16 & 7);
          cp_async_16(kbase + doff, P.k + goff);
          cp_async_16(vbase + doff, P.v + goff);
        }
        const uint32_t bar = smem_u32(&sm.full[stage]);
        asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(bar);
        next_stage();
        // shift the remaining staged columns down
        const int rem = nstaged - n;
        __syncwarp();
        int tr0 = 0, tr1 = 0;
        uint32_t tb0 = 0, tb1 = 0;
        if (lane < rem) { tr0 = sm.stage_rows[n + lane]; tb0 = sm.stage_bits[n + lane]; }
        if (lane + 32 < rem) { tr1 = sm.stage_rows[n + lane + 32]; tb1 = sm.stage_bits[n + lane + 32]; }
        __syncwarp();
        if (lane < rem) { sm.stage_rows[lane] = tr0; sm.stage_bits[lane] = tb0; }
        if (lane + 32 < rem) { sm.stage_rows[lane + 32] = tr1; sm.stage_bits[lane + 32] = tb1; }
        __syncwarp();
        nstaged = rem;
      };
      for (int base = vb; base < ve; base += 32) {
        const int i = base + lane;
        int m = 0;
        bool in0 = false, in1 = false;
        bool more = false;
        if (i < ve) {
          m = vc[i];
          const int blk = m >> 6;
          if (blk < glim) {
            more = true;
            in0 = blk < g0 && !plan_has_slash(pl, h, g0 - blk);
            in1 = v1 && blk < g1 && !plan_has_slash(pl, h, g1 - blk);
          }
        }
        const bool keep = in0 || in1;
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        const int pos = __popc(bal & ((1u << lane) - 1u));
        if (keep) {
          const int blk = m >> 6;
          sm.stage_rows[nstaged + pos] = ((blk - P.s) / W) * 64 + (m & 63);
          sm.stage_bits[nstaged + pos] = (in0 ? 1u : 0u) | (in1 ? 2u : 0u);
        }
        __syncwarp();
        nstaged += __popc(bal);
        if (nstaged >= 64) emit(64);
        if (!__any_sync(0xffffffffu, more)) break;  // sorted: later columns are beyond glim
      }
      if (nstaged > 0) emit(nstaged);
    }

    // ---- END marker
    acquire();
    if (lane == 0) {
      sm.meta[stage].kind = kEnd;
      mbar_arrive(smem_u32(&sm.full[stage]));
    }
    __syncwarp();
    next_stage();
  }
}

// ------------------------------------------------------------------ MMA issuer
__device__ void mma_issuer(Smem& sm, const Params& P, uint32_t tmem) {
  const uint32_t idesc_s = make_idesc_bf16(128, 64, false, false);
  const uint32_t idesc_o = make_idesc_bf16(128, 128, false, true);
  const uint32_t tm_o = tmem;           // O: columns [0, 128)
  int stage = 0;
  uint32_t fphase = 0;
  int b = 0;
  uint32_t sfree_phase[2] = {0, 0};
  uint32_t pfull_phase = 0, qfull_phase = 0;
  const uint32_t q0 = smem_u32(sm.q), p0 = smem_u32(sm.p);

  for (int tile = blockIdx.x; tile < P.n_tiles; tile += gridDim.x) {
    mbar_wait(smem_u32(&sm.qfull), qfull_phase);
    qfull_phase ^= 1;
    tc_fence_after();
    bool have_prev = false, o_started = false;
    int prev_stage = 0;
    for (;;) {
      mbar_wait(smem_u32(&sm.full[stage]), fphase);
      const ChunkMeta& m = sm.meta[stage];
      const int kind = m.kind;
      if (kind == kBar) fence_proxy_async_smem();
      tc_fence_after();
      // S buffer b must be free (softmax done reading it)
      mbar_wait(smem_u32(&sm.sfree[b]), sfree_phase[b] ^ 1);
      sfree_phase[b] ^= 1;
      sm.smeta[b].kind = kind;
      sm.smeta[b].flags = m.flags;
      sm.smeta[b].mask[0] = m.mask[0];
      sm.smeta[b].mask[1] = m.mask[1];
      mbar_arrive(smem_u32(&sm.sfull[b]));  // 1st of 2 arrivals: publishes smeta[b]
      if (kind != kEnd) {
        const uint32_t kb0 = smem_u32(sm.k[stage]);
        const uint32_t tm_s = tmem + 128 + 64 * b;
#pragma unroll
        for (int kk = 0; kk < 128; kk += 16) {
          const uint64_t ad = make_sdesc(q0 + (kk >> 6) * 16384 + (kk & 63) * 2, 16, 1024);
          const uint64_t bd = make_sdesc(kb0 + (kk >> 6) * 8192 + (kk & 63) * 2, 16, 1024);
          mma_ss(tm_s, ad, bd, idesc_s, kk > 0);
        }
        mma_commit(smem_u32(&sm.sfull[b]));  // 2nd arrival: S ready
      } else {
        mma_commit(smem_u32(&sm.qempty));  // all S MMAs of this tile done -> Q reusable
      }
      // O += P(prev) V(prev)
      if (have_prev) {
        mbar_wait(smem_u32(&sm.pfull), pfull_phase);
        pfull_phase ^= 1;
        tc_fence_after();
        const uint32_t vb0 = smem_u32(sm.v[prev_stage]);
#pragma unroll
        for (int kk = 0; kk < 64; kk += 16) {
          const uint64_t ad = make_sdesc(p0 + kk * 2, 16, 1024);
          const uint64_t bd = make_sdesc(vb0 + kk * 128, 8192, 1024);
          mma_ss(tm_o, ad, bd, idesc_o, (o_started || kk > 0) ? 1u : 0u);
        }
        o_started = true;
        mma_commit(smem_u32(&sm.pvdone));
        mma_commit(smem_u32(&sm.empty[prev_stage]));
      }
      if (kind == kEnd) {
        mbar_arrive(smem_u32(&sm.empty[stage]));
        mbar_arrive(smem_u32(&sm.sfull[b]));
      }
      have_prev = (kind != kEnd);
      prev_stage = stage;
      b ^= 1;
      if (++stage == kStages) { stage = 0; fphase ^= 1; }
      if (kind == kEnd) break;
    }
  }
}

// ------------------------------------------------------------------ softmax + epilogue
__device__ void softmax_epilogue(Smem& sm, const Params& P, uint32_t tmem) {
  const int wq = warp_id() & 3;                 // TMEM lane quadrant
  const int row = wq * 32 + lane_id();          // tile row == TMEM lane
  const int slot = row >> 6, i = row & 63;
  const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
  const VSPlan& pl = P.plan;
  const int Hq = pl.Hq;
  const int64_t S_loc = (int64_t)P.nloc * 64;
  int b = 0;
  uint32_t sfull_phase[2] = {0, 0};
  uint32_t pv_waits = 0;
  const uint32_t prow = smem_u32(sm.p) + row * 128;

  for (int tile = blockIdx.x; tile < P.n_tiles; tile += gridDim.x) {
    int h, j0;
    tile_coords(P, tile, h, j0);
    const int jx = j0 + slot;
    const bool valid = jx < P.nloc;
    float m_run = -INFINITY, l_run = 0.f;
    int nchunks = 0;
    for (;;) {
      mbar_wait(smem_u32(&sm.sfull[b]), sfull_phase[b]);
      sfull_phase[b] ^= 1;
      const int kind = sm.smeta[b].kind;
      if (kind == kEnd) {
        mbar_arrive(smem_u32(&sm.sfree[b]));
        b ^= 1;
        break;
      }
      const uint32_t flags = sm.smeta[b].flags;
      const uint64_t cmask = sm.smeta[b].mask[slot];
      tc_fence_after();
      uint32_t sr[64];
      tmem_ld32(tmem + lane_base + 128 + 64 * b, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
      tmem_ld32(tmem + lane_base + 128 + 64 * b + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(smem_u32(&sm.sfree[b]));
      // masks
      bool use;
      uint64_t vis;  // visible columns of this row
      if (kind == kBlock) {
        use = (flags >> slot) & 1u;
        const bool diag = (flags >> (2 + slot)) & 1u;
        vis = diag ? ((i == 63) ? ~0ull : ((2ull << i) - 1ull)) : ~0ull;
      } else {
        vis = cmask;
        use = true;
      }
      if (!use || !valid) vis = 0ull;
      float x[64];
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 64; ++c) {
        x[c] = ((vis >> c) & 1ull) ? __uint_as_float(sr[c]) * P.scale_log2 : -INFINITY;
        mx = fmaxf(mx, x[c]);
      }
      // conditional rescale: move the stabiliser only when the max grew by > 8 (log2)
      float alpha = 1.f;
      bool resc = false;
      if (mx > m_run + 8.f || (m_run == -INFINITY && mx > -INFINITY)) {
        const float m_new = mx;
        alpha = (m_run == -INFINITY) ? 0.f : exp2f(m_run - m_new);
        resc = (m_run != -INFINITY);
        m_run = m_new;
      }
      float lsum = 0.f;
      uint32_t pk[32];
#pragma unroll
      for (int c = 0; c < 64; c += 2) {
        const float p0 = (x[c] == -INFINITY) ? 0.f : exp2f(x[c] - m_run);
        const float p1 = (x[c + 1] == -INFINITY) ? 0.f : exp2f(x[c + 1] - m_run);
        lsum += p0 + p1;
        pk[c >> 1] = pack_bf16x2(p0, p1);
      }
      l_run = l_run * alpha + lsum;
      // previous PV must be complete: P buffer free, O stable
      if (nchunks > 0) {
        mbar_wait(smem_u32(&sm.pvdone), pv_waits & 1);
        ++pv_waits;
        tc_fence_after();
        if (__any_sync(0xffffffffu, resc)) {
          const float a = resc ? alpha : 1.f;
#pragma unroll 1
          for (int c0 = 0; c0 < 128; c0 += 32) {
            uint32_t o[32];
            tmem_ld32(tmem + lane_base + c0, o);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * a);
            tmem_st32(tmem + lane_base + c0, o);
          }
          tmem_st_wait();
        }
      }
      // P row -> smem (K-major SW128: 8 x 16-byte pieces)
#pragma unroll
      for (int c16 = 0; c16 < 8; ++c16) {
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(prow + ((c16 ^ (row & 7)) << 4)),
                     "r"(pk[4 * c16]), "r"(pk[4 * c16 + 1]), "r"(pk[4 * c16 + 2]),
                     "r"(pk[4 * c16 + 3])
                     : "memory");
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(smem_u32(&sm.pfull));
      ++nchunks;
      b ^= 1;
    }

    // ---- epilogue: O' = O / l, LSE' = (m + log2 l) ln 2; merge into the running result
    float inv_l = 0.f, lse_new = -INFINITY;
    if (nchunks > 0) {
      mbar_wait(smem_u32(&sm.pvdone), pv_waits & 1);
      ++pv_waits;
      tc_fence_after();
    }
    if (l_run > 0.f) {
      inv_l = 1.f / l_run;
      lse_new = (m_run + __log2f(l_run)) * 0.69314718055994531f;
    }
    const int64_t tok = (int64_t)jx * 64 + i;
    float* lse_p = valid ? P.lse + (int64_t)h * S_loc + tok : nullptr;
    float lse_old = -INFINITY;
    if (!P.first && valid) lse_old = *lse_p;
    const float lse_m = fmaxf(lse_old, lse_new);
    float w_old = 0.f, w_new = 0.f, lse_out = -INFINITY;
    if (lse_m > -INFINITY) {
      const float eo = (lse_old == -INFINITY) ? 0.f : __expf(lse_old - lse_m);
      const float en = (lse_new == -INFINITY) ? 0.f : __expf(lse_new - lse_m);
      const float tot = eo + en;
      lse_out = lse_m + __logf(tot);
      w_old = eo / tot;
      w_new = en / tot * inv_l;
    }
    const size_t obase = ((size_t)tok * Hq + h) * 128;
#pragma unroll 1
    for (int c0 = 0; c0 < 128; c0 += 32) {
      uint32_t o[32];
      if (nchunks > 0) {
        tmem_ld32(tmem + lane_base + c0, o);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) o[c] = 0u;
      }
      if (!valid) continue;
      float res[32];
      if (!P.first) {
        const float4* src = reinterpret_cast<const float4*>(P.o_acc + obase + c0);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float4 a = src[c];
          res[4 * c] = a.x * w_old;
          res[4 * c + 1] = a.y * w_old;
          res[4 * c + 2] = a.z * w_old;
          res[4 * c + 3] = a.w * w_old;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) res[c] = 0.f;
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) res[c] += __uint_as_float(o[c]) * w_new;
      if (P.last) {
        uint4* dst = reinterpret_cast<uint4*>(P.o + obase + c0);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          dst[c] = make_uint4(pack_bf16x2(res[8 * c], res[8 * c + 1]),
                              pack_bf16x2(res[8 * c + 2], res[8 * c + 3]),
                              pack_bf16x2(res[8 * c + 4], res[8 * c + 5]),
                              pack_bf16x2(res[8 * c + 6], res[8 * c + 7]));
      } else {
        float4* dst = reinterpret_cast<float4*>(P.o_acc + obase + c0);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          dst[c] = make_float4(res[4 * c], res[4 * c + 1], res[4 * c + 2], res[4 * c + 3]);
      }
    }
    if (valid) *lse_p = lse_out;
    tc_fence_before();
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ Params P, const __grid_constant__ CUtensorMap tmq,
                    const __grid_constant__ CUtensorMap tmk,
                    const __grid_constant__ CUtensorMap tmv) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~uintptr_t(1023));
  const int warp = warp_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(smem_u32(&sm.full[s]), 1);
      mbar_init(smem_u32(&sm.empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&sm.sfull[b]), 2);
      mbar_init(smem_u32(&sm.sfree[b]), 128);
    }
    mbar_init(smem_u32(&sm.qfull), 1);
    mbar_init(smem_u32(&sm.qempty), 1);
    mbar_init(smem_u32(&sm.pfull), 128);
    mbar_init(smem_u32(&sm.pvdone), 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(smem_u32(&sm.tmem_base), 256);
  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tmq);
    tma_prefetch_desc(&tmk);
    tma_prefetch_desc(&tmv);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    producer(sm, P, &tmq, &tmk, &tmv);
  } else if (warp == 1) {
    if (lane_id() == 0) mma_issuer(sm, P, tmem);
    __syncwarp();
  } else {
    softmax_epilogue(sm, P, tmem);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 256);
}

}  // namespace fwd

size_t fwd_smem_bytes() { return sizeof(fwd::Smem) + 1024; }

// One ring step of the forward (or the whole forward when W = 1).
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
  P.n_tiles = plan.Hq * ((nloc + 1) / 2);
  P.first = first;
  P.last = last;
  P.scale_log2 = 1.4426950408889634f / sqrtf(128.f);
  P.k = static_cast<const __nv_bfloat16*>(k);
  P.v = static_cast<const __nv_bfloat16*>(v);
  P.o = static_cast<__nv_bfloat16*>(o);
  P.o_acc = o_acc;
  P.lse = lse;
  const uint64_t S_loc = (uint64_t)nloc * 64;
  CUtensorMap tmq, tmk, tmv;
  if (make_tmap_bf16_3d(&tmq, q, 128, plan.Hq, S_loc, 64, 1, 64) ||
      make_tmap_bf16_3d(&tmk, k, 128, plan.Hkv, S_loc, 64, 1, 64) ||
      make_tmap_bf16_3d(&tmv, v, 128, plan.Hkv, S_loc, 64, 1, 64))
    return fail(MT_ECUDA, "cuTensorMapEncodeTiled failed");
  const size_t smem = fwd_smem_bytes();
  static bool attr_done = false;
  if (!attr_done) {
    if (cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return fail(MT_ECUDA, "cudaFuncSetAttribute(attn_fwd) failed");
    attr_done = true;
  }
  const int grid = P.n_tiles < num_sms ? P.n_tiles : num_sms;
  if (grid > 0) attn_fwd_kernel<<<grid, kThreads, smem, st>>>(P, tmq, tmk, tmv);
  return check_launch("attn_fwd_kernel");
}

}  // namespace mt
