/* _vsidx_ref.c — VS-IDX v1 steps I1-I6 in plain C (oracle fast path).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Same arithmetic as
 * oracle/vsidx.py (window_scores, window_stats, column_and_slash_scores),
 * written out loop by loop so it can be read against PAPER.md Alg. 1
 * and DESIGN.md §2.1.  Compile with -ffp-contract=off and without fast-math:
 * every float operation below is one IEEE binary32 round-to-nearest-even op,
 * except I1's fused multiply-add, written as (float)((double)acc + (double)q *
 * (double)k): the bf16 x bf16 product is exact in double and the double sum is
 * either exact or too far from a float rounding boundary for the second
 * rounding to matter (R11), so it equals fmaf(q, k, acc).
 *
 *   I1 t[i,m] = fold_c RN(acc + q[i,c]*k[m,c])   (fused: the product is not rounded)
 *   I2 M_i = max over causal m (m <= n_i = S-nq+i)
 *   I3 e = exp2s(RN(RN(t - M_i) * C_d))
 *   I4 E_i = sum floor(e * 2^31)
 *   I5 l_i = RN((float)E_i) * 2^-31 ; p = RN(e / l_i) ; w = floor(p * 2^32)
 *   I6 V_m = sum_i w[i,m]
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static const uint32_t EXP2_COEF_BITS[8] = {0x3F800000u, 0x3F317218u, 0x3E75FDF0u, 0x3D635847u,
                                           0x3C1D955Bu, 0x3AAEC3FFu, 0x39218489u, 0x377FE5FEu};

static float f32_bits(uint32_t b) {
  float f;
  memcpy(&f, &b, 4);
  return f;
}

/* I3: specified 2^y, y <= 0. */
static float exp2s(float y, const float* c) {
  if (!(y >= -125.0f)) return 0.0f;
  float j = rintf(y); /* default rounding mode: nearest, ties to even */
  float f = y - j;    /* exact */
  float p = c[7];
  for (int k = 6; k >= 0; --k) {
    p = p * f;
    p = p + c[k];
  }
  return ldexpf(p, (int)j);
}

/* V[m] for one head.  q: [nq][d], k: [S][d] (float32 holding bf16 values). */
int vsidx_ref_column_scores(const float* q, const float* k, int64_t S, int d, int nq,
                            uint32_t cd_bits, uint64_t* V) {
  float c[8];
  for (int i = 0; i < 8; ++i) c[i] = f32_bits(EXP2_COEF_BITS[i]);
  const float Cd = f32_bits(cd_bits);
  float* t = (float*)malloc((size_t)nq * (size_t)S * sizeof(float));
  if (!t) return 1;
  float M[256];
  uint64_t E[256];
  float l[256];
  if (nq > 256) {
    free(t);
    return 2;
  }

  /* I1 + I2.  kT = k transposed to [d][S] so the inner loop runs over m: every
   * m keeps its own sequential fold over channels (same bits as the plain
   * per-(i,m) loop; the loop order only lets the compiler vectorise across m). */
  float* kT = (float*)malloc((size_t)d * (size_t)S * sizeof(float));
  if (!kT) {
    free(t);
    return 1;
  }
#pragma omp parallel for schedule(static)
  for (int64_t m = 0; m < S; ++m)
    for (int ch = 0; ch < d; ++ch) kT[(size_t)ch * S + m] = k[(size_t)m * d + ch];
  for (int i = 0; i < nq; ++i) {
    const int64_t n = S - nq + i;
    float* ti = t + (size_t)i * S;
    float mx = -INFINITY;
#pragma omp parallel reduction(max : mx)
    {
#pragma omp for schedule(static)
      for (int64_t m0 = 0; m0 <= n; m0 += 1024) {
        const int64_t m1 = (m0 + 1024 <= n + 1) ? m0 + 1024 : n + 1;
        for (int64_t m = m0; m < m1; ++m) ti[m] = 0.0f;
        for (int ch = 0; ch < d; ++ch) {
          const float qc = q[(size_t)i * d + ch];
          const float* kc = kT + (size_t)ch * S;
          for (int64_t m = m0; m < m1; ++m) {
            ti[m] = (float)((double)ti[m] + (double)qc * (double)kc[m]);
          }
        }
        for (int64_t m = m0; m < m1; ++m)
          if (ti[m] > mx) mx = ti[m];
      }
    }
    M[i] = mx;
  }
  free(kT);
  /* I3 + I4 (uint64 sums: exact under any order) */
  for (int i = 0; i < nq; ++i) {
    const int64_t n = S - nq + i;
    uint64_t Ei = 0;
#pragma omp parallel for reduction(+ : Ei) schedule(static)
    for (int64_t m = 0; m <= n; ++m) {
      float y = t[(size_t)i * S + m] - M[i];
      y = y * Cd;
      float e = exp2s(y, c);
      t[(size_t)i * S + m] = e;
      Ei += (uint64_t)floor((double)(e * 2147483648.0f));
    }
    E[i] = Ei;
    l[i] = ((float)(int64_t)Ei) * f32_bits(0x30000000u); /* 2^-31 */
  }
  /* I5 + I6 */
#pragma omp parallel for schedule(static)
  for (int64_t m = 0; m < S; ++m) {
    uint64_t acc = 0;
    for (int i = 0; i < nq; ++i) {
      const int64_t n = S - nq + i;
      if (m > n) continue;
      float p = t[(size_t)i * S + m] / l[i];
      acc += (uint64_t)floor((double)(p * 4294967296.0f));
    }
    V[m] = acc;
  }
  free(t);
  return 0;
}
