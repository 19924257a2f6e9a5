// rope.cuh — the rotary embedding arithmetic shared by mt_rope (rope.cu) and the
// RoPE-fused index builder (vs_index.cu), so both produce the same bf16 values bit for
// bit.  PAPER.md Appendix A: the half-split pair (x_i, x_{i+d/2}) at position
// n rotates by n theta_i.  Every operation is one explicitly rounded IEEE op (no FMA
// contraction): the angle in fp64 reduced mod 2 pi, sin/cos in fp32, the rotation and
// the YaRN scale in fp32; the caller rounds to bf16 once.
#pragma once
#include <cstdint>

namespace mt {

struct RopeArgs {
  double theta[64];  // theta_i, i < d/2 (mt_rope_inv_freq)
  float mscale;      // YaRN attention scale (1 without YaRN)
};

__device__ __forceinline__ void rope_sincos(int64_t pos, double theta, float* s, float* c) {
  double ang = __dmul_rn((double)pos, theta);
  ang = __dsub_rn(ang, __dmul_rn(floor(__dmul_rn(ang, 0.15915494309189535)), 6.283185307179586));
  sincosf((float)ang, s, c);
}

// (yl, yh) = mscale R(angle) (xl, xh); s -> -s gives the inverse rotation
__device__ __forceinline__ void rope_rotate(float xl, float xh, float s, float c, float mscale,
                                            float* yl, float* yh) {
  *yl = __fmul_rn(mscale, __fsub_rn(__fmul_rn(xl, c), __fmul_rn(xh, s)));
  *yh = __fmul_rn(mscale, __fadd_rn(__fmul_rn(xh, c), __fmul_rn(xl, s)));
}

}  // namespace mt
