// rope.cu — rotary position embedding with optional YaRN scaling (SURVEY §8(f)
// f3: the step upstream of the path).  PAPER.md Appendix A: the
// half-split pairs (x[i], x[i + d/2]) of the vector at position n rotate by
// n * theta_i, theta_i = base^(-2i/d); YaRN, factor 32.  Readings (base,
// YaRN parametrisation): DESIGN.md R-rope.
//
// Memory-bound: one thread per (token, head, 8 pairs) moves 2 x 16 B.  Angles are
// formed in fp64 (n theta reaches ~5e5 rad at 512K, beyond fp32's resolution),
// reduced mod 2 pi, then sin/cos and the rotation run in fp32; output bf16.
#include <cuda_bf16.h>

#include <cmath>

#include "common.cuh"
#include "plan.cuh"
#include "rope.cuh"
#include "../../include/mtsa.h"

namespace mt {
namespace {

struct RopeParams {
  double theta[64];
  float mscale;
  int inverse;
  int64_t rows;  // local tokens
  int H, W, r;
  int layout, zc;  // rank layout of the rows (plan.cuh)
};

__global__ void rope_kernel(const __grid_constant__ RopeParams p, const __nv_bfloat16* src,
                            __nv_bfloat16* x) {
  const int64_t n_items = p.rows * p.H * 8;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < n_items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int gi = (int)(it & 7);
    const int64_t th = it >> 3;  // token * H + head
    const int64_t j = th / p.H;
    const int64_t pos = (int64_t)layout_l2g(p.layout, p.W, p.zc, p.r, (int)(j >> 6)) * 64 + (j & 63);
    __nv_bfloat16* v = x + th * 128;
    const __nv_bfloat16* vs = src + th * 128;
    uint4 lo = *reinterpret_cast<const uint4*>(vs + 8 * gi);
    uint4 hi = *reinterpret_cast<const uint4*>(vs + 64 + 8 * gi);
    __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(&lo);
    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&hi);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 a = __bfloat1622float2(l2[e]), b = __bfloat1622float2(h2[e]);
      float ra[2], rb[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = 8 * gi + 2 * e + u;
        float s, c;
        rope_sincos(pos, p.theta[i], &s, &c);  // rope.cuh: shared with the fused index
        if (p.inverse) s = -s;
        const float xl = u ? a.y : a.x, xh = u ? b.y : b.x;
        rope_rotate(xl, xh, s, c, p.mscale, &ra[u], &rb[u]);
      }
      l2[e] = __floats2bfloat162_rn(ra[0], ra[1]);
      h2[e] = __floats2bfloat162_rn(rb[0], rb[1]);
    }
    *reinterpret_cast<uint4*>(v + 8 * gi) = lo;
    *reinterpret_cast<uint4*>(v + 64 + 8 * gi) = hi;
  }
}

}  // namespace

// x_out = RoPE(x_in) on a rank's token-major [S/W][H][128] bf16 slice in `layout`
// (in place when x_out == x_in); used by mt_rope and the RoPE-fused index
mt_status rope_launch(const RopeArgs& ra, int inverse, int64_t seq_len, int world, int rank,
                      int layout, int n_heads, const void* x_in, void* x_out, cudaStream_t st) {
  RopeParams p{};
  for (int i = 0; i < 64; ++i) p.theta[i] = ra.theta[i];
  p.mscale = ra.mscale;
  p.inverse = inverse;
  p.rows = seq_len / world;
  p.H = n_heads;
  p.W = world;
  p.r = rank;
  p.layout = world > 1 ? layout : 0;
  p.zc = p.layout ? (int)(seq_len / 64 / (2 * world)) : 0;
  const int64_t n = p.rows * n_heads * 8;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  rope_kernel<<<(unsigned)blocks, 256, 0, st>>>(p, static_cast<const __nv_bfloat16*>(x_in),
                                               static_cast<__nv_bfloat16*>(x_out));
  return check_launch("rope_kernel");
}

}  // namespace mt

using namespace mt;

extern "C" mt_status mt_rope_inv_freq(int head_dim, double base, double yarn_factor,
                                      int64_t original_max_position, double* theta,
                                      float* mscale) {
  if (head_dim != 128 || !theta || !mscale || base <= 1.0 || yarn_factor < 1.0)
    return fail(MT_ESHAPE, "rope: head_dim must be 128, base > 1, factor >= 1");
  const int h = head_dim / 2;
  for (int i = 0; i < h; ++i) theta[i] = pow(base, -2.0 * i / head_dim);
  *mscale = 1.0f;
  if (yarn_factor == 1.0) return MT_OK;
  if (original_max_position <= 0) return fail(MT_ESHAPE, "rope: original_max_position <= 0");
  // NTK-by-parts: keep theta where the rotation count over the original context
  // exceeds beta_fast = 32, divide by the factor below beta_slow = 1, ramp between
  auto dim_of = [&](double beta) {
    return head_dim * log((double)original_max_position / (beta * 2.0 * M_PI)) / (2.0 * log(base));
  };
  double lo = floor(dim_of(32.0)), hi = ceil(dim_of(1.0));
  lo = lo < 0 ? 0 : lo;
  hi = hi > h - 1 ? h - 1 : hi;
  if (lo == hi) hi += 0.001;
  for (int i = 0; i < h; ++i) {
    double ramp = (i - lo) / (hi - lo);
    ramp = ramp < 0 ? 0 : (ramp > 1 ? 1 : ramp);
    theta[i] = theta[i] * (1.0 - ramp) + theta[i] / yarn_factor * ramp;
  }
  *mscale = (float)(0.1 * log(yarn_factor) + 1.0);
  return MT_OK;
}

extern "C" mt_status mt_rope(int64_t seq_len, int world, int rank, int n_heads,
                             const double* theta, float mscale, int inverse, void* x,
                             mt_stream_t stream) {
  if (!theta || !x || n_heads <= 0 || world <= 0 || rank < 0 || rank >= world)
    return fail(MT_ESHAPE, "rope: bad arguments");
  if (seq_len < 64 || seq_len % 64) return fail(MT_EWINDOW, "rope: seq_len must be a multiple of 64");
  if (seq_len % (64LL * world)) return fail(MT_ELAYOUT, "rope: seq_len %% (64 world) != 0");
  RopeArgs ra{};
  for (int i = 0; i < 64; ++i) ra.theta[i] = theta[i];
  ra.mscale = mscale;
  return rope_launch(ra, inverse, seq_len, world, rank, MT_LAYOUT_STRIPED, n_heads, x, x,
                     static_cast<cudaStream_t>(stream));
}
