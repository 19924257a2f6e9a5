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
#include "../../include/mtsa.h"

namespace mt {
namespace {

struct RopeParams {
  double theta[64];
  float mscale;
  int inverse;
  int64_t rows;  // local tokens
  int H, W, r;
};

__global__ void rope_kernel(const __grid_constant__ RopeParams p, __nv_bfloat16* x) {
  const int64_t n_items = p.rows * p.H * 8;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < n_items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int gi = (int)(it & 7);
    const int64_t th = it >> 3;  // token * H + head
    const int64_t j = th / p.H;
    const int64_t pos = ((j >> 6) * p.W + p.r) * 64 + (j & 63);  // block-striped global position
    __nv_bfloat16* v = x + th * 128;
    uint4 lo = *reinterpret_cast<const uint4*>(v + 8 * gi);
    uint4 hi = *reinterpret_cast<const uint4*>(v + 64 + 8 * gi);
    __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(&lo);
    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&hi);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 a = __bfloat1622float2(l2[e]), b = __bfloat1622float2(h2[e]);
      float ra[2], rb[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = 8 * gi + 2 * e + u;
        double ang = (double)pos * p.theta[i];
        ang -= floor(ang * 0.15915494309189535) * 6.283185307179586;  // mod 2 pi
        float s, c;
        sincosf((float)ang, &s, &c);
        if (p.inverse) s = -s;
        const float xl = u ? a.y : a.x, xh = u ? b.y : b.x;
        ra[u] = p.mscale * (xl * c - xh * s);
        rb[u] = p.mscale * (xh * c + xl * s);
      }
      l2[e] = __floats2bfloat162_rn(ra[0], ra[1]);
      h2[e] = __floats2bfloat162_rn(rb[0], rb[1]);
    }
    *reinterpret_cast<uint4*>(v + 8 * gi) = lo;
    *reinterpret_cast<uint4*>(v + 64 + 8 * gi) = hi;
  }
}

}  // namespace
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
  RopeParams p{};
  for (int i = 0; i < 64; ++i) p.theta[i] = theta[i];
  p.mscale = mscale;
  p.inverse = inverse;
  p.rows = seq_len / world;
  p.H = n_heads;
  p.W = world;
  p.r = rank;
  const int64_t n = p.rows * n_heads * 8;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  rope_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      p, static_cast<__nv_bfloat16*>(x));
  return check_launch("rope_kernel");
}
