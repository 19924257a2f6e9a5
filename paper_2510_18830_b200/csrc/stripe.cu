// stripe.cu — layout copies global <-> rank-local: block-striped (
// SURVEY §8 a1) and zigzag (Fig. 1, the f1 ablation; plan.cuh layouts).
// A 64-token block is contiguous in both layouts, so the copy is a gather of
// nloc contiguous segments of 64 * row_bytes bytes: one 16-byte vector per
// thread, grid-stride, coalesced on both sides (HBM-bound).
#include "common.cuh"
#include "plan.cuh"
#include "../../include/mtsa.h"

namespace mt {
namespace {

// dir 0: local <- global (stripe); dir 1: global <- local (unstripe)
__global__ void stripe_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                              int64_t nloc, int64_t seg16, int W, int r, int dir, int layout,
                              int zc) {
  const int64_t total = nloc * seg16;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lb = i / seg16, o = i - lb * seg16;
    const int64_t g = (int64_t)layout_l2g(layout, W, zc, r, (int)lb) * seg16 + o;  // global
    if (dir == 0)
      dst[i] = src[g];
    else
      dst[g] = src[i];
  }
}

mt_status stripe_copy(int layout, int64_t S, int64_t row_bytes, int W, int r, const void* src,
                      void* dst, int dir, cudaStream_t st) {
  if (!src || !dst || row_bytes <= 0 || row_bytes % 16 || W <= 0 || r < 0 || r >= W)
    return fail(MT_ESHAPE, "stripe: bad pointer/row_bytes/rank");
  if (layout != MT_LAYOUT_STRIPED && layout != MT_LAYOUT_ZIGZAG)
    return fail(MT_ESHAPE, "stripe: unknown layout %d", layout);
  if (S < 64 || S % 64) return fail(MT_EWINDOW, "stripe: S=%lld not a positive multiple of 64", (long long)S);
  if (S % (64LL * W)) return fail(MT_ELAYOUT, "stripe: S %% (64 W) != 0");
  if (layout == MT_LAYOUT_ZIGZAG && S % (128LL * W)) return fail(MT_ELAYOUT, "zigzag: S %% (128 W) != 0");
  const int zc = layout == MT_LAYOUT_ZIGZAG ? (int)(S / 64 / (2 * W)) : 0;
  const int64_t nloc = S / 64 / W, seg16 = 64 * row_bytes / 16;
  const int64_t total = nloc * seg16;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 512;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  if (blocks < 1) blocks = 1;
  stripe_kernel<<<(unsigned)blocks, threads, 0, st>>>(static_cast<const uint4*>(src),
                                                       static_cast<uint4*>(dst), nloc, seg16, W, r,
                                                       dir, layout, zc);
  return check_launch("stripe_kernel");
}

}  // namespace
}  // namespace mt

extern "C" mt_status mt_stripe(int64_t seq_len, int64_t row_bytes, int world, int rank,
                               const void* global, void* local, mt_stream_t stream) {
  return mt::stripe_copy(MT_LAYOUT_STRIPED, seq_len, row_bytes, world, rank, global, local, 0,
                         static_cast<cudaStream_t>(stream));
}

extern "C" mt_status mt_unstripe(int64_t seq_len, int64_t row_bytes, int world, int rank,
                                 const void* local, void* global, mt_stream_t stream) {
  return mt::stripe_copy(MT_LAYOUT_STRIPED, seq_len, row_bytes, world, rank, local, global, 1,
                         static_cast<cudaStream_t>(stream));
}

extern "C" mt_status mt_layout_to_local(int layout, int64_t seq_len, int64_t row_bytes, int world,
                                        int rank, const void* global, void* local,
                                        mt_stream_t stream) {
  return mt::stripe_copy(layout, seq_len, row_bytes, world, rank, global, local, 0,
                         static_cast<cudaStream_t>(stream));
}

extern "C" mt_status mt_layout_to_global(int layout, int64_t seq_len, int64_t row_bytes,
                                         int world, int rank, const void* local, void* global,
                                         mt_stream_t stream) {
  return mt::stripe_copy(layout, seq_len, row_bytes, world, rank, local, global, 1,
                         static_cast<cudaStream_t>(stream));
}
