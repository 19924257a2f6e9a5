// tmap.cuh — host-side TMA tensor-map construction through the driver entry
// point (no -lcuda link needed).  Used by every kernel that stages tiles by TMA.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace mt {

// Encode a rank-3 bf16 tensor map over a token-major [n2][n1][n0] array
// (n0 innermost, contiguous).  Box = {b0, b1, b2}; SWIZZLE_128B (b0*2 must be 128).
// Returns 0 on success.
int make_tmap_bf16_3d(CUtensorMap* out, const void* base, uint64_t n0, uint64_t n1, uint64_t n2,
                      uint32_t b0, uint32_t b1, uint32_t b2);
// Rank-3 fp32 map over a token-major [n2][n1][n0] array (used as the destination
// of bulk tensor reduce-adds).  Box = {b0, b1, b2}; swizzle128 needs b0 * 4 == 128.
int make_tmap_f32_3d(CUtensorMap* out, const void* base, uint64_t n0, uint64_t n1, uint64_t n2,
                     uint32_t b0, uint32_t b1, uint32_t b2, bool swizzle128 = false);
// Rank-2 bf16 map over [n1][n0] with row pitch `pitch_bytes`.
int make_tmap_bf16_2d(CUtensorMap* out, const void* base, uint64_t n0, uint64_t n1,
                      uint64_t pitch_bytes, uint32_t b0, uint32_t b1);

}  // namespace mt
