// Device helpers shared by the bank kernels (internal).
#pragma once
#include "common.cuh"

namespace casc {


template <int MS>
struct TmemCols {
  static constexpr int value = MS < 32 ? 32 : MS;
};

// Warp-private staged store of the warp's 32 consecutive rows (32 x MS fp32, contiguous in
// global): lane r deposits row r in an XOR-swizzled 8 KB smem slab, then the warp writes the
// slab out as 512-byte coalesced runs. `stage` points at this warp's slab (32*MS floats).
template <int MS>
__device__ __forceinline__ void warp_store_rows(float* stage, const float* v, float* gdst, int lane,
                                                int valid_rows) {
  constexpr int CH = MS / 4;                      // 16-byte chunks per row
#pragma unroll
  for (int j = 0; j < CH; ++j)
    *reinterpret_cast<float4*>(stage + lane * MS + ((j ^ (lane % CH)) * 4)) =
        make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  __syncwarp();
  constexpr int ROWS_PER_IT = 32 / CH;            // rows covered by one 32-lane sweep
#pragma unroll
  for (int it = 0; it < 32 / ROWS_PER_IT; ++it) {
    const int r = it * ROWS_PER_IT + lane / CH, j = lane % CH;
    if (r < valid_rows)
      *reinterpret_cast<float4*>(gdst + r * MS + j * 4) =
          *reinterpret_cast<const float4*>(stage + r * MS + ((j ^ (r % CH)) * 4));
  }
  __syncwarp();
}

}  // namespace casc
