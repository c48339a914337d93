// Block-wide exclusive scan of small integers (blockDim.x <= 1024, multiple of 32).
#pragma once
#include <cuda_runtime.h>

namespace hdr {

// Returns the exclusive prefix of v over the block; *total = block sum.
// `scratch` must hold 32 ints. Contains __syncthreads(): call uniformly.
__device__ __forceinline__ int block_exclusive_scan(int v, int* scratch, int* total) {
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int nwarps = (blockDim.x + 31) >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int y = __shfl_up_sync(0xffffffff, x, off);
    if (lane >= off) x += y;
  }
  __syncthreads();  // scratch may still be read by a previous call
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int s = lane < nwarps ? scratch[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int y = __shfl_up_sync(0xffffffff, s, off);
      if (lane >= off) s += y;
    }
    if (lane < nwarps) scratch[lane] = s;
  }
  __syncthreads();
  int warp_base = warp ? scratch[warp - 1] : 0;
  *total = scratch[nwarps - 1];
  return warp_base + x - v;
}

}  // namespace hdr
