// scan.cuh -- exclusive prefix sum over u32 (reduce-then-scan, 3 launches).
#pragma once
#include "common.cuh"

namespace tpx {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096

// Block-wide exclusive scan of one value per thread; returns the prefix and
// writes the block total to *total.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t warp_sums[kScanThreads / 32];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= (unsigned)o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t s = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(kFull, s, o);
      if (lane >= (unsigned)o) s += y;
    }
    if (lane < kScanThreads / 32) warp_sums[lane] = s;
  }
  __syncthreads();
  uint32_t warp_prefix = warp ? warp_sums[warp - 1] : 0;
  *total = warp_sums[kScanThreads / 32 - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t* __restrict__ in, uint64_t n,
                                                              uint32_t* __restrict__ partials) {
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  uint32_t s = 0;
#pragma unroll
  for (int r = 0; r < kScanItems; ++r) {
    uint64_t i = base + (uint64_t)r * kScanThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  uint32_t total;
  block_exclusive_scan(s, &total);
  if (threadIdx.x == 0) partials[blockIdx.x] = total;
}

// Single block: exclusive scan of the tile partials in place, total -> *out_total.
__global__ void __launch_bounds__(kScanThreads) k_scan_partials(uint32_t* partials, uint32_t n_tiles,
                                                               uint32_t* out_total) {
  uint32_t carry = 0;
  for (uint32_t base = 0; base < n_tiles; base += kScanThreads) {
    uint32_t i = base + threadIdx.x;
    uint32_t v = i < n_tiles ? partials[i] : 0;
    uint32_t total;
    uint32_t ex = block_exclusive_scan(v, &total);
    if (i < n_tiles) partials[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0 && out_total) *out_total = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(const uint32_t* __restrict__ in, uint64_t n,
                                                           const uint32_t* __restrict__ partials,
                                                           uint32_t* __restrict__ out) {
  __shared__ uint32_t tile[kScanTile];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
#pragma unroll
  for (int r = 0; r < kScanItems; ++r) {
    uint64_t i = base + (uint64_t)r * kScanThreads + threadIdx.x;
    tile[r * kScanThreads + threadIdx.x] = i < n ? in[i] : 0;
  }
  __syncthreads();
  uint32_t local[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    // blocked ownership with a skewed index to avoid bank conflicts
    local[k] = tile[threadIdx.x * kScanItems + k];
    s += local[k];
  }
  uint32_t total;
  uint32_t ex = block_exclusive_scan(s, &total) + partials[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    tile[threadIdx.x * kScanItems + k] = ex;
    ex += local[k];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kScanItems; ++r) {
    uint64_t i = base + (uint64_t)r * kScanThreads + threadIdx.x;
    if (i < n) out[i] = tile[r * kScanThreads + threadIdx.x];
  }
}

}  // namespace tpx
