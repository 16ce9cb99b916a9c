// group.cuh -- cluster-contiguous output and shape records.
//
// Alg. "High-level GPU clustering" Step 6 (§4 l.175): "Sort clusters
// by their minimum time of arrival, causing the hits from the same cluster to
// form adjacent memory blocks".  Reading R18: a cluster's place is that of its
// earliest hit in the (toa, input index) order -- the sorted stream S the run
// already holds -- and inside a block the hits keep that order.  The block
// order is therefore a stable sort of S by the rank of each hit's cluster:
//
//   G0  root bits  bit i = (labels[i] == i); popc + scan -> ordinal(label)
//   G1  first[c]   = min sorted position of cluster c (atomicMin), cpos[p] = c
//   G2  first bits bit first[c]; popc + scan -> grank[c] = block index of c
//   G3  block table cluster_of[g], sizes -> offsets (scan)
//   G4  keys       (grank[cpos[p]], S[p].idx) in S order, then a stable LSD
//                  radix sort on ceil(log2 k) bits (sort.cuh) -> order
//   G5  shapes     bounding box (§3.3 l.132) and second moments
//                  (reading R19), one segmented pass over the blocks.
#pragma once
#include "common.cuh"
#include "sort.cuh"

namespace tpx {

// Same 32-byte layout as tpx_cluster_shape (include/tpx_cluster.h).
struct shape_rec {
  uint16_t x_min, x_max, y_min, y_max;
  unsigned long long sum_xx, sum_xy, sum_yy;
};
static_assert(sizeof(shape_rec) == 32, "shape record");

// G0: one thread per 32 labels -> one bitmap word (no atomics).
__global__ void k_root_bits(const uint32_t* __restrict__ labels, uint64_t n, uint32_t* __restrict__ bits) {
  const uint64_t nwords = (n + 31) / 32;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t b = 0;
    const uint64_t i0 = w * 32;
    const uint32_t cnt = (uint32_t)min((uint64_t)32, n - i0);
    for (uint32_t k = 0; k < cnt; ++k) b |= (uint32_t)(labels[i0 + k] == (uint32_t)(i0 + k)) << k;
    bits[w] = b;
  }
}

__device__ __forceinline__ uint32_t bit_rank(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ wbase,
                                             uint32_t i) {
  const uint32_t w = i >> 5;
  return wbase[w] + __popc(bits[w] & ((1u << (i & 31)) - 1u));
}

// G1: cluster ordinal of every sorted position and each cluster's first one.
__global__ void k_group_first(const srec* __restrict__ S, uint64_t n, const uint32_t* __restrict__ labels,
                              const uint32_t* __restrict__ rbits, const uint32_t* __restrict__ rbase,
                              uint32_t* __restrict__ cpos, uint32_t* __restrict__ first) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t idx = S[p].idx;
    const uint32_t c = bit_rank(rbits, rbase, labels[idx]);
    cpos[p] = c;
    atomicMin(first + c, (uint32_t)p);
  }
}

// G1 when the tile path recorded each cluster's first sorted position:
// cluster ordinal per sorted position (no atomics) ...
__global__ void k_group_cpos(const srec* __restrict__ S, uint64_t n, const uint32_t* __restrict__ labels,
                             const uint32_t* __restrict__ rbits, const uint32_t* __restrict__ rbase,
                             uint32_t* __restrict__ cpos) {
  // 4 positions per thread and iteration: their dependent load chains
  // (index -> label -> rank words) are in flight together
  constexpr int U = 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < n; p0 += U * stride) {
    uint32_t lab[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t p = p0 + u * stride;
      lab[u] = p < n ? labels[__ldg(&S[p].idx)] : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t p = p0 + u * stride;
      if (p < n) cpos[p] = bit_rank(rbits, rbase, lab[u]);
    }
  }
}

// ... and the first position per cluster from its label.
__global__ void k_group_first_of(const tpx_cluster_features* __restrict__ feats, uint64_t k,
                                 const uint32_t* __restrict__ first_of_label, uint32_t* __restrict__ first) {
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < k; c += (uint64_t)gridDim.x * blockDim.x)
    first[c] = first_of_label[feats[c].label];
}

__global__ void k_mark_first(const uint32_t* __restrict__ first, uint64_t k, uint32_t* __restrict__ fbits) {
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < k; c += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f = first[c];
    atomicOr(fbits + (f >> 5), 1u << (f & 31));
  }
}

// G3: block index of each cluster, the block table and the block sizes.
__global__ void k_group_rank(const uint32_t* __restrict__ first, uint64_t k, const uint32_t* __restrict__ fbits,
                             const uint32_t* __restrict__ fbase, const tpx_cluster_features* __restrict__ feats,
                             uint32_t* __restrict__ grank, uint32_t* __restrict__ cluster_of,
                             uint32_t* __restrict__ gsize) {
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < k; c += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t g = bit_rank(fbits, fbase, first[c]);
    grank[c] = g;
    cluster_of[g] = (uint32_t)c;
    gsize[g] = feats[c].size;
  }
}

// G4: radix keys and payloads in S order.
__global__ void k_group_keys(const srec* __restrict__ S, uint64_t n, const uint32_t* __restrict__ cpos,
                             const uint32_t* __restrict__ grank, uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ vals) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    keys[p] = grank[cpos[p]];
    vals[p] = S[p].idx;
  }
}

struct shape_acc {
  uint32_t xmin, xmax, ymin, ymax;
  unsigned long long xx, xy, yy;
  __device__ __forceinline__ void init() {
    xmin = ymin = 0xffffffffu;
    xmax = ymax = 0;
    xx = xy = yy = 0;
  }
  __device__ __forceinline__ void add(uint32_t x, uint32_t y) {
    xmin = min(xmin, x);
    xmax = max(xmax, x);
    ymin = min(ymin, y);
    ymax = max(ymax, y);
    xx += (unsigned long long)x * x;
    xy += (unsigned long long)x * y;
    yy += (unsigned long long)y * y;
  }
  __device__ __forceinline__ void store(shape_rec* d) const {
    shape_rec r;
    r.x_min = (uint16_t)xmin;
    r.x_max = (uint16_t)xmax;
    r.y_min = (uint16_t)ymin;
    r.y_max = (uint16_t)ymax;
    r.sum_xx = xx;
    r.sum_xy = xy;
    r.sum_yy = yy;
    *d = r;
  }
};

constexpr uint32_t kShapeWarpMin = 32;  // blocks at least this large are reduced by a warp

// G5a: one thread per block of fewer than kShapeWarpMin hits.
__global__ void k_shapes_small(const tpx_hit* __restrict__ hits, const uint32_t* __restrict__ order,
                               const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ cluster_of,
                               uint64_t k, shape_rec* __restrict__ shapes) {
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < k; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t o0 = offsets[g], o1 = offsets[g + 1];
    if (o1 - o0 >= kShapeWarpMin) continue;
    shape_acc s;
    s.init();
    uint32_t j = o0;
    for (; j + 4 <= o1; j += 4) {  // 4 gathers in flight
      uint32_t ix[4];
      hit4 h[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) ix[u] = order[j + u];
#pragma unroll
      for (int u = 0; u < 4; ++u) h[u] = load_hit(hits + ix[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) s.add(h[u].x, h[u].y);
    }
    for (; j < o1; ++j) {
      const hit4 h = load_hit(hits + order[j]);
      s.add(h.x, h.y);
    }
    s.store(shapes + cluster_of[g]);
  }
}

// G5b: one warp per large block (the others are skipped by a cheap test).
__global__ void k_shapes_large(const tpx_hit* __restrict__ hits, const uint32_t* __restrict__ order,
                               const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ cluster_of,
                               uint64_t k, shape_rec* __restrict__ shapes) {
  const unsigned lane = lane_id();
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t g0 = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; g0 < k; g0 += nw * 32) {
    // 32 candidate blocks per warp step: lanes test, the warp reduces each hit
    const uint64_t gl = g0 + lane;
    const bool is_big = gl < k && offsets[gl + 1] - offsets[gl] >= kShapeWarpMin;
    unsigned todo = __ballot_sync(kFull, is_big);
    while (todo) {
      const int b = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint64_t g = g0 + b;
      const uint32_t o0 = offsets[g], o1 = offsets[g + 1];
      shape_acc s;
      s.init();
      for (uint32_t j = o0 + lane; j < o1; j += 32) {
        const hit4 h = load_hit(hits + order[j]);
        s.add(h.x, h.y);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        s.xmin = min(s.xmin, __shfl_xor_sync(kFull, s.xmin, o));
        s.xmax = max(s.xmax, __shfl_xor_sync(kFull, s.xmax, o));
        s.ymin = min(s.ymin, __shfl_xor_sync(kFull, s.ymin, o));
        s.ymax = max(s.ymax, __shfl_xor_sync(kFull, s.ymax, o));
        s.xx += __shfl_xor_sync(kFull, s.xx, o);
        s.xy += __shfl_xor_sync(kFull, s.xy, o);
        s.yy += __shfl_xor_sync(kFull, s.yy, o);
      }
      if (lane == 0) s.store(shapes + cluster_of[g]);
    }
  }
}

}  // namespace tpx
