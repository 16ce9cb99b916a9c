// shard.cuh -- kernels of the ToA-sharded multi-GPU path.
//
// Rank r owns the contiguous input-index block [o_r, o_r + n_r) of the
// t-ordered stream.  Because edges only join hits within dt_max in ToA
// (§2 (iii)(a) l.39) and a rank's block is a contiguous ToA range up
// to the readout disorder, rank r only needs rank r+1's hits with
// toa <= maxToA(r) + dt_max (the "forward halo", cf. the paper's temporal
// splitting, §3.2.3 l.117-119: "we only need to examine the dt_max-time
// neighborhood around each border").  Border clusters are merged by a union
// pass over (label on rank r, label on rank r+1) pairs of the halo hits --
// the B200 counterpart of the paper's merge step (§3.3 l.121-139).
#pragma once
#include "common.cuh"
#include "sort.cuh"
#include "tile_cc.cuh"

namespace tpx {

__global__ void k_range_init(unsigned long long* mm) {
  mm[0] = ~0ull;
  mm[1] = 0ull;
}

__global__ void k_toa_range(const tpx_hit* __restrict__ hits, uint64_t n, unsigned long long* mm) {
  unsigned long long lo = ~0ull, hi = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = load_hit(hits + i).toa;
    lo = min(lo, (unsigned long long)t);
    hi = max(hi, (unsigned long long)t);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(kFull, lo, o));
    hi = max(hi, __shfl_xor_sync(kFull, hi, o));
  }
  if (lane_id() == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

__global__ void k_halo_flags(const tpx_hit* __restrict__ hits, uint64_t n, uint64_t toa_limit,
                             uint32_t* __restrict__ flags) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    flags[i] = load_hit(hits + i).toa <= toa_limit;
}

__global__ void k_halo_scatter(const tpx_hit* __restrict__ hits, uint64_t n, const uint32_t* __restrict__ flags,
                               const uint32_t* __restrict__ ord, tpx_hit* __restrict__ out,
                               uint32_t* __restrict__ idx_out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (!flags[i]) continue;
    const uint32_t k = ord[i];
    reinterpret_cast<uint4*>(out)[k] = __ldg(reinterpret_cast<const uint4*>(hits) + i);
    idx_out[k] = (uint32_t)i;
  }
}

// Local labels of [owned | halo] -> global input indices.
__global__ void k_translate(uint32_t* labels, uint64_t n, uint64_t n_owned, uint64_t own_off,
                            const uint32_t* __restrict__ halo_idx, uint64_t next_off) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t L = labels[i];
    labels[i] = L < n_owned ? (uint32_t)(own_off + L) : (uint32_t)(next_off + halo_idx[L - n_owned]);
  }
}

__global__ void k_offset_labels(tpx_cluster_features* f, uint64_t k, uint32_t off) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x)
    f[i].label += off;
}

__global__ void k_gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx, uint64_t n,
                             uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = src[idx[i]];
}

// Pairs (a_i, b_i) with a_i != b_i, compacted (order irrelevant).
__global__ void k_make_pairs(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t n,
                             uint2* __restrict__ pairs, unsigned long long* count) {
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    const bool v = i < n && a[i] != b[i];
    const uint32_t slot = warp_append(v, count);
    if (v) pairs[slot] = make_uint2(a[i], b[i]);
  }
}

__global__ void k_unique_flags(const uint32_t* __restrict__ k, uint64_t n, uint32_t* __restrict__ flags) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    flags[i] = i == 0 || k[i] != k[i - 1];
}

__global__ void k_unique_scatter(const uint32_t* __restrict__ k, uint64_t n, const uint32_t* __restrict__ flags,
                                 const uint32_t* __restrict__ ord, uint32_t* __restrict__ uniq,
                                 uint32_t* __restrict__ parent) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (!flags[i]) continue;
    uniq[ord[i]] = k[i];
    parent[ord[i]] = ord[i];
  }
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t key) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Union of the two labels of every pair over indices into the sorted unique
// label array: linking the larger index under the smaller makes every root
// the smallest label of its set (label = smallest input index, reading R6).
__global__ void k_pair_union(const uint2* __restrict__ pairs, uint64_t n_pairs, const uint32_t* __restrict__ uniq,
                             const uint32_t* __restrict__ n_uniq, uint32_t* parent) {
  const uint32_t u = *n_uniq;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pairs;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 p = pairs[i];
    uf_unite(parent, lower_bound_u32(uniq, u, p.x), lower_bound_u32(uniq, u, p.y));
  }
}

__global__ void k_pair_finals(const uint32_t* __restrict__ uniq, const uint32_t* __restrict__ n_uniq,
                              const uint32_t* parent, uint32_t* __restrict__ finals) {
  const uint32_t u = *n_uniq;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < u; i += gridDim.x * blockDim.x)
    finals[i] = uniq[uf_root(parent, i)];
}

// labels[i] <- final(labels[i]) for labels in the map (sorted keys).
__global__ void k_relabel(uint32_t* labels, uint64_t n, const uint32_t* __restrict__ keys,
                          const uint32_t* __restrict__ vals, const unsigned long long* __restrict__ n_map) {
  const uint32_t m = (uint32_t)*n_map;
  if (m == 0) return;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t L = labels[i];
    const uint32_t p = lower_bound_u32(keys, m, L);
    if (p < m && keys[p] == L) labels[i] = vals[p];
  }
}

// Split records: labels in the map become partials (keyed by their final
// label); the rest are kept in order (flags for an order-preserving scan).
__global__ void k_split_flags(const tpx_cluster_features* __restrict__ f, uint64_t k, const uint32_t* __restrict__ keys,
                              const uint32_t* __restrict__ vals, const unsigned long long* __restrict__ n_map,
                              uint32_t* __restrict__ keep, tpx_cluster_features* __restrict__ partials,
                              unsigned long long* n_partials) {
  const uint32_t m = (uint32_t)*n_map;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < k; i0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    bool inv = false;
    uint32_t fin = 0;
    if (i < k) {
      const uint32_t L = f[i].label;
      const uint32_t p = m ? lower_bound_u32(keys, m, L) : 0;
      inv = p < m && keys[p] == L;
      if (inv) fin = vals[p];
      keep[i] = !inv;
    }
    const uint32_t slot = warp_append(inv, n_partials);
    if (inv) {
      tpx_cluster_features r = f[i];
      r.label = fin;
      partials[slot] = r;
    }
  }
}

__global__ void k_compact_records(const tpx_cluster_features* __restrict__ f, uint64_t k,
                                  const uint32_t* __restrict__ flag, const uint32_t* __restrict__ ord,
                                  tpx_cluster_features* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x)
    if (flag[i]) out[ord[i]] = f[i];
}

// Partials of this rank's block: keys (label) + payload (index) for sorting.
__global__ void k_fold_keys(const tpx_cluster_features* __restrict__ p, uint64_t q, uint64_t lo, uint64_t hi,
                            uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, unsigned long long* count) {
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < q; i0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    const bool v = i < q && p[i].label >= lo && p[i].label < hi;
    const uint32_t slot = warp_append(v, count);
    if (v) {
      keys[slot] = p[i].label;
      vals[slot] = (uint32_t)i;
    }
  }
}

// Combine runs of equal labels (run heads flagged, ord = exclusive scan).
__global__ void k_fold_runs(const tpx_cluster_features* __restrict__ p, const uint32_t* __restrict__ keys,
                            const uint32_t* __restrict__ vals, const unsigned long long* __restrict__ count,
                            const uint32_t* __restrict__ head, const uint32_t* __restrict__ ord,
                            tpx_cluster_features* __restrict__ merged) {
  const uint64_t q = *count;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q; i += (uint64_t)gridDim.x * blockDim.x) {
    if (!head[i]) continue;
    tpx_cluster_features r = p[vals[i]];
    for (uint64_t j = i + 1; j < q && keys[j] == keys[i]; ++j) {
      const tpx_cluster_features s = p[vals[j]];
      r.size += s.size;
      r.toa_min = min(r.toa_min, s.toa_min);
      r.toa_max = max(r.toa_max, s.toa_max);
      r.tot_sum += s.tot_sum;
      r.sum_x += s.sum_x;
      r.sum_y += s.sum_y;
      r.sum_tot_x += s.sum_tot_x;
      r.sum_tot_y += s.sum_tot_y;
    }
    merged[ord[i]] = r;
  }
}

__global__ void k_run_heads(const uint32_t* __restrict__ keys, const unsigned long long* __restrict__ count,
                            uint32_t* __restrict__ head) {
  const uint64_t q = *count;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q; i += (uint64_t)gridDim.x * blockDim.x)
    head[i] = i == 0 || keys[i] != keys[i - 1];
}

__device__ __forceinline__ uint64_t count_less(const tpx_cluster_features* a, uint64_t n, uint32_t label) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid].label < label) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Merge two label-sorted, label-disjoint record lists into out (merge path).
__global__ void k_merge_records(const tpx_cluster_features* __restrict__ a, uint64_t na,
                                const tpx_cluster_features* __restrict__ b, const uint32_t* __restrict__ nb_dev,
                                tpx_cluster_features* __restrict__ out, uint64_t capacity) {
  const uint64_t nb = *nb_dev;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na + nb;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (i < na) {
      const uint64_t pos = i + count_less(b, nb, a[i].label);
      if (pos < capacity) out[pos] = a[i];
    } else {
      const uint64_t j = i - na;
      const uint64_t pos = j + count_less(a, na, b[j].label);
      if (pos < capacity) out[pos] = b[j];
    }
  }
}

}  // namespace tpx
