// cluster.cuh -- windowed neighbour search, union-find, canonical labels,
// compaction flags and segmented feature reductions (global-memory path).
#pragma once
#include "common.cuh"

namespace tpx {

// A3+A4: for every sorted position i, every later j with
// toa_j - toa_i <= dt and Chebyshev distance <= 1 (§2 (ii)+(iii)(a),
// §4.1 l.217: "the 8 neighboring pixels plus the pixel itself") is united
// with i.  Sorted order makes the candidate set a contiguous window.
__global__ void k_window_union(const srec* __restrict__ rec, uint64_t n, uint64_t dt, uint32_t* parent) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    srec a = load_srec(rec + i);
    const uint64_t ta = srec_toa(a);
    const int xa = (int)srec_x(a), ya = (int)srec_y(a);
    for (uint64_t j = i + 1; j < n; ++j) {
      srec b = load_srec(rec + j);
      if (srec_toa(b) - ta > dt) break;
      int dx = (int)srec_x(b) - xa, dy = (int)srec_y(b) - ya;
      if (dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1) uf_unite(parent, (uint32_t)i, (uint32_t)j);
    }
  }
}

__global__ void k_iota(uint32_t* parent, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    parent[i] = (uint32_t)i;
}

// Flatten: parent[i] = root(i).
__global__ void k_flatten(uint32_t* parent, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    parent[i] = uf_root(parent, (uint32_t)i);
}

// A5: minidx[root] = smallest input index of the cluster.
__global__ void k_minidx(const srec* __restrict__ rec, const uint32_t* __restrict__ root, uint64_t n,
                         uint32_t* minidx) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    atomicMin(minidx + root[i], rec[i].idx);
}

// labels_out[input index] = cluster label.
__global__ void k_labels(const srec* __restrict__ rec, const uint32_t* __restrict__ root,
                         const uint32_t* __restrict__ minidx, uint64_t n, uint32_t* __restrict__ labels) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    labels[rec[i].idx] = minidx[root[i]];
}

// A6: flag[j] = (labels[j] == j)  (j is the label of its cluster).
__global__ void k_flags(const uint32_t* __restrict__ labels, uint64_t n, uint64_t n_owned,
                        uint32_t* __restrict__ flags) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    flags[j] = labels[j] == (uint32_t)j && j < n_owned;
}

// Feature records initialised at their ordinal (ascending label).
__global__ void k_feat_init(const uint32_t* __restrict__ labels, const uint32_t* __restrict__ ord, uint64_t n,
                            uint64_t n_owned, tpx_cluster_features* __restrict__ feats, uint64_t capacity) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    if (labels[j] != (uint32_t)j || !(j + 1 <= n_owned)) continue;
    uint32_t k = ord[j];
    if (k >= capacity) continue;
    tpx_cluster_features f;
    f.label = (uint32_t)j;
    f.size = 0;
    f.toa_min = ~0ull;
    f.toa_max = 0;
    f.tot_sum = f.sum_x = f.sum_y = f.sum_tot_x = f.sum_tot_y = 0;
    feats[k] = f;
  }
}

// A7: integer feature reductions (u64 atomics; order-independent, bit-exact).
__global__ void k_feat_accum(const srec* __restrict__ rec, const uint32_t* __restrict__ root,
                             const uint32_t* __restrict__ minidx, const uint32_t* __restrict__ ord, uint64_t n,
                             uint64_t n_owned, tpx_cluster_features* feats, uint64_t capacity) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    srec r = load_srec(rec + i);
    if (r.idx >= n_owned) continue;  // halo hit of a sharded run: no features
    uint32_t k = ord[minidx[root[i]]];
    if (k >= capacity) continue;
    tpx_cluster_features* f = feats + k;
    const unsigned long long t = srec_toa(r), tot = srec_tot(r), x = srec_x(r), y = srec_y(r);
    atomicAdd(&f->size, 1u);
    atomicMin((unsigned long long*)&f->toa_min, t);
    atomicMax((unsigned long long*)&f->toa_max, t);
    atomicAdd((unsigned long long*)&f->tot_sum, tot);
    atomicAdd((unsigned long long*)&f->sum_x, x);
    atomicAdd((unsigned long long*)&f->sum_y, y);
    atomicAdd((unsigned long long*)&f->sum_tot_x, tot * x);
    atomicAdd((unsigned long long*)&f->sum_tot_y, tot * y);
  }
}

// A8: fp64 centroid, one correctly rounded division per coordinate.
__global__ void k_centroids(const tpx_cluster_features* __restrict__ f, uint64_t k, double* __restrict__ cxy) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x) {
    tpx_cluster_features r = f[i];
    double cx, cy;
    if (r.tot_sum) {
      cx = __ddiv_rn((double)r.sum_tot_x, (double)r.tot_sum);
      cy = __ddiv_rn((double)r.sum_tot_y, (double)r.tot_sum);
    } else {
      cx = __ddiv_rn((double)r.sum_x, (double)r.size);
      cy = __ddiv_rn((double)r.sum_y, (double)r.size);
    }
    cxy[2 * i] = cx;
    cxy[2 * i + 1] = cy;
  }
}

}  // namespace tpx
