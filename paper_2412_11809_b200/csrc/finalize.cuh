// finalize.cuh -- global merge of border-crossing ("open") components and the
// ordered emission of feature records (A4 across tiles, A5, A6, A7).
//
// Only hits of open components take part in the global union-find; for the
// 40 Mhit/s mixed stream that is a few percent of the hits.
#pragma once
#include "common.cuh"
#include "sort.cuh"
#include "tile_cc.cuh"

namespace tpx {

constexpr int kListThreads = 256;
#ifndef TPX_LIST_GRID
#define TPX_LIST_GRID (148 * 32)  // swept 148 x {4, 8, 16, 32}: 32 best (mixed merge + emit 1.08 -> 1.01 ms)
#endif
constexpr int kListGrid = TPX_LIST_GRID;

__device__ __forceinline__ void flag_internal(dev_hdr* hdr) { atomicOr(&hdr->err, 2u); }

// Open bitmap over sorted positions (bit p = hit p belongs to an open
// component), one word per warp and output round of the tile kernels.  Edges
// of the global pass must join open hits only; a closed endpoint means the
// tile path was inconsistent (checked, never expected).
__device__ __forceinline__ bool is_open(const uint32_t* openbm, uint64_t p) {
  return (__ldcg(openbm + (p >> 5)) >> (p & 31)) & 1u;
}

// Hits whose forward window left the staged halo: scan the rest of the window
// (from the first position the tile did not stage) in global memory, one warp
// per hit (lane = candidate, 32 per step); any j it reaches belongs to an open
// component.
__global__ void __launch_bounds__(kListThreads) k_overflow_unions(const srec* __restrict__ S, uint64_t n, uint64_t dt,
                                                                  const uint2* __restrict__ list, dev_hdr* hdr,
                                                                  uint32_t* parent_g, const uint32_t* openbm) {
  const uint64_t cnt = hdr->n_overflow;
  const unsigned lane = lane_id();
  const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t t = wid; t < cnt; t += nw) {
    const uint2 e = list[t];
    const uint32_t i = e.x;
    const srec a = load_srec(S + i);
    const uint64_t ta = srec_toa(a);
    for (uint64_t j0 = e.y; j0 < n; j0 += 32) {
      const uint64_t j = j0 + lane;
      bool in = false, adj = false;
      if (j < n) {
        const srec b = load_srec(S + j);
        in = srec_toa(b) - ta <= dt;
        adj = in && adjacent(a.xy, b.xy);
      }
      if (adj) {
        if (!is_open(openbm, j)) flag_internal(hdr);
        else uf_unite_il(parent_g, i, (uint32_t)j);
      }
      if (!__all_sync(kFull, in)) break;  // past the window (sorted by ToA)
    }
  }
}

// After all unions: parent_g[pos] <- root for every open hit (read-only walk;
// every stored value is a final root), so later lookups are one load.
__global__ void __launch_bounds__(kListThreads) k_flatten_open(const uint32_t* __restrict__ open_hits, dev_hdr* hdr,
                                                               uint32_t* parent_g) {
  const uint64_t nh = hdr->n_open_hits;
  // 4 hits per thread and iteration: their dependent root walks overlap
  constexpr int U = 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < nh; t0 += U * stride) {
    uint32_t pos[U], cur[U];
#pragma unroll
    for (int u = 0; u < U; ++u) pos[u] = t0 + u * stride < nh ? open_hits[t0 + u * stride] : 0xffffffffu;
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = pos[u] != 0xffffffffu ? ld_cg(parent_g + pos[u]) : 0u;
    // the four root walks advance in lock step (one round = up to 4 loads)
    for (bool more = true; more;) {
      more = false;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (pos[u] == 0xffffffffu) continue;
        const uint32_t nx = ld_cg(parent_g + cur[u]);
        if (nx != cur[u]) {
          cur[u] = nx;
          more = true;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (pos[u] != 0xffffffffu) parent_g[pos[u]] = cur[u];
  }
}

__global__ void __launch_bounds__(kListThreads) k_pair_unions(const uint2* __restrict__ pairs, dev_hdr* hdr,
                                                              uint32_t* parent_g, const uint32_t* openbm) {
  const uint64_t cnt = hdr->n_pairs;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 p = pairs[t];
    if (!is_open(openbm, p.x) || !is_open(openbm, p.y)) {
      flag_internal(hdr);
      return;
    }
    uf_unite_il(parent_g, p.x, p.y);
  }
}

// Fold every open component's partial record into its final root's record.
__global__ void __launch_bounds__(kListThreads) k_merge_open(const uint32_t* __restrict__ open_comps, dev_hdr* hdr,
                                                             const uint32_t* __restrict__ parent_g,
                                                             const uint32_t* __restrict__ slot_of,
                                                             tpx_cluster_features* stage) {
  const uint64_t cnt = hdr->n_open_comps;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = open_comps[t];
    const uint32_t R = parent_g[r];  // flattened
    if (R == r) continue;
    tpx_cluster_features* src = stage + slot_of[r];
    tpx_cluster_features* dst = stage + slot_of[R];
    const tpx_cluster_features f = *src;
    atomicMin(&dst->label, f.label);
    atomicAdd(&dst->size, f.size);
    atomicMin((unsigned long long*)&dst->toa_min, (unsigned long long)f.toa_min);
    atomicMax((unsigned long long*)&dst->toa_max, (unsigned long long)f.toa_max);
    atomicAdd((unsigned long long*)&dst->tot_sum, (unsigned long long)f.tot_sum);
    atomicAdd((unsigned long long*)&dst->sum_x, (unsigned long long)f.sum_x);
    atomicAdd((unsigned long long*)&dst->sum_y, (unsigned long long)f.sum_y);
    atomicAdd((unsigned long long*)&dst->sum_tot_x, (unsigned long long)f.sum_tot_x);
    atomicAdd((unsigned long long*)&dst->sum_tot_y, (unsigned long long)f.sum_tot_y);
    src->size = 0;  // merged away: k_emit skips it
  }
}

// Labels of open hits; label bits of open final roots.
__global__ void __launch_bounds__(kListThreads) k_open_labels(const srec* __restrict__ S,
                                                              const uint32_t* __restrict__ open_hits,
                                                              const uint32_t* __restrict__ open_comps, dev_hdr* hdr,
                                                              const uint32_t* __restrict__ parent_g,
                                                              const uint32_t* __restrict__ slot_of,
                                                              const tpx_cluster_features* __restrict__ stage,
                                                              uint32_t* __restrict__ labels, uint32_t* bitmap,
                                                              uint32_t n_owned, uint32_t* __restrict__ first_of_label,
                                                              label_map lm) {
  const uint64_t nh = hdr->n_open_hits, nc = hdr->n_open_comps;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  constexpr int U = 4;  // 4 dependent load chains in flight per thread
  for (uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < nh; t0 += U * stride) {
    uint32_t pos[U], idx[U], lab[U];
#pragma unroll
    for (int u = 0; u < U; ++u) pos[u] = t0 + u * stride < nh ? open_hits[t0 + u * stride] : 0xffffffffu;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (pos[u] != 0xffffffffu) {
        idx[u] = S[pos[u]].idx;
        lab[u] = stage[slot_of[parent_g[pos[u]]]].label;  // flattened
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (pos[u] != 0xffffffffu) store_label(labels, n_owned, lm, idx[u], lab[u]);
  }
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nc; t += stride) {
    const uint32_t r = open_comps[t];
    if (parent_g[r] == r) {
      const uint32_t lab = stage[slot_of[r]].label;
      if (lab < n_owned) {
        set_label_bit(bitmap, lab);
        // the final root is the smallest sorted position of the component
        if (first_of_label) first_of_label[lab] = r;
      }
    }
  }
}

// Window-density probe on the sorted stream: for 128 evenly spaced hits, the
// number of later hits within dt_max (binary search).  The host uses it to
// pick the tile configuration (sparse tile_csr.cuh / dense tile_cc.cuh).
constexpr int kProbeSamples = 128;
// a sampled window longer than this counts as dense (the sparse kernels stage
// 512 forward-halo hits; > 10 % of the samples above it selects k_tile_cc<dense>)
constexpr uint32_t kDenseWindow = 640;
__global__ void k_density_probe(const srec* __restrict__ S, uint64_t n, uint64_t dt, uint32_t* __restrict__ out) {
  const uint32_t k = threadIdx.x;
  if (k >= kProbeSamples) return;
  const uint64_t p = (n - 1) * k / (kProbeSamples - 1);
  const uint64_t t = srec_key_toa(S, p);
  uint64_t lo = p + 1, hi = p + (1ull << 16) < n ? p + (1ull << 16) : n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (srec_key_toa(S, mid) <= t + dt) lo = mid + 1; else hi = mid;
  }
  out[k] = (uint32_t)(lo - p - 1);
}

__global__ void k_popc(const uint32_t* __restrict__ bitmap, uint64_t nwords, uint32_t* __restrict__ cnt) {
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += (uint64_t)gridDim.x * blockDim.x)
    cnt[w] = __popc(bitmap[w]);
}

// A6 + A7: ordinal of a label = set bits below it in the label bitmap; copy
// the staged record to features_out[ordinal] (ascending label order).  One
// warp per tile (persistent grid): the tile's records are read as a flat run
// of 16-byte words, so every load instruction covers 512 contiguous bytes.
constexpr int kEmitThreads = 256;
__global__ void __launch_bounds__(kEmitThreads) k_emit(const tpx_cluster_features* __restrict__ stage,
                                                       const uint32_t* __restrict__ comp_count, uint32_t n_tiles,
                                                       uint32_t tile,
                                                       const uint32_t* __restrict__ bitmap,
                                                       const uint32_t* __restrict__ wbase,
                                                       tpx_cluster_features* __restrict__ out, uint64_t capacity,
                                                       uint32_t label_off, tpx_cluster_features* __restrict__ removed,
                                                       unsigned long long* n_removed) {
  const unsigned lane = lane_id();
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n_tiles; t += nw) {
    const uint32_t cc = comp_count[t];
    const uint4* src = reinterpret_cast<const uint4*>(stage + (uint64_t)t * tile);
    // kU 32-word steps per iteration: their loads (record words, then bitmap
    // words, then ordinal bases) are in flight together
    constexpr int kU = 4;
    for (uint32_t q0 = 0; q0 < cc * 4; q0 += 32 * kU) {  // warp-uniform trip count
      uint4 v[kU];
      uint32_t label[kU], size[kU], bits[kU], base[kU];
      bool valid[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t q = q0 + 32 * u + lane;
        valid[u] = q < cc * 4;
        v[u] = make_uint4(0, 0, 0, 0);
        if (valid[u]) v[u] = __ldcs(src + q);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        // the record's first word (label, size) sits in the group's first lane
        label[u] = __shfl_sync(kFull, v[u].x, lane & ~3u);
        size[u] = __shfl_sync(kFull, v[u].y, lane & ~3u);
        valid[u] = valid[u] && size[u] != 0;
        bits[u] = valid[u] ? bitmap[label[u] >> 5] : 0u;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) base[u] = valid[u] ? wbase[label[u] >> 5] : 0u;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (!valid[u]) continue;
        const uint32_t q = q0 + 32 * u + lane;
        if ((q & 3) == 0) v[u].x = label[u] + label_off;  // global label (sharded runs)
        if (!((bits[u] >> (label[u] & 31)) & 1u)) {
          // bit cleared by the sharded boundary merge: the record moves to the
          // rank owning the cluster's final label (one slot per record)
          if (!removed) continue;
          uint32_t slot = 0;
          if ((q & 3) == 0) slot = (uint32_t)atomicAdd(n_removed, 1ull);
          slot = __shfl_sync(0xfu << (lane & ~3u), slot, lane & ~3u);  // the record's 4 lanes take this branch together
          reinterpret_cast<uint4*>(removed + slot)[q & 3] = v[u];
          continue;
        }
        const uint64_t ord = (uint64_t)base[u] + __popc(bits[u] & ((1u << (label[u] & 31)) - 1u));
        if (ord >= capacity) continue;
        TPX_BOUND(label[u], (uint64_t)n_tiles * tile);  // labels are input indices
        reinterpret_cast<uint4*>(out + ord)[q & 3] = v[u];
      }
    }
  }
}

}  // namespace tpx
