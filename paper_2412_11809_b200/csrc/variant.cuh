// variant.cuh -- variants (iii)(b) "global" and (iii)(c) "static" time
// neighbourhoods (§2 l.40-41) on the GPU.
//
// Both are defined by the streaming convention (R11, R21; the
// oracle's oracle_cluster_streaming): hits in (toa, index) order; a hit joins
// every existing cluster that has a member on one of its 9 neighbouring
// pixels and satisfies
//     (b) toa - cluster.maxToA <= dt_max      (c) toa - cluster.minToA <= dt_max
// and all joinable clusters are merged.  The process is sequential, but it is
// local in space-time, which gives independent islands:
//   * islands = connected components of the (a)-graph with window W (adjacent
//     and |dToA| <= W), computed by the (a) path itself, hits of an island in
//     (toa, index) order (tpx_cluster_run_grouped);
//   * inside an island the process is simulated exactly, a candidate member
//     taken only from the last W ticks;
//   * (c): W = dt_max is exact (a member older than dt_max cannot satisfy the
//     minToA test);
//   * (b): exact iff every simulated cluster spans <= W - dt_max (a missed
//     candidate would have joined a cluster already spanning more), which is
//     checked; otherwise W grows and the pass repeats.
// One thread simulates a small island, one warp a large one (the window scan
// in parallel, the merge as a warp min-reduction).
#pragma once
#include "common.cuh"
#include "group.cuh"

namespace tpx {

struct variant_args {
  const tpx_hit* ih;        // hits gathered in grouped order (ih[p] = hits[order[p]])
  const uint32_t* order;    // grouped order: input index per position
  const uint32_t* offsets;  // island blocks
  uint64_t k;               // islands
  uint64_t dt, window;
  int rule;                 // TPX_VARIANT_GLOBAL or TPX_VARIANT_STATIC
  uint32_t* par;            // union-find over positions (parent <= child)
  unsigned long long* cmin;  // per root position
  unsigned long long* cmax;
  uint32_t* stamp;          // candidate marks: stamp[root] = position + 1
};

#ifndef TPX_VAR_WARP_MIN
#define TPX_VAR_WARP_MIN 16
#endif
constexpr uint32_t kVarWarpMin = TPX_VAR_WARP_MIN;  // islands this large get a warp

__device__ __forceinline__ uint32_t var_find(uint32_t* par, uint32_t x) {
  uint32_t p;
  while ((p = par[x]) != x) {
    const uint32_t g = par[p];
    par[x] = g;  // path halving (any ancestor is a valid parent)
    x = g;
  }
  return x;
}

__device__ __forceinline__ bool var_pred(const variant_args& a, uint32_t r, uint64_t ti) {
  const uint64_t ref = a.rule == TPX_VARIANT_GLOBAL ? a.cmax[r] : a.cmin[r];
  return ti - ref <= a.dt;  // ref <= ti: members precede the hit
}

__device__ __forceinline__ bool var_adjacent(const hit4& p, const hit4& q) {
  const int dx = (int)p.x - (int)q.x, dy = (int)p.y - (int)q.y;
  return dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1;
}

// Hits in grouped (island) order, so the window scans below read contiguous
// records instead of a dependent order -> hit gather per candidate.
__global__ void k_gather_hits(const tpx_hit* __restrict__ hits, const uint32_t* __restrict__ order, uint64_t n,
                              tpx_hit* __restrict__ out) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x)
    out[p] = hits[order[p]];
}

// Small islands: one thread runs the process over the island's hits.
__global__ void k_variant_small(variant_args a) {
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < a.k; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t o0 = a.offsets[g], o1 = a.offsets[g + 1];
    if (o1 - o0 >= kVarWarpMin) continue;
    for (uint32_t p = o0; p < o1; ++p) {
      const hit4 hi = load_hit(a.ih + p);
      const uint64_t ti = hi.toa;
      // pass 1: mark the roots that may take the hit (states before merging)
      for (uint32_t q = p; q-- > o0;) {
        const hit4 hq = load_hit(a.ih + q);
        if (hq.toa + a.window < ti) break;
        if (!var_adjacent(hi, hq)) continue;
        const uint32_t r = var_find(a.par, q);
        if (var_pred(a, r, ti)) a.stamp[r] = p + 1;
      }
      // pass 2: merge the marked roots and the hit (target = smallest root)
      uint32_t target = 0xffffffffu;
      unsigned long long mn = ti, mx = ti;
      for (uint32_t q = p; q-- > o0;) {
        const hit4 hq = load_hit(a.ih + q);
        if (hq.toa + a.window < ti) break;
        if (!var_adjacent(hi, hq)) continue;
        const uint32_t r = var_find(a.par, q);
        if (a.stamp[r] != p + 1) continue;
        mn = min(mn, a.cmin[r]);
        mx = max(mx, a.cmax[r]);
        if (target == 0xffffffffu) {
          target = r;
        } else if (r != target) {
          const uint32_t lo = min(r, target), hi2 = max(r, target);
          a.par[hi2] = lo;  // parent < child
          target = lo;
        }
      }
      if (target == 0xffffffffu) target = p;
      a.par[p] = target;
      a.cmin[target] = mn;
      a.cmax[target] = mx;
    }
  }
}

// Large islands: one warp per island; lanes scan the window 32 at a time.
constexpr uint32_t kVarAdjCap = 256;  // listed adjacent candidates per warp and hit

__global__ void __launch_bounds__(256) k_variant_large(variant_args a) {
  __shared__ uint32_t s_adj[256 / 32][kVarAdjCap];
  uint32_t* adj = s_adj[threadIdx.x >> 5];
  const unsigned lane = lane_id();
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t g0 = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; g0 < a.k; g0 += nw * 32) {
    const uint64_t gl = g0 + lane;
    const bool is_big = gl < a.k && a.offsets[gl + 1] - a.offsets[gl] >= kVarWarpMin;
    unsigned todo = __ballot_sync(kFull, is_big);
    while (todo) {
      const uint64_t g = g0 + (__ffs(todo) - 1);
      todo &= todo - 1;
      const uint32_t o0 = a.offsets[g], o1 = a.offsets[g + 1];
      for (uint32_t p = o0; p < o1; ++p) {
        const hit4 hi = load_hit(a.ih + p);
        const uint64_t ti = hi.toa;
        // pass 1 (no linking: concurrent path halving is benign); the
        // adjacent candidates are listed so passes 2 and 3 visit only them
        uint32_t nadj = 0;
        for (uint32_t base = p; base > o0;) {
          const uint32_t q = base > lane ? base - 1 - lane : 0xffffffffu;
          bool in = false, isadj = false;
          uint32_t r1 = 0;
          if (q != 0xffffffffu && q >= o0) {
            const hit4 hq = load_hit(a.ih + q);
            in = hq.toa + a.window >= ti;
            isadj = in && var_adjacent(hi, hq);
            if (isadj) {
              r1 = var_find(a.par, q);
              if (var_pred(a, r1, ti)) a.stamp[r1] = p + 1;
            }
          }
          // the list keeps the candidate's ROOT: nothing links before pass 3,
          // so passes 2 and 3 need no second walk
          const unsigned bm = __ballot_sync(kFull, isadj);
          if (isadj && nadj + __popc(bm) <= kVarAdjCap) adj[nadj + __popc(bm & lanemask_lt())] = r1;
          nadj += __popc(bm);
          if (!__any_sync(kFull, in)) break;
          base = base > 32 ? base - 32 : 0;
        }
        __syncwarp();
        const bool listed = nadj <= kVarAdjCap;
        // pass 2: candidate roots -> warp min (target), min/max of their spans
        uint32_t tmin = 0xffffffffu;
        unsigned long long mn = ti, mx = ti;
        auto take = [&](uint32_t q) {
          uint32_t r = q;
          while (a.par[r] != r) r = a.par[r];  // read-only: no writes in this pass
          if (a.stamp[r] == p + 1) {
            tmin = min(tmin, r);
            mn = min(mn, a.cmin[r]);
            mx = max(mx, a.cmax[r]);
          }
        };
        if (listed) {
          for (uint32_t i = lane; i < nadj; i += 32) {
            const uint32_t r = adj[i];  // a root (pass 1)
            if (a.stamp[r] == p + 1) {
              tmin = min(tmin, r);
              mn = min(mn, a.cmin[r]);
              mx = max(mx, a.cmax[r]);
            }
          }
        } else {
          for (uint32_t base = p; base > o0;) {
            const uint32_t q = base > lane ? base - 1 - lane : 0xffffffffu;
            bool in = false;
            if (q != 0xffffffffu && q >= o0) {
              const hit4 hq = load_hit(a.ih + q);
              in = hq.toa + a.window >= ti;
              if (in && var_adjacent(hi, hq)) take(q);
            }
            if (!__any_sync(kFull, in)) break;
            base = base > 32 ? base - 32 : 0;
          }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          tmin = min(tmin, __shfl_xor_sync(kFull, tmin, o));
          mn = min(mn, __shfl_xor_sync(kFull, mn, o));
          mx = max(mx, __shfl_xor_sync(kFull, mx, o));
        }
        __syncwarp();
        // pass 3: link every candidate root under the target
        if (tmin != 0xffffffffu) {
          auto link = [&](uint32_t q) {
            uint32_t r = q;
            while (a.par[r] != r && a.stamp[r] != p + 1) r = a.par[r];
            if (a.stamp[r] == p + 1 && r != tmin) a.par[r] = tmin;  // same value from every lane
          };
          if (listed) {
            for (uint32_t i = lane; i < nadj; i += 32) {
              const uint32_t r = adj[i];
              if (a.stamp[r] == p + 1 && r != tmin) a.par[r] = tmin;  // same value from every lane
            }
          } else {
            for (uint32_t base = p; base > o0;) {
              const uint32_t q = base > lane ? base - 1 - lane : 0xffffffffu;
              bool in = false;
              if (q != 0xffffffffu && q >= o0) {
                const hit4 hq = load_hit(a.ih + q);
                in = hq.toa + a.window >= ti;
                if (in && var_adjacent(hi, hq)) link(q);
              }
              if (!__any_sync(kFull, in)) break;
              base = base > 32 ? base - 32 : 0;
            }
          }
        }
        __syncwarp();
        if (lane == 0) {
          const uint32_t t = tmin == 0xffffffffu ? p : tmin;
          a.par[p] = t;
          a.cmin[t] = mn;
          a.cmax[t] = mx;
        }
        __syncwarp();
      }
    }
  }
}

// Roots of every position, smallest input index per root, largest span.
__global__ void k_variant_roots(uint32_t* __restrict__ par, const uint32_t* __restrict__ order, uint64_t n,
                                const unsigned long long* __restrict__ cmin, const unsigned long long* __restrict__ cmax,
                                uint32_t* __restrict__ root_of, uint32_t* __restrict__ minidx,
                                unsigned long long* __restrict__ max_span) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t r = (uint32_t)p;
    while (par[r] != r) r = par[r];
    root_of[p] = r;
    atomicMin(minidx + r, order[p]);
    if (r == p) {
      // one address for every root: read before the atomic, so only spans
      // above the running maximum serialise on it
      const unsigned long long sp = cmax[r] - cmin[r];
      if (sp > *reinterpret_cast<volatile unsigned long long*>(max_span)) atomicMax(max_span, sp);
    }
  }
}

__global__ void k_variant_labels(const uint32_t* __restrict__ root_of, const uint32_t* __restrict__ order, uint64_t n,
                                 const uint32_t* __restrict__ minidx, uint32_t* __restrict__ labels) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x)
    labels[order[p]] = minidx[root_of[p]];
}

// Records in ascending label order: ordinal = rank of the label among roots.
__global__ void k_variant_feat_init(uint64_t n, const uint32_t* __restrict__ rbits, const uint32_t* __restrict__ rbase,
                                    tpx_cluster_features* __restrict__ feats, uint64_t capacity) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (!((rbits[i >> 5] >> (i & 31)) & 1u)) continue;
    const uint64_t o = bit_rank(rbits, rbase, (uint32_t)i);
    if (o >= capacity) continue;
    tpx_cluster_features f;
    f.label = (uint32_t)i;
    f.size = 0;
    f.toa_min = ~0ull;
    f.toa_max = 0;
    f.tot_sum = f.sum_x = f.sum_y = f.sum_tot_x = f.sum_tot_y = 0;
    feats[o] = f;
  }
}

// Feature accumulation over the hits in island order (ih[p] = hits[order[p]]):
// positions of one record are mostly adjacent there, and within an island
// in (toa, index) order, so lanes with the same record are reduced first
// and one lane per group issues the atomics (ToA min / max = the group's
// first / last lane).
__global__ void k_variant_feat_accum_grouped(const tpx_hit* __restrict__ ih, const uint32_t* __restrict__ order,
                                             uint64_t n, const uint32_t* __restrict__ labels,
                                             const uint32_t* __restrict__ rbits, const uint32_t* __restrict__ rbase,
                                             tpx_cluster_features* __restrict__ feats, uint64_t capacity) {
  const unsigned lane = lane_id();
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned am = __activemask();
    const uint64_t o = bit_rank(rbits, rbase, labels[order[p]]);
    const hit4 h = load_hit(ih + p);
    const unsigned peers = __match_any_sync(am, (unsigned)o);  // o < 2^32 (o < n)
    const uint32_t tx = (uint32_t)h.tot * h.x, ty = (uint32_t)h.tot * h.y;  // < 2^32 each
    const uint32_t s_tot = __reduce_add_sync(peers, (uint32_t)h.tot);
    const uint32_t s_x = __reduce_add_sync(peers, (uint32_t)h.x);
    const uint32_t s_y = __reduce_add_sync(peers, (uint32_t)h.y);
    const uint64_t s_tx = (uint64_t)__reduce_add_sync(peers, tx & 0xffffu) +
                          ((uint64_t)__reduce_add_sync(peers, tx >> 16) << 16);
    const uint64_t s_ty = (uint64_t)__reduce_add_sync(peers, ty & 0xffffu) +
                          ((uint64_t)__reduce_add_sync(peers, ty >> 16) << 16);
    if (o >= capacity) continue;
    tpx_cluster_features* f = feats + o;
    if ((int)lane == __ffs(peers) - 1) {
      atomicAdd(&f->size, (uint32_t)__popc(peers));
      atomicMin((unsigned long long*)&f->toa_min, (unsigned long long)h.toa);
      atomicAdd((unsigned long long*)&f->tot_sum, (unsigned long long)s_tot);
      atomicAdd((unsigned long long*)&f->sum_x, (unsigned long long)s_x);
      atomicAdd((unsigned long long*)&f->sum_y, (unsigned long long)s_y);
      atomicAdd((unsigned long long*)&f->sum_tot_x, (unsigned long long)s_tx);
      atomicAdd((unsigned long long*)&f->sum_tot_y, (unsigned long long)s_ty);
    }
    if ((int)lane == 31 - __clz(peers)) atomicMax((unsigned long long*)&f->toa_max, (unsigned long long)h.toa);
  }
}

}  // namespace tpx
