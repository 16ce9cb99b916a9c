// sort.cuh -- ToA sort (Alg. GPU Step 3: "Sort hits by their
// time of arrival. A fast option is the parallel radix sort").
//
// Global LSD radix sort on key = toa - toa_min with the input index as the
// payload; every pass is stable, so the final order is (toa, input index).
#pragma once
#include "common.cuh"

namespace tpx {

struct dev_hdr {
  unsigned long long toa_min;
  unsigned long long toa_max;
  unsigned int err;          // bit 0: coordinate / ToA range violation; bit 1: internal;
                             // bit 2: a sort window spans >= 2^32 ticks (windowed sort impossible)
                             // bit 3: a packed sort window's ToA range exceeds 28 bits
                             // bit 4: a ToA outside [radix_base, radix_base + 2^32) (speculative radix base)
  unsigned int sort_bad;     // windowed-sort verification failures
  unsigned long long n_clusters;
  unsigned long long n_pairs;       // cross-tile union pairs
  unsigned long long n_open_comps;  // components touching a tile border
  unsigned long long n_open_hits;   // hits of those components
  unsigned long long n_overflow;    // hits whose window left the staged halo
  unsigned long long radix_base;    // key origin of the radix fallback (toa - radix_base < 2^32)
  unsigned long long pad[7];
  unsigned long long phase_cycles[16];  // k_tile_cc per-phase clock totals (profiling)
};
static_assert(sizeof(dev_hdr) == 256, "dev_hdr layout");

constexpr int kMMThreads = 256;

// Fused validation + min/max ToA (one read of the hits).
__global__ void __launch_bounds__(kMMThreads) k_validate_minmax(hit_src hits, uint64_t n,
                                                                uint32_t width, uint32_t height,
                                                                dev_hdr* hdr) {
  uint64_t mn = ~0ull, mx = 0;
  unsigned bad = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    hit4 h = load_hit(hits + i);
    mn = min(mn, h.toa);
    mx = max(mx, h.toa);
    bad |= (h.x >= width) | (h.y >= height) | (h.toa >> 48 != 0);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(kFull, mn, o));
    mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    bad |= __shfl_xor_sync(kFull, bad, o);
  }
  if (lane_id() == 0) {
    atomicMin(&hdr->toa_min, mn);
    atomicMax(&hdr->toa_max, mx);
    if (bad) atomicOr(&hdr->err, 1u);
  }
}

// Guessed key origin of the radix fallback: the smallest ToA of the first
// kRadixBaseSample hits less 2^28 ticks (t-ordered input: no hit precedes its
// neighbourhood by anything near that).  The histogram kernel checks every key
// against it (err bit 4) and validates the hits, so the ToA range needs no
// separate pass and no read-back before the sort; a stream that breaks the
// guess is re-sorted with the exact minimum.
constexpr uint32_t kRadixBaseSample = 8192;
constexpr unsigned long long kRadixBaseMargin = 1ull << 28;
__global__ void __launch_bounds__(256) k_radix_base(hit_src hits, uint64_t n, dev_hdr* hdr) {
  __shared__ unsigned long long red[8];
  unsigned long long mn = ~0ull;
  const uint64_t m = n < kRadixBaseSample ? n : kRadixBaseSample;
  for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) mn = min(mn, (unsigned long long)load_hit(hits + i).toa);
#pragma unroll
  for (int o = 16; o; o >>= 1) mn = min(mn, __shfl_xor_sync(kFull, mn, o));
  if (lane_id() == 0) red[threadIdx.x >> 5] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) mn = min(mn, red[w]);
    hdr->radix_base = mn == ~0ull ? 0ull : (mn > kRadixBaseMargin ? mn - kRadixBaseMargin : 0ull);
  }
}

constexpr int kRadixThreads = 256;
constexpr int kRadixItems = 16;
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // 4096 keys per tile
constexpr int kRadixBins = 256;
#ifndef TPX_RSCAT_MINB
#define TPX_RSCAT_MINB 3  // resident CTAs per SM of k_radix_scatter_tile
#endif
#ifndef TPX_RSCAT_MINB
#define TPX_RSCAT_MINB 3
#endif

template <typename KeyT, bool kFromHits>
__device__ __forceinline__ KeyT radix_key(const hit_src& hits, const KeyT* keys, uint64_t i, uint64_t toa_min) {
  if constexpr (kFromHits) {
    return (KeyT)(load_hit(hits + i).toa - toa_min);
  } else {
    return keys[i];
  }
}

// Per-tile digit histogram, written digit-major: hist[d * n_tiles + tile].
template <typename KeyT, bool kFromHits>
__global__ void __launch_bounds__(kRadixThreads) k_radix_hist(hit_src hits,
                                                             const KeyT* __restrict__ keys, uint64_t n,
                                                             uint64_t toa_min, int shift,
                                                             uint32_t* __restrict__ hist, uint32_t n_tiles) {
  __shared__ uint32_t h[kRadixBins];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kRadixTile;
  // all digits first (16 independent loads in flight per thread), then the counting
  unsigned dg[kRadixItems];
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    uint64_t i = base + (uint64_t)r * kRadixThreads + threadIdx.x;
    dg[r] = i < n ? (unsigned)((radix_key<KeyT, kFromHits>(hits, keys, i, toa_min) >> shift) & 0xffu) : 256u;
  }
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const unsigned d = dg[r];
    unsigned peers = __match_any_sync(kFull, d);
    if (d < 256 && (__ffs(peers) - 1) == (int)lane_id()) atomicAdd(&h[d], (uint32_t)__popc(peers));
  }
  __syncthreads();
  hist[(uint64_t)threadIdx.x * n_tiles + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter: rank = global digit offset of this tile + number of earlier
// (round, warp, lane)-ordered elements of the tile with the same digit.
template <typename KeyT, bool kFromHits>
__global__ void __launch_bounds__(kRadixThreads) k_radix_scatter(hit_src hits,
                                                                const KeyT* __restrict__ keys_in,
                                                                const uint32_t* __restrict__ vals_in, uint64_t n,
                                                                uint64_t toa_min, int shift,
                                                                const uint32_t* __restrict__ offsets,
                                                                uint32_t n_tiles, KeyT* __restrict__ keys_out,
                                                                uint32_t* __restrict__ vals_out) {
  constexpr int kWarps = kRadixThreads / 32;
  __shared__ uint32_t base[kRadixBins];
  __shared__ uint32_t wcnt[kWarps][kRadixBins];
  base[threadIdx.x] = offsets[(uint64_t)threadIdx.x * n_tiles + blockIdx.x];
#pragma unroll
  for (int w = 0; w < kWarps; ++w) wcnt[w][threadIdx.x] = 0;
  __syncthreads();
  const unsigned warp = threadIdx.x >> 5, lane = lane_id();
  const uint64_t tbase = (uint64_t)blockIdx.x * kRadixTile;
  for (int r = 0; r < kRadixItems; ++r) {
    uint64_t i = tbase + (uint64_t)r * kRadixThreads + threadIdx.x;
    bool valid = i < n;
    KeyT key = 0;
    uint32_t val = 0;
    unsigned d = 256;
    if (valid) {
      key = radix_key<KeyT, kFromHits>(hits, keys_in, i, toa_min);
      val = kFromHits ? (uint32_t)i : vals_in[i];
      d = (unsigned)((key >> shift) & 0xffu);
    }
    unsigned peers = __match_any_sync(kFull, d);
    unsigned lrank = __popc(peers & lanemask_lt());
    if (valid && lrank == 0) wcnt[warp][d] = (uint32_t)__popc(peers);
    __syncthreads();
    if (valid) {
      uint32_t pos = base[d] + lrank;
      for (unsigned w = 0; w < warp; ++w) pos += wcnt[w][d];
      keys_out[pos] = key;
      vals_out[pos] = val;
    }
    __syncthreads();
    uint32_t add = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      add += wcnt[w][threadIdx.x];
      wcnt[w][threadIdx.x] = 0;
    }
    base[threadIdx.x] += add;
    __syncthreads();
  }
}

// Stable scatter for 32-bit keys, ranked in shared memory: the tile's 4096
// elements are ranked by digit with warp-private counters (warp w owns tile
// positions [512 w, 512 w + 512), so (warp, round, lane) order is index
// order), placed digit-sorted in shared memory, and written out in that
// order -- runs of equal digits go to consecutive global positions, so the
// stores coalesce, and the tile needs four barriers instead of three per
// 256 elements.
template <bool kFromHits>
__global__ void __launch_bounds__(kRadixThreads, TPX_RSCAT_MINB) k_radix_scatter_tile(hit_src hits,
                                                                     const uint32_t* __restrict__ keys_in,
                                                                     const uint32_t* __restrict__ vals_in,
                                                                     uint64_t n, uint64_t toa_min, int shift,
                                                                     const uint32_t* __restrict__ offsets,
                                                                     uint32_t n_tiles, uint32_t* __restrict__ keys_out,
                                                                     uint32_t* __restrict__ vals_out) {
  constexpr int kWarps = kRadixThreads / 32;
  constexpr int kPerWarp = kRadixItems * 32;
  static_assert(kRadixThreads == kRadixBins, "one scan thread per digit");
  __shared__ uint32_t skey[kRadixTile];
  __shared__ uint32_t sval[kRadixTile];
  __shared__ uint32_t wc[kWarps * kRadixBins];  // warp-major digit counters, then offsets
  __shared__ uint32_t gb[kRadixBins];           // global position - tile-local position, by digit
  __shared__ uint32_t dsum[kWarps];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t tbase = (uint64_t)blockIdx.x * kRadixTile;
  const uint32_t m = (uint32_t)min((uint64_t)kRadixTile, n - tbase);
  for (int i = threadIdx.x; i < kWarps * kRadixBins; i += kRadixThreads) wc[i] = 0;
  uint32_t key[kRadixItems], val[kRadixItems], rk[kRadixItems];
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const uint32_t p = warp * kPerWarp + r * 32 + lane;
    key[r] = 0;
    val[r] = 0;
    if (p < m) {
      const uint64_t i = tbase + p;
      if constexpr (kFromHits) {
        key[r] = (uint32_t)(load_hit(hits + i).toa - toa_min);
        val[r] = (uint32_t)i;
      } else {
        key[r] = keys_in[i];
        val[r] = vals_in[i];
      }
    }
  }
  __syncthreads();
  uint32_t* w = wc + warp * kRadixBins;
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const uint32_t p = warp * kPerWarp + r * 32 + lane;
    const bool valid = p < m;
    const unsigned d = valid ? (key[r] >> shift) & 0xffu : 256u;
    const unsigned peers = __match_any_sync(kFull, d);
    uint32_t b = 0;
    if (valid) b = w[d];
    rk[r] = b + __popc(peers & lanemask_lt());
    __syncwarp();
    if (valid && (__ffs(peers) - 1) == (int)lane) w[d] = b + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    const unsigned d = threadIdx.x;
    uint32_t tot = 0;
#pragma unroll
    for (int w2 = 0; w2 < kWarps; ++w2) tot += wc[w2 * kRadixBins + d];
    uint32_t x = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) dsum[warp] = x;
    __syncthreads();
    uint32_t start = x - tot;
    for (unsigned w2 = 0; w2 < warp; ++w2) start += dsum[w2];
    gb[d] = offsets[(uint64_t)d * n_tiles + blockIdx.x] - start;
#pragma unroll
    for (int w2 = 0; w2 < kWarps; ++w2) {
      const uint32_t c = wc[w2 * kRadixBins + d];
      wc[w2 * kRadixBins + d] = start;
      start += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const uint32_t p = warp * kPerWarp + r * 32 + lane;
    if (p < m) {
      const uint32_t q = w[(key[r] >> shift) & 0xffu] + rk[r];
      skey[q] = key[r];
      sval[q] = val[r];
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < m; i += kRadixThreads) {
    const uint32_t k = skey[i];
    const uint32_t pos = gb[(k >> shift) & 0xffu] + i;
    keys_out[pos] = k;
    vals_out[pos] = sval[i];
  }
}

// Sorted records + union-find init: rec[i] = hit[perm[i]], parent[i] = i.
// Four elements per thread and iteration: the permutation loads, then the
// dependent hit gathers, are issued together (memory-level parallelism).
__global__ void k_gather_init(hit_src hits, const uint32_t* __restrict__ perm, uint64_t n,
                              srec* __restrict__ rec, uint32_t* __restrict__ parent) {
  constexpr int U = 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += stride * U) {
    uint32_t j[U];
    hit4 h[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * stride;
      j[u] = i < n ? (perm ? perm[i] : (uint32_t)i) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n) h[u] = load_hit(hits + j[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < n) {
        srec r;
        r.tt = (h[u].toa << 16) | h[u].tot;
        r.xy = (h[u].y << 16) | h[u].x;
        r.idx = j[u];
        store_srec(rec + i, r);
        parent[i] = (uint32_t)i;
      }
    }
  }
}

}  // namespace tpx
