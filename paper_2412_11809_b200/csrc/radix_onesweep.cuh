// radix_onesweep.cuh -- single-sweep LSD radix passes for the global ToA sort
// (the fallback of sort_window.cuh; "parallel radix sort").
//
// The earlier passes (sort.cuh: per pass a tile histogram kernel, a scan of
// tiles x 256 counters and a scatter kernel) read every key twice per pass.
// Here one kernel reads the keys once for the digit totals of every pass;
// each pass is then one kernel: a CTA takes the next tile in order (a global
// ticket, so every earlier tile is already running), ranks its 4096 keys by
// digit in shared memory (stable: warp w owns tile positions
// [512 w, 512 w + 512)), publishes its per-digit count, and obtains the
// number of keys with the same digit in all earlier tiles by looking back
// over their published words (decoupled look-back: a word is either this
// tile's count -- keep walking -- or the inclusive prefix -- stop), then
// publishes its own inclusive prefix and scatters digit runs to
// consecutive global positions.  Stability of every pass keeps the final
// order (toa, input index).  The last pass writes the sorted 16-byte records
// themselves (each gathered by its input index), so no permutation makes a
// round trip through HBM.
#pragma once
#include "common.cuh"
#include "sort.cuh"

namespace tpx {

constexpr int kOsPasses = 4;  // 32-bit keys, 8-bit digits
#ifndef TPX_OS_MINB
#define TPX_OS_MINB 3  // resident CTAs per SM of a pass (80 registers; 4 CTAs at 64 spill: 2.71 vs 2.53 ms per 50M)
#endif
constexpr unsigned long long kOsAgg = 1ull << 62;  // word holds this tile's count
constexpr unsigned long long kOsInc = 2ull << 62;  // word holds the inclusive prefix
constexpr unsigned long long kOsVal = (1ull << 62) - 1;

// Scratch layout (bytes, inside the radix histogram region of the workspace).
struct os_layout {
  static constexpr size_t gcount = 0;                                  // u32 [kOsPasses][256] digit totals
  static constexpr size_t ticket = gcount + kOsPasses * kRadixBins * 4;  // u32 [kOsPasses] tile tickets
  static constexpr size_t status = 8192;                               // u64 [kOsPasses][tiles][256]
  static_assert(ticket + kOsPasses * 4 <= status, "scratch layout");
  static size_t bytes(uint32_t tiles) { return status + (size_t)kOsPasses * tiles * kRadixBins * 8; }
};

// Digit totals of every pass (one read of the hits).
__global__ void __launch_bounds__(256) k_os_hist(hit_src hits, uint64_t n, const unsigned long long* base_ptr,
                                                 int passes, uint32_t* __restrict__ gcount, uint32_t width,
                                                 uint32_t height, dev_hdr* hdr) {
  __shared__ uint32_t h[kOsPasses][kRadixBins];
  for (int i = threadIdx.x; i < kOsPasses * kRadixBins; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint64_t toa_min = *base_ptr;
  // validate (fused): coordinates / ToA range, and every key inside
  // [base, base + 2^32) when the base was guessed (hdr != nullptr)
  unsigned bad = 0, out = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const hit4 hi = load_hit(hits + i);
    const uint64_t d = hi.toa - toa_min;
    if (hdr) {
      bad |= (hi.x >= width) | (hi.y >= height) | (hi.toa >> 48 != 0);
      out |= (hi.toa < toa_min) | ((d >> 32) != 0);
    }
    const uint32_t k = (uint32_t)d;
#pragma unroll
    for (int p = 0; p < kOsPasses; ++p)
      if (p < passes) atomicAdd(&h[p][(k >> (8 * p)) & 0xffu], 1u);
  }
  if (hdr) {  // the warp's flags, not lane 0's own
    const unsigned wb = __ballot_sync(kFull, bad), wo = __ballot_sync(kFull, out);
    if ((wb | wo) && lane_id() == 0) atomicOr(&hdr->err, (wb ? 1u : 0u) | (wo ? 16u : 0u));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadixBins; i += blockDim.x) {
    const uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(gcount + i, v);
  }
}

// One pass.  kFromHits: keys computed from the hits (first pass), payload =
// input index.
template <bool kFromHits>
__global__ void __launch_bounds__(kRadixThreads, TPX_OS_MINB) k_os_pass(
    hit_src hits, const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint64_t n,
    const unsigned long long* base_ptr, int pass, uint32_t n_tiles, const uint32_t* __restrict__ gcount, uint32_t* ticket,
    unsigned long long* status, uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
    srec* __restrict__ s_out) {
  constexpr int kWarps = kRadixThreads / 32;
  constexpr int kPerWarp = kRadixItems * 32;
  static_assert(kRadixThreads == kRadixBins, "one look-back thread per digit");
  __shared__ uint32_t skey[kRadixTile];
  __shared__ uint32_t sval[kRadixTile];
  __shared__ uint32_t wc[kWarps * kRadixBins];  // warp-major digit counters, then tile-local offsets
  __shared__ uint32_t gb[kRadixBins];           // global position - tile-local position, by digit
  __shared__ uint32_t s_tile;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const int shift = 8 * pass;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket + pass, 1u);
  for (int i = threadIdx.x; i < kWarps * kRadixBins; i += kRadixThreads) wc[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t tbase = (uint64_t)tile * kRadixTile;
  const uint32_t m = (uint32_t)min((uint64_t)kRadixTile, n - tbase);
  uint32_t key[kRadixItems], val[kRadixItems], rk[kRadixItems];
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const uint32_t p = warp * kPerWarp + r * 32 + lane;
    key[r] = 0;
    val[r] = 0;
    if (p < m) {
      const uint64_t i = tbase + p;
      if constexpr (kFromHits) {
        key[r] = (uint32_t)(load_hit(hits + i).toa - *base_ptr);
        val[r] = (uint32_t)i;
      } else {
        key[r] = keys_in[i];
        val[r] = vals_in[i];
      }
    }
  }
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
    // tile-local digit totals and offsets; thread d owns digit d
    const unsigned d = threadIdx.x;
    uint32_t tot = 0;
#pragma unroll
    for (int w2 = 0; w2 < kWarps; ++w2) tot += wc[w2 * kRadixBins + d];
    // publish this tile's count at once, then look back for the prefix
    unsigned long long* st = status + ((size_t)pass * n_tiles) * kRadixBins;
    volatile unsigned long long* vst = st;
    unsigned long long excl = 0;
    if (tile == 0) {
      vst[d] = kOsInc | tot;
    } else {
      vst[(size_t)tile * kRadixBins + d] = kOsAgg | tot;
      for (int64_t t = (int64_t)tile - 1; t >= 0; --t) {
        unsigned long long x;
        do {
          x = vst[(size_t)t * kRadixBins + d];
        } while ((x >> 62) == 0);
        excl += x & kOsVal;
        if ((x >> 62) == 2) break;
      }
      vst[(size_t)tile * kRadixBins + d] = kOsInc | (excl + tot);
    }
    // global digit start: totals of the smaller digits of this pass
    uint32_t x = gcount[pass * kRadixBins + d];
    const uint32_t cnt_d = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= (unsigned)o) x += y;
    }
    uint32_t lx = tot;  // tile-local exclusive offsets by digit
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, lx, o);
      if (lane >= (unsigned)o) lx += y;
    }
    __shared__ uint32_t gsum[kWarps], lsum[kWarps];
    if (lane == 31) {
      gsum[warp] = x;
      lsum[warp] = lx;
    }
    __syncthreads();
    uint32_t gstart = x - cnt_d, start = lx - tot;
    for (unsigned w2 = 0; w2 < warp; ++w2) {
      gstart += gsum[w2];
      start += lsum[w2];
    }
    gb[d] = (uint32_t)(gstart + excl) - start;
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
      TPX_BOUND(q, m);
      skey[q] = key[r];
      sval[q] = val[r];
    }
  }
  __syncthreads();
  if (s_out) {  // last pass: the sorted records themselves (gathered by input index, kGU per thread in flight)
    constexpr int kGU = TPX_RADIX_GATHER_U;
    for (uint32_t i0 = threadIdx.x; i0 < m; i0 += kGU * kRadixThreads) {
      uint4 v[kGU];
      uint32_t pos[kGU], gi[kGU];
#pragma unroll
      for (int u = 0; u < kGU; ++u) {
        const uint32_t i = i0 + u * kRadixThreads;
        if (i < m) {
          pos[u] = gb[(skey[i] >> shift) & 0xffu] + i;
          gi[u] = sval[i];
          TPX_BOUND(pos[u], n);
          v[u] = __ldg(reinterpret_cast<const uint4*>(hits + gi[u]));
        }
      }
#pragma unroll
      for (int u = 0; u < kGU; ++u) {
        const uint32_t i = i0 + u * kRadixThreads;
        if (i < m) {
          const uint64_t toa = (uint64_t)v[u].x | ((uint64_t)v[u].y << 32);
          const uint64_t tt = (toa << 16) | (v[u].w & 0xffffu);
          *reinterpret_cast<uint4*>(s_out + pos[u]) = make_uint4((uint32_t)tt, (uint32_t)(tt >> 32), v[u].z, gi[u]);
        }
      }
    }
  } else {
    for (uint32_t i = threadIdx.x; i < m; i += kRadixThreads) {
      const uint32_t k = skey[i];
      const uint32_t pos = gb[(k >> shift) & 0xffu] + i;
      TPX_BOUND(pos, n);
      keys_out[pos] = k;
      vals_out[pos] = sval[i];
    }
  }
}

}  // namespace tpx
