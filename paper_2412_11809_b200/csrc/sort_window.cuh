// sort_window.cuh -- bounded-disorder ToA sort (A2), one pass over HBM.
//
// The input is t-ordered (§3.1 l.99-100): hits arrive almost in ToA
// order.  If no hit is displaced by more than D positions from its place in
// the (toa, input index) order, the hits that land in output positions
// [kT, (k+1)T) all come from input window [kT-D, (k+1)T+D), and exactly the
// first kT-ws of that window (ws = max(0, kT-D)) precede them.  So CTA k
// loads the window, sorts it in shared memory with a stable LSD radix sort on
// toa - window_min (ties keep input order => (toa, index) order), and writes
// the middle T records.  Whether D held is verified afterwards: the
// concatenation is correct iff it is strictly increasing in (toa, index)
// across CTA borders (k_sort_check, run right after the sort, checks every
// border and is the sole verifier); otherwise the host
// retries with a larger D and finally with the global radix sort (sort.cuh).
// Fused: coordinate / ToA-range validation of every hit.
#pragma once
#include "common.cuh"
#include "sort.cuh"

namespace tpx {

constexpr int kWSortThreads = 512;
constexpr int kWSortWarps = kWSortThreads / 32;
constexpr int kWSortTile = 4096;   // output records per CTA (T)
constexpr int kWDigitBits = 9;     // radix digit: 512 bins, so a 18-bit window key takes 2 passes
constexpr int kWRadix = 1 << kWDigitBits;
static_assert(kWRadix <= kWSortThreads, "one scan thread per digit");

// windowed sort attempts of tpx_cluster_run: 0 -> 8192 outputs per CTA from
// a 10240-hit window (IT = 20, D = 1024, 1.25x redundancy); 1 -> 5120 outputs
// (D = 2560, 2x: Timepix4-rate streams, displacement up to ~2300); 2 -> 4096
// outputs (D = 3072, 2.5x)
constexpr int kSortT0 = 8192;
constexpr int kSortTm = 5120;
constexpr int kSortT1 = 4096;

template <int IT, int T = kWSortTile, int NT = kWSortThreads>
struct wsort_cfg {
  static constexpr int W = NT * IT;                    // window capacity
  static constexpr int kT = T;                         // output records per CTA
  static constexpr int D = (W - T) / 2;                // displacement bound
  static constexpr int PER_WARP = IT * 32;
};

__device__ __forceinline__ unsigned long long block_min_u64(unsigned long long v, unsigned long long* sm) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
  if (lane_id() == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long x = threadIdx.x < blockDim.x / 32 ? sm[threadIdx.x] : ~0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) x = min(x, __shfl_xor_sync(kFull, x, o));
    if (threadIdx.x == 0) sm[32] = x;
  }
  __syncthreads();
  unsigned long long r = sm[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ unsigned long long block_max_u64(unsigned long long v, unsigned long long* sm) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
  if (lane_id() == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long x = threadIdx.x < blockDim.x / 32 ? sm[threadIdx.x] : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) x = max(x, __shfl_xor_sync(kFull, x, o));
    if (threadIdx.x == 0) sm[32] = x;
  }
  __syncthreads();
  unsigned long long r = sm[32];
  __syncthreads();
  return r;
}

template <int IT, int T, int NT = kWSortThreads>
__global__ void __launch_bounds__(NT, 1024 / NT) k_window_sort(hit_src hits, uint64_t n,
                                                                   uint32_t width, uint32_t height,
                                                                   srec* __restrict__ out, dev_hdr* hdr) {
  using C = wsort_cfg<IT, T, NT>;
  constexpr int kWarps = NT / 32;
  static_assert(kWRadix <= NT, "one scan thread per digit");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* skey = reinterpret_cast<uint32_t*>(smem_raw);                       // [W]
  uint16_t* sval = reinterpret_cast<uint16_t*>(skey + C::W);                     // [W]
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sval + C::W);                      // [kWRadix * warps]
  __shared__ unsigned long long red[33];

  const uint64_t k0 = (uint64_t)blockIdx.x * T;
  const uint64_t ws = k0 > (uint64_t)C::D ? k0 - C::D : 0;
  const uint64_t we = min(n, k0 + T + C::D);
  const uint32_t m = (uint32_t)(we - ws);
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;

  // ---- load the window (warp-blocked: warp w owns positions [w*PER_WARP, ...)).
  // Keys are kept as 32-bit offsets from a provisional origin (the window's
  // first ToA - 2^31), so no 64-bit ToA array lives in registers; a ToA more
  // than 2^31 ticks from the first one (only possible if the window spans
  // >= 2^31 ticks) sends the window to the fallback like a >= 2^32 span.
  const uint64_t org = (uint64_t)__ldg(reinterpret_cast<const unsigned long long*>(hits + ws)) - 0x80000000ull;
  uint32_t key[IT];
  uint32_t mn = 0xffffffffu, mx = 0;
  unsigned bad = 0, far = 0;
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    const uint32_t p = warp * C::PER_WARP + r * 32 + lane;
    key[r] = 0;
    if (p < m) {
      hit4 h = load_hit(hits + (ws + p));
      const uint64_t d = h.toa - org;
      far |= (d >> 32) != 0;
      key[r] = (uint32_t)d;
      mn = min(mn, key[r]);
      mx = max(mx, key[r]);
      bad |= (h.x >= width) | (h.y >= height) | (h.toa >> 48 != 0);
    }
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(&hdr->err, 1u);
  const uint32_t kmin = (uint32_t)block_min_u64(mn, red);
  const uint32_t kmax = (uint32_t)block_max_u64(mx, red);
  if (__syncthreads_or(far)) {  // window wider than 2^31 ticks: leave it to the fallback
    if (threadIdx.x == 0) {
      atomicAdd(&hdr->sort_bad, 1u);
      atomicOr(&hdr->err, 4u);  // a wider displacement bound cannot help: radix for this run only
    }
    return;
  }
  const uint32_t range = kmax - kmin;
  const int bits = range ? 32 - __clz(range) : 0;
  const int passes = (bits + kWDigitBits - 1) / kWDigitBits;
  uint32_t vl[IT];  // low 16 bits: window position (payload); high 16: rank within the warp
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    const uint32_t p = warp * C::PER_WARP + r * 32 + lane;
    key[r] -= kmin;
    vl[r] = p;
  }

  // ---- stable LSD radix passes, 8 bits each, ranks via warp-private counters
  // cnt is warp-major (cnt[w * kWRadix + d]): lanes of a warp touch banks d % 32,
  // so counter traffic is (nearly) conflict-free; equal digits are grouped by
  // __match_any_sync and only the group leader writes.
  __shared__ uint32_t dsum[NT / 32];
  for (int pass = 0; pass < passes || pass == 0; ++pass) {
    const int shift = pass * kWDigitBits;
    for (int i = threadIdx.x; i < kWRadix * kWarps; i += NT) cnt[i] = 0;
    __syncthreads();
    uint32_t* wc = cnt + warp * kWRadix;
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      const uint32_t p = warp * C::PER_WARP + r * 32 + lane;
      const bool valid = p < m;
      const unsigned d = valid ? (key[r] >> shift) & (kWRadix - 1) : (unsigned)kWRadix;
      const unsigned peers = __match_any_sync(kFull, d);
      uint32_t b = 0;
      if (valid) b = wc[d];
      vl[r] = (vl[r] & 0xffffu) | ((b + __popc(peers & lanemask_lt())) << 16);
      __syncwarp();
      if (valid && (__ffs(peers) - 1) == (int)lane) wc[d] = b + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // offsets in (digit, warp) order, every thread busy: thread t owns digit
    // t / kSplit and the kWarps / kSplit warps (t % kSplit)-th slice of it
    {
      constexpr int kSplit = NT / kWRadix;
      constexpr int kPer = kWarps / kSplit;
      static_assert(kSplit * kWRadix == NT && kPer * kSplit == kWarps, "offset scan layout");
      const uint32_t dd = threadIdx.x / kSplit, w0 = (threadIdx.x % kSplit) * kPer;
      uint32_t tot = 0;
#pragma unroll 4
      for (int w = 0; w < kPer; ++w) tot += cnt[(w0 + w) * kWRadix + dd];
      uint32_t x = tot;  // inclusive scan over threads (= (digit, slice) order)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= (unsigned)o) x += y;
      }
      if (lane == 31) dsum[warp] = x;
      __syncthreads();
      if (warp == 0) {
        uint32_t v = lane < (unsigned)kWarps ? dsum[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, v, o);
          if (lane >= (unsigned)o) v += y;
        }
        if (lane < (unsigned)kWarps) dsum[lane] = v;
      }
      __syncthreads();
      uint32_t basev = x - tot + (warp ? dsum[warp - 1] : 0u);
#pragma unroll 4
      for (int w = 0; w < kPer; ++w) {
        const uint32_t c = cnt[(w0 + w) * kWRadix + dd];
        cnt[(w0 + w) * kWRadix + dd] = basev;
        basev += c;
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      const uint32_t p = warp * C::PER_WARP + r * 32 + lane;
      if (p < m) {
        const unsigned d = (key[r] >> shift) & (kWRadix - 1);
        const uint32_t q = wc[d] + (vl[r] >> 16);
        skey[q] = key[r];
        sval[q] = (uint16_t)vl[r];
      }
    }
    __syncthreads();
    if (pass + 1 < passes) {
#pragma unroll
      for (int r = 0; r < IT; ++r) {
        const uint32_t p = warp * C::PER_WARP + r * 32 + lane;
        if (p < m) {
          key[r] = skey[p];
          vl[r] = sval[p];
        }
      }
      __syncthreads();
    }
  }

  // ---- write the middle T records (window-local ranks [k0-ws, k0-ws+T))
  const uint32_t ofs = (uint32_t)(k0 - ws);
  const uint32_t cnt_out = (uint32_t)min((uint64_t)T, n - k0);
  for (uint32_t j = threadIdx.x; j < cnt_out; j += NT) {
    const uint64_t gi = ws + sval[ofs + j];
    hit4 h = load_hit(hits + gi);
    srec r;
    r.tt = (h.toa << 16) | h.tot;
    r.xy = (h.y << 16) | h.x;
    r.idx = (uint32_t)gi;
    store_srec(out + k0 + j, r);
  }
}

// Packed variant: the registers hold one word per key instead of two.  Pass 0
// ranks the plain keys (the payload, the window position, is implicit in the
// (warp, round, lane) layout) and scatters (key >> 9) << 14 | position; later
// passes take their digit from that word.  Ranks are 16-bit halves.  So the
// register arrays are 1.5 x IT words, a 26-key window (W = 13312) fits 64
// registers, and the window redundancy drops (D = 1024: 11264 outputs of
// 13312 instead of 8192 of 10240; D = 2560: 8192 instead of 5120).  Key
// ranges up to 10 + 18 = 28 bits (2.7e8 ticks, 0.42 s) fit; a wider window
// flags err bit 3 and the run takes the unpacked kernel.  Digits are 10 bits
// wide with 16-bit counters (ranks and offsets are < 2^16 in a 13312-hit
// window), so a 20-bit window range -- the 40 Mhit/s mixed stream's 13312-hit
// windows span up to ~3.2e5 ticks -- still sorts in two passes.
#ifndef TPX_SORT_L2HINT
#define TPX_SORT_L2HINT 1
#endif
constexpr int kPackPosBits = 14;
constexpr int kPDigitBits = 10;
constexpr int kPRadix = 1 << kPDigitBits;
constexpr int kPackKeyBits = kPDigitBits + 32 - kPackPosBits;

template <int IT, int T, int NT = kWSortThreads>
__global__ void __launch_bounds__(NT, 1024 / NT) k_window_sort_packed(hit_src hits, uint64_t n, uint32_t width,
                                                                      uint32_t height, srec* __restrict__ out,
                                                                      dev_hdr* hdr) {
  using C = wsort_cfg<IT, T, NT>;
  constexpr int kWarps = NT / 32;
  static_assert(C::W <= (1 << kPackPosBits), "window positions fit the packed field");
  static_assert(3 * kPDigitBits >= kPackKeyBits && C::W < 65536, "three passes; 16-bit counters");
  static_assert(kPRadix % NT == 0, "whole digits per scan thread");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* skey = reinterpret_cast<uint32_t*>(smem_raw);  // [W] key << 14 | position
  uint16_t* cnt = reinterpret_cast<uint16_t*>(skey + C::W);  // [kPRadix * warps], warp-major
  __shared__ unsigned long long red[33];
  __shared__ uint32_t dsum[NT / 32];

  const uint64_t k0 = (uint64_t)blockIdx.x * T;
  const uint64_t ws = k0 > (uint64_t)C::D ? k0 - C::D : 0;
  const uint64_t we = min(n, k0 + T + C::D);
  const uint32_t m = (uint32_t)(we - ws);
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;

  const uint64_t org = (uint64_t)__ldg(reinterpret_cast<const unsigned long long*>(hits + ws)) - 0x80000000ull;
  uint32_t pk[IT];
  uint32_t mn = 0xffffffffu, mx = 0;
  unsigned bad = 0, far = 0;
#if TPX_SORT_L2HINT
  const uint64_t pol_keep = l2_policy_evict_last();
#endif
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    const uint32_t p = warp * C::PER_WARP + r * 32 + lane;
    pk[r] = 0;
    if (p < m) {
#if TPX_SORT_L2HINT
      hit4 h = load_hit_hint(hits + (ws + p), pol_keep);
#else
      hit4 h = load_hit(hits + (ws + p));
#endif
      const uint64_t d = h.toa - org;
      far |= (d >> 32) != 0;
      pk[r] = (uint32_t)d;
      mn = min(mn, pk[r]);
      mx = max(mx, pk[r]);
      bad |= (h.x >= width) | (h.y >= height) | (h.toa >> 48 != 0);
    }
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(&hdr->err, 1u);
  const uint32_t kmin = (uint32_t)block_min_u64(mn, red);
  const uint32_t kmax = (uint32_t)block_max_u64(mx, red);
  if (__syncthreads_or(far)) {  // window wider than 2^31 ticks: leave it to the fallback
    if (threadIdx.x == 0) {
      atomicAdd(&hdr->sort_bad, 1u);
      atomicOr(&hdr->err, 4u);
    }
    return;
  }
  const uint32_t range = kmax - kmin;
  const int bits = range ? 32 - __clz(range) : 0;
  if (bits > kPackKeyBits) {  // too wide for the packed words: the unpacked kernel takes this run
    if (threadIdx.x == 0) {
      atomicAdd(&hdr->sort_bad, 1u);
      atomicOr(&hdr->err, 8u);
    }
    return;
  }
  const int passes = (bits + kPDigitBits - 1) / kPDigitBits;
#pragma unroll
  for (int r = 0; r < IT; ++r) pk[r] -= kmin;  // pass 0: plain keys
  uint32_t rk2[(IT + 1) / 2];  // rank within the warp's digit run, two 16-bit halves per word
  for (int pass = 0; pass < passes || pass == 0; ++pass) {
    // digit position: plain key in pass 0, packed word (key >> 9) << 14 | pos after
    const int shift = pass == 0 ? 0 : kPackPosBits + (pass - 1) * kPDigitBits;
    {
      uint4* c4 = reinterpret_cast<uint4*>(cnt);
      for (int i = threadIdx.x; i < kPRadix * kWarps / 8; i += NT) c4[i] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    uint16_t* wc = cnt + warp * kPRadix;
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      const uint32_t p = warp * C::PER_WARP + r * 32 + lane;
      const bool valid = p < m;
      const unsigned d = valid ? (pk[r] >> shift) & (kPRadix - 1) : (unsigned)kPRadix;
      const unsigned peers = __match_any_sync(kFull, d);
      uint32_t b = 0;
      if (valid) b = wc[d];
      const uint32_t rank = b + __popc(peers & lanemask_lt());
      if (r & 1) rk2[r / 2] |= rank << 16;
      else rk2[r / 2] = rank;
      __syncwarp();
      if (valid && (__ffs(peers) - 1) == (int)lane) wc[d] = (uint16_t)(b + __popc(peers));
      __syncwarp();
    }
    __syncthreads();
    {
      // offsets in (digit, warp) order: thread t owns digits [t * kDpt, (t + 1) * kDpt)
      constexpr int kDpt = kPRadix / NT;
      const uint32_t d0 = threadIdx.x * kDpt;
      uint32_t tot = 0;
#pragma unroll
      for (int dd = 0; dd < kDpt; ++dd)
#pragma unroll 4
        for (int w = 0; w < kWarps; ++w) tot += cnt[w * kPRadix + d0 + dd];
      uint32_t x = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= (unsigned)o) x += y;
      }
      if (lane == 31) dsum[warp] = x;
      __syncthreads();
      if (warp == 0) {
        uint32_t v = lane < (unsigned)kWarps ? dsum[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, v, o);
          if (lane >= (unsigned)o) v += y;
        }
        if (lane < (unsigned)kWarps) dsum[lane] = v;
      }
      __syncthreads();
      uint32_t basev = x - tot + (warp ? dsum[warp - 1] : 0u);
#pragma unroll
      for (int dd = 0; dd < kDpt; ++dd)
#pragma unroll 4
        for (int w = 0; w < kWarps; ++w) {
          const uint32_t c = cnt[w * kPRadix + d0 + dd];
          cnt[w * kPRadix + d0 + dd] = (uint16_t)basev;
          basev += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      const uint32_t p = warp * C::PER_WARP + r * 32 + lane;
      if (p < m) {
        const unsigned d = (pk[r] >> shift) & (kPRadix - 1);
        const uint32_t w = pass == 0 ? ((pk[r] >> kPDigitBits) << kPackPosBits) | p : pk[r];
        TPX_BOUND(wc[d] + ((rk2[r / 2] >> (16 * (r & 1))) & 0xffffu), m);
        skey[wc[d] + ((rk2[r / 2] >> (16 * (r & 1))) & 0xffffu)] = w;
      }
    }
    __syncthreads();
    if (pass + 1 < passes) {
#pragma unroll
      for (int r = 0; r < IT; ++r) {
        const uint32_t p = warp * C::PER_WARP + r * 32 + lane;
        if (p < m) pk[r] = skey[p];
      }
      __syncthreads();
    }
  }

  // ---- write the middle T records (window-local ranks [k0-ws, k0-ws+T))
  const uint32_t ofs = (uint32_t)(k0 - ws);
  const uint32_t cnt_out = (uint32_t)min((uint64_t)T, n - k0);
#if TPX_SORT_L2HINT
  const uint64_t pol_drop = l2_policy_evict_first();
#endif
  // kGU records per thread in flight: their shared-memory positions, then
  // their gathers, then their stores
  constexpr int kGU = TPX_WSORT_GATHER_U;
  for (uint32_t j0 = threadIdx.x; j0 < cnt_out; j0 += kGU * NT) {
    uint4 v[kGU];
    uint32_t gi[kGU];
#pragma unroll
    for (int u = 0; u < kGU; ++u) {
      const uint32_t j = j0 + u * NT;
      gi[u] = 0;
      if (j < cnt_out) {
        TPX_BOUND(ofs + j, m);
        gi[u] = skey[ofs + j] & ((1u << kPackPosBits) - 1);
      }
    }
#pragma unroll
    for (int u = 0; u < kGU; ++u) {
      const uint32_t j = j0 + u * NT;
      if (j < cnt_out) {
        TPX_BOUND(ws + gi[u], we);
#if TPX_SORT_L2HINT
        v[u] = ldg_v4_hint(hits + (ws + gi[u]), pol_drop);
#else
        v[u] = __ldg(reinterpret_cast<const uint4*>(hits + (ws + gi[u])));
#endif
      }
    }
#pragma unroll
    for (int u = 0; u < kGU; ++u) {
      const uint32_t j = j0 + u * NT;
      if (j < cnt_out) {
        TPX_BOUND(k0 + j, n);
        // tpx_hit {toa, x | y << 16, tot | reserved << 16} -> srec {toa << 16 | tot, y << 16 | x, index}
        const uint64_t toa = (uint64_t)v[u].x | ((uint64_t)v[u].y << 32);
        const uint64_t tt = (toa << 16) | (v[u].w & 0xffffu);
        const uint4 o = make_uint4((uint32_t)tt, (uint32_t)(tt >> 32), v[u].z, (uint32_t)(ws + gi[u]));
#if TPX_SORT_L2HINT
        stg_v4_hint(out + k0 + j, o, pol_drop);
#else
        *reinterpret_cast<uint4*>(out + k0 + j) = o;
#endif
      }
    }
  }
}

template <int IT, int NT = kWSortThreads>
constexpr size_t window_sort_packed_smem() {
  return (size_t)wsort_cfg<IT, kWSortTile, NT>::W * 4 + (size_t)kPRadix * (NT / 32) * 2;
}

template <int IT, int NT = kWSortThreads>
constexpr size_t window_sort_smem() {
  return (size_t)wsort_cfg<IT, kWSortTile, NT>::W * 6 + (size_t)kWRadix * (NT / 32) * 4;
}

// Verification of a windowed sort right after it (before any clustering
// work): the output is the sorted permutation iff it is strictly increasing
// in (toa, index) at every CTA border (each CTA's range is sorted by
// construction; n strictly increasing entries drawn from the input are a
// permutation of it).  One thread per border.
__global__ void k_sort_check(const srec* __restrict__ S, uint64_t n, uint32_t tile, dev_hdr* hdr) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1;
  const uint64_t b = k * tile;
  if (b >= n) return;
  const srec p = load_srec(S + b - 1), q = load_srec(S + b);
  const uint64_t tp = srec_toa(p), tq = srec_toa(q);
  if (!(tp < tq || (tp == tq && p.idx < q.idx))) atomicAdd(&hdr->sort_bad, 1u);
}

// ---------------------------------------------------------------------------
// Windowed stable sort of (key, payload) arrays whose keys are nearly sorted
// (every element within D positions of its place in the stable key order).
// Used by the grouping step (group.cuh): a hit's block rank, read in the ToA
// order S, is displaced from its output position by at most the span of its
// cluster in S.  CTA k sorts window [kT-D, kT+T+D) by key in shared memory
// (stable LSD radix, digits as k_window_sort) and writes the payloads of the
// middle T; the first / last (key, position) it emits go to `edge` so a
// border check can verify the displacement bound (k_kv_check), exactly as the
// ToA sort is verified.
// Keys are gathered as grank[cpos[p]] (block rank of the hit at sorted
// position p) and payloads as S[p].idx, so the grouping needs no separate
// key/value arrays.
template <int IT>
__global__ void __launch_bounds__(kWSortThreads, 2) k_window_sort_kv(const uint32_t* __restrict__ cpos,
                                                                      const uint32_t* __restrict__ grank,
                                                                      const srec* __restrict__ S, uint64_t n,
                                                                      uint32_t* __restrict__ out,
                                                                      uint4* __restrict__ edge, dev_hdr* hdr) {
  using C = wsort_cfg<IT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* skey = reinterpret_cast<uint32_t*>(smem_raw);                       // [W]
  uint16_t* sval = reinterpret_cast<uint16_t*>(skey + C::W);                     // [W]
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sval + C::W);                      // [kWRadix * warps]
  __shared__ unsigned long long red[33];

  const uint64_t k0 = (uint64_t)blockIdx.x * kWSortTile;
  const uint64_t ws = k0 > (uint64_t)C::D ? k0 - C::D : 0;
  const uint64_t we = min(n, k0 + kWSortTile + C::D);
  const uint32_t m = (uint32_t)(we - ws);
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;

  uint32_t key[IT];
  uint32_t vl[IT];  // low 16 bits: window position (payload); high 16: rank within the warp
  unsigned long long mn = ~0ull, mx = 0;
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    const uint32_t p = warp * C::PER_WARP + r * 32 + lane;
    key[r] = 0;
    vl[r] = p;
    if (p < m) {
      key[r] = __ldg(grank + __ldg(cpos + ws + p));
      mn = min(mn, (unsigned long long)key[r]);
      mx = max(mx, (unsigned long long)key[r]);
    }
  }
  const uint32_t base = (uint32_t)block_min_u64(mn, red);
  const uint32_t top = (uint32_t)block_max_u64(mx, red);
  const uint32_t range = top - base;
  const int bits = range ? 32 - __clz(range) : 0;
  const int passes = (bits + kWDigitBits - 1) / kWDigitBits;
#pragma unroll
  for (int r = 0; r < IT; ++r) key[r] -= base;

  __shared__ uint32_t dsum[kWSortThreads / 32];
  for (int pass = 0; pass < passes || pass == 0; ++pass) {
    const int shift = pass * kWDigitBits;
    for (int i = threadIdx.x; i < kWRadix * kWSortWarps; i += kWSortThreads) cnt[i] = 0;
    __syncthreads();
    uint32_t* wc = cnt + warp * kWRadix;
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      const uint32_t p = warp * C::PER_WARP + r * 32 + lane;
      const bool valid = p < m;
      const unsigned d = valid ? (key[r] >> shift) & (kWRadix - 1) : (unsigned)kWRadix;
      const unsigned peers = __match_any_sync(kFull, d);
      uint32_t b = 0;
      if (valid) b = wc[d];
      vl[r] = (vl[r] & 0xffffu) | ((b + __popc(peers & lanemask_lt())) << 16);
      __syncwarp();
      if (valid && (__ffs(peers) - 1) == (int)lane) wc[d] = b + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    {
      uint32_t tot = 0;
      if (threadIdx.x < kWRadix) {
#pragma unroll
        for (int w = 0; w < kWSortWarps; ++w) tot += cnt[w * kWRadix + threadIdx.x];
      }
      uint32_t x = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= (unsigned)o) x += y;
      }
      if (lane == 31) dsum[warp] = x;
      __syncthreads();
      if (threadIdx.x < kWRadix) {
        uint32_t basev = x - tot;
        for (unsigned w2 = 0; w2 < warp; ++w2) basev += dsum[w2];
#pragma unroll
        for (int w = 0; w < kWSortWarps; ++w) {
          const uint32_t c = cnt[w * kWRadix + threadIdx.x];
          cnt[w * kWRadix + threadIdx.x] = basev;
          basev += c;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      const uint32_t p = warp * C::PER_WARP + r * 32 + lane;
      if (p < m) {
        const unsigned d = (key[r] >> shift) & (kWRadix - 1);
        const uint32_t q = wc[d] + (vl[r] >> 16);
        skey[q] = key[r];
        sval[q] = (uint16_t)vl[r];
      }
    }
    __syncthreads();
    if (pass + 1 < passes) {
#pragma unroll
      for (int r = 0; r < IT; ++r) {
        const uint32_t p = warp * C::PER_WARP + r * 32 + lane;
        if (p < m) {
          key[r] = skey[p];
          vl[r] = sval[p];
        }
      }
      __syncthreads();
    }
  }
  const uint32_t ofs = (uint32_t)(k0 - ws);
  const uint32_t cnt_out = (uint32_t)min((uint64_t)kWSortTile, n - k0);
  for (uint32_t j = threadIdx.x; j < cnt_out; j += kWSortThreads) out[k0 + j] = __ldg(&S[ws + sval[ofs + j]].idx);
  if (threadIdx.x == 0) {
    const uint32_t a = ofs, b = ofs + cnt_out - 1;
    edge[blockIdx.x] = make_uint4(skey[a] + base, (uint32_t)(ws + sval[a]), skey[b] + base, (uint32_t)(ws + sval[b]));
  }
}

template <int IT>
constexpr size_t window_sort_kv_smem() {
  return window_sort_smem<IT>();
}

// Border check of k_window_sort_kv: (key, position) strictly increasing from
// every CTA's last output to the next CTA's first.
__global__ void k_kv_check(const uint4* __restrict__ edge, uint32_t n_ctas, dev_hdr* hdr) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (k >= n_ctas) return;
  const uint4 a = edge[k - 1], b = edge[k];
  if (!(a.z < b.x || (a.z == b.x && a.w < b.y))) atomicAdd(&hdr->sort_bad, 1u);
}

}  // namespace tpx
