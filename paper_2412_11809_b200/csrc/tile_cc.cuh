// tile_cc.cuh -- A3 + A4 + A5 + A7 for one tile of the ToA-sorted stream,
// entirely in shared memory (the B200 counterpart of the paper's Step 4 chunk
// clustering, and Step 5 border stitching, l.173).
//
// CTA k owns sorted positions [kT, kT+T).  It stages its tile plus the hits
// within dt_max after it (forward halo) and before it (back halo):
//   1. column index: the tile + forward-halo hits are bucketed by pixel
//      column (counting sort, then ranked by time inside each bucket), so a
//      hit's spatial neighbours live in 3 short, time-ordered buckets (the
//      role the paper's 256x256 "last hit per pixel" matrix plays, l.171);
//   2. window search: for every tile hit i and each neighbouring column
//      bucket, the later hits j with toa_j - toa_i <= dt are tested for
//      Chebyshev distance <= 1 (one packed subtraction, adjacent()); edges
//      are buffered, then united in a shared-memory union-find (atomicCAS,
//      larger root under smaller => root = earliest hit: the paper's
//      time-invariant, l.219-221);
//   3. every tile hit within dt of the previous tile looks back into the back
//      halo; an edge there (or a back halo cut by its capacity) makes its
//      component "open"; so does a forward window that leaves the staged halo
//      (those hits are finished in global memory, finalize.cuh);
//   4. forward-halo hits that joined a tile component become cross pairs for
//      the global merge and make that component open;
//   5. closed components are final: label = smallest input index, features
//      reduced (warp REDUX + shared-memory atomics), labels_out written, one
//      64-byte record staged; open components stage a partial record that the
//      global pass merges.
#pragma once
#include "common.cuh"
#include "sort.cuh"

namespace tpx {

constexpr int kTileThreads = 512;
constexpr int kTile = 2048;                    // tile hits per CTA
constexpr int kHaloCap = 1024;                 // staged halo hits per side
constexpr int kFwdMax = kTile + kHaloCap;      // tile + forward halo (local index l)
constexpr int kBuckets = 4096;                 // column buckets (x >> shift)
constexpr int kBucketCap = 512;                // longer buckets: the tile takes the global path
constexpr int kItemsPerThread = kTile / kTileThreads;      // 4
constexpr int kStageItems = kFwdMax / kTileThreads;        // 6
constexpr uint32_t kSentinel = 0xffffffffu;
constexpr uint32_t kEdgeBuf = 8;               // buffered edges per thread and chunk
static_assert(kFwdMax % kTileThreads == 0, "staging layout");

struct tile_args {
  const srec* S;
  uint64_t n;
  uint64_t dt;
  uint32_t width;
  uint32_t bucket_shift;     // bucket = x >> bucket_shift  (< kBuckets buckets)
  uint32_t* labels;          // labels_out (input order)
  uint32_t* parent_g;        // global union-find over sorted positions (open hits only)
  uint32_t* slot_of;         // root position -> stage slot (open components)
  tpx_cluster_features* stage;  // [n_tiles * kTile]
  uint32_t* comp_count;      // [n_tiles]
  uint32_t* bitmap;          // label bitmap (input-index space)
  uint32_t* open_hits;       // sorted positions of hits in open components
  uint32_t* open_comps;      // sorted positions of open component roots
  uint2* pairs;              // cross pairs (halo hit position, tile root position)
  uint32_t* overflow;        // tile hits whose forward window exceeded the halo
  dev_hdr* hdr;
  uint32_t verify_stride;    // sorted-tile size whose borders are verified
};

// |dx| <= 1 and |dy| <= 1 for packed (y << 16 | x) with x, y < 2^15:
// d = (dy + 1) * 2^16 + (dx + 1) (mod 2^32); the low field is in [0, 2] iff
// |dx| <= 1 (a negative dx + 1 wraps to >= 2^15 + 2), and then no borrow
// reached the high field, which is in [0, 2] iff |dy| <= 1.
__device__ __forceinline__ bool adjacent(uint32_t a, uint32_t b) {
  const uint32_t d = b - a + 0x00010001u;
  return ((d & 0xffffu) <= 2u) & ((d >> 16) <= 2u);
}

__device__ __forceinline__ uint32_t s_find(volatile uint32_t* par, uint32_t x) {
  uint32_t p;
  while ((p = par[x]) != x) {
    const uint32_t g = par[p];
    par[x] = g;
    x = g;
  }
  return x;
}

__device__ __forceinline__ void s_unite(uint32_t* par, uint32_t a, uint32_t b) {
  a = s_find(par, a);
  b = s_find(par, b);
  while (a != b) {
    if (a > b) {
      const uint32_t t = a;
      a = b;
      b = t;
    }
    const uint32_t old = atomicCAS(par + b, b, a);
    if (old == b) break;
    b = s_find(par, old);
    a = s_find(par, a);
  }
}

__device__ __forceinline__ uint64_t srec_key_toa(const srec* S, uint64_t i) { return __ldg(&S[i].tt) >> 16; }

// Warp-aggregated append of `pred` items to a global list; returns the slot.
__device__ __forceinline__ uint32_t warp_append(bool pred, unsigned long long* counter) {
  const unsigned m = __ballot_sync(kFull, pred);
  uint32_t base = 0;
  const unsigned lane = lane_id();
  if (m) {
    const int leader = __ffs(m) - 1;
    if ((int)lane == leader) base = (uint32_t)atomicAdd(counter, (unsigned long long)__popc(m));
    base = __shfl_sync(kFull, base, leader);
  }
  return base + __popc(m & lanemask_lt());
}

__device__ __forceinline__ void stage_write(tpx_cluster_features* dst, uint32_t label, uint32_t size,
                                            uint64_t tmin, uint64_t tmax, uint64_t tot, uint64_t sx, uint64_t sy,
                                            uint64_t stx, uint64_t sty) {
  uint4* d = reinterpret_cast<uint4*>(dst);
  d[0] = make_uint4(label, size, (uint32_t)tmin, (uint32_t)(tmin >> 32));
  d[1] = make_uint4((uint32_t)tmax, (uint32_t)(tmax >> 32), (uint32_t)tot, (uint32_t)(tot >> 32));
  d[2] = make_uint4((uint32_t)sx, (uint32_t)(sx >> 32), (uint32_t)sy, (uint32_t)(sy >> 32));
  d[3] = make_uint4((uint32_t)stx, (uint32_t)(stx >> 32), (uint32_t)sty, (uint32_t)(sty >> 32));
}

__device__ __forceinline__ void set_label_bit(uint32_t* bitmap, uint32_t label) {
  atomicOr(bitmap + (label >> 5), 1u << (label & 31));
}

// Shared-memory carve-up (bytes).  Region A holds the column index during the
// clustering phase and the per-component accumulators afterwards.
struct tile_smem_layout {
  static constexpr size_t csort = 0;                                  // uint2 [kFwdMax]
  static constexpr size_t csli = csort + (size_t)kFwdMax * 8;          // u16   [kFwdMax]
  static constexpr size_t cltmp = csli + (size_t)kFwdMax * 2;          // u16   [kFwdMax]
  static constexpr size_t myrank = cltmp + (size_t)kFwdMax * 2;        // u16   [kFwdMax]
  static constexpr size_t region_a = myrank + (size_t)kFwdMax * 2;     // 43008
  static constexpr size_t hb = region_a;                               // uint2 [kHaloCap]
  static constexpr size_t bcnt = hb + (size_t)kHaloCap * 8;            // u32   [kBuckets/2 + 1] (u16 pairs)
  static constexpr size_t par = bcnt + ((size_t)kBuckets / 2 + 4) * 4;  // u32   [kFwdMax]
  static constexpr size_t csize = par + (size_t)kFwdMax * 4;           // u32   [kTile]
  static constexpr size_t crank = csize + (size_t)kTile * 4;           // u16   [kTile]
  static constexpr size_t cacc = crank + (size_t)kTile * 2;            // u16   [kTile]
  static constexpr size_t eb = cacc + (size_t)kTile * 2;               // u16   [kEdgeBuf * threads]
  static constexpr size_t copen = eb + (size_t)kEdgeBuf * kTileThreads * 2;  // u8 [kTile]
  static constexpr size_t hflag = copen + kTile;                       // u8    [kTile]
  static constexpr size_t total = hflag + kTile;
};
static_assert(10 * (kTile / 2) * 4 <= tile_smem_layout::region_a, "accumulators alias region A");
constexpr size_t kTileSmem = tile_smem_layout::total;

__global__ void __launch_bounds__(kTileThreads, 2) k_tile_cc(tile_args a) {
  using SL = tile_smem_layout;
  extern __shared__ __align__(16) unsigned char sm[];
  uint2* csort = reinterpret_cast<uint2*>(sm + SL::csort);      // (toa - base, y<<16|x), bucket-sorted
  uint16_t* csli = reinterpret_cast<uint16_t*>(sm + SL::csli);  // local index of csort entries
  uint16_t* cltmp = reinterpret_cast<uint16_t*>(sm + SL::cltmp);
  uint16_t* myrank = reinterpret_cast<uint16_t*>(sm + SL::myrank);  // local index -> csort position
  uint2* hb = reinterpret_cast<uint2*>(sm + SL::hb);            // back halo, index order
  uint32_t* bcnt = reinterpret_cast<uint32_t*>(sm + SL::bcnt);  // bucket counts / starts, 2 x u16 per word
  uint32_t* par = reinterpret_cast<uint32_t*>(sm + SL::par);
  uint32_t* csize = reinterpret_cast<uint32_t*>(sm + SL::csize);
  uint16_t* crank = reinterpret_cast<uint16_t*>(sm + SL::crank);
  uint16_t* cacc = reinterpret_cast<uint16_t*>(sm + SL::cacc);
  uint16_t* eb = reinterpret_cast<uint16_t*>(sm + SL::eb);
  uint8_t* copen = sm + SL::copen;
  uint8_t* hflag = sm + SL::hflag;  // per tile hit: bit0 open mark, bit1 overflow
  // accumulators (region A, after clustering)
  uint32_t* a_tot = reinterpret_cast<uint32_t*>(sm);
  uint32_t* a_sx = a_tot + kTile / 2;
  uint32_t* a_sy = a_sx + kTile / 2;
  uint32_t* a_vxl = a_sy + kTile / 2;  // sum(tot*x) and sum(tot*y) in 16-bit halves
  uint32_t* a_vxh = a_vxl + kTile / 2;
  uint32_t* a_vyl = a_vxh + kTile / 2;
  uint32_t* a_vyh = a_vyl + kTile / 2;
  uint32_t* a_tmin = a_vyh + kTile / 2;
  uint32_t* a_tmax = a_tmin + kTile / 2;
  uint32_t* a_midx = a_tmax + kTile / 2;
  __shared__ uint64_t s_meta[8];
  __shared__ uint32_t s_wsum[kTileThreads / 32];
  __shared__ uint32_t s_chunk, s_bmax;

  const uint64_t n = a.n, dt = a.dt;
  const srec* __restrict__ S = a.S;
  const uint64_t t0 = (uint64_t)blockIdx.x * kTile;
  const uint64_t t1 = min(n, t0 + kTile);
  const uint32_t nt = (uint32_t)(t1 - t0);
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t shift = a.bucket_shift;

  // ---- halo ranges (binary searches in the sorted stream), sort verification
  if (threadIdx.x == 0) {
    const uint64_t toa_first = srec_key_toa(S, t0), toa_last = srec_key_toa(S, t1 - 1);
    const uint64_t blim = t0 > (uint64_t)kHaloCap ? t0 - kHaloCap : 0;
    uint64_t lo = blim, hi = t0;  // back halo: first position with toa + dt >= toa_first
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (srec_key_toa(S, mid) + dt < toa_first) lo = mid + 1; else hi = mid;
    }
    const uint64_t b0 = lo;
    const bool btrunc = b0 == blim && blim > 0 && srec_key_toa(S, blim - 1) + dt >= toa_first;
    const uint64_t flim = min(n, t1 + kHaloCap);
    lo = t1;
    hi = flim;  // forward halo: first position with toa > toa_last + dt
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (srec_key_toa(S, mid) <= toa_last + dt) lo = mid + 1; else hi = mid;
    }
    const uint64_t f1 = lo;
    const bool ftrunc = f1 == flim && flim < n && srec_key_toa(S, flim) <= toa_last + dt;
    const uint64_t base = srec_key_toa(S, b0);
    const bool wide = (srec_key_toa(S, f1 - 1) - base) >> 32 != 0;
    s_meta[0] = b0;
    s_meta[1] = f1;
    s_meta[2] = base;
    s_meta[3] = (btrunc ? 1u : 0u) | (ftrunc ? 2u : 0u) | (wide ? 4u : 0u);
    s_meta[4] = ftrunc ? srec_key_toa(S, f1) : 0;  // ToA of the first hit not staged
    s_meta[5] = t0 ? srec_key_toa(S, t0 - 1) : 0;  // ToA of the previous tile's last hit
    if (t0 > 0 && (t0 % a.verify_stride) == 0) {   // sort verification at sorted-tile borders
      const srec p = load_srec(S + t0 - 1), q = load_srec(S + t0);
      const uint64_t tp = srec_toa(p), tq = srec_toa(q);
      if (!(tp < tq || (tp == tq && p.idx < q.idx))) atomicAdd(&a.hdr->sort_bad, 1u);
    }
    s_chunk = 0;
    s_bmax = 0;
  }
  for (uint32_t w = threadIdx.x; w < kBuckets / 2 + 4; w += kTileThreads) bcnt[w] = 0;
  for (uint32_t j = threadIdx.x; j < kTile; j += kTileThreads) {
    csize[j] = 0;
    copen[j] = 0;
    hflag[j] = 0;
  }
  __syncthreads();
  const uint64_t b0 = s_meta[0], f1 = s_meta[1], base = s_meta[2];
  const uint32_t flags = (uint32_t)s_meta[3];
  const bool btrunc = flags & 1u, ftrunc = flags & 2u;
  bool wide = flags & 4u;
  const uint32_t nb = (uint32_t)(t0 - b0);
  const uint32_t m = (uint32_t)(f1 - t0);  // tile + forward halo
  const uint32_t nf = m - nt;
  const uint32_t dt32 = dt > 0xffffffffull ? 0xffffffffu : (uint32_t)dt;  // rel. ToAs differ by < 2^32

  // ---- stage: back halo, and tile + forward halo counted into column buckets
  uint2 ev[kStageItems];
  uint32_t eslot[kStageItems];
  if (!wide) {
    for (uint32_t k = threadIdx.x; k < nb; k += kTileThreads) {
      const srec r = load_srec(S + b0 + k);
      hb[k] = make_uint2((uint32_t)(srec_toa(r) - base), r.xy);
    }
#pragma unroll
    for (int q = 0; q < kStageItems; ++q) {
      const uint32_t l = threadIdx.x + q * kTileThreads;
      if (l < m) {
        const srec r = load_srec(S + t0 + l);
        ev[q] = make_uint2((uint32_t)(srec_toa(r) - base), r.xy);
        const uint32_t b = (r.xy & 0xffffu) >> shift;
        const uint32_t old = atomicAdd(bcnt + (b >> 1), 1u << ((b & 1) * 16));
        eslot[q] = (old >> ((b & 1) * 16)) & 0xffffu;
      }
    }
  }
  __syncthreads();
  // exclusive scan of the bucket counts (in place, u16 pairs), max bucket length
  if (!wide) {
    constexpr int PT = kBuckets / kTileThreads;  // 8 buckets per thread
    uint32_t cnts[PT];
    uint32_t s = 0, mx = 0;
#pragma unroll
    for (int i = 0; i < PT; ++i) {
      const uint32_t b = threadIdx.x * PT + i;
      cnts[i] = (bcnt[b >> 1] >> ((b & 1) * 16)) & 0xffffu;
      s += cnts[i];
      mx = max(mx, cnts[i]);
    }
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= (unsigned)o) x += y;
    }
    mx = __reduce_max_sync(kFull, mx);
    if (lane == 31) s_wsum[warp] = x;
    if (lane == 0) atomicMax(&s_bmax, mx);
    __syncthreads();
    if (warp == 0) {
      uint32_t t = lane < kTileThreads / 32 ? s_wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, t, o);
        if (lane >= (unsigned)o) t += y;
      }
      if (lane < kTileThreads / 32) s_wsum[lane] = t;
    }
    __syncthreads();
    uint32_t ex = (warp ? s_wsum[warp - 1] : 0) + x - s;
    // write starts back as u16 pairs (each thread owns 8 consecutive buckets = 4 words)
#pragma unroll
    for (int i = 0; i < PT; i += 2) {
      const uint32_t lo16 = ex;
      const uint32_t hi16 = ex + cnts[i];
      bcnt[(threadIdx.x * PT + i) >> 1] = lo16 | (hi16 << 16);
      ex += cnts[i] + cnts[i + 1];
    }
    if (threadIdx.x == kTileThreads - 1) bcnt[kBuckets / 2] = m;  // start of the sentinel bucket
  }
  __syncthreads();
  if (s_bmax > (uint32_t)kBucketCap) wide = true;  // degenerate column: global path

  auto bstart = [&](uint32_t b) -> uint32_t { return (bcnt[b >> 1] >> ((b & 1) * 16)) & 0xffffu; };

  if (wide) {
    // Every hit becomes its own open component; the global pass does the work.
    for (uint32_t j = threadIdx.x; j < kTile; j += kTileThreads) {
      const bool v = j < nt;
      srec r;
      if (v) r = load_srec(S + t0 + j);
      const uint32_t oh = warp_append(v, &a.hdr->n_open_hits);
      const uint32_t oc = warp_append(v, &a.hdr->n_open_comps);
      const uint32_t ov = warp_append(v, &a.hdr->n_overflow);
      if (v) {
        const uint64_t pos = t0 + j;
        const uint64_t toa = srec_toa(r), tot = srec_tot(r), x = srec_x(r), y = srec_y(r);
        a.parent_g[pos] = (uint32_t)pos;
        a.slot_of[pos] = (uint32_t)(t0 + j);
        stage_write(a.stage + t0 + j, r.idx, 1, toa, toa, tot, x, y, tot * x, tot * y);
        a.open_hits[oh] = (uint32_t)pos;
        a.open_comps[oc] = (uint32_t)pos;
        a.overflow[ov] = (uint32_t)pos;
      }
    }
    if (threadIdx.x == 0) a.comp_count[blockIdx.x] = nt;
    return;
  }

  // ---- unordered scatter into buckets, then rank by time inside each bucket
#pragma unroll
  for (int q = 0; q < kStageItems; ++q) {
    const uint32_t l = threadIdx.x + q * kTileThreads;
    if (l < m) cltmp[bstart((ev[q].y & 0xffffu) >> shift) + eslot[q]] = (uint16_t)l;
  }
  for (uint32_t l = threadIdx.x; l < m; l += kTileThreads) par[l] = l;
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kStageItems; ++q) {
    const uint32_t l = threadIdx.x + q * kTileThreads;
    if (l < m) {
      const uint32_t b = (ev[q].y & 0xffffu) >> shift;
      const uint32_t s0 = bstart(b), s1 = bstart(b + 1);
      uint32_t r = 0;
      for (uint32_t p = s0; p < s1; ++p) r += cltmp[p] < l;
      const uint32_t fin = s0 + r;
      csort[fin] = ev[q];
      csli[fin] = (uint16_t)l;
      myrank[l] = (uint16_t)fin;
    }
  }
  __syncthreads();

  // ---- window search over the 3 neighbouring column buckets (dynamic warp
  // chunks; edges buffered, united after each chunk)
  const uint64_t prev_last = s_meta[5];
  const uint64_t first_unstaged = s_meta[4];
  const uint32_t wmax = a.width - 1;
  const uint32_t n_chunks = (nt + 31) / 32;
  for (;;) {
    uint32_t chunk = 0;
    if (lane == 0) chunk = atomicAdd(&s_chunk, 1u);
    chunk = __shfl_sync(kFull, chunk, 0);
    if (chunk >= n_chunks) break;
    const uint32_t j = chunk * 32 + lane;
    uint32_t ne = 0;
    if (j < nt) {
      const uint32_t pself = myrank[j];
      const uint2 h = csort[pself];
      const uint32_t x = h.y & 0xffffu;
      const uint32_t bl = (x ? x - 1 : x) >> shift, bm = x >> shift, br = (x < wmax ? x + 1 : x) >> shift;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const uint32_t b = c == 0 ? bl : (c == 1 ? bm : br);
        if ((c == 0 && b == bm) || (c == 2 && b == bm) || (c == 2 && b == bl)) continue;
        uint32_t p, pe = bstart(b + 1);
        if (b == bm) {
          p = pself + 1;
        } else {  // first entry of the bucket with local index > j (entries are time-ordered)
          uint32_t lo = bstart(b), hi = pe;
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (csli[mid] <= j) lo = mid + 1; else hi = mid;
          }
          p = lo;
        }
        for (; p < pe; ++p) {
          const uint2 g = csort[p];
          if (g.x - h.x > dt32) break;
          if (adjacent(h.y, g.y)) {
            const uint32_t lj = csli[p];
            if (ne < kEdgeBuf) eb[ne++ * kTileThreads + threadIdx.x] = (uint16_t)lj;
            else s_unite(par, j, lj);
          }
        }
      }
      uint8_t fl = 0;
      if (ftrunc && first_unstaged <= base + h.x + dt) fl = 3;  // window continues past the halo
      if (t0 > 0 && base + h.x <= prev_last + dt) {           // could an earlier tile reach it?
        bool found = false;
        int lb = (int)nb - 1;
        for (; lb >= 0; --lb) {
          const uint2 g = hb[lb];
          if (h.x - g.x > dt32) break;
          if (adjacent(h.y, g.y)) {
            found = true;
            break;
          }
        }
        if (found || (lb < 0 && btrunc)) fl |= 1;
      }
      hflag[j] = fl;
    }
    __syncwarp();
    for (uint32_t e = 0; e < ne; ++e) s_unite(par, j, eb[e * kTileThreads + threadIdx.x]);
    __syncwarp();
  }
  __syncthreads();

  // ---- flatten (read-only root walk; every stored value is a final root)
  for (uint32_t l = threadIdx.x; l < m; l += kTileThreads) {
    uint32_t c = par[l], nx;
    while (c != (nx = par[c])) c = nx;
    par[l] = c;
  }
  __syncthreads();

  // ---- sizes (warp-aggregated by root), open flags, cross pairs
#pragma unroll
  for (int q = 0; q < kItemsPerThread; ++q) {
    const uint32_t j = threadIdx.x + q * kTileThreads;
    const uint32_t r = j < nt ? par[j] : 0xffffffffu;
    const unsigned peers = __match_any_sync(kFull, r);
    if (j < nt) {
      if ((__ffs(peers) - 1) == (int)lane) atomicAdd(&csize[r], (uint32_t)__popc(peers));
      if (hflag[j] & 1u) copen[r] = 1;
    }
  }
  for (uint32_t h0 = 0; h0 < nf; h0 += kTileThreads) {
    const uint32_t h = h0 + threadIdx.x;
    bool joined = false;
    uint32_t r = 0, l = 0;
    if (h < nf) {
      l = nt + h;
      r = par[l];
      joined = r != l;
    }
    const uint32_t slot = warp_append(joined, &a.hdr->n_pairs);
    if (joined) {
      copen[r] = 1;
      a.pairs[slot] = make_uint2((uint32_t)(t0 + l), (uint32_t)(t0 + r));
    }
  }
  __syncthreads();

  // ---- compact roots (stage rank) and multi-hit roots (accumulator slot)
  {
    uint32_t packed[kItemsPerThread];
    uint32_t my = 0;
#pragma unroll
    for (int q = 0; q < kItemsPerThread; ++q) {
      const uint32_t j = threadIdx.x * kItemsPerThread + q;  // blocked for rank order
      uint32_t v = 0;
      if (j < nt && par[j] == j) v = 1u | ((csize[j] >= 2 ? 1u : 0u) << 16);
      packed[q] = v;
      my += v;
    }
    uint32_t x = my;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t t = lane < kTileThreads / 32 ? s_wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, t, o);
        if (lane >= (unsigned)o) t += y;
      }
      if (lane < kTileThreads / 32) s_wsum[lane] = t;
    }
    __syncthreads();
    uint32_t ex = (warp ? s_wsum[warp - 1] : 0) + x - my;
    const uint32_t total = s_wsum[kTileThreads / 32 - 1];
#pragma unroll
    for (int q = 0; q < kItemsPerThread; ++q) {
      const uint32_t j = threadIdx.x * kItemsPerThread + q;
      if (packed[q]) {
        crank[j] = (uint16_t)(ex & 0xffffu);
        if (packed[q] >> 16) {
          const uint32_t s = ex >> 16;
          cacc[j] = (uint16_t)s;
          a_tot[s] = 0;
          a_sx[s] = 0;
          a_sy[s] = 0;
          a_vxl[s] = 0;
          a_vxh[s] = 0;
          a_vyl[s] = 0;
          a_vyh[s] = 0;
          a_tmin[s] = 0xffffffffu;
          a_tmax[s] = 0;
          a_midx[s] = 0xffffffffu;
        }
      }
      ex += packed[q];
    }
    if (threadIdx.x == 0) a.comp_count[blockIdx.x] = total & 0xffffu;
  }
  __syncthreads();

  // ---- feature reductions of multi-hit components: lanes of a warp that
  // share a root reduce with REDUX first, then one shared-memory atomic per
  // field and group (64-bit sums are split into 16-bit halves so that every
  // atomic is a native 32-bit one: no CAS loops).
  srec rq[kItemsPerThread];
#pragma unroll
  for (int q = 0; q < kItemsPerThread; ++q) {
    const uint32_t j = threadIdx.x + q * kTileThreads;
    uint32_t key = 0xffffffffu;
    if (j < nt) {
      rq[q] = load_srec(S + t0 + j);
      const uint32_t r = par[j];
      if (csize[r] >= 2) key = cacc[r];
    }
    const unsigned peers = __match_any_sync(kFull, key);
    uint32_t tot = 0, x = 0, y = 0, rel = 0, idx = 0;
    if (key != 0xffffffffu) {
      tot = srec_tot(rq[q]);
      x = srec_x(rq[q]);
      y = srec_y(rq[q]);
      rel = (uint32_t)(srec_toa(rq[q]) - base);
      idx = rq[q].idx;
    }
    const uint32_t vx = tot * x, vy = tot * y;  // < 2^31 (tot < 2^16, x, y < 2^15)
    const uint32_t s_tot = __reduce_add_sync(peers, tot);
    const uint32_t s_x = __reduce_add_sync(peers, x);
    const uint32_t s_y = __reduce_add_sync(peers, y);
    const uint32_t s_vxl = __reduce_add_sync(peers, vx & 0xffffu);
    const uint32_t s_vxh = __reduce_add_sync(peers, vx >> 16);
    const uint32_t s_vyl = __reduce_add_sync(peers, vy & 0xffffu);
    const uint32_t s_vyh = __reduce_add_sync(peers, vy >> 16);
    const uint32_t m_tmin = __reduce_min_sync(peers, rel);
    const uint32_t m_tmax = __reduce_max_sync(peers, rel);
    const uint32_t m_idx = __reduce_min_sync(peers, idx);
    if (key != 0xffffffffu && (__ffs(peers) - 1) == (int)lane) {
      atomicAdd(&a_tot[key], s_tot);
      atomicAdd(&a_sx[key], s_x);
      atomicAdd(&a_sy[key], s_y);
      atomicAdd(&a_vxl[key], s_vxl);
      atomicAdd(&a_vxh[key], s_vxh);
      atomicAdd(&a_vyl[key], s_vyl);
      atomicAdd(&a_vyh[key], s_vyh);
      atomicMin(&a_tmin[key], m_tmin);
      atomicMax(&a_tmax[key], m_tmax);
      atomicMin(&a_midx[key], m_idx);
    }
  }
  __syncthreads();

  // ---- outputs: staged records, labels, bitmap, open lists
#pragma unroll
  for (int q = 0; q < kItemsPerThread; ++q) {
    const uint32_t j = threadIdx.x + q * kTileThreads;
    const bool v = j < nt;
    uint32_t r = 0;
    bool is_root = false, open = false, multi = false;
    if (v) {
      r = par[j];
      is_root = r == j;
      open = copen[r] != 0;
      multi = csize[r] >= 2;
    }
    const uint32_t label = !v ? 0u : (multi ? a_midx[cacc[r]] : rq[q].idx);
    const uint64_t pos = t0 + j;
    if (is_root) {  // staged record for every component root
      const uint64_t slot = t0 + crank[j];
      if (multi) {
        const uint32_t s = cacc[j];
        stage_write(a.stage + slot, label, csize[j], base + a_tmin[s], base + a_tmax[s], a_tot[s], a_sx[s], a_sy[s],
                    ((uint64_t)a_vxh[s] << 16) + a_vxl[s], ((uint64_t)a_vyh[s] << 16) + a_vyl[s]);
      } else {
        const uint64_t toa = srec_toa(rq[q]), tot = srec_tot(rq[q]), x = srec_x(rq[q]), y = srec_y(rq[q]);
        stage_write(a.stage + slot, label, 1, toa, toa, tot, x, y, tot * x, tot * y);
      }
      if (!open) set_label_bit(a.bitmap, label);
      else a.slot_of[pos] = (uint32_t)slot;
    }
    const uint32_t oc = warp_append(is_root && open, &a.hdr->n_open_comps);
    if (is_root && open) a.open_comps[oc] = (uint32_t)pos;
    const uint32_t oh = warp_append(v && open, &a.hdr->n_open_hits);
    const bool ovf = v && (hflag[j] & 2u);
    const uint32_t ov = warp_append(ovf, &a.hdr->n_overflow);
    if (v) {
      if (open) {
        a.parent_g[pos] = (uint32_t)(t0 + r);
        a.open_hits[oh] = (uint32_t)pos;
      } else {
        a.parent_g[pos] = kSentinel;
        a.labels[rq[q].idx] = label;
      }
      if (ovf) a.overflow[ov] = (uint32_t)pos;
    }
  }
}

}  // namespace tpx
