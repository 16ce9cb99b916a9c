// tile_cc.cuh -- A3 + A4 + A5 + A7 for one tile of the ToA-sorted stream,
// entirely in shared memory (the B200 counterpart of the paper's Step 4 chunk
// clustering, and Step 5 border stitching, l.173): the
// dense-stream (heavy-ion) configuration, chosen by the window-density probe,
// plus the helpers every tile kernel shares (tile_args, label stores, record
// writes, block scan, shared-memory union-find).
//
// CTA k owns sorted positions [kT, kT+T).  It stages its tile plus the hits
// within dt_max after it (forward halo) and before it (back halo):
//   1. pixel hash: every staged hit is pushed onto the list of its pixel in an
//      open-addressing table (slot word = pixel << 14 | list head) -- a
//      compact, per-CTA stand-in for the paper's 256x256 "last hit per pixel"
//      matrix (l.171); back-halo hits join the lists with local indices
//      m + k, so a tile hit learns from its own 9 lookups whether an earlier
//      tile reaches it;
//   2. search: for each of its 9 neighbouring pixels a tile hit takes only
//      the FIRST later hit on that pixel within dt (later hits there reach it
//      through their own same-pixel edge: the last-hit-per-pixel rule read
//      forwards); edges are buffered, then united in a shared-memory
//      union-find (atomicCAS, larger root under smaller => root = earliest
//      hit: the paper's time-invariant, l.219-221);
//   3. an edge into the back halo (or a back halo cut by its capacity) makes
//      a component "open"; so does a forward window that leaves the staged
//      halo (those hits are finished in global memory, finalize.cuh);
//   4. forward-halo hits that joined a tile component become cross pairs for
//      the global merge and make that component open;
//   5. closed components are final: label = smallest input index, features
//      reduced over a member array grouped by component (one thread per small
//      component, one warp per large one), labels_out written, one 64-byte
//      record staged; open components stage a partial record that the global
//      pass merges.
// (Round 1's sparse column-bucket configuration of this kernel was removed in
// round 2: the sparse path is tile_csr.cuh.)
#pragma once
#include <type_traits>

#include "common.cuh"
#include "sort.cuh"

namespace tpx {

constexpr int kTile = 1024;                    // smallest tile (comp_count sizing)
constexpr int kMaxTile = 4096;                 // largest tile (stage slot sizing)
#ifndef TPX_BACK_CAP
#define TPX_BACK_CAP 64  // swept 64 / 128 / 256: 64 fastest on mixed, heavy-ion and Timepix4 (fewer idle loads; a truncated back halo only marks hits open)
#endif
constexpr int kBackCap = TPX_BACK_CAP;         // staged back-halo hits (openness only)
constexpr int kHeadBits = 14;                  // dense pixel hash: slot word = pixel << 14 | list head
constexpr uint32_t kHeadMask = (1u << kHeadBits) - 1;
constexpr uint32_t kPixEmpty = 0xffffffffu >> kHeadBits;  // empty hash slot key (pixel ids must be < 2^18 - 1)
constexpr uint32_t kMaxTilePixels = kPixEmpty - 1;  // sensors with more pixels take the global path
constexpr uint16_t kNil = 0xffffu;             // end of a pixel list
constexpr int kMaxTileWidth = 1024;            // sensors wider than this take the global pipeline
constexpr uint32_t kSentinel = 0xffffffffu;
constexpr uint32_t kEdgeBuf = 8;               // buffered edges per thread and chunk

// Tile configurations: the forward halo must hold the hits within dt_max of
// the tile's last hit.  Sparse streams (windows of tens of hits) use a 1024
// halo and fit 4 CTAs per SM; dense heavy-ion streams (windows of ~1-3k hits,
// SURVEY H1) use a 3072 halo at 2 CTAs per SM so that windows stay on chip.
template <int kTileHits, int kThreadsPerCta, int kHaloHits, int kMinBlocks, bool kHashIndex>
struct tile_cfg {
  static constexpr int kTile = kTileHits;                         // tile hits per CTA
  static constexpr int kThreads = kThreadsPerCta;
  static constexpr int kItems = kTileHits / kThreadsPerCta;       // tile hits per thread
  static constexpr int kHalo = kHaloHits;
  static constexpr int kFwdMax = kTile + kHaloHits;               // tile + forward halo (local index l)
  static constexpr int kStageItems = kFwdMax / kThreads;
  static constexpr bool kRegStage = kStageItems <= 8;             // stage in registers, else re-read S
  static constexpr int kBlocks = kMinBlocks;
  static constexpr bool kHash = kHashIndex;                       // pixel hash (dense) vs column buckets (sparse)
  static constexpr int kSlotBits = kFwdMax <= 2048 ? 12 : kFwdMax <= 4096 ? 13 : 14;  // pixel hash slots (load <= 1/2)
  static constexpr int kSlots = 1 << kSlotBits;
  static_assert(kFwdMax % kThreads == 0 && kTile % kThreads == 0 && kTile % ::tpx::kTile == 0 &&
                    kTile <= kMaxTile, "staging layout");
  static_assert(kFwdMax + 256 <= (1 << kHeadBits), "list heads: tile + halos fit kHeadBits");
  static_assert(kSlots >= 2 * kFwdMax, "hash load");
};
using tile_dense = tile_cfg<4096, 1024, 4096, 1, true>;

// Where the final label of a hit goes (sharded runs, sharded.cuh): labels of
// owned hits (input index < n_owned) into `labels`, of halo hits into
// `halo_labels`, translated to global input indices -- own_off + l for an
// owned label l, next_off + halo_idx[l - n_owned] for a label that is a halo
// hit.  halo_idx == nullptr: one array, local labels (every other run).
struct label_map {
  uint32_t* halo_labels;
  const uint32_t* halo_idx;
  uint32_t own_off, next_off;
};
__device__ __forceinline__ void store_label(uint32_t* labels, uint32_t n_owned, const label_map& m, uint32_t idx,
                                            uint32_t label) {
  if (!m.halo_idx) {
    labels[idx] = label;
    return;
  }
  const uint32_t g = label < n_owned ? label + m.own_off : m.next_off + m.halo_idx[label - n_owned];
  if (idx < n_owned) labels[idx] = g;
  else m.halo_labels[idx - n_owned] = g;
}

struct tile_args {
  const srec* S;
  uint64_t n;
  uint64_t dt;
  uint32_t width;
  uint32_t height;
  uint32_t n_owned;          // hits with input index >= n_owned carry no features (sharded halo)
  uint32_t* labels;          // labels_out (input order)
  uint32_t* parent_g;        // global union-find over sorted positions (open hits only)
  uint32_t* openbm;          // open bitmap over sorted positions (finalize.cuh is_open)
  uint32_t* slot_of;         // root position -> stage slot (open components)
  tpx_cluster_features* stage;  // [n_tiles * kTile]
  uint32_t* comp_count;      // [n_tiles]
  uint32_t* bitmap;          // label bitmap (input-index space)
  uint32_t* open_hits;       // sorted positions of hits in open components
  uint32_t* open_comps;      // sorted positions of open component roots
  uint2* pairs;              // cross pairs (halo hit position, tile root position)
  uint2* overflow;           // (position, first unscanned position) of tile hits whose window exceeded the halo
  dev_hdr* hdr;
  uint32_t verify_stride;    // sorted-tile size whose borders are verified
  unsigned long long* phase_cycles;  // optional per-phase clock totals (profiling), may be null
  const uint64_t* tile_meta;  // k_tile_bounds output (k_tile_cell only)
  uint32_t* first_of_label;   // optional (grouped runs): label -> sorted position of the cluster's first hit
  label_map lm;               // label destinations (sharded runs)
};

#define TPX_PHASE(k)                                                         \
  do {                                                                       \
    if (a.phase_cycles && threadIdx.x == 0) {                                \
      const long long now_ = clock64();                                      \
      atomicAdd(a.phase_cycles + (k), (unsigned long long)(now_ - t_phase)); \
      t_phase = now_;                                                        \
    }                                                                        \
  } while (0)

// |dx| <= 1 and |dy| <= 1 for packed (y << 16 | x) with x, y < 2^15:
// d = (dy + 1) * 2^16 + (dx + 1) (mod 2^32); the low field is in [0, 2] iff
// |dx| <= 1 (a negative dx + 1 wraps to >= 2^15 + 2), and then no borrow
// reached the high field, which is in [0, 2] iff |dy| <= 1.
__device__ __forceinline__ bool adjacent(uint32_t a, uint32_t b) {
  const uint32_t d = b - a + 0x00010001u;
  return ((d & 0xffffu) <= 2u) & ((d >> 16) <= 2u);
}

// Shared-memory atomic min without a return value (RED.MIN on shared memory).
__device__ __forceinline__ void red_min_shared(uint32_t* p, uint32_t v) {
  asm volatile("red.shared.min.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

// Find with path halving.  Parents only decrease along a path (a root is
// linked under a smaller one), so every ancestor is a valid parent and the
// halving store can be an atomic min: concurrent finds on the same path then
// never race (compute-sanitizer racecheck reports 0 hazards), and a halving
// store can never move a node back down below a concurrently written one.
__device__ __forceinline__ uint32_t s_find(uint32_t* par, uint32_t x) {
  volatile uint32_t* vp = par;
  uint32_t p;
  while ((p = vp[x]) != x) {
    const uint32_t g = vp[p];
    if (g != p) red_min_shared(par + x, g);
    x = g;
  }
  return x;
}

__device__ __forceinline__ void s_unite(uint32_t* par, uint32_t a, uint32_t b) {
  // start one level up: an edge inside an already-merged component (most
  // edges of a compact cluster once its first edges are united) usually has
  // both ends under the same parent and costs two loads
  a = reinterpret_cast<volatile uint32_t*>(par)[a];
  b = reinterpret_cast<volatile uint32_t*>(par)[b];
  if (a == b) return;
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

// The same union with both finds climbing in lockstep: each step issues the
// two parent loads together (independent), so a union costs about one find's
// latency instead of two, and stops as soon as the two walks meet.
__device__ __forceinline__ void s_unite_il(uint32_t* par, uint32_t a, uint32_t b) {
  volatile uint32_t* vp = par;
  a = vp[a];
  b = vp[b];
  for (;;) {
    if (a == b) return;
    const uint32_t pa = vp[a], pb = vp[b];
    if (pa == a && pb == b) {  // two roots: larger under smaller
      const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
      const uint32_t old = atomicCAS(par + hi, hi, lo);
      if (old == hi) return;
      a = lo;
      b = old;  // hi was linked meanwhile: go on from its new parent
      continue;
    }
    if (pa != a) {
      const uint32_t ga = vp[pa];
      if (ga != pa) red_min_shared(par + a, ga);
      a = ga;
    }
    if (pb != b) {
      const uint32_t gb = vp[pb];
      if (gb != pb) red_min_shared(par + b, gb);
      b = gb;
    }
  }
}

__device__ __forceinline__ uint64_t srec_key_toa(const srec* S, uint64_t i) { return __ldg(&S[i].tt) >> 16; }

// First p in [lo, hi) with pred(p) (hi if none) for a monotone pred, one warp:
// 32 probes per round shrink the range 31-fold (3 dependent loads for 1024).
template <typename Pred>
__device__ __forceinline__ uint64_t warp_lower_bound(uint64_t lo, uint64_t hi, Pred pred) {
  const unsigned lane = lane_id();
  while (hi > lo) {  // invariant: the answer is in [lo, hi], pred(hi) taken as true
    const uint64_t step = (hi - lo) / 31 + 1;
    const uint64_t p = lo + lane * step;
    const bool v = p >= hi ? true : pred(p);
    const int f = __ffs(__ballot_sync(kFull, v)) - 1;  // lane 31 probes >= hi
    if (f == 0) return lo;
    const uint64_t nhi = min(hi, lo + (uint64_t)f * step);
    lo = lo + (uint64_t)(f - 1) * step + 1;
    hi = nhi;
  }
  return lo;
}

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

// Shared-memory carve-up of the pixel-hash index (dense configuration), bytes.
// Region A holds the hash index during the clustering phase and the staged hits + member array + labels afterwards.
template <class C>
struct tile_smem_hash {
  static constexpr size_t kFwdMax = C::kFwdMax;
  static constexpr size_t kTile = C::kTile;
  static constexpr size_t kTileThreads = C::kThreads;
  static constexpr size_t tab = 0;                                      // u32 [kSlots] pixel << 14 | list head
  static constexpr size_t kIdx = kFwdMax + kBackCap;                    // local indices: tile + fwd halo, then back halo
  static constexpr size_t stoa = tab + (size_t)C::kSlots * 4;           // u32 [kIdx] toa - base
  static constexpr size_t nxt = stoa + kIdx * 4;                        // u16 [kIdx] next in pixel list
  static constexpr size_t sxy = nxt + kIdx * 2;                         // u32 [kTile]   y << 16 | x
  static constexpr size_t region_a = sxy + (size_t)kTile * 4;
  // reduction-phase aliases of region A
  static constexpr size_t stile = 0;                                    // uint4 [kTile]
  static constexpr size_t mem = stile + (size_t)kTile * 16;             // u16   [kTile]
  static constexpr size_t big = mem + (size_t)kTile * 2;                // u16   [kTile]
  static constexpr size_t mlabel = big + (size_t)kTile * 2;             // u32   [kTile]
  static constexpr size_t bacc = mlabel + (size_t)kTile * 4;           // big_acc [kMaxBig] (segmented big components)
  static constexpr size_t kMaxBig = kTile / 24 + 1;                     // kBigComp = 24
  static_assert(bacc + kMaxBig * 64 <= region_a, "reduction arrays alias region A");
  static constexpr size_t hb = region_a;                                // uint2 [kBackCap]
  static constexpr size_t par = hb + (size_t)kBackCap * 8;              // u32   [kFwdMax]
  static constexpr size_t csize = par + (size_t)kFwdMax * 4;            // u32   [kTile/2] (u16 pairs)
  static constexpr size_t crank = csize + (size_t)kTile * 2;            // u16   [kTile]
  static constexpr size_t coff = crank + (size_t)kTile * 2;             // u16   [kTile]
  static constexpr size_t eb = coff + (size_t)kTile * 2;                // u16   [kEdgeBuf * threads]
  static constexpr size_t eb_bytes = (size_t)kEdgeBuf * kTileThreads * 2;
  static constexpr size_t ccur = eb;                                    // u32   [kTile]   (alias)
  static_assert((size_t)kTile * 4 <= eb_bytes, "cursor alias");
  static_assert((size_t)kTileThreads * kEdgeBuf <= (size_t)kTile * 4, "edge owners alias crank + coff");
  static constexpr size_t copen = eb + eb_bytes;                        // u8    [kTile]
  static constexpr size_t hflag = copen + kTile;                        // u8    [kTile]
  static constexpr size_t total = hflag + kTile;
};
template <class C>
using tile_smem_layout = tile_smem_hash<C>;
template <class C>
constexpr size_t tile_smem_bytes() {
  return tile_smem_layout<C>::total;
}
constexpr uint32_t kBigComp = 24;  // components this large are reduced by whole warps
constexpr uint32_t kBigSeg = 256;  // member hits per warp work item of a large component (swept 64 / 128 / 256 / 512 / 1024: 256)

// Partial-sum accumulator of one large component (reduced in kBigSeg-hit
// segments by several warps, merged by shared-memory atomics; the warp that
// merges the last segment writes the record).  64 bytes.
struct big_acc {
  unsigned long long tot, sx, sy, stx, sty;
  uint32_t tmin, tmax, midx, cnt, segbase, done;
};
static_assert(sizeof(big_acc) == 64, "big_acc is 64 bytes");

// Block-wide exclusive scan (kTileThreads threads) of one u32 per thread.
template <int kTileThreads>
__device__ __forceinline__ uint32_t tile_block_scan(uint32_t v, uint32_t* total, uint32_t* s_wsum) {
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t x = v;
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
  *total = s_wsum[kTileThreads / 32 - 1];
  const uint32_t r = (warp ? s_wsum[warp - 1] : 0) + x - v;
  __syncthreads();
  return r;
}

// Feature accumulator.  Only hits with input index < n_owned contribute
// features (sharded runs: halo hits connect clusters but belong to the next
// rank); the label (smallest input index) is taken over all hits.
struct feat_acc {
  uint32_t tmin, tmax, midx, cnt;
  uint64_t tot, sx, sy, stx, sty;
  __device__ __forceinline__ void init() {
    tmin = 0xffffffffu;
    tmax = 0;
    midx = 0xffffffffu;
    cnt = 0;
    tot = sx = sy = stx = sty = 0;
  }
  // one staged hit: (toa - base, y<<16|x, tot, input index)
  __device__ __forceinline__ void add(const uint4 h, uint32_t n_owned) {
    midx = min(midx, h.w);
    if (h.w >= n_owned) return;
    const uint32_t x = h.y & 0xffffu, y = h.y >> 16, t = h.z;
    cnt += 1;
    tmin = min(tmin, h.x);
    tmax = max(tmax, h.x);
    tot += t;
    sx += x;
    sy += y;
    stx += (uint64_t)t * x;
    sty += (uint64_t)t * y;
  }
  __device__ __forceinline__ void warp_reduce() {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      tmin = min(tmin, __shfl_xor_sync(kFull, tmin, o));
      tmax = max(tmax, __shfl_xor_sync(kFull, tmax, o));
      midx = min(midx, __shfl_xor_sync(kFull, midx, o));
      cnt += __shfl_xor_sync(kFull, cnt, o);
      tot += __shfl_xor_sync(kFull, tot, o);
      sx += __shfl_xor_sync(kFull, sx, o);
      sy += __shfl_xor_sync(kFull, sy, o);
      stx += __shfl_xor_sync(kFull, stx, o);
      sty += __shfl_xor_sync(kFull, sty, o);
    }
  }
};

template <class C>
__global__ void __launch_bounds__(C::kThreads, C::kBlocks) k_tile_cc(tile_args a) {
  using SL = tile_smem_layout<C>;
  constexpr int kTile = C::kTile;
  constexpr int kTileThreads = C::kThreads;
  constexpr int kItemsPerThread = C::kItems;
  constexpr int kStageItems = C::kStageItems;
  extern __shared__ __align__(16) unsigned char sm[];
  // index arrays of the two configurations (only one set is used):
  // sparse -- column buckets ranked by (row, time); dense -- pixel hash
  uint32_t* tab = nullptr;    // pixel hash: pixel << 13 | list head, open addressing
  uint32_t* stoa = nullptr;   // toa - base by local index
  uint16_t* nxt = nullptr;    // next local index on the same pixel
  uint32_t* sxy = nullptr;    // y << 16 | x of tile hits
  {
    tab = reinterpret_cast<uint32_t*>(sm + SL::tab);
    stoa = reinterpret_cast<uint32_t*>(sm + SL::stoa);
    nxt = reinterpret_cast<uint16_t*>(sm + SL::nxt);
    sxy = reinterpret_cast<uint32_t*>(sm + SL::sxy);
  }
  uint4* stile = reinterpret_cast<uint4*>(sm + SL::stile);      // tile hits (toa - base, xy, tot, idx)
  uint16_t* mem = reinterpret_cast<uint16_t*>(sm + SL::mem);    // member array grouped by component
  uint16_t* big = reinterpret_cast<uint16_t*>(sm + SL::big);    // roots of large components
  uint2* hb = reinterpret_cast<uint2*>(sm + SL::hb);            // back halo, index order
  uint32_t* mlabel = reinterpret_cast<uint32_t*>(sm + SL::mlabel);  // label by tile root (reductions)
  uint32_t* par = reinterpret_cast<uint32_t*>(sm + SL::par);
  uint32_t* csize2 = reinterpret_cast<uint32_t*>(sm + SL::csize);  // component sizes, two u16 per word
  uint16_t* crank = reinterpret_cast<uint16_t*>(sm + SL::crank);  // stage rank by root
  uint16_t* coff = reinterpret_cast<uint16_t*>(sm + SL::coff);    // member offset by root
  uint16_t* eb = reinterpret_cast<uint16_t*>(sm + SL::eb);
  uint32_t* ccur = reinterpret_cast<uint32_t*>(sm + SL::ccur);
  uint8_t* copen = sm + SL::copen;
  uint8_t* hflag = sm + SL::hflag;  // per tile hit: bit0 open mark, bit1 overflow
  __shared__ uint64_t s_meta[8];
  __shared__ uint32_t s_wsum[kTileThreads / 32];
  __shared__ uint32_t s_chunk, s_nbig, s_bigq, s_nseg;
  __shared__ uint32_t s_app[3];  // output phase: open components / open hits / overflow of this CTA, then their list bases
  big_acc* bacc = reinterpret_cast<big_acc*>(sm + SL::bacc);

  const uint64_t n = a.n, dt = a.dt;
  const srec* __restrict__ S = a.S;
  const uint64_t t0 = (uint64_t)blockIdx.x * kTile;
  const uint64_t t1 = min(n, t0 + kTile);
  const uint32_t nt = (uint32_t)(t1 - t0);
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  long long t_phase = clock64();

  // ---- halo ranges: precomputed by k_tile_bounds (one load), else 32-ary
  // warp searches in the sorted stream (warp 0 the back halo, warp 1 the
  // forward halo) while the other warps clear the index
  if (a.tile_meta) {
    if (threadIdx.x < 8) s_meta[threadIdx.x] = a.tile_meta[(uint64_t)blockIdx.x * 8 + threadIdx.x];
    if (threadIdx.x == 0) {
      s_chunk = 0;
      s_nbig = 0;
      s_bigq = 0;
    }
  } else if (warp == 0) {
    const uint64_t toa_first = srec_key_toa(S, t0);
    const uint64_t blim = t0 > (uint64_t)kBackCap ? t0 - kBackCap : 0;
    // back halo: first position with toa + dt >= toa_first
    const uint64_t b0 = warp_lower_bound(blim, t0, [&](uint64_t p) { return srec_key_toa(S, p) + dt >= toa_first; });
    if (lane == 0) {
      const bool btrunc = b0 == blim && blim > 0 && srec_key_toa(S, blim - 1) + dt >= toa_first;
      s_meta[0] = b0;
      s_meta[2] = srec_key_toa(S, b0);               // base: the smallest staged ToA
      s_meta[3] = btrunc ? 1u : 0u;
      s_chunk = 0;
      s_nbig = 0;
      s_bigq = 0;
    }
  } else if (warp == 1) {
    const uint64_t toa_last = srec_key_toa(S, t1 - 1);
    const uint64_t flim = min(n, t1 + (uint64_t)C::kHalo);
    // forward halo: first position with toa > toa_last + dt
    const uint64_t f1 = warp_lower_bound(t1, flim, [&](uint64_t p) { return srec_key_toa(S, p) > toa_last + dt; });
    if (lane == 0) {
      const bool ftrunc = f1 == flim && flim < n && srec_key_toa(S, flim) <= toa_last + dt;
      s_meta[1] = f1;
      s_meta[4] = ftrunc ? srec_key_toa(S, f1) : 0;  // ToA of the first hit not staged
      s_meta[6] = srec_key_toa(S, f1 - 1);           // largest staged ToA
      s_meta[7] = ftrunc ? 2u : 0u;
    }
  }
  {
    for (uint32_t b = threadIdx.x; b < (uint32_t)C::kSlots; b += kTileThreads) tab[b] = 0xffffffffu;
  }
  for (uint32_t j = threadIdx.x; j < kTile; j += kTileThreads) {
    copen[j] = 0;
    hflag[j] = 0;
  }
  for (uint32_t w = threadIdx.x; w < kTile / 2; w += kTileThreads) csize2[w] = 0;
  if (threadIdx.x < 3) s_app[threadIdx.x] = 0;
  __syncthreads();
  TPX_PHASE(0);
  const uint64_t b0 = s_meta[0], f1 = s_meta[1], base = s_meta[2];
  const uint32_t flags = (uint32_t)(s_meta[3] | s_meta[7]);
  const bool btrunc = flags & 1u, ftrunc = flags & 2u;
  bool wide = ((s_meta[6] - base) >> 32) != 0;  // staged ToA span exceeds 32 bits
  const uint32_t nb = (uint32_t)(t0 - b0);
  const uint32_t m = (uint32_t)(f1 - t0);  // tile + forward halo
  const uint32_t nf = m - nt;
  const uint32_t dt32 = dt > 0xffffffffull ? 0xffffffffu : (uint32_t)dt;  // rel. ToAs differ by < 2^32

  const uint32_t W = a.width;
  auto slot_of_pixel = [&](uint32_t pix) { return (pix * 0x9E3779B1u) >> (32 - C::kSlotBits); };
  auto run_wide = [&]() {
    // Every hit becomes its own open component; the global pass does the work.
    for (uint32_t j = threadIdx.x; j < kTile; j += kTileThreads) {
      const bool v = j < nt;
      srec r;
      if (v) r = load_srec(S + t0 + j);
      const uint32_t oh = warp_append(v, &a.hdr->n_open_hits);
      const uint32_t oc = warp_append(v, &a.hdr->n_open_comps);
      const uint32_t ov = warp_append(v, &a.hdr->n_overflow);
      {
        const unsigned om = __ballot_sync(kFull, v);  // every hit is open
        if (lane_id() == 0) a.openbm[(t0 + j) >> 5] = om;
      }
      if (v) {
        const uint64_t pos = t0 + j;
        const bool own = r.idx < a.n_owned;
        const uint64_t toa = srec_toa(r), tot = own ? srec_tot(r) : 0, x = own ? srec_x(r) : 0,
                       y = own ? srec_y(r) : 0;
        a.parent_g[pos] = (uint32_t)pos;
        a.slot_of[pos] = (uint32_t)(t0 + j);
        stage_write(a.stage + t0 + j, r.idx, own ? 1 : 0, own ? toa : ~0ull, own ? toa : 0, tot, x, y, tot * x,
                    tot * y);
        a.open_hits[oh] = (uint32_t)pos;
        a.open_comps[oc] = (uint32_t)pos;
        a.overflow[ov] = make_uint2((uint32_t)pos, (uint32_t)pos + 1);
      }
    }
    if (threadIdx.x == 0) a.comp_count[blockIdx.x] = nt;
  };

  {}
  {
    // ---- stage: back halo; tile + forward halo into a pixel hash index.  Each
    // occupied pixel owns one open-addressing slot (pixel << 13 | head) and a
    // list of its local indices threaded through nxt[] -- a compact, per-CTA
    // stand-in for the paper's 256x256 "last hit per pixel" matrix (P:171,
    // P:310).  Inserts are lock-free pushes (atomicCAS on the slot word).
    auto staged = [&](uint32_t l) {
      const srec r = load_srec(S + t0 + l);
      return make_uint2((uint32_t)(srec_toa(r) - base), r.xy);
    };
    auto insert = [&](uint32_t l, uint2 e) {
      TPX_BOUND(l, C::kFwdMax);
      stoa[l] = e.x;
      if (l < nt) sxy[l] = e.y;
      par[l] = l;
      const uint32_t pix = (e.y >> 16) * W + (e.y & 0xffffu);
      uint32_t h = slot_of_pixel(pix);
      uint32_t cur = tab[h];
      for (;;) {
        const uint32_t ck = cur >> kHeadBits;
        if (ck != kPixEmpty && ck != pix) {  // another pixel: linear probing
          h = (h + 1) & (C::kSlots - 1);
          cur = tab[h];
          continue;
        }
        nxt[l] = ck == pix ? (uint16_t)(cur & kHeadMask) : kNil;
        const uint32_t old = atomicCAS(tab + h, cur, (pix << kHeadBits) | l);
        if (old == cur) break;
        cur = old;
      }
    };
    // back-halo hits go into the same pixel lists with local indices m + k:
    // a tile hit finds the earlier hits next to it through its 9 lookups
    // instead of scanning the back halo
    auto insert_back = [&](uint32_t l, uint2 e) {
      TPX_BOUND(l, SL::kIdx);
      stoa[l] = e.x;
      const uint32_t pix = (e.y >> 16) * W + (e.y & 0xffffu);
      uint32_t h = slot_of_pixel(pix);
      uint32_t cur = tab[h];
      for (;;) {
        const uint32_t ck = cur >> kHeadBits;
        if (ck != kPixEmpty && ck != pix) {
          h = (h + 1) & (C::kSlots - 1);
          cur = tab[h];
          continue;
        }
        nxt[l] = ck == pix ? (uint16_t)(cur & kHeadMask) : kNil;
        const uint32_t old = atomicCAS(tab + h, cur, (pix << kHeadBits) | l);
        if (old == cur) break;
        cur = old;
      }
    };
    if (!wide) {
      for (uint32_t k = threadIdx.x; k < nb; k += kTileThreads) {
        const srec r = load_srec(S + b0 + k);
        insert_back(m + k, make_uint2((uint32_t)(srec_toa(r) - base), r.xy));
      }
      if constexpr (C::kRegStage) {
        uint2 ev[kStageItems];
  #pragma unroll
        for (int q = 0; q < kStageItems; ++q) {  // all loads first, then the inserts
          const uint32_t l = threadIdx.x + q * kTileThreads;
          if (l < m) ev[q] = staged(l);
        }
  #pragma unroll
        for (int q = 0; q < kStageItems; ++q) {
          const uint32_t l = threadIdx.x + q * kTileThreads;
          if (l < m) insert(l, ev[q]);
        }
      } else {
        for (uint32_t l = threadIdx.x; l < m; l += kTileThreads) insert(l, staged(l));
      }
    }
    __syncthreads();
    TPX_PHASE(1);


    if (wide) {
      run_wide();
      return;
    }
  }
  TPX_PHASE(2);

  // ---- pixel-exact neighbour search.  For a hit at (x, y) with local index j
  // only the FIRST later hit on each of its 9 neighbouring pixels needs an edge
  // (later hits on that pixel are within dt of the first one and reach it via
  // their own same-pixel edge; this is the paper's last-hit-per-pixel rule,
  // P:171, read forwards).  Sparse: column x' in {x-1, x, x+1} is a
  // bucket sorted by (row, time); one binary search finds row y-1 after j,
  // then a short walk over rows y-1..y+1 takes the first entry per row with
  // local index > j.  Dense: per neighbouring pixel one hash probe sequence,
  // then the smallest local index > j in its list.  Either way the work per
  // hit is independent of the window density.
  const uint64_t first_unstaged = s_meta[4];
  const uint32_t wmax = W - 1;
  const uint32_t n_chunks = (nt + 31) / 32;
  for (;;) {
    uint32_t chunk = 0;
    if (lane == 0) chunk = atomicAdd(&s_chunk, 1u);
    chunk = __shfl_sync(kFull, chunk, 0);
    if (chunk >= n_chunks) break;
    const uint32_t j = chunk * 32 + lane;
    uint32_t ne = 0;
    if (j < nt) {
      uint32_t xy, tj;
      auto edge = [&](uint32_t lj) {
        if (ne < kEdgeBuf) eb[ne++ * kTileThreads + threadIdx.x] = (uint16_t)lj;
        else s_unite_il(par, j, lj);
      };
      bool back_near = false;
      {
        xy = sxy[j];
        tj = stoa[j];
        const uint32_t x = xy & 0xffffu, y = xy >> 16;
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy) {
#pragma unroll
          for (int dx = -1; dx <= 1; ++dx) {
            if ((dy < 0 && y == 0) || (dx < 0 && x == 0) || (dx > 0 && x == wmax)) continue;
            // row y + 1 == height gives a pixel id >= W * H: never present
            const uint32_t pix = (y + dy) * W + (x + dx);
            uint32_t h = slot_of_pixel(pix);
            uint32_t cur;
            while (((cur = tab[h]) >> kHeadBits) != pix) {
              if ((cur >> kHeadBits) == kPixEmpty) break;
              h = (h + 1) & (C::kSlots - 1);
            }
            if ((cur >> kHeadBits) != pix) continue;
            uint32_t best = 0xffffu;
            for (uint32_t q = cur & kHeadMask; q != kNil; q = nxt[q]) {
              TPX_BOUND(q, SL::kIdx);
              if (q >= m) back_near |= tj - stoa[q] <= dt32;  // back-halo hit (earlier)
              else if (q > j && q < best) best = q;
            }
            if (best != 0xffffu && stoa[best] - tj <= dt32) edge(best);
          }
        }
      }
      uint8_t fl = 0;
      if (ftrunc && first_unstaged <= base + tj + dt) fl = 3;  // window continues past the halo
      {
        // adjacent back-halo hit within dt, or a truncated back halo whose
        // earliest staged hit (relative ToA 0) is still within dt
        if (back_near || (t0 > 0 && btrunc && tj <= dt32)) fl |= 1;
      }
      hflag[j] = fl;
    }
    // unions of the buffered edges, spread over the warp (edge e of the
    // warp's E to lane e % 32; owner lanes in crank/coff, unused until the
    // compaction)
    {
      uint32_t pre = ne;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, pre, o);
        if (lane >= (unsigned)o) pre += y;
      }
      const uint32_t E = __shfl_sync(kFull, pre, 31);
      pre -= ne;
      uint8_t* owner = reinterpret_cast<uint8_t*>(crank) + (threadIdx.x >> 5) * (32 * kEdgeBuf);
      for (uint32_t k = 0; k < ne; ++k) owner[pre + k] = (uint8_t)lane;
      __syncwarp();
      const uint32_t wbase = threadIdx.x & ~31u;
      for (uint32_t b = 0; b < E; b += 32) {
        const uint32_t e = b + lane;
        const uint32_t L = e < E ? owner[e] : 0u;
        const uint32_t pL = __shfl_sync(kFull, pre, L);
        TPX_BOUND(e < E ? e - pL : 0u, kEdgeBuf);
        if (e < E) s_unite_il(par, chunk * 32 + L, eb[(e - pL) * kTileThreads + wbase + L]);
      }
    }
    __syncwarp();
  }
  __syncthreads();
  TPX_PHASE(3);

  // ---- flatten (read-only root walk; every stored value is a final root)
  for (uint32_t l = threadIdx.x; l < m; l += kTileThreads) {
    const uint32_t p0 = par[l];
    TPX_BOUND(p0, m);
    uint32_t c = p0, nx;
    while (c != (nx = par[c])) c = nx;
    if (c != p0) red_min_shared(par + l, c);  // atomic: other threads' walks read par[l]
  }
  __syncthreads();
  TPX_PHASE(4);

  // ---- sizes (warp-aggregated by root), open flags, cross pairs; stage the
  // tile hits for the reductions (region A is free now)
  srec rq[kItemsPerThread];
#pragma unroll
  for (int q = 0; q < kItemsPerThread; ++q) {
    const uint32_t j = threadIdx.x + q * kTileThreads;
    const uint32_t r = j < nt ? par[j] : 0xffffffffu;
    const unsigned peers = __match_any_sync(kFull, r);
    if (j < nt) {
      if ((__ffs(peers) - 1) == (int)lane) atomicAdd(csize2 + (r >> 1), (uint32_t)__popc(peers) << ((r & 1) * 16));
      if (hflag[j] & 1u) copen[r] = 1;
      rq[q] = load_srec(S + t0 + j);
      stile[j] = make_uint4((uint32_t)(srec_toa(rq[q]) - base), rq[q].xy, srec_tot(rq[q]), rq[q].idx);
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
  TPX_PHASE(5);

  // ---- compact roots (stage rank) and member offsets of multi-hit components
  {
    uint32_t packed[kItemsPerThread];
    uint32_t my = 0;
#pragma unroll
    for (int q = 0; q < kItemsPerThread; ++q) {
      const uint32_t j = threadIdx.x * kItemsPerThread + q;  // blocked for rank order
      uint32_t v = 0;
      if (j < nt && par[j] == j) {
        const uint32_t sz = (csize2[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
        v = 1u | ((sz >= 2 ? sz : 0u) << 16);
      }
      packed[q] = v;
      my += v;
    }
    uint32_t total;
    uint32_t ex = tile_block_scan<kTileThreads>(my, &total, s_wsum);
#pragma unroll
    for (int q = 0; q < kItemsPerThread; ++q) {
      const uint32_t j = threadIdx.x * kItemsPerThread + q;
      if (packed[q]) {
        crank[j] = (uint16_t)(ex & 0xffffu);
        coff[j] = (uint16_t)(ex >> 16);
        ccur[j] = 0;
        if ((packed[q] >> 16) >= kBigComp) big[atomicAdd(&s_nbig, 1u)] = (uint16_t)j;
      }
      ex += packed[q];
    }
    if (threadIdx.x == 0) a.comp_count[blockIdx.x] = total & 0xffffu;
  }
  __syncthreads();
  // member array: hits of every multi-hit component, contiguous per component
#pragma unroll
  for (int q = 0; q < kItemsPerThread; ++q) {
    const uint32_t j = threadIdx.x + q * kTileThreads;
    if (j < nt) {
      const uint32_t r = par[j];
      if (((csize2[r >> 1] >> ((r & 1) * 16)) & 0xffffu) >= 2) {
        const uint32_t mi = coff[r] + atomicAdd(&ccur[r], 1u);
        TPX_BOUND(mi, kTile);
        mem[mi] = (uint16_t)j;
      }
    }
  }
  if (warp == 0) {  // large components: segment counts -> work-item prefix; accumulators
    const uint32_t nbig = s_nbig;
    uint32_t run = 0;
    for (uint32_t g0 = 0; g0 < nbig; g0 += 32) {
      const uint32_t bi = g0 + lane;
      uint32_t ns = 0;
      if (bi < nbig) {
        TPX_BOUND(bi, SL::kMaxBig);
        const uint32_t r = big[bi], sz = (csize2[r >> 1] >> ((r & 1) * 16)) & 0xffffu;
        ns = (sz + kBigSeg - 1) / kBigSeg;
      }
      uint32_t x = ns;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= (unsigned)o) x += y;
      }
      if (bi < nbig) {
        big_acc& A = bacc[bi];
        A.tot = A.sx = A.sy = A.stx = A.sty = 0;
        A.tmin = 0xffffffffu;
        A.tmax = 0;
        A.midx = 0xffffffffu;
        A.cnt = 0;
        A.segbase = run + x - ns;
        A.done = 0;
      }
      run += __shfl_sync(kFull, x, 31);
    }
    if (lane == 0) s_nseg = run;
  }
  __syncthreads();
  TPX_PHASE(6);

  // ---- A7 reductions: small components by their root thread, large ones by
  // a whole warp (shuffle reduction); records staged, labels kept in smem
#pragma unroll
  for (int q = 0; q < kItemsPerThread; ++q) {
    const uint32_t j = threadIdx.x + q * kTileThreads;
    if (j < nt && par[j] == j) {
      const uint32_t sz = (csize2[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
      if (sz < kBigComp) {
        feat_acc f;
        f.init();
        if (sz == 1) {
          f.add(stile[j], a.n_owned);
        } else {
          const uint32_t o = coff[j];
          for (uint32_t k = 0; k < sz; ++k) f.add(stile[mem[o + k]], a.n_owned);
        }
        mlabel[j] = f.midx;
        TPX_BOUND(t0 + crank[j], t1);
        stage_write(a.stage + t0 + crank[j], f.midx, f.cnt, base + f.tmin, base + f.tmax, f.tot, f.sx, f.sy, f.stx,
                    f.sty);
      }
    }
  }
  // large components: kBigSeg-hit segments as warp work items (a 5000-hit
  // blob is spread over ~40 warps instead of holding one warp while the
  // others wait at the barrier)
  const uint32_t nbig = s_nbig, nseg = s_nseg;
  for (;;) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(&s_bigq, 1u);
    t = __shfl_sync(kFull, t, 0);
    if (t >= nseg) break;
    uint32_t bi = 0;  // the component whose segments contain t: (# segbase <= t) - 1
    for (uint32_t g0 = 0; g0 < nbig; g0 += 32) {
      const bool le = g0 + lane < nbig && bacc[g0 + lane].segbase <= t;
      bi += __popc(__ballot_sync(kFull, le));
    }
    bi -= 1;
    TPX_BOUND(bi, nbig);
    const uint32_t r = big[bi], sz = (csize2[r >> 1] >> ((r & 1) * 16)) & 0xffffu, o = coff[r];
    const uint32_t seg = t - bacc[bi].segbase, ns = (sz + kBigSeg - 1) / kBigSeg;
    const uint32_t k1 = min(sz, (seg + 1) * kBigSeg);
    feat_acc f;
    f.init();
    for (uint32_t k = seg * kBigSeg + lane; k < k1; k += 32) f.add(stile[mem[o + k]], a.n_owned);
    f.warp_reduce();
    if (lane == 0) {
      bool last = ns == 1;
      if (!last) {
        big_acc& A = bacc[bi];
        atomicAdd(&A.tot, (unsigned long long)f.tot);
        atomicAdd(&A.sx, (unsigned long long)f.sx);
        atomicAdd(&A.sy, (unsigned long long)f.sy);
        atomicAdd(&A.stx, (unsigned long long)f.stx);
        atomicAdd(&A.sty, (unsigned long long)f.sty);
        atomicMin(&A.tmin, f.tmin);
        atomicMax(&A.tmax, f.tmax);
        atomicMin(&A.midx, f.midx);
        atomicAdd(&A.cnt, f.cnt);
        __threadfence_block();
        last = atomicAdd(&A.done, 1u) == ns - 1;
        if (last) {  // every other segment merged before its done increment
          __threadfence_block();
          const volatile big_acc& V = A;
          f.tot = V.tot;
          f.sx = V.sx;
          f.sy = V.sy;
          f.stx = V.stx;
          f.sty = V.sty;
          f.tmin = V.tmin;
          f.tmax = V.tmax;
          f.midx = V.midx;
          f.cnt = V.cnt;
        }
      }
      if (last) {
        mlabel[r] = f.midx;
        TPX_BOUND(t0 + crank[r], t1);
        stage_write(a.stage + t0 + crank[r], f.midx, f.cnt, base + f.tmin, base + f.tmax, f.tot, f.sx, f.sy, f.stx,
                    f.sty);
      }
    }
  }
  __syncthreads();
  TPX_PHASE(7);

  // ---- outputs: labels, bitmap, open lists.  The open-list appends are
  // aggregated per CTA (warp counts -> shared offsets -> one global atomic
  // per list and CTA): with half of a heavy-ion stream's hits open, per-warp
  // global appends queue on the three list counters.
  uint32_t wofs[kItemsPerThread][3];
#pragma unroll
  for (int q = 0; q < kItemsPerThread; ++q) {
    const uint32_t j = threadIdx.x + q * kTileThreads;
    const bool v = j < nt;
    bool is_root = false, open = false;
    if (v) {
      const uint32_t r = par[j];
      is_root = r == j;
      open = copen[r] != 0;
    }
    const bool ovf = v && (hflag[j] & 2u);
    const unsigned mc = __ballot_sync(kFull, is_root && open), mh = __ballot_sync(kFull, v && open),
                   mo = __ballot_sync(kFull, ovf);
    uint32_t b0 = 0, b1 = 0, b2 = 0;
    if (lane == 0) {
      if (mc) b0 = atomicAdd(&s_app[0], (uint32_t)__popc(mc));
      if (mh) b1 = atomicAdd(&s_app[1], (uint32_t)__popc(mh));
      if (mo) b2 = atomicAdd(&s_app[2], (uint32_t)__popc(mo));
    }
    const unsigned lt = lanemask_lt();
    wofs[q][0] = __shfl_sync(kFull, b0, 0) + __popc(mc & lt);
    wofs[q][1] = __shfl_sync(kFull, b1, 0) + __popc(mh & lt);
    wofs[q][2] = __shfl_sync(kFull, b2, 0) + __popc(mo & lt);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t c0 = s_app[0], c1 = s_app[1], c2 = s_app[2];
    s_app[0] = c0 ? (uint32_t)atomicAdd(&a.hdr->n_open_comps, (unsigned long long)c0) : 0u;
    s_app[1] = c1 ? (uint32_t)atomicAdd(&a.hdr->n_open_hits, (unsigned long long)c1) : 0u;
    s_app[2] = c2 ? (uint32_t)atomicAdd(&a.hdr->n_overflow, (unsigned long long)c2) : 0u;
  }
  __syncthreads();
  const uint32_t base_oc = s_app[0], base_oh = s_app[1], base_ov = s_app[2];
#pragma unroll
  for (int q = 0; q < kItemsPerThread; ++q) {
    const uint32_t j = threadIdx.x + q * kTileThreads;
    const bool v = j < nt;
    uint32_t r = 0, label = 0;
    bool is_root = false, open = false;
    if (v) {
      r = par[j];
      is_root = r == j;
      open = copen[r] != 0;
      label = mlabel[r];
    }
    const uint64_t pos = t0 + j;
    if (is_root) {
      if (!open && label < a.n_owned) {
        set_label_bit(a.bitmap, label);
        if (a.first_of_label) a.first_of_label[label] = (uint32_t)pos;  // grouping: cluster's first sorted position
      }
      else a.slot_of[pos] = (uint32_t)(t0 + crank[j]);
    }
    {  // open word of these 32 positions (lane 0's position is 32-aligned; zeroed before the kernel)
      const unsigned om = __ballot_sync(kFull, v && open);
      if (lane_id() == 0 && om) a.openbm[pos >> 5] = om;
    }
    if (is_root && open) a.open_comps[base_oc + wofs[q][0]] = (uint32_t)pos;
    const bool ovf = v && (hflag[j] & 2u);
    if (v) {
      if (open) {
        a.parent_g[pos] = (uint32_t)(t0 + r);
        a.open_hits[base_oh + wofs[q][1]] = (uint32_t)pos;
      } else {
        store_label(a.labels, a.n_owned, a.lm, rq[q].idx, label);
      }
      if (ovf) a.overflow[base_ov + wofs[q][2]] = make_uint2((uint32_t)pos, (uint32_t)(t0 + m));  // staged part done in-tile
    }
  }
  TPX_PHASE(8);
}

}  // namespace tpx
