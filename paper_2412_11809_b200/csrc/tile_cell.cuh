// tile_cell.cuh -- A3 + A4 + A5 + A7 for one tile of the ToA-sorted stream
// with a 2x2-pixel cell index (the sparse-stream configuration).
//
// Same contract as k_tile_cc (tile_cc.cuh): CTA k owns sorted positions
// [kT, kT+T), stages the forward halo (hits within dt_max after the tile) and
// the back halo (within dt_max before it, openness only), and leaves closed
// components final (labels, one 64-byte record, label bit) and open ones as
// partial records + global union-find entries for finalize.cuh.
//
// What differs is the neighbour index, the union schedule and the feature
// reduction:
//  * cell index: every staged hit is pushed onto the list of its 2x2-pixel
//    cell (16-bit heads in shared memory, 128 x 128 cells; larger sensors
//    alias modulo 256 pixels and the true coordinates are compared).  The 3x3
//    neighbourhood of a pixel ("the 8 neighboring pixels plus
//    the pixel itself") always lies in at most 2 x 2 cells, so a hit reads 4
//    list heads and tests the few hits on those lists: later (local index >
//    j), within dt_max (l.39, inclusive) and Chebyshev-adjacent.  This is a
//    compact, per-CTA stand-in for the paper's 256x256 "last hit per pixel"
//    matrix (l.171, l.310): the work per hit is the number of hits near it in
//    space inside the staged time span, independent of the window density.
//    The first entry of each list is tested with predicated, unconditional
//    loads; longer lists continue in one warp-uniform loop, so the warp stays
//    converged (no per-lane re-execution of the code after the search).
//  * unions: each lane buffers its edges (j, q), q > j, and unites them
//    after its chunk's search (lock-free CAS, larger root under smaller ->
//    root = earliest hit, the paper's time-invariant l.219-221).
//  * features: tile hits are mapped to lanes in local-index (= time) order;
//    lanes with the same root form runs, a segmented warp scan sums each run
//    and the run's last lane folds it into the component's shared-memory
//    accumulator (32-bit integer atomics, order independent; the two 64-bit
//    sums carry explicitly).  First/last owned member (ToA min/max: local
//    index order is ToA order) and the owned count come from ballots, not
//    from the scan.  Single-hit components skip the accumulators entirely.
#pragma once
#include "tile_cc.cuh"

namespace tpx {

template <int kTileHits, int kThreadsPerCta, int kHaloHits, int kMinBlocks>
struct cell_cfg {
  static constexpr int kTile = kTileHits;
  static constexpr int kThreads = kThreadsPerCta;
  static constexpr int kItems = kTileHits / kThreadsPerCta;  // tile hits per thread
  static constexpr int kHalo = kHaloHits;
  static constexpr int kFwdMax = kTile + kHaloHits;          // tile + forward halo (local index l)
  static constexpr int kStage = kFwdMax / kThreads;          // staged hits per thread
  static constexpr int kBlocks = kMinBlocks;
  static constexpr int kCellBits = 7;                        // 2^7 x 2^7 cells of 2x2 pixels
  static constexpr int kCells = 1 << (2 * kCellBits);
  static constexpr int kMulti = kTile / 2;                   // components with >= 2 tile hits
  static_assert(kFwdMax % kThreads == 0 && kTile % kThreads == 0, "staging layout");
  static_assert(kFwdMax < 0xffff, "16-bit local indices");
  static_assert(kTile % ::tpx::kTile == 0 && kTile <= kMaxTile, "stage slots");
};
#ifndef TPX_CELL_HALO
#define TPX_CELL_HALO 512  // forward-halo cap; swept 512 / 1024 / 1536: 512 fastest (mixed tile 11.54 -> 11.36 ms per 200M)
#endif
using cell_sparse = cell_cfg<2048, 512, TPX_CELL_HALO, 2>;

// Shared-memory carve-up, bytes.  Region A holds the cell heads during the
// search and the multi-hit component accumulators afterwards; the edge buffer
// aliases crank/aslot (both written only after the search).
template <class C>
struct cell_smem {
  static constexpr size_t kM = C::kFwdMax, kT = C::kTile, kA = C::kMulti;
  static constexpr size_t heads = 0;                                   // u16 [kCells]
  // accumulators: u32 arrays [kMulti] (shared-memory atomics are native for
  // 32 bits only; the two 64-bit sums are (lo, hi) pairs with explicit carry)
  static constexpr size_t accN = 0;                                    // owned hit count
  static constexpr size_t accT = accN + kA * 4;                        // sum ToT
  static constexpr size_t accX = accT + kA * 4;                        // sum x
  static constexpr size_t accY = accX + kA * 4;                        // sum y
  static constexpr size_t accTX = accY + kA * 4;                       // sum ToT*x (lo [kA], hi [kA])
  static constexpr size_t accTY = accTX + kA * 8;                      // sum ToT*y (lo [kA], hi [kA])
  static constexpr size_t accE = accTY + kA * 8;                       // min input index
  static constexpr size_t accF = accE + kA * 4;                        // first owned local idx
  static constexpr size_t accG = accF + kA * 4;                        // last owned local idx
  static constexpr size_t acc_end = accG + kA * 4;
  static constexpr size_t heads_end = (size_t)C::kCells * 2;
  // edge owners during the search (u8 lane per buffered edge, one array of
  // 32 * kEdgeBuf per warp), after the heads in region A
  static constexpr size_t owner = heads_end;
  static constexpr size_t owner_end = owner + (size_t)(C::kThreads / 32) * 32 * kEdgeBuf;
  static constexpr size_t region_a0 = acc_end > heads_end ? acc_end : heads_end;
  static constexpr size_t region_a = region_a0 > owner_end ? region_a0 : owner_end;
  static constexpr size_t rec = region_a;                              // uint2 [kM] (toa - base, y<<16|x)
  static constexpr size_t par = rec + kM * 8;                          // u32 [kM]
  static constexpr size_t nxt = par + kM * 4;                          // u16 [kM]
  static constexpr size_t hb = nxt + kM * 2;                           // uint2 [kBackCap]
  static constexpr size_t crank = hb + (size_t)kBackCap * 8;           // u16 [kT] stage rank by root
  static constexpr size_t aslot = crank + kT * 2;                      // u16 [kT] accumulator slot by root
  static_assert(aslot == crank + kT * 2 && (size_t)kEdgeBuf * C::kThreads * 2 <= kT * 4,
                "per-lane edge buffers alias crank + aslot");
  static constexpr size_t hflag = aslot + kT * 2;                      // u8 [kT] bit0 open mark, bit1 overflow
  static constexpr size_t copen = hflag + kT;                          // u8 [kT]
  static constexpr size_t multi = copen + kT;                          // u8 [kT]
  static constexpr size_t total = multi + kT;
};
template <class C>
constexpr size_t cell_smem_bytes() {
  return cell_smem<C>::total;
}

// Exact 64-bit add into a (lo, hi) pair of u32 words with 32-bit atomics:
// the carry out of the low word is known from the value atomicAdd returns.
__device__ __forceinline__ void add_u64_pair(uint32_t* lo, uint32_t* hi, uint64_t v) {
  const uint32_t vl = (uint32_t)v;
  const uint32_t old = atomicAdd(lo, vl);
  const uint32_t vh = (uint32_t)(v >> 32) + ((uint32_t)(old + vl) < old ? 1u : 0u);
  if (vh) atomicAdd(hi, vh);
}

// Plain shared-memory fetch-add (the compiler would otherwise wrap a single
// lane's atomicAdd in its warp-aggregation sequence).
__device__ __forceinline__ uint32_t atom_add_shared(uint32_t* p, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;"
               : "=r"(r)
               : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v)
               : "memory");
  return r;
}

__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
  asm volatile("" : "+r"(x));
  return x;
}

// Every hit of a tile whose staged ToA span exceeds 32 bits becomes its own
// open component; the global pass does the work (same as k_tile_cc).
__device__ __forceinline__ void tile_run_wide(const tile_args& a, uint64_t t0, uint32_t nt, uint32_t tile_cap) {
  for (uint32_t j = threadIdx.x; j < tile_cap; j += blockDim.x) {
    const bool v = j < nt;
    srec r;
    if (v) r = load_srec(a.S + t0 + j);
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
      const uint64_t toa = srec_toa(r), tot = own ? srec_tot(r) : 0, x = own ? srec_x(r) : 0, y = own ? srec_y(r) : 0;
      a.parent_g[pos] = (uint32_t)pos;
      a.slot_of[pos] = (uint32_t)(t0 + j);
      stage_write(a.stage + t0 + j, r.idx, own ? 1 : 0, own ? toa : ~0ull, own ? toa : 0, tot, x, y, tot * x, tot * y);
      a.open_hits[oh] = (uint32_t)pos;
      a.open_comps[oc] = (uint32_t)pos;
      a.overflow[ov] = make_uint2((uint32_t)pos, (uint32_t)pos + 1);
    }
  }
  if (threadIdx.x == 0) a.comp_count[blockIdx.x] = nt;
}

// Per-tile staging bounds, one warp per tile (run before k_tile_cell so the
// tile kernel starts its loads at once instead of waiting for two dependent
// binary searches): the 8-word record k_tile_cell keeps in s_meta --
//   [0] b0 (back halo start)  [1] f1 (forward halo end)  [2] base ToA
//   [3] back-truncated flag   [4] ToA of the first unstaged hit (if truncated)
//   [5] ToA of the previous tile's last hit   [6] largest staged ToA
//   [7] forward-truncated flag (2)
// (the sort order itself is verified by k_sort_check right after the sort).
template <class C>
__global__ void __launch_bounds__(256) k_tile_bounds(const srec* __restrict__ S, uint64_t n, uint64_t dt,
                                                     uint32_t n_tiles, uint32_t verify_stride,
                                                     uint64_t* __restrict__ meta, dev_hdr* hdr) {
  const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned lane = lane_id();
  if (t >= n_tiles) return;
  const uint64_t t0 = (uint64_t)t * C::kTile, t1 = min(n, t0 + C::kTile);
  const uint64_t toa_first = srec_key_toa(S, t0), toa_last = srec_key_toa(S, t1 - 1);
  const uint64_t blim = t0 > (uint64_t)kBackCap ? t0 - kBackCap : 0;
  const uint64_t b0 = warp_lower_bound(blim, t0, [&](uint64_t p) { return srec_key_toa(S, p) + dt >= toa_first; });
  const uint64_t flim = min(n, t1 + (uint64_t)C::kHalo);
  const uint64_t f1 = warp_lower_bound(t1, flim, [&](uint64_t p) { return srec_key_toa(S, p) > toa_last + dt; });
  uint64_t v = 0;
  const bool btrunc = b0 == blim && blim > 0;
  const bool ftrunc = f1 == flim && flim < n;
  switch (lane) {
    case 0: v = b0; break;
    case 1: v = f1; break;
    case 2: v = srec_key_toa(S, b0); break;
    case 3: v = (btrunc && srec_key_toa(S, blim - 1) + dt >= toa_first) ? 1u : 0u; break;
    case 4: v = (ftrunc && srec_key_toa(S, flim) <= toa_last + dt) ? srec_key_toa(S, f1) : 0; break;
    case 5: v = t0 ? srec_key_toa(S, t0 - 1) : 0; break;
    case 6: v = srec_key_toa(S, f1 - 1); break;
    case 7: v = (ftrunc && srec_key_toa(S, flim) <= toa_last + dt) ? 2u : 0u; break;
    default: break;
  }
  if (lane < 8) meta[(uint64_t)t * 8 + lane] = v;
}

template <class C>
__global__ void __launch_bounds__(C::kThreads, C::kBlocks) k_tile_cell(tile_args a) {
  using SL = cell_smem<C>;
  constexpr int kT = C::kTile;
  constexpr int kTh = C::kThreads;
  constexpr uint32_t kCellMask = (1u << C::kCellBits) - 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // One opaque 32-bit shared base: without it the compiler rematerialises the
  // shared window base (S2R SR_CgaCtaId) inside the hot loops.
  const uint32_t sbase = opaque_u32((uint32_t)__cvta_generic_to_shared(smem_raw));
  auto sp = [&](size_t off) { return __cvta_shared_to_generic(sbase + (uint32_t)off); };
  uint16_t* heads = reinterpret_cast<uint16_t*>(sp(SL::heads));
  uint8_t* owner = reinterpret_cast<uint8_t*>(sp(SL::owner)) + (threadIdx.x >> 5) * (32 * kEdgeBuf);
  uint32_t* accN = reinterpret_cast<uint32_t*>(sp(SL::accN));
  uint32_t* accT = reinterpret_cast<uint32_t*>(sp(SL::accT));
  uint32_t* accX = reinterpret_cast<uint32_t*>(sp(SL::accX));
  uint32_t* accY = reinterpret_cast<uint32_t*>(sp(SL::accY));
  uint32_t* accTX = reinterpret_cast<uint32_t*>(sp(SL::accTX));
  uint32_t* accTY = reinterpret_cast<uint32_t*>(sp(SL::accTY));
  uint32_t* accE = reinterpret_cast<uint32_t*>(sp(SL::accE));
  uint32_t* accF = reinterpret_cast<uint32_t*>(sp(SL::accF));
  uint32_t* accG = reinterpret_cast<uint32_t*>(sp(SL::accG));
  uint2* rec = reinterpret_cast<uint2*>(sp(SL::rec));
  uint32_t* par = reinterpret_cast<uint32_t*>(sp(SL::par));
  uint16_t* nxt = reinterpret_cast<uint16_t*>(sp(SL::nxt));
  uint2* hb = reinterpret_cast<uint2*>(sp(SL::hb));
  uint16_t* crank = reinterpret_cast<uint16_t*>(sp(SL::crank));
  uint16_t* aslot = reinterpret_cast<uint16_t*>(sp(SL::aslot));
  uint8_t* hflag = reinterpret_cast<uint8_t*>(sp(SL::hflag));
  uint8_t* copen = reinterpret_cast<uint8_t*>(sp(SL::copen));
  uint8_t* multi = reinterpret_cast<uint8_t*>(sp(SL::multi));
  __shared__ uint64_t s_meta[8];
  __shared__ uint32_t s_wsum[kTh / 32];
  __shared__ uint32_t s_chunk;

  const uint64_t n = a.n, dt = a.dt;
  const srec* __restrict__ S = a.S;
  const uint64_t t0 = (uint64_t)blockIdx.x * kT;
  const uint64_t t1 = min(n, t0 + kT);
  const uint32_t nt = (uint32_t)(t1 - t0);
  const unsigned lane = lane_id();
  long long t_phase = clock64();

  // ---- staging bounds (k_tile_bounds); the tile's own records are loaded
  // right away (they do not depend on the bounds), the halo after the barrier
  if (threadIdx.x < 8) s_meta[threadIdx.x] = a.tile_meta[(uint64_t)blockIdx.x * 8 + threadIdx.x];
  // all global loads are issued here, before the bounds are known: the tile,
  // the largest forward halo the configuration stages (kept if < f1 after the
  // barrier) and the largest back halo (kept if >= b0) -- one memory round
  // trip per tile instead of three
  srec rr[C::kStage];
  const uint64_t lim = min(n, t1 + (uint64_t)C::kHalo);
#pragma unroll
  for (int s = 0; s < C::kStage; ++s) {
    const uint32_t l = threadIdx.x + s * kTh;
    if (t0 + l < lim) rr[s] = load_srec(S + t0 + l);
  }
  static_assert(kBackCap <= C::kThreads, "one back-halo record per thread");
  const bool has_back = threadIdx.x < (uint32_t)kBackCap && t0 + threadIdx.x >= (uint64_t)kBackCap;
  const uint64_t bpos = t0 + threadIdx.x - kBackCap;
  srec rb;
  if (has_back) rb = load_srec(S + bpos);
  if (threadIdx.x == 0) {
    s_chunk = 0;
  }
  {
    uint4* h4 = reinterpret_cast<uint4*>(heads);
    for (uint32_t b = threadIdx.x; b < (uint32_t)C::kCells / 8; b += kTh) h4[b] = make_uint4(~0u, ~0u, ~0u, ~0u);
    uint32_t* f4 = reinterpret_cast<uint32_t*>(hflag);  // hflag, copen, multi are contiguous
    for (uint32_t w = threadIdx.x; w < 3 * (uint32_t)kT / 4; w += kTh) f4[w] = 0;
  }
  __syncthreads();
  TPX_PHASE(0);
  const uint64_t b0 = s_meta[0], f1 = s_meta[1], base = s_meta[2];
  const uint32_t flags = (uint32_t)(s_meta[3] | s_meta[7]);
  const bool btrunc = flags & 1u, ftrunc = flags & 2u;
  if (((s_meta[6] - base) >> 32) != 0) {  // staged ToA span exceeds 32 bits
    tile_run_wide(a, t0, nt, kT);
    return;
  }
  const uint32_t nb = (uint32_t)(t0 - b0);
  const uint32_t m = (uint32_t)(f1 - t0);  // tile + forward halo
  const uint32_t dt32 = dt > 0xffffffffull ? 0xffffffffu : (uint32_t)dt;
  const uint32_t wmax = a.width - 1, hmax = a.height - 1;

  // ---- stage: back halo; tile + forward halo into rec[] and the cell lists.
  // Tile hits' input index and ToT stay in registers (thread owns j = tid + q*kTh).
  uint32_t tidx[C::kItems], ttot[C::kItems];
  if (has_back && bpos >= b0) hb[bpos - b0] = make_uint2((uint32_t)(srec_toa(rb) - base), rb.xy);
  {
#pragma unroll
    for (int s = 0; s < C::kStage; ++s) {
      const uint32_t l = threadIdx.x + s * kTh;
      if (s < C::kItems) {
        tidx[s] = rr[s].idx;
        ttot[s] = srec_tot(rr[s]);
      }
      if (l < m) {
        const uint32_t xy = rr[s].xy;
        rec[l] = make_uint2((uint32_t)(srec_toa(rr[s]) - base), xy);
        par[l] = l;
        const uint32_t c = ((((xy >> 16) >> 1) & kCellMask) << C::kCellBits) | (((xy & 0xffffu) >> 1) & kCellMask);
        // lock-free push onto the cell list: 16-bit head inside a 32-bit word
        uint32_t* w32 = reinterpret_cast<uint32_t*>(heads) + (c >> 1);
        const uint32_t sh = (c & 1u) * 16u;
        uint32_t cur = *w32;
        for (;;) {
          const uint32_t nw = (cur & ~(0xffffu << sh)) | (l << sh);
          const uint32_t old = atomicCAS(w32, cur, nw);
          if (old == cur) break;
          cur = old;
        }
        nxt[l] = (uint16_t)(cur >> sh);
      }
    }
  }
  __syncthreads();
  TPX_PHASE(1);

  // ---- neighbour search (dynamic 32-hit chunks).  Edges (j, q) with q > j
  // only: every tile pair is found from its earlier end, tile-halo pairs from
  // the tile end; halo-halo pairs belong to the next tile.
  // flag thresholds in relative ToA (32-bit compares per hit):
  //  fwd: window continues past the staged halo  <=>  tj >= fwd_thr (if ftrunc)
  //  back: an earlier tile could reach the hit   <=>  tj <= back_thr (if t0 > 0)
  const uint64_t prev_last = s_meta[5];
  const uint64_t first_unstaged = s_meta[4];
  const uint32_t fwd_thr = !ftrunc ? 0xffffffffu
                           : (first_unstaged <= base + dt ? 0u : (uint32_t)min((unsigned long long)(first_unstaged - base - dt), 0xffffffffull));
  const bool fwd_any = ftrunc;
  const bool back_any = t0 > 0 && prev_last + dt >= base;
  const uint32_t back_thr = back_any ? (uint32_t)min((unsigned long long)(prev_last + dt - base), 0xffffffffull) : 0u;
  const uint32_t n_chunks = (nt + 31) / 32;
  uint16_t* eb = crank;  // per-lane edge buffers (kEdgeBuf per thread), alias of crank/aslot
  {
    for (;;) {
      uint32_t chunk = 0;
      if (lane == 0) chunk = atom_add_shared(&s_chunk, 1u);
      chunk = __shfl_sync(kFull, chunk, 0);
      if (chunk >= n_chunks) break;
      const uint32_t j = chunk * 32 + lane;
      const bool act = j < nt;
      uint32_t ne = 0;
      uint32_t xy = 0, tj = 0;
      // q may be kNil: loads are unconditional (clamped index) so the common
      // case runs predicated; only a found edge branches
      auto visit = [&](uint32_t q) {
        const uint32_t qq = q < m ? q : 0u;
        const uint2 e = rec[qq];
        const bool ok = (q > j) & (q < m) & (e.x - tj <= dt32) & adjacent(xy, e.y);
        // branch-free append: the slot is written every time and kept only
        // if ok (ne advances); a full buffer unites directly (rare)
        const uint32_t slot = ne < kEdgeBuf ? ne : kEdgeBuf - 1;
        const bool full = ne >= kEdgeBuf;
        if (!full) eb[slot * kTh + threadIdx.x] = (uint16_t)q;
        ne += (ok & !full) ? 1u : 0u;
        if (ok & full) s_unite_il(par, j, q);
      };
      uint64_t hq = ~0ull;  // queue of list continuations (16 bits each, kNil-padded)
      if (act) {
        const uint2 hj = rec[j];
        xy = hj.y;
        tj = hj.x;
      }
      const uint32_t x = xy & 0xffffu, y = xy >> 16;
      {
        uint32_t hd[4];  // list heads of the (up to) 2 x 2 cells
        {
          const uint32_t cx0 = (x ? x - 1 : 0) >> 1, cx1 = min(x + 1, wmax) >> 1;
          const uint32_t cy0 = (y ? y - 1 : 0) >> 1, cy1 = min(y + 1, hmax) >> 1;
          const uint32_t r0 = (cy0 & kCellMask) << C::kCellBits, r1 = (cy1 & kCellMask) << C::kCellBits;
          const uint32_t k0 = cx0 & kCellMask, k1 = cx1 & kCellMask;
          const bool two_x = cx1 != cx0, two_y = cy1 != cy0;
          hd[0] = heads[r0 | k0];
          hd[1] = heads[r0 | k1];
          hd[2] = heads[r1 | k0];
          hd[3] = heads[r1 | k1];
          if (!act) hd[0] = kNil;
          if (!act || !two_x) hd[1] = kNil;
          if (!act || !two_y) hd[2] = kNil;
          if (!act || !two_x || !two_y) hd[3] = kNil;
        }
        // first entry of every list: independent loads, no loop
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t q = hd[c];
          const uint32_t nq = nxt[q < m ? q : 0u];
          visit(q);
          hd[c] = q == kNil ? kNil : nq;
        }
#pragma unroll
        for (int c = 3; c >= 0; --c)
          if (hd[c] != kNil) hq = (hq << 16) | hd[c];
      }
      // remaining entries: warp-uniform loop (the warp stays converged, so the
      // code after it runs once per chunk)
      while (__any_sync(kFull, ((uint32_t)hq & 0xffffu) != kNil)) {
        const uint32_t q = (uint32_t)hq & 0xffffu;
        if (q != kNil) {
          const uint32_t nq = nxt[q];
          hq = nq == kNil ? ((hq >> 16) | 0xffff000000000000ull) : ((hq & ~0xffffull) | nq);
          visit(q);
        }
      }
      if (act) {
        uint8_t fl = (fwd_any && tj >= fwd_thr) ? 3 : 0;  // window continues past the halo
        if (back_any && tj <= back_thr) {                 // could an earlier tile reach it?
          bool found = false;
          int lb = (int)nb - 1;
          for (; lb >= 0; --lb) {
            const uint2 g = hb[lb];
            if (tj - g.x > dt32) break;
            if (adjacent(xy, g.y)) {
              found = true;
              break;
            }
          }
          if (found || (lb < 0 && btrunc)) fl |= 1;
        }
        hflag[j] = fl;
      }
      // unions of the buffered edges (larger root under smaller), spread over
      // the warp: edge e of the warp's E goes to lane e % 32, so a round
      // keeps every lane busy instead of iterating max(ne) times with the
      // lanes that have few edges idle
      {
        uint32_t pre = ne;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, pre, o);
          if (lane >= (unsigned)o) pre += y;
        }
        const uint32_t E = __shfl_sync(kFull, pre, 31);
        pre -= ne;
        for (uint32_t k = 0; k < ne; ++k) owner[pre + k] = (uint8_t)lane;
        __syncwarp();
        const uint32_t wbase = threadIdx.x & ~31u;
        for (uint32_t b = 0; b < E; b += 32) {
          const uint32_t e = b + lane;
          const uint32_t L = e < E ? owner[e] : 0u;
          const uint32_t pL = __shfl_sync(kFull, pre, L);
          if (e < E) s_unite_il(par, chunk * 32 + L, eb[(e - pL) * kTh + wbase + L]);
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  TPX_PHASE(3);

  // ---- flatten; multi-hit marks; open marks; cross pairs (halo hits that
  // joined a tile component).  Roots are found first (reads only), stored
  // after a barrier: no thread writes a parent another thread's walk reads.
  uint32_t root[C::kStage];
#pragma unroll
  for (int s = 0; s < C::kStage; ++s) {
    const uint32_t l = threadIdx.x + s * kTh;
    uint32_t c = 0;
    if (l < m) {
      uint32_t nx;
      c = par[l];
      while (c != (nx = par[c])) c = nx;
    }
    root[s] = c;
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < C::kStage; ++s) {
    const uint32_t l = threadIdx.x + s * kTh;
    const uint32_t c = root[s];
    bool joined = false;
    if (l < m) {
      par[l] = c;
      if (l < nt) {
        if (c != l) multi[c] = 1;
        if (hflag[l] & 1u) copen[c] = 1;
      } else {
        joined = c != l;
        if (joined) copen[c] = 1;
      }
    }
    if (__ballot_sync(kFull, joined)) {
      const uint32_t slot = warp_append(joined, &a.hdr->n_pairs);
      if (joined) a.pairs[slot] = make_uint2((uint32_t)(t0 + l), (uint32_t)(t0 + c));
    }
  }
  __syncthreads();
  TPX_PHASE(4);

  // ---- compaction: stage rank of every root, accumulator slot of every
  // multi-hit root (blocked order so ranks follow local index order)
  {
    uint32_t packed[C::kItems];
    uint32_t my = 0;
#pragma unroll
    for (int q = 0; q < C::kItems; ++q) {
      const uint32_t j = threadIdx.x * C::kItems + q;
      uint32_t v = 0;
      if (j < nt && par[j] == j) v = 1u | ((uint32_t)multi[j] << 16);
      packed[q] = v;
      my += v;
    }
    uint32_t total;
    uint32_t ex = tile_block_scan<kTh>(my, &total, s_wsum);
#pragma unroll
    for (int q = 0; q < C::kItems; ++q) {
      const uint32_t j = threadIdx.x * C::kItems + q;
      if (packed[q]) {
        crank[j] = (uint16_t)(ex & 0xffffu);
        const bool mu = packed[q] >> 16;
        const uint32_t sl = ex >> 16;
        aslot[j] = mu ? (uint16_t)sl : (uint16_t)0xffffu;
        if (mu) {
          accN[sl] = 0;
          accT[sl] = 0;
          accX[sl] = 0;
          accY[sl] = 0;
          accTX[sl] = 0;
          accTX[sl + C::kMulti] = 0;
          accTY[sl] = 0;
          accTY[sl + C::kMulti] = 0;
          accE[sl] = 0xffffffffu;
          accF[sl] = 0xffffffffu;
          accG[sl] = 0;
        }
      }
      ex += packed[q];
    }
    if (threadIdx.x == 0) a.comp_count[blockIdx.x] = total & 0xffffu;
  }
  __syncthreads();
  TPX_PHASE(6);

  // ---- A7: segmented run reduction (lanes = consecutive local indices)
  const unsigned lmask_le = lanemask_lt() | (1u << lane);
#pragma unroll
  for (int q = 0; q < C::kItems; ++q) {
    const uint32_t j = threadIdx.x + q * kTh;
    const bool valid = j < nt;
    const uint32_t r = valid ? par[j] : 0xffffffffu;
    const uint32_t slot = valid ? aslot[r] : 0xffffu;
    const bool own = valid && tidx[q] < a.n_owned;
    const uint32_t prev = __shfl_up_sync(kFull, r, 1);
    const bool head = lane == 0 || prev != r;
    const unsigned heads_m = __ballot_sync(kFull, head);
    const unsigned any_multi = __ballot_sync(kFull, slot != 0xffffu);
    if (!any_multi) continue;  // warp-uniform: only single-hit components here
    const uint32_t s = 31 - __clz(heads_m & lmask_le);
    const unsigned later = heads_m & ~lmask_le;
    const uint32_t e = later ? (uint32_t)__ffs(later) - 2 : 31u;
    const unsigned run = (e == 31 ? kFull : ((2u << e) - 1u)) & ~((1u << s) - 1u);
    const unsigned ownm = __ballot_sync(kFull, own) & run;
    const uint32_t len = e - s + 1;
    const uint32_t maxlen = __reduce_max_sync(kFull, slot != 0xffffu ? len : 1u);
    uint32_t x = 0, y = 0, tot = 0, midx = valid ? tidx[q] : 0xffffffffu;
    uint64_t stx = 0, sty = 0;
    if (own) {
      const uint32_t xy = rec[j].y;
      x = xy & 0xffffu;
      y = xy >> 16;
      tot = ttot[q];
      stx = (uint64_t)tot * x;
      sty = (uint64_t)tot * y;
    }
    for (uint32_t d = 1; d < maxlen; d <<= 1) {
      const uint32_t x2 = __shfl_up_sync(kFull, x, d), y2 = __shfl_up_sync(kFull, y, d);
      const uint32_t t2 = __shfl_up_sync(kFull, tot, d), m2 = __shfl_up_sync(kFull, midx, d);
      const uint64_t sx2 = __shfl_up_sync(kFull, stx, d), sy2 = __shfl_up_sync(kFull, sty, d);
      if (lane >= s + d) {
        x += x2;
        y += y2;
        tot += t2;
        midx = min(midx, m2);
        stx += sx2;
        sty += sy2;
      }
    }
    if (lane == e && slot != 0xffffu) {
      const uint32_t cnt = __popc(ownm);
      const uint32_t jbase = j - lane;
      if (cnt) {
        atomicAdd(accN + slot, cnt);
        atomicAdd(accT + slot, tot);
        atomicAdd(accX + slot, x);
        atomicAdd(accY + slot, y);
        add_u64_pair(accTX + slot, accTX + slot + C::kMulti, stx);
        add_u64_pair(accTY + slot, accTY + slot + C::kMulti, sty);
      }
      atomicMin(accE + slot, midx);
      if (ownm) {
        atomicMin(accF + slot, jbase + __ffs(ownm) - 1);
        atomicMax(accG + slot, jbase + 31 - __clz(ownm));
      }
    }
  }
  __syncthreads();
  TPX_PHASE(7);

  // ---- outputs: records (roots), labels, bitmap, open lists
#pragma unroll
  for (int q = 0; q < C::kItems; ++q) {
    const uint32_t j = threadIdx.x + q * kTh;
    const bool v = j < nt;
    uint32_t r = 0, label = 0;
    bool is_root = false, open = false;
    if (v) {
      r = par[j];
      is_root = r == j;
      open = copen[r] != 0;
      const uint32_t sl = aslot[r];
      label = sl == 0xffffu ? tidx[q] : accE[sl];
      if (is_root) {
        tpx_cluster_features* dst = a.stage + t0 + crank[j];
        if (sl == 0xffffu) {
          const bool own = tidx[q] < a.n_owned;
          const uint32_t xy = rec[j].y;
          const uint64_t tot = own ? ttot[q] : 0, x = own ? (xy & 0xffffu) : 0, y = own ? (xy >> 16) : 0;
          const uint64_t toa = base + rec[j].x;
          stage_write(dst, label, own ? 1 : 0, own ? toa : base + 0xffffffffull, own ? toa : base, tot, x, y,
                      tot * x, tot * y);
        } else {
          const uint32_t cnt = accN[sl];
          const uint64_t tmin = cnt ? base + rec[accF[sl]].x : base + 0xffffffffull;
          const uint64_t tmax = cnt ? base + rec[accG[sl]].x : base;
          const uint64_t stx = ((uint64_t)accTX[sl + C::kMulti] << 32) | accTX[sl];
          const uint64_t sty = ((uint64_t)accTY[sl + C::kMulti] << 32) | accTY[sl];
          stage_write(dst, label, cnt, tmin, tmax, accT[sl], accX[sl], accY[sl], stx, sty);
        }
      }
    }
    const uint64_t pos = t0 + j;
    if (is_root) {
      if (!open && label < a.n_owned) {
        set_label_bit(a.bitmap, label);
        if (a.first_of_label) a.first_of_label[label] = (uint32_t)pos;  // grouping: cluster's first sorted position
      }
      else a.slot_of[pos] = (uint32_t)(t0 + crank[j]);
    }
    const bool ovf = v && (hflag[j] & 2u);
    if (__ballot_sync(kFull, (v && open) || ovf)) {  // warp-uniform: most warps have no open hit
      const unsigned om = __ballot_sync(kFull, v && open);  // open word (zeroed before the kernel)
      if (lane_id() == 0 && om) a.openbm[pos >> 5] = om;  // lane 0's position is 32-aligned
      const uint32_t oc = warp_append(is_root && open, &a.hdr->n_open_comps);
      if (is_root && open) a.open_comps[oc] = (uint32_t)pos;
      const uint32_t oh = warp_append(v && open, &a.hdr->n_open_hits);
      const uint32_t ov = warp_append(ovf, &a.hdr->n_overflow);
      if (v && open) a.open_hits[oh] = (uint32_t)pos;
      if (ovf) a.overflow[ov] = make_uint2((uint32_t)pos, (uint32_t)(t0 + m));  // staged part done in-tile
    }
    if (v) {
      if (open) {
        a.parent_g[pos] = (uint32_t)(t0 + r);
      } else {
        store_label(a.labels, a.n_owned, a.lm, tidx[q], label);
      }
    }
  }
  TPX_PHASE(8);
}

}  // namespace tpx
