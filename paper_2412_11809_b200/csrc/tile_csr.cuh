// tile_csr.cuh -- A3 + A4 + A5 + A7 for one tile of the ToA-sorted stream
// (the sparse-stream configuration): a counting-sorted cell index and
// backward hooking.
//
// Same contract as k_tile_cell (tile_cell.cuh) and k_tile_cc: CTA k owns
// sorted positions [kT, kT+T), stages the forward halo (hits within dt_max
// after the tile) and the back halo (within dt_max before it), and leaves
// closed components final (labels, one 64-byte record, label bit) and open
// ones as partial records + global union-find entries for finalize.cuh.
//
// What differs is how neighbours are found and united:
//  * cell index in CSR form: every staged hit (back halo, tile, forward halo)
//    is counted into its 2x2-pixel cell (a 16-bit counter, the returned value
//    is its rank), the 128 x 128 counters are scanned into offsets and the
//    hits are scattered into a cell-ordered array of 8-byte entries
//    {toa - base, L << 20 | y << 10 | x} (L = staged index).  Cells of one row
//    are adjacent in that array, so the 3x3 neighbourhood of a pixel
//    ("the 8 neighboring pixels plus the pixel itself") is
//    covered by at most two contiguous ranges (one per cell row): the search
//    walks them with independent loads and a warp-uniform trip count (no
//    list pointers, no per-lane loop exits).  This is a compact, per-CTA
//    stand-in for the paper's 256x256 "last hit per pixel" matrix (l.171).
//  * one packed subtraction tests a candidate: Chebyshev adjacency in the two
//    10-bit coordinate fields, "earlier in (ToA, input index) order" from the
//    L field (one unsigned compare of the words); |dToA| <= dt_max (l.39,
//    inclusive) in a second compare.  Every edge is found once, from its later end.
//  * hooking: a hit's parent is set to its smallest earlier neighbour (one
//    CAS from par[j] == j; parent < child keeps the forest acyclic with the
//    earliest hit as root -- the paper's time-invariant, l.219-221).  Only
//    the remaining backward edges (~0.4 per hit on the mixed stream, against
//    ~1.1 edges per hit) need a union (lock-free CAS, larger root under
//    smaller); a lane keeps up to four of them in registers and unites them
//    after its visits (more: it re-walks its ranges and unites every edge).  If a union of another lane linked j
//    before j's hook, the hook CAS fails and j is united with its neighbour
//    instead, so hooks and unions may interleave freely.
//  * back-halo neighbours only mark the hit open (as in k_tile_cell);
//    forward-halo hits search too (their edges among themselves are true
//    edges and harmless), and those rooted in a tile component become cross
//    pairs for the global merge.
//  * flatten, compaction, segmented feature reduction and outputs are the
//    k_tile_cell ones (tile hits in local-index order on lanes).
// Sensor coordinates must be < 1024 (10-bit fields); wider sensors use
// k_tile_cell.
#pragma once
#include "tile_cell.cuh"

namespace tpx {

template <int kTileHits, int kThreadsPerCta, int kHaloHits, int kMinBlocks, int kCellW = 1, int kCellH = 1,
          int kCellBx = 7, int kCellBy = 7>
struct csr_cfg {
  static constexpr int kTile = kTileHits;
  static constexpr int kThreads = kThreadsPerCta;
  static constexpr int kItems = kTileHits / kThreadsPerCta;  // tile hits per thread
  static constexpr int kHalo = kHaloHits;
  static constexpr int kFwdMax = kTile + kHaloHits;          // tile + forward halo (local index l)
  static constexpr int kStage = kFwdMax / kThreads;          // staged hits per thread
  static constexpr int kBlocks = kMinBlocks;
  // cells of 2^kCellW x 2^kCellH pixels (both >= 2: a 3-pixel range spans at
  // most two cells), 2^kCellBx x 2^kCellBy of them (coordinates alias modulo
  // the grid; the packed compare checks true coordinates)
  static constexpr int kCwShift = kCellW, kChShift = kCellH, kCbx = kCellBx, kCby = kCellBy;
  static_assert(kCellW >= 1 && kCellH >= 1, "cells at least 2 pixels wide and high");
  static constexpr int kCells = 1 << (kCellBx + kCellBy);
  static constexpr int kMulti = kTile / 2;                   // components with >= 2 tile hits
  static constexpr int kCntWords = kCells / 2;               // two 16-bit counters per word
  static constexpr int kCntPerThread = kCntWords / kThreads; // scan: words per thread
  static_assert(kFwdMax % kThreads == 0 && kTile % kThreads == 0, "staging layout");
  static_assert(kBackCap + kFwdMax < 4096, "12-bit staged index in the entry word");
  static_assert(kCntWords % (4 * kThreads) == 0, "scan: uint4 words per thread");
  static_assert(kTile % ::tpx::kTile == 0 && kTile <= kMaxTile, "stage slots");
};
using csr_sparse = csr_cfg<2048, 512, TPX_CELL_HALO, 2>;
#ifndef TPX_CSR_JUMPS
#define TPX_CSR_JUMPS 2  // pointer-jumping rounds of the in-chunk hook targets (swept 0/1/2/3/5: 2 fastest)
#endif                 // 2x2-pixel cells, 128 x 128
constexpr uint32_t kCsrMaxCoord = 1023;  // 10-bit coordinate fields in the entry word

// Shared-memory carve-up, bytes.  Region A holds the cell counters / offsets
// during staging and search and the multi-hit accumulators afterwards; the
// extra-edge list aliases crank/aslot (both written only after the unions).
template <class C>
struct csr_smem {
  static constexpr size_t kM = C::kFwdMax, kT = C::kTile, kA = C::kMulti;
  static constexpr size_t off = 0;                                     // u16 [kCells + 2]
  static constexpr size_t off_end = (size_t)(C::kCells + 8) * 2;
  static constexpr size_t accN = 0;                                    // owned hit count
  static constexpr size_t accT = accN + kA * 4;                        // sum ToT
  static constexpr size_t accX = accT + kA * 4;                        // sum x
  static constexpr size_t accY = accX + kA * 4;                        // sum y
  static constexpr size_t accTX = accY + kA * 4;                       // sum ToT*x: low 16-bit halves [kA], high halves [kA]
  static constexpr size_t accTY = accTX + kA * 8;                      // sum ToT*y: same
  static constexpr size_t accE = accTY + kA * 8;                       // min input index
  static constexpr size_t accF = accE + kA * 4;                        // first owned local idx
  static constexpr size_t accG = accF + kA * 4;                        // last owned local idx
  static constexpr size_t acc_end = accG + kA * 4;
  static constexpr size_t region_a0 = acc_end > off_end ? acc_end : off_end;
  static constexpr size_t region_a = (region_a0 + 15) & ~(size_t)15;
  static constexpr size_t ent = region_a;                              // uint2 [kBackCap + kM], cell order (root_of u16 [kM] after the search)
  static constexpr size_t rec = ent + (size_t)(kBackCap + kM) * 8;     // uint2 [kM] (toa - base, y<<16|x)
  static constexpr size_t par = rec + kM * 8;                          // u32 [kM]
  static constexpr size_t crank = par + kM * 4;                        // u16 [kT] stage rank by root
  static constexpr size_t aslot = crank + kT * 2;                      // u16 [kT] accumulator slot by root
  static constexpr size_t hflag = aslot + kT * 2;                      // u8 [kT] bit0 open mark, bit1 overflow
  static constexpr size_t copen = hflag + kT;                          // u8 [kT]
  static constexpr size_t multi = copen + kT;                          // u8 [kT]
  static constexpr size_t total = multi + kT;
};
template <class C>
constexpr size_t csr_smem_bytes() {
  return csr_smem<C>::total;
}

// Entry word of a staged hit: L << 20 | y << 10 | x (x, y < 1024, L < 4096).
__device__ __forceinline__ uint32_t csr_pack(uint32_t xy, uint32_t L) {
  return (L << 20) | ((xy >> 16) << 10) | (xy & 0x3ffu);
}

// d = pe - pq + 0x401 (mod 2^32) for entry words pe (candidate) and pq
// (query): the low two 10-bit fields hold dx + 1 and dy + 1 (mod 1024), which
// are in [0, 2] iff |dx| <= 1 and |dy| <= 1 (coordinates < 1024: no other
// residue is reachable; a negative dx + 1 borrows from the y field, but then
// the x test already fails).  The candidate is earlier in the staged order
// iff Le < Lq, i.e. pe < pq (L is the top field and unique per hit).
__device__ __forceinline__ bool csr_back_adjacent(uint32_t pe, uint32_t pq) {
  const uint32_t d = pe - pq + 0x401u;
  return ((d & 0x3ffu) <= 2u) & ((d & 0xffc00u) <= 0x800u) & (pe < pq);
}

template <class C>
__global__ void __launch_bounds__(C::kThreads, C::kBlocks) k_tile_csr(tile_args a) {
  using SL = csr_smem<C>;
  constexpr int kT = C::kTile;
  constexpr int kTh = C::kThreads;
  constexpr uint32_t kMaskX = (1u << C::kCbx) - 1, kMaskY = (1u << C::kCby) - 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t sbase = opaque_u32((uint32_t)__cvta_generic_to_shared(smem_raw));
  auto sp = [&](size_t off) { return __cvta_shared_to_generic(sbase + (uint32_t)off); };
  uint16_t* off16 = reinterpret_cast<uint16_t*>(sp(SL::off));
  uint32_t* cnt32 = reinterpret_cast<uint32_t*>(sp(SL::off));
  uint32_t* accN = reinterpret_cast<uint32_t*>(sp(SL::accN));
  uint32_t* accT = reinterpret_cast<uint32_t*>(sp(SL::accT));
  uint32_t* accX = reinterpret_cast<uint32_t*>(sp(SL::accX));
  uint32_t* accY = reinterpret_cast<uint32_t*>(sp(SL::accY));
  uint32_t* accTX = reinterpret_cast<uint32_t*>(sp(SL::accTX));
  uint32_t* accTY = reinterpret_cast<uint32_t*>(sp(SL::accTY));
  uint32_t* accE = reinterpret_cast<uint32_t*>(sp(SL::accE));
  uint32_t* accF = reinterpret_cast<uint32_t*>(sp(SL::accF));
  uint32_t* accG = reinterpret_cast<uint32_t*>(sp(SL::accG));
  uint2* ent = reinterpret_cast<uint2*>(sp(SL::ent));
  uint2* rec = reinterpret_cast<uint2*>(sp(SL::rec));
  uint32_t* par = reinterpret_cast<uint32_t*>(sp(SL::par));
  uint16_t* root_of = reinterpret_cast<uint16_t*>(sp(SL::ent));  // after the search: root of each staged hit
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

  // ---- staging bounds (k_tile_bounds); all global loads issued at once:
  // the tile, the largest forward halo (kept if < f1) and back halo (>= b0)
  if (threadIdx.x < 8) s_meta[threadIdx.x] = a.tile_meta[(uint64_t)blockIdx.x * 8 + threadIdx.x];
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
    uint4* c4 = reinterpret_cast<uint4*>(cnt32);
    for (uint32_t b = threadIdx.x; b < (uint32_t)C::kCntWords / 4; b += kTh) c4[b] = make_uint4(0, 0, 0, 0);
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
  const uint32_t m = (uint32_t)(f1 - t0);  // tile + forward halo
  const uint32_t dt32 = dt > 0xffffffffull ? 0xffffffffu : (uint32_t)dt;
  const uint32_t wmax = a.width - 1, hmax = a.height - 1;
  auto cell_of = [&](uint32_t xy) {
    return ((((xy >> 16) >> C::kChShift) & kMaskY) << C::kCbx) | (((xy & 0xffffu) >> C::kCwShift) & kMaskX);
  };

  // ---- stage: rec[] in local-index order; count every staged hit into its
  // cell (the returned counter value is its rank inside the cell)
  uint32_t tidx[C::kItems], ttot2[(C::kItems + 1) / 2];  // ToT (16 bits) of tile hit q in half q & 1 of ttot2[q / 2]
  uint32_t key[C::kStage];  // cell << 12 | rank
  uint32_t keyb = 0, tb = 0, xyb = 0;
  const bool back_in = has_back && bpos >= b0;
#pragma unroll
  for (int s = 0; s < C::kStage; ++s) {
    const uint32_t l = threadIdx.x + s * kTh;
    if (s < C::kItems) {
      tidx[s] = rr[s].idx;
      if (s & 1) ttot2[s / 2] |= srec_tot(rr[s]) << 16;
      else ttot2[s / 2] = srec_tot(rr[s]);
    }
    key[s] = 0;
    if (l < m) {
      const uint32_t xy = rr[s].xy;
      TPX_BOUND(l, C::kFwdMax);
      rec[l] = make_uint2((uint32_t)(srec_toa(rr[s]) - base), xy);
      par[l] = l;
      const uint32_t c = cell_of(xy);
      TPX_BOUND(c >> 1, C::kCntWords);
      const uint32_t sh = (c & 1u) * 16u;
      const uint32_t old = atomicAdd(cnt32 + (c >> 1), 1u << sh);
      key[s] = (c << 12) | ((old >> sh) & 0xfffu);
    }
  }
  if (back_in) {
    xyb = rb.xy;
    tb = (uint32_t)(srec_toa(rb) - base);
    const uint32_t c = cell_of(xyb);
    const uint32_t sh = (c & 1u) * 16u;
    const uint32_t old = atomicAdd(cnt32 + (c >> 1), 1u << sh);
    keyb = (c << 12) | ((old >> sh) & 0xfffu);
  }
  __syncthreads();
  TPX_PHASE(1);

  // ---- exclusive scan of the 16-bit counters into cell offsets (in place):
  // a word holds counters lo | hi << 16; its offsets are run | (run + lo) << 16
  {
    constexpr int kV = C::kCntPerThread / 4;
    uint4* c4 = reinterpret_cast<uint4*>(cnt32) + threadIdx.x * kV;
    uint4 v[kV];
    uint32_t my = 0;
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      v[i] = c4[i];
      my += ((v[i].x * 0x10001u) >> 16) + ((v[i].y * 0x10001u) >> 16) + ((v[i].z * 0x10001u) >> 16) +
            ((v[i].w * 0x10001u) >> 16);
    }
    uint32_t total;
    uint32_t run = tile_block_scan<kTh>(my, &total, s_wsum);
    auto step = [&](uint32_t w) {
      const uint32_t o = run * 0x10001u + (w << 16);
      run += (w * 0x10001u) >> 16;
      return o;
    };
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      uint4 o;
      o.x = step(v[i].x);
      o.y = step(v[i].y);
      o.z = step(v[i].z);
      o.w = step(v[i].w);
      c4[i] = o;
    }
    if (threadIdx.x == 0) off16[C::kCells] = (uint16_t)total;
  }
  __syncthreads();
  TPX_PHASE(2);

  // ---- scatter the staged hits into cell order: {toa - base, L << 20 | y << 10 | x},
  // L = l + kBackCap (back-halo hits have l < 0)
#pragma unroll
  for (int s = 0; s < C::kStage; ++s) {
    const uint32_t l = threadIdx.x + s * kTh;
    if (l < m) {
      const uint2 e = rec[l];
      const uint32_t k = key[s];
      TPX_BOUND(off16[k >> 12] + (k & 0xfffu), kBackCap + C::kFwdMax);
      ent[off16[k >> 12] + (k & 0xfffu)] = make_uint2(e.x, csr_pack(e.y, l + kBackCap));
    }
  }
  TPX_BOUND(back_in ? off16[keyb >> 12] + (keyb & 0xfffu) : 0u, kBackCap + C::kFwdMax);
  if (back_in) ent[off16[keyb >> 12] + (keyb & 0xfffu)] = make_uint2(tb, csr_pack(xyb, kBackCap - (uint32_t)(t0 - bpos)));
  __syncthreads();
  TPX_PHASE(3);

  // ---- search (dynamic 32-hit chunks over tile + forward-halo hits): every
  // backward edge (e, j), e earlier than j.  bm = the smallest earlier
  // neighbour's staged index; every other neighbour (L >= kBackCap: tile or
  // forward halo) is an extra edge.  j is hooked under bm with a CAS (a union
  // of another lane may already have linked j: then it is united instead),
  // extras are united at the end of the chunk (the first two, from
  // registers) or at once (rare).  A back-halo neighbour (L < kBackCap) is
  // the smallest if present: it only marks j open.
  const uint64_t first_unstaged = s_meta[4];
  const uint32_t fwd_thr = !ftrunc ? 0xffffffffu
                           : (first_unstaged <= base + dt ? 0u : (uint32_t)min((unsigned long long)(first_unstaged - base - dt), 0xffffffffull));
  const uint32_t n_chunks = (m + 31) / 32;
  constexpr uint32_t kNone = 0xfffu;
  {
    for (;;) {
      uint32_t chunk = 0;
      if (lane == 0) chunk = atom_add_shared(&s_chunk, 1u);
      chunk = __shfl_sync(kFull, chunk, 0);
      if (chunk >= n_chunks) break;
      const uint32_t j = chunk * 32 + lane;
      const bool act = j < m;
      uint32_t tj = 0, xy = 0;
      if (act) {
        const uint2 hj = rec[j];
        tj = hj.x;
        xy = hj.y;
      }
      const uint32_t pj = csr_pack(xy, j + kBackCap);
      // the (up to) two cell rows around the pixel: one contiguous range each
      // unless the row's two cells alias across the 256-pixel wrap (sensors
      // wider than 256 only; handled below)
      const uint32_t x = xy & 0xffffu, y = xy >> 16;
      const uint32_t cx0 = (x ? x - 1 : 0) >> C::kCwShift, cx1 = min(x + 1, wmax) >> C::kCwShift;
      const uint32_t cy0 = (y ? y - 1 : 0) >> C::kChShift, cy1 = min(y + 1, hmax) >> C::kChShift;
      const uint32_t r0 = (cy0 & kMaskY) << C::kCbx, r1 = (cy1 & kMaskY) << C::kCbx;
      const uint32_t k0 = cx0 & kMaskX, k1 = cx1 & kMaskX;
      const bool two_y = act && cy1 != cy0;
      const bool wrap = act && cx1 != cx0 && k1 != k0 + 1;
      const uint32_t kend = k0 + ((cx1 != cx0 && !wrap) ? 2u : 1u);
      const uint32_t lo0 = off16[r0 + k0], lo1r = off16[r1 + k0];
      const uint32_t len0 = act ? (uint32_t)off16[r0 + kend] - lo0 : 0u;
      const uint32_t len1 = two_y ? (uint32_t)off16[r1 + kend] - lo1r : 0u;
      uint32_t bm = kNone, ne = 0;
      uint32_t exl = 0, exh = 0;  // up to four extra neighbours (16-bit staged indices), newest in the low half of exl
      auto visit = [&](uint32_t p, bool valid) {
        TPX_BOUND(p, (SL::total - SL::ent) / 8);
        const uint2 e = ent[p];  // p may run past the ranges (masked by valid; inside the CTA's smem)
        const bool edge = valid & csr_back_adjacent(e.y, pj) & (tj - e.x <= dt32);
        const uint32_t le = e.y >> 20;
        const uint32_t hi = max(bm, le);
        if (edge) bm = min(bm, le);
        // every neighbour but the smallest is an extra (back-halo ones excepted)
        const bool push = edge & (hi - (uint32_t)kBackCap < kNone - (uint32_t)kBackCap);
        // shift hi in (predicated, no branch): exh:exl = (exh:exl << 16) | hi
        const uint32_t nl = __byte_perm(hi, exl, 0x5410), nh = __byte_perm(exl, exh, 0x5432);
        exl = push ? nl : exl;
        exh = push ? nh : exh;
        ne += push ? 1u : 0u;
      };
      {
        const uint32_t V = len0 + len1;
        const uint32_t Vw = __reduce_max_sync(kFull, V);
        const uint32_t jump = lo1r - lo0 - len0;
#pragma unroll 4
        for (uint32_t k = 0; k < Vw; ++k) visit(lo0 + k + (k >= len0 ? jump : 0u), k < V);
      }
      if (__any_sync(kFull, wrap)) {  // sensors wider than 256: the cells at the wrap
        const uint32_t w0 = off16[r0 + k1], w1 = off16[r1 + k1];
        const uint32_t wl0 = wrap ? (uint32_t)off16[r0 + k1 + 1] - w0 : 0u;
        const uint32_t wl1 = (wrap && two_y) ? (uint32_t)off16[r1 + k1 + 1] - w1 : 0u;
        const uint32_t V = wl0 + wl1;
        const uint32_t Vw = __reduce_max_sync(kFull, V);
        const uint32_t jump = w1 - w0 - wl0;
        for (uint32_t k = 0; k < Vw; ++k) visit(w0 + k + (k >= wl0 ? jump : 0u), k < V);
      }
      // hook target: the smallest earlier neighbour; chains inside the chunk
      // are shortened by pointer jumping over the lanes (TPX_CSR_JUMPS rounds:
      // two shorten a chain 4-fold, which measured faster than the 5 rounds
      // that collapse any 32-lane chain -- the unions after the hook climb
      // what is left), a target in an earlier chunk by one hop to its current
      // parent
      {
        const uint32_t cb = chunk * 32;
        uint32_t tgt = (bm != kNone && bm >= (uint32_t)kBackCap) ? bm - kBackCap : j;
#pragma unroll
        for (int r = 0; r < TPX_CSR_JUMPS; ++r) {
          const uint32_t t2 = __shfl_sync(kFull, tgt, (tgt - cb) & 31u);
          if (tgt >= cb) tgt = t2;
        }
        if (act && tgt != j) {
          TPX_BOUND(tgt, m);
          TPX_BOUND(j, m);
          if (tgt < cb) tgt = par[tgt];
          if (atomicCAS(par + j, j, tgt) != j) s_unite_il(par, j, tgt);
        }
      }
      if (act) {
        if (ne <= 4) {
          for (uint32_t q = 0; q < ne; ++q) s_unite_il(par, j, ((q < 2 ? exl : exh) >> (16 * (q & 1)) & 0xffffu) - kBackCap);
        } else {  // more than four extras (very rare): unite every tile / forward-halo neighbour
          auto all = [&](uint32_t lo, uint32_t len) {
            for (uint32_t k = 0; k < len; ++k) {
              const uint2 e = ent[lo + k];
              const uint32_t le = e.y >> 20;
              if (csr_back_adjacent(e.y, pj) && tj - e.x <= dt32 && le >= (uint32_t)kBackCap) s_unite_il(par, j, le - kBackCap);
            }
          };
          all(lo0, len0);
          all(lo1r, len1);
          if (wrap) {
            all(off16[r0 + k1], (uint32_t)off16[r0 + k1 + 1] - off16[r0 + k1]);
            if (two_y) all(off16[r1 + k1], (uint32_t)off16[r1 + k1 + 1] - off16[r1 + k1]);
          }
        }
        if (j < nt) {
          TPX_BOUND(j, kT);
          uint8_t fl = (ftrunc && tj >= fwd_thr) ? 3 : 0;  // window continues past the halo
          // an earlier neighbour in the back halo, or one that was not staged
          if (bm < (uint32_t)kBackCap || (btrunc && tj <= dt32)) fl |= 1;
          hflag[j] = fl;
        }
      }
    }
  }
  __syncthreads();
  TPX_PHASE(4);

  // ---- flatten (one read-only root walk per staged hit into root_of[],
  // which reuses the entry array: par is not written, so no walk races a
  // store); multi-hit marks; open marks; cross pairs (forward-halo hits rooted
  // in a tile component)
  // the kStage walks of a thread advance in lockstep: their parent loads are
  // independent and overlap
  uint32_t rc[C::kStage];
#pragma unroll
  for (int s = 0; s < C::kStage; ++s) {
    const uint32_t l = threadIdx.x + s * kTh;
    rc[s] = l < m ? par[l] : 0u;
  }
  for (;;) {
    bool more = false;
#pragma unroll
    for (int s = 0; s < C::kStage; ++s) {
      const uint32_t nx = par[rc[s]];
      more |= nx != rc[s];
      rc[s] = nx;
    }
    if (!more) break;
  }
#pragma unroll
  for (int s = 0; s < C::kStage; ++s) {
    const uint32_t l = threadIdx.x + s * kTh;
    const uint32_t c = rc[s];
    bool joined = false;
    if (l < m) {
      TPX_BOUND(c, m);
      TPX_BOUND(c <= l ? 0u : 1u, 1u);  // roots are the smallest staged index of their tree
      root_of[l] = (uint16_t)c;
      if (l < nt) {
        if (c != l) multi[c] = 1;
        if (hflag[l] & 1u) copen[c] = 1;
      } else {
        joined = c < nt;
        if (joined) copen[c] = 1;
      }
    }
    if (__ballot_sync(kFull, joined)) {
      const uint32_t slot = warp_append(joined, &a.hdr->n_pairs);
      if (joined) a.pairs[slot] = make_uint2((uint32_t)(t0 + l), (uint32_t)(t0 + c));
    }
  }
  __syncthreads();
  TPX_PHASE(6);

  // ---- compaction: stage rank of every root, accumulator slot of every
  // multi-hit root (blocked order so ranks follow local index order: records
  // of a tile stay in label order, which keeps k_emit's stores coalesced)
  {
    uint32_t packed[C::kItems];
    uint32_t my = 0;
#pragma unroll
    for (int q = 0; q < C::kItems; ++q) {
      const uint32_t j = threadIdx.x * C::kItems + q;
      uint32_t v = 0;
      if (j < nt && root_of[j] == j) v = 1u | ((uint32_t)multi[j] << 16);
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
        TPX_BOUND(j, kT);
        TPX_BOUND(mu ? sl : 0u, C::kMulti);
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
  TPX_PHASE(7);

  // ---- A7: segmented run reduction (lanes = consecutive local indices)
  const unsigned lmask_le = lanemask_lt() | (1u << lane);
#pragma unroll
  for (int q = 0; q < C::kItems; ++q) {
    const uint32_t j = threadIdx.x + q * kTh;
    const bool valid = j < nt;
    const uint32_t r = valid ? (uint32_t)root_of[j] : 0xffffffffu;
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
    // 32-bit run sums (a run has <= 32 hits; x, y < 1024, ToT < 2^16): x + y
    // packed as x | y << 16 (sum of x < 2^15), ToT*x and ToT*y < 2^31
    uint32_t pxy = 0, tot = 0, stx = 0, sty = 0, midx = valid ? tidx[q] : 0xffffffffu;
    if (own) {
      const uint32_t xy = rec[j].y;
      pxy = xy;
      tot = (ttot2[q / 2] >> (16 * (q & 1))) & 0xffffu;
      stx = tot * (xy & 0xffffu);
      sty = tot * (xy >> 16);
    }
    for (uint32_t d = 1; d < maxlen; d <<= 1) {
      const uint32_t p2 = __shfl_up_sync(kFull, pxy, d), t2 = __shfl_up_sync(kFull, tot, d);
      const uint32_t m2 = __shfl_up_sync(kFull, midx, d);
      const uint32_t sx2 = __shfl_up_sync(kFull, stx, d), sy2 = __shfl_up_sync(kFull, sty, d);
      if (lane >= s + d) {
        pxy += p2;
        tot += t2;
        midx = min(midx, m2);
        stx += sx2;
        sty += sy2;
      }
    }
    if (lane == e && slot != 0xffffu) {
      TPX_BOUND(slot, C::kMulti);
      const uint32_t cnt = __popc(ownm);
      const uint32_t jbase = j - lane;
      if (cnt) {
        atomicAdd(accN + slot, cnt);
        atomicAdd(accT + slot, tot);
        atomicAdd(accX + slot, pxy & 0xffffu);
        atomicAdd(accY + slot, pxy >> 16);
        // ToT*x, ToT*y (< 2^31 per run) as low and high 16-bit halves in two
        // 32-bit sums each (<= 2048 runs per component: no overflow), so no
        // atomic waits for its return value to propagate a carry
        atomicAdd(accTX + slot, stx & 0xffffu);
        atomicAdd(accTX + slot + C::kMulti, stx >> 16);
        atomicAdd(accTY + slot, sty & 0xffffu);
        atomicAdd(accTY + slot + C::kMulti, sty >> 16);
      }
      atomicMin(accE + slot, midx);
      if (ownm) {
        atomicMin(accF + slot, jbase + __ffs(ownm) - 1);
        atomicMax(accG + slot, jbase + 31 - __clz(ownm));
      }
    }
  }
  __syncthreads();
  TPX_PHASE(8);

  // ---- outputs: records (roots), labels, bitmap, open lists
#pragma unroll
  for (int q = 0; q < C::kItems; ++q) {
    const uint32_t j = threadIdx.x + q * kTh;
    const bool v = j < nt;
    uint32_t r = 0, label = 0;
    bool is_root = false, open = false;
    if (v) {
      r = root_of[j];
      is_root = r == j;
      open = copen[r] != 0;
      const uint32_t sl = aslot[r];
      label = sl == 0xffffu ? tidx[q] : accE[sl];
      if (is_root) {
        TPX_BOUND(t0 + crank[j], t1);
        tpx_cluster_features* dst = a.stage + t0 + crank[j];
        if (sl == 0xffffu) {
          const bool own = tidx[q] < a.n_owned;
          const uint32_t xy = rec[j].y;
          const uint64_t tot = own ? (ttot2[q / 2] >> (16 * (q & 1))) & 0xffffu : 0, x = own ? (xy & 0xffffu) : 0, y = own ? (xy >> 16) : 0;
          const uint64_t toa = base + rec[j].x;
          stage_write(dst, label, own ? 1 : 0, own ? toa : base + 0xffffffffull, own ? toa : base, tot, x, y,
                      tot * x, tot * y);
        } else {
          const uint32_t cnt = accN[sl];
          TPX_BOUND(cnt ? accF[sl] : 0u, nt);
          TPX_BOUND(cnt ? accG[sl] : 0u, nt);
          const uint64_t tmin = cnt ? base + rec[accF[sl]].x : base + 0xffffffffull;
          const uint64_t tmax = cnt ? base + rec[accG[sl]].x : base;
          const uint64_t stx = ((uint64_t)accTX[sl + C::kMulti] << 16) + accTX[sl];
          const uint64_t sty = ((uint64_t)accTY[sl + C::kMulti] << 16) + accTY[sl];
          stage_write(dst, label, cnt, tmin, tmax, accT[sl], accX[sl], accY[sl], stx, sty);
        }
      }
    }
    const uint64_t pos = t0 + j;
    if (is_root) {
      TPX_BOUND(pos, a.n);
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
  TPX_PHASE(9);
}

}  // namespace tpx
