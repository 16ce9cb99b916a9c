// tpx_cluster.cu -- the C ABI (include/tpx_cluster.h) over the sm_100a kernels.
//
// Fast path per run (one host synchronisation, at the end):
//   k_window_sort      bounded-disorder ToA sort            (sort_window.cuh)
//   k_tile_cc          tile-local window search + union-find, labels and
//                      features of tile-closed components  (tile_cc.cuh)
//   k_overflow_unions, k_pair_unions, k_merge_open, k_open_labels
//                      global merge of border-crossing components
//   k_popc + scan + k_emit
//                      ordinals by label, ordered feature records (finalize.cuh)
// Fallbacks (taken only when the fast path reports it cannot be exact):
//   wider sort window -> global LSD radix sort (sort.cuh) -> global
//   union-find pipeline (cluster.cuh).
#include <nvtx3/nvToolsExt.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "cluster.cuh"
#include "common.cuh"
#include "finalize.cuh"
#include "tile_cell.cuh"
#include "tile_csr.cuh"
#include "group.cuh"
#include "variant.cuh"
#include "scan.cuh"
#include "sort.cuh"
#include "sort_window.cuh"
#include "radix_onesweep.cuh"
#include "tile_cc.cuh"

using namespace tpx;

// NVTX range over a stage's launches (host timeline; header-only NVTX v3,
// a no-op unless a profiler is attached).
struct nvtx_range {
  explicit nvtx_range(const char* name) { nvtxRangePushA(name); }
  ~nvtx_range() { nvtxRangePop(); }
  nvtx_range(const nvtx_range&) = delete;
  nvtx_range& operator=(const nvtx_range&) = delete;
};

namespace {

constexpr int kMaxStages = 16;
const char* const kStageNames[kMaxStages] = {"sort", "tile_cc", "border_merge", "emit", "", "", "", "",
                                             "",     "",        "",             "",     "", "", "", ""};

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }
uint32_t n_tiles_of(uint64_t n, int tile) { return (uint32_t)((n + tile - 1) / tile); }

struct layout {
  size_t hdr, probe, S, parent, openbm, slot_of, stage, comp_count, tmeta, open_hits, open_comps, overflow, pairs, bitmap, wcnt, partials;
  size_t keys0, keys1, vals0, vals1, hist, minidx, flags, ord;
  size_t total;
  uint32_t tiles, nwords;
};

layout make_layout(uint64_t n) {
  layout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  L.tiles = n_tiles_of(n, kTile);
  L.nwords = (uint32_t)((n + 31) / 32);
  const uint32_t rt = n_tiles_of(n, kRadixTile);
  uint32_t st = n_tiles_of((uint64_t)rt * kRadixBins, kScanTile);
  st = st > n_tiles_of(n, kScanTile) ? st : n_tiles_of(n, kScanTile);
  L.hdr = take(sizeof(dev_hdr));
  L.probe = take(kProbeSamples * 4);
  L.S = take(n * 16);
  L.parent = take(n * 4);
  L.openbm = take((size_t)n_tiles_of(n, kMaxTile) * kMaxTile / 8);  // one bit per position of every tile
  L.slot_of = take(n * 4);
  L.stage = take((size_t)n_tiles_of(n, kMaxTile) * kMaxTile * 64);
  L.comp_count = take((size_t)L.tiles * 4);
  L.tmeta = take((size_t)L.tiles * 64);
  L.open_hits = take(n * 4);
  L.open_comps = take(n * 4);
  L.overflow = take(n * 8);
  L.pairs = take(n * 8);
  L.bitmap = take((size_t)L.nwords * 4);
  L.wcnt = take((size_t)L.nwords * 4);
  L.partials = take((size_t)st * 4 + 4);
  // fallback-only buffers
  L.keys0 = take(n * 8);
  L.keys1 = take(n * 8);
  L.vals0 = take(n * 4);
  L.vals1 = take(n * 4);
  {
    const size_t hb = (size_t)rt * kRadixBins * 4, ob = os_layout::bytes(rt);  // tile histograms / onesweep words
    L.hist = take(hb > ob ? hb : ob);
  }
  L.minidx = take(n * 4);
  L.flags = take(n * 4);
  L.ord = take(n * 4);
  L.total = off;
  return L;
}

}  // namespace

constexpr size_t kHostMapBytes = 4096;  // mapped pinned read-back area per context

struct tpx_cluster {
  uint64_t dt;
  int variant;
  uint32_t width, height;
  dev_hdr* host_hdr;  // mapped pinned, 4 KB: the header, then scratch for other read-backs
  char* host_scratch;
  int profiling;
  int tile_mode;  // TPX_TILE_*
  cudaEvent_t ev[kMaxStages + 1];
  tpx_run_stats stats;
  int cuda_ready;  // CUDA resources are created lazily by the first run
  int bitmap_valid;  // the last run left the label bitmap + its word scan in the workspace (tile path)
  int want_first;    // next run records each cluster's first sorted position (grouped runs)
  int sort_start;  // first sort attempt (0: D=1024 window, 1: D=2560, 2: D=3072, 3: global radix);
                   // raised to the attempt that succeeded, so a stream whose disorder exceeds
                   // the window bound pays the failed attempts once, not on every run; it
                   // decays back to 0 after kSortProbeRuns runs (the stream may have calmed
                   // down), and a window spanning >= 2^32 ticks (a beam pause) sends only
                   // that run to the radix sort without raising it
  int runs_at_start;  // runs since sort_start was last raised
  tpx_cluster* island;  // variants (b)/(c): (a)-context whose components are the islands
  uint64_t island_dt;
};

#define TPX_CUDA(call)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "tpx_cluster: %s failed: %s\n", #call, cudaGetErrorString(e_)); \
      return TPX_ERR_CUDA;                                                             \
    }                                                                                  \
  } while (0)

#define TPX_LAUNCHED(ctx)                                                          \
  do {                                                                             \
    (ctx)->stats.kernel_launches++;                                                \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "tpx_cluster: launch failed: %s\n", cudaGetErrorString(e_)); \
      return TPX_ERR_CUDA;                                                         \
    }                                                                              \
  } while (0)

// Pinned header + timing events + kernel attributes, created on first use so
// that contexts can be created (and arguments validated) without a GPU.
static int ensure_cuda(tpx_cluster* c) {
  if (c->cuda_ready) return TPX_OK;
  if (cudaFuncSetAttribute(k_window_sort_kv<12>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)window_sort_kv_smem<12>()) != cudaSuccess ||
      cudaFuncSetAttribute(k_tile_csr<csr_sparse>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)csr_smem_bytes<csr_sparse>()) != cudaSuccess ||
      cudaFuncSetAttribute(k_tile_cc<tile_dense>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tile_smem_bytes<tile_dense>()) != cudaSuccess ||
      cudaFuncSetAttribute(k_tile_cell<cell_sparse>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)cell_smem_bytes<cell_sparse>()) != cudaSuccess)
    return TPX_ERR_CUDA;
  if (cudaHostAlloc((void**)&c->host_hdr, kHostMapBytes, cudaHostAllocMapped) != cudaSuccess) return TPX_ERR_CUDA;
  c->host_scratch = reinterpret_cast<char*>(c->host_hdr) + sizeof(dev_hdr);
  for (int i = 0; i <= kMaxStages; ++i) {
    if (cudaEventCreate(&c->ev[i]) != cudaSuccess) {
      for (int k = 0; k < i; ++k) cudaEventDestroy(c->ev[k]);
      cudaFreeHost(c->host_hdr);
      return TPX_ERR_CUDA;
    }
  }
  c->cuda_ready = 1;
  return TPX_OK;
}

static int grid_for(uint64_t n, int threads) {
  uint64_t g = (n + threads - 1) / threads;
  const uint64_t cap = 148ull * 32;  // grid-stride loops beyond 32 CTAs per SM
  if (g > cap) g = cap;
  return (int)(g ? g : 1);
}

static int exclusive_scan(tpx_cluster* c, const uint32_t* in, uint64_t n, uint32_t* out, uint32_t* partials,
                          uint32_t* total, cudaStream_t s) {
  uint32_t tiles = n_tiles_of(n, kScanTile);
  k_scan_reduce<<<tiles, kScanThreads, 0, s>>>(in, n, partials);
  TPX_LAUNCHED(c);
  k_scan_partials<<<1, kScanThreads, 0, s>>>(partials, tiles, total);
  TPX_LAUNCHED(c);
  k_scan_down<<<tiles, kScanThreads, 0, s>>>(in, n, partials, out);
  TPX_LAUNCHED(c);
  return TPX_OK;
}

// s_out: if not null and the single-sweep path runs, its last pass writes the
// sorted records there and *perm_out is set to a null permutation with
// *gathered = true.
template <typename KeyT>
static int radix_sort(tpx_cluster* c, hit_src hits, uint64_t n, uint64_t toa_min, int passes, char* ws,
                      const layout& L, uint32_t** perm_out, cudaStream_t s, srec* s_out, bool* gathered,
                      const unsigned long long* base_ptr = nullptr, dev_hdr* vhdr = nullptr) {
  KeyT* k0 = (KeyT*)(ws + L.keys0);
  KeyT* k1 = (KeyT*)(ws + L.keys1);
  uint32_t* v0 = (uint32_t*)(ws + L.vals0);
  uint32_t* v1 = (uint32_t*)(ws + L.vals1);
  uint32_t* hist = (uint32_t*)(ws + L.hist);
  uint32_t* partials = (uint32_t*)(ws + L.partials);
  const uint32_t tiles = n_tiles_of(n, kRadixTile);
  if constexpr (sizeof(KeyT) == 4) {
    // single-sweep passes (radix_onesweep.cuh): one digit-total read, then
    // one kernel per pass
    if (passes > 0) {
      char* sc = (char*)hist;
      uint32_t* gcount = (uint32_t*)(sc + os_layout::gcount);
      uint32_t* ticket = (uint32_t*)(sc + os_layout::ticket);
      unsigned long long* status = (unsigned long long*)(sc + os_layout::status);
      TPX_CUDA(cudaMemsetAsync(sc, 0, os_layout::bytes(tiles), s));
      const uint32_t hg = tiles < 148 * 8 ? tiles : 148 * 8;
      // key origin on the device (base_ptr): the exact minimum, or a guess
      // the histogram checks (vhdr: validation fused into the histogram)
      k_os_hist<<<hg, 256, 0, s>>>(hits, n, base_ptr, passes, gcount, c->width, c->height, vhdr);
      TPX_LAUNCHED(c);
      for (int p = 0; p < passes; ++p) {
        srec* so = (p + 1 == passes) ? s_out : nullptr;
        if (p == 0)
          k_os_pass<true><<<tiles, kRadixThreads, 0, s>>>(hits, nullptr, nullptr, n, base_ptr, p, tiles, gcount, ticket,
                                                          status, (uint32_t*)k1, v1, so);
        else
          k_os_pass<false><<<tiles, kRadixThreads, 0, s>>>(hits, (const uint32_t*)k0, v0, n, base_ptr, p, tiles, gcount,
                                                           ticket, status, (uint32_t*)k1, v1, so);
        TPX_LAUNCHED(c);
        KeyT* tk = k0;
        k0 = k1;
        k1 = tk;
        uint32_t* tv = v0;
        v0 = v1;
        v1 = tv;
      }
    }
    *perm_out = passes ? v0 : nullptr;
    if (gathered) *gathered = passes > 0 && s_out;
    return TPX_OK;
  } else {
  // 64-bit keys (ToA spans >= 2^32 ticks): histogram + scan + scatter per pass
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    if (p == 0) {
      k_radix_hist<KeyT, true><<<tiles, kRadixThreads, 0, s>>>(hits, nullptr, n, toa_min, shift, hist, tiles);
    } else {
      k_radix_hist<KeyT, false><<<tiles, kRadixThreads, 0, s>>>(hits, k0, n, toa_min, shift, hist, tiles);
    }
    TPX_LAUNCHED(c);
    int rc = exclusive_scan(c, hist, (uint64_t)tiles * kRadixBins, hist, partials, nullptr, s);
    if (rc) return rc;
    if (p == 0) {
      k_radix_scatter<KeyT, true><<<tiles, kRadixThreads, 0, s>>>(hits, nullptr, nullptr, n, toa_min, shift, hist,
                                                                  tiles, k1, v1);
    } else {
      k_radix_scatter<KeyT, false><<<tiles, kRadixThreads, 0, s>>>(hits, k0, v0, n, toa_min, shift, hist, tiles,
                                                                   k1, v1);
    }
    TPX_LAUNCHED(c);
    KeyT* tk = k0;
    k0 = k1;
    k1 = tk;
    uint32_t* tv = v0;
    v0 = v1;
    v1 = tv;
  }
  *perm_out = passes ? v0 : nullptr;
  return TPX_OK;
  }
}

struct run_ptrs {
  hit_src hits;
  uint64_t n;
  uint64_t n_owned;
  uint32_t* labels;
  tpx_cluster_features* feats;
  uint64_t capacity;
  char* ws;
  layout L;
  cudaStream_t s;
  bool dense;   // tile configuration chosen by the density probe
  uint32_t sort_T = kWSortTile;  // output tile of the sort that produced S (its borders are verified)
  bool csr = false;  // counting-sorted cell index + backward hooking (tile_csr.cuh)
  // sharded runs (sharded.cuh): labels written as global indices into two
  // arrays, emission deferred until the boundary clusters are merged
  label_map lm = {};
  bool defer_emit = false;
};

// The header is initialised by a kernel, not by an H2D copy of a host
// struct: with several buffers in flight (tpx_pipeline, the streaming path)
// a small H2D would queue on the copy engine behind another buffer's bulk
// H2D and hold this run until it drained.
__global__ void k_reset_hdr(dev_hdr* h) {
  static_assert(sizeof(dev_hdr) % 8 == 0 && offsetof(dev_hdr, toa_min) == 0, "header layout");
  unsigned long long* w = reinterpret_cast<unsigned long long*>(h);
  for (uint32_t i = threadIdx.x; i < sizeof(dev_hdr) / 8; i += blockDim.x) w[i] = i == 0 ? ~0ull : 0ull;
}

static int reset_header(tpx_cluster* c, const run_ptrs& r) {
  k_reset_hdr<<<1, 32, 0, r.s>>>((dev_hdr*)(r.ws + r.L.hdr));
  TPX_LAUNCHED(c);
  TPX_CUDA(cudaMemsetAsync(r.ws + r.L.bitmap, 0, (size_t)r.L.nwords * 4, r.s));
  // open bitmap: tile kernels store only the words that have an open hit
  TPX_CUDA(cudaMemsetAsync(r.ws + r.L.openbm, 0, (size_t)n_tiles_of(r.n, kMaxTile) * kMaxTile / 8, r.s));
  return TPX_OK;
}

static int read_header(tpx_cluster* c, const run_ptrs& r) {
  TPX_CUDA(readback_async(c->host_hdr, r.ws + r.L.hdr, sizeof(dev_hdr), r.s));
  c->stats.kernel_launches++;
  TPX_CUDA(cudaStreamSynchronize(r.s));
  return TPX_OK;
}

// Small read-back into a host variable through the context's mapped scratch.
static int readback_sync(tpx_cluster* c, void* dst, const void* dev, size_t bytes, cudaStream_t s) {
  if (bytes > kHostMapBytes - sizeof(dev_hdr)) return TPX_ERR_INVALID_ARG;
  TPX_CUDA(readback_async(c->host_scratch, dev, bytes, s));
  c->stats.kernel_launches++;
  TPX_CUDA(cudaStreamSynchronize(s));
  memcpy(dst, c->host_scratch, bytes);
  return TPX_OK;
}

// Global LSD radix sort into S (fallback when the windowed sort cannot prove
// its displacement bound).  First with a guessed key origin (k_radix_base;
// 4 passes, validation and the range check fused into the histogram, no host
// sync); if the guess fails (err bit 4, seen at the run's post-sort
// read-back), exact: the ToA range first (one extra host sync), then
// ceil(bits / 8) passes from the true minimum.
static int sort_global(tpx_cluster* c, const run_ptrs& r, bool exact) {
  nvtx_range nv("tpx:sort_radix");
  dev_hdr* hdr = (dev_hdr*)(r.ws + r.L.hdr);
  srec* S = (srec*)(r.ws + r.L.S);
  if (!exact) {
    k_radix_base<<<1, 256, 0, r.s>>>(r.hits, r.n, hdr);
    TPX_LAUNCHED(c);
    uint32_t* perm = nullptr;
    bool gathered = false;
    int rc = radix_sort<uint32_t>(c, r.hits, r.n, 0, 4, r.ws, r.L, &perm, r.s, S, &gathered, &hdr->radix_base, hdr);
    (void)gathered;  // 4 passes with s_out: the last pass wrote S
    return rc;
  }
  const int g = grid_for(r.n, kMMThreads) < 148 * 8 ? grid_for(r.n, kMMThreads) : 148 * 8;
  k_validate_minmax<<<g, kMMThreads, 0, r.s>>>(r.hits, r.n, c->width, c->height, hdr);
  TPX_LAUNCHED(c);
  int rc = read_header(c, r);
  if (rc) return rc;
  if (c->host_hdr->err & 1u) return TPX_ERR_COORD_RANGE;
  const uint64_t toa_min = c->host_hdr->toa_min, range = c->host_hdr->toa_max - toa_min;
  const int bits = range ? 64 - __builtin_clzll(range) : 0;
  const int passes = (bits + 7) / 8;
  uint32_t* perm = nullptr;
  bool gathered = false;
  rc = (bits <= 32) ? radix_sort<uint32_t>(c, r.hits, r.n, toa_min, passes, r.ws, r.L, &perm, r.s, S, &gathered,
                                           &hdr->toa_min)
                    : radix_sort<uint64_t>(c, r.hits, r.n, toa_min, passes, r.ws, r.L, &perm, r.s, nullptr, nullptr);
  if (rc) return rc;
  if (gathered) return TPX_OK;  // the last pass wrote S
  k_gather_init<<<grid_for(r.n, 256), 256, 0, r.s>>>(r.hits, perm, r.n, (srec*)(r.ws + r.L.S),
                                                     (uint32_t*)(r.ws + r.L.parent));
  TPX_LAUNCHED(c);
  return TPX_OK;
}

static int emit_sorted(tpx_cluster* c, const run_ptrs& r, tpx_cluster_features* removed_out,
                       unsigned long long* n_removed);

// One packed windowed-sort attempt (sort_window.cuh k_window_sort_packed).
template <int IT, int T>
static int window_sort_packed(tpx_cluster* c, run_ptrs& r, srec* S, dev_hdr* hdr) {
  constexpr int NT = kWSortThreads;
  static_assert(window_sort_packed_smem<IT, NT>() <= 113 * 1024, "two CTAs per SM");
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_window_sort_packed<IT, T, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)window_sort_packed_smem<IT, NT>()) != cudaSuccess)
      return TPX_ERR_CUDA;
    attr = true;
  }
  r.sort_T = T;
  const uint32_t sort_tiles = n_tiles_of(r.n, T);
  k_window_sort_packed<IT, T, NT><<<sort_tiles, NT, window_sort_packed_smem<IT, NT>(), r.s>>>(
      r.hits, r.n, c->width, c->height, S, hdr);
  TPX_LAUNCHED(c);
  k_sort_check<<<grid_for(sort_tiles, 256), 256, 0, r.s>>>(S, r.n, T, hdr);
  TPX_LAUNCHED(c);
  return TPX_OK;
}

// One windowed-sort attempt (sort_window.cuh): T outputs per CTA from a
// window of IT * NT hits (D = (IT * NT - T) / 2), then the border check.
template <int IT, int T, int NT>
static int window_sort(tpx_cluster* c, run_ptrs& r, srec* S, dev_hdr* hdr) {
  static_assert(window_sort_smem<IT, NT>() <= 227 * 1024, "window sort shared memory");
  static bool attr = false;  // once per process (the attribute is per function)
  if (!attr) {
    if (cudaFuncSetAttribute(k_window_sort<IT, T, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)window_sort_smem<IT, NT>()) != cudaSuccess)
      return TPX_ERR_CUDA;
    attr = true;
  }
  r.sort_T = T;
  const uint32_t sort_tiles = n_tiles_of(r.n, T);
  k_window_sort<IT, T, NT><<<sort_tiles, NT, window_sort_smem<IT, NT>(), r.s>>>(r.hits, r.n, c->width, c->height, S,
                                                                               hdr);
  TPX_LAUNCHED(c);
  k_sort_check<<<grid_for(sort_tiles, 256), 256, 0, r.s>>>(S, r.n, T, hdr);
  TPX_LAUNCHED(c);
  return TPX_OK;
}

// Tile clustering + border merge + ordered emission on a sorted S.
static int cluster_sorted(tpx_cluster* c, const run_ptrs& r) {
  nvtx_range nv("tpx:tile+border_merge");
  char* ws = r.ws;
  const layout& L = r.L;
  dev_hdr* hdr = (dev_hdr*)(ws + L.hdr);
  const srec* S = (const srec*)(ws + L.S);
  uint32_t* parent_g = (uint32_t*)(ws + L.parent);
  uint32_t* slot_of = (uint32_t*)(ws + L.slot_of);
  tpx_cluster_features* stage = (tpx_cluster_features*)(ws + L.stage);
  uint32_t* comp_count = (uint32_t*)(ws + L.comp_count);
  uint32_t* open_hits = (uint32_t*)(ws + L.open_hits);
  uint32_t* open_comps = (uint32_t*)(ws + L.open_comps);
  uint2* overflow = (uint2*)(ws + L.overflow);
  uint2* pairs = (uint2*)(ws + L.pairs);
  uint32_t* bitmap = (uint32_t*)(ws + L.bitmap);

  if (c->profiling) cudaEventRecord(c->ev[1], r.s);
  tile_args a;
  a.S = S;
  a.n = r.n;
  a.dt = c->dt;
  a.width = c->width;
  a.height = c->height;
  a.n_owned = (uint32_t)r.n_owned;
  a.labels = r.labels;
  a.parent_g = parent_g;
  a.openbm = (uint32_t*)(ws + L.openbm);
  a.slot_of = slot_of;
  a.stage = stage;
  a.comp_count = comp_count;
  a.bitmap = bitmap;
  a.open_hits = open_hits;
  a.open_comps = open_comps;
  a.pairs = pairs;
  a.overflow = overflow;
  a.hdr = hdr;
  a.verify_stride = r.sort_T;
  a.phase_cycles = c->profiling >= 2 ? hdr->phase_cycles : nullptr;
  a.tile_meta = nullptr;
  a.first_of_label = c->want_first ? (uint32_t*)(ws + L.minidx) : nullptr;
  a.lm = r.lm;
  if (r.dense) {
    const uint32_t nt = n_tiles_of(r.n, tile_dense::kTile);
    a.tile_meta = (const uint64_t*)(ws + L.tmeta);
    k_tile_bounds<tile_dense><<<(nt + 7) / 8, 256, 0, r.s>>>(S, r.n, c->dt, nt, r.sort_T, (uint64_t*)(ws + L.tmeta),
                                                            hdr);
    TPX_LAUNCHED(c);
    k_tile_cc<tile_dense><<<nt, tile_dense::kThreads, tile_smem_bytes<tile_dense>(), r.s>>>(a);
  }
  else if (r.csr) {
    static_assert(csr_sparse::kTile == cell_sparse::kTile && csr_sparse::kHalo == cell_sparse::kHalo, "shared bounds");
    const uint32_t nt = n_tiles_of(r.n, csr_sparse::kTile);
    a.tile_meta = (const uint64_t*)(ws + L.tmeta);
    k_tile_bounds<cell_sparse><<<(nt + 7) / 8, 256, 0, r.s>>>(S, r.n, c->dt, nt, r.sort_T, (uint64_t*)(ws + L.tmeta),
                                                             hdr);
    TPX_LAUNCHED(c);
    k_tile_csr<csr_sparse><<<nt, csr_sparse::kThreads, csr_smem_bytes<csr_sparse>(), r.s>>>(a);
  } else {
    const uint32_t nt = n_tiles_of(r.n, cell_sparse::kTile);
    a.tile_meta = (const uint64_t*)(ws + L.tmeta);
    k_tile_bounds<cell_sparse><<<(nt + 7) / 8, 256, 0, r.s>>>(S, r.n, c->dt, nt, r.sort_T, (uint64_t*)(ws + L.tmeta),
                                                             hdr);
    TPX_LAUNCHED(c);
    k_tile_cell<cell_sparse><<<nt, cell_sparse::kThreads, cell_smem_bytes<cell_sparse>(), r.s>>>(a);
  }
  TPX_LAUNCHED(c);

  if (c->profiling) cudaEventRecord(c->ev[2], r.s);
  k_overflow_unions<<<kListGrid, kListThreads, 0, r.s>>>(S, r.n, c->dt, overflow, hdr, parent_g, a.openbm);
  TPX_LAUNCHED(c);
  k_pair_unions<<<kListGrid, kListThreads, 0, r.s>>>(pairs, hdr, parent_g, a.openbm);
  TPX_LAUNCHED(c);
  k_flatten_open<<<kListGrid, kListThreads, 0, r.s>>>(open_hits, hdr, parent_g);
  TPX_LAUNCHED(c);
  k_merge_open<<<kListGrid, kListThreads, 0, r.s>>>(open_comps, hdr, parent_g, slot_of, stage);
  TPX_LAUNCHED(c);
  k_open_labels<<<kListGrid, kListThreads, 0, r.s>>>(S, open_hits, open_comps, hdr, parent_g, slot_of, stage,
                                                     r.labels, bitmap, (uint32_t)r.n_owned, a.first_of_label, r.lm);
  TPX_LAUNCHED(c);
  if (r.defer_emit) return TPX_OK;  // sharded: emit_sorted() after the boundary merge
  return emit_sorted(c, r, nullptr, nullptr);
}

// A6 + A7 emission: ordinal of every label bit, records copied in label
// order.  removed_out (sharded runs): records whose label bit was cleared by
// the boundary merge are appended there (global labels) instead.
static int emit_sorted(tpx_cluster* c, const run_ptrs& r, tpx_cluster_features* removed_out,
                       unsigned long long* n_removed) {
  nvtx_range nv("tpx:emit");
  char* ws = r.ws;
  const layout& L = r.L;
  dev_hdr* hdr = (dev_hdr*)(ws + L.hdr);
  const tpx_cluster_features* stage = (const tpx_cluster_features*)(ws + L.stage);
  const uint32_t* comp_count = (const uint32_t*)(ws + L.comp_count);
  uint32_t* bitmap = (uint32_t*)(ws + L.bitmap);
  uint32_t* wcnt = (uint32_t*)(ws + L.wcnt);
  uint32_t* partials = (uint32_t*)(ws + L.partials);

  if (c->profiling) cudaEventRecord(c->ev[3], r.s);
  k_popc<<<grid_for(L.nwords, 256), 256, 0, r.s>>>(bitmap, L.nwords, wcnt);
  TPX_LAUNCHED(c);
  int rc = exclusive_scan(c, wcnt, L.nwords, wcnt, partials, (uint32_t*)&hdr->n_clusters, r.s);
  if (rc) return rc;
  if (r.capacity || removed_out) {
    const uint32_t tile = r.dense ? tile_dense::kTile : cell_sparse::kTile;
    k_emit<<<kListGrid, kEmitThreads, 0, r.s>>>(stage, comp_count, n_tiles_of(r.n, tile), tile, bitmap, wcnt, r.feats,
                                                r.capacity, r.lm.own_off, removed_out, n_removed);
    TPX_LAUNCHED(c);
  }
  if (c->profiling) cudaEventRecord(c->ev[4], r.s);
  return TPX_OK;
}

// Global union-find pipeline (cluster.cuh) on a sorted S -- the internal
// fallback if the tile path ever reports an inconsistency.
static int cluster_global(tpx_cluster* c, const run_ptrs& r) {
  char* ws = r.ws;
  const layout& L = r.L;
  dev_hdr* hdr = (dev_hdr*)(ws + L.hdr);
  const srec* S = (const srec*)(ws + L.S);
  uint32_t* parent = (uint32_t*)(ws + L.parent);
  uint32_t* minidx = (uint32_t*)(ws + L.minidx);
  uint32_t* flags = (uint32_t*)(ws + L.flags);
  uint32_t* ord = (uint32_t*)(ws + L.ord);
  uint32_t* partials = (uint32_t*)(ws + L.partials);
  const uint64_t n = r.n;
  if (c->profiling) cudaEventRecord(c->ev[1], r.s);
  k_iota<<<grid_for(n, 256), 256, 0, r.s>>>(parent, n);
  TPX_LAUNCHED(c);
  k_window_union<<<grid_for(n, 256), 256, 0, r.s>>>(S, n, c->dt, parent);
  TPX_LAUNCHED(c);
  k_flatten<<<grid_for(n, 256), 256, 0, r.s>>>(parent, n);
  TPX_LAUNCHED(c);
  if (c->profiling) cudaEventRecord(c->ev[2], r.s);
  TPX_CUDA(cudaMemsetAsync(minidx, 0xff, n * 4, r.s));
  k_minidx<<<grid_for(n, 256), 256, 0, r.s>>>(S, parent, n, minidx);
  TPX_LAUNCHED(c);
  k_labels<<<grid_for(n, 256), 256, 0, r.s>>>(S, parent, minidx, n, r.labels);
  TPX_LAUNCHED(c);
  k_flags<<<grid_for(n, 256), 256, 0, r.s>>>(r.labels, n, r.n_owned, flags);
  TPX_LAUNCHED(c);
  if (c->profiling) cudaEventRecord(c->ev[3], r.s);
  int rc = exclusive_scan(c, flags, n, ord, partials, (uint32_t*)&hdr->n_clusters, r.s);
  if (rc) return rc;
  if (r.capacity) {
    k_feat_init<<<grid_for(n, 256), 256, 0, r.s>>>(r.labels, ord, n, r.n_owned, r.feats, r.capacity);
    TPX_LAUNCHED(c);
    k_feat_accum<<<grid_for(n, 256), 256, 0, r.s>>>(S, parent, minidx, ord, n, r.n_owned, r.feats, r.capacity);
    TPX_LAUNCHED(c);
  }
  if (c->profiling) cudaEventRecord(c->ev[4], r.s);
  return TPX_OK;
}

// ---------------------------------------------------------------- variants
// (iii)(b) GLOBAL / (iii)(c) STATIC (variant.cuh): islands from an (a)-run
// with window W, the streaming process simulated per island, records by
// label.  Workspace: the island run's own, then the arrays below.
struct variant_layout {
  size_t labels, feats, order, offsets, cluster_of, par, cmin, cmax, stamp, root_of, minidx, rbits, rbase, misc,
      total;
};

static variant_layout make_variant_layout(uint64_t n) {
  variant_layout V;
  size_t off = make_layout(n).total;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  const uint64_t nwords = (n + 31) / 32;
  V.labels = take(n * 4);
  V.feats = take(n * 64);
  V.order = take(n * 4);
  V.offsets = take(n * 4 + 4);
  V.cluster_of = take(n * 4);
  V.par = take(n * 4);
  V.cmin = take(n * 8);
  V.cmax = take(n * 8);
  V.stamp = take(n * 4);
  V.root_of = take(n * 4);
  V.minidx = take(n * 4);
  V.rbits = take(nwords * 4);
  V.rbase = take(nwords * 4);
  V.misc = take(256);
  V.total = off;
  return V;
}

static size_t run_ws_total(const tpx_cluster* c, uint64_t n) {
  return c->variant == TPX_VARIANT_LOCAL ? make_layout(n).total : make_variant_layout(n).total;
}

__global__ void k_fill_iota32(uint32_t* __restrict__ a, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = (uint32_t)i;
}

static int run_variant(tpx_cluster* c, const tpx_hit* hits, uint64_t n, uint32_t* labels_out,
                       tpx_cluster_features* features_out, uint64_t capacity, uint64_t* n_clusters_out, char* ws,
                       size_t ws_bytes, cudaStream_t s) {
  const variant_layout V = make_variant_layout(n);
  uint32_t* order = (uint32_t*)(ws + V.order);
  uint32_t* offsets = (uint32_t*)(ws + V.offsets);
  uint32_t* par = (uint32_t*)(ws + V.par);
  unsigned long long* cmin = (unsigned long long*)(ws + V.cmin);
  unsigned long long* cmax = (unsigned long long*)(ws + V.cmax);
  uint32_t* stamp = (uint32_t*)(ws + V.stamp);
  uint32_t* root_of = (uint32_t*)(ws + V.root_of);
  uint32_t* minidx = (uint32_t*)(ws + V.minidx);
  uint32_t* rbits = (uint32_t*)(ws + V.rbits);
  uint32_t* rbase = (uint32_t*)(ws + V.rbase);
  unsigned long long* d_span = (unsigned long long*)(ws + V.misc);
  uint32_t* partials = (uint32_t*)(ws + make_layout(n).partials);
  const uint64_t dt = c->dt;
  // (c): W = dt is exact; (b): start at 4 dt and grow until the span test holds
  uint64_t W = c->variant == TPX_VARIANT_STATIC ? dt : 4 * dt + 64;
  int rc;
  for (int round = 0;; ++round) {
    if (!c->island || c->island_dt != W) {
      tpx_cluster_destroy(c->island);
      c->island = nullptr;
      if ((rc = tpx_cluster_create(W, TPX_VARIANT_LOCAL, c->width, c->height, &c->island))) return rc;
      c->island_dt = W;
    }
    uint64_t k_is = 0;
    rc = tpx_cluster_run_grouped(c->island, hits, n, (uint32_t*)(ws + V.labels), (tpx_cluster_features*)(ws + V.feats),
                                 nullptr, n, &k_is, order, offsets, (uint32_t*)(ws + V.cluster_of), ws,
                                 make_layout(n).total, s);
    if (rc) return rc;
    c->stats.kernel_launches += c->island->stats.kernel_launches;
    const int gn = grid_for(n, 256), gk = grid_for(k_is, 256);
    k_fill_iota32<<<gn, 256, 0, s>>>(par, n);
    TPX_LAUNCHED(c);
    TPX_CUDA(cudaMemsetAsync(stamp, 0, n * 4, s));
    // the island features are not needed past the grouped run: their space
    // holds the hits gathered in island order
    tpx_hit* ih = (tpx_hit*)(ws + V.feats);
    k_gather_hits<<<gn, 256, 0, s>>>(hits, order, n, ih);
    TPX_LAUNCHED(c);
    variant_args a;
    a.ih = ih;
    a.order = order;
    a.offsets = offsets;
    a.k = k_is;
    a.dt = dt;
    a.window = W;
    a.rule = c->variant;
    a.par = par;
    a.cmin = cmin;
    a.cmax = cmax;
    a.stamp = stamp;
    k_variant_small<<<gk, 256, 0, s>>>(a);
    TPX_LAUNCHED(c);
    k_variant_large<<<gk, 256, 0, s>>>(a);
    TPX_LAUNCHED(c);
    TPX_CUDA(cudaMemsetAsync(minidx, 0xff, n * 4, s));
    TPX_CUDA(cudaMemsetAsync(d_span, 0, 8, s));
    k_variant_roots<<<gn, 256, 0, s>>>(par, order, n, cmin, cmax, root_of, minidx, d_span);
    TPX_LAUNCHED(c);
    if (c->variant == TPX_VARIANT_GLOBAL) {
      unsigned long long span = 0;
      if ((rc = readback_sync(c, &span, d_span, 8, s))) return rc;
      if (span + dt > W) {  // a candidate older than W might have been missed
        const uint64_t grow = 2 * (span + dt) + 64;
        W = grow > 4 * W ? grow : 4 * W;
        c->stats.sort_retries++;
        continue;
      }
    }
    break;
  }
  k_variant_labels<<<grid_for(n, 256), 256, 0, s>>>(root_of, order, n, minidx, labels_out);
  TPX_LAUNCHED(c);
  // records in ascending label order
  const uint64_t nwords = (n + 31) / 32;
  k_root_bits<<<grid_for(nwords, 256), 256, 0, s>>>(labels_out, n, rbits);
  TPX_LAUNCHED(c);
  k_popc<<<grid_for(nwords, 256), 256, 0, s>>>(rbits, nwords, rbase);
  TPX_LAUNCHED(c);
  if ((rc = exclusive_scan(c, rbase, nwords, rbase, partials, (uint32_t*)(ws + V.misc + 64), s))) return rc;
  if (capacity) {
    k_variant_feat_init<<<grid_for(n, 256), 256, 0, s>>>(n, rbits, rbase, features_out, capacity);
    TPX_LAUNCHED(c);
    k_variant_feat_accum_grouped<<<grid_for(n, 256), 256, 0, s>>>((const tpx_hit*)(ws + V.feats), order, n, labels_out,
                                                                   rbits, rbase, features_out, capacity);
    TPX_LAUNCHED(c);
  }
  uint32_t k = 0;
  if ((rc = readback_sync(c, &k, ws + V.misc + 64, 4, s))) return rc;
  *n_clusters_out = k;
  c->stats.n_clusters = k;
  c->stats.cross_pairs = W;  // diagnostics: final island window (ticks)
  return k > capacity ? TPX_ERR_CAPACITY : TPX_OK;
}

static int run_core(tpx_cluster* c, run_ptrs& r);
static void finish_stats(tpx_cluster* c);

extern "C" {

int tpx_abi_version(void) { return TPX_ABI_VERSION; }

const char* tpx_status_string(int s) {
  switch (s) {
    case TPX_OK: return "ok";
    case TPX_ERR_INVALID_ARG: return "invalid argument";
    case TPX_ERR_UNSUPPORTED:
      return "unsupported (variant (iii)(a) only for sharded runs and streams; sharded runs: sensor width <= 1024, "
             "no rank-skipping edge, halo <= TPX_SHARD_HALO_CAP)";
    case TPX_ERR_COORD_RANGE: return "hit coordinate outside the sensor or toa >= 2^48";
    case TPX_ERR_TOO_MANY_HITS: return "too many hits (n must be < 2^32 - 1)";
    case TPX_ERR_CAPACITY: return "feature capacity too small (n_clusters_out holds the required count)";
    case TPX_ERR_OOM: return "workspace too small";
    case TPX_ERR_CUDA: return "CUDA error";
    case TPX_ERR_NCCL: return "NCCL error";
    default: return "unknown status";
  }
}

const char* tpx_cluster_stage_name(int i) { return (i >= 0 && i < kMaxStages) ? kStageNames[i] : ""; }

int tpx_cluster_create(uint64_t dt_max_ticks, int variant, uint32_t width, uint32_t height, tpx_cluster** out) {
  if (!out) return TPX_ERR_INVALID_ARG;
  *out = nullptr;
  if (variant < TPX_VARIANT_LOCAL || variant > TPX_VARIANT_STATIC) return TPX_ERR_INVALID_ARG;
  if (width == 0 || height == 0 || width > 32768 || height > 32768) return TPX_ERR_INVALID_ARG;
  if (dt_max_ticks >= (1ull << 48)) return TPX_ERR_INVALID_ARG;
  tpx_cluster* c = new (std::nothrow) tpx_cluster;
  if (!c) return TPX_ERR_OOM;
  memset(c, 0, sizeof(*c));
  c->dt = dt_max_ticks;
  c->variant = variant;
  c->width = width;
  c->height = height;
  *out = c;
  return TPX_OK;
}

void tpx_cluster_destroy(tpx_cluster* c) {
  if (!c) return;
  tpx_cluster_destroy(c->island);
  if (c->cuda_ready) {
    for (int i = 0; i <= kMaxStages; ++i) cudaEventDestroy(c->ev[i]);
    cudaFreeHost(c->host_hdr);
  }
  delete c;
}

int tpx_cluster_workspace_bytes(const tpx_cluster* c, uint64_t n, size_t* bytes) {
  if (!c || !bytes) return TPX_ERR_INVALID_ARG;
  if (n >= 0xffffffffull) return TPX_ERR_TOO_MANY_HITS;
  *bytes = run_ws_total(c, n);
  return TPX_OK;
}

int tpx_cluster_set_profiling(tpx_cluster* c, int enable) {
  if (!c) return TPX_ERR_INVALID_ARG;
  if (enable < 0 || enable > 2) return TPX_ERR_INVALID_ARG;
  c->profiling = enable;
  return TPX_OK;
}

int tpx_cluster_set_tile_mode(tpx_cluster* c, int mode) {
  // TPX_TILE_COLUMN (round 1's column-bucket kernel) was removed in round 2
  if (!c || mode < TPX_TILE_AUTO || mode > TPX_TILE_CELL || mode == TPX_TILE_COLUMN) return TPX_ERR_INVALID_ARG;
  c->tile_mode = mode;
  return TPX_OK;
}

int tpx_cluster_last_stats(const tpx_cluster* c, tpx_run_stats* out) {
  if (!c || !out) return TPX_ERR_INVALID_ARG;
  *out = c->stats;
  return TPX_OK;
}

int tpx_cluster_run(tpx_cluster* c, const tpx_hit* hits, uint64_t n, uint32_t* labels_out,
                    tpx_cluster_features* features_out, uint64_t capacity, uint64_t* n_clusters_out, void* workspace,
                    size_t workspace_bytes, void* stream) {
  return tpx_cluster_run_partial(c, hits, n, n, labels_out, features_out, capacity, n_clusters_out, workspace,
                                 workspace_bytes, stream);
}

int tpx_cluster_run_partial(tpx_cluster* c, const tpx_hit* hits, uint64_t n, uint64_t n_owned, uint32_t* labels_out,
                            tpx_cluster_features* features_out, uint64_t capacity, uint64_t* n_clusters_out,
                            void* workspace, size_t workspace_bytes, void* stream) {
  if (!c || !n_clusters_out) return TPX_ERR_INVALID_ARG;
  *n_clusters_out = 0;
  if (n >= 0xffffffffull) return TPX_ERR_TOO_MANY_HITS;
  if (n_owned > n) return TPX_ERR_INVALID_ARG;
  memset(&c->stats, 0, sizeof(c->stats));
  c->stats.n_hits = n;
  if (n == 0) return TPX_OK;
  if (!hits || !labels_out || !workspace || (!features_out && capacity)) return TPX_ERR_INVALID_ARG;
  if (((uintptr_t)hits & 15) || ((uintptr_t)workspace & 255) || ((uintptr_t)features_out & 15) ||
      ((uintptr_t)labels_out & 3))
    return TPX_ERR_INVALID_ARG;
  if (c->variant != TPX_VARIANT_LOCAL) {
    if (n_owned != n) return TPX_ERR_UNSUPPORTED;  // sharded runs: variant (a) only
    if (workspace_bytes < run_ws_total(c, n)) return TPX_ERR_OOM;
    if (ensure_cuda(c)) return TPX_ERR_CUDA;
    return run_variant(c, hits, n, labels_out, features_out, capacity, n_clusters_out, (char*)workspace,
                       workspace_bytes, (cudaStream_t)stream);
  }
  run_ptrs r;
  r.L = make_layout(n);
  if (workspace_bytes < r.L.total) return TPX_ERR_OOM;
  if (ensure_cuda(c)) return TPX_ERR_CUDA;
  r.hits = hit_src(hits);
  r.n = n;
  r.n_owned = n_owned;
  r.labels = labels_out;
  r.feats = features_out;
  r.capacity = capacity;
  r.ws = (char*)workspace;
  r.s = (cudaStream_t)stream;
  int rc = run_core(c, r);
  if (rc) return rc;
  const uint64_t k = c->stats.n_clusters;
  *n_clusters_out = k;
  return k > capacity ? TPX_ERR_CAPACITY : TPX_OK;
}

}  // extern "C"

// Sort attempts + clustering + (unless r.defer_emit) emission for a prepared
// run; fills c->stats (n_clusters from the emission's scan).  Deferred runs
// (sharded.cuh) return after the clustering kernels are queued, without a
// host synchronisation: the caller finishes with emit_sorted().
static int run_core(tpx_cluster* c, run_ptrs& r) {
  const uint64_t n = r.n;
  srec* S = (srec*)(r.ws + r.L.S);
  dev_hdr* hdr = (dev_hdr*)(r.ws + r.L.hdr);

  int rc;
  // windowed sorts: 0 packed D = 1024 (13312-hit window, 11264 outputs),
  // 1 unpacked D = 1024 (10240 / 8192: windows spanning >= 2^27 ticks),
  // 2 packed D = 2560 (13312 / 8192), 3 unpacked D = 2560 (10240 / 5120),
  // 4 unpacked D = 3072 (10240 / 4096); 5 global radix sort; 6 global
  // union-find pipeline (internal fallback)
  constexpr int kRadixAttempt = 5;
  constexpr int kSortProbeRuns = 64;
  if (c->sort_start > 0 && ++c->runs_at_start > kSortProbeRuns) {
    c->sort_start = 0;
    c->runs_at_start = 0;
  }
  const int first_attempt = c->sort_start;
  bool radix_exact = false;  // the guessed radix key origin failed: exact range first
  nvtx_range nv_run("tpx:run");
  for (int attempt = first_attempt; attempt <= kRadixAttempt + 1; ++attempt) {
    nvtx_range nv_sort(attempt <= 1   ? "tpx:sort_window"
                       : attempt <= 3 ? "tpx:sort_window_d2560"
                       : attempt == 4 ? "tpx:sort_window_d3072"
                                      : "tpx:sort_fallback");
    if ((rc = reset_header(c, r))) return rc;
    if (c->profiling) cudaEventRecord(c->ev[0], r.s);
    if (attempt == 0) {
      if ((rc = window_sort_packed<26, 11264>(c, r, S, hdr))) return rc;  // D = 1024
    } else if (attempt == 1) {
      if ((rc = window_sort<20, kSortT0, 512>(c, r, S, hdr))) return rc;  // D = 1024
    } else if (attempt == 2) {
      if ((rc = window_sort_packed<26, 8192>(c, r, S, hdr))) return rc;  // D = 2560
    } else if (attempt == 3) {
      if ((rc = window_sort<20, kSortTm, 512>(c, r, S, hdr))) return rc;  // D = 2560
    } else if (attempt == 4) {
      if ((rc = window_sort<20, kSortT1, 512>(c, r, S, hdr))) return rc;  // D = 3072
    } else {
      if ((rc = sort_global(c, r, radix_exact))) return rc;
    }
    c->stats.sort_path = attempt >= kRadixAttempt ? 1 : 0;
    // one small read-back after the sort: validation and window-sort status
    // (a window wider than 32 bits of ticks leaves its output tile unwritten,
    // so the tile kernel must not run on it) and the window-density probe
    // (dense heavy-ion windows use the large-halo tile configuration)
    {
      const bool probe_on = c->tile_mode == TPX_TILE_AUTO;
      uint32_t* probe = (uint32_t*)(r.ws + r.L.probe);
      uint32_t hprobe[kProbeSamples];
      if (probe_on) {
        k_density_probe<<<1, kProbeSamples, 0, r.s>>>(S, n, c->dt, probe);
        TPX_LAUNCHED(c);
        TPX_CUDA(readback_async(c->host_scratch, probe, sizeof(hprobe), r.s));
        c->stats.kernel_launches++;
      }
      if ((rc = read_header(c, r))) return rc;  // synchronises the stream: the probe samples are in as well
      if (probe_on) memcpy(hprobe, c->host_scratch, sizeof(hprobe));
      if (c->host_hdr->err & 1u) return TPX_ERR_COORD_RANGE;
      if (attempt >= kRadixAttempt && !radix_exact && (c->host_hdr->err & 16u)) {  // ToA outside the guessed key range
        radix_exact = true;
        --attempt;
        continue;
      }
      if (attempt < kRadixAttempt && (c->host_hdr->err & 4u)) {  // >= 2^32-tick window: radix, this run only
        attempt = kRadixAttempt - 1;
        continue;
      }
      if (attempt < kRadixAttempt && c->host_hdr->sort_bad) {  // displacement bound violated: widen / fall back
        // a packed attempt that failed on displacement (not on its 18-bit key
        // range) skips the unpacked attempt with the same bound
        if ((attempt == 0 || attempt == 2) && !(c->host_hdr->err & 8u)) ++attempt;
        if (attempt + 1 > c->sort_start) {
          c->sort_start = attempt + 1;
          c->runs_at_start = 0;
        }
        continue;
      }
      if (probe_on) {
        int big = 0;
        for (int i = 0; i < kProbeSamples; ++i) big += hprobe[i] > kDenseWindow;
        r.dense = big * 10 > kProbeSamples;  // > 10 % of the samples have windows near the sparse halo
      } else {
        r.dense = c->tile_mode == TPX_TILE_DENSE;
      }
      r.csr = !r.dense && c->tile_mode != TPX_TILE_CELL && c->width <= kCsrMaxCoord + 1 &&
              c->height <= kCsrMaxCoord + 1;
      c->stats.tile_dense = r.dense ? 1 : 0;
    }
    c->stats.sort_retries = (attempt < kRadixAttempt ? attempt : kRadixAttempt) -
                            (first_attempt < kRadixAttempt ? first_attempt : kRadixAttempt);
    // the tile kernel indexes one bucket per pixel column (sparse) or packs
    // pixel ids in 20 bits (dense): larger sensors take the global pipeline
    const bool big_sensor =
        c->width > (uint32_t)kMaxTileWidth || (uint64_t)c->width * c->height + c->width > kMaxTilePixels;
    c->bitmap_valid = !(attempt == kRadixAttempt + 1 || big_sensor);
    if (r.defer_emit && !c->bitmap_valid) return TPX_ERR_UNSUPPORTED;  // sharded: tile path only
    rc = c->bitmap_valid ? cluster_sorted(c, r) : cluster_global(c, r);
    if (rc) return rc;
    if (r.defer_emit) return TPX_OK;
    if ((rc = read_header(c, r))) return rc;
    const dev_hdr& h = *c->host_hdr;
    if (h.err & 1u) return TPX_ERR_COORD_RANGE;
    if (attempt < kRadixAttempt && h.sort_bad) {  // displacement bound violated: widen / fall back
      if (attempt + 1 > c->sort_start) {
        c->sort_start = attempt + 1;
        c->runs_at_start = 0;
      }
      continue;
    }
    if (attempt <= kRadixAttempt && (h.err & 2u)) {  // tile path inconsistency: global pipeline
      attempt = kRadixAttempt;
      continue;
    }
    break;
  }
  finish_stats(c);
  return TPX_OK;
}

// Counters of the last run from the (synchronised) host header.
static void finish_stats(tpx_cluster* c) {
  const dev_hdr& h = *c->host_hdr;
  const uint64_t k = (uint32_t)h.n_clusters;  // low word written by the scan
  c->stats.n_clusters = k;
  c->stats.cross_pairs = h.n_pairs;
  c->stats.open_hits = h.n_open_hits;
  c->stats.overflow_hits = h.n_overflow;
  for (int i = 0; i < 16; ++i) c->stats.tile_phase_cycles[i] = h.phase_cycles[i];
  if (c->profiling) {
    c->stats.n_stages = 4;
    for (int i = 0; i < 4; ++i) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]) != cudaSuccess) ms = -1.f;
      c->stats.stage_ms[i] = ms;
    }
  }
}

extern "C" {


// G4 fallback: stable global LSD radix sort of (block index, input index)
// on ceil(log2 k) bits.
static int group_radix(tpx_cluster* c, uint64_t n, uint64_t k, uint32_t* k0, uint32_t* v0, uint32_t* k1,
                       uint32_t* v1, uint32_t* hist, uint32_t* partials, uint32_t* order_out, cudaStream_t s) {
  int rc;
  const int bits = k > 1 ? 64 - __builtin_clzll(k - 1) : 0;
  const int passes = bits ? (bits + 7) / 8 : 0;
  const uint32_t tiles = n_tiles_of(n, kRadixTile);
  if (passes == 0) {
    TPX_CUDA(cudaMemcpyAsync(order_out, v0, n * 4, cudaMemcpyDeviceToDevice, s));
  }
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    const bool last = p == passes - 1;
    uint32_t* vout = last ? order_out : v1;
    k_radix_hist<uint32_t, false><<<tiles, kRadixThreads, 0, s>>>(nullptr, k0, n, 0, shift, hist, tiles);
    TPX_LAUNCHED(c);
    if ((rc = exclusive_scan(c, hist, (uint64_t)tiles * kRadixBins, hist, partials, nullptr, s))) return rc;
    k_radix_scatter_tile<false><<<tiles, kRadixThreads, 0, s>>>(nullptr, k0, v0, n, 0, shift, hist, tiles, k1, vout);
    TPX_LAUNCHED(c);
    uint32_t* t = k0;
    k0 = k1;
    k1 = t;
    t = v0;
    v0 = v1;
    v1 = t;
  }
  return TPX_OK;
}

int tpx_cluster_run_grouped(tpx_cluster* c, const tpx_hit* hits, uint64_t n, uint32_t* labels_out,
                            tpx_cluster_features* features_out, tpx_cluster_shape* shapes_out, uint64_t capacity,
                            uint64_t* n_clusters_out, uint32_t* order_out, uint32_t* offsets_out,
                            uint32_t* cluster_of_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!c || !n_clusters_out) return TPX_ERR_INVALID_ARG;
  *n_clusters_out = 0;
  if (n && (!order_out || !offsets_out || !cluster_of_out || !features_out || capacity == 0)) return TPX_ERR_INVALID_ARG;
  if (((uintptr_t)order_out & 3) || ((uintptr_t)offsets_out & 3) || ((uintptr_t)cluster_of_out & 3) ||
      ((uintptr_t)shapes_out & 15))
    return TPX_ERR_INVALID_ARG;
  uint64_t k = 0;
  c->want_first = 1;
  int rc = tpx_cluster_run_partial(c, hits, n, n, labels_out, features_out, capacity, &k, workspace,
                                   workspace_bytes, stream);
  c->want_first = 0;
  *n_clusters_out = k;
  cudaStream_t s = (cudaStream_t)stream;
  if (rc == TPX_OK && n == 0 && offsets_out) {
    TPX_CUDA(cudaMemsetAsync(offsets_out, 0, 4, s));
    TPX_CUDA(cudaStreamSynchronize(s));
  }
  if (rc != TPX_OK || n == 0) return rc;
  const layout L = make_layout(n);
  char* ws = (char*)workspace;
  // after the run only S (sorted records) is live; the scratch regions are reused
  const srec* S = (const srec*)(ws + L.S);
  uint32_t* rbits = (uint32_t*)(ws + L.bitmap);
  uint32_t* rbase = (uint32_t*)(ws + L.wcnt);
  uint32_t* fbits = (uint32_t*)(ws + L.open_hits);
  uint32_t* fbase = (uint32_t*)(ws + L.open_comps);
  uint32_t* cpos = (uint32_t*)(ws + L.keys1);        // per sorted position (k1 is free until the fallback)
  const uint32_t* first_of_label = (const uint32_t*)(ws + L.minidx);  // written by the run (tile path)
  uint32_t* first = (uint32_t*)(ws + L.flags);
  uint32_t* grank = (uint32_t*)(ws + L.ord);
  uint32_t* gsize = (uint32_t*)(ws + L.parent);
  uint32_t* k0 = (uint32_t*)(ws + L.keys0);
  uint32_t* k1 = (uint32_t*)(ws + L.keys1);
  uint32_t* v0 = (uint32_t*)(ws + L.vals0);
  uint32_t* v1 = (uint32_t*)(ws + L.vals1);
  uint32_t* hist = (uint32_t*)(ws + L.hist);
  uint32_t* partials = (uint32_t*)(ws + L.partials);
  const uint64_t nwords = L.nwords;
  const int gn = grid_for(n, 256), gk = grid_for(k, 256), gw = grid_for(nwords, 256);
  // G0: label -> ordinal (the tile path already left the label bitmap and its
  // word scan in the workspace: bit i is set iff labels[i] == i)
  if (!c->bitmap_valid) {
    k_root_bits<<<gw, 256, 0, s>>>(labels_out, n, rbits);
    TPX_LAUNCHED(c);
    k_popc<<<gw, 256, 0, s>>>(rbits, nwords, rbase);
    TPX_LAUNCHED(c);
    if ((rc = exclusive_scan(c, rbase, nwords, rbase, partials, nullptr, s))) return rc;
  }
  // G1: first sorted position per cluster (recorded by the tile path; atomics
  // over all hits otherwise)
  if (c->bitmap_valid) {
    k_group_cpos<<<gn, 256, 0, s>>>(S, n, labels_out, rbits, rbase, cpos);
    TPX_LAUNCHED(c);
    k_group_first_of<<<gk, 256, 0, s>>>(features_out, k, first_of_label, first);
    TPX_LAUNCHED(c);
  } else {
    TPX_CUDA(cudaMemsetAsync(first, 0xff, k * 4, s));
    k_group_first<<<gn, 256, 0, s>>>(S, n, labels_out, rbits, rbase, cpos, first);
    TPX_LAUNCHED(c);
  }
  // G2/G3: block index of each cluster, block table, offsets
  TPX_CUDA(cudaMemsetAsync(fbits, 0, nwords * 4, s));
  k_mark_first<<<gk, 256, 0, s>>>(first, k, fbits);
  TPX_LAUNCHED(c);
  k_popc<<<gw, 256, 0, s>>>(fbits, nwords, fbase);
  TPX_LAUNCHED(c);
  if ((rc = exclusive_scan(c, fbase, nwords, fbase, partials, nullptr, s))) return rc;
  k_group_rank<<<gk, 256, 0, s>>>(first, k, fbits, fbase, features_out, grank, cluster_of_out, gsize);
  TPX_LAUNCHED(c);
  if ((rc = exclusive_scan(c, gsize, k, offsets_out, partials, offsets_out + k, s))) return rc;
  // G4: stable sort of (block index, input index) in S order.  The block
  // index of a hit is displaced from its output place by at most its
  // cluster's span in S, so the windowed sort does it in one pass over HBM
  // (verified at every CTA border); the global LSD radix sort is the fallback.
  {
    dev_hdr* hdr = (dev_hdr*)(ws + L.hdr);
    const uint32_t ctas = n_tiles_of(n, kWSortTile);
    uint4* edge = (uint4*)hist;
    TPX_CUDA(cudaMemsetAsync(&hdr->sort_bad, 0, sizeof(hdr->sort_bad), s));
    k_window_sort_kv<12><<<ctas, kWSortThreads, window_sort_kv_smem<12>(), s>>>(cpos, grank, S, n, order_out, edge,
                                                                               hdr);
    TPX_LAUNCHED(c);
    if (ctas > 1) {
      k_kv_check<<<grid_for(ctas, 256), 256, 0, s>>>(edge, ctas, hdr);
      TPX_LAUNCHED(c);
    }
    unsigned int bad = 0;
    if ((rc = readback_sync(c, &bad, &hdr->sort_bad, sizeof(bad), s))) return rc;
    if (bad) {
      c->stats.sort_retries += 1;
      k_group_keys<<<gn, 256, 0, s>>>(S, n, cpos, grank, k0, v0);
      TPX_LAUNCHED(c);
      if ((rc = group_radix(c, n, k, k0, v0, k1, v1, hist, partials, order_out, s))) return rc;
    }
  }
  // G5: shape records
  if (shapes_out) {
    k_shapes_small<<<gk, 256, 0, s>>>(hits, order_out, offsets_out, cluster_of_out, k, (shape_rec*)shapes_out);
    TPX_LAUNCHED(c);
    k_shapes_large<<<gk, 256, 0, s>>>(hits, order_out, offsets_out, cluster_of_out, k, (shape_rec*)shapes_out);
    TPX_LAUNCHED(c);
  }
  TPX_CUDA(cudaStreamSynchronize(s));
  return TPX_OK;
}

int tpx_cluster_host_workspace_bytes(const tpx_cluster* c, uint64_t n, uint64_t capacity, size_t* bytes) {
  if (!c || !bytes) return TPX_ERR_INVALID_ARG;
  if (n >= 0xffffffffull) return TPX_ERR_TOO_MANY_HITS;
  *bytes = align256(n * 16) + align256(n * 4) + align256(capacity * 64) + run_ws_total(c, n);
  return TPX_OK;
}

int tpx_cluster_run_host(tpx_cluster* c, const tpx_hit* hits_host, uint64_t n, uint32_t* labels_host,
                         tpx_cluster_features* features_host, uint64_t capacity, uint64_t* n_clusters_out,
                         void* workspace, size_t workspace_bytes, void* stream) {
  if (!c || !n_clusters_out) return TPX_ERR_INVALID_ARG;
  *n_clusters_out = 0;
  if (n >= 0xffffffffull) return TPX_ERR_TOO_MANY_HITS;
  if (n == 0) return TPX_OK;
  if (!hits_host || !labels_host || !workspace || (!features_host && capacity)) return TPX_ERR_INVALID_ARG;
  size_t need = 0;
  tpx_cluster_host_workspace_bytes(c, n, capacity, &need);
  if (workspace_bytes < need) return TPX_ERR_OOM;
  if ((uintptr_t)workspace & 255) return TPX_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  tpx_hit* d_hits = (tpx_hit*)ws;
  uint32_t* d_labels = (uint32_t*)(ws + align256(n * 16));
  tpx_cluster_features* d_feats = (tpx_cluster_features*)(ws + align256(n * 16) + align256(n * 4));
  char* inner = ws + align256(n * 16) + align256(n * 4) + align256(capacity * 64);
  size_t inner_bytes = workspace_bytes - (size_t)(inner - ws);
  TPX_CUDA(cudaMemcpyAsync(d_hits, hits_host, n * 16, cudaMemcpyHostToDevice, s));
  uint64_t k = 0;
  int rc = tpx_cluster_run(c, d_hits, n, d_labels, d_feats, capacity, &k, inner, inner_bytes, stream);
  if (rc != TPX_OK && rc != TPX_ERR_CAPACITY) return rc;
  *n_clusters_out = k;
  TPX_CUDA(cudaMemcpyAsync(labels_host, d_labels, n * 4, cudaMemcpyDeviceToHost, s));
  uint64_t kk = k < capacity ? k : capacity;
  if (kk) TPX_CUDA(cudaMemcpyAsync(features_host, d_feats, kk * 64, cudaMemcpyDeviceToHost, s));
  TPX_CUDA(cudaStreamSynchronize(s));
  return rc;
}

int tpx_cluster_centroids(const tpx_cluster_features* features, uint64_t k, double* cxy, void* stream) {
  if (k == 0) return TPX_OK;
  if (!features || !cxy) return TPX_ERR_INVALID_ARG;
  k_centroids<<<grid_for(k, 256), 256, 0, (cudaStream_t)stream>>>(features, k, cxy);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TPX_OK : TPX_ERR_CUDA;
}

}  // extern "C"

#include "sharded.cuh"
#include "stream.cuh"
