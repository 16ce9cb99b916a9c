// sharded.cuh -- tpx_cluster_run_sharded: the ToA-sharded multi-GPU run
// (include/tpx_cluster.h "ToA-sharded multi-GPU clustering").
// Included at the end of tpx_cluster.cu (it drives the run internals there).
//
// Method: temporal splitting (§3.2.3 l.117-119) -- a rank's block is
// a contiguous ToA range up to the readout disorder, and an edge joins hits
// within dt_max (§2 (iii)(a) l.39), so only the dt_max neighbourhood of each
// border needs the neighbour's hits; border stitching (§4 l.173) becomes a
// union over (label on rank r, label on rank r+1) pairs of the lent hits.
//
// Per run, on the caller's stream (3 host synchronisations):
//   k_shard_range       validation, min/max ToA, per-4096-hit tile minima
//   allgather           [n, minToA, maxToA, flags] of every rank
//   k_shard_select      hits with toa <= maxToA(r-1) + dt (tile minima skip
//                       the rest), in input order -> lent to rank r-1
//   allgather           lent counts                    -> sync 1 (host sizes)
//   send/recv           lent hits + their block positions
//   run_core            sort + tile clustering of [owned | halo] (sync 2:
//                       sort status), labels written as global indices
//   send/recv           rank r+1's labels of the lent hits
//   k_shard_pairs       pairs (my label, peer label) of halo hits
//   allgather           pairs of every rank
//   k_hash_*            union of all pairs in a hash table (smallest wins)
//   k_shard_changed     label bits of merged-away labels cleared
//   k_shard_relabel     owned labels -> final labels
//   emit_sorted         records; merged-away ones become partials
//   allgather           partials of every rank (+ error flags)
//   k_shard_fold        partials folded into the owner's records -> sync 3
#pragma once
#include <memory>

#include "comm.h"

namespace tpx {

constexpr int kShardTile = 4096;  // hits per tile minimum (halo selection index)
constexpr uint32_t kHashEmpty = 0xffffffffu;

// Device-side state of one sharded run (256 B).
struct shard_state {
  unsigned long long hdr[4];  // this rank: n, minToA, maxToA, flags (bit 0 coordinates)
  unsigned long long c_send;  // hits selected for rank r-1 (may exceed the capacity)
  unsigned long long n_removed;
  unsigned long long kmin, kmax;  // range of merged-away labels in this rank's block
  unsigned long long any_err;     // OR of every rank's error flags
  unsigned long long pad[23];
};
static_assert(sizeof(shard_state) == 256, "shard_state layout");

__global__ void k_shard_init(shard_state* st, uint64_t n, unsigned long long* pair_count) {
  if (threadIdx.x == 0) {
    st->hdr[0] = n;
    st->hdr[1] = ~0ull;
    st->hdr[2] = 0;
    st->hdr[3] = 0;
    st->c_send = 0;
    st->n_removed = 0;
    st->kmin = ~0ull;
    st->kmax = 0;
    st->any_err = 0;
    *pair_count = 0;
  }
}

__device__ __forceinline__ void block_minmax(unsigned long long& mn, unsigned long long& mx, unsigned& bad,
                                             unsigned long long* sm) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(kFull, mn, o));
    mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    bad |= __shfl_xor_sync(kFull, bad, o);
  }
  const unsigned w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane_id() == 0) {
    sm[w] = mn;
    sm[32 + w] = mx;
    sm[64 + w] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (unsigned i = 1; i < nw; ++i) {
      mn = min(mn, sm[i]);
      mx = max(mx, sm[32 + i]);
      bad |= (unsigned)sm[64 + i];
    }
  }
}

// One CTA per 4096-hit tile: coordinates / ToA range, block min / max
// ToA, tile minimum (the halo selection reads only tiles that can qualify).
__global__ void __launch_bounds__(256) k_shard_range(const tpx_hit* __restrict__ hits, uint64_t n, uint32_t width,
                                                     uint32_t height, unsigned long long* __restrict__ tile_min,
                                                     shard_state* st) {
  __shared__ unsigned long long sm[96];
  const uint64_t t0 = (uint64_t)blockIdx.x * kShardTile;
  unsigned long long mn = ~0ull, mx = 0;
  unsigned bad = 0;
#pragma unroll 4
  for (int k = 0; k < kShardTile / 256; ++k) {
    const uint64_t i = t0 + (uint64_t)k * 256 + threadIdx.x;
    if (i < n) {
      const hit4 h = load_hit(hits + i);
      mn = min(mn, (unsigned long long)h.toa);
      mx = max(mx, (unsigned long long)h.toa);
      bad |= (h.x >= width) | (h.y >= height) | (h.toa >> 48 != 0);
    }
  }
  block_minmax(mn, mx, bad, sm);
  if (threadIdx.x == 0) {
    tile_min[blockIdx.x] = mn;
    atomicMin(&st->hdr[1], mn);
    atomicMax(&st->hdr[2], mx);
    if (bad) atomicOr(&st->hdr[3], 1ull);
  }
}

// Lent hits for rank r-1 (r > 0): every hit with toa <= maxToA(r-1) + dt, in
// input order (one CTA; tiles whose minimum exceeds the limit are skipped).
constexpr int kSelThreads = 1024;
__global__ void __launch_bounds__(kSelThreads) k_shard_select(const tpx_hit* __restrict__ hits, uint64_t n,
                                                              const unsigned long long* __restrict__ tile_min,
                                                              uint32_t n_tiles,
                                                              const unsigned long long* __restrict__ all_hdr, int rank,
                                                              uint64_t dt, tpx_hit* __restrict__ out,
                                                              uint32_t* __restrict__ idx_out, uint32_t cap,
                                                              shard_state* st) {
  __shared__ uint32_t cand[kSelThreads];
  __shared__ uint32_t wsum[kSelThreads / 32];
  __shared__ uint32_t s_nc;
  if (rank == 0) return;  // c_send stays 0
  const unsigned long long limit = all_hdr[(rank - 1) * 4 + 2] + dt;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  // block-wide exclusive scan of a 0/1 flag in thread order
  auto scan = [&](bool f, uint32_t* total) -> uint32_t {
    const unsigned b = __ballot_sync(kFull, f);
    if (lane == 0) wsum[warp] = __popc(b);
    __syncthreads();
    uint32_t before = 0, tot = 0;
    for (unsigned w = 0; w < kSelThreads / 32; ++w) {
      const uint32_t v = wsum[w];
      before += w < warp ? v : 0;
      tot += v;
    }
    __syncthreads();
    *total = tot;
    return before + __popc(b & lanemask_lt());
  };
  uint64_t base = 0;
  for (uint32_t t0 = 0; t0 < n_tiles; t0 += kSelThreads) {
    const uint32_t t = t0 + threadIdx.x;
    const bool c = t < n_tiles && tile_min[t] <= limit;
    uint32_t nc;
    const uint32_t pos = scan(c, &nc);
    if (c) cand[pos] = t;
    if (threadIdx.x == 0) s_nc = nc;
    __syncthreads();
    nc = s_nc;
    for (uint32_t k = 0; k < nc; ++k) {
      const uint64_t tb = (uint64_t)cand[k] * kShardTile;
      for (int q = 0; q < kShardTile / kSelThreads; ++q) {
        const uint64_t i = tb + (uint64_t)q * kSelThreads + threadIdx.x;
        bool sel = false;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (i < n) {
          v = __ldg(reinterpret_cast<const uint4*>(hits + i));
          sel = (((unsigned long long)v.y << 32) | v.x) <= limit;
        }
        uint32_t tot;
        const uint32_t p = scan(sel, &tot);
        if (sel && base + p < cap) {
          reinterpret_cast<uint4*>(out)[base + p] = v;
          idx_out[base + p] = (uint32_t)i;
        }
        base += tot;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) st->c_send = base;
}

// out[k] = labels[idx[k]]: this rank's labels of the hits it lent.
__global__ void k_shard_gather_labels(const uint32_t* __restrict__ labels, const uint32_t* __restrict__ idx,
                                      uint64_t c, uint32_t* __restrict__ out) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < c; k += (uint64_t)gridDim.x * blockDim.x)
    out[k] = labels[idx[k]];
}

// Boundary pairs (my label, next rank's label) of the halo hits, a != b;
// slot 0 of `pairs` is the count (u64).
__global__ void k_shard_pairs(const uint32_t* __restrict__ mine, const uint32_t* __restrict__ peer, uint64_t c,
                              uint2* __restrict__ pairs) {
  unsigned long long* count = reinterpret_cast<unsigned long long*>(pairs);
  for (uint64_t k0 = (uint64_t)blockIdx.x * blockDim.x; k0 < c; k0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = k0 + threadIdx.x;
    const bool v = k < c && mine[k] != peer[k];
    const uint32_t slot = warp_append(v, count);
    if (v) pairs[1 + slot] = make_uint2(mine[k], peer[k]);
  }
}

// ---------------------------------------------------------------- hash union
// Open-addressing table of the labels in all pairs (T = 2^bits slots), a
// lock-free union-find over its slots: a root with the larger label is linked
// under the one with the smaller, so every root holds the smallest label of
// its set -- the label of the merged cluster (reading R6).  Every rank runs
// it on the same gathered pairs and reaches the same partition.
__device__ __forceinline__ uint32_t hash_slot(uint32_t key, uint32_t mask) { return (key * 0x9E3779B1u) & mask; }

__device__ __forceinline__ uint32_t hash_lookup(const uint32_t* keys, uint32_t mask, uint32_t key) {
  for (uint32_t s = hash_slot(key, mask);; s = (s + 1) & mask) {
    const uint32_t k = keys[s];
    if (k == key) return s;
    if (k == kHashEmpty) return kHashEmpty;
  }
}

__global__ void k_hash_init(uint32_t* keys, uint32_t* parent, uint32_t T) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < T; i += gridDim.x * blockDim.x) {
    keys[i] = kHashEmpty;
    parent[i] = i;
  }
}

__device__ __forceinline__ void hash_insert(uint32_t* keys, uint32_t mask, uint32_t key) {
  for (uint32_t s = hash_slot(key, mask);; s = (s + 1) & mask) {
    const uint32_t old = atomicCAS(keys + s, kHashEmpty, key);
    if (old == kHashEmpty || old == key) return;
  }
}

// Iterate the gathered pairs: world segments of `stride` uint2, count in slot 0.
template <typename F>
__device__ __forceinline__ void for_all_pairs(const uint2* all, int world, uint64_t stride, F f) {
  for (int g = 0; g < world; ++g) {
    const uint2* seg = all + (uint64_t)g * stride;
    const uint64_t cnt = *reinterpret_cast<const unsigned long long*>(seg);
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += (uint64_t)gridDim.x * blockDim.x)
      f(seg[1 + k]);
  }
}

__global__ void k_hash_insert(const uint2* __restrict__ all, int world, uint64_t stride, uint32_t* keys, uint32_t mask) {
  for_all_pairs(all, world, stride, [&](uint2 p) {
    hash_insert(keys, mask, p.x);
    hash_insert(keys, mask, p.y);
  });
}

__device__ __forceinline__ uint32_t slot_root(const uint32_t* parent, uint32_t s) {
  uint32_t nx;
  while (s != (nx = ld_cg(parent + s))) s = nx;
  return s;
}

__global__ void k_hash_union(const uint2* __restrict__ all, int world, uint64_t stride, const uint32_t* __restrict__ keys,
                             uint32_t mask, uint32_t* parent) {
  for_all_pairs(all, world, stride, [&](uint2 p) {
    uint32_t a = slot_root(parent, hash_lookup(keys, mask, p.x));
    uint32_t b = slot_root(parent, hash_lookup(keys, mask, p.y));
    while (a != b) {
      if (keys[a] > keys[b]) {  // link the root with the larger label under the smaller
        const uint32_t t = a;
        a = b;
        b = t;
      }
      const uint32_t old = atomicCAS(parent + b, b, a);
      if (old == b) break;
      b = slot_root(parent, old);
      a = slot_root(parent, a);
    }
  });
}

// final[s] = label of s's set; merged-away labels of this rank's block get
// their label bit cleared (k_emit turns their records into partials) and
// bound the relabel pass.
__global__ void k_shard_changed(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ parent, uint32_t T,
                                uint32_t* __restrict__ finals, uint64_t own_off, uint64_t n, uint32_t* bitmap,
                                shard_state* st) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < T; s += gridDim.x * blockDim.x) {
    const uint32_t k = keys[s];
    if (k == kHashEmpty) continue;
    const uint32_t f = keys[slot_root(parent, s)];
    finals[s] = f;
    if (f != k && k >= own_off && k < own_off + n) {
      const uint32_t l = (uint32_t)(k - own_off);
      atomicAnd(bitmap + (l >> 5), ~(1u << (l & 31)));
      atomicMin(&st->kmin, (unsigned long long)k);
      atomicMax(&st->kmax, (unsigned long long)k);
    }
  }
}

__global__ void k_shard_relabel(uint32_t* labels, uint64_t n, const uint32_t* __restrict__ keys,
                                const uint32_t* __restrict__ finals, uint32_t mask, const shard_state* st) {
  const unsigned long long lo = st->kmin, hi = st->kmax;
  if (lo > hi) return;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t L = labels[i];
    if (L < lo || L > hi) continue;
    const uint32_t s = hash_lookup(keys, mask, L);
    if (s != kHashEmpty) labels[i] = finals[s];
  }
}

// Partials: the removed records (global labels) relabelled to their final
// label; slot 0 = header {count, error flags of this rank}.
__global__ void k_shard_partials(tpx_cluster_features* part, const uint32_t* __restrict__ keys,
                                 const uint32_t* __restrict__ finals, uint32_t mask, const shard_state* st,
                                 const dev_hdr* hdr) {
  const uint64_t cnt = st->n_removed;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = hash_lookup(keys, mask, part[1 + k].label);
    part[1 + k].label = s == kHashEmpty ? part[1 + k].label : finals[s];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long* h = reinterpret_cast<unsigned long long*>(part);
    h[0] = cnt;
    h[1] = hdr->err;
  }
}

// Owner fold: every gathered partial whose final label is in this block is
// added into that record (integer add / min / max: exact, order independent).
__global__ void k_shard_fold(const tpx_cluster_features* __restrict__ all, int world, uint64_t stride,
                             uint64_t own_off, uint64_t n, tpx_cluster_features* out, uint64_t capacity,
                             const dev_hdr* hdr, shard_state* st) {
  const uint64_t k = min((uint64_t)(uint32_t)hdr->n_clusters, capacity);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long e = 0;
    for (int g = 0; g < world; ++g) e |= reinterpret_cast<const unsigned long long*>(all + (uint64_t)g * stride)[1];
    st->any_err = e;
  }
  for (int g = 0; g < world; ++g) {
    const tpx_cluster_features* seg = all + (uint64_t)g * stride;
    const uint64_t cnt = reinterpret_cast<const unsigned long long*>(seg)[0];
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (uint64_t)gridDim.x * blockDim.x) {
      const tpx_cluster_features f = seg[1 + q];
      if (f.label < own_off || f.label >= own_off + n) continue;
      uint64_t lo = 0, hi = k;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (out[mid].label < f.label) lo = mid + 1; else hi = mid;
      }
      if (lo >= k || out[lo].label != f.label) continue;  // truncated by the capacity
      tpx_cluster_features* d = out + lo;
      atomicAdd(&d->size, f.size);
      atomicMin((unsigned long long*)&d->toa_min, (unsigned long long)f.toa_min);
      atomicMax((unsigned long long*)&d->toa_max, (unsigned long long)f.toa_max);
      atomicAdd((unsigned long long*)&d->tot_sum, (unsigned long long)f.tot_sum);
      atomicAdd((unsigned long long*)&d->sum_x, (unsigned long long)f.sum_x);
      atomicAdd((unsigned long long*)&d->sum_y, (unsigned long long)f.sum_y);
      atomicAdd((unsigned long long*)&d->sum_tot_x, (unsigned long long)f.sum_tot_x);
      atomicAdd((unsigned long long*)&d->sum_tot_y, (unsigned long long)f.sum_tot_y);
    }
  }
}

}  // namespace tpx

namespace {

constexpr uint32_t kHaloCap = TPX_SHARD_HALO_CAP;

struct shard_layout {
  size_t run, state, all_hdr, counts, tile_min, send_hits, send_idx, recv_hits, recv_idx, halo_labels, lent_labels,
      peer_labels, pairs, all_pairs, hkeys, hparent, hfinal, part, all_part, total;
  uint64_t hash_slots, pair_stride, part_stride;
};

uint32_t hash_slots_for(uint64_t keys) {
  uint64_t t = 1024;
  while (t < 2 * keys) t <<= 1;
  return (uint32_t)t;
}

// Workspace of a sharded run: the run itself for n + kHaloCap hits, then the
// exchange buffers sized for world ranks each lending at most kHaloCap hits.
shard_layout make_shard_layout(uint64_t n, int world) {
  shard_layout S;
  size_t off = make_layout(n + kHaloCap).total;
  S.run = 0;
  auto take = [&](size_t b) {
    size_t o = off;
    off += align256(b);
    return o;
  };
  const uint64_t cap = kHaloCap;
  S.hash_slots = hash_slots_for(2ull * cap * world);
  S.pair_stride = cap + 1;
  S.part_stride = 2 * cap + 1;
  S.state = take(sizeof(shard_state));
  S.all_hdr = take((size_t)world * 32);
  S.counts = take((size_t)world * 8);
  S.tile_min = take((size_t)n_tiles_of(n, kShardTile) * 8);
  S.send_hits = take(cap * 16);
  S.send_idx = take(cap * 4);
  S.recv_hits = take(cap * 16);
  S.recv_idx = take(cap * 4);
  S.halo_labels = take(cap * 4);
  S.lent_labels = take(cap * 4);
  S.peer_labels = take(cap * 4);
  S.pairs = take(S.pair_stride * 8);
  S.all_pairs = take((size_t)world * S.pair_stride * 8);
  S.hkeys = take(S.hash_slots * 4);
  S.hparent = take(S.hash_slots * 4);
  S.hfinal = take(S.hash_slots * 4);
  S.part = take(S.part_stride * 64);
  S.all_part = take((size_t)world * S.part_stride * 64);
  S.total = off;
  return S;
}

#define TPX_SH(call)           \
  do {                         \
    int rc_ = (call);          \
    if (rc_ != TPX_OK) return rc_; \
  } while (0)

}  // namespace

extern "C" {

int tpx_cluster_sharded_workspace_bytes(const tpx_cluster* c, uint64_t n_local, int world, size_t* bytes) {
  if (!c || !bytes || world < 1 || world > 64) return TPX_ERR_INVALID_ARG;
  if (n_local + kHaloCap >= 0xffffffffull) return TPX_ERR_TOO_MANY_HITS;
  *bytes = make_shard_layout(n_local, world).total;
  return TPX_OK;
}

int tpx_cluster_run_sharded(tpx_cluster* c, tpx_comm* comm, const tpx_hit* local_hits, uint64_t n_local,
                            uint32_t* labels_out, tpx_cluster_features* features_out, uint64_t capacity,
                            uint64_t* n_clusters_out, uint64_t* global_offset_out, void* workspace,
                            size_t workspace_bytes, void* stream) {
  if (!c || !comm || !n_clusters_out) return TPX_ERR_INVALID_ARG;
  *n_clusters_out = 0;
  const int G = comm_world(comm), R = comm_rank(comm);
  if (G > 64) return TPX_ERR_INVALID_ARG;
  // argument checks are local but identical in meaning on every rank; a rank
  // that fails them returns before any collective (caller error)
  if (n_local == 0 || !local_hits || !labels_out || !workspace || (!features_out && capacity)) return TPX_ERR_INVALID_ARG;
  if (((uintptr_t)local_hits & 15) || ((uintptr_t)workspace & 255) || ((uintptr_t)features_out & 15) ||
      ((uintptr_t)labels_out & 3))
    return TPX_ERR_INVALID_ARG;
  if (c->variant != TPX_VARIANT_LOCAL) return TPX_ERR_UNSUPPORTED;
  if (c->width > (uint32_t)kMaxTileWidth || (uint64_t)c->width * c->height + c->width > kMaxTilePixels)
    return TPX_ERR_UNSUPPORTED;  // the global pipeline has no sharded emission
  if (n_local + kHaloCap >= 0xffffffffull) return TPX_ERR_TOO_MANY_HITS;
  const shard_layout SL = make_shard_layout(n_local, G);
  if (workspace_bytes < SL.total) return TPX_ERR_OOM;
  if (ensure_cuda(c)) return TPX_ERR_CUDA;
  memset(&c->stats, 0, sizeof(c->stats));
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  shard_state* st = (shard_state*)(ws + SL.state);
  unsigned long long* all_hdr = (unsigned long long*)(ws + SL.all_hdr);
  unsigned long long* counts = (unsigned long long*)(ws + SL.counts);
  unsigned long long* tile_min = (unsigned long long*)(ws + SL.tile_min);
  tpx_hit* send_hits = (tpx_hit*)(ws + SL.send_hits);
  uint32_t* send_idx = (uint32_t*)(ws + SL.send_idx);
  tpx_hit* recv_hits = (tpx_hit*)(ws + SL.recv_hits);
  uint32_t* recv_idx = (uint32_t*)(ws + SL.recv_idx);
  uint32_t* halo_labels = (uint32_t*)(ws + SL.halo_labels);
  uint32_t* lent_labels = (uint32_t*)(ws + SL.lent_labels);
  uint32_t* peer_labels = (uint32_t*)(ws + SL.peer_labels);
  uint2* pairs = (uint2*)(ws + SL.pairs);
  uint2* all_pairs = (uint2*)(ws + SL.all_pairs);
  uint32_t* hkeys = (uint32_t*)(ws + SL.hkeys);
  uint32_t* hparent = (uint32_t*)(ws + SL.hparent);
  uint32_t* hfinal = (uint32_t*)(ws + SL.hfinal);
  tpx_cluster_features* part = (tpx_cluster_features*)(ws + SL.part);
  tpx_cluster_features* all_part = (tpx_cluster_features*)(ws + SL.all_part);
  const uint64_t n = n_local, dt = c->dt;

  // ---- 1. ranges, lent hits, counts
  nvtx_range nv_all("tpx:sharded_run");
  std::unique_ptr<nvtx_range> nv(new nvtx_range("tpx:shard_exchange"));
  k_shard_init<<<1, 32, 0, s>>>(st, n, reinterpret_cast<unsigned long long*>(pairs));
  TPX_LAUNCHED(c);
  const uint32_t ntiles = n_tiles_of(n, kShardTile);
  k_shard_range<<<ntiles, 256, 0, s>>>(local_hits, n, c->width, c->height, tile_min, st);
  TPX_LAUNCHED(c);
  TPX_SH(comm_allgather(comm, st->hdr, all_hdr, 32, s));
  k_shard_select<<<1, kSelThreads, 0, s>>>(local_hits, n, tile_min, ntiles, all_hdr, R, dt, send_hits, send_idx,
                                           kHaloCap, st);
  TPX_LAUNCHED(c);
  TPX_SH(comm_allgather(comm, &st->c_send, counts, 8, s));
  // sync 1: every rank's [n, min, max, flags] and lent count on the host
  struct {
    unsigned long long hdr[64][4];
    unsigned long long cnt[64];
  } h;
  TPX_SH(readback_sync(c, h.hdr, all_hdr, (size_t)G * 32, s));
  TPX_SH(readback_sync(c, h.cnt, counts, (size_t)G * 8, s));
  uint64_t o_r = 0, total = 0;
  int flags = 0;
  for (int g = 0; g < G; ++g) {
    if (g < R) o_r += h.hdr[g][0];
    total += h.hdr[g][0];
    flags |= (int)h.hdr[g][3];
  }
  if (global_offset_out) *global_offset_out = o_r;
  if (flags & 1) return TPX_ERR_COORD_RANGE;
  if (total >= 0xffffffffull) return TPX_ERR_TOO_MANY_HITS;
  for (int g = 0; g < G; ++g) {
    if (h.cnt[g] > kHaloCap) return TPX_ERR_UNSUPPORTED;  // halo above TPX_SHARD_HALO_CAP
    for (int t = g + 2; t < G; ++t)
      if (h.hdr[t][1] <= h.hdr[g][2] + dt) return TPX_ERR_UNSUPPORTED;  // an edge could skip a rank
  }
  const uint64_t c_send = h.cnt[R], c_recv = R + 1 < G ? h.cnt[R + 1] : 0;
  const uint64_t next_off = o_r + n;
  TPX_SH(comm_group_start(comm));
  TPX_SH(comm_sendrecv(comm, R - 1, send_hits, c_send * 16, R + 1, recv_hits, c_recv * 16, s));
  TPX_SH(comm_sendrecv(comm, R - 1, send_idx, c_send * 4, R + 1, recv_idx, c_recv * 4, s));
  TPX_SH(comm_group_end(comm));

  nv.reset();
  // ---- 2. cluster [owned | halo]: sort (sync 2) + tiles + border merge
  run_ptrs r;
  r.L = make_layout(n + c_recv);
  r.hits = hit_src(local_hits, n, recv_hits);
  r.n = n + c_recv;
  r.n_owned = n;
  r.labels = labels_out;
  r.feats = features_out;
  r.capacity = capacity;
  r.ws = ws;
  r.s = s;
  r.lm.halo_labels = halo_labels;
  r.lm.halo_idx = recv_idx;
  r.lm.own_off = (uint32_t)o_r;
  r.lm.next_off = (uint32_t)next_off;
  r.defer_emit = true;
  TPX_SH(run_core(c, r));

  // ---- 3. boundary pairs of every rank, union
  nv.reset(new nvtx_range("tpx:shard_union"));
  if (c_send) {
    k_shard_gather_labels<<<grid_for(c_send, 256), 256, 0, s>>>(labels_out, send_idx, c_send, lent_labels);
    TPX_LAUNCHED(c);
  }
  TPX_SH(comm_sendrecv(comm, R - 1, lent_labels, c_send * 4, R + 1, peer_labels, c_recv * 4, s));
  if (c_recv) {
    k_shard_pairs<<<grid_for(c_recv, 256), 256, 0, s>>>(halo_labels, peer_labels, c_recv, pairs);
    TPX_LAUNCHED(c);
  }
  uint64_t pmax = 0, psum = 0, qmax = 0;
  for (int g = 0; g < G; ++g) {
    const uint64_t cr = g + 1 < G ? h.cnt[g + 1] : 0;  // pairs of rank g <= its halo
    pmax = cr > pmax ? cr : pmax;
    psum += cr;
    const uint64_t q = cr + h.cnt[g];  // merged-away records of rank g <= its two borders
    qmax = q > qmax ? q : qmax;
  }
  const uint64_t pstride = pmax + 1, qstride = qmax + 1;
  dev_hdr* hdr = (dev_hdr*)(ws + r.L.hdr);
  uint32_t* bitmap = (uint32_t*)(ws + r.L.bitmap);
  const uint32_t T = hash_slots_for(2 * psum);
  const uint32_t mask = T - 1;
  if (G > 1) {
    TPX_SH(comm_allgather(comm, pairs, all_pairs, pstride * 8, s));
    k_hash_init<<<grid_for(T, 256), 256, 0, s>>>(hkeys, hparent, T);
    TPX_LAUNCHED(c);
    if (psum) {
      const int gp = grid_for(pmax, 256);
      k_hash_insert<<<gp, 256, 0, s>>>(all_pairs, G, pstride, hkeys, mask);
      TPX_LAUNCHED(c);
      k_hash_union<<<gp, 256, 0, s>>>(all_pairs, G, pstride, hkeys, mask, hparent);
      TPX_LAUNCHED(c);
      k_shard_changed<<<grid_for(T, 256), 256, 0, s>>>(hkeys, hparent, T, hfinal, o_r, n, bitmap, st);
      TPX_LAUNCHED(c);
      k_shard_relabel<<<grid_for(n, 256), 256, 0, s>>>(labels_out, n, hkeys, hfinal, mask, st);
      TPX_LAUNCHED(c);
    }
  }

  nv.reset();
  // ---- 4. records: emission (merged-away records -> partials), owner fold
  unsigned long long* n_removed = &st->n_removed;
  TPX_SH(emit_sorted(c, r, part + 1, n_removed));
  if (G > 1) {
    k_shard_partials<<<grid_for(qmax, 256), 256, 0, s>>>(part, hkeys, hfinal, mask, st, hdr);
    TPX_LAUNCHED(c);
    TPX_SH(comm_allgather(comm, part, all_part, qstride * 64, s));
    k_shard_fold<<<grid_for(qmax * G, 256), 256, 0, s>>>(all_part, G, qstride, o_r, n, features_out, capacity, hdr, st);
    TPX_LAUNCHED(c);
  }
  // sync 3: counts, error flags of every rank
  TPX_CUDA(readback_async(c->host_scratch, st, sizeof(shard_state), s));
  c->stats.kernel_launches++;
  TPX_SH(read_header(c, r));
  shard_state hs;
  memcpy(&hs, c->host_scratch, sizeof(hs));
  finish_stats(c);
  c->stats.n_hits = n + c_recv;
  c->stats.cross_pairs = psum;
  const unsigned long long errs = (G > 1 ? hs.any_err : c->host_hdr->err) | c->host_hdr->err;
  if (errs & 2u) return TPX_ERR_UNSUPPORTED;  // tile-path inconsistency (never observed): unsharded run needed
  if (hs.n_removed > qmax) return TPX_ERR_UNSUPPORTED;
  const uint64_t k = c->stats.n_clusters;
  *n_clusters_out = k;
  return k > capacity ? TPX_ERR_CAPACITY : TPX_OK;
}

}  // extern "C"
