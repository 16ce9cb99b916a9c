// stream.cuh -- streaming ingest with exact cross-buffer carry-over
// (included at the end of tpx_cluster.cu, whose host helpers
// it uses).
//
// The paper's GPU driver (Alg. "High-level GPU clustering", §4
// l.160-182) fills host buffers with Alg. "Hit buffer filling" (l.184-213,
// buffill.h), copies each to the device, clusters it, orders the clusters by
// time (Step 6) and copies hits and labels back (Step 8).  Border clusters
// are stitched exactly here: after buffer k (cut C_k, every later hit has
// toa >= C_k) a cluster is OPEN iff some hit has toa + dt_max >= C_k -- only
// those can still meet a later hit (l.119: "we only need to examine the
// dt_max-time neighborhood around each border").  Closed clusters are final
// and emitted; the hits of open clusters are carried on the device into
// buffer k+1, merged with its new hits by arrival index, so that a local
// position order equals the arrival order and a cluster's label (its
// smallest local position) maps to its smallest arrival index.  The union of
// all emitted clusters equals the clustering of the whole stream.
#pragma once
#include <cuda_runtime.h>

#include <cstring>
#include <deque>
#include <new>
#include <vector>

#include "buffill.h"

namespace tpx {

// Same 80-byte layout as tpx_stream_cluster.
static_assert(sizeof(tpx_stream_cluster) == 80, "stream cluster record");

// Merge the carried hits (ascending arrival index) with the new hits
// (ascending arrival index): each element's place = its own rank + the number
// of elements of the other list with a smaller index (indices are distinct).
__device__ __forceinline__ uint32_t count_less(const uint64_t* __restrict__ a, uint32_t n, uint64_t v) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_stream_merge(const tpx_hit* __restrict__ carry, const uint64_t* __restrict__ carry_g, uint32_t nc,
                               const tpx_hit* __restrict__ fresh, const uint64_t* __restrict__ fresh_g, uint32_t nn,
                               tpx_hit* __restrict__ out, uint64_t* __restrict__ out_g) {
  const uint64_t total = (uint64_t)nc + nn;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (i < nc) {
      const uint64_t g = carry_g[i];
      const uint64_t pos = i + count_less(fresh_g, nn, g);
      reinterpret_cast<uint4*>(out)[pos] = reinterpret_cast<const uint4*>(carry)[i];
      out_g[pos] = g;
    } else {
      const uint32_t j = (uint32_t)(i - nc);
      const uint64_t g = fresh_g[j];
      const uint64_t pos = j + count_less(carry_g, nc, g);
      reinterpret_cast<uint4*>(out)[pos] = __ldcs(reinterpret_cast<const uint4*>(fresh) + j);
      out_g[pos] = g;
    }
  }
}

// Per cluster block (Step-6 order): closed unless a hit lies within dt_max of
// the cut; flags and sizes for the two scans.
__global__ void k_stream_blocks(const uint32_t* __restrict__ cluster_of, const tpx_cluster_features* __restrict__ feats,
                                uint64_t k, uint64_t cut, uint64_t dt, int final_buffer,
                                uint32_t* __restrict__ closed_flag, uint32_t* __restrict__ closed_size) {
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < k; g += (uint64_t)gridDim.x * blockDim.x) {
    const tpx_cluster_features f = feats[cluster_of[g]];
    const bool open = !final_buffer && f.toa_max + dt >= cut;
    closed_flag[g] = open ? 0u : 1u;
    closed_size[g] = open ? 0u : f.size;
  }
}

struct stream_emit_args {
  const tpx_hit* hits;          // merged buffer (arrival order)
  const uint64_t* gidx;         // arrival index per local position
  const uint32_t* order;        // Step-6 order (local positions)
  const uint32_t* offsets;      // block offsets
  const uint32_t* cluster_of;   // block -> feature record
  const tpx_cluster_features* feats;
  const uint32_t* closed_flag;  // per block
  const uint32_t* cidx;         // closed block -> output cluster index
  const uint32_t* hoff;         // closed block -> output hit offset
  uint64_t k;
  tpx_stream_cluster* out_cl;
  tpx_hit* out_hits;            // may be null (one-shot run: the caller has the hits)
  uint64_t* out_g;              // arrival index per output hit (u64), or null
  uint32_t* out_g32;            // arrival index per output hit (u32), or null
  uint64_t hoff_base;           // added to record offsets (one-shot: position in order_out)
  uint32_t* open_flag;          // per local position: hit of an open cluster
};

__device__ __forceinline__ void stream_put_hit(const stream_emit_args& a, uint64_t q, uint32_t p) {
  if (a.out_hits) reinterpret_cast<uint4*>(a.out_hits)[q] = reinterpret_cast<const uint4*>(a.hits)[p];
  if (a.out_g) a.out_g[q] = a.gidx[p];
  if (a.out_g32) a.out_g32[q] = (uint32_t)a.gidx[p];
}

__device__ __forceinline__ void stream_block_head(const stream_emit_args& a, uint64_t g) {
  const uint32_t c = a.cluster_of[g];
  const tpx_cluster_features f = a.feats[c];
  tpx_stream_cluster r;
  r.label = a.gidx[f.label];  // smallest local position = smallest arrival index
  r.offset = a.hoff_base + a.hoff[g];
  r.size = f.size;
  r.reserved = 0;
  r.toa_min = f.toa_min;
  r.toa_max = f.toa_max;
  r.tot_sum = f.tot_sum;
  r.sum_x = f.sum_x;
  r.sum_y = f.sum_y;
  r.sum_tot_x = f.sum_tot_x;
  r.sum_tot_y = f.sum_tot_y;
  a.out_cl[a.cidx[g]] = r;
}

constexpr uint32_t kStreamWarpMin = 32;

// Small blocks: one thread each.  Closed: record + hits gathered into the
// batch; open: mark the hits for the carry.
__global__ void k_stream_emit_small(stream_emit_args a) {
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < a.k; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t o0 = a.offsets[g], o1 = a.offsets[g + 1];
    if (o1 - o0 >= kStreamWarpMin) continue;
    if (a.closed_flag[g]) {
      stream_block_head(a, g);
      const uint64_t h0 = a.hoff[g];
      for (uint32_t j = o0; j < o1; ++j) stream_put_hit(a, h0 + (j - o0), a.order[j]);
    } else {
      for (uint32_t j = o0; j < o1; ++j) a.open_flag[a.order[j]] = 1u;
    }
  }
}

// Large blocks: one warp each.
__global__ void k_stream_emit_large(stream_emit_args a) {
  const unsigned lane = lane_id();
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t g0 = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; g0 < a.k; g0 += nw * 32) {
    const uint64_t gl = g0 + lane;
    const bool is_big = gl < a.k && a.offsets[gl + 1] - a.offsets[gl] >= kStreamWarpMin;
    unsigned todo = __ballot_sync(kFull, is_big);
    while (todo) {
      const uint64_t g = g0 + (__ffs(todo) - 1);
      todo &= todo - 1;
      const uint32_t o0 = a.offsets[g], o1 = a.offsets[g + 1];
      if (a.closed_flag[g]) {
        if (lane == 0) stream_block_head(a, g);
        const uint64_t h0 = a.hoff[g];
        for (uint32_t j = o0 + lane; j < o1; j += 32) stream_put_hit(a, h0 + (j - o0), a.order[j]);
      } else {
        for (uint32_t j = o0 + lane; j < o1; j += 32) a.open_flag[a.order[j]] = 1u;
      }
    }
  }
}

// Arrival indices of a run of consecutive input hits.
__global__ void k_iota64(uint64_t* __restrict__ g, uint64_t n, uint64_t base) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    g[i] = base + i;
}

// Carried hits in local (= arrival) order.
__global__ void k_stream_carry(const tpx_hit* __restrict__ hits, const uint64_t* __restrict__ gidx, uint64_t n,
                               const uint32_t* __restrict__ open_flag, const uint32_t* __restrict__ cpos,
                               tpx_hit* __restrict__ carry, uint64_t* __restrict__ carry_g) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (!open_flag[i]) continue;
    const uint32_t q = cpos[i];
    reinterpret_cast<uint4*>(carry)[q] = reinterpret_cast<const uint4*>(hits)[i];
    carry_g[q] = gidx[i];
  }
}

// Growable pinned host array (H2D / D2H at full PCIe speed).
template <typename T>
struct pinned_vec {
  T* p = nullptr;
  size_t n = 0, cap = 0;
  bool ok = true;
  pinned_vec() = default;
  pinned_vec(const pinned_vec&) = delete;
  pinned_vec& operator=(const pinned_vec&) = delete;
  ~pinned_vec() {
    if (p) cudaFreeHost(p);
  }
  size_t size() const { return n; }
  void clear() { n = 0; }
  bool reserve(size_t want) {
    if (want <= cap) return true;
    size_t nc = cap ? cap : 1024;
    while (nc < want) nc *= 2;
    T* q = nullptr;
    if (cudaHostAlloc((void**)&q, nc * sizeof(T), cudaHostAllocDefault) != cudaSuccess) {
      ok = false;
      return false;
    }
    if (n) memcpy(q, p, n * sizeof(T));
    if (p) cudaFreeHost(p);
    p = q;
    cap = nc;
    return true;
  }
  void push_back(const T& v) {
    if (n == cap && !reserve(n + 1)) return;
    p[n++] = v;
  }
  void swap(pinned_vec& o) {
    T* tp = p;
    p = o.p;
    o.p = tp;
    size_t t = n;
    n = o.n;
    o.n = t;
    t = cap;
    cap = o.cap;
    o.cap = t;
    bool b = ok;
    ok = o.ok;
    o.ok = b;
  }
};

struct stream_batch_store {
  uint64_t seq = 0, k = 0, nh = 0;
  pinned_vec<tpx_stream_cluster> cl;
  pinned_vec<tpx_hit> hits;
  pinned_vec<uint64_t> g;
};

// Device state of one stream: the carry and the per-buffer scratch.
struct stream_dev {
  tpx_cluster* ctx = nullptr;
  cudaStream_t s = nullptr;
  uint64_t cap = 0, dt = 0;
  tpx_hit *d_hits = nullptr, *d_carry = nullptr;
  uint64_t *d_g = nullptr, *d_carry_g = nullptr;
  uint32_t *d_labels = nullptr, *d_order = nullptr, *d_offsets = nullptr, *d_cluster_of = nullptr;
  uint32_t *d_flag = nullptr, *d_size = nullptr, *d_cidx = nullptr, *d_hoff = nullptr, *d_open = nullptr,
           *d_cpos = nullptr, *d_counts = nullptr, *d_partials = nullptr;
  tpx_cluster_features* d_feats = nullptr;
  char* d_run_ws = nullptr;
  size_t run_ws_bytes = 0;
  uint64_t n_carry = 0;
  uint32_t* h_counts = nullptr;  // pinned [4]
};

struct stream_out {
  tpx_stream_cluster* cl;
  tpx_hit* hits;
  uint64_t* g;
  uint32_t* g32;
  uint64_t hoff_base;
};

// Shared scratch (bytes) of a stream_dev for `cap` device hits per buffer.
struct stream_dev_layout {
  size_t hits, g, carry, carry_g, labels, order, offsets, cluster_of, flag, size, cidx, hoff, open, cpos, counts,
      partials, feats, run_ws, total;
};

static size_t stream_dev_layout_of(uint64_t cap, size_t off, stream_dev_layout* L) {
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  L->hits = take(cap * 16);
  L->g = take(cap * 8);
  L->carry = take(cap * 16);
  L->carry_g = take(cap * 8);
  L->labels = take(cap * 4);
  L->order = take(cap * 4);
  L->offsets = take(cap * 4 + 4);
  L->cluster_of = take(cap * 4);
  L->flag = take(cap * 4);
  L->size = take(cap * 4);
  L->cidx = take(cap * 4);
  L->hoff = take(cap * 4);
  L->open = take(cap * 4);
  L->cpos = take(cap * 4);
  L->counts = take(64);
  L->partials = take((size_t)n_tiles_of(cap, kScanTile) * 4 + 64);
  L->feats = take(cap * 64);
  L->run_ws = off;
  off += align256(make_layout(cap).total);
  L->total = off;
  return off;
}

static void stream_dev_bind(stream_dev* d, char* w, const stream_dev_layout& L, size_t ws_end) {
  d->d_hits = (tpx_hit*)(w + L.hits);
  d->d_g = (uint64_t*)(w + L.g);
  d->d_carry = (tpx_hit*)(w + L.carry);
  d->d_carry_g = (uint64_t*)(w + L.carry_g);
  d->d_labels = (uint32_t*)(w + L.labels);
  d->d_order = (uint32_t*)(w + L.order);
  d->d_offsets = (uint32_t*)(w + L.offsets);
  d->d_cluster_of = (uint32_t*)(w + L.cluster_of);
  d->d_flag = (uint32_t*)(w + L.flag);
  d->d_size = (uint32_t*)(w + L.size);
  d->d_cidx = (uint32_t*)(w + L.cidx);
  d->d_hoff = (uint32_t*)(w + L.hoff);
  d->d_open = (uint32_t*)(w + L.open);
  d->d_cpos = (uint32_t*)(w + L.cpos);
  d->d_counts = (uint32_t*)(w + L.counts);
  d->d_partials = (uint32_t*)(w + L.partials);
  d->d_feats = (tpx_cluster_features*)(w + L.feats);
  d->d_run_ws = w + L.run_ws;
  d->run_ws_bytes = ws_end - L.run_ws;
}

// One buffer on the device: merge the carried hits with the nn fresh ones
// (device, arrival order), cluster + group, emit the closed clusters into
// `out`, keep the open ones' hits as the next carry.  Returns the emitted
// cluster and hit counts (one small read-back; all work on d->s).
static int stream_pass(stream_dev* d, const tpx_hit* fresh, const uint64_t* fresh_g, uint64_t nn, uint64_t cut,
                       bool final_buffer, const stream_out& out, uint64_t* kc_out, uint64_t* nh_out) {
  tpx_cluster* c = d->ctx;
  const uint64_t nc = d->n_carry;
  const uint64_t n = nn + nc;
  *kc_out = *nh_out = 0;
  if (n == 0) return TPX_OK;
  if (n > d->cap) return TPX_ERR_CAPACITY;
  cudaStream_t st = d->s;
  const tpx_hit* hits = fresh;
  const uint64_t* gidx = fresh_g;
  if (nc) {
    k_stream_merge<<<grid_for(n, 256), 256, 0, st>>>(d->d_carry, d->d_carry_g, (uint32_t)nc, fresh, fresh_g,
                                                      (uint32_t)nn, d->d_hits, d->d_g);
    TPX_LAUNCHED(c);
    hits = d->d_hits;
    gidx = d->d_g;
  }
  uint64_t k = 0;
  int rc = tpx_cluster_run_grouped(c, hits, n, d->d_labels, d->d_feats, nullptr, n, &k, d->d_order, d->d_offsets,
                                   d->d_cluster_of, d->d_run_ws, d->run_ws_bytes, st);
  if (rc) return rc;
  const int gk = grid_for(k, 256), gn = grid_for(n, 256);
  k_stream_blocks<<<gk, 256, 0, st>>>(d->d_cluster_of, d->d_feats, k, cut, d->dt, final_buffer ? 1 : 0, d->d_flag,
                                      d->d_size);
  TPX_LAUNCHED(c);
  if ((rc = exclusive_scan(c, d->d_flag, k, d->d_cidx, d->d_partials, d->d_counts + 0, st))) return rc;
  if ((rc = exclusive_scan(c, d->d_size, k, d->d_hoff, d->d_partials, d->d_counts + 1, st))) return rc;
  TPX_CUDA(cudaMemsetAsync(d->d_open, 0, n * 4, st));
  stream_emit_args a;
  a.hits = hits;
  a.gidx = gidx;
  a.order = d->d_order;
  a.offsets = d->d_offsets;
  a.cluster_of = d->d_cluster_of;
  a.feats = d->d_feats;
  a.closed_flag = d->d_flag;
  a.cidx = d->d_cidx;
  a.hoff = d->d_hoff;
  a.k = k;
  a.out_cl = out.cl;
  a.out_hits = out.hits;
  a.out_g = out.g;
  a.out_g32 = out.g32;
  a.hoff_base = out.hoff_base;
  a.open_flag = d->d_open;
  k_stream_emit_small<<<gk, 256, 0, st>>>(a);
  TPX_LAUNCHED(c);
  k_stream_emit_large<<<gk, 256, 0, st>>>(a);
  TPX_LAUNCHED(c);
  if ((rc = exclusive_scan(c, d->d_open, n, d->d_cpos, d->d_partials, d->d_counts + 2, st))) return rc;
  k_stream_carry<<<gn, 256, 0, st>>>(hits, gidx, n, d->d_open, d->d_cpos, d->d_carry, d->d_carry_g);
  TPX_LAUNCHED(c);
  TPX_CUDA(readback_async(d->h_counts, d->d_counts, 12, st));
  c->stats.kernel_launches++;
  TPX_CUDA(cudaStreamSynchronize(st));
  *kc_out = d->h_counts[0];
  *nh_out = d->h_counts[1];
  d->n_carry = d->h_counts[2];
  return TPX_OK;
}

}  // namespace tpx

struct tpx_stream {
  tpx_stream_config cfg;
  tpx::stream_dev dev;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  tpx::buffill_t<tpx::pinned_vec<tpx_hit>, tpx::pinned_vec<uint64_t>> bf;
  uint64_t arrivals = 0, last_cut = 0, seq = 0;
  bool have_cut = false, flushed = false;
  tpx_hit* d_new = nullptr;
  uint64_t* d_new_g = nullptr;
  tpx_hit* d_out_hits = nullptr;
  uint64_t* d_out_g = nullptr;
  tpx_stream_cluster* d_out_cl = nullptr;
  std::deque<tpx::stream_batch_store*> ready, pool;
  tpx::stream_batch_store* current = nullptr;  // last popped batch (valid until the next pop)
  tpx_stream_stats st;
};

namespace tpx {

struct stream_layout {
  size_t new_h, new_g, out_hits, out_g, out_cl, total;
  stream_dev_layout dev;
};

static int stream_layout_of(const tpx_stream_config* cfg, stream_layout* L) {
  const uint64_t cap = cfg->max_device_hits;
  const uint64_t fresh = cfg->buffer_hits + cfg->reserve_hits;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  L->new_h = take(fresh * 16);
  L->new_g = take(fresh * 8);
  L->out_hits = take(cap * 16);
  L->out_g = take(cap * 8);
  L->out_cl = take(cap * 80);
  L->total = stream_dev_layout_of(cap, off, &L->dev);
  return TPX_OK;
}

static void stream_release(tpx_stream* s, stream_batch_store* b) {
  if (b) s->pool.push_back(b);
}

// Cluster the current buffer (bf.buf + carried hits) with cut `cut`; queue a
// batch of the closed clusters; keep the open ones' hits on the device.
static int stream_process(tpx_stream* s, uint64_t cut, bool final_buffer) {
  const uint64_t nn = s->bf.buf.size();
  if (nn + s->dev.n_carry == 0) return TPX_OK;
  if (nn > s->cfg.buffer_hits + s->cfg.reserve_hits) return TPX_ERR_CAPACITY;
  if (!s->bf.buf.ok || !s->bf.buf_g.ok) return TPX_ERR_OOM;
  cudaStream_t st = s->dev.s;
  TPX_CUDA(cudaEventRecord(s->ev0, st));
  if (nn) {
    TPX_CUDA(cudaMemcpyAsync(s->d_new, s->bf.buf.p, nn * 16, cudaMemcpyHostToDevice, st));
    TPX_CUDA(cudaMemcpyAsync(s->d_new_g, s->bf.buf_g.p, nn * 8, cudaMemcpyHostToDevice, st));
  }
  stream_out out{s->d_out_cl, s->d_out_hits, s->d_out_g, nullptr, 0};
  uint64_t kc = 0, nh = 0;
  int rc = stream_pass(&s->dev, s->d_new, s->d_new_g, nn, cut, final_buffer, out, &kc, &nh);
  if (rc) return rc;
  // batch of closed clusters (pinned, from the pool)
  stream_batch_store* b = nullptr;
  if (!s->pool.empty()) {
    b = s->pool.front();
    s->pool.pop_front();
  } else {
    b = new (std::nothrow) stream_batch_store;
    if (!b) return TPX_ERR_OOM;
  }
  if (!b->cl.reserve(kc ? kc : 1) || !b->hits.reserve(nh ? nh : 1) || !b->g.reserve(nh ? nh : 1)) {
    stream_release(s, b);
    return TPX_ERR_OOM;
  }
  if (kc) TPX_CUDA(cudaMemcpyAsync(b->cl.p, s->d_out_cl, kc * 80, cudaMemcpyDeviceToHost, st));
  if (nh) {
    TPX_CUDA(cudaMemcpyAsync(b->hits.p, s->d_out_hits, nh * 16, cudaMemcpyDeviceToHost, st));
    TPX_CUDA(cudaMemcpyAsync(b->g.p, s->d_out_g, nh * 8, cudaMemcpyDeviceToHost, st));
  }
  TPX_CUDA(cudaEventRecord(s->ev1, st));
  TPX_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, s->ev0, s->ev1);
  b->seq = s->seq++;
  b->k = kc;
  b->nh = nh;
  b->cl.n = kc;
  b->hits.n = nh;
  b->g.n = nh;
  s->ready.push_back(b);
  s->st.buffers++;
  s->st.clusters_out += kc;
  s->st.hits_out += nh;
  s->st.carried_last = s->dev.n_carry;
  if (s->dev.n_carry > s->st.carried_max) s->st.carried_max = s->dev.n_carry;
  s->st.device_ms += ms;
  return TPX_OK;
}

}  // namespace tpx

extern "C" {

int tpx_stream_workspace_bytes(const tpx_stream_config* cfg, size_t* bytes) {
  if (!cfg || !bytes) return TPX_ERR_INVALID_ARG;
  if (cfg->buffer_hits <= cfg->reserve_hits || cfg->max_device_hits < cfg->buffer_hits + cfg->reserve_hits ||
      cfg->max_device_hits >= 0xffffffffull)
    return TPX_ERR_INVALID_ARG;
  tpx::stream_layout L;
  tpx::stream_layout_of(cfg, &L);
  *bytes = L.total;
  return TPX_OK;
}

void tpx_stream_destroy(tpx_stream* s) {
  if (!s) return;
  if (s->dev.s) cudaStreamSynchronize(s->dev.s);
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev1) cudaEventDestroy(s->ev1);
  if (s->dev.h_counts) cudaFreeHost(s->dev.h_counts);
  for (auto* b : s->ready) delete b;
  for (auto* b : s->pool) delete b;
  delete s->current;
  tpx_cluster_destroy(s->dev.ctx);
  delete s;
}

int tpx_stream_create(const tpx_stream_config* cfg, void* workspace, size_t workspace_bytes, void* cuda_stream,
                      tpx_stream** out) {
  if (!out || !cfg || !workspace || ((uintptr_t)workspace & 255)) return TPX_ERR_INVALID_ARG;
  *out = nullptr;
  size_t need = 0;
  int rc = tpx_stream_workspace_bytes(cfg, &need);
  if (rc) return rc;
  if (workspace_bytes < need) return TPX_ERR_OOM;
  tpx_stream* s = new (std::nothrow) tpx_stream;
  if (!s) return TPX_ERR_OOM;
  memset(&s->st, 0, sizeof(s->st));
  s->cfg = *cfg;
  rc = tpx_cluster_create(cfg->dt_max_ticks, TPX_VARIANT_LOCAL, cfg->width, cfg->height, &s->dev.ctx);
  if (rc) {
    delete s;
    return rc;
  }
  s->dev.s = (cudaStream_t)cuda_stream;
  s->dev.cap = cfg->max_device_hits;
  s->dev.dt = cfg->dt_max_ticks;
  s->bf.b = cfg->buffer_hits;
  s->bf.b_t = cfg->reserve_hits;
  s->bf.t = cfg->disorder_ticks;
  s->bf.t_closing = cfg->closing_ticks;
  tpx::stream_layout L;
  tpx::stream_layout_of(cfg, &L);
  char* w = (char*)workspace;
  s->d_new = (tpx_hit*)(w + L.new_h);
  s->d_new_g = (uint64_t*)(w + L.new_g);
  s->d_out_hits = (tpx_hit*)(w + L.out_hits);
  s->d_out_g = (uint64_t*)(w + L.out_g);
  s->d_out_cl = (tpx_stream_cluster*)(w + L.out_cl);
  tpx::stream_dev_bind(&s->dev, w, L.dev, workspace_bytes);
  if (cudaEventCreate(&s->ev0) != cudaSuccess || cudaEventCreate(&s->ev1) != cudaSuccess ||
      cudaHostAlloc((void**)&s->dev.h_counts, 64, cudaHostAllocMapped) != cudaSuccess || !s->bf.buf.reserve(1024) || !s->bf.next.reserve(1024) ||
      !s->bf.buf_g.reserve(1024) || !s->bf.next_g.reserve(1024)) {
    tpx_stream_destroy(s);
    return TPX_ERR_CUDA;
  }
  *out = s;
  return TPX_OK;
}

int tpx_stream_push(tpx_stream* s, const tpx_hit* hits, uint64_t n) {
  if (!s || (n && !hits) || s->flushed) return TPX_ERR_INVALID_ARG;
  for (uint64_t i = 0; i < n; ++i) {
    const tpx_hit& h = hits[i];
    if (s->have_cut && h.toa < s->last_cut) s->st.late_hits++;  // stream not t-ordered
    uint64_t cut = 0;
    const bool send = s->bf.store(h, s->arrivals++, &cut);
    if (!s->bf.buf.ok || !s->bf.next.ok || !s->bf.buf_g.ok || !s->bf.next_g.ok) return TPX_ERR_OOM;
    if (send) {
      const int rc = tpx::stream_process(s, cut, false);
      if (rc) return rc;
      s->last_cut = cut;
      s->have_cut = true;
      s->bf.rotate();
    }
  }
  s->st.hits_in += n;
  return TPX_OK;
}

int tpx_stream_flush(tpx_stream* s) {
  if (!s) return TPX_ERR_INVALID_ARG;
  if (s->flushed) return TPX_OK;
  int rc;
  if (s->bf.next.size()) {  // reading R20: the open buffer first, with its cut
    const uint64_t cut = s->bf.toa_max + s->bf.t_closing;
    if ((rc = tpx::stream_process(s, cut, false))) return rc;
    s->bf.rotate();
  }
  if ((rc = tpx::stream_process(s, ~0ull, true))) return rc;
  s->bf.buf.clear();
  s->bf.buf_g.clear();
  s->flushed = true;
  return TPX_OK;
}

int tpx_stream_pop(tpx_stream* s, tpx_stream_batch* out) {
  if (!s || !out) return TPX_ERR_INVALID_ARG;
  memset(out, 0, sizeof(*out));
  tpx::stream_release(s, s->current);
  s->current = nullptr;
  if (s->ready.empty()) return 0;
  tpx::stream_batch_store* b = s->ready.front();
  s->ready.pop_front();
  s->current = b;
  out->seq = b->seq;
  out->n_clusters = b->k;
  out->n_hits = b->nh;
  out->clusters = b->cl.p;
  out->hits = b->hits.p;
  out->hit_index = b->g.p;
  return 1;
}

int tpx_stream_get_stats(const tpx_stream* s, tpx_stream_stats* out) {
  if (!s || !out) return TPX_ERR_INVALID_ARG;
  *out = s->st;
  out->carried_last = s->dev.n_carry;
  return TPX_OK;
}

int tpx_buffill_assign(const tpx_hit* hits, uint64_t n, uint64_t b, uint64_t b_t, uint64_t t, uint64_t t_closing,
                       uint32_t* buffer_id_out, uint64_t* cuts_out, uint64_t cuts_cap, uint64_t* n_buffers_out) {
  if ((n && (!hits || !buffer_id_out)) || !n_buffers_out || b <= b_t) return TPX_ERR_INVALID_ARG;
  tpx::buffill f;
  f.b = b;
  f.b_t = b_t;
  f.t = t;
  f.t_closing = t_closing;
  uint64_t nb = 0;
  // hits are identified by their arrival index (stored in the g-vectors)
  auto send = [&](uint64_t cut) {
    for (uint64_t g : f.buf_g) buffer_id_out[g] = (uint32_t)nb;
    if (nb < cuts_cap && cuts_out) cuts_out[nb] = cut;
    ++nb;
  };
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t cut = 0;
    if (f.store(hits[i], i, &cut)) {
      send(cut);
      f.rotate();
    }
  }
  if (!f.next.empty()) {
    send(f.toa_max + f.t_closing);
    f.rotate();
  }
  if (!f.buf.empty()) send(~0ull);
  *n_buffers_out = nb;
  return nb > cuts_cap && cuts_out ? TPX_ERR_CAPACITY : TPX_OK;
}

}  // extern "C"

#include "stream_host.cuh"
