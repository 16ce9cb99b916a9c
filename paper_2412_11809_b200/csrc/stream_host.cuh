// stream_host.cuh -- one-shot host-to-host streaming run (included by
// stream.cuh).
//
// The paper's GPU benchmark (§5 l.278-280): "The clock starts once
// the host buffer is populated with data and ends after the clustered data is
// transferred back to the host."  tpx_stream_run_host takes a whole stream in
// host memory and runs Alg. "Hit buffer filling" over it without copying on
// the host: a buffer = [hits moved from the previous nextBuffer | a run of
// consecutive input hits (the phase where every hit joins) | hits routed in
// by the toa_max + t_closing test], and the run goes to the device straight
// from the caller's memory.  Copies overlap compute (l.310): buffer k+1's run
// is in flight on the H2D stream while buffer k is clustered, and buffer k's
// results drain on the D2H stream while buffer k+1 is clustered.  Results are
// those of tpx_stream_push/flush (same BufFill decisions, same carry).
#pragma once
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace tpx {

struct run_host_layout {
  size_t new_h[2], new_g[2], out_cl[2], out_g32[2], scan[2], total;
  stream_dev_layout dev;
};

static void run_host_layout_of(const tpx_stream_config* cfg, run_host_layout* L) {
  const uint64_t cap = cfg->max_device_hits;
  const uint64_t fresh = cfg->buffer_hits + cfg->reserve_hits;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  for (int i = 0; i < 2; ++i) {
    L->new_h[i] = take(fresh * 16);
    L->new_g[i] = take(fresh * 8);
    L->out_cl[i] = take(cap * 80);
    L->out_g32[i] = take(cap * 4);
    L->scan[i] = take(64);
  }
  L->total = stream_dev_layout_of(cap, off, &L->dev);
}

// Largest ToA of a run (BufFill's toa_max over its phase-1 hits) and the
// number of hits with toa < last_cut (t-orderedness violations), computed on
// the device right after the run's H2D (out[0] = max, out[1] = late; zeroed
// by the caller).
__global__ void k_run_scan(const tpx_hit* __restrict__ h, uint64_t n, uint64_t last_cut, int have_cut,
                           unsigned long long* __restrict__ out) {
  unsigned long long mx = 0, late = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long t = __ldg(reinterpret_cast<const unsigned long long*>(h + i));
    mx = t > mx ? t : mx;
    late += (have_cut && t < last_cut) ? 1ull : 0ull;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    late += __shfl_xor_sync(kFull, late, o);
  }
  if (lane_id() == 0) {
    atomicMax(out, mx);
    if (late) atomicAdd(out + 1, late);
  }
}

// One buffer's plan: [moved (m0) | run [run_a, run_b) | extras], its cut.
struct buf_plan {
  int slot = 0;
  uint64_t m0 = 0, run_a = 0, run_b = 0, n_extra = 0;
  uint64_t cut = ~0ull;
  bool final_buffer = false;
  uint64_t resume = 0;  // first input position after this buffer's routing
};

}  // namespace tpx

extern "C" {

int tpx_stream_run_host_workspace_bytes(const tpx_stream_config* cfg, size_t* bytes) {
  if (!cfg || !bytes) return TPX_ERR_INVALID_ARG;
  size_t dummy = 0;
  int rc = tpx_stream_workspace_bytes(cfg, &dummy);  // same argument checks
  if (rc) return rc;
  tpx::run_host_layout L;
  tpx::run_host_layout_of(cfg, &L);
  *bytes = L.total;
  return TPX_OK;
}

int tpx_stream_run_host(const tpx_stream_config* cfg, const tpx_hit* hits, uint64_t n, uint32_t* order_out,
                        tpx_stream_cluster* clusters_out, uint64_t capacity, uint64_t* n_clusters_out,
                        void* workspace, size_t workspace_bytes, void* cuda_stream, tpx_stream_stats* stats_out) {
  using namespace tpx;
  if (!cfg || !n_clusters_out || !workspace || ((uintptr_t)workspace & 255)) return TPX_ERR_INVALID_ARG;
  *n_clusters_out = 0;
  if (n >= 0xffffffffull) return TPX_ERR_TOO_MANY_HITS;
  if (n && (!hits || !order_out || (!clusters_out && capacity))) return TPX_ERR_INVALID_ARG;
  size_t need = 0;
  int rc = tpx_stream_run_host_workspace_bytes(cfg, &need);
  if (rc) return rc;
  if (workspace_bytes < need) return TPX_ERR_OOM;
  tpx_stream_stats st;
  memset(&st, 0, sizeof(st));
  if (n == 0) {
    if (stats_out) *stats_out = st;
    return TPX_OK;
  }
  run_host_layout L;
  run_host_layout_of(cfg, &L);
  char* w = (char*)workspace;
  stream_dev d;
  if ((rc = tpx_cluster_create(cfg->dt_max_ticks, TPX_VARIANT_LOCAL, cfg->width, cfg->height, &d.ctx))) return rc;
  d.s = (cudaStream_t)cuda_stream;
  d.cap = cfg->max_device_hits;
  d.dt = cfg->dt_max_ticks;
  stream_dev_bind(&d, w, L.dev, workspace_bytes);
  tpx_hit* d_new[2] = {(tpx_hit*)(w + L.new_h[0]), (tpx_hit*)(w + L.new_h[1])};
  uint64_t* d_new_g[2] = {(uint64_t*)(w + L.new_g[0]), (uint64_t*)(w + L.new_g[1])};
  tpx_stream_cluster* d_out_cl[2] = {(tpx_stream_cluster*)(w + L.out_cl[0]), (tpx_stream_cluster*)(w + L.out_cl[1])};
  uint32_t* d_out_g32[2] = {(uint32_t*)(w + L.out_g32[0]), (uint32_t*)(w + L.out_g32[1])};

  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t e_in[2] = {nullptr, nullptr}, e_out[2] = {nullptr, nullptr}, e_scan[2] = {nullptr, nullptr},
              e_done = nullptr, t0 = nullptr, t1 = nullptr;
  unsigned long long* d_scan[2] = {(unsigned long long*)(w + L.scan[0]), (unsigned long long*)(w + L.scan[1])};
  unsigned long long* h_scan = nullptr;  // pinned [2 slots][2]
  pinned_vec<tpx_hit> moved_h[2], extra_h[2];
  pinned_vec<uint64_t> moved_g[2], extra_g[2];
  const uint64_t b = cfg->buffer_hits, b_t = cfg->reserve_hits, fresh = b + b_t;
  const uint64_t t_dis = cfg->disorder_ticks, t_cl = cfg->closing_ticks;
  uint64_t toa_max = 0, last_cut = 0, k_total = 0, h_total = 0;
  bool have_cut = false;
  auto cleanup = [&]() {
    if (d.s) cudaStreamSynchronize(d.s);
    if (s_h2d) {
      cudaStreamSynchronize(s_h2d);
      cudaStreamDestroy(s_h2d);
    }
    if (s_d2h) {
      cudaStreamSynchronize(s_d2h);
      cudaStreamDestroy(s_d2h);
    }
    for (int i = 0; i < 2; ++i) {
      if (e_in[i]) cudaEventDestroy(e_in[i]);
      if (e_out[i]) cudaEventDestroy(e_out[i]);
      if (e_scan[i]) cudaEventDestroy(e_scan[i]);
    }
    if (h_scan) cudaFreeHost(h_scan);
    if (e_done) cudaEventDestroy(e_done);
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
    if (d.h_counts) cudaFreeHost(d.h_counts);
    tpx_cluster_destroy(d.ctx);
  };
#define TPX_RH(call)            \
  do {                          \
    if ((call) != cudaSuccess) { \
      cleanup();                \
      return TPX_ERR_CUDA;      \
    }                           \
  } while (0)
  TPX_RH(cudaStreamCreateWithFlags(&s_h2d, cudaStreamNonBlocking));
  TPX_RH(cudaStreamCreateWithFlags(&s_d2h, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    TPX_RH(cudaEventCreateWithFlags(&e_in[i], cudaEventDisableTiming));
    TPX_RH(cudaEventCreateWithFlags(&e_out[i], cudaEventDisableTiming));
    TPX_RH(cudaEventCreateWithFlags(&e_scan[i], cudaEventDisableTiming));
    if (!moved_h[i].reserve(1024) || !moved_g[i].reserve(1024) || !extra_h[i].reserve(1024) ||
        !extra_g[i].reserve(1024)) {
      cleanup();
      return TPX_ERR_OOM;
    }
  }
  TPX_RH(cudaEventCreateWithFlags(&e_done, cudaEventDisableTiming));
  TPX_RH(cudaEventCreate(&t0));
  TPX_RH(cudaEventCreate(&t1));
  TPX_RH(cudaHostAlloc((void**)&d.h_counts, 64, cudaHostAllocMapped));
  TPX_RH(cudaHostAlloc((void**)&h_scan, 64, cudaHostAllocMapped));
  TPX_RH(cudaEventRecord(t0, d.s));

  // issue the H2D of a plan's moved hits and run (the run straight from the
  // caller's memory), arrival indices of the run by a device iota
  auto issue_run = [&](const buf_plan& p, uint64_t cut_before, bool have) -> int {
    const int sl = p.slot;
    if (cudaMemsetAsync(d_scan[sl], 0, 16, s_h2d) != cudaSuccess) return TPX_ERR_CUDA;
    if (p.m0) {
      if (cudaMemcpyAsync(d_new[sl], moved_h[sl].p, p.m0 * 16, cudaMemcpyHostToDevice, s_h2d) != cudaSuccess ||
          cudaMemcpyAsync(d_new_g[sl], moved_g[sl].p, p.m0 * 8, cudaMemcpyHostToDevice, s_h2d) != cudaSuccess)
        return TPX_ERR_CUDA;
    }
    const uint64_t rl = p.run_b - p.run_a;
    if (rl) {
      if (cudaMemcpyAsync(d_new[sl] + p.m0, hits + p.run_a, rl * 16, cudaMemcpyHostToDevice, s_h2d) != cudaSuccess)
        return TPX_ERR_CUDA;
      k_iota64<<<grid_for(rl, 256), 256, 0, s_h2d>>>(d_new_g[sl] + p.m0, rl, p.run_a);
      k_run_scan<<<grid_for(rl, 256), 256, 0, s_h2d>>>(d_new[sl] + p.m0, rl, cut_before, have ? 1 : 0, d_scan[sl]);
      if (cudaGetLastError() != cudaSuccess) return TPX_ERR_CUDA;
    }
    if (readback_async(h_scan + 2 * sl, d_scan[sl], 16, s_h2d) != cudaSuccess ||
        cudaEventRecord(e_scan[sl], s_h2d) != cudaSuccess)
      return TPX_ERR_CUDA;
    return TPX_OK;
  };
  // toa_max over the run's hits (BufFill phase 1) and its late hits
  auto take_scan = [&](int sl) -> int {
    if (cudaEventSynchronize(e_scan[sl]) != cudaSuccess) return TPX_ERR_CUDA;
    toa_max = std::max<uint64_t>(toa_max, h_scan[2 * sl]);
    st.late_hits += h_scan[2 * sl + 1];
    return TPX_OK;
  };
  // phase 2 of BufFill after the run: route hits into extras (this buffer) or
  // moved[other slot] (the next buffer) until a hit sends the buffer
  auto route = [&](buf_plan& p) -> int {
    const int sl = p.slot, ns = sl ^ 1;
    extra_h[sl].clear();
    extra_g[sl].clear();
    moved_h[ns].clear();
    moved_g[ns].clear();
    uint64_t q = p.run_b;
    bool sent = false;
    for (; q < n; ++q) {
      const tpx_hit& h = hits[q];
      if (have_cut && h.toa < last_cut) st.late_hits++;
      if (h.toa < toa_max + t_cl) {
        extra_h[sl].push_back(h);
        extra_g[sl].push_back(q);
      } else {
        moved_h[ns].push_back(h);
        moved_g[ns].push_back(q);
      }
      if (h.toa > toa_max + t_dis + t_cl) {
        sent = true;
        ++q;
        break;
      }
    }
    if (!extra_h[sl].ok || !extra_g[sl].ok || !moved_h[ns].ok || !moved_g[ns].ok) return TPX_ERR_OOM;
    p.n_extra = extra_h[sl].size();
    p.resume = q;
    if (sent) {
      p.cut = toa_max + t_cl;
      p.final_buffer = false;
    } else if (moved_h[ns].size()) {  // end of stream, nextBuffer non-empty (R20)
      p.cut = toa_max + t_cl;
      p.final_buffer = false;
    } else {
      p.cut = ~0ull;
      p.final_buffer = true;
    }
    if (p.m0 + (p.run_b - p.run_a) + p.n_extra > fresh) return TPX_ERR_CAPACITY;
    if (p.n_extra) {
      const uint64_t o = p.m0 + (p.run_b - p.run_a);
      if (cudaMemcpyAsync(d_new[sl] + o, extra_h[sl].p, p.n_extra * 16, cudaMemcpyHostToDevice, s_h2d) !=
              cudaSuccess ||
          cudaMemcpyAsync(d_new_g[sl] + o, extra_g[sl].p, p.n_extra * 8, cudaMemcpyHostToDevice, s_h2d) !=
              cudaSuccess)
        return TPX_ERR_CUDA;
    }
    if (cudaEventRecord(e_in[sl], s_h2d) != cudaSuccess) return TPX_ERR_CUDA;
    return TPX_OK;
  };
  auto plan_after = [&](const buf_plan& p) {
    buf_plan x;
    x.slot = p.slot ^ 1;
    x.m0 = moved_h[x.slot].size();
    x.run_a = p.resume;
    const uint64_t room = x.m0 < b - b_t ? (b - b_t) - x.m0 : 0;  // phase 1: buffer below b - b_t
    x.run_b = std::min<uint64_t>(n, x.run_a + room);
    return x;
  };

  buf_plan cur;
  cur.slot = 0;
  cur.run_a = 0;
  cur.run_b = std::min<uint64_t>(n, b - b_t);
  if ((rc = issue_run(cur, 0, false)) || (rc = take_scan(cur.slot)) || (rc = route(cur))) {
    cleanup();
    return rc;
  }
  bool use_prev_out[2] = {false, false};
  const bool trace = getenv("TPX_STREAM_TRACE") != nullptr;
  double tr[5] = {0, 0, 0, 0, 0};  // issue_run, stream_pass, d2h issue, take_scan, route
  auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double ta = now();
  for (;;) {
    const int sl = cur.slot;
    // the next buffer's run goes out now (overlaps this buffer's kernels),
    // its toa_max scan runs on the device right behind it
    buf_plan nxt;
    const bool more = !cur.final_buffer;
    if (more) {
      nxt = plan_after(cur);
      if ((rc = issue_run(nxt, cur.cut, true))) break;
    }
    if (trace) { double tb = now(); tr[0] += tb - ta; ta = tb; }
    // cluster this buffer
    if (cudaStreamWaitEvent(d.s, e_in[sl], 0) != cudaSuccess) {
      rc = TPX_ERR_CUDA;
      break;
    }
    if (use_prev_out[sl] && cudaStreamWaitEvent(d.s, e_out[sl], 0) != cudaSuccess) {
      rc = TPX_ERR_CUDA;
      break;
    }
    const uint64_t nn = cur.m0 + (cur.run_b - cur.run_a) + cur.n_extra;
    stream_out out{d_out_cl[sl], nullptr, nullptr, d_out_g32[sl], h_total};
    uint64_t kc = 0, nh = 0;
    if ((rc = stream_pass(&d, d_new[sl], d_new_g[sl], nn, cur.cut, cur.final_buffer, out, &kc, &nh))) break;
    if (trace) { double tb = now(); tr[1] += tb - ta; ta = tb; }
    // drain the results on the D2H stream
    if (cudaEventRecord(e_done, d.s) != cudaSuccess || cudaStreamWaitEvent(s_d2h, e_done, 0) != cudaSuccess) {
      rc = TPX_ERR_CUDA;
      break;
    }
    const uint64_t kfit = k_total >= capacity ? 0 : std::min<uint64_t>(kc, capacity - k_total);
    if (kfit && cudaMemcpyAsync(clusters_out + k_total, d_out_cl[sl], kfit * 80, cudaMemcpyDeviceToHost, s_d2h) !=
                    cudaSuccess) {
      rc = TPX_ERR_CUDA;
      break;
    }
    if (nh && cudaMemcpyAsync(order_out + h_total, d_out_g32[sl], nh * 4, cudaMemcpyDeviceToHost, s_d2h) !=
                  cudaSuccess) {
      rc = TPX_ERR_CUDA;
      break;
    }
    if (cudaEventRecord(e_out[sl], s_d2h) != cudaSuccess) {
      rc = TPX_ERR_CUDA;
      break;
    }
    use_prev_out[sl] = true;
    if (trace) { double tb = now(); tr[2] += tb - ta; ta = tb; }
    k_total += kc;
    h_total += nh;
    st.buffers++;
    st.carried_last = d.n_carry;
    st.carried_max = std::max(st.carried_max, d.n_carry);
    if (!more) break;
    last_cut = cur.cut;
    have_cut = true;
    if ((rc = take_scan(nxt.slot))) break;
    if (trace) { double tb = now(); tr[3] += tb - ta; ta = tb; }
    cur = nxt;
    if ((rc = route(cur))) break;
    if (trace) { double tb = now(); tr[4] += tb - ta; ta = tb; }
  }
  if (trace)
    fprintf(stderr, "stream trace (ms): issue_run %.2f stream_pass %.2f d2h_issue %.2f take_scan %.2f route %.2f buffers %llu\n",
            tr[0], tr[1], tr[2], tr[3], tr[4], (unsigned long long)st.buffers);
#undef TPX_RH
  if (rc == TPX_OK) {
    if (cudaEventRecord(t1, s_d2h) != cudaSuccess || cudaEventSynchronize(t1) != cudaSuccess) rc = TPX_ERR_CUDA;
    float ms = 0.f;
    if (rc == TPX_OK && cudaEventElapsedTime(&ms, t0, t1) == cudaSuccess) st.device_ms = ms;
  }
  cleanup();
  st.hits_in = n;
  st.hits_out = h_total;
  st.clusters_out = k_total;
  if (stats_out) *stats_out = st;
  *n_clusters_out = k_total;
  if (rc) return rc;
  if (h_total != n) return TPX_ERR_CAPACITY;  // cannot happen for a complete stream
  return k_total > capacity ? TPX_ERR_CAPACITY : TPX_OK;
}

}  // extern "C"
