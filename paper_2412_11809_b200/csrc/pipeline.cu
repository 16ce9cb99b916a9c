// pipeline.cu -- host-buffer pipeline: copy/compute overlap across buffers.
//
// The paper's GPU driver (Alg. "High-level GPU clustering", PAPER.md
// l.160-182) fills a host buffer (Step 1), copies it to the device (Step 2),
// clusters it (Steps 3-7), copies the result back (Step 8) and recycles the
// buffer (Step 9, "in use" / "reusable" l.164, l.180); "overlapping copy and
// compute using CUDA streams hid the latency of data copying" (l.310).  Here
// `depth` slots each own a context, a CUDA stream and a slice of a
// caller-provided device workspace; a native worker thread per slot runs
// [H2D -> tpx_cluster_run -> D2H] for the buffers assigned to it, so the
// copies of one buffer overlap the kernels of another.  Buffers are
// independent closed streams (reading R14).
//
// The copies of all slots go through two pipeline-wide streams (one per
// direction, FIFO in submission order) and the kernels through the slot's
// own stream, joined by events.  With a copy stream per slot the copy
// engine interleaved the H2D of every buffer in flight, so all of them
// finished late and the slots fell into lock step (H2D together, then D2H
// together: little duplex overlap).  FIFO copies finish one buffer's H2D at
// full bandwidth while the previous buffer's labels and records go back in
// the other direction, so the steady state is max(H2D, kernels, D2H) per
// buffer instead of roughly their sum.
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "tpx_cluster.h"

namespace {

struct job {
  const tpx_hit* hits;
  uint64_t n;
  uint32_t* labels;
  tpx_cluster_features* feats;
  uint64_t capacity;
  uint64_t n_clusters = 0;
  int status = TPX_OK;
  bool done = false;
};

struct slot {
  tpx_cluster* ctx = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t t_start = nullptr, t_stop = nullptr;
  cudaEvent_t ev_in = nullptr, ev_run = nullptr, ev_out = nullptr;  // H2D done, kernels done, D2H done
  char* ws = nullptr;
  size_t ws_bytes = 0;
  std::thread th;
  std::deque<job*> q;
};

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

}  // namespace

struct tpx_pipeline {
  int device = 0;
  uint64_t max_hits = 0, capacity = 0;
  std::vector<slot> slots;
  cudaStream_t h2d = nullptr, d2h = nullptr;  // pipeline-wide copy streams (FIFO per direction)
  cudaEvent_t c_start[2] = {nullptr, nullptr}, c_stop[2] = {nullptr, nullptr};
  std::mutex m;
  std::condition_variable cv_work, cv_done;
  std::map<uint64_t, job*> jobs;
  uint64_t next_ticket = 0;
  bool stop = false;
};

// tpx_cluster_run_host with the copies on the pipeline's copy streams (same
// workspace layout: hits, labels, records, then the run's own workspace).
static int run_job(tpx_pipeline* p, slot& s, job* j, uint64_t* k_out) {
  *k_out = 0;
  const uint64_t n = j->n;
  if (n >= 0xffffffffull) return TPX_ERR_TOO_MANY_HITS;
  if (n == 0) return TPX_OK;
  if (!j->hits || !j->labels || (!j->feats && j->capacity)) return TPX_ERR_INVALID_ARG;
  size_t need = 0;
  tpx_cluster_host_workspace_bytes(s.ctx, n, j->capacity, &need);
  if (s.ws_bytes < need) return TPX_ERR_OOM;
  char* ws = s.ws;
  tpx_hit* d_hits = (tpx_hit*)ws;
  uint32_t* d_labels = (uint32_t*)(ws + align256(n * 16));
  tpx_cluster_features* d_feats = (tpx_cluster_features*)(ws + align256(n * 16) + align256(n * 4));
  char* inner = ws + align256(n * 16) + align256(n * 4) + align256(j->capacity * 64);
  const size_t inner_bytes = s.ws_bytes - (size_t)(inner - ws);
  if (cudaMemcpyAsync(d_hits, j->hits, n * 16, cudaMemcpyHostToDevice, p->h2d) != cudaSuccess ||
      cudaEventRecord(s.ev_in, p->h2d) != cudaSuccess || cudaStreamWaitEvent(s.stream, s.ev_in, 0) != cudaSuccess)
    return TPX_ERR_CUDA;
  uint64_t k = 0;
  const int rc = tpx_cluster_run(s.ctx, d_hits, n, d_labels, d_feats, j->capacity, &k, inner, inner_bytes, s.stream);
  if (rc != TPX_OK && rc != TPX_ERR_CAPACITY) return rc;
  *k_out = k;
  const uint64_t kk = k < j->capacity ? k : j->capacity;
  if (cudaEventRecord(s.ev_run, s.stream) != cudaSuccess || cudaStreamWaitEvent(p->d2h, s.ev_run, 0) != cudaSuccess ||
      cudaMemcpyAsync(j->labels, d_labels, n * 4, cudaMemcpyDeviceToHost, p->d2h) != cudaSuccess ||
      (kk && cudaMemcpyAsync(j->feats, d_feats, kk * 64, cudaMemcpyDeviceToHost, p->d2h) != cudaSuccess) ||
      cudaEventRecord(s.ev_out, p->d2h) != cudaSuccess || cudaEventSynchronize(s.ev_out) != cudaSuccess)
    return TPX_ERR_CUDA;
  return rc;
}

static void worker(tpx_pipeline* p, size_t si) {
  cudaSetDevice(p->device);
  slot& s = p->slots[si];
  for (;;) {
    job* j = nullptr;
    {
      std::unique_lock<std::mutex> lk(p->m);
      p->cv_work.wait(lk, [&] { return p->stop || !s.q.empty(); });
      if (s.q.empty()) return;  // stop requested and nothing left
      j = s.q.front();
      s.q.pop_front();
    }
    uint64_t k = 0;
    const int rc = run_job(p, s, j, &k);
    {
      std::lock_guard<std::mutex> lk(p->m);
      j->status = rc;
      j->n_clusters = k;
      j->done = true;
    }
    p->cv_done.notify_all();
  }
}

extern "C" {

int tpx_pipeline_workspace_bytes(const tpx_cluster* proto, uint64_t max_hits, uint64_t capacity, int depth,
                                 size_t* bytes) {
  if (!proto || !bytes || depth < 1 || depth > 16) return TPX_ERR_INVALID_ARG;
  size_t one = 0;
  const int rc = tpx_cluster_host_workspace_bytes(proto, max_hits, capacity, &one);
  if (rc) return rc;
  *bytes = align256(one) * (size_t)depth;
  return TPX_OK;
}

int tpx_pipeline_create(uint64_t dt_max_ticks, int variant, uint32_t width, uint32_t height, uint64_t max_hits,
                        uint64_t capacity, int depth, void* workspace, size_t workspace_bytes, tpx_pipeline** out) {
  if (!out || depth < 1 || depth > 16 || !workspace || ((uintptr_t)workspace & 255)) return TPX_ERR_INVALID_ARG;
  *out = nullptr;
  tpx_pipeline* p = new (std::nothrow) tpx_pipeline;
  if (!p) return TPX_ERR_OOM;
  p->max_hits = max_hits;
  p->capacity = capacity;
  if (cudaGetDevice(&p->device) != cudaSuccess) {
    delete p;
    return TPX_ERR_CUDA;
  }
  p->slots.resize((size_t)depth);
  size_t one = 0;
  int rc = TPX_OK;
  for (int i = 0; i < depth && rc == TPX_OK; ++i) {
    slot& s = p->slots[(size_t)i];
    rc = tpx_cluster_create(dt_max_ticks, variant, width, height, &s.ctx);
    if (rc) break;
    rc = tpx_cluster_host_workspace_bytes(s.ctx, max_hits, capacity, &one);
    if (rc) break;
    one = align256(one);
    if (workspace_bytes < one * (size_t)depth) {
      rc = TPX_ERR_OOM;
      break;
    }
    s.ws = (char*)workspace + one * (size_t)i;
    s.ws_bytes = one;
    if (cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&s.t_start) != cudaSuccess || cudaEventCreate(&s.t_stop) != cudaSuccess ||
        cudaEventCreateWithFlags(&s.ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s.ev_run, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s.ev_out, cudaEventDisableTiming | cudaEventBlockingSync) != cudaSuccess)
      rc = TPX_ERR_CUDA;
  }
  if (rc == TPX_OK &&
      (cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking) != cudaSuccess ||
       cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking) != cudaSuccess))
    rc = TPX_ERR_CUDA;
  for (int i = 0; i < 2 && rc == TPX_OK; ++i)
    if (cudaEventCreate(&p->c_start[i]) != cudaSuccess || cudaEventCreate(&p->c_stop[i]) != cudaSuccess)
      rc = TPX_ERR_CUDA;
  if (rc) {
    tpx_pipeline_destroy(p);
    return rc;
  }
  for (size_t i = 0; i < p->slots.size(); ++i) p->slots[i].th = std::thread(worker, p, i);
  *out = p;
  return TPX_OK;
}

int tpx_pipeline_submit(tpx_pipeline* p, const tpx_hit* hits_host, uint64_t n, uint32_t* labels_host,
                        tpx_cluster_features* features_host, uint64_t capacity, uint64_t* ticket) {
  if (!p || !ticket || n > p->max_hits || capacity > p->capacity) return TPX_ERR_INVALID_ARG;
  job* j = new (std::nothrow) job;
  if (!j) return TPX_ERR_OOM;
  j->hits = hits_host;
  j->n = n;
  j->labels = labels_host;
  j->feats = features_host;
  j->capacity = capacity;
  {
    std::lock_guard<std::mutex> lk(p->m);
    const uint64_t t = p->next_ticket++;
    p->jobs[t] = j;
    p->slots[t % p->slots.size()].q.push_back(j);
    *ticket = t;
  }
  p->cv_work.notify_all();
  return TPX_OK;
}

int tpx_pipeline_wait(tpx_pipeline* p, uint64_t ticket, uint64_t* n_clusters_out) {
  if (!p || !n_clusters_out) return TPX_ERR_INVALID_ARG;
  std::unique_lock<std::mutex> lk(p->m);
  auto it = p->jobs.find(ticket);
  if (it == p->jobs.end()) return TPX_ERR_INVALID_ARG;
  job* j = it->second;
  p->cv_done.wait(lk, [&] { return j->done; });
  *n_clusters_out = j->n_clusters;
  const int rc = j->status;
  p->jobs.erase(it);
  delete j;
  return rc;
}

int tpx_pipeline_mark(tpx_pipeline* p, int which) {
  if (!p || (which != 0 && which != 1)) return TPX_ERR_INVALID_ARG;
  for (slot& s : p->slots)
    if (cudaEventRecord(which ? s.t_stop : s.t_start, s.stream) != cudaSuccess) return TPX_ERR_CUDA;
  if (cudaEventRecord(which ? p->c_stop[0] : p->c_start[0], p->h2d) != cudaSuccess ||
      cudaEventRecord(which ? p->c_stop[1] : p->c_start[1], p->d2h) != cudaSuccess)
    return TPX_ERR_CUDA;
  return TPX_OK;
}

int tpx_pipeline_elapsed_ms(tpx_pipeline* p, float* ms) {
  if (!p || !ms) return TPX_ERR_INVALID_ARG;
  float best = 0.f;
  // span from the earliest start to the latest stop over the slot streams and
  // the two copy streams
  std::vector<cudaEvent_t> st, sp;
  for (slot& s : p->slots) {
    st.push_back(s.t_start);
    sp.push_back(s.t_stop);
  }
  for (int i = 0; i < 2; ++i) {
    st.push_back(p->c_start[i]);
    sp.push_back(p->c_stop[i]);
  }
  for (cudaEvent_t e0 : st)
    for (cudaEvent_t e1 : sp) {
      float v = 0.f;
      if (cudaEventSynchronize(e1) != cudaSuccess) return TPX_ERR_CUDA;
      if (cudaEventElapsedTime(&v, e0, e1) != cudaSuccess) return TPX_ERR_CUDA;
      if (v > best) best = v;
    }
  *ms = best;
  return TPX_OK;
}

void tpx_pipeline_destroy(tpx_pipeline* p) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(p->m);
    p->stop = true;
  }
  p->cv_work.notify_all();
  for (slot& s : p->slots)
    if (s.th.joinable()) s.th.join();
  for (slot& s : p->slots) {
    if (s.stream) {
      cudaStreamSynchronize(s.stream);
      cudaStreamDestroy(s.stream);
    }
    if (s.t_start) cudaEventDestroy(s.t_start);
    if (s.t_stop) cudaEventDestroy(s.t_stop);
    if (s.ev_in) cudaEventDestroy(s.ev_in);
    if (s.ev_run) cudaEventDestroy(s.ev_run);
    if (s.ev_out) cudaEventDestroy(s.ev_out);
    tpx_cluster_destroy(s.ctx);
  }
  for (cudaStream_t cs : {p->h2d, p->d2h})
    if (cs) {
      cudaStreamSynchronize(cs);
      cudaStreamDestroy(cs);
    }
  for (int i = 0; i < 2; ++i) {
    if (p->c_start[i]) cudaEventDestroy(p->c_start[i]);
    if (p->c_stop[i]) cudaEventDestroy(p->c_stop[i]);
  }
  for (auto& kv : p->jobs) delete kv.second;
  delete p;
}

}  // extern "C"
