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
  std::mutex m;
  std::condition_variable cv_work, cv_done;
  std::map<uint64_t, job*> jobs;
  uint64_t next_ticket = 0;
  bool stop = false;
};

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
    const int rc = tpx_cluster_run_host(s.ctx, j->hits, j->n, j->labels, j->feats, j->capacity, &k, s.ws, s.ws_bytes,
                                        s.stream);
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
        cudaEventCreate(&s.t_start) != cudaSuccess || cudaEventCreate(&s.t_stop) != cudaSuccess)
      rc = TPX_ERR_CUDA;
  }
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
  return TPX_OK;
}

int tpx_pipeline_elapsed_ms(tpx_pipeline* p, float* ms) {
  if (!p || !ms) return TPX_ERR_INVALID_ARG;
  float best = 0.f;
  // span from the earliest start to the latest stop over the slot streams
  for (slot& s0 : p->slots)
    for (slot& s1 : p->slots) {
      float v = 0.f;
      if (cudaEventSynchronize(s1.t_stop) != cudaSuccess) return TPX_ERR_CUDA;
      if (cudaEventElapsedTime(&v, s0.t_start, s1.t_stop) != cudaSuccess) return TPX_ERR_CUDA;
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
    tpx_cluster_destroy(s.ctx);
  }
  for (auto& kv : p->jobs) delete kv.second;
  delete p;
}

}  // extern "C"
