// comm.cu -- tpx_comm: the rank communicator of the ToA-sharded run
// (include/tpx_cluster.h "ToA-sharded multi-GPU clustering", comm.h).
//
// NCCL is loaded with dlopen (libnccl.so.2: the copy PyTorch already loaded
// into the process if there is one, else the system library), so the C ABI
// library has no link-time NCCL dependency and loads on machines without it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>

#include "comm.h"

namespace {

struct nccl_api {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  bool ok;
};

nccl_api g_nccl;
std::once_flag g_nccl_once;

template <typename F>
bool sym(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  return out != nullptr;
}

const nccl_api* nccl() {
  std::call_once(g_nccl_once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      fprintf(stderr, "tpx_comm: libnccl.so.2 not found: %s\n", dlerror());
      return;
    }
    nccl_api& a = g_nccl;
    a.ok = sym(h, "ncclGetUniqueId", a.GetUniqueId) && sym(h, "ncclCommInitRank", a.CommInitRank) &&
           sym(h, "ncclCommDestroy", a.CommDestroy) && sym(h, "ncclAllGather", a.AllGather) &&
           sym(h, "ncclSend", a.Send) && sym(h, "ncclRecv", a.Recv) && sym(h, "ncclGroupStart", a.GroupStart) &&
           sym(h, "ncclGroupEnd", a.GroupEnd) && sym(h, "ncclGetErrorString", a.GetErrorString);
  });
  return g_nccl.ok ? &g_nccl : nullptr;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return TPX_OK;
  fprintf(stderr, "tpx_comm: %s failed: %s\n", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
  return TPX_ERR_NCCL;
}

}  // namespace

struct tpx_comm {
  int rank, world;
  ncclComm_t nccl;  // NCCL transport (owned), else nullptr
  tpx_allgather_fn allgather;
  tpx_sendrecv_fn sendrecv;
  void* user;
  char* hbuf;  // pinned staging (host transport): [send | recv]
  size_t hcap;
};

namespace tpx {

int comm_rank(const tpx_comm* c) { return c->rank; }
int comm_world(const tpx_comm* c) { return c->world; }

static int host_reserve(tpx_comm* c, size_t bytes) {
  if (bytes <= c->hcap) return TPX_OK;
  if (c->hbuf) cudaFreeHost(c->hbuf);
  c->hbuf = nullptr;
  c->hcap = 0;
  size_t cap = bytes < (1u << 20) ? (1u << 20) : bytes;
  if (cudaHostAlloc((void**)&c->hbuf, cap, cudaHostAllocDefault) != cudaSuccess) return TPX_ERR_CUDA;
  c->hcap = cap;
  return TPX_OK;
}

int comm_allgather(tpx_comm* c, const void* d_send, void* d_recv, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return TPX_OK;
  if (c->nccl) return nccl_check(g_nccl.AllGather(d_send, d_recv, bytes, ncclUint8, c->nccl, s), "ncclAllGather");
  const size_t total = bytes * (size_t)(c->world + 1);
  int rc = host_reserve(c, total);
  if (rc) return rc;
  char* hs = c->hbuf;
  char* hr = c->hbuf + bytes;
  if (cudaMemcpyAsync(hs, d_send, bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return TPX_ERR_CUDA;
  if (c->allgather(c->user, hs, hr, bytes) != 0) return TPX_ERR_NCCL;
  if (cudaMemcpyAsync(d_recv, hr, bytes * c->world, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return TPX_ERR_CUDA;
  return TPX_OK;
}

int comm_sendrecv(tpx_comm* c, int to, const void* d_send, size_t send_bytes, int from, void* d_recv,
                  size_t recv_bytes, cudaStream_t s) {
  if (to < 0 || send_bytes == 0) to = -1, send_bytes = 0;
  if (from < 0 || recv_bytes == 0) from = -1, recv_bytes = 0;
  if (to < 0 && from < 0) return TPX_OK;
  if (c->nccl) {
    int rc = TPX_OK;
    if ((rc = nccl_check(g_nccl.GroupStart(), "ncclGroupStart"))) return rc;
    if (to >= 0) rc = nccl_check(g_nccl.Send(d_send, send_bytes, ncclUint8, to, c->nccl, s), "ncclSend");
    if (!rc && from >= 0) rc = nccl_check(g_nccl.Recv(d_recv, recv_bytes, ncclUint8, from, c->nccl, s), "ncclRecv");
    const int rc2 = nccl_check(g_nccl.GroupEnd(), "ncclGroupEnd");
    return rc ? rc : rc2;
  }
  int rc = host_reserve(c, send_bytes + recv_bytes);
  if (rc) return rc;
  char* hs = c->hbuf;
  char* hr = c->hbuf + send_bytes;
  if (send_bytes && cudaMemcpyAsync(hs, d_send, send_bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return TPX_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return TPX_ERR_CUDA;
  if (c->sendrecv(c->user, to, hs, send_bytes, from, hr, recv_bytes) != 0) return TPX_ERR_NCCL;
  if (recv_bytes && (cudaMemcpyAsync(d_recv, hr, recv_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess ||
                     cudaStreamSynchronize(s) != cudaSuccess))
    return TPX_ERR_CUDA;
  return TPX_OK;
}

int comm_group_start(tpx_comm* c) { return c->nccl ? nccl_check(g_nccl.GroupStart(), "ncclGroupStart") : TPX_OK; }
int comm_group_end(tpx_comm* c) { return c->nccl ? nccl_check(g_nccl.GroupEnd(), "ncclGroupEnd") : TPX_OK; }

}  // namespace tpx

extern "C" {

int tpx_nccl_unique_id(uint8_t id_out[128]) {
  if (!id_out) return TPX_ERR_INVALID_ARG;
  const nccl_api* a = nccl();
  if (!a) return TPX_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  int rc = nccl_check(a->GetUniqueId(&id), "ncclGetUniqueId");
  if (rc) return rc;
  memcpy(id_out, &id, 128);
  return TPX_OK;
}

int tpx_nccl_comm_init(int rank, int world, const uint8_t id[128], tpx_comm** out) {
  if (!out || !id || world < 1 || rank < 0 || rank >= world) return TPX_ERR_INVALID_ARG;
  *out = nullptr;
  const nccl_api* a = nccl();
  if (!a) return TPX_ERR_NCCL;
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  ncclComm_t comm = nullptr;
  int rc = nccl_check(a->CommInitRank(&comm, world, uid, rank), "ncclCommInitRank");
  if (rc) return rc;
  tpx_comm* c = new (std::nothrow) tpx_comm();
  if (!c) {
    a->CommDestroy(comm);
    return TPX_ERR_OOM;
  }
  c->rank = rank;
  c->world = world;
  c->nccl = comm;
  *out = c;
  return TPX_OK;
}

int tpx_comm_create_host(int rank, int world, tpx_allgather_fn allgather, tpx_sendrecv_fn sendrecv, void* user,
                         tpx_comm** out) {
  if (!out || !allgather || !sendrecv || world < 1 || rank < 0 || rank >= world) return TPX_ERR_INVALID_ARG;
  tpx_comm* c = new (std::nothrow) tpx_comm();
  if (!c) return TPX_ERR_OOM;
  c->rank = rank;
  c->world = world;
  c->allgather = allgather;
  c->sendrecv = sendrecv;
  c->user = user;
  *out = c;
  return TPX_OK;
}

void tpx_comm_destroy(tpx_comm* c) {
  if (!c) return;
  if (c->nccl && g_nccl.CommDestroy) g_nccl.CommDestroy(c->nccl);
  if (c->hbuf) cudaFreeHost(c->hbuf);
  delete c;
}

int tpx_comm_rank(const tpx_comm* c, int* rank, int* world) {
  if (!c) return TPX_ERR_INVALID_ARG;
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  return TPX_OK;
}

// Byte pattern of rank r at position i (self test).
static unsigned char pat(int r, size_t i) { return (unsigned char)((r * 131 + i * 7 + (i >> 8)) & 0xff); }

int tpx_comm_selftest(tpx_comm* c, size_t bytes) {
  if (!c || bytes == 0) return TPX_ERR_INVALID_ARG;
  if (c->nccl) return TPX_ERR_UNSUPPORTED;  // device buffers: exercised by the sharded GPU tests
  const int W = c->world, r = c->rank;
  unsigned char* send = new (std::nothrow) unsigned char[bytes];
  unsigned char* recv = new (std::nothrow) unsigned char[bytes * W];
  if (!send || !recv) {
    delete[] send;
    delete[] recv;
    return TPX_ERR_OOM;
  }
  int rc = TPX_OK;
  for (size_t i = 0; i < bytes; ++i) send[i] = pat(r, i);
  if (c->allgather(c->user, send, recv, bytes) != 0) rc = TPX_ERR_NCCL;
  for (int q = 0; q < W && !rc; ++q)
    for (size_t i = 0; i < bytes; ++i)
      if (recv[(size_t)q * bytes + i] != pat(q, i)) {
        rc = TPX_ERR_INVALID_ARG;
        break;
      }
  // neighbour exchange: to r-1, from r+1 (the halo direction of the sharded run)
  const int to = r > 0 ? r - 1 : -1, from = r + 1 < W ? r + 1 : -1;
  if (!rc && c->sendrecv(c->user, to, send, to >= 0 ? bytes : 0, from, recv, from >= 0 ? bytes : 0) != 0)
    rc = TPX_ERR_NCCL;
  for (size_t i = 0; i < bytes && !rc && from >= 0; ++i)
    if (recv[i] != pat(from, i)) rc = TPX_ERR_INVALID_ARG;
  delete[] send;
  delete[] recv;
  return rc;
}

}  // extern "C"
