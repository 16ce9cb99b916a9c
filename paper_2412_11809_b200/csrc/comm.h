// comm.h -- internal interface of the rank communicator behind tpx_comm
// (comm.cu): the exchange steps of the ToA-sharded run (sharded.cuh).
//
// Two transports, one interface:
//  * NCCL (the multi-GPU product path): collectives and point-to-point
//    transfers of device buffers on the run stream, one process per GPU,
//    NVLink / NVSwitch.  libnccl is loaded with dlopen on first use, so the
//    library itself has no link-time NCCL dependency.
//  * host callbacks: device buffers staged through pinned host memory and
//    moved by caller-supplied functions (in-process virtual ranks, gloo
//    process groups, several ranks sharing one GPU: functional runs only).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

#include "tpx_cluster.h"

namespace tpx {

int comm_rank(const tpx_comm* c);
int comm_world(const tpx_comm* c);
// All-gather `bytes` per rank: d_recv[r * bytes ...] = rank r's d_send.
int comm_allgather(tpx_comm* c, const void* d_send, void* d_recv, size_t bytes, cudaStream_t s);
// Send d_send (send_bytes) to rank `to` and receive recv_bytes from rank
// `from` into d_recv; -1 skips a direction.  Both sides agree on the sizes.
int comm_sendrecv(tpx_comm* c, int to, const void* d_send, size_t send_bytes, int from, void* d_recv,
                  size_t recv_bytes, cudaStream_t s);
// Batch the operations issued in between (NCCL group); no-op for callbacks.
int comm_group_start(tpx_comm* c);
int comm_group_end(tpx_comm* c);

}  // namespace tpx
