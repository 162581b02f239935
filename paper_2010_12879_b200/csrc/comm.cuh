// Inter-GPU transport for the z-slab decomposition.
//
// Two implementations of one small interface:
//  * NcclComm  -- ncclSend/ncclRecv (grouped) and ncclAllGather on the
//    solve stream; NCCL is loaded with dlopen so single-GPU use needs no
//    NCCL at all.  This is the production path (NVLink 5 / NVSwitch).
//  * HostComm  -- calls host callbacks (e.g. torch.distributed gloo from
//    Python) after synchronising the stream; used to test the distributed
//    algorithm with several processes sharing one GPU.
#pragma once
#include <vector>

#include "common.cuh"

namespace spfd {

struct Comm {
    int rank = 0, size = 1;
    virtual ~Comm() {}
    // point-to-point exchange group: queue sends/recvs, then run them
    virtual void begin() = 0;
    virtual void send(int peer, const void *buf, size_t bytes) = 0;
    virtual void recv(int peer, void *buf, size_t bytes) = 0;
    virtual void end(cudaStream_t s) = 0;
    // rank-ordered concatenation of `bytes` from every rank into recv
    virtual void allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) = 0;
    // every operation is stream-ordered (no host synchronisation), so a
    // sequence of them can be captured into a CUDA graph
    virtual bool stream_ordered() const { return false; }
};

Comm *comm_nccl(const void *unique_id, int rank, int size);
void nccl_unique_id(void *out128);
Comm *comm_host(const spfd_comm_callbacks &cb, int rank, int size);

}  // namespace spfd
