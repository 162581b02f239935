// NCCL (dlopen) and host-callback transports for the z-slab decomposition.
#include <dlfcn.h>

#include <cstring>
#include <string>

#include "comm.cuh"

namespace spfd {

namespace {

// minimal NCCL ABI (nccl.h 2.2x): opaque comm, 128-byte unique id
typedef struct ncclComm *ncclComm_t;
struct ncclUniqueId {
    char internal[128];
};
typedef int ncclResult_t;
constexpr int kNcclInt8 = 0;

struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl() {
    static NcclApi api;
    if (api.h) return api;
    // SPFD_NCCL_LIB (the Python side sets it to the nvidia-nccl wheel's library
    // when it is not set, distributed.py), else the loader's search path
    const char *env = getenv("SPFD_NCCL_LIB");
    const char *cands[] = {env, "libnccl.so.2"};
    for (const char *c : cands) {
        if (!c) continue;
        api.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
        if (api.h) break;
    }
    SPFD_CHECK(api.h != nullptr, SPFD_ENCCL, "cannot load libnccl.so.2 (set SPFD_NCCL_LIB)");
    auto sym = [&](const char *n) {
        void *f = dlsym(api.h, n);
        SPFD_CHECK(f != nullptr, SPFD_ENCCL, std::string("NCCL symbol missing: ") + n);
        return f;
    };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    return api;
}

#define SPFD_NCCL(expr)                                                                       \
    do {                                                                                      \
        ncclResult_t _r = (expr);                                                             \
        if (_r != 0) throw Error(SPFD_ENCCL, std::string(#expr) + ": " + nccl().GetErrorString(_r)); \
    } while (0)

struct NcclComm : Comm {
    ncclComm_t c = nullptr;
    bool stream_ordered() const override { return true; }
    struct Op {
        int peer, kind;
        void *buf;
        size_t bytes;
    };
    std::vector<Op> q;
    ~NcclComm() override {
        if (c) nccl().CommDestroy(c);
    }
    void begin() override { q.clear(); }
    void send(int peer, const void *buf, size_t bytes) override {
        if (bytes) q.push_back({peer, 0, const_cast<void *>(buf), bytes});
    }
    void recv(int peer, void *buf, size_t bytes) override {
        if (bytes) q.push_back({peer, 1, buf, bytes});
    }
    void end(cudaStream_t s) override {
        if (q.empty()) return;
        NcclApi &n = nccl();
        SPFD_NCCL(n.GroupStart());
        for (auto &o : q) {
            if (o.kind == 0) SPFD_NCCL(n.Send(o.buf, o.bytes, kNcclInt8, o.peer, c, s));
            else SPFD_NCCL(n.Recv(o.buf, o.bytes, kNcclInt8, o.peer, c, s));
        }
        SPFD_NCCL(n.GroupEnd());
        q.clear();
    }
    void allgather(const void *sendb, void *recvb, size_t bytes, cudaStream_t s) override {
        SPFD_NCCL(nccl().AllGather(sendb, recvb, bytes, kNcclInt8, c, s));
    }
};

struct HostComm : Comm {
    spfd_comm_callbacks cb;
    std::vector<int> peer, kind;
    std::vector<void *> buf;
    std::vector<int64_t> bytes;
    void begin() override { peer.clear(); kind.clear(); buf.clear(); bytes.clear(); }
    void send(int p, const void *b, size_t n) override {
        if (!n) return;
        peer.push_back(p); kind.push_back(0); buf.push_back(const_cast<void *>(b)); bytes.push_back((int64_t)n);
    }
    void recv(int p, void *b, size_t n) override {
        if (!n) return;
        peer.push_back(p); kind.push_back(1); buf.push_back(b); bytes.push_back((int64_t)n);
    }
    void end(cudaStream_t s) override {
        if (peer.empty()) return;
        SPFD_CUDA(cudaStreamSynchronize(s));
        int rc = cb.exchange(cb.user, (int)peer.size(), peer.data(), kind.data(), buf.data(), bytes.data());
        SPFD_CHECK(rc == 0, SPFD_ENCCL, "host transport exchange failed");
        begin();
    }
    void allgather(const void *sendb, void *recvb, size_t n, cudaStream_t s) override {
        SPFD_CUDA(cudaStreamSynchronize(s));
        int rc = cb.allgather(cb.user, sendb, recvb, (int64_t)n);
        SPFD_CHECK(rc == 0, SPFD_ENCCL, "host transport allgather failed");
    }
};

}  // namespace

void nccl_unique_id(void *out) {
    ncclUniqueId id;
    SPFD_NCCL(nccl().GetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
}

Comm *comm_nccl(const void *unique_id, int rank, int size) {
    auto *c = new NcclComm();
    c->rank = rank;
    c->size = size;
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    try {
        SPFD_NCCL(nccl().CommInitRank(&c->c, size, id, rank));
    } catch (...) {
        delete c;
        throw;
    }
    return c;
}

Comm *comm_host(const spfd_comm_callbacks &cb, int rank, int size) {
    SPFD_CHECK(cb.exchange && cb.allgather, SPFD_EINVAL, "null transport callback");
    auto *c = new HostComm();
    c->cb = cb;
    c->rank = rank;
    c->size = size;
    return c;
}

}  // namespace spfd
