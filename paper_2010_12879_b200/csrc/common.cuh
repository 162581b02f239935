// Shared helpers for the spfd_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <chrono>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/spfd_b200.h"
#include <nvtx3/nvToolsExt.h>

namespace spfd {

// NVTX range over a C-ABI call (visible in Nsight Systems / ncu --nvtx)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};


// ---------------------------------------------------------------- errors --
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string &msg);

#define SPFD_CUDA(expr)                                                        \
    do {                                                                       \
        cudaError_t _e = (expr);                                               \
        if (_e != cudaSuccess)                                                 \
            throw ::spfd::Error(SPFD_ECUDA, std::string(#expr) + ": " +        \
                                                cudaGetErrorString(_e));       \
    } while (0)

#define SPFD_CHECK(cond, code, msg)                                            \
    do {                                                                       \
        if (!(cond)) throw ::spfd::Error((code), (msg));                       \
    } while (0)

// Every kernel launch on the library's paths is followed by this check; it
// also counts launches (bench.py reports them as `gpu_launches`).
int64_t launch_count();
void count_launch();
#define SPFD_LAUNCH_CHECK()                                                    \
    do {                                                                       \
        ::spfd::count_launch();                                                \
        SPFD_CUDA(cudaGetLastError());                                         \
    } while (0)

// ------------------------------------------------------- device buffers --
// RAII device allocation (stream-ordered).  Handles own their buffers; the
// Python side owns every input/output tensor.
// The library's private stream-ordered memory pool on the current device
// (created on first use; null if the driver has no pool support).
inline cudaMemPool_t lib_pool() {
    static cudaMemPool_t pools[64] = {};
    static bool made[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    if (!made[dev]) {
        made[dev] = true;
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&pools[dev], &props) != cudaSuccess) {
            cudaGetLastError();
            pools[dev] = nullptr;
        } else {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    return pools[dev];
}

// Bytes the pool currently hands out / its high-water mark since the last reset.
inline size_t pool_used() {
    size_t v = 0;
    if (cudaMemPool_t pool = lib_pool()) cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &v);
    return v;
}
inline size_t pool_used_high_reset() {
    size_t v = 0;
    if (cudaMemPool_t pool = lib_pool()) {
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &v);
        size_t zero = 0;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero);
    }
    return v;
}

// Grow the pool in one step so that `bytes` more can be handed out without
// mapping memory again.  Growing it allocation by allocation is slow and
// erratic on the B200 driver: single 35-816 MB requests that had to map
// memory took 5-176 ms each (C3 setup 0.6-2.8 s, SPFD_ALLOC_TRACE=1).
inline void pool_reserve(size_t bytes) {
    cudaMemPool_t pool = lib_pool();
    if (!pool || bytes == 0) return;
    size_t reserved = 0, used = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    if (reserved >= used + bytes) return;
    // (trimming the free blocks first and mapping one block for the whole
    // estimate measured no steadier)
    cudaDeviceSynchronize();
    void *p = nullptr;
    if (cudaMallocFromPoolAsync(&p, used + bytes - reserved, pool, 0) == cudaSuccess) {
        cudaFreeAsync(p, 0);
        cudaStreamSynchronize(0);
    } else {
        cudaGetLastError();  // not enough memory for the whole estimate: grow per allocation
    }
}

// Return the pool's unused reservations (setup temporaries) to the device,
// keeping a floor of SPFD_POOL_KEEP_MB (default 4096 MB of the 180 GB) mapped
// so that the next setup does not pay the page mapping again (C3 repeat
// setups varied 1.6-4.4 s with a full trim).
inline void pool_trim() {
    if (cudaMemPool_t pool = lib_pool()) {
        static long long keep_mb = -1;
        if (keep_mb < 0) {
            const char *e = getenv("SPFD_POOL_KEEP_MB");
            keep_mb = e ? atoll(e) : 4096;
            if (keep_mb < 0) keep_mb = 0;
        }
        cudaDeviceSynchronize();
        cudaMemPoolTrimTo(pool, (size_t)keep_mb << 20);
    }
}

template <class T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf &operator=(DevBuf &&o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    // Device memory comes from the library's own stream-ordered pool (one per
    // device, unlimited release threshold): setup allocates and frees many
    // large temporaries (SpGEMM expansions, sorts), and recycling pool memory
    // avoids re-mapping pages every time (plain cudaMalloc/cudaFree made the C3
    // setup vary between 2 and 12 s).  The pool is private, so the default
    // pool other libraries (PyTorch's cudaMallocAsync backend) use keeps its
    // own policy, and pool_trim() hands the setup temporaries back at the end
    // of every setup entry point.  Frees first synchronise the device, like
    // cudaFree, so no stream can still be using the buffer.
    void alloc(size_t count) {
        release();
        if (count == 0) count = 1;
        cudaMemPool_t pool = lib_pool();
        static const bool tr = getenv("SPFD_ALLOC_TRACE") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        cudaError_t e = pool ? cudaMallocFromPoolAsync((void **)&p, count * sizeof(T), pool, 0)
                             : cudaMallocAsync((void **)&p, count * sizeof(T), 0);
        const auto t1 = std::chrono::steady_clock::now();
        if (e == cudaSuccess) e = cudaStreamSynchronize(0);
        if (tr) {
            const auto t2 = std::chrono::steady_clock::now();
            const double a_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
            const double s_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
            if (a_ms + s_ms > 5.0)
                fprintf(stderr, "[alloc] %10.1f MB  malloc %8.1f ms  sync %8.1f ms\n", count * sizeof(T) / 1e6, a_ms, s_ms);
        }
        if (e != cudaSuccess) {
            p = nullptr;
            throw Error(SPFD_ENOMEM, std::string("device allocation failed: ") + cudaGetErrorString(e));
        }
        n = count;
    }
    void release() {
        if (p) {
            static const bool tr = getenv("SPFD_ALLOC_TRACE") != nullptr;
            const auto t0 = std::chrono::steady_clock::now();
            cudaDeviceSynchronize();
            const auto t1 = std::chrono::steady_clock::now();
            cudaFreeAsync(p, 0);
            if (tr) {
                const auto t2 = std::chrono::steady_clock::now();
                const double a_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
                const double f_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
                if (a_ms + f_ms > 5.0)
                    fprintf(stderr, "[free ] %10.1f MB  sync %8.1f ms  free %8.1f ms\n", n * sizeof(T) / 1e6, a_ms, f_ms);
            }
        }
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
    T *get() const { return p; }
};

// int32 -> int64 widening functor for CUB scans over int32 counts
struct WidenI32 {
    __host__ __device__ int64_t operator()(int v) const { return (int64_t)v; }
};
struct RootFlag {  // operator construction: bit 2 marks a component root
    __host__ __device__ uint8_t operator()(uint8_t f) const { return (f & 2) ? 1 : 0; }
};

inline int grid_for(int64_t n, int threads, int cap = 148 * 16) {
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

// ---------------------------------------------- exact (no-FMA) arithmetic --
// The reference computes with numpy/scipy (no fused multiply-add); the bit-
// exact kernels use explicitly rounded ops so nvcc cannot contract them.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// ---------------------------------------------- deterministic reductions --
// Block-level sum of K values per thread in a FIXED tree order (xor-shuffle
// within warps, then warp 0 over the per-warp partials).  Result valid in
// thread 0.  No atomics: the order depends only on blockDim.
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double *smem /* [32*K] */) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) smem[warp * K + k] = v[k];
    }
    __syncwarp();      // reconverge the warp before the CTA barrier (synccheck)
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double t = lane < nwarps ? smem[lane * K + k] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            v[k] = t;
        }
    }
    __syncwarp();      // reconverge warp 0 after its reduction (synccheck)
    __syncthreads();
}

}  // namespace spfd
