// Probe: HBM -> shared-memory throughput of 1-D bulk copies (cp.async.bulk)
// issued by one producer warp per CTA, with S stages of B bytes split into
// NC copies each, consumers only release the stage.  Also the same for a
// plain coalesced LDG read loop.  Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a tools/tma_probe.cu -o /tmp/tma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, unsigned n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned par) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
                     : "=r"(done) : "r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void *d, const void *s, unsigned n, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(su32(d)),
                 "l"(s), "r"(n), "r"(su32(b)) : "memory");
}

__global__ void k_tma(const char *src, size_t total, int B, int S, int NC, double *sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[8], empty[8];
    const int tid = threadIdx.x, nc = blockDim.x - 32;
    if (tid == 0) {
        for (int k = 0; k < S; ++k) { mbar_init(&full[k], 1); mbar_init(&empty[k], nc / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const size_t ntile = total / B;
    if (tid >= nc) {
        const int lane = tid & 31;
        int i = 0;
        for (size_t t = blockIdx.x; t < ntile; t += gridDim.x, ++i) {
            const int st = i % S;
            if (i >= S) mbar_wait(&empty[st], ((i / S) - 1) & 1);
            if (lane == 0) mbar_expect(&full[st], B);
            __syncwarp();
            const int part = B / NC;
            if (lane < NC) bulk(sm + (size_t)st * B + lane * part, src + t * B + lane * part, part, &full[st]);
        }
        return;
    }
    double acc = 0;
    int i = 0;
    for (size_t t = blockIdx.x; t < ntile; t += gridDim.x, ++i) {
        const int st = i % S;
        mbar_wait(&full[st], (i / S) & 1);
        acc += reinterpret_cast<const double *>(sm + (size_t)st * B)[tid];
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[st]);
    }
    if (acc == 12345.0) sink[0] = acc;
}

__global__ void k_ldg(const double2 *src, size_t n, double *sink) {
    double2 acc = make_double2(0, 0);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double2 v = src[i];
        acc.x += v.x; acc.y += v.y;
    }
    if (acc.x == 12345.0) sink[0] = acc.y;
}

int main() {
    const size_t total = (size_t)2 << 30;
    char *src; double *sink;
    cudaMalloc(&src, total); cudaMalloc(&sink, 8);
    cudaMemset(src, 0, total);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    int Bs[] = {8192, 16384, 32768, 65536};
    int Ss[] = {2, 3, 4};
    int NCs[] = {1, 4, 16};
    for (int B : Bs) for (int S : Ss) for (int NC : NCs) {
        if ((size_t)B * S > 200 * 1024) continue;
        for (int cps = 1; cps <= 2; ++cps) {
            if ((size_t)B * S * cps > 220 * 1024) continue;
            if (cps == 2) cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, B * S);
            float best = 1e9;
            for (int rep = 0; rep < 4; ++rep) {
                cudaEventRecord(a);
                k_tma<<<nsm * cps, 256 + 32, B * S>>>(src, total, B, S, NC, sink);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
            }
            cudaError_t e = cudaGetLastError();
            printf("tma B=%6d S=%d NC=%2d ctas/sm=%d : %7.1f GB/s %s\n", B, S, NC, cps, total / best / 1e6, e ? cudaGetErrorString(e) : "");
            cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        }
    }
    for (int g = 1; g <= 8; g *= 2) {
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(a);
            k_ldg<<<nsm * g, 256>>>((const double2 *)src, total / 16, sink);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        printf("ldg ctas/sm=%d : %7.1f GB/s\n", g, total / best / 1e6);
    }
    return 0;
}
