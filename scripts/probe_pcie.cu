// Probe: which SM-side load form reads mapped pinned host memory most efficiently over
// PCIe on B200?  (Standalone; nvcc -gencode arch=compute_100a,code=sm_100a probe_pcie.cu)
// Prints GB/s for each variant copying 1 GiB host -> HBM, plus the copy-engine figure.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

template <int V>
__device__ __forceinline__ uint4 ld(const uint4* p) {
    uint4 v;
    if constexpr (V == 0)
        asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if constexpr (V == 1)
        asm volatile("ld.global.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if constexpr (V == 2)
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else
        asm volatile("ld.global.L1::no_allocate.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int V, int U>
__global__ void __launch_bounds__(512) copy_k(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
    const size_t stride = (size_t)gridDim.x * blockDim.x * U;
    for (size_t base = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < n; base += stride) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            size_t i = base + (size_t)u * blockDim.x;
            if (i < n) r[u] = ld<V>(s + i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            size_t i = base + (size_t)u * blockDim.x;
            if (i < n) d[i] = r[u];
        }
    }
}

// L2 bulk prefetch ahead of plain loads: one thread per CTA issues cp.async.bulk.prefetch.L2
// for the CTA's next chunk, then the CTA reads the current chunk (hits L2 if prefetched).
template <int CHUNK>
__global__ void __launch_bounds__(512) copy_prefetch(const char* __restrict__ s, char* __restrict__ d, size_t bytes) {
    const size_t nchunks = bytes / CHUNK;
    size_t c = blockIdx.x;
    if (threadIdx.x == 0 && c < nchunks)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s + c * CHUNK), "r"(CHUNK) : "memory");
    for (; c < nchunks; c += gridDim.x) {
        size_t nx = c + gridDim.x;
        if (threadIdx.x == 0 && nx < nchunks)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s + nx * CHUNK), "r"(CHUNK) : "memory");
        const uint4* sp = reinterpret_cast<const uint4*>(s + c * CHUNK);
        uint4* dp = reinterpret_cast<uint4*>(d + c * CHUNK);
        constexpr int NV = CHUNK / 16;
        for (int i = threadIdx.x; i < NV; i += blockDim.x) dp[i] = ld<0>(sp + i);
    }
}

int main() {
    const size_t bytes = 1ull << 30;
    char *h, *hd, *d;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
    CK(cudaMalloc(&d, bytes));
    for (size_t i = 0; i < bytes; i += 4096) h[i] = (char)i;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto launch) {
        float best = 1e9;
        for (int r = 0; r < 4; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r) best = ms < best ? ms : best;
        }
        cudaError_t e = cudaGetLastError();
        printf("%-40s %8.2f GB/s %s\n", name, bytes / (best * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    const size_t n = bytes / 16;
    for (int g : {16, 32, 148}) {
        char nm[64];
        snprintf(nm, 64, "ld plain U8 grid %d", g);
        timeit(nm, [&] { copy_k<0, 8><<<g, 512>>>((const uint4*)hd, (uint4*)d, n); });
        snprintf(nm, 64, "ld L2::256B U8 grid %d", g);
        timeit(nm, [&] { copy_k<1, 8><<<g, 512>>>((const uint4*)hd, (uint4*)d, n); });
        snprintf(nm, 64, "ld.nc L2::256B U8 grid %d", g);
        timeit(nm, [&] { copy_k<2, 8><<<g, 512>>>((const uint4*)hd, (uint4*)d, n); });
        snprintf(nm, 64, "ld L2::128B U8 grid %d", g);
        timeit(nm, [&] { copy_k<3, 8><<<g, 512>>>((const uint4*)hd, (uint4*)d, n); });
        snprintf(nm, 64, "bulk prefetch.L2 64K grid %d", g);
        timeit(nm, [&] { copy_prefetch<65536><<<g, 512>>>(hd, d, bytes); });
    }
    timeit("copy engine cudaMemcpyAsync", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice); });
    return 0;
}
