// Probe: K1 bytes-in-flight vs (a) H2D bandwidth and (b) the latency a small concurrent
// H2D transfer (a decision call's inputs) sees while K1 saturates the link.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 probe_inflight.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

template <int U>
__global__ void copy_k(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
    const size_t stride = (size_t)gridDim.x * blockDim.x * U;
    for (size_t base = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < n; base += stride) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            size_t i = base + (size_t)u * blockDim.x;
            if (i < n) asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r[u].x), "=r"(r[u].y), "=r"(r[u].z), "=r"(r[u].w) : "l"(s + i));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            size_t i = base + (size_t)u * blockDim.x;
            if (i < n) d[i] = r[u];
        }
    }
}

__global__ void touch(const uint4* s, uint4* d, int n) {  // a 1-CTA decision-like reader of host memory
    for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = s[i];
}

int main() {
    const size_t bytes = 1ull << 30;
    char *h, *hd, *d, *hs, *hsd, *ds;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
    CK(cudaMalloc(&d, bytes));
    const int small = 64 << 10;
    CK(cudaHostAlloc(&hs, small, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&hsd, hs, 0));
    CK(cudaMalloc(&ds, small));
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const size_t n = bytes / 16;
    struct Cfg { int grid, block, unroll; } cfgs[] = {{32, 512, 8}, {16, 512, 8}, {8, 512, 8}, {8, 512, 4}, {8, 256, 4},
                                                     {4, 512, 4}, {4, 256, 4}, {16, 256, 2}, {8, 128, 4}, {2, 512, 4}};
    auto small_latency = [&](bool zero_copy) {
        // 20 round trips, host wall each
        double tot = 0;
        for (int i = 0; i < 20; ++i) {
            auto t0 = std::chrono::steady_clock::now();
            if (zero_copy) touch<<<1, 1024, 0, b>>>((const uint4*)hsd, (uint4*)ds, small / 16);
            else cudaMemcpyAsync(ds, hs, small, cudaMemcpyHostToDevice, b);
            cudaStreamSynchronize(b);
            tot += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        }
        return tot / 20;
    };
    printf("idle link: memcpy64K %.1f us, zero-copy64K %.1f us\n", small_latency(false), small_latency(true));
    for (auto c : cfgs) {
        auto launch = [&] {
            if (c.unroll == 8) copy_k<8><<<c.grid, c.block, 0, a>>>((const uint4*)hd, (uint4*)d, n);
            else if (c.unroll == 4) copy_k<4><<<c.grid, c.block, 0, a>>>((const uint4*)hd, (uint4*)d, n);
            else copy_k<2><<<c.grid, c.block, 0, a>>>((const uint4*)hd, (uint4*)d, n);
        };
        launch();
        cudaStreamSynchronize(a);
        cudaEventRecord(e0, a);
        launch();
        cudaEventRecord(e1, a);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        launch();  // under load
        double lat_m = small_latency(false), lat_z = small_latency(true);
        cudaStreamSynchronize(a);
        printf("grid %3d block %3d unroll %d inflight %7d KB: %6.2f GB/s | under load: memcpy64K %7.1f us, zero-copy64K %7.1f us\n",
               c.grid, c.block, c.unroll, c.grid * c.block * c.unroll * 16 / 1024, bytes / (ms * 1e-3) / 1e9, lat_m, lat_z);
    }
    return 0;
}
