// Probe: do TMA *tensor* loads (cp.async.bulk.tensor.2d) read mapped pinned host memory over
// PCIe faster than the SM load forms in probe_pcie.cu (all saturate at ~51.5 GB/s vs the
// copy engine's 55.6)?  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 probe_tma_h2d.cu -o probe_tma_h2d
// 1 GiB host -> HBM: each CTA streams 16 KiB boxes (2 KiB rows x 8) through a 4-stage smem ring
// -- TMA tensor load (mbarrier complete_tx) then a 1D bulk store smem -> HBM -- for several grid
// sizes and box shapes; then the same with 1D cp.async.bulk loads, and the copy engine.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int kStages = 4;

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <bool TENSOR>
__global__ void __launch_bounds__(32) tma_copy(const __grid_constant__ CUtensorMap tm, const char* src, char* dst,
                                               uint32_t box_rows, uint32_t row_bytes, uint32_t rows_total) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[kStages];
    const uint32_t box = box_rows * row_bytes;
    const uint32_t nbox = rows_total / box_rows;
    if (threadIdx.x != 0) return;
    for (int s = 0; s < kStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t phase[kStages] = {0, 0, 0, 0};
    auto load = [&](uint32_t b, int s) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(box) : "memory");
        if constexpr (TENSOR) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    sa(sm + s * box)),
                "l"(&tm), "r"(0), "r"(b * box_rows), "r"(sa(&bar[s]))
                : "memory");
        } else {
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             sa(sm + s * box)),
                         "l"(src + static_cast<uint64_t>(b) * box), "r"(box), "r"(sa(&bar[s]))
                         : "memory");
        }
    };
    // boxes blockIdx.x, blockIdx.x + grid, ...
    uint32_t next = blockIdx.x;
    int issued = 0;
    for (int s = 0; s < kStages && next < nbox; ++s, next += gridDim.x, ++issued) load(next, s);
    uint32_t b = blockIdx.x;
    for (int k = 0; b < nbox; ++k, b += gridDim.x) {
        const int s = k % kStages;
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                         : "=r"(done)
                         : "r"(sa(&bar[s])), "r"(phase[s])
                         : "memory");
        phase[s] ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + static_cast<uint64_t>(b) * box),
                     "r"(sa(sm + s * box)), "r"(box)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem slot free again
        if (next < nbox) {
            load(next, s);
            next += gridDim.x;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const size_t bytes = 1ull << 30;
    char *h = nullptr, *hd = nullptr, *d = nullptr;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hd), h, 0));
    CK(cudaMalloc(&d, bytes));
    for (size_t i = 0; i < bytes; i += 4096) h[i] = static_cast<char>(i >> 12);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    EncodeFn encode = reinterpret_cast<EncodeFn>(fn);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    struct Shape { uint32_t row_bytes, box_rows; };
    const Shape shapes[] = {{2048, 8}, {2048, 16}, {1024, 32}, {512, 64}};
    for (int tensor = 1; tensor >= 0; --tensor) {
        for (const Shape& sh : shapes) {
            if (!tensor && sh.row_bytes != 2048) continue;
            const uint32_t box = sh.row_bytes * sh.box_rows;
            const uint64_t rows = bytes / sh.row_bytes;
            CUtensorMap tm;
            cuuint64_t dims[2] = {sh.row_bytes / 8, rows};  // uint64 elements x rows
            cuuint64_t strides[1] = {sh.row_bytes};
            cuuint32_t boxd[2] = {sh.row_bytes / 8 > 256 ? 256u : sh.row_bytes / 8, sh.box_rows};
            cuuint32_t es[2] = {1, 1};
            if (boxd[0] * 8 != sh.row_bytes) continue;  // box inner dim is at most 256 elements
            CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, hd, dims, strides, boxd, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) {
                printf("encode failed (%d) for row %u box rows %u\n", static_cast<int>(r), sh.row_bytes, sh.box_rows);
                continue;
            }
            const size_t smem = static_cast<size_t>(kStages) * box;
            auto kern = tensor ? tma_copy<true> : tma_copy<false>;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            for (int grid : {16, 32, 64, 148, 296}) {
                float best = 1e9f;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(a);
                    kern<<<grid, 32, smem>>>(tm, hd, d, sh.box_rows, sh.row_bytes, static_cast<uint32_t>(rows));
                    cudaEventRecord(b);
                    CK(cudaEventSynchronize(b));
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                CK(cudaGetLastError());
                printf("%-12s row %5u B x %3u rows (%5u B box) grid %3d  %6.2f GB/s\n", tensor ? "tma tensor" : "tma 1d bulk",
                       sh.row_bytes, sh.box_rows, box, grid, bytes / (best * 1e-3) / 1e9);
            }
        }
    }
    float best = 1e9f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    printf("copy engine cudaMemcpyAsync                                  %6.2f GB/s\n", bytes / (best * 1e-3) / 1e9);
    // spot check the last tensor copy's bytes
    char* back = new char[4096];
    CK(cudaMemcpy(back, d + (bytes - 4096), 4096, cudaMemcpyDeviceToHost));
    printf("bytes %s\n", back[0] == h[bytes - 4096] ? "ok" : "MISMATCH");
    return 0;
}
