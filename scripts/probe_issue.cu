// Host cost of the CUDA calls a transfer issue makes (event records, stream waits, launches
// with small vs 1.5 KB parameter blocks).  nvcc -gencode arch=compute_100a,code=sm_100a -O2 probe_issue.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

struct Big { char b[1600]; };
struct Small { char b[64]; };
__global__ void kbig(const __grid_constant__ Big p) { if (p.b[0] == 42 && threadIdx.x == 999) printf("x"); }
__global__ void ksmall(const __grid_constant__ Small p) { if (p.b[0] == 42 && threadIdx.x == 999) printf("x"); }

template <typename F>
double us_per(int n, F f) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) f(i);
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / n;
}

int main() {
    cudaStream_t s, s2;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    const int N = 2000;
    std::vector<cudaEvent_t> tev(N), nev(N);
    for (int i = 0; i < N; ++i) {
        cudaEventCreate(&tev[i]);
        cudaEventCreateWithFlags(&nev[i], cudaEventDisableTiming);
    }
    Big big{};
    Small small{};
    for (int rep = 0; rep < 2; ++rep) {
        cudaDeviceSynchronize();
        double a = us_per(N, [&](int i) { cudaEventRecord(tev[i], s); });
        cudaDeviceSynchronize();
        double b = us_per(N, [&](int i) { cudaEventRecord(nev[i], s); });
        cudaDeviceSynchronize();
        double c = us_per(N, [&](int i) { cudaStreamWaitEvent(s2, nev[i], 0); });
        cudaDeviceSynchronize();
        double d = us_per(N, [&](int) { kbig<<<8, 256, 0, s>>>(big); });
        cudaDeviceSynchronize();
        double e = us_per(N, [&](int) { ksmall<<<8, 256, 0, s>>>(small); });
        cudaDeviceSynchronize();
        double f = us_per(N, [&](int i) {
            cudaEventRecord(tev[i], s);
            kbig<<<8, 256, 0, s>>>(big);
            cudaEventRecord(tev[(i + 1) % N], s);
        });
        cudaDeviceSynchronize();
        double g = us_per(200, [&](int i) {
            cudaEventRecord(tev[i], s);
            ksmall<<<8, 256, 0, s>>>(small);
            cudaEventRecord(nev[i], s);
            cudaEventSynchronize(nev[i]);
        });
        printf("record(timing) %.2f  record(no timing) %.2f  streamWaitEvent %.2f  launch(1.6KB) %.2f  launch(64B) %.2f  "
               "rec+big+rec %.2f  rec+small+rec+sync %.2f us\n", a, b, c, d, e, f, g);
    }
    return 0;
}
