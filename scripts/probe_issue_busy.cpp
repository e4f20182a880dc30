// Host cost of a K1 issue through the C-ABI with the H2D stream idle vs busy (a 1 GiB K1 in
// flight on it), and of a K2 issue beside that K1.  Diagnostics for the transfer-issue share
// of the decision time.
//   g++ -O2 -std=c++17 -Iinclude scripts/probe_issue_busy.cpp -Lpaper_2507_07400_b200 -lkvflow \
//       -Wl,-rpath,paper_2507_07400_b200 -o scripts/probe_issue_busy
#include <chrono>
#include <cstdio>

#include "kvflow.h"

int main() {
    kvf_geometry g{32, 8, 8, 0, 128, 2};  // Llama-3-8B KV: 128 KiB per token
    kvf_engine_config c{0, 16384, 16384, 0, KVF_COPY_SM_VEC, 0, -1};
    kvf_engine* e = nullptr;
    if (kvf_engine_create(&g, &c, &e)) { std::printf("create: %s\n", kvf_last_error()); return 1; }
    kvf_engine_set_job_timing(e, KVF_JOB_TIMING_STAMPS);
    kvf_run big_h{0, 8192}, big_d{0, 8192}, h{9000, 16}, d{9000, 16};
    for (int busy = 0; busy < 2; ++busy) {
        double k1 = 0, k2 = 0;
        const int N = 200;
        for (int i = 0; i < N; ++i) {
            if (busy && i % 50 == 0) {
                kvf_h2d_gather(e, 1, &big_h, 1, &big_d, 1);
            }
            auto t0 = std::chrono::steady_clock::now();
            kvf_h2d_gather(e, 1000 + i, &h, 1, &d, 1);
            auto t1 = std::chrono::steady_clock::now();
            uint64_t job = 5000 + i;
            uint32_t one = 1;
            kvf_d2h_scatter_batch(e, 1, &job, &d, &one, &h, &one);
            auto t2 = std::chrono::steady_clock::now();
            k1 += std::chrono::duration<double, std::micro>(t1 - t0).count();
            k2 += std::chrono::duration<double, std::micro>(t2 - t1).count();
            kvf_job_wait(e, 1000 + i);
            kvf_job_release(e, 1000 + i);
            kvf_job_wait(e, job);
            kvf_job_release(e, job);
            if (busy && i % 50 == 49) { kvf_job_wait(e, 1); kvf_job_release(e, 1); }
        }
        std::printf("%s: K1 issue %.2f us, K2 issue %.2f us\n", busy ? "busy (1 GiB K1 in flight)" : "idle", k1 / N, k2 / N);
    }
    kvf_engine_destroy(e);
    return 0;
}
