// Host cost of one K1 / K2 issue through the engine C-ABI (kvf_h2d_gather, kvf_d2h_scatter_batch)
// with stamp-timed jobs, vs a bare kernel launch (scripts/probe_issue.cu).  Diagnostics.
//   g++ -O2 -std=c++17 -Iinclude scripts/probe_issue_engine.cpp -Lpaper_2507_07400_b200 -lkvflow \
//       -Wl,-rpath,paper_2507_07400_b200 -o scripts/probe_issue_engine
#include <chrono>
#include <cstdio>
#include <vector>

#include "kvflow.h"

int main() {
    kvf_geometry g{32, 8, 1, 7, 128, 2};
    kvf_engine_config c{0, 4096, 4096, 0, KVF_COPY_SM_VEC, 0, -1};
    kvf_engine* e = nullptr;
    if (kvf_engine_create(&g, &c, &e)) { std::printf("create: %s\n", kvf_last_error()); return 1; }
    kvf_engine_set_job_timing(e, KVF_JOB_TIMING_STAMPS);
    kvf_run h{0, 16}, d{0, 16};
    const int N = 3000;
    for (int mode = 0; mode < 2; ++mode) {
        double issue = 0;
        for (int i = 0; i < N; ++i) {
            const uint64_t job = 1000 + i;
            auto t0 = std::chrono::steady_clock::now();
            int rc;
            if (mode == 0) {
                rc = kvf_h2d_gather(e, job, &h, 1, &d, 1);
            } else {
                uint32_t one = 1;
                rc = kvf_d2h_scatter_batch(e, 1, &job, &d, &one, &h, &one);
            }
            issue += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
            if (rc) { std::printf("rc %d %s\n", rc, kvf_last_error()); return 1; }
            kvf_job_release(e, job);
        }
        std::printf("%s issue: %.2f us per call\n", mode ? "K2 batch(1)" : "K1 gather", issue / N);
    }
    kvf_engine_destroy(e);
    return 0;
}
