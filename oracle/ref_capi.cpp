// C-ABI shim over the UNMODIFIED reference library (compiled in place from
// /root/reference/proj/src into oracle/_ref/).  TEST/BASELINE INFRASTRUCTURE ONLY:
// bench.py --impl reference and the cpu_baseline leg call it to time the reference's
// own decision path (Simulator::run, scheduler.cpp:80-148) on the box's host cores.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>

#include "kvsim/cost_model.hpp"
#include "kvsim/scheduler.hpp"
#include "kvsim/workload.hpp"

using namespace kvsim;

extern "C" {

struct ref_sim_cfg {
    uint32_t agents, iterations, warmup, workflows;
    uint64_t fixed, dyn, out, shared_prefix, vocab;
    uint64_t bytes_per_token, gpu_cap, cpu_cap, seed;
    uint32_t max_running, max_prefetch;
    int32_t topology;  // 0 SEQ 1 CYCLIC 2 BRANCH_MAX 3 BRANCH_MIN 4 PEER
    int32_t policy;    // 0 LRU_GPU_ONLY 1 HICACHE 2 KVFLOW
};

struct ref_job {
    uint64_t id, node_id, bytes;
    int32_t dir, purpose;
    double enqueue, start, complete;
};

// Returns 0 on success; wall_s = host seconds spent inside Simulator::run().
int ref_sim_run(const ref_sim_cfg* c, ref_job* jobs, uint64_t max_jobs, uint64_t* n_jobs, double* wall_s,
                uint64_t* events, char* err, uint64_t err_len) {
    try {
        WorkloadSpec w;
        static const Topology topo[] = {Topology::Sequential, Topology::Cyclic, Topology::BranchMax,
                                        Topology::BranchMin, Topology::PeerStyle};
        w.topology = topo[c->topology];
        w.num_agents = c->agents;
        w.iterations = c->iterations;
        w.warmup_rounds = c->warmup;
        w.num_workflows = c->workflows;
        w.fixed_len = c->fixed;
        w.dyn_len = c->dyn;
        w.out_len = c->out;
        w.shared_prefix_len = c->shared_prefix;
        w.vocab_size = c->vocab;
        CostModel cost = profile_by_name("h100-qwen32b");
        cost.bytes_per_token = c->bytes_per_token;
        SchedulerConfig sc;
        static const Policy pol[] = {Policy::LruGpuOnly, Policy::LruReactiveHicache, Policy::Kvflow};
        sc.policy = pol[c->policy];
        sc.apply_policy_defaults();
        sc.max_running = c->max_running;
        sc.max_concurrent_prefetch = c->max_prefetch;
        Simulator sim(cost, sc, w, c->gpu_cap, c->cpu_cap, c->seed);
        uint64_t ev = 0;
        sim.post_event_hook = [&](VirtualTime) { ++ev; };
        auto t0 = std::chrono::steady_clock::now();
        SimResult r = sim.run();
        auto t1 = std::chrono::steady_clock::now();
        *wall_s = std::chrono::duration<double>(t1 - t0).count();
        *events = ev;
        *n_jobs = r.transfers.size();
        for (uint64_t i = 0; i < r.transfers.size() && i < max_jobs; ++i) {
            const TransferJob& j = r.transfers[i];
            jobs[i] = ref_job{j.id, j.node_id, j.bytes, static_cast<int32_t>(j.dir), static_cast<int32_t>(j.purpose),
                              j.enqueue, j.start, j.complete};
        }
        return 0;
    } catch (const std::exception& e) {
        if (err && err_len) {
            std::strncpy(err, e.what(), err_len - 1);
            err[err_len - 1] = 0;
        }
        return 1;
    }
}

}  // extern "C"
