/* kvflow_host.h -- C-ABI over the C++ control plane (libkvflow_host.so).
 *
 * Drives the lockstep workflow driver (kvf::Simulator, include/kvflow/scheduler.hpp) on a
 * GPU engine from C / Python / bench.py.  It stands where the reference's experiment
 * runner calls Simulator::run (proj/src/experiment.cpp:44-54, proj/src/scheduler.cpp:80-148),
 * and emits the same trace records the golden extractor (oracle/ref_trace.cpp) prints for
 * the reference, so parity is a line-by-line comparison.
 *
 * Same conventions as kvflow.h: extern "C", no exceptions, int status (kvsim ErrorCode + 1,
 * engine codes >= 100), kvfh_last_error() for the text.
 */
#ifndef KVFLOW_HOST_H
#define KVFLOW_HOST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kvfh_sim kvfh_sim;

typedef struct {
    /* workload (WorkloadSpec, proj/include/kvsim/workload.hpp:31-46) */
    int32_t topology; /* 0 SEQUENTIAL 1 CYCLIC 2 BRANCH_MAX 3 BRANCH_MIN 4 PEER_STYLE */
    uint32_t agents, iterations, warmup, workflows;
    uint64_t fixed, dyn, out, shared_prefix, vocab;
    /* scheduling (SchedulerConfig, proj/include/kvsim/scheduler.hpp:36-51) */
    int32_t policy; /* 0 LRU_GPU_ONLY 1 LRU_REACTIVE_HICACHE 2 KVFLOW */
    uint32_t max_running, max_prefetch;
    int32_t prefetch;  /* -1 policy default, else 0/1 */
    int32_t eviction;  /* -1 policy default, 0 LRU, 1 WORKFLOW_AWARE */
    int32_t heuristic_boundary;
    double overlap_fraction;
    /* timing profile for virtual time: 0 h100-qwen32b 1 a10g-llama8b 2 micro (test cost) */
    int32_t profile;
    uint64_t bytes_per_token; /* ledger bytes per token on this shard (= engine token bytes) */
    uint64_t gpu_cap, cpu_cap, seed;
    /* data plane: KV geometry of this shard and engine options */
    uint32_t layers, kv_heads_total, kv_heads_local, head_offset, head_dim;
    int32_t device;
    uint64_t host_slots; /* 0: sized from the workload's upper bound */
    uint32_t pcie_mode, pcie_ctas;
    int32_t numa_node;
    int32_t audit;        /* TierManager::audit after every event */
    int32_t verify_loads; /* GPU checksum of every H2D-loaded node vs its host copy */
    int32_t timing;       /* 0 modeled (lockstep parity), 1 measured (hardware in the loop) */
    /* clock: 0 virtual (event-driven on modeled/measured times), 1 wall clock -- transfers and
     * model compute (spin kernels on the engine's compute stream, cost-model durations scaled
     * by compute_scale) complete when their CUDA events fire; stalls are real seconds. */
    int32_t clock;
    double compute_scale;   /* wall clock: emulated compute = cost-model time * scale (0 -> 1) */
    uint32_t compute_ctas;  /* wall clock: CTAs the compute emulation spins on (0 -> 128) */
    int32_t prefetch_retry; /* re-run the step-1 prefetch whenever a transfer lands */
    int32_t layered_gate;   /* wall clock: HiCache-gated prefills consume layer-pipelined loads */
    int32_t d2h_unbatched;  /* 1: one K2 launch per write-back instead of one per evict call */
    int32_t d2h_coalesce;   /* 1 (default): write-backs booked by consecutive evict calls leave
                               together at the next fence; 0: one K2 launch per evict call */
} kvfh_sim_config;

typedef struct {
    double makespan, end_of_run;
    uint64_t loaded_bytes, offloaded_bytes, wasted_prefetch_bytes;
    uint64_t events, nodes, requests;
    double wall_s;            /* host wall time of run() */
    /* hot path (HotPathStats) */
    uint64_t arrivals;
    double decision_us_total, decision_us_max;
    uint64_t prefetch_jobs, reactive_jobs, offload_jobs;
    uint64_t prefetch_bytes, reactive_bytes, offload_bytes;
    double prefetch_device_ms, reactive_device_ms, offload_device_ms, fence_wait_us;
    uint64_t priority_calls, evict_calls;
    double priority_us, evict_us;
    uint64_t kernel_launches;
    uint64_t verified_loads, verify_failures;
    uint64_t audits;
    uint64_t d2h_batches;     /* K2 batch launches (one per evict call with write-backs) */
    /* stalls (RequestTrace::stall_seconds, virtual seconds) over measured requests */
    double stall_total_s;
    uint64_t stalled_requests, measured_requests;
    /* decision calls as the engine saw them (kvf_get_stats): in-kernel time (globaltimer) and
       C-ABI call time, K4 + K5 together -- the rest of priority_us / evict_us is host packing */
    uint64_t engine_decisions;
    double engine_decision_kernel_ms, engine_decision_call_us;
    /* HBM tree mirror (kvf_tree): who served the decisions, records shipped */
    uint64_t resident_served, oneshot_served, resident_launches, mirror_records;
    /* host-time breakdown (us): waiting for queued K4 results, K5 calls, applying victims
       (ledger + K2 issue), issuing K1/K2 on the engine */
    double k4_join_us, k5_us, apply_us, issue_us;
    /* the part of decision_us_total spent issuing K1 / K2 (launch + stop event) inside arrivals:
       real byte movement the reference's ledger-only decisions do not have */
    double decision_issue_us;
    /* K4 calls that ran on the GPU (priority_calls minus the ones a newer call replaced unread) */
    uint64_t priority_issued;
} kvfh_sim_result;

const char* kvfh_last_error(void);
void kvfh_default_config(kvfh_sim_config* c);
int kvfh_sim_create(const kvfh_sim_config* c, kvfh_sim** out);
int kvfh_sim_run(kvfh_sim* s);
int kvfh_sim_result_get(const kvfh_sim* s, kvfh_sim_result* out);
/* JSON-lines trace ("tr", "job", "req", "res", "dump" records; oracle/ref_trace.cpp format).
 * Copies min(cap, len) bytes; *len gets the full length. */
int kvfh_sim_trace(const kvfh_sim* s, char* buf, size_t cap, size_t* len);
/* Expected-vs-device payload check of every node resident in HBM after the run:
 * GPU checksum of its slots vs GPU checksum of a fresh fill of its content ids. */
int kvfh_sim_verify_resident(kvfh_sim* s, uint64_t* nodes_checked, uint64_t* mismatches);
int kvfh_sim_destroy(kvfh_sim* s);

#ifdef __cplusplus
}
#endif
#endif /* KVFLOW_HOST_H */
