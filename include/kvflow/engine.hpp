// kvflow host API -- RAII C++ handle over the CUDA engine's C-ABI (include/kvflow.h).
// The host control plane (RadixCache, TierManager) talks to the GPU only through this.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "kvflow.h"
#include "kvflow/errors.hpp"

namespace kvf {

using Run = kvf_run;
using RunList = std::vector<Run>;

inline uint64_t run_tokens(const RunList& r) {
    uint64_t t = 0;
    for (const Run& x : r) t += x.len;
    return t;
}

// Split `runs` after `tokens` tokens: returns the head, leaves the tail in `runs`.
RunList split_runs(RunList& runs, uint64_t tokens);

// Maps an engine status onto the reference's ErrorCode convention (code = status - 1).
[[noreturn]] void throw_engine(int status, const std::string& what);

class Engine;

// Drop-in for code written against the engine-less reference API (kvsim): a process-wide
// factory that the RadixCache / TierManager / Simulator constructors ask for an engine when
// none is passed (same bytes_per_token => the same engine, so a cache and a tier manager built
// separately share it).  Unset -- the default -- nothing changes: no engine, no GPU path.
using EngineFactory = std::function<Engine*(uint64_t bytes_per_token)>;
void set_default_engine_factory(EngineFactory factory);
Engine* default_engine(uint64_t bytes_per_token);  // nullptr when no factory is installed

struct EngineOptions {
    uint32_t layers = 32, kv_heads_total = 8, kv_heads_local = 8, head_offset = 0, head_dim = 128;
    int device = 0;
    uint64_t gpu_slots = 0, host_slots = 0;
    uint32_t pcie_mode = KVF_COPY_SM_VEC, pcie_ctas = 0, hbm_ctas = 0;
    int numa_node = -1;
};

class Engine {
public:
    explicit Engine(const EngineOptions& opt);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    kvf_engine* raw() const { return e_; }
    uint64_t token_bytes() const { return token_bytes_; }
    const EngineOptions& options() const { return opt_; }

    RunList alloc(int tier, uint64_t tokens);
    void free(int tier, const RunList& runs);
    uint64_t free_tokens(int tier) const;

    void h2d(uint64_t job, const RunList& host, const RunList& dev);
    // layer-pipelined K1 with engine-owned per-layer landed counters
    void h2d_layered(uint64_t job, const RunList& host, const RunList& dev);
    void d2h(uint64_t job, const RunList& dev, const RunList& host);
    // one K2 launch for several nodes (each job keeps its id and events)
    void d2h_batch(const std::vector<uint64_t>& jobs, const std::vector<const RunList*>& dev,
                   const std::vector<const RunList*>& host);
    bool query(uint64_t job);
    void wait(uint64_t job);
    float elapsed_ms(uint64_t job);
    void release(uint64_t job);
    void sync();

    // emulated model compute on the engine's compute stream (wall-clock driver)
    void compute_begin(uint64_t job);
    void compute_end(uint64_t job);
    void compute_wait_job(uint64_t transfer_job);
    void compute_wait_job_layer(uint64_t transfer_job, uint32_t layer);
    void compute_spin(uint64_t ns, uint32_t ctas);

    void fill(int tier, const RunList& runs, const std::vector<uint64_t>& cids);
    uint64_t checksum(int tier, const RunList& runs);
    uint64_t payload_checksum(const std::vector<uint64_t>& cids);

    std::vector<int64_t> priorities(const std::vector<int32_t>& parent, const std::vector<int32_t>& bidx,
                                    const std::vector<int64_t>& cand);
    void victims(const kvf_tree_view& tree, const kvf_evict_request& req, std::vector<int32_t>& idx,
                 std::vector<uint8_t>& action, uint64_t& immediate, uint64_t& pending);
    kvf_stats stats() const;
    // KVF_JOB_TIMING_EVENTS / KVF_JOB_TIMING_STAMPS for K1 / K2 jobs (kvflow.h)
    void set_job_timing(uint32_t mode);

private:
    kvf_engine* e_ = nullptr;
    EngineOptions opt_;
    uint64_t token_bytes_ = 0;
};

}  // namespace kvf
