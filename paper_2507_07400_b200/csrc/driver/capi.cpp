// C-ABI over the control plane (include/kvflow_host.h): create a GPU engine shard, run
// the lockstep driver on it, and export its decision trace in the golden-trace format.
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "kvflow/scheduler.hpp"
#include "kvflow_host.h"

using namespace kvf;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const SimError& e) {
        return fail(static_cast<int>(e.code()) + 1, e.what());
    } catch (const std::exception& e) {
        return fail(KVF_E_INTERNAL, e.what());
    }
}

std::string jd(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

std::string js(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') {
            o += '\\';
            o += c;
        } else if (c == '\n') {
            o += "\\n";
        } else {
            o += c;
        }
    }
    return o + "\"";
}

CostModel cost_for(const kvfh_sim_config& c) {
    CostModel m;
    if (c.profile == 2) {  // the reference test suite's hand-calibrated cost (test_scheduler.cpp:23-36)
        m.name = "micro";
        m.prefill_a = 1e-5;
        m.prefill_b = 1e-3;
        m.decode_base = 1e-3;
        m.decode_per_seq = 1e-4;
        m.h2d_bandwidth = 2e9;
        m.d2h_bandwidth = 1e9;
        m.pcie_efficiency = 0.5;
        m.fixed_latency = 1e-3;
    } else {
        m = profile_by_name(c.profile == 1 ? "a10g-llama8b" : "h100-qwen32b");
    }
    m.bytes_per_token = c.bytes_per_token;
    return m;
}

}  // namespace

struct kvfh_sim {
    kvfh_sim_config cfg{};
    std::unique_ptr<Engine> engine;
    std::unique_ptr<Simulator> sim;
    SimResult result;
    std::string trace;
    uint64_t events = 0, audits = 0;
    double wall_s = 0;
    bool ran = false;
};

extern "C" {

const char* kvfh_last_error(void) { return g_err.c_str(); }

void kvfh_default_config(kvfh_sim_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->topology = 1;
    c->agents = 4;
    c->iterations = 10;
    c->warmup = 1;
    c->workflows = 1;
    c->fixed = 2048;
    c->dyn = 64;
    c->out = 64;
    c->vocab = 32000;
    c->policy = 2;
    c->max_running = 8;
    c->max_prefetch = 2;
    c->prefetch = -1;
    c->eviction = -1;
    c->overlap_fraction = 0.5;
    c->profile = 0;
    c->bytes_per_token = 131072;
    c->seed = 1;
    c->layers = 32;
    c->kv_heads_total = 8;
    c->kv_heads_local = 8;
    c->head_dim = 128;
    c->numa_node = -1;
    c->compute_scale = 1.0;
    c->compute_ctas = 128;
    c->d2h_coalesce = 1;
}

int kvfh_sim_create(const kvfh_sim_config* c, kvfh_sim** out) {
    if (!c || !out) return fail(KVF_E_INVALID_ARG, "null argument");
    *out = nullptr;
    auto s = std::make_unique<kvfh_sim>();
    s->cfg = *c;
    int rc = guarded([&] {
        WorkloadSpec w;
        w.topology = static_cast<Topology>(c->topology);
        w.num_agents = c->agents;
        w.iterations = c->iterations;
        w.warmup_rounds = c->warmup;
        w.num_workflows = c->workflows;
        w.fixed_len = c->fixed;
        w.dyn_len = c->dyn;
        w.out_len = c->out;
        w.shared_prefix_len = c->shared_prefix;
        w.vocab_size = c->vocab;
        SchedulerConfig sc;
        sc.policy = static_cast<Policy>(c->policy);
        sc.apply_policy_defaults();
        sc.max_running = c->max_running;
        sc.max_concurrent_prefetch = c->max_prefetch;
        if (c->prefetch >= 0) sc.prefetch_enabled = c->prefetch != 0;
        if (c->eviction >= 0) sc.eviction = c->eviction ? EvictionPolicy::WorkflowAware : EvictionPolicy::Lru;
        if (c->heuristic_boundary) sc.boundary_mode = BoundaryMode::Heuristic;
        sc.overlap_fraction = c->overlap_fraction;
        CostModel cost = cost_for(*c);
        if (c->bytes_per_token == 0) throw_error(ErrorCode::ConfigError, "bytes_per_token must be > 0");

        EngineOptions eo;
        eo.layers = c->layers;
        eo.kv_heads_total = c->kv_heads_total;
        eo.kv_heads_local = c->kv_heads_local;
        eo.head_offset = c->head_offset;
        eo.head_dim = c->head_dim;
        eo.device = c->device;
        eo.gpu_slots = c->gpu_cap / c->bytes_per_token;
        uint64_t host = c->host_slots;
        if (host == 0) {  // every token the run could ever back up (write-once host copies)
            w.validate();
            // the generator's own bound (PEER_STYLE lengths are drawn per agent from the seed)
            host = WorkloadController(w, c->seed).max_cached_tokens() + 1024;
            if (c->cpu_cap) host = std::min<uint64_t>(host, c->cpu_cap / c->bytes_per_token + 1024);
        }
        eo.host_slots = host;
        eo.pcie_mode = c->pcie_mode;
        eo.pcie_ctas = c->pcie_ctas;
        eo.numa_node = c->numa_node;
        s->engine = std::make_unique<Engine>(eo);
        s->sim = std::make_unique<Simulator>(cost, sc, w, c->gpu_cap, c->cpu_cap, c->seed, s->engine.get());
        s->sim->verify_loads = c->verify_loads != 0;
        if (c->timing == 1) s->sim->tier().set_timing(TransferTiming::Measured);
        if (c->clock == 1) {
            s->sim->clock = ClockMode::WallClock;
            s->sim->wall.compute_scale = c->compute_scale > 0 ? c->compute_scale : 1.0;
            s->sim->wall.compute_ctas = c->compute_ctas ? c->compute_ctas : 128;
        }
        s->sim->wall.prefetch_retry = c->prefetch_retry != 0;
        s->sim->wall.layered_gate = c->layered_gate != 0;
        if (c->d2h_unbatched) s->sim->tier().set_offload_batching(false);
        s->sim->tier().set_offload_coalescing(c->d2h_coalesce != 0 && !c->d2h_unbatched);
        // record every transition, tagged with the event index (same stream as ref_trace)
        auto prev = s->sim->tier().transition_observer;
        kvfh_sim* raw = s.get();
        s->sim->tier().transition_observer = [raw, prev](const CacheNode& n, NodeStatus from, NodeStatus to) {
            char b[160];
            std::snprintf(b, sizeof b, "{\"t\":\"tr\",\"ev\":%" PRIu64 ",\"node\":%" PRIu64 ",\"from\":%d,\"to\":%d,\"tokens\":%zu}\n",
                          raw->events, n.id, static_cast<int>(from), static_cast<int>(to), n.key.size());
            raw->trace += b;
            if (prev) prev(n, from, to);
        };
        const bool audit = c->audit != 0;
        s->sim->observe_ranks = audit;
        s->sim->post_event_hook = [raw, audit](VirtualTime) {
            if (audit) {
                raw->sim->tier().audit(raw->sim->cache());
                raw->audits++;
            }
            raw->events++;
        };
    });
    if (rc) return rc;
    *out = s.release();
    return 0;
}

int kvfh_sim_run(kvfh_sim* s) {
    if (!s || !s->sim) return fail(KVF_E_INVALID_ARG, "null sim");
    if (s->ran) return fail(KVF_E_INVALID_ARG, "simulation already ran");
    return guarded([&] {
        auto t0 = std::chrono::steady_clock::now();
        s->result = s->sim->run();
        s->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        s->ran = true;
        std::string& o = s->trace;
        char b[512];
        for (const TransferJob& j : s->result.transfers) {
            std::snprintf(b, sizeof b,
                          "{\"t\":\"job\",\"id\":%" PRIu64 ",\"dir\":%d,\"purpose\":%d,\"node\":%" PRIu64 ",\"bytes\":%" PRIu64
                          ",\"enqueue\":%s,\"start\":%s,\"complete\":%s,\"tc\":%u,\"tn\":%s,\"device_ms\":%s}\n",
                          j.id, static_cast<int>(j.dir), static_cast<int>(j.purpose), j.node_id, j.bytes,
                          jd(j.enqueue).c_str(), jd(j.start).c_str(), jd(j.complete).c_str(), j.target_agent.client,
                          js(j.target_agent.name).c_str(), jd(j.device_ms).c_str());
            o += b;
        }
        for (const RequestTrace& t : s->result.traces) {
            std::snprintf(b, sizeof b,
                          "{\"t\":\"req\",\"id\":%" PRIu64 ",\"client\":%u,\"agent\":%s,\"seq\":%" PRIu64 ",\"iter\":%u,"
                          "\"measured\":%d,\"arrival\":%s,\"prefill_start\":%s,\"first_token\":%s,\"done\":%s,"
                          "\"prompt\":%" PRIu64 ",\"matched\":%" PRIu64 ",\"loaded\":%" PRIu64 ",\"recomputed\":%" PRIu64
                          ",\"fixed\":%" PRIu64 ",\"output\":%" PRIu64 ",\"loaded_bytes\":%" PRIu64 ",\"stall\":%s%s}\n",
                          t.request_id, t.client, js(t.agent).c_str(), t.arrival_seq, t.iteration, t.measured ? 1 : 0,
                          jd(t.arrival).c_str(), jd(t.prefill_start).c_str(), jd(t.first_token).c_str(),
                          jd(t.done).c_str(), t.prompt_tokens, t.matched_tokens, t.loaded_tokens, t.recomputed_tokens,
                          t.fixed_tokens, t.output_tokens, t.loaded_bytes, jd(t.stall_seconds).c_str(),
                          t.load_wait_seconds < 0 ? "" : (",\"load_wait\":" + jd(t.load_wait_seconds)).c_str());
            o += b;
        }
        std::snprintf(b, sizeof b,
                      "{\"t\":\"res\",\"makespan\":%s,\"end_of_run\":%s,\"loaded_bytes\":%" PRIu64 ",\"offloaded_bytes\":%" PRIu64
                      ",\"wasted\":%" PRIu64 ",\"events\":%" PRIu64 ",\"nodes\":%zu,\"wall_s\":%s}\n",
                      jd(s->result.makespan).c_str(), jd(s->result.end_of_run).c_str(), s->result.loaded_bytes,
                      s->result.offloaded_bytes, s->result.wasted_prefetch_bytes, s->events, s->sim->cache().node_count(),
                      jd(s->wall_s).c_str());
        o += b;
        o += "{\"t\":\"dump\",\"text\":" + js(s->sim->cache().dump()) + "}\n";
    });
}

int kvfh_sim_result_get(const kvfh_sim* s, kvfh_sim_result* r) {
    if (!s || !r || !s->sim) return fail(KVF_E_INVALID_ARG, "null argument");
    return guarded([&] {
        std::memset(r, 0, sizeof(*r));
        r->makespan = s->result.makespan;
        r->end_of_run = s->result.end_of_run;
        r->loaded_bytes = s->result.loaded_bytes;
        r->offloaded_bytes = s->result.offloaded_bytes;
        r->wasted_prefetch_bytes = s->result.wasted_prefetch_bytes;
        r->events = s->events;
        r->nodes = s->sim->cache().node_count();
        r->requests = s->result.traces.size();
        r->wall_s = s->wall_s;
        const HotPathStats& h = s->sim->hot_path();
        r->arrivals = h.arrivals;
        r->decision_us_total = h.decision_us_total;
        r->decision_us_max = h.decision_us_max;
        r->prefetch_jobs = h.prefetch_jobs;
        r->reactive_jobs = h.reactive_jobs;
        r->offload_jobs = h.offload_jobs;
        r->prefetch_bytes = h.prefetch_bytes;
        r->reactive_bytes = h.reactive_bytes;
        r->offload_bytes = h.offload_bytes;
        r->prefetch_device_ms = h.prefetch_device_ms;
        r->reactive_device_ms = h.reactive_device_ms;
        r->offload_device_ms = h.offload_device_ms;
        r->fence_wait_us = h.fence_wait_us;
        const auto& d = s->sim->cache().decision_stats();
        r->priority_calls = d.priority_calls;
        r->evict_calls = d.evict_calls;
        r->priority_us = d.priority_us;
        r->evict_us = d.evict_us;
        const kvf_stats es = s->engine->stats();
        r->kernel_launches = es.kernel_launches;
        r->engine_decisions = es.decisions;
        r->engine_decision_kernel_ms = es.decision_kernel_ms;
        r->engine_decision_call_us = es.decision_call_us;
        r->resident_served = es.resident_served;
        r->oneshot_served = es.oneshot_served;
        r->resident_launches = es.resident_launches;
        r->mirror_records = es.mirror_records;
        r->k4_join_us = d.k4_join_us;
        r->k5_us = d.k5_us;
        r->apply_us = d.apply_us;
        r->issue_us = s->sim->tier().issue_us();
        r->decision_issue_us = h.decision_issue_us;
        r->priority_issued = d.priority_issued;
        r->verified_loads = s->sim->verified_loads;
        r->verify_failures = s->sim->verify_failures;
        r->audits = s->audits;
        r->d2h_batches = s->sim->tier().batched_launches();
        for (const RequestTrace& t : s->result.traces) {
            if (!t.measured) continue;
            r->measured_requests++;
            r->stall_total_s += t.stall_seconds;
            if (t.stall_seconds > 1e-12) r->stalled_requests++;
        }
    });
}

int kvfh_sim_trace(const kvfh_sim* s, char* buf, size_t cap, size_t* len) {
    if (!s || !len) return fail(KVF_E_INVALID_ARG, "null argument");
    *len = s->trace.size();
    if (buf && cap) std::memcpy(buf, s->trace.data(), std::min(cap, s->trace.size()));
    return 0;
}

int kvfh_sim_verify_resident(kvfh_sim* s, uint64_t* checked, uint64_t* mismatches) {
    if (!s || !s->sim || !checked || !mismatches) return fail(KVF_E_INVALID_ARG, "null argument");
    return guarded([&] {
        uint64_t k = 0, bad = 0;
        RadixCache& cache = s->sim->cache();
        Engine& e = *s->engine;
        e.sync();
        cache.for_each_node([&](const CacheNode& n) {
            const std::vector<uint64_t> cids = cache.node_cids(n);
            const uint64_t want = e.payload_checksum(cids);
            if (n.status == NodeStatus::InGpu) {
                ++k;
                if (e.checksum(KVF_TIER_DEVICE, n.dev_runs) != want) ++bad;
            }
            if (n.cpu_backed && n.status != NodeStatus::Offloading) {
                ++k;
                if (e.checksum(KVF_TIER_HOST, n.host_runs) != want) ++bad;
            }
        });
        *checked = k;
        *mismatches = bad;
    });
}

int kvfh_sim_destroy(kvfh_sim* s) {
    if (!s) return 0;
    s->sim.reset();  // returns every slot before the engine goes away
    s->engine.reset();
    delete s;
    return 0;
}

}  // extern "C"
