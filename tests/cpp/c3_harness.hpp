// C3 harness (BASELINE configs[2]): a 16-agent Agent Step Graph with conditional branches
// (MIN+1 joins) and a synchronisation barrier (MAX+1 join), mixed 1k-8k fixed prompts behind
// a 256-token system prompt shared by every agent.  The reference's workload generator
// cannot express this graph (branch topologies are capped at 4 agents,
// proj/src/workload.cpp:35-36), so this driver calls the cache-manager components directly
// -- StepGraph, RadixCache, TierManager, EventQueue -- and restates the scheduler's
// make_room (proj/src/scheduler.cpp:396-405) and maybe_prefetch (418-435) on their public
// API.  The same source compiles against the reference (KV_NS = kvsim, oracle/ref_c3.cpp,
// golden generation) and against this repo (KV_NS = kvf, tests/cpp/c3_kvf.cpp, GPU
// engine attached), so the two traces must match record for record.
//
// Sequential execution (one agent request at a time), transfers drained after each
// request; deterministic in the seed.
#pragma once

#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <optional>
#include <random>
#include <string>
#include <vector>

#ifndef KV_NS
#error "define KV_NS (kvsim or kvf) before including c3_harness.hpp"
#endif

namespace c3 {

namespace K = KV_NS;

struct Agent {
    K::AgentId id;
    K::TokenSeq fixed;
};

struct Result {
    std::string trace;  // JSON lines: tr / job / req / dump
};

inline std::vector<K::GraphNode> nodes_of(const std::vector<Agent>& ag) {
    std::vector<K::GraphNode> v;
    for (size_t i = 0; i < ag.size(); ++i) {
        // joins after a conditional branch wait for ANY predecessor; the barrier for ALL
        const bool min_join = i == 4 || i == 14;
        v.push_back({ag[i].id, min_join ? K::AggregationKind::MinPlusOne : K::AggregationKind::MaxPlusOne});
    }
    return v;
}

inline std::vector<K::GraphEdge> edges_of(const std::vector<Agent>& ag) {
    std::vector<std::pair<int, int>> e = {{0, 1}, {0, 2}, {0, 3}, {1, 4}, {2, 4}, {3, 4}};   // plan -> 3-way branch -> MIN join
    for (int w = 5; w <= 10; ++w) {
        e.push_back({4, w});   // fan-out to six workers
        e.push_back({w, 11});  // barrier: MAX join over all six
    }
    e.push_back({11, 12});
    e.push_back({11, 13});
    e.push_back({12, 14});  // 2-way conditional -> MIN join
    e.push_back({13, 14});
    e.push_back({14, 15});
    e.push_back({15, 0});  // iterate
    std::vector<K::GraphEdge> out;
    for (auto [a, b] : e) out.push_back({ag[a].id, ag[b].id});
    return out;
}

template <class Tier, class Cache, class Events, class Cost>
class Driver {
public:
    Driver(Tier& tier, Cache& cache, Events& ev, const Cost& cost, uint64_t seed)
        : tier_(tier), cache_(cache), ev_(ev), cost_(cost), rng_(seed) {
        const size_t lens[] = {1024, 2048, 4096, 8192};
        K::TokenSeq system(256);
        for (auto& t : system) t = static_cast<K::TokenId>(rng_() % 32000);
        for (int i = 0; i < 16; ++i) {
            Agent a;
            char name[8];
            std::snprintf(name, sizeof name, "c3_%02d", i);
            a.id = K::AgentId{0, name};
            a.fixed = system;
            a.fixed.push_back(static_cast<K::TokenId>(32000 + i));  // agent-private tail starts here
            const size_t len = lens[rng_() % 4];
            while (a.fixed.size() < len) a.fixed.push_back(static_cast<K::TokenId>(rng_() % 32000));
            agents_.push_back(std::move(a));
        }
        graph_ = std::make_unique<K::StepGraph>(K::StepGraph::build(nodes_of(agents_), edges_of(agents_)));
        tier_.transition_observer = [this](const K::CacheNode& n, K::NodeStatus from, K::NodeStatus to) {
            char b[160];
            std::snprintf(b, sizeof b, "{\"t\":\"tr\",\"req\":%zu,\"node\":%" PRIu64 ",\"from\":%d,\"to\":%d,\"tokens\":%zu}\n",
                          req_, n.id, static_cast<int>(from), static_cast<int>(to), n.key.size());
            out_.trace += b;
        };
    }

    Result run(int iterations) {
        for (int it = 0; it < iterations; ++it) {
            std::vector<int> order = {0, 1 + static_cast<int>(rng_() % 3), 4, 5, 6, 7, 8, 9, 10, 11,
                                      12 + static_cast<int>(rng_() % 2), 14, 15};
            for (int a : order) request(a);
        }
        drain();
        for (const auto& j : tier_.completed_jobs()) {
            char b[256];
            std::snprintf(b, sizeof b,
                          "{\"t\":\"job\",\"id\":%" PRIu64 ",\"dir\":%d,\"purpose\":%d,\"node\":%" PRIu64 ",\"bytes\":%" PRIu64
                          ",\"enqueue\":%.17g,\"start\":%.17g,\"complete\":%.17g}\n",
                          j.id, static_cast<int>(j.dir), static_cast<int>(j.purpose), j.node_id, j.bytes, j.enqueue,
                          j.start, j.complete);
            out_.trace += b;
        }
        std::string d = cache_.dump(), esc;
        for (char ch : d) esc += ch == '\n' ? std::string("\\n") : std::string(1, ch);
        out_.trace += "{\"t\":\"dump\",\"text\":\"" + esc + "\"}\n";
        return out_;
    }

private:
    void drain() {
        while (!ev_.empty()) {
            auto e = ev_.pop();
            now_ = std::max(now_, e.time);
            tier_.complete(e.id, e.time);
        }
    }

    bool make_room(K::Bytes bytes, std::optional<int64_t> floor) {  // scheduler.cpp:396-405
        if (tier_.free_bytes() >= bytes) return true;
        K::EvictRequest req;
        req.needed = bytes - tier_.free_bytes();
        req.policy = K::EvictionPolicy::WorkflowAware;
        req.mode = K::TierMode::Offload;
        req.rank_floor_exclusive = floor;
        cache_.evict(req, tier_, now_);
        return tier_.free_bytes() >= bytes;
    }

    void prefetch(const K::StepMap& steps) {  // scheduler.cpp:418-435
        for (const K::AgentId& agent : K::next_step_agents(steps)) {
            K::CacheNode* b = cache_.boundary_node(agent);
            if (!b) continue;
            std::vector<K::CacheNode*> path;
            for (K::CacheNode* n = b; n && !n->is_root(); n = n->parent) path.push_back(n);
            std::reverse(path.begin(), path.end());
            for (K::CacheNode* n : path) {
                if (n->status != K::NodeStatus::BackupInCpu) continue;
                if (tier_.inflight_loads(K::TransferPurpose::Prefetch) >= 2) return;
                const K::Bytes bytes = cache_.node_bytes(*n);
                if (!make_room(bytes, K::rank_for_step(1))) return;
                tier_.begin_load(*n, now_, bytes, K::TransferPurpose::Prefetch, agent);
            }
        }
    }

    void request(int a) {
        ++req_;
        const Agent& ag = agents_[a];
        K::TokenSeq prompt = ag.fixed;
        for (int i = 0; i < 64; ++i) prompt.push_back(static_cast<K::TokenId>(rng_() % 32000));
        K::TokenSeq output;
        for (int i = 0; i < 32; ++i) output.push_back(static_cast<K::TokenId>(rng_() % 32000));
        const K::StepMap steps = graph_->compute_steps({ag.id});
        cache_.set_agent_priorities(steps);
        // reactive loads of any host-resident part of the prefix, then the fence
        {
            K::MatchResult m = cache_.peek_prefix(prompt);
            std::vector<K::CacheNode*> host;
            K::Bytes total = 0;
            for (K::CacheNode* n : m.needed_nodes())
                if (n->status == K::NodeStatus::BackupInCpu) {
                    host.push_back(n);
                    total += cache_.node_bytes(*n);
                }
            if (!host.empty() && make_room(total, std::nullopt))
                for (K::CacheNode* n : host) tier_.begin_load(*n, now_, cache_.node_bytes(*n), K::TransferPurpose::Reactive, ag.id);
            drain();
        }
        K::MatchResult m = cache_.match_prefix(prompt, now_);
        std::vector<K::CacheNode*> needed = m.needed_nodes();
        K::CacheNode* deepest = needed.empty() ? nullptr : needed.back();
        cache_.lock_root_path(deepest);
        const uint64_t uncached = prompt.size() - m.matched_tokens;
        const K::Bytes working = cost_.kv_bytes(uncached + output.size());
        // offloads started by make_room free their bytes only on completion: evict, fence,
        // repeat while that makes progress
        for (K::Bytes before = 0; tier_.free_bytes() < working && tier_.free_bytes() != before;) {
            before = tier_.free_bytes();
            make_room(working, std::nullopt);
            drain();
        }
        if (tier_.free_bytes() < working) {
            char b[160];
            std::snprintf(b, sizeof b, "{\"t\":\"skip\",\"req\":%zu,\"free\":%" PRIu64 ",\"working\":%" PRIu64 "}\n", req_,
                          static_cast<uint64_t>(tier_.free_bytes()), static_cast<uint64_t>(working));
            out_.trace += b;
            cache_.unlock_root_path(deepest);
            return;
        }
        tier_.reserve_working(working);
        now_ += cost_.prefill_time(uncached) + cost_.decode_iter_time(1) * static_cast<double>(output.size());
        cache_.unlock_root_path(deepest);
        K::TokenSeq full = prompt;
        full.insert(full.end(), output.begin(), output.end());
        K::InsertResult ins = cache_.insert(full, now_);
        tier_.convert_working(working, ins.new_bytes);
        cache_.mark_fixed_boundary(ag.id, full, ag.fixed.size());
        char b[200];
        std::snprintf(b, sizeof b, "{\"t\":\"req\",\"req\":%zu,\"agent\":\"%s\",\"matched\":%zu,\"prompt\":%zu,\"now\":%.17g}\n", req_,
                      ag.id.name.c_str(), m.matched_tokens, prompt.size(), now_);
        out_.trace += b;
        prefetch(graph_->compute_steps({ag.id}));
    }

    Tier& tier_;
    Cache& cache_;
    Events& ev_;
    const Cost& cost_;
    std::mt19937_64 rng_;
    std::vector<Agent> agents_;
    std::unique_ptr<K::StepGraph> graph_;
    double now_ = 0;
    size_t req_ = 0;
    Result out_;
};

inline K::CostModel c3_cost(K::Bytes bpt) {
    K::CostModel c = K::profile_by_name("h100-qwen32b");
    c.bytes_per_token = bpt;
    return c;
}

}  // namespace c3
