// Golden-trace extractor.  TEST INFRASTRUCTURE ONLY: links the UNMODIFIED reference
// library (oracle/_ref/libkvsim_ref.a, compiled in place from /root/reference/proj/src)
// and drives it through its public API, printing JSON lines that tests/golden/ holds.
//
//   ref_trace sim   key=value...   full Simulator run: every status
//                                   transition (radix_cache.cpp evict / tier_manager.cpp
//                                   set_status), every completed TransferJob
//                                   (tier_manager.cpp:95-124), every request trace row,
//                                   the run result and the final RadixCache::dump().
//   ref_trace evict key=value...   random trees snapshotted as SoA + one RadixCache::evict
//                                   call each (radix_cache.cpp:302-372): the K5 golden vectors.
//   ref_trace prio  key=value...   random trees + boundaries + StepMap ->
//                                   RadixCache::set_agent_priorities (radix_cache.cpp:266-285):
//                                   the K4 golden vectors.
//   ref_trace steps key=value...   random step graphs -> StepGraph::compute_steps
//                                   (step_graph.cpp:46-103) and next_step_agents (105-111).
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <random>
#include <string>
#include <unordered_map>
#include <vector>

#include "kvsim/cost_model.hpp"
#include "kvsim/radix_cache.hpp"
#include "kvsim/scheduler.hpp"
#include "kvsim/sim_engine.hpp"
#include "kvsim/step_graph.hpp"
#include "kvsim/tier_manager.hpp"
#include "kvsim/workload.hpp"

using namespace kvsim;

namespace {

std::map<std::string, std::string> parse_kv(int argc, char** argv, int first) {
    std::map<std::string, std::string> kv;
    for (int i = first; i < argc; ++i) {
        std::string a = argv[i];
        auto eq = a.find('=');
        if (eq == std::string::npos) {
            std::fprintf(stderr, "bad arg %s\n", a.c_str());
            std::exit(2);
        }
        kv[a.substr(0, eq)] = a.substr(eq + 1);
    }
    return kv;
}

std::string get(const std::map<std::string, std::string>& kv, const std::string& k, const std::string& dflt) {
    auto it = kv.find(k);
    return it == kv.end() ? dflt : it->second;
}
uint64_t getu(const std::map<std::string, std::string>& kv, const std::string& k, uint64_t dflt) {
    auto it = kv.find(k);
    return it == kv.end() ? dflt : std::strtoull(it->second.c_str(), nullptr, 10);
}
double getd(const std::map<std::string, std::string>& kv, const std::string& k, double dflt) {
    auto it = kv.find(k);
    return it == kv.end() ? dflt : std::strtod(it->second.c_str(), nullptr);
}

int status_code(NodeStatus s) {
    switch (s) {
        case NodeStatus::InGpu: return 0;
        case NodeStatus::BackupInCpu: return 1;
        case NodeStatus::Loading: return 2;
        case NodeStatus::Offloading: return 3;
    }
    return -1;
}

std::string jstr(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') { o += '\\'; o += c; }
        else if (c == '\n') o += "\\n";
        else o += c;
    }
    return o + "\"";
}

// %.17g round-trips every double exactly.
std::string jd(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

// ------------------------------------------------------------------ sim ----
int run_sim(const std::map<std::string, std::string>& kv) {
    WorkloadSpec w;
    w.topology = topology_from_name(get(kv, "topology", "CYCLIC"));
    w.num_agents = static_cast<uint32_t>(getu(kv, "agents", 4));
    w.iterations = static_cast<uint32_t>(getu(kv, "iterations", 10));
    w.warmup_rounds = static_cast<uint32_t>(getu(kv, "warmup", 1));
    w.num_workflows = static_cast<uint32_t>(getu(kv, "workflows", 1));
    w.fixed_len = getu(kv, "fixed", 2048);
    w.dyn_len = getu(kv, "dyn", 64);
    w.out_len = getu(kv, "out", 64);
    w.shared_prefix_len = getu(kv, "shared_prefix", 0);
    w.vocab_size = getu(kv, "vocab", 32000);

    CostModel cost;
    std::string prof = get(kv, "profile", "h100-qwen32b");
    if (prof == "micro") {
        cost.name = "micro";
        cost.prefill_a = 1e-5;
        cost.prefill_b = 1e-3;
        cost.decode_base = 1e-3;
        cost.decode_per_seq = 1e-4;
        cost.h2d_bandwidth = 2e9;
        cost.d2h_bandwidth = 1e9;
        cost.pcie_efficiency = 0.5;
        cost.fixed_latency = 1e-3;
    } else {
        cost = profile_by_name(prof);
    }
    cost.bytes_per_token = getu(kv, "bpt", 131072);

    SchedulerConfig sc;
    sc.policy = policy_from_name(get(kv, "policy", "KVFLOW"));
    sc.apply_policy_defaults();
    sc.max_running = static_cast<uint32_t>(getu(kv, "max_running", 8));
    sc.max_concurrent_prefetch = static_cast<uint32_t>(getu(kv, "max_prefetch", 2));
    if (kv.count("prefetch")) sc.prefetch_enabled = getu(kv, "prefetch", 1) != 0;
    if (kv.count("eviction")) sc.eviction = get(kv, "eviction", "") == "WA" ? EvictionPolicy::WorkflowAware : EvictionPolicy::Lru;
    if (get(kv, "boundary", "explicit") == "heuristic") sc.boundary_mode = BoundaryMode::Heuristic;
    sc.overlap_fraction = getd(kv, "overlap", 0.5);

    Bytes gpu_cap = getu(kv, "gpu_cap", 0);
    Bytes cpu_cap = getu(kv, "cpu_cap", 0);
    uint64_t seed = getu(kv, "seed", 1);

    Simulator sim(cost, sc, w, gpu_cap, cpu_cap, seed);
    uint64_t ev = 0;
    std::string args;
    for (const auto& [k, v] : kv) args += (args.empty() ? "" : ",") + jstr(k) + ":" + jstr(v);
    std::printf("{\"t\":\"cfg\",\"workload\":%s,\"policy\":%s,\"bpt\":%" PRIu64 ",\"gpu_cap\":%" PRIu64
                ",\"cpu_cap\":%" PRIu64 ",\"seed\":%" PRIu64 ",\"profile\":%s,\"args\":{%s}}\n",
                jstr(w.label()).c_str(), jstr(policy_name(sc.policy)).c_str(), cost.bytes_per_token, gpu_cap, cpu_cap,
                seed, jstr(prof).c_str(), args.c_str());
    auto prev = sim.tier().transition_observer;
    sim.tier().transition_observer = [&](const CacheNode& n, NodeStatus from, NodeStatus to) {
        std::printf("{\"t\":\"tr\",\"ev\":%" PRIu64 ",\"node\":%" PRIu64 ",\"from\":%d,\"to\":%d,\"tokens\":%zu}\n", ev,
                    n.id, status_code(from), status_code(to), n.key.size());
        if (prev) prev(n, from, to);
    };
    bool audit = getu(kv, "audit", 0) != 0;
    sim.post_event_hook = [&](VirtualTime) {
        if (audit) sim.tier().audit(sim.cache());
        ++ev;
    };
    auto t0 = std::chrono::steady_clock::now();
    SimResult r = sim.run();
    auto t1 = std::chrono::steady_clock::now();
    for (const TransferJob& j : r.transfers) {
        std::printf("{\"t\":\"job\",\"id\":%" PRIu64 ",\"dir\":%d,\"purpose\":%d,\"node\":%" PRIu64 ",\"bytes\":%" PRIu64
                    ",\"enqueue\":%s,\"start\":%s,\"complete\":%s,\"tc\":%u,\"tn\":%s}\n",
                    j.id, static_cast<int>(j.dir), static_cast<int>(j.purpose), j.node_id, j.bytes, jd(j.enqueue).c_str(),
                    jd(j.start).c_str(), jd(j.complete).c_str(), j.target_agent.client, jstr(j.target_agent.name).c_str());
    }
    for (const RequestTrace& t : r.traces) {
        std::printf("{\"t\":\"req\",\"id\":%" PRIu64 ",\"client\":%u,\"agent\":%s,\"seq\":%" PRIu64 ",\"iter\":%u,\"measured\":%d,"
                    "\"arrival\":%s,\"prefill_start\":%s,\"first_token\":%s,\"done\":%s,\"prompt\":%" PRIu64 ",\"matched\":%" PRIu64
                    ",\"loaded\":%" PRIu64 ",\"recomputed\":%" PRIu64 ",\"fixed\":%" PRIu64 ",\"output\":%" PRIu64
                    ",\"loaded_bytes\":%" PRIu64 ",\"stall\":%s}\n",
                    t.request_id, t.client, jstr(t.agent).c_str(), t.arrival_seq, t.iteration, t.measured ? 1 : 0,
                    jd(t.arrival).c_str(), jd(t.prefill_start).c_str(), jd(t.first_token).c_str(), jd(t.done).c_str(),
                    t.prompt_tokens, t.matched_tokens, t.loaded_tokens, t.recomputed_tokens, t.fixed_tokens,
                    t.output_tokens, t.loaded_bytes, jd(t.stall_seconds).c_str());
    }
    std::printf("{\"t\":\"res\",\"makespan\":%s,\"end_of_run\":%s,\"loaded_bytes\":%" PRIu64 ",\"offloaded_bytes\":%" PRIu64
                ",\"wasted\":%" PRIu64 ",\"events\":%" PRIu64 ",\"nodes\":%zu,\"wall_s\":%s}\n",
                jd(r.makespan).c_str(), jd(r.end_of_run).c_str(), r.loaded_bytes, r.offloaded_bytes,
                r.wasted_prefetch_bytes, ev, sim.cache().node_count(),
                jd(std::chrono::duration<double>(t1 - t0).count()).c_str());
    if (getu(kv, "dump", 1)) std::printf("{\"t\":\"dump\",\"text\":%s}\n", jstr(sim.cache().dump()).c_str());
    return 0;
}

// ------------------------------------------------------- random trees ----
CostModel flat_cost(Bytes bpt) {
    CostModel c;
    c.name = "flat";
    c.bytes_per_token = bpt;
    c.prefill_a = 1e-5;
    c.prefill_b = 1e-3;
    c.decode_base = 1e-3;
    c.decode_per_seq = 1e-4;
    c.h2d_bandwidth = 1e9;
    c.d2h_bandwidth = 1e9;
    c.pcie_efficiency = 1.0;
    c.fixed_latency = 0;
    return c;
}

TokenSeq rand_seq(std::mt19937_64& rng, const std::vector<TokenSeq>& prior, int vocab, int lo, int hi) {
    TokenSeq s;
    if (!prior.empty() && rng() % 3 != 0) {
        const TokenSeq& b = prior[rng() % prior.size()];
        size_t keep = 1 + rng() % b.size();
        s.assign(b.begin(), b.begin() + static_cast<long>(keep));
    }
    int n = lo + static_cast<int>(rng() % static_cast<uint64_t>(hi - lo + 1));
    for (int i = 0; i < n; ++i) s.push_back(static_cast<TokenId>(rng() % static_cast<uint64_t>(vocab)));
    return s;
}

struct Snapshot {
    std::vector<const CacheNode*> nodes;  // preorder, [0] = root
    std::unordered_map<const CacheNode*, int> index;
};

Snapshot snapshot(const RadixCache& cache) {
    Snapshot s;
    s.nodes.push_back(&cache.root());
    s.index[&cache.root()] = 0;
    cache.for_each_node([&](const CacheNode& n) {
        s.index[&n] = static_cast<int>(s.nodes.size());
        s.nodes.push_back(&n);
    });
    return s;
}

void print_tree(const RadixCache& cache, const Snapshot& s) {
    std::string par, st, lk, rk, tm, sq, id, tk, bk;
    for (size_t i = 0; i < s.nodes.size(); ++i) {
        const CacheNode* n = s.nodes[i];
        const char* sep = i ? "," : "";
        par += sep + std::to_string(n->parent ? s.index.at(n->parent) : -1);
        st += sep + std::to_string(status_code(n->status));
        lk += sep + std::to_string(n->lock_count);
        rk += sep + std::to_string(n->rank);
        tm += sep + jd(n->last_access.time);
        sq += sep + std::to_string(n->last_access.seq);
        id += sep + std::to_string(n->id);
        tk += sep + std::to_string(n->key.size());
        bk += sep + std::to_string(n->cpu_backed ? 1 : 0);
    }
    std::printf("\"bpt\":%" PRIu64 ",\"parent\":[%s],\"status\":[%s],\"lock\":[%s],\"rank\":[%s],\"time\":[%s],\"seq\":[%s],"
                "\"id\":[%s],\"tokens\":[%s],\"backed\":[%s]",
                cache.bytes_per_token(), par.c_str(), st.c_str(), lk.c_str(), rk.c_str(), tm.c_str(), sq.c_str(),
                id.c_str(), tk.c_str(), bk.c_str());
}

// Builds a random tree through the public API with mixed statuses, locks, backups and ranks.
struct Scenario {
    Bytes bpt;
    CostModel cost;
    EventQueue events;
    TierManager tier;
    RadixCache cache;
    std::vector<TokenSeq> seqs;
    Scenario(Bytes b, Bytes cpu_cap) : bpt(b), cost(flat_cost(b)), tier(Bytes(1) << 50, cpu_cap, cost, events), cache(b) {}
};

void grow(Scenario& sc, std::mt19937_64& rng, size_t target_nodes, int vocab, VirtualTime& now) {
    size_t guard = 0, count = sc.cache.node_count();
    while (count < target_nodes && guard++ < target_nodes * 8) {
        if (guard % 64 == 0) count = sc.cache.node_count();  // O(n): not every insert
        else count += 2;                                      // an insert adds <= 2 nodes
        TokenSeq s = rand_seq(rng, sc.seqs, vocab, 1, 12);
        InsertResult ins = sc.cache.insert(s, now += static_cast<double>(rng() % 3));  // equal times happen
        sc.tier.reserve_working(ins.new_bytes);
        sc.tier.convert_working(ins.new_bytes, ins.new_bytes);
        sc.seqs.push_back(std::move(s));
        if (rng() % 4 == 0) sc.cache.match_prefix(sc.seqs[rng() % sc.seqs.size()], now);
    }
}

std::vector<CacheNode*> all_nodes(RadixCache& cache) {
    std::vector<CacheNode*> v;
    cache.for_each_node([&](const CacheNode& n) { v.push_back(const_cast<CacheNode*>(&n)); });
    return v;
}

void randomize(Scenario& sc, std::mt19937_64& rng, VirtualTime& now, bool allow_tiers, bool inflight) {
    // boundaries + priorities
    size_t agents = 1 + rng() % 6;
    StepMap steps;
    for (size_t a = 0; a < agents; ++a) {
        AgentId id{static_cast<ClientId>(rng() % 2), "ag" + std::to_string(a)};
        const TokenSeq& s = sc.seqs[rng() % sc.seqs.size()];
        size_t flen = 1 + rng() % s.size();
        sc.cache.mark_fixed_boundary(id, s, flen);
        uint64_t r = rng() % 10;
        if (r < 7) steps[id] = static_cast<StepValue>(rng() % 6);
        else if (r == 7) steps[id] = kStepUnreachable;
    }
    sc.cache.set_agent_priorities(steps);
    if (allow_tiers) {
        auto nodes = all_nodes(sc.cache);
        // Offload + complete a subset (becomes BackupInCpu, cpu_backed)
        for (CacheNode* n : nodes) {
            if (rng() % 3 == 0 && n->status == NodeStatus::InGpu && n->lock_count == 0) {
                sc.tier.begin_offload(*n, now, sc.cache.node_bytes(*n));
                Event e = sc.events.pop();
                sc.tier.complete(e.id, e.time);
                now = std::max(now, e.time);
            }
        }
        // Load some back (InGpu + cpu_backed)
        for (CacheNode* n : nodes) {
            if (rng() % 2 == 0 && n->status == NodeStatus::BackupInCpu) {
                sc.tier.begin_load(*n, now, sc.cache.node_bytes(*n), TransferPurpose::Reactive);
                Event e = sc.events.pop();
                sc.tier.complete(e.id, e.time);
                now = std::max(now, e.time);
            }
        }
    }
    // locks
    {
        auto nodes = all_nodes(sc.cache);
        size_t nl = rng() % 3;
        for (size_t i = 0; i < nl && !nodes.empty(); ++i) sc.cache.lock_root_path(nodes[rng() % nodes.size()]);
    }
    if (allow_tiers && inflight) {
        auto nodes = all_nodes(sc.cache);
        for (CacheNode* n : nodes) {
            uint64_t r = rng() % 12;
            if (r == 0 && n->status == NodeStatus::InGpu && n->lock_count == 0)
                sc.tier.begin_offload(*n, now, sc.cache.node_bytes(*n));
            else if (r == 1 && n->status == NodeStatus::BackupInCpu)
                sc.tier.begin_load(*n, now, sc.cache.node_bytes(*n), TransferPurpose::Prefetch);
        }
    }
    // more touches after everything (recency shuffle)
    size_t touches = rng() % 4;
    for (size_t i = 0; i < touches; ++i) sc.cache.match_prefix(sc.seqs[rng() % sc.seqs.size()], now += 1.0);
}

int run_evict(const std::map<std::string, std::string>& kv) {
    std::mt19937_64 rng(getu(kv, "seed", 7));
    size_t cases = getu(kv, "cases", 100);
    size_t max_nodes = getu(kv, "max_nodes", 200);
    size_t min_nodes = getu(kv, "min_nodes", 1);
    int vocab = static_cast<int>(getu(kv, "vocab", 6));
    for (size_t c = 0; c < cases; ++c) {
        uint64_t kind = rng() % 10;
        bool discard = kind == 0;          // GPU-only tree, Discard mode
        bool bounded = kind == 1;          // bounded CPU store (may hit the reference defect)
        Bytes bpt = 1 + rng() % 64;
        Scenario sc(bpt, 0);
        VirtualTime now = 0;
        size_t target = min_nodes + rng() % (max_nodes - min_nodes + 1);
        grow(sc, rng, target, vocab, now);
        randomize(sc, rng, now, !discard, !discard && rng() % 2 == 0);
        Snapshot snap = snapshot(sc.cache);
        Bytes total = 0;
        sc.cache.for_each_node([&](const CacheNode& n) { total += sc.cache.node_bytes(n); });
        EvictRequest req;
        req.needed = rng() % 5 == 0 ? total + 1 : rng() % (total + 2);
        req.policy = rng() % 2 ? EvictionPolicy::WorkflowAware : EvictionPolicy::Lru;
        req.mode = discard ? TierMode::Discard : TierMode::Offload;
        if (rng() % 3 == 0) req.rank_floor_exclusive = static_cast<int64_t>(rng() % 5);
        Bytes cpu_cap = 0, cpu_used = sc.tier.cpu_used();
        if (bounded) {
            cpu_cap = cpu_used + rng() % (total / 2 + 2);
            // rebuild the TierManager's cap is not possible; emulate via a fresh manager is also
            // impossible (ledger state), so bounded cases use a second scenario below.
        }
        std::printf("{\"t\":\"evict\",\"case\":%zu,", c);
        print_tree(sc.cache, snap);
        std::printf(",\"needed\":%" PRIu64 ",\"policy\":%d,\"mode\":%d,\"has_floor\":%d,\"floor\":%" PRId64
                    ",\"cpu_used\":%" PRIu64 ",\"cpu_cap\":%" PRIu64,
                    req.needed, req.policy == EvictionPolicy::WorkflowAware ? 1 : 0, req.mode == TierMode::Offload ? 1 : 0,
                    req.rank_floor_exclusive ? 1 : 0, req.rank_floor_exclusive.value_or(0), cpu_used, sc.tier.cpu_capacity());
        (void)cpu_cap;
        try {
            auto t0 = std::chrono::steady_clock::now();
            EvictOutcome out = sc.cache.evict(req, sc.tier, now + 1.0);
            const double evict_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
            std::printf(",\"evict_us\":%.3f", evict_us);
            std::string v;
            for (size_t i = 0; i < out.victims.size(); ++i) {
                const auto& x = out.victims[i];
                v += (i ? "," : "") + std::string("[") + std::to_string(x.node_id) + "," + std::to_string(x.bytes) + "," +
                     (x.immediate ? "1" : "0") + "]";
            }
            std::printf(",\"victims\":[%s],\"immediate\":%" PRIu64 ",\"pending\":%" PRIu64 ",\"sufficient\":%d}\n", v.c_str(),
                        out.immediate_freed, out.pending_freed, out.sufficient ? 1 : 0);
            sc.tier.audit(sc.cache);
        } catch (const SimError& e) {
            std::printf(",\"error\":%d}\n", static_cast<int>(e.code()));
        }
    }
    return 0;
}

// Bounded-CPU evictions need the cap at TierManager construction: replay the same
// random construction with a capped manager.
int run_evict_bounded(const std::map<std::string, std::string>& kv) {
    std::mt19937_64 rng(getu(kv, "seed", 9));
    size_t cases = getu(kv, "cases", 50);
    size_t max_nodes = getu(kv, "max_nodes", 60);
    for (size_t c = 0; c < cases; ++c) {
        Bytes bpt = 1 + rng() % 16;
        Bytes cap = 1 + rng() % 4000;
        Scenario sc(bpt, cap);
        VirtualTime now = 0;
        grow(sc, rng, 2 + rng() % max_nodes, 5, now);
        // statuses without exceeding the cap: only offload while room remains
        size_t agents = 1 + rng() % 4;
        StepMap steps;
        for (size_t a = 0; a < agents; ++a) {
            AgentId id{0, "b" + std::to_string(a)};
            const TokenSeq& s = sc.seqs[rng() % sc.seqs.size()];
            sc.cache.mark_fixed_boundary(id, s, 1 + rng() % s.size());
            steps[id] = static_cast<StepValue>(rng() % 4);
        }
        sc.cache.set_agent_priorities(steps);
        for (CacheNode* n : all_nodes(sc.cache)) {
            if (rng() % 4 == 0 && n->status == NodeStatus::InGpu && sc.tier.cpu_has_room(sc.cache.node_bytes(*n))) {
                sc.tier.begin_offload(*n, now, sc.cache.node_bytes(*n));
                Event e = sc.events.pop();
                sc.tier.complete(e.id, e.time);
                now = std::max(now, e.time);
            }
        }
        Snapshot snap = snapshot(sc.cache);
        Bytes total = 0;
        sc.cache.for_each_node([&](const CacheNode& n) { total += sc.cache.node_bytes(n); });
        EvictRequest req;
        req.needed = rng() % (total + 2);
        req.policy = rng() % 2 ? EvictionPolicy::WorkflowAware : EvictionPolicy::Lru;
        req.mode = TierMode::Offload;
        std::printf("{\"t\":\"evict\",\"case\":%zu,", c);
        print_tree(sc.cache, snap);
        std::printf(",\"needed\":%" PRIu64 ",\"policy\":%d,\"mode\":1,\"has_floor\":0,\"floor\":0,\"cpu_used\":%" PRIu64
                    ",\"cpu_cap\":%" PRIu64,
                    req.needed, req.policy == EvictionPolicy::WorkflowAware ? 1 : 0, sc.tier.cpu_used(), sc.tier.cpu_capacity());
        try {
            auto t0 = std::chrono::steady_clock::now();
            EvictOutcome out = sc.cache.evict(req, sc.tier, now + 1.0);
            const double evict_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
            std::printf(",\"evict_us\":%.3f", evict_us);
            std::string v;
            for (size_t i = 0; i < out.victims.size(); ++i) {
                const auto& x = out.victims[i];
                v += (i ? "," : "") + std::string("[") + std::to_string(x.node_id) + "," + std::to_string(x.bytes) + "," +
                     (x.immediate ? "1" : "0") + "]";
            }
            std::printf(",\"victims\":[%s],\"immediate\":%" PRIu64 ",\"pending\":%" PRIu64 ",\"sufficient\":%d}\n", v.c_str(),
                        out.immediate_freed, out.pending_freed, out.sufficient ? 1 : 0);
        } catch (const SimError& e) {
            std::printf(",\"error\":%d}\n", static_cast<int>(e.code()));
        }
    }
    return 0;
}

int run_prio(const std::map<std::string, std::string>& kv) {
    std::mt19937_64 rng(getu(kv, "seed", 11));
    size_t cases = getu(kv, "cases", 100);
    size_t max_nodes = getu(kv, "max_nodes", 200);
    // optional (the default stream of random draws, and so every golden vector, is unchanged):
    // min_nodes / agents override the drawn sizes, time=1 adds the call's steady_clock time
    const size_t min_nodes = getu(kv, "min_nodes", 0), agents_fixed = getu(kv, "agents", 0);
    const bool timed = getu(kv, "time", 0) != 0;
    for (size_t c = 0; c < cases; ++c) {
        Scenario sc(16, 0);
        VirtualTime now = 0;
        grow(sc, rng, std::max<size_t>(min_nodes, 1 + rng() % max_nodes), static_cast<int>(3 + rng() % 6), now);
        size_t agents = 1 + rng() % 12;
        if (agents_fixed) agents = agents_fixed;
        std::vector<AgentId> ids;
        for (size_t a = 0; a < agents; ++a) {
            AgentId id{static_cast<ClientId>(rng() % 3), "p" + std::to_string(a)};
            const TokenSeq& s = sc.seqs[rng() % sc.seqs.size()];
            sc.cache.mark_fixed_boundary(id, s, 1 + rng() % s.size());
            ids.push_back(id);
        }
        StepMap steps;
        for (const AgentId& id : ids) {
            uint64_t r = rng() % 10;
            if (r < 7) steps[id] = static_cast<StepValue>(rng() % 9);
            else if (r == 7) steps[id] = kStepUnreachable;
        }
        const auto t0 = std::chrono::steady_clock::now();
        sc.cache.set_agent_priorities(steps);
        const double prio_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        Snapshot snap = snapshot(sc.cache);
        std::printf("{\"t\":\"prio\",\"case\":%zu,", c);
        if (timed) std::printf("\"prio_us\":%.3f,", prio_us);
        print_tree(sc.cache, snap);
        // boundary agents (node index, candidate rank) in map order of the agent id
        std::map<AgentId, int> bidx;
        for (const AgentId& id : ids) {
            CacheNode* b = sc.cache.boundary_node(id);
            if (b) bidx[id] = snap.index.at(b);
        }
        std::string bl;
        bool first = true;
        for (const auto& [id, idx] : bidx) {
            auto it = steps.find(id);
            int64_t cand = rank_for_step(it == steps.end() ? kStepUnreachable : it->second);
            bl += (first ? "" : ",") + std::string("[") + std::to_string(idx) + "," + std::to_string(cand) + "," +
                  std::to_string(id.client) + "," + jstr(id.name) + "," +
                  (it == steps.end() ? std::string("null") : std::to_string(it->second)) + "]";
            first = false;
        }
        std::printf(",\"boundaries\":[%s]}\n", bl.c_str());
    }
    return 0;
}

int run_steps(const std::map<std::string, std::string>& kv) {
    std::mt19937_64 rng(getu(kv, "seed", 13));
    size_t cases = getu(kv, "cases", 100);
    int max_n = static_cast<int>(getu(kv, "max_nodes", 16));
    for (size_t c = 0; c < cases; ++c) {
        int n = 2 + static_cast<int>(rng() % static_cast<uint64_t>(max_n - 1));
        std::vector<GraphNode> nodes;
        for (int i = 0; i < n; ++i)
            nodes.push_back({AgentId{static_cast<ClientId>(rng() % 2), "s" + std::to_string(i)},
                             rng() % 2 ? AggregationKind::MaxPlusOne : AggregationKind::MinPlusOne});
        std::vector<GraphEdge> edges;
        std::string es;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                if (i != j && rng() % 5 == 0) {
                    edges.push_back({nodes[i].id, nodes[j].id});
                    es += (es.empty() ? "" : ",") + std::string("[") + std::to_string(i) + "," + std::to_string(j) + "]";
                }
        StepGraph g = StepGraph::build(nodes, edges);
        std::vector<AgentId> active;
        std::string as;
        size_t na = 1 + rng() % 3;
        for (size_t a = 0; a < na; ++a) {
            int v = static_cast<int>(rng() % static_cast<uint64_t>(n));
            active.push_back(nodes[v].id);
            as += (as.empty() ? "" : ",") + std::to_string(v);
        }
        StepMap sm = g.compute_steps(active);
        std::string ns, ks, ss, fr;
        for (int i = 0; i < n; ++i) {
            ns += (i ? "," : "") + std::string("[") + std::to_string(nodes[i].id.client) + "," + jstr(nodes[i].id.name) + "]";
            ks += (i ? "," : "") + std::to_string(nodes[i].kind == AggregationKind::MinPlusOne ? 1 : 0);
            StepValue v = sm.at(nodes[i].id);
            ss += (i ? "," : "") + (v == kStepUnreachable ? std::string("-1") : std::to_string(v));
        }
        for (const AgentId& a : next_step_agents(sm)) fr += (fr.empty() ? "" : ",") + jstr(std::to_string(a.client) + "/" + a.name);
        std::printf("{\"t\":\"steps\",\"case\":%zu,\"nodes\":[%s],\"kinds\":[%s],\"edges\":[%s],\"active\":[%s],\"steps\":[%s],"
                    "\"frontier\":[%s]}\n",
                    c, ns.c_str(), ks.c_str(), es.c_str(), as.c_str(), ss.c_str(), fr.c_str());
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_trace sim|evict|evict_bounded|prio|steps key=value...\n");
        return 2;
    }
    std::string mode = argv[1];
    auto kv = parse_kv(argc, argv, 2);
    try {
        if (mode == "sim") return run_sim(kv);
        if (mode == "evict") return run_evict(kv);
        if (mode == "evict_bounded") return run_evict_bounded(kv);
        if (mode == "prio") return run_prio(kv);
        if (mode == "steps") return run_steps(kv);
    } catch (const SimError& e) {
        std::fprintf(stderr, "SimError %d: %s\n", static_cast<int>(e.code()), e.what());
        return 3;
    }
    std::fprintf(stderr, "unknown mode %s\n", mode.c_str());
    return 2;
}
