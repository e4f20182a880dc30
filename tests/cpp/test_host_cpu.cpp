// CPU unit tests of the C++ control plane (no GPU): step graph, cost model, event queue,
// radix tree structure, the tier ledger (bare ledger: no engine attached), workload
// generator.  Cases restate the reference's own suites (proj/tests/test_step_graph.cpp,
// test_cost_model.cpp, test_radix_cache.cpp, test_tier_manager.cpp, test_workload.cpp)
// against the kvf API.  GPU-backed cases live in test_host_gpu.cpp.
#include <algorithm>
#include <deque>
#include <map>
#include <memory>
#include <numeric>
#include <random>

#include "kvflow/cost_model.hpp"
#include "kvflow/radix_cache.hpp"
#include "kvflow/sim_engine.hpp"
#include "kvflow/step_graph.hpp"
#include "kvflow/tier_manager.hpp"
#include "kvflow/workload.hpp"
#include "tinytest.hpp"

using namespace kvf;

namespace {

AgentId ag(const std::string& n, ClientId c = 0) { return AgentId{c, n}; }
GraphNode gnode(const std::string& n, AggregationKind k = AggregationKind::MaxPlusOne) { return {ag(n), k}; }

StepGraph chain(int n) {
    std::vector<GraphNode> ns;
    std::vector<GraphEdge> es;
    for (int i = 0; i < n; ++i) ns.push_back(gnode("n" + std::to_string(i)));
    for (int i = 0; i + 1 < n; ++i) es.push_back({ns[i].id, ns[i + 1].id});
    return StepGraph::build(ns, es);
}

constexpr Bytes kBpt = 16;

CostModel flat_cost() {  // h2d 1 GB/s, d2h 0.5 GB/s effective, 1 ms setup (test_tier_manager.cpp:19-32)
    CostModel c;
    c.name = "test";
    c.bytes_per_token = kBpt;
    c.prefill_a = 1e-4;
    c.prefill_b = 1e-3;
    c.decode_base = 1e-3;
    c.decode_per_seq = 1e-4;
    c.h2d_bandwidth = 2e9;
    c.d2h_bandwidth = 1e9;
    c.pcie_efficiency = 0.5;
    c.fixed_latency = 1e-3;
    return c;
}

TokenSeq iota_seq(TokenId base, size_t n) {
    TokenSeq s(n);
    std::iota(s.begin(), s.end(), base);
    return s;
}

CacheNode* resident(RadixCache& cache, TierManager& tier, TokenId base, size_t n, VirtualTime now) {
    InsertResult ins = cache.insert(iota_seq(base, n), now);
    tier.reserve_working(ins.new_bytes);
    tier.convert_working(ins.new_bytes, ins.new_bytes);
    return ins.path.back();
}

void backed(RadixCache& cache, TierManager& tier, EventQueue& ev, CacheNode* n, VirtualTime now) {
    tier.begin_offload(*n, now, cache.node_bytes(*n));
    Event e = ev.pop();
    REQUIRE(e.kind == EventKind::TransferDone);
    tier.complete(e.id, e.time);
    REQUIRE(n->status == NodeStatus::BackupInCpu);
}

const CacheNode* by_key(const RadixCache& cache, const TokenSeq& key) {
    const CacheNode* f = nullptr;
    cache.for_each_node([&](const CacheNode& n) {
        if (n.key == key) f = &n;
    });
    return f;
}

}  // namespace

// ---------------------------------------------------------------- step graph ------------
TEST("step graph: four-agent ring counts forward from the active agent") {
    std::vector<GraphNode> ns = {gnode("planner"), gnode("executor"), gnode("expresser"), gnode("reviewer")};
    std::vector<GraphEdge> es = {{ag("planner"), ag("executor")}, {ag("executor"), ag("expresser")},
                                 {ag("expresser"), ag("reviewer")}, {ag("reviewer"), ag("planner")}};
    StepGraph g = StepGraph::build(ns, es);
    StepMap s = g.compute_steps({ag("executor")});
    CHECK(s.at(ag("executor")) == 0);
    CHECK(s.at(ag("expresser")) == 1);
    CHECK(s.at(ag("reviewer")) == 2);
    CHECK(s.at(ag("planner")) == 3);
    StepMap s2 = g.compute_steps({ag("executor"), ag("reviewer")});
    CHECK(s2.at(ag("reviewer")) == 0);
    CHECK(s2.at(ag("planner")) == 1);
    CHECK(s2.at(ag("expresser")) == 1);
}

TEST("step graph: chains, MIN vs MAX, islands, frontier order") {
    StepMap s = chain(10).compute_steps({ag("n5")});
    for (int i = 0; i < 5; ++i) CHECK(s.at(ag("n" + std::to_string(i))) == kStepUnreachable);
    for (int i = 5; i < 10; ++i) CHECK(s.at(ag("n" + std::to_string(i))) == i - 5);
    std::vector<GraphEdge> es = {{ag("a"), ag("b")}, {ag("b"), ag("c")}, {ag("c"), ag("d")}, {ag("a"), ag("d")}};
    CHECK(StepGraph::build({gnode("a"), gnode("b"), gnode("c"), gnode("d")}, es).compute_steps({ag("a")}).at(ag("d")) == 3);
    CHECK(StepGraph::build({gnode("a"), gnode("b"), gnode("c"), gnode("d", AggregationKind::MinPlusOne)}, es)
              .compute_steps({ag("a")})
              .at(ag("d")) == 1);
    StepMap m;
    m[ag("zeta")] = 1;
    m[ag("alpha")] = 1;
    m[ag("mid")] = 2;
    m[ag("gone")] = kStepUnreachable;
    m[ag("x", 1)] = 1;
    std::vector<AgentId> f = next_step_agents(m);
    REQUIRE(f.size() == 3);
    CHECK(f[0].name == "alpha");
    CHECK(f[1].name == "zeta");
    CHECK(f[2].client == 1);
}

TEST("step graph: malformed graphs and active sets are rejected") {
    EXPECT_CODE(StepGraph::build({gnode("a"), gnode("a")}, {}), ErrorCode::DuplicateAgent);
    EXPECT_CODE(StepGraph::build({gnode("a"), gnode("b")}, {{ag("a"), ag("a")}}), ErrorCode::SelfLoop);
    EXPECT_CODE(StepGraph::build({gnode("a"), gnode("b")}, {{ag("a"), ag("ghost")}}), ErrorCode::UnknownAgent);
    StepGraph g = StepGraph::build({gnode("a"), gnode("b")}, {{ag("a"), ag("b")}, {ag("a"), ag("b")}});
    CHECK(g.preds_of(1).size() == 1);
    EXPECT_CODE(chain(3).compute_steps({}), ErrorCode::EmptyActiveSet);
    EXPECT_CODE(chain(3).compute_steps({ag("ghost")}), ErrorCode::UnknownAgent);
}

TEST("step graph: random DAGs agree with a topological-order DP; rings with the closed form") {
    std::mt19937_64 rng(97);
    for (int tc = 0; tc < 300; ++tc) {
        const int n = 2 + static_cast<int>(rng() % 19);
        std::vector<GraphNode> ns;
        std::vector<AggregationKind> kinds;
        for (int i = 0; i < n; ++i) {
            kinds.push_back(rng() % 2 ? AggregationKind::MinPlusOne : AggregationKind::MaxPlusOne);
            ns.push_back({ag("v" + std::to_string(i)), kinds.back()});
        }
        std::vector<GraphEdge> es;
        std::vector<std::vector<int>> preds(n);
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j)
                if (rng() % 4 == 0) {
                    es.push_back({ns[i].id, ns[j].id});
                    preds[j].push_back(i);
                }
        std::vector<bool> act(n, false);
        std::vector<AgentId> active;
        for (int k = 0; k < 1 + static_cast<int>(rng() % 3); ++k) {
            int v = static_cast<int>(rng() % n);
            if (!act[v]) {
                act[v] = true;
                active.push_back(ns[v].id);
            }
        }
        StepMap got = StepGraph::build(ns, es).compute_steps(active);
        std::vector<StepValue> want(n, kStepUnreachable);  // nodes are already in topological order
        for (int v = 0; v < n; ++v) {
            if (act[v]) {
                want[v] = 0;
                continue;
            }
            bool any = false;
            StepValue best = 0;
            for (int p : preds[v]) {
                if (want[p] == kStepUnreachable) continue;
                best = !any ? want[p] : (kinds[v] == AggregationKind::MinPlusOne ? std::min(best, want[p]) : std::max(best, want[p]));
                any = true;
            }
            want[v] = any ? best + 1 : kStepUnreachable;
        }
        for (int v = 0; v < n; ++v) CHECK(got.at(ns[v].id) == want[v]);
    }
    for (int tc = 0; tc < 100; ++tc) {
        const int n = 2 + static_cast<int>(rng() % 15);
        std::vector<GraphNode> ns;
        std::vector<GraphEdge> es;
        for (int i = 0; i < n; ++i) ns.push_back({ag("r" + std::to_string(i)), rng() % 2 ? AggregationKind::MinPlusOne : AggregationKind::MaxPlusOne});
        for (int i = 0; i < n; ++i) es.push_back({ns[i].id, ns[(i + 1) % n].id});
        const int a = static_cast<int>(rng() % n);
        StepMap got = StepGraph::build(ns, es).compute_steps({ns[a].id});
        for (int v = 0; v < n; ++v) CHECK(got.at(ns[v].id) == ((v - a) % n + n) % n);
    }
}

// ---------------------------------------------------------------- cost model ------------
TEST("cost model: geometry, frozen profiles, affine formulas, validation") {
    CHECK(kv_bytes_per_token(32, 8, 128, 2) == 131072);
    CHECK(kv_bytes_per_token(80, 8, 128, 2) == 327680);
    CostModel a = profile_by_name("a10g-llama8b");
    CHECK(a.bytes_per_token == 131072);
    CHECK(a.kv_bytes(8192) == 1073741824ull);
    CHECK_APPROX(a.prefill_a, 400e-6);
    CHECK_APPROX(a.decode_iter_time(8), 28e-3);
    CostModel h = profile_by_name("h100-qwen32b");
    CHECK(h.bytes_per_token == 262144);
    CHECK_APPROX(h.h2d_bandwidth, 64e9);
    CHECK((profile_names() == std::vector<std::string>{"a10g-llama8b", "h100-qwen32b"}));
    EXPECT_CODE(profile_by_name("tpu-v9"), ErrorCode::ConfigError);
    CHECK_APPROX(a.h2d_seconds(a.kv_bytes(8192)), static_cast<double>(1073741824ull) / (2e9 * 0.6) + 50e-6);
    for (const std::string& n : profile_names()) {
        CostModel m = profile_by_name(n);
        for (uint64_t t : {512u, 1024u, 4096u, 8192u}) CHECK(m.h2d_seconds(m.kv_bytes(t)) < m.prefill_time(t) - m.prefill_b);
    }
    CostModel bad = a;
    bad.pcie_efficiency = 1.5;
    EXPECT_CODE(bad.validate(), ErrorCode::ConfigError);
    bad = a;
    bad.bytes_per_token = 0;
    EXPECT_CODE(bad.validate(), ErrorCode::ConfigError);
}

TEST("event queue: (time, push order) total order") {
    EventQueue q;
    q.push(2.0, EventKind::Arrival, 1);
    q.push(1.0, EventKind::PrefillDone, 2);
    q.push(1.0, EventKind::DecodeIter, 3);
    q.push(0.5, EventKind::TransferDone, 4);
    std::vector<uint64_t> ids;
    while (!q.empty()) ids.push_back(q.pop().id);
    CHECK((ids == std::vector<uint64_t>{4, 2, 3, 1}));
    ComputeClock c;
    c.occupy(0, 2);
    CHECK(!c.idle(1.0));
    CHECK_APPROX(c.busy_integral(1.0), 1.0);
    CHECK(c.idle(2.0));
    // wall clock: a booked occupation that really ended early / late
    ComputeClock w;
    w.occupy(0, 2);
    w.finish_at(1.5);
    CHECK(w.idle(1.5));
    CHECK_APPROX(w.busy_integral(3.0), 1.5);
    w.occupy(3.0, 4.0);
    w.finish_at(4.5);
    CHECK(!w.idle(4.2));
    CHECK_APPROX(w.busy_integral(5.0), 3.0);
}

// ------------------------------------------------------------- radix tree ---------------
TEST("radix: matches agree with a one-token-per-node trie over random workloads") {
    std::mt19937_64 rng(20260822);
    for (int w = 0; w < 300; ++w) {
        RadixCache cache(16);
        std::map<TokenSeq, bool> prefixes;  // every cached prefix
        std::vector<TokenSeq> used;
        VirtualTime now = 0;
        auto longest = [&](const TokenSeq& s) {
            size_t k = 0;
            while (k < s.size() && prefixes.count(TokenSeq(s.begin(), s.begin() + static_cast<long>(k) + 1))) ++k;
            return k;
        };
        for (int op = 0; op < 30; ++op) {
            TokenSeq s;
            if (!used.empty() && rng() % 2) {
                const TokenSeq& b = used[rng() % used.size()];
                s.assign(b.begin(), b.begin() + static_cast<long>(1 + rng() % b.size()));
            }
            for (int i = 0, e = 1 + static_cast<int>(rng() % 10); i < e; ++i) s.push_back(static_cast<TokenId>(rng() % 6));
            now += 1;
            if (rng() % 10 < 7) {
                cache.insert(s, now);
                for (size_t k = 1; k <= s.size(); ++k) prefixes[TokenSeq(s.begin(), s.begin() + static_cast<long>(k))] = true;
            } else {
                MatchResult m = cache.match_prefix(s, now);
                CHECK(m.matched_tokens == longest(s));
                size_t cov = m.partial_len;
                for (CacheNode* n : m.path) cov += n->key.size();
                CHECK(cov == m.matched_tokens);
                CHECK(cache.peek_prefix(s).matched_tokens == m.matched_tokens);
            }
            used.push_back(s);
        }
        size_t tokens = 0;
        cache.for_each_node([&](const CacheNode& n) { tokens += n.key.size(); });
        CHECK(tokens == prefixes.size());
    }
}

TEST("radix: split conserves tokens and charges only fresh suffixes") {
    RadixCache cache(kBpt);
    InsertResult a = cache.insert({1, 2, 3, 10, 11, 12}, 1.0);
    CHECK(a.new_nodes == 1);
    CHECK(a.new_bytes == 6 * kBpt);
    InsertResult b = cache.insert({1, 2, 3, 20, 21}, 2.0);
    CHECK(b.new_nodes == 1);
    CHECK(b.new_bytes == 2 * kBpt);
    CHECK(cache.node_count() == 3);
    CHECK(by_key(cache, {1, 2, 3}) != nullptr);
    CHECK(by_key(cache, {10, 11, 12}) != nullptr);
    size_t path = 0;
    for (const CacheNode* n : b.path) path += n->key.size();
    CHECK(path == 5);
    // content ids survive the split: the tail's prefix is the upper half's end
    const CacheNode* up = by_key(cache, {1, 2, 3});
    const CacheNode* tail = by_key(cache, {10, 11, 12});
    CHECK(tail->prefix_cid == up->end_cid);
    CHECK(cache.node_cids(*tail).back() == tail->end_cid);
}

TEST("radix: partial match does not split; insert does") {
    RadixCache cache(kBpt);
    cache.insert({1, 2, 3, 4}, 1.0);
    MatchResult m = cache.match_prefix({1, 2, 9}, 2.0);
    CHECK(m.matched_tokens == 2);
    CHECK(m.path.empty());
    REQUIRE(m.partial != nullptr);
    CHECK(m.partial_len == 2);
    CHECK(cache.node_count() == 1);
    CHECK(m.needed_nodes().size() == 1);
    cache.insert({1, 2, 9}, 3.0);
    CHECK(cache.node_count() == 3);
    CHECK(by_key(cache, {9}) != nullptr);
}

TEST("radix: locks survive splits; unlock balances and underflow is an error") {
    RadixCache cache(kBpt);
    CacheNode* deep = cache.insert({1, 2, 3, 4}, 1.0).path.back();
    cache.lock_root_path(deep);
    cache.insert({1, 2, 9}, 2.0);
    CHECK(deep->key == (TokenSeq{3, 4}));
    CHECK(deep->lock_count == 1);
    CHECK(by_key(cache, {1, 2})->lock_count == 1);
    CHECK(by_key(cache, {9})->lock_count == 0);
    cache.unlock_root_path(deep);
    cache.for_each_node([&](const CacheNode& n) { CHECK(n.lock_count == 0); });
    EXPECT_CODE(cache.unlock_root_path(deep), ErrorCode::UnderflowUnlock);
}

TEST("radix: fixed boundaries land on node ends") {
    AgentId w{0, "writer"};
    {
        RadixCache c(kBpt);
        c.insert({1, 2, 3, 4, 5}, 1.0);
        CacheNode* b = c.mark_fixed_boundary(w, {1, 2, 3, 4, 5}, 2);
        CHECK(b->key == (TokenSeq{1, 2}));
        CHECK(c.node_count() == 2);
        CHECK(c.boundary_node(w) == b);
        CacheNode* b2 = c.mark_fixed_boundary(w, {1, 2, 3, 4, 5}, 4);
        CHECK(b2->key == (TokenSeq{3, 4}));
        CHECK(b->fixed_boundary_for.empty());
        CHECK(c.boundary_node(w) == b2);
    }
    {
        RadixCache c(kBpt);
        c.insert({1, 2, 3}, 1.0);
        c.insert({1, 2, 3, 4, 5}, 2.0);
        CHECK(c.mark_fixed_boundary(w, {1, 2, 3, 4, 5}, 3)->key == (TokenSeq{1, 2, 3}));
        CHECK(c.node_count() == 2);
        EXPECT_CODE(c.mark_fixed_boundary(w, {1, 2, 3, 9, 9}, 5), ErrorCode::BoundaryBeyondCache);
        EXPECT_CODE(c.mark_fixed_boundary(w, {1, 2, 3}, 0), ErrorCode::BoundaryBeyondCache);
    }
    {
        RadixCache c(kBpt);
        c.insert({1, 2, 3, 4}, 1.0);
        EXPECT_CODE(c.mark_fixed_boundary(w, {1, 2, 9, 9}, 4), ErrorCode::BoundaryBeyondCache);
    }
}

TEST("radix: fixed-length heuristic takes the window minimum") {
    CHECK(update_fixed_heuristic({512, 520, 512, 518}, 4) == 512);
    CHECK(update_fixed_heuristic({8, 9}, 4) == 8);
    CHECK(update_fixed_heuristic({100, 512, 520, 518}, 3) == 512);
    EXPECT_CODE(update_fixed_heuristic({512}, 4), ErrorCode::InsufficientHistory);
    EXPECT_CODE(update_fixed_heuristic({512, 513}, 0), ErrorCode::ConfigError);
}

TEST("radix: decisions have no CPU path -- priorities and eviction need the GPU engine") {
    RadixCache cache(kBpt);
    cache.insert({1, 2, 3}, 1.0);
    EXPECT_CODE(cache.set_agent_priorities(StepMap{}), ErrorCode::NoDevice);
    EventQueue ev;
    TierManager tier(1 << 20, 0, flat_cost(), ev);
    EXPECT_CODE(cache.evict(EvictRequest{1, EvictionPolicy::Lru, TierMode::Discard, {}}, tier, 2.0), ErrorCode::NoDevice);
    CHECK(cache.dump() == "root\n  [1..+2] IN_GPU SUFFIX lock=0\n");
}

// ------------------------------------------------------------- tier ledger ---------------
TEST("tier ledger: timing follows bandwidth, efficiency and setup latency") {
    EventQueue ev;
    TierManager tier(4u << 20, 0, flat_cost(), ev);
    RadixCache cache(kBpt);
    CacheNode* n = resident(cache, tier, 1, 62500, 0.0);  // 1 MB
    const Bytes mb = 1000000;
    uint64_t off = tier.begin_offload(*n, 1.0, mb);
    Event e = ev.pop();
    CHECK(e.id == off);
    CHECK_APPROX(e.time, 1.003);
    const TransferJob& d2h = tier.complete(e.id, e.time);
    CHECK_APPROX(d2h.start, 1.0);
    CHECK(tier.cpu_used() == mb);
    tier.begin_load(*n, 2.0, mb, TransferPurpose::Reactive);
    REQUIRE(tier.load_completion_for_node(n->id).has_value());
    CHECK_APPROX(*tier.load_completion_for_node(n->id), 2.002);
    Event l = ev.pop();
    tier.complete(l.id, l.time);
    CHECK(n->status == NodeStatus::InGpu);
    CHECK(n->cpu_backed);
    CHECK(!tier.load_completion_for_node(n->id).has_value());
    tier.audit(cache);
}

TEST("tier ledger: measured / wall-clock timing need the GPU engine (no CPU path)") {
    EventQueue ev;
    TierManager tier(4u << 20, 0, flat_cost(), ev);
    EXPECT_CODE(tier.set_timing(TransferTiming::Measured), ErrorCode::NoDevice);
    EXPECT_CODE(tier.set_timing(TransferTiming::WallClock), ErrorCode::NoDevice);
    CHECK(tier.timing() == TransferTiming::Modeled);
    CHECK(tier.inflight_ids().empty());
}

TEST("tier ledger: per-direction FIFO channels, full duplex across directions") {
    EventQueue ev;
    TierManager tier(8u << 20, 0, flat_cost(), ev);
    RadixCache cache(kBpt);
    CacheNode* a = resident(cache, tier, 1, 62500, 0.0);
    CacheNode* b = resident(cache, tier, 100000, 31250, 0.0);
    CacheNode* c = resident(cache, tier, 200000, 62500, 0.0);
    backed(cache, tier, ev, a, 0.0);
    backed(cache, tier, ev, b, 0.01);
    tier.begin_load(*a, 1.0, 1000000, TransferPurpose::Reactive);
    tier.begin_load(*b, 1.0, 500000, TransferPurpose::Reactive);
    tier.begin_offload(*c, 1.0, 1000000);
    CHECK_APPROX(tier.channel_busy_until(TransferDirection::HostToDevice), 1.0035);
    CHECK_APPROX(tier.channel_busy_until(TransferDirection::DeviceToHost), 1.003);
    Event e1 = ev.pop();
    const TransferJob& j1 = tier.complete(e1.id, e1.time);
    CHECK(j1.node_id == a->id);
    Event e2 = ev.pop();
    CHECK_APPROX(e2.time, 1.003);  // the D2H finishes between the two loads
    tier.complete(e2.id, e2.time);
    Event e3 = ev.pop();
    const TransferJob& j3 = tier.complete(e3.id, e3.time);
    CHECK(j3.node_id == b->id);
    CHECK_APPROX(j3.start, 1.002);
    tier.audit(cache);
}

TEST("tier ledger: illegal moves are rejected with the ledger untouched") {
    EventQueue ev;
    TierManager tier(8u << 20, 0, flat_cost(), ev);
    RadixCache cache(kBpt);
    CacheNode* g = resident(cache, tier, 1, 100, 0.0);
    CacheNode* h = resident(cache, tier, 1000, 100, 0.0);
    backed(cache, tier, ev, h, 0.0);
    const Bytes b = 100 * kBpt;
    EXPECT_CODE(tier.begin_offload(*h, 1.0, b), ErrorCode::IllegalState);
    EXPECT_CODE(tier.begin_load(*g, 1.0, b, TransferPurpose::Reactive), ErrorCode::IllegalState);
    EXPECT_CODE(tier.discard_to_backup(*g, 1.0, b), ErrorCode::IllegalState);
    cache.lock_root_path(g);
    EXPECT_CODE(tier.begin_offload(*g, 1.0, b), ErrorCode::IllegalState);
    cache.unlock_root_path(g);
    uint64_t id = tier.begin_offload(*g, 1.0, b);
    EXPECT_CODE(tier.discard_release(*g, b), ErrorCode::IllegalState);
    Event e = ev.pop();
    EXPECT_CODE(tier.complete(e.id, e.time + 1.0), ErrorCode::InternalError);  // drifted
    EXPECT_CODE(tier.complete(id, e.time), ErrorCode::InternalError);          // already consumed
    EXPECT_CODE(tier.complete(999, 0.0), ErrorCode::InternalError);
}

TEST("tier ledger: GPU memory cannot be overcommitted; working conversions are bounded") {
    EventQueue ev;
    const Bytes cap = 1500000;
    TierManager tier(cap, 0, flat_cost(), ev);
    RadixCache cache(kBpt);
    CacheNode* n = resident(cache, tier, 1, 62500, 0.0);
    backed(cache, tier, ev, n, 0.0);
    CHECK(tier.free_bytes() == cap);
    tier.reserve_working(1000000);
    EXPECT_CODE(tier.begin_load(*n, 1.0, 1000000, TransferPurpose::Reactive), ErrorCode::OutOfGpuMemory);
    CHECK(n->status == NodeStatus::BackupInCpu);
    CHECK(tier.pool().reserved == 0);
    EXPECT_CODE(tier.reserve_working(cap), ErrorCode::OutOfGpuMemory);
    EXPECT_CODE(tier.convert_working(1000000, 2000000), ErrorCode::InternalError);
    EXPECT_CODE(tier.convert_working(5000000, 100), ErrorCode::InternalError);
    tier.convert_working(1000000, 400);
    CHECK(tier.pool().working == 0);
    CHECK(tier.pool().used == 400);
}

TEST("tier ledger: every move is tracked and the audit catches drift") {
    EventQueue ev;
    TierManager tier(8u << 20, 0, flat_cost(), ev);
    RadixCache cache(kBpt);
    CacheNode* n = resident(cache, tier, 1, 1000, 0.0);
    const Bytes b = 1000 * kBpt;
    tier.begin_offload(*n, 1.0, b);
    CHECK(tier.pool().used == b);
    tier.audit(cache);
    Event off = ev.pop();
    tier.complete(off.id, off.time);
    CHECK(tier.pool().used == 0);
    tier.begin_load(*n, 2.0, b, TransferPurpose::Reactive);
    CHECK(tier.pool().reserved == b);
    tier.audit(cache);
    Event ld = ev.pop();
    tier.complete(ld.id, ld.time);
    tier.begin_offload(*n, 3.0, b);  // re-offload of backed content: CPU charged once
    Event again = ev.pop();
    tier.complete(again.id, again.time);
    CHECK(tier.cpu_used() == b);
    tier.begin_load(*n, 4.0, b, TransferPurpose::Reactive);
    Event back = ev.pop();
    tier.complete(back.id, back.time);
    tier.discard_release(*n, b);
    EXPECT_CODE(tier.audit(cache), ErrorCode::InternalError);
}

TEST("tier ledger: instant discard issues no transfer; job records and inflight counts") {
    EventQueue ev;
    TierManager tier(8u << 20, 0, flat_cost(), ev);
    RadixCache cache(kBpt);
    CacheNode* n = resident(cache, tier, 1, 62500, 0.0);
    backed(cache, tier, ev, n, 5.0);
    AgentId target{3, "writer"};
    tier.begin_load(*n, 7.0, 1000000, TransferPurpose::Prefetch, target);
    CHECK(tier.inflight_loads(TransferPurpose::Prefetch) == 1);
    CHECK(tier.inflight_loads(TransferPurpose::Reactive) == 0);
    CHECK(tier.inflight_load_bytes() == 1000000);
    Event e = ev.pop();
    tier.complete(e.id, e.time);
    REQUIRE(tier.completed_jobs().size() == 2);
    const TransferJob& off = tier.completed_jobs()[0];
    CHECK(off.dir == TransferDirection::DeviceToHost);
    CHECK(off.purpose == TransferPurpose::EvictionBackup);
    const TransferJob& ld = tier.completed_jobs()[1];
    CHECK(ld.purpose == TransferPurpose::Prefetch);
    CHECK(ld.target_agent.client == 3);
    CHECK(ld.target_agent.name == "writer");
    CHECK_APPROX(ld.complete, 7.002);
    CHECK(n->prefetched_unused);
    CHECK(std::string(direction_name(ld.dir)) == "H2D");
    CHECK(std::string(purpose_name(off.purpose)) == "eviction_backup");
    const size_t before = tier.inflight_count();
    tier.discard_to_backup(*n, 8.0, 1000000);
    CHECK(n->status == NodeStatus::BackupInCpu);
    CHECK(tier.inflight_count() == before);
    CHECK(ev.empty());
    tier.audit(cache);
}

// ------------------------------------------------------------- workload -------------------
TEST("workload: release order, ids, warmup prompts, validation") {
    WorkloadSpec w;
    w.topology = Topology::Cyclic;
    w.num_agents = 3;
    w.iterations = 2;
    w.warmup_rounds = 1;
    w.fixed_len = 40;
    w.dyn_len = 5;
    w.out_len = 3;
    w.num_workflows = 2;
    w.vocab_size = 1000;
    WorkloadController wc(w, 1);
    std::vector<RequestSpec> first = wc.start();
    REQUIRE(first.size() == 2);
    CHECK(first[0].id == 0);
    CHECK(first[1].id == 1000000);
    CHECK(first[0].prompt.size() == 40);  // warmup: fixed part only
    CHECK(first[0].output.empty());
    CHECK(first[0].prompt[0] == 0);       // reserved first token client 0 agent 0
    CHECK(first[1].prompt[0] == 4);       // client 1 base = 1 * (3 + 1)
    CHECK(first[0].step_metadata.at(AgentId{0, "a01"}) == 1);
    size_t total = 2;
    std::deque<RequestSpec> q(first.begin(), first.end());
    while (!q.empty()) {
        RequestSpec r = q.front();
        q.pop_front();
        if (r.measured) {
            CHECK(r.prompt.size() == 45);
            CHECK(r.output.size() == 3);
        }
        for (RequestSpec& n : wc.on_done(r.id)) {
            q.push_back(n);
            ++total;
        }
    }
    CHECK(total == 2u * 3u * 3u);
    CHECK(wc.all_finished());
    CHECK(wc.max_request_tokens() == 48);
    WorkloadSpec bad = w;
    bad.topology = Topology::BranchMax;
    EXPECT_CODE(WorkloadController(bad, 1), ErrorCode::ConfigError);
    bad = w;
    bad.fixed_len = 1;
    EXPECT_CODE(WorkloadController(bad, 1), ErrorCode::ConfigError);
    bad = w;
    bad.vocab_size = 5;
    EXPECT_CODE(WorkloadController(bad, 1), ErrorCode::ConfigError);
    CHECK(w.label() == "CYCLIC-a3-i2-w2-f40-d5-o3");
}

TT_MAIN
