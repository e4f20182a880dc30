// GPU-backed unit tests of the C++ control plane: eviction order and actions (K5),
// priorities (K4), and TierManager transfers that move real bytes (K1/K2).  Cases restate
// the reference's radix-cache and tier-manager suites (proj/tests/test_radix_cache.cpp:143-349,
// 435-452; test_tier_manager.cpp) on the kvf API with an Engine attached.
#include <algorithm>
#include <map>
#include <numeric>
#include <random>

#include "kvflow/radix_cache.hpp"
#include "kvflow/scheduler.hpp"
#include "kvflow/sim_engine.hpp"
#include "kvflow/tier_manager.hpp"
#include "tinytest.hpp"

using namespace kvf;

namespace {

constexpr Bytes kBpt = 16;  // 1 layer x 1 head x 4 dims x bf16 x {K,V}

Engine& engine() {
    // intentionally leaked: a static Engine would be destroyed after the CUDA runtime's own
    // atexit teardown
    static Engine& e = *new Engine([] {
        EngineOptions o;
        o.layers = 1;
        o.kv_heads_total = 1;
        o.kv_heads_local = 1;
        o.head_dim = 4;
        o.gpu_slots = 1 << 20;
        o.host_slots = 1 << 20;
        return o;
    }());
    return e;
}

CostModel flat_cost() {
    CostModel c;
    c.bytes_per_token = kBpt;
    c.prefill_a = 1e-4;
    c.prefill_b = 1e-3;
    c.decode_base = 1e-3;
    c.decode_per_seq = 1e-4;
    c.h2d_bandwidth = 1e9;
    c.d2h_bandwidth = 1e9;
    c.pcie_efficiency = 1.0;
    c.fixed_latency = 0;
    return c;
}

struct Rig {
    EventQueue ev;
    TierManager tier;
    RadixCache cache;
    explicit Rig(Bytes cpu_cap = 0) : tier(1 << 20, cpu_cap, flat_cost(), ev, &engine()), cache(kBpt, &engine()) {
        cache.set_prefill_emulation(true);  // the payload checks below need the synthetic KV
    }
    InsertResult put(const TokenSeq& s, VirtualTime now) {
        InsertResult ins = cache.insert(s, now);
        tier.reserve_working(ins.new_bytes);
        tier.convert_working(ins.new_bytes, ins.new_bytes);
        return ins;
    }
    uint64_t id_of(const TokenSeq& key) const {
        uint64_t id = 0;
        cache.for_each_node([&](const CacheNode& n) {
            if (n.key == key) id = n.id;
        });
        return id;
    }
    CacheNode* node(const TokenSeq& key) {
        CacheNode* f = nullptr;
        cache.for_each_node([&](const CacheNode& n) {
            if (n.key == key) f = const_cast<CacheNode*>(&n);
        });
        return f;
    }
    // the node's HBM bytes equal its expected payload (GPU checksum vs GPU payload hash)
    bool dev_ok(const CacheNode& n) {
        return engine().checksum(KVF_TIER_DEVICE, n.dev_runs) == engine().payload_checksum(cache.node_cids(n));
    }
    bool host_ok(const CacheNode& n) {
        return engine().checksum(KVF_TIER_HOST, n.host_runs) == engine().payload_checksum(cache.node_cids(n));
    }
};

}  // namespace

TEST("evict: LRU takes the least recently accessed first; discard frees the slots") {
    Rig r;
    const uint64_t free0 = engine().free_tokens(KVF_TIER_DEVICE);
    r.put({1, 11, 12}, 1.0);
    r.put({2, 21, 22}, 2.0);
    r.put({3, 31, 32}, 3.0);
    CHECK(engine().free_tokens(KVF_TIER_DEVICE) == free0 - 9);
    const uint64_t a = r.id_of({1, 11, 12});
    EvictOutcome out = r.cache.evict({1, EvictionPolicy::Lru, TierMode::Discard, {}}, r.tier, 4.0);
    REQUIRE(out.victims.size() == 1);
    CHECK(out.victims[0].node_id == a);
    CHECK(out.victims[0].immediate);
    CHECK(out.immediate_freed == 3 * kBpt);
    CHECK(r.cache.peek_prefix({1, 11, 12}).matched_tokens == 0);
    CHECK(r.tier.pool().used == 6 * kBpt);
    CHECK(engine().free_tokens(KVF_TIER_DEVICE) == free0 - 6);
    r.tier.audit(r.cache);
}

TEST("evict: match refreshes recency, peek does not") {
    for (bool use_match : {false, true}) {
        Rig r;
        r.put({1, 11}, 1.0);
        r.put({2, 22}, 2.0);
        if (use_match) CHECK(r.cache.match_prefix({1, 11}, 4.0).matched_tokens == 2);
        else CHECK(r.cache.peek_prefix({1, 11}).matched_tokens == 2);
        const uint64_t want = r.id_of(use_match ? TokenSeq{2, 22} : TokenSeq{1, 11});  // before it is removed
        EvictOutcome out = r.cache.evict({1, EvictionPolicy::Lru, TierMode::Discard, {}}, r.tier, 5.0);
        REQUIRE(out.victims.size() == 1);
        CHECK(out.victims[0].node_id == want);
    }
}

TEST("evict: workflow-aware order (suffix, then larger steps) and the rank floor") {
    for (bool floor : {false, true}) {
        Rig r;
        r.put({1, 11, 12}, 1.0);
        r.put({2, 21, 22}, 2.0);
        r.put({3, 31, 32}, 3.0);
        AgentId a{0, "a"}, b{0, "b"};
        r.cache.mark_fixed_boundary(a, {1, 11, 12}, 3);
        r.cache.mark_fixed_boundary(b, {2, 21, 22}, 3);
        StepMap steps;
        steps[a] = 5;
        steps[b] = 1;
        r.cache.set_agent_priorities(steps);  // K4
        EvictRequest req{floor ? Bytes(1 << 20) : 9 * kBpt, EvictionPolicy::WorkflowAware, TierMode::Discard, {}};
        if (floor) req.rank_floor_exclusive = rank_for_step(1);
        const uint64_t a_id = r.id_of({1, 11, 12}), b_id = r.id_of({2, 21, 22}), c_id = r.id_of({3, 31, 32});
        EvictOutcome out = r.cache.evict(req, r.tier, 4.0);  // K5
        REQUIRE(out.victims.size() == (floor ? 2u : 3u));
        CHECK(out.victims[0].node_id == c_id);
        CHECK(out.victims[1].node_id == a_id);
        if (!floor) CHECK(out.victims[2].node_id == b_id);
        CHECK(out.sufficient == !floor);
        if (floor) CHECK(r.cache.peek_prefix({2, 21, 22}).matched_tokens == 3);
    }
}

TEST("evict: leaves before parents, a freed parent follows in the same pass; locks protect") {
    {
        Rig r;
        r.put({1, 2}, 1.0);
        r.put({1, 2, 3}, 2.0);
        const uint64_t p = r.id_of({1, 2}), l = r.id_of({3});
        EvictOutcome out = r.cache.evict({3 * kBpt, EvictionPolicy::Lru, TierMode::Discard, {}}, r.tier, 3.0);
        REQUIRE(out.victims.size() == 2);
        CHECK(out.victims[0].node_id == l);
        CHECK(out.victims[1].node_id == p);
        CHECK(r.cache.node_count() == 0);
    }
    {
        Rig r;
        InsertResult a = r.put({1, 11}, 1.0);
        r.put({2, 22}, 2.0);
        r.cache.lock_root_path(a.path.back());
        const uint64_t b_id = r.id_of({2, 22});
        EvictOutcome out = r.cache.evict({1 << 20, EvictionPolicy::Lru, TierMode::Discard, {}}, r.tier, 3.0);
        REQUIRE(out.victims.size() == 1);
        CHECK(out.victims[0].node_id == b_id);
        CHECK(!out.sufficient);
        r.cache.unlock_root_path(a.path.back());
    }
}

TEST("queued K4: records shipped while it is pending keep its ranks; K5 behind it sees them; late join") {
    // Two caches built the same way: A joins every K4 at once (the reference's synchronous
    // set_agent_priorities), B leaves it queued while locks and an eviction's status changes
    // ship records (KVF_REC_KEEP_RANK), then joins at the end.  Victims and dumps must agree.
    std::mt19937_64 rng(7);
    for (int trial = 0; trial < 40; ++trial) {
        Rig ra, rb;
        std::vector<TokenSeq> used;
        const size_t nseq = 4 + rng() % 12;
        for (size_t k = 0; k < nseq; ++k) {
            TokenSeq s;
            const size_t len = 2 + rng() % 6;
            for (size_t t = 0; t < len; ++t) s.push_back(static_cast<TokenId>(1 + rng() % 4));
            used.push_back(s);
            ra.put(s, 1.0 + k);
            rb.put(s, 1.0 + k);
        }
        std::vector<std::pair<AgentId, std::pair<TokenSeq, size_t>>> marks;
        for (size_t a = 0, na = 1 + rng() % 5; a < na; ++a) {
            const TokenSeq& s = used[rng() % used.size()];
            marks.push_back({AgentId{0, "agent" + std::to_string(a)}, {s, 1 + rng() % s.size()}});
        }
        for (auto& m : marks) {
            ra.cache.mark_fixed_boundary(m.first, m.second.first, m.second.second);
            rb.cache.mark_fixed_boundary(m.first, m.second.first, m.second.second);
        }
        StepMap steps;
        for (auto& m : marks)
            if (rng() % 4) steps[m.first] = static_cast<StepValue>(rng() % 6);
        ra.cache.set_agent_priorities(steps);
        rb.cache.set_agent_priorities_async(steps);
        CHECK(rb.cache.priorities_pending());
        // lock one sequence's path in both (its nodes ship lock records while B's K4 is queued)
        const TokenSeq& locked = used[rng() % used.size()];
        MatchResult ma = ra.cache.peek_prefix(locked), mb = rb.cache.peek_prefix(locked);
        REQUIRE(!ma.path.empty() && !mb.path.empty());
        ra.cache.lock_root_path(ma.path.back());
        rb.cache.lock_root_path(mb.path.back());
        const TierMode mode = trial % 2 ? TierMode::Offload : TierMode::Discard;
        const EvictRequest req{Bytes(1 + rng() % 12) * kBpt, EvictionPolicy::WorkflowAware, mode, {}};
        EvictOutcome oa = ra.cache.evict(req, ra.tier, 50.0);
        EvictOutcome ob = rb.cache.evict(req, rb.tier, 50.0);
        CHECK(rb.cache.priorities_pending());  // K5 ran behind the queued K4 without a join
        REQUIRE(oa.victims.size() == ob.victims.size());
        for (size_t k = 0; k < oa.victims.size(); ++k) {
            CHECK(oa.victims[k].node_id == ob.victims[k].node_id);
            CHECK(oa.victims[k].immediate == ob.victims[k].immediate);
        }
        // a second eviction ships the first one's status records, still under the queued K4
        EvictOutcome oa2 = ra.cache.evict(req, ra.tier, 51.0);
        EvictOutcome ob2 = rb.cache.evict(req, rb.tier, 51.0);
        REQUIRE(oa2.victims.size() == ob2.victims.size());
        for (size_t k = 0; k < oa2.victims.size(); ++k) CHECK(oa2.victims[k].node_id == ob2.victims[k].node_id);
        ra.cache.unlock_root_path(ma.path.back());
        rb.cache.unlock_root_path(mb.path.back());
        rb.cache.join_priorities();
        CHECK(!rb.cache.priorities_pending());
        CHECK(ra.cache.dump() == rb.cache.dump());
        for (Rig* r : {&ra, &rb})  // fence the write-backs (K2) before the rigs go
            while (!r->ev.empty()) {
                Event done = r->ev.pop();
                r->tier.complete(done.id, done.time);
            }
    }
}

TEST("offload eviction moves real bytes; a backed copy makes the next eviction instant") {
    Rig r;
    r.put({1, 11, 12}, 1.0);
    CacheNode* n = r.node({1, 11, 12});
    REQUIRE(r.dev_ok(*n));
    EvictOutcome out = r.cache.evict({1, EvictionPolicy::Lru, TierMode::Offload, {}}, r.tier, 2.0);
    REQUIRE(out.victims.size() == 1);
    CHECK(!out.victims[0].immediate);
    CHECK(n->status == NodeStatus::Offloading);
    Event done = r.ev.pop();
    r.tier.complete(done.id, done.time);  // K2 fence
    CHECK(n->status == NodeStatus::BackupInCpu);
    CHECK(n->dev_runs.empty());
    CHECK(r.host_ok(*n));
    r.tier.audit(r.cache);
    r.tier.begin_load(*n, done.time, 3 * kBpt, TransferPurpose::Reactive);
    Event loaded = r.ev.pop();
    r.tier.complete(loaded.id, loaded.time);  // K1 fence
    CHECK(n->status == NodeStatus::InGpu);
    CHECK(r.dev_ok(*n));
    EvictOutcome again = r.cache.evict({1, EvictionPolicy::Lru, TierMode::Offload, {}}, r.tier, loaded.time + 1);
    REQUIRE(again.victims.size() == 1);
    CHECK(again.victims[0].immediate);
    CHECK(n->status == NodeStatus::BackupInCpu);
    CHECK(r.ev.empty());
    r.tier.audit(r.cache);
}

TEST("a full backup tier falls back to plain discard") {
    Rig r(3 * kBpt);
    r.put({1, 11, 12}, 1.0);
    r.put({2, 21, 22}, 2.0);
    EvictOutcome first = r.cache.evict({1, EvictionPolicy::Lru, TierMode::Offload, {}}, r.tier, 3.0);
    REQUIRE(first.victims.size() == 1);
    Event done = r.ev.pop();
    r.tier.complete(done.id, done.time);
    CHECK(r.tier.cpu_used() == 3 * kBpt);
    EvictOutcome second = r.cache.evict({1, EvictionPolicy::Lru, TierMode::Offload, {}}, r.tier, 4.0);
    REQUIRE(second.victims.size() == 1);
    CHECK(second.victims[0].immediate);
    CHECK(r.cache.peek_prefix({2, 21, 22}).matched_tokens == 0);
    CHECK(r.ev.empty());
    r.tier.audit(r.cache);
}

TEST("dump renders priorities deterministically (reference golden string)") {
    Rig r;
    r.cache.insert({1, 2, 3, 4}, 1.0);
    r.cache.insert({1, 2, 5}, 2.0);
    r.cache.insert({7}, 3.0);
    AgentId w{0, "writer"};
    r.cache.mark_fixed_boundary(w, {1, 2, 5}, 3);
    StepMap s;
    s[w] = 2;
    r.cache.set_agent_priorities(s);
    CHECK(r.cache.dump() ==
          "root\n"
          "  [1..+1] IN_GPU STEP(2) lock=0\n"
          "    [3..+1] IN_GPU SUFFIX lock=0\n"
          "    [5] IN_GPU STEP(2) lock=0 boundary{c0/writer}\n"
          "  [7] IN_GPU SUFFIX lock=0\n");
}

TEST("K4 priorities equal brute force on random trees; splits keep every node's bytes") {
    std::mt19937_64 rng(20260822);
    for (int t = 0; t < 60; ++t) {
        Rig r;
        std::vector<TokenSeq> used;
        VirtualTime now = 0;
        for (int i = 0, e = 5 + static_cast<int>(rng() % 21); i < e; ++i) {
            TokenSeq s;
            if (!used.empty() && rng() % 2) {
                const TokenSeq& b = used[rng() % used.size()];
                s.assign(b.begin(), b.begin() + static_cast<long>(1 + rng() % b.size()));
            }
            for (int k = 0, m = 4 + static_cast<int>(rng() % 17); k < m; ++k) s.push_back(static_cast<TokenId>(rng() % 4));
            r.put(s, now += 1.0);
            used.push_back(s);
        }
        std::vector<std::pair<AgentId, std::pair<TokenSeq, size_t>>> marks;
        for (size_t a = 0, na = 1 + rng() % 6; a < na; ++a) {
            AgentId id{static_cast<ClientId>(rng() % 2), "agent" + std::to_string(a)};
            const TokenSeq& s = used[rng() % used.size()];
            size_t fl = 1 + rng() % s.size();
            r.cache.mark_fixed_boundary(id, s, fl);
            marks.push_back({id, {s, fl}});
        }
        StepMap steps;
        for (auto& m : marks) {
            uint64_t x = rng() % 10;
            if (x < 7) steps[m.first] = static_cast<StepValue>(rng() % 9);
            else if (x == 7) steps[m.first] = kStepUnreachable;
        }
        r.cache.set_agent_priorities(steps);
        std::map<const CacheNode*, int64_t> want;
        r.cache.for_each_node([&](const CacheNode& n) { want[&n] = kRankSuffix; });
        for (auto& m : marks) {
            CacheNode* b = r.cache.boundary_node(m.first);
            REQUIRE(b != nullptr);
            auto it = steps.find(m.first);
            int64_t v = rank_for_step(it == steps.end() ? kStepUnreachable : it->second);
            for (CacheNode* n = b; n && !n->is_root(); n = n->parent) want[n] = std::min(want[n], v);
        }
        r.cache.for_each_node([&](const CacheNode& n) {
            CHECK(n.rank == want[&n]);
            CHECK(r.dev_ok(n));
        });
    }
}

TEST("tier manager with bytes: FIFO jobs, fences, write-once host copies, audit") {
    Rig r;
    r.put({1, 2, 3, 4, 5, 6, 7, 8}, 0.0);
    r.put({9, 10, 11}, 0.0);
    CacheNode* a = r.node({1, 2, 3, 4, 5, 6, 7, 8});
    CacheNode* b = r.node({9, 10, 11});
    r.tier.begin_offload(*a, 1.0, r.cache.node_bytes(*a));
    r.tier.begin_offload(*b, 1.0, r.cache.node_bytes(*b));
    CHECK(r.tier.inflight_count() == 2);
    while (!r.ev.empty()) {
        Event e = r.ev.pop();
        const TransferJob& j = r.tier.complete(e.id, e.time);
        CHECK(j.device_ms >= 0.0f);
    }
    CHECK(r.host_ok(*a));
    CHECK(r.host_ok(*b));
    const RunList host_before = a->host_runs;
    r.tier.begin_load(*a, 2.0, r.cache.node_bytes(*a), TransferPurpose::Prefetch, AgentId{1, "x"});
    Event e = r.ev.pop();
    r.tier.complete(e.id, e.time);
    CHECK(a->prefetched_unused);
    CHECK(r.dev_ok(*a));
    r.tier.begin_offload(*a, 3.0, r.cache.node_bytes(*a));  // re-offload: same host slots
    Event e2 = r.ev.pop();
    r.tier.complete(e2.id, e2.time);
    CHECK(a->host_runs.size() == host_before.size() && a->host_runs[0].start == host_before[0].start);
    CHECK(r.tier.cpu_used() == (8 + 3) * kBpt);
    CHECK(r.host_ok(*a));
    r.tier.audit(r.cache);
    // split of a backed node splits both run lists; bytes stay put and stay correct
    r.tier.begin_load(*a, 4.0, r.cache.node_bytes(*a), TransferPurpose::Reactive);
    Event e3 = r.ev.pop();
    r.tier.complete(e3.id, e3.time);
    r.put({1, 2, 3, 99}, 5.0);
    CacheNode* up = r.node({1, 2, 3});
    REQUIRE(up != nullptr);
    CHECK(r.dev_ok(*up) && r.dev_ok(*a) && r.host_ok(*up) && r.host_ok(*a));
    r.tier.audit(r.cache);
}

TT_MAIN

TEST("evict: a victim that throws (bounded-CPU remove defect) still launches the booked write-backs") {
    Rig r(4 * kBpt);
    r.tier.set_offload_batching(true);
    InsertResult c = r.put({9}, 0.5);
    r.cache.lock_root_path(c.path.back());  // keep {9} out of the first two evictions
    r.put({1, 2, 3, 4}, 1.0);
    r.put({1, 2, 3, 5}, 2.0);  // A = [1,2,3] with children [4], [5]
    for (VirtualTime t : {3.0, 4.0}) {  // [4] then [5] -> backed copies (cpu_used = 2 tokens)
        EvictOutcome o = r.cache.evict({kBpt, EvictionPolicy::Lru, TierMode::Offload, {}}, r.tier, t);
        REQUIRE(o.victims.size() == 1);
        Event done = r.ev.pop();
        r.tier.complete(done.id, done.time);
    }
    r.cache.unlock_root_path(c.path.back());
    CHECK(r.tier.cpu_used() == 2 * kBpt);
    // victims: {9} (fits the CPU tier: offload, booked) then A (3 tokens, no CPU room: remove,
    // but it still has BACKUP_IN_CPU children -> the reference's InternalError)
    const uint64_t d2h0 = engine().stats().d2h_jobs;
    bool threw = false;
    try {
        r.cache.evict({4 * kBpt, EvictionPolicy::Lru, TierMode::Offload, {}}, r.tier, 5.0);
    } catch (const SimError& e) {
        threw = e.code() == ErrorCode::InternalError;
    }
    CHECK(threw);
    CHECK(engine().stats().d2h_jobs == d2h0 + 1);  // {9}'s write-back left before the throw escaped
    Event done = r.ev.pop();
    r.tier.complete(done.id, done.time);
    CHECK(r.host_ok(*r.node({9})));
}

TEST("Simulator refuses a ledger larger than the engine's slot pools") {
    WorkloadSpec w;
    w.topology = Topology::Cyclic;
    w.num_agents = 2;
    w.iterations = 1;
    w.fixed_len = 8;
    w.dyn_len = 2;
    w.out_len = 2;
    SchedulerConfig sc;
    sc.policy = Policy::Kvflow;
    sc.apply_policy_defaults();
    CostModel cost = flat_cost();
    auto code_of = [&](Bytes gpu_cap, Bytes cpu_cap) {
        try {
            Simulator sim(cost, sc, w, gpu_cap, cpu_cap, 1, &engine());
        } catch (const SimError& e) {
            return static_cast<int>(e.code());
        }
        return -1;
    };
    CHECK(code_of((1ull << 20) * kBpt, 0) == -1);                              // fits exactly
    CHECK(code_of((1ull << 21) * kBpt, 0) == static_cast<int>(ErrorCode::ConfigError));  // HBM pool too small
    CHECK(code_of(1 << 20, 0) == -1);                                          // unbounded CPU: caller's bound
    CHECK(code_of(1 << 20, 1ull << 40) == -1);  // bounded, but above anything the run can cache
}
