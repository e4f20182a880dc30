// C3 trace from this repo's components on the GPU engine: the shared harness
// (tests/cpp/c3_harness.hpp) compiled against kvf.  Same arguments as oracle/ref_c3.
#include <cstdio>
#include <cstdlib>

#include "kvflow/cost_model.hpp"
#include "kvflow/radix_cache.hpp"
#include "kvflow/sim_engine.hpp"
#include "kvflow/step_graph.hpp"
#include "kvflow/tier_manager.hpp"
#define KV_NS kvf
#include "c3_harness.hpp"

int main(int argc, char** argv) {
    const uint64_t seed = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 3;
    const int iters = argc > 2 ? std::atoi(argv[2]) : 4;
    const kvf::Bytes bpt = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 16384;
    const kvf::Bytes cap = argc > 4 ? std::strtoull(argv[4], nullptr, 10) : 24000ull * 16384;
    kvf::EngineOptions eo;  // one Llama-3-8B KV head (16 KiB/token) unless bpt says otherwise
    eo.layers = 32;
    eo.kv_heads_total = 8;
    eo.kv_heads_local = static_cast<uint32_t>(bpt / (2 * 32 * 128 * 2));
    eo.head_offset = 8 - eo.kv_heads_local;
    eo.head_dim = 128;
    eo.gpu_slots = cap / bpt;
    eo.host_slots = 16 * 8192 + 64 * 16 * 100;
    kvf::Engine engine(eo);
    kvf::CostModel cost = c3::c3_cost(bpt);
    kvf::EventQueue ev;
    kvf::TierManager tier(cap, 0, cost, ev, &engine);
    kvf::RadixCache cache(bpt, &engine);
    cache.set_prefill_emulation(true);  // the byte checks below need the synthetic KV
    try {
        c3::Driver<kvf::TierManager, kvf::RadixCache, kvf::EventQueue, kvf::CostModel> d(tier, cache, ev, cost, seed);
        std::fputs(d.run(iters).trace.c_str(), stdout);
        // bytes: every resident / backed node holds its expected payload
        uint64_t bad = 0, checked = 0;
        cache.for_each_node([&](const kvf::CacheNode& n) {
            const uint64_t want = engine.payload_checksum(cache.node_cids(n));
            if (n.status == kvf::NodeStatus::InGpu) { ++checked; bad += engine.checksum(KVF_TIER_DEVICE, n.dev_runs) != want; }
            if (n.cpu_backed) { ++checked; bad += engine.checksum(KVF_TIER_HOST, n.host_runs) != want; }
        });
        std::printf("{\"t\":\"bytes\",\"checked\":%llu,\"bad\":%llu}\n", (unsigned long long)checked, (unsigned long long)bad);
    } catch (const kvf::SimError& e) {
        std::printf("{\"t\":\"error\",\"code\":%d}\n", static_cast<int>(e.code()));
    }
    return 0;
}
