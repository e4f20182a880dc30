// Golden C3 trace from the UNMODIFIED reference components (TEST INFRASTRUCTURE ONLY):
// the shared harness tests/cpp/c3_harness.hpp compiled against kvsim.
//   oracle/_ref/ref_c3 <seed> <iterations> <bytes_per_token> <gpu_cap>
#include <cstdio>
#include <cstdlib>

#include "kvsim/cost_model.hpp"
#include "kvsim/radix_cache.hpp"
#include "kvsim/sim_engine.hpp"
#include "kvsim/step_graph.hpp"
#include "kvsim/tier_manager.hpp"
#define KV_NS kvsim
#include "../tests/cpp/c3_harness.hpp"

int main(int argc, char** argv) {
    const uint64_t seed = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 3;
    const int iters = argc > 2 ? std::atoi(argv[2]) : 4;
    const kvsim::Bytes bpt = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 16384;
    const kvsim::Bytes cap = argc > 4 ? std::strtoull(argv[4], nullptr, 10) : 24000ull * 16384;
    kvsim::CostModel cost = c3::c3_cost(bpt);
    kvsim::EventQueue ev;
    kvsim::TierManager tier(cap, 0, cost, ev);
    kvsim::RadixCache cache(bpt);
    try {
        c3::Driver<kvsim::TierManager, kvsim::RadixCache, kvsim::EventQueue, kvsim::CostModel> d(tier, cache, ev, cost, seed);
        std::fputs(d.run(iters).trace.c_str(), stdout);
    } catch (const kvsim::SimError& e) {
        std::printf("{\"t\":\"error\",\"code\":%d}\n", static_cast<int>(e.code()));
    }
    return 0;
}
