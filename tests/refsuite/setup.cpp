// Default-engine factory for the reference suites run against the B200 host API
// (test infrastructure, tests/refsuite/README.md).  The reference's tests build RadixCache /
// TierManager / Simulator with no engine (kvsim has none); kvf::set_default_engine_factory
// makes each of them land on a GPU engine whose token geometry matches the ledger's
// bytes_per_token -- the same engine for the same bytes_per_token, so a cache and a tier
// manager built separately share their pools.  Engines live until process exit.
#include <execinfo.h>
#include <unistd.h>

#include <csignal>
#include <cstdio>
#include <map>
#include <memory>
#include <mutex>

#include "kvflow/engine.hpp"

namespace {

bool geometry_for(uint64_t bpt, kvf::EngineOptions& o) {
    const uint64_t per_head_layer = 2 * 128 * 2;  // K and V planes, head_dim 128, bf16
    if (bpt % per_head_layer == 0) {
        const uint64_t units = bpt / per_head_layer;  // layers x heads
        for (uint32_t h : {8u, 4u, 2u, 1u})
            if (units % h == 0) {
                o.layers = static_cast<uint32_t>(units / h);
                o.kv_heads_total = o.kv_heads_local = h;
                o.head_dim = 128;
                return true;
            }
    }
    if (bpt % 16 == 0) {  // one layer, one head, head_dim = bpt / 4 (e.g. the suites' 16 B/token)
        o.layers = 1;
        o.kv_heads_total = o.kv_heads_local = 1;
        o.head_dim = static_cast<uint32_t>(bpt / 4);
        return true;
    }
    return false;
}

void on_crash(int sig) {  // a crash inside a suite names its frames (no debugger on the GPU box)
    void* frames[64];
    const int n = backtrace(frames, 64);
    std::fprintf(stderr, "refsuite: signal %d\n", sig);
    backtrace_symbols_fd(frames, n, 2);
    _exit(128 + sig);
}

struct Install {
    Install() {
        std::signal(SIGSEGV, on_crash);
        std::signal(SIGABRT, on_crash);
        kvf::set_default_engine_factory([](uint64_t bpt) -> kvf::Engine* {
            static std::mutex mu;
            static std::map<uint64_t, kvf::Engine*> engines;  // leaked on purpose: outlive every cache
            std::lock_guard<std::mutex> lk(mu);
            auto it = engines.find(bpt);
            if (it != engines.end()) return it->second;
            kvf::EngineOptions o;
            if (!geometry_for(bpt, o)) {
                std::fprintf(stderr, "refsuite: no bf16 geometry for %llu bytes/token\n",
                             static_cast<unsigned long long>(bpt));
                return engines[bpt] = nullptr;
            }
            const uint64_t budget = 1ull << 30;  // 1 GiB per tier: far above any suite's ledger
            o.gpu_slots = o.host_slots = std::min<uint64_t>(budget / bpt, 1ull << 24);
            return engines[bpt] = new kvf::Engine(o);
        });
    }
} install;

}  // namespace
