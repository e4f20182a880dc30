// C++ handle over the CUDA engine C-ABI (include/kvflow.h).  Every failure becomes a
// SimError with the reference's ErrorCode convention (status - 1), engine-specific
// statuses become DeviceError / NoDevice.
#include "kvflow/engine.hpp"

#include <algorithm>
#include <mutex>

namespace kvf {

RunList split_runs(RunList& runs, uint64_t tokens) {
    RunList head;
    size_t i = 0;
    while (tokens > 0 && i < runs.size()) {
        Run& r = runs[i];
        if (r.len <= tokens) {
            head.push_back(r);
            tokens -= r.len;
            ++i;
        } else {
            head.push_back(Run{r.start, tokens});
            r.start += tokens;
            r.len -= tokens;
            tokens = 0;
        }
    }
    runs.erase(runs.begin(), runs.begin() + static_cast<long>(i));
    return head;
}

void throw_engine(int status, const std::string& what) {
    std::string msg = what + ": " + kvf_last_error();
    if (status >= 1 && status <= 14) throw_error(static_cast<ErrorCode>(status - 1), msg);
    if (status == KVF_E_NO_DEVICE) throw_error(ErrorCode::NoDevice, msg);
    if (status == KVF_E_OUT_OF_HOST_SLOTS) throw_error(ErrorCode::OutOfHostMemory, msg);
    throw_error(ErrorCode::DeviceError, msg);
}

#define KVF_CALL(expr)                          \
    do {                                        \
        int _rc = (expr);                       \
        if (_rc != KVF_OK) throw_engine(_rc, #expr); \
    } while (0)

namespace {
std::mutex g_factory_mu;
EngineFactory g_factory;
}  // namespace

void set_default_engine_factory(EngineFactory factory) {
    std::lock_guard<std::mutex> lk(g_factory_mu);
    g_factory = std::move(factory);
}

Engine* default_engine(uint64_t bytes_per_token) {
    std::lock_guard<std::mutex> lk(g_factory_mu);
    return g_factory ? g_factory(bytes_per_token) : nullptr;
}

Engine::Engine(const EngineOptions& opt) : opt_(opt) {
    kvf_geometry g{opt.layers, opt.kv_heads_total, opt.kv_heads_local, opt.head_offset, opt.head_dim, 2};
    kvf_engine_config c{opt.device, opt.gpu_slots, opt.host_slots, opt.pcie_ctas, opt.pcie_mode, opt.hbm_ctas,
                        opt.numa_node};
    KVF_CALL(kvf_engine_create(&g, &c, &e_));
    KVF_CALL(kvf_engine_token_bytes(e_, nullptr, &token_bytes_));
}

Engine::~Engine() { kvf_engine_destroy(e_); }

RunList Engine::alloc(int tier, uint64_t tokens) {
    // the allocator keeps runs long (best fit, else largest first): a handful of entries is
    // the common case -- a 4096-entry buffer zeroed per call cost ~3 us on every load / insert
    RunList out(static_cast<size_t>(std::max<uint64_t>(1, std::min<uint64_t>(tokens, 16))));
    uint32_t n = 0;
    int rc = kvf_slots_alloc(e_, tier, tokens, out.data(), static_cast<uint32_t>(out.size()), &n);
    for (size_t cap = 4096; rc == KVF_E_TOO_LARGE && out.size() < (1u << 20); cap = 1u << 20) {
        out.resize(std::min<uint64_t>(std::max<uint64_t>(tokens, 1), cap));  // fragmented pool: room for more runs
        rc = kvf_slots_alloc(e_, tier, tokens, out.data(), static_cast<uint32_t>(out.size()), &n);
    }
    if (rc != KVF_OK) throw_engine(rc, "kvf_slots_alloc");
    out.resize(n);
    return out;
}

void Engine::free(int tier, const RunList& runs) {
    if (!runs.empty()) KVF_CALL(kvf_slots_free(e_, tier, runs.data(), static_cast<uint32_t>(runs.size())));
}

uint64_t Engine::free_tokens(int tier) const {
    uint64_t t = 0;
    KVF_CALL(kvf_slots_free_count(e_, tier, &t, nullptr));
    return t;
}

void Engine::h2d(uint64_t job, const RunList& host, const RunList& dev) {
    KVF_CALL(kvf_h2d_gather(e_, job, host.data(), static_cast<uint32_t>(host.size()), dev.data(),
                            static_cast<uint32_t>(dev.size())));
}

void Engine::h2d_layered(uint64_t job, const RunList& host, const RunList& dev) {
    KVF_CALL(kvf_h2d_gather_layered(e_, job, host.data(), static_cast<uint32_t>(host.size()), dev.data(),
                                    static_cast<uint32_t>(dev.size()), nullptr, nullptr));
}

void Engine::d2h(uint64_t job, const RunList& dev, const RunList& host) {
    KVF_CALL(kvf_d2h_scatter(e_, job, dev.data(), static_cast<uint32_t>(dev.size()), host.data(),
                             static_cast<uint32_t>(host.size())));
}

void Engine::d2h_batch(const std::vector<uint64_t>& jobs, const std::vector<const RunList*>& dev,
                       const std::vector<const RunList*>& host) {
    std::vector<Run> d, h;
    std::vector<uint32_t> dc, hc;
    for (size_t k = 0; k < jobs.size(); ++k) {
        d.insert(d.end(), dev[k]->begin(), dev[k]->end());
        h.insert(h.end(), host[k]->begin(), host[k]->end());
        dc.push_back(static_cast<uint32_t>(dev[k]->size()));
        hc.push_back(static_cast<uint32_t>(host[k]->size()));
    }
    KVF_CALL(kvf_d2h_scatter_batch(e_, static_cast<uint32_t>(jobs.size()), jobs.data(), d.data(), dc.data(), h.data(),
                                   hc.data()));
}

bool Engine::query(uint64_t job) {
    int32_t done = 0;
    KVF_CALL(kvf_job_query(e_, job, &done));
    return done != 0;
}

void Engine::wait(uint64_t job) { KVF_CALL(kvf_job_wait(e_, job)); }

float Engine::elapsed_ms(uint64_t job) {
    float ms = 0;
    KVF_CALL(kvf_job_elapsed_ms(e_, job, &ms));
    return ms;
}

void Engine::release(uint64_t job) { KVF_CALL(kvf_job_release(e_, job)); }
void Engine::compute_begin(uint64_t job) { KVF_CALL(kvf_compute_job_begin(e_, job)); }
void Engine::compute_end(uint64_t job) { KVF_CALL(kvf_compute_job_end(e_, job)); }
void Engine::compute_wait_job(uint64_t job) { KVF_CALL(kvf_compute_wait_job(e_, job)); }
void Engine::compute_wait_job_layer(uint64_t job, uint32_t layer) {
    KVF_CALL(kvf_compute_wait_job_layer(e_, job, layer));
}
void Engine::compute_spin(uint64_t ns, uint32_t ctas) { KVF_CALL(kvf_compute_spin(e_, ns, ctas)); }
void Engine::sync() { KVF_CALL(kvf_sync_all(e_)); }

void Engine::fill(int tier, const RunList& runs, const std::vector<uint64_t>& cids) {
    KVF_CALL(kvf_fill_payload(e_, tier, runs.data(), static_cast<uint32_t>(runs.size()), cids.data(), cids.size()));
}

uint64_t Engine::checksum(int tier, const RunList& runs) {
    uint64_t s = 0;
    KVF_CALL(kvf_checksum(e_, tier, runs.data(), static_cast<uint32_t>(runs.size()), &s));
    return s;
}

uint64_t Engine::payload_checksum(const std::vector<uint64_t>& cids) {
    uint64_t s = 0;
    KVF_CALL(kvf_payload_checksum(e_, cids.data(), cids.size(), &s));
    return s;
}

std::vector<int64_t> Engine::priorities(const std::vector<int32_t>& parent, const std::vector<int32_t>& bidx,
                                        const std::vector<int64_t>& cand) {
    std::vector<int64_t> out(parent.size());
    KVF_CALL(kvf_priority_propagate(e_, parent.data(), static_cast<uint32_t>(parent.size()), bidx.data(), cand.data(),
                                    static_cast<uint32_t>(bidx.size()), out.data()));
    return out;
}

void Engine::victims(const kvf_tree_view& tree, const kvf_evict_request& req, std::vector<int32_t>& idx,
                     std::vector<uint8_t>& action, uint64_t& immediate, uint64_t& pending) {
    idx.resize(std::max<uint32_t>(1, tree.n));
    action.resize(idx.size());
    uint32_t cnt = 0;
    KVF_CALL(kvf_victim_select(e_, &tree, &req, idx.data(), action.data(), &cnt, &immediate, &pending));
    idx.resize(cnt);
    action.resize(cnt);
}

kvf_stats Engine::stats() const {
    kvf_stats s{};
    KVF_CALL(kvf_get_stats(e_, &s));
    return s;
}

void Engine::set_job_timing(uint32_t mode) {
    if (int rc = kvf_engine_set_job_timing(e_, mode)) throw_engine(rc, "kvf_engine_set_job_timing");
}

}  // namespace kvf
