// CostModel geometry + the two calibrated timing profiles of the reference
// (proj/src/cost_model.cpp:5-55).  Profile numbers are configuration data.
#include "kvflow/cost_model.hpp"

namespace kvf {

Bytes kv_bytes_per_token(uint64_t layers, uint64_t kv_heads, uint64_t head_dim, uint64_t dtype_bytes) {
    return 2ULL * layers * kv_heads * head_dim * dtype_bytes;
}

void CostModel::validate() const {
    auto bad = [](const char* m) { throw_error(ErrorCode::ConfigError, m); };
    if (bytes_per_token == 0) bad("bytes_per_token must be > 0");
    if (prefill_a < 0 || prefill_b < 0) bad("prefill coefficients must be >= 0");
    if (decode_base < 0 || decode_per_seq < 0) bad("decode coefficients must be >= 0");
    if (h2d_bandwidth <= 0 || d2h_bandwidth <= 0) bad("bandwidth must be > 0");
    if (pcie_efficiency <= 0 || pcie_efficiency > 1) bad("pcie_efficiency must be in (0,1]");
    if (fixed_latency < 0) bad("fixed_latency must be >= 0");
}

namespace {
struct Profile {
    const char* name;
    uint64_t layers;
    double pa, pb, db, dps, bw;
};
// {name, layers (8 KV heads x 128 x bf16), prefill_a, prefill_b, decode_base, decode_per_seq, pcie bw}
constexpr Profile kProfiles[] = {
    {"a10g-llama8b", 32, 400e-6, 5e-3, 20e-3, 1e-3, 2e9},
    {"h100-qwen32b", 64, 60e-6, 3e-3, 4e-3, 0.2e-3, 64e9},
};
}  // namespace

CostModel profile_by_name(const std::string& name) {
    for (const Profile& p : kProfiles) {
        if (name != p.name) continue;
        CostModel m;
        m.name = name;
        m.bytes_per_token = kv_bytes_per_token(p.layers, 8, 128, 2);
        m.prefill_a = p.pa;
        m.prefill_b = p.pb;
        m.decode_base = p.db;
        m.decode_per_seq = p.dps;
        m.h2d_bandwidth = m.d2h_bandwidth = p.bw;
        m.pcie_efficiency = 0.6;
        m.fixed_latency = 50e-6;
        m.validate();
        return m;
    }
    throw_error(ErrorCode::ConfigError, "unknown profile: " + name);
}

std::vector<std::string> profile_names() {
    std::vector<std::string> v;
    for (const Profile& p : kProfiles) v.emplace_back(p.name);
    return v;
}

}  // namespace kvf
