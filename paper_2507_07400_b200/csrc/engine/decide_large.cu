// K5, device-wide path for trees above the single-CTA limit (4096 nodes).
//
// Same closed form as the single-CTA kernel (decide.cu), spread over the
// whole GPU:
//   1. stage flags (self-eligible, releases-parent) per node            -- 1 grid kernel
//   2. `before` order of the candidates as a stable LSD radix sort       -- CUB onesweep, one
//      pass per key word, least significant first: id, seq, time, (rank)  pass per word
//      and finally a 1-bit "not a candidate" word so non-candidates sort last
//   3. ord, blocked root walks, R, eff root walks                         -- 4 grid kernels
//      (global atomics with early exit, as in the CTA version)
//   4. victims: R sorted by (eff asc, depth desc)                         -- CUB radix sort
//   5. byte prefix in victim order + the `needed` cut + actions           -- CUB scan + 1 kernel
// No host round trip between phases; one H2D of the packed SoA and one D2H of the result.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "engine_internal.hpp"

using namespace kvf_impl;

namespace {

constexpr int64_t kSuffix = INT64_MAX / 2;
constexpr int64_t kUnreach = INT64_MAX / 4;

struct BigTree {
    const int32_t* parent;
    const uint16_t* depth;
    const uint8_t* status;
    const int32_t* lock;
    const int64_t* rank;
    const double* time;
    const uint64_t* seq;
    const uint64_t* id;
    const uint64_t* tokens;
    const uint8_t* backed;
    uint32_t n;
};

struct BigReq {  // lives in device memory (part of the uploaded blob): the graph is reusable
    uint64_t needed;
    int64_t floor;
    uint64_t cpu_used, cpu_cap;
    int32_t wa, offload, has_floor;
    uint64_t bpt;  // bytes per token (per call: not baked into the graph)
    int64_t rank_max;  // rank_bytes < 8: every rank is SUFFIX, UNREACHABLE or in [0, rank_max]
};

__device__ __forceinline__ uint64_t time_order(double t) {
    const uint64_t b = t == 0.0 ? 0ull : static_cast<uint64_t>(__double_as_longlong(t));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void big_stage(BigTree t, const BigReq* __restrict__ q, uint8_t* flags, uint32_t* blocked, uint32_t* vals) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < t.n; i += gridDim.x * blockDim.x) {
        const uint64_t bytes = t.tokens[i] * q->bpt;
        const bool cpu_room = q->cpu_cap == 0 || q->cpu_used + bytes <= q->cpu_cap;
        const bool selfok =
            i > 0 && t.lock[i] == 0 && t.status[i] == 0 && (!q->has_floor || t.rank[i] > q->floor);
        const bool releases = !q->offload || t.backed[i] || !cpu_room;
        flags[i] = (selfok ? 1 : 0) | (releases ? 2 : 0);
        blocked[i] = 0;
        vals[i] = i;
    }
}

// keys[k] = word `w` of node vals[k]'s `before` key (ascending = earlier).  Only the relative
// order of candidates matters downstream (ord is read for R nodes only), so non-candidates
// need no extra pass to sort last.
// WA rank word, descending.  Compact form (rank_bytes < 8, decided on the host): SUFFIX -> 0,
// UNREACHABLE -> 1, r in [0, rank_max] -> 2 + rank_max - r -- the same order in a few bytes.
__device__ __forceinline__ uint64_t rank_key(int64_t r, const BigReq* q, bool compact) {
    if (!compact) return ~(static_cast<uint64_t>(r) ^ 0x8000000000000000ull);
    if (r == kSuffix) return 0;
    if (r == kUnreach) return 1;
    return 2 + static_cast<uint64_t>(q->rank_max - r);
}

__global__ void big_gather_key(BigTree t, const BigReq* q, const uint32_t* vals, uint64_t* keys, int w,
                               bool compact_rank) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < t.n; k += gridDim.x * blockDim.x) {
        const uint32_t i = vals[k];
        uint64_t key;
        switch (w) {
            case 0: key = t.id[i]; break;
            case 1: key = t.seq[i]; break;
            case 2: key = time_order(t.time[i]); break;
            default: key = rank_key(t.rank[i], q, compact_rank); break;  // rank desc
        }
        keys[k] = key;
    }
}

__global__ void big_ord(uint32_t n, const uint32_t* vals, int32_t* ord) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) ord[vals[k]] = k;
}

__global__ void big_blocked(BigTree t, const uint8_t* flags, uint32_t* blocked) {
    for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x + 1; m < t.n; m += gridDim.x * blockDim.x) {
        const uint8_t f = flags[m];
        if (t.status[m] == 1 || ((f & 1) && (f & 2))) continue;
        for (int32_t cur = static_cast<int32_t>(m);;) {
            const int32_t p = t.parent[cur];
            if (p <= 0) break;
            if (atomicOr(&blocked[p], 1u)) break;
            if (t.status[p] == 1) break;
            cur = p;
        }
    }
}

__global__ void big_r_init(uint32_t n, uint8_t* flags, const uint32_t* blocked, const int32_t* ord, int32_t* eff) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const bool r = (flags[i] & 1) && !blocked[i];
        if (r) flags[i] |= 4;
        eff[i] = r ? ord[i] : -1;
    }
}

__global__ void big_eff(BigTree t, const uint8_t* flags, const int32_t* ord, int32_t* eff) {
    for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x + 1; m < t.n; m += gridDim.x * blockDim.x) {
        if (!(flags[m] & 4)) continue;
        const int32_t v = ord[m];
        for (int32_t cur = static_cast<int32_t>(m);;) {
            const int32_t p = t.parent[cur];
            if (p <= 0 || !(flags[p] & 4)) break;
            if (atomicMax(&eff[p], v) >= v) break;
            cur = p;
        }
    }
}

// victim key (eff asc, depth desc) in 16 + log2(n) + 1 bits; non-R nodes sort last
__global__ void big_victim_keys(BigTree t, const uint8_t* flags, const int32_t* eff, uint64_t* keys, uint32_t* vals) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < t.n; i += gridDim.x * blockDim.x) {
        keys[i] = (flags[i] & 4) ? (static_cast<uint64_t>(static_cast<uint32_t>(eff[i])) << 16) |
                                       (0xFFFFu - static_cast<uint32_t>(t.depth[i]))
                                 : ~0ull;
        vals[i] = i;
    }
}

__global__ void big_bytes(BigTree t, const BigReq* __restrict__ q, const uint64_t* keys, const uint32_t* vals,
                          uint64_t* bytes) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < t.n; k += gridDim.x * blockDim.x)
        bytes[k] = keys[k] == ~0ull ? 0 : t.tokens[vals[k]] * q->bpt;
}

// victim k is popped iff the bytes freed before it are < needed (radix_cache.cpp:335);
// idx / action go straight to mapped pinned host memory (posted writes, no D2H copy)
__global__ void big_cut(BigTree t, const BigReq* __restrict__ q, const uint64_t* keys, const uint32_t* vals,
                        const uint64_t* before, int32_t* out_idx, uint8_t* out_act, unsigned long long* header) {
    uint64_t imm = 0, pend = 0;
    uint32_t cnt = 0;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < t.n; k += gridDim.x * blockDim.x) {
        if (keys[k] == ~0ull || before[k] >= q->needed) continue;
        const uint32_t v = vals[k];
        const uint64_t bytes = t.tokens[v] * q->bpt;
        uint8_t act;
        if (!q->offload) act = KVF_ACT_REMOVE;
        else if (t.backed[v]) act = KVF_ACT_DISCARD_TO_BACKUP;
        else if (!(q->cpu_cap == 0 || q->cpu_used + bytes <= q->cpu_cap)) act = KVF_ACT_REMOVE;
        else act = KVF_ACT_OFFLOAD;
        out_idx[k] = static_cast<int32_t>(v);
        out_act[k] = act;
        (act == KVF_ACT_OFFLOAD ? pend : imm) += bytes;
        cnt = max(cnt, k + 1);
    }
    for (int o = 16; o; o >>= 1) {
        imm += __shfl_xor_sync(0xffffffffu, imm, o);
        pend += __shfl_xor_sync(0xffffffffu, pend, o);
        cnt = max(cnt, __shfl_xor_sync(0xffffffffu, cnt, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (cnt) atomicMax(header, static_cast<unsigned long long>(cnt));
        if (imm) atomicAdd(header + 1, static_cast<unsigned long long>(imm));
        if (pend) atomicAdd(header + 2, static_cast<unsigned long long>(pend));
    }
}

template <typename T>
T* take(char*& p, size_t count) {
    T* r = reinterpret_cast<T*>(p);
    p += (count * sizeof(T) + 255) & ~size_t(255);
    return r;
}

// Bucketed size: n rounded up to a quarter of its octave (<= 25 % padding), so a captured
// graph serves every tree size in the bucket.
uint32_t bucket(uint32_t n) {
    uint32_t p = 1;
    while (p * 2 <= n) p *= 2;
    const uint32_t step = std::max<uint32_t>(1024, p / 4);
    return (n + step - 1) / step * step;
}

uint32_t bits_for(uint32_t x) {  // bits to hold 0..x
    uint32_t b = 0;
    while ((1ull << b) <= x) ++b;
    return b;
}

}  // namespace

namespace kvf_impl {

int victim_select_large(kvf_engine* e, const kvf_tree_view* t, const kvf_evict_request* q, int32_t* out_idx,
                        uint8_t* out_action, uint32_t* out_count, uint64_t* out_imm, uint64_t* out_pend) {
    const uint32_t n = t->n;
    const uint32_t np = bucket(n);
    const bool wa = q->workflow_aware != 0;
    cudaStream_t s = e->s_dec;
    size_t sort_tmp = 0, scan_tmp = 0;
    KVF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, static_cast<uint64_t*>(nullptr),
                                             static_cast<uint64_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                             static_cast<uint32_t*>(nullptr), static_cast<int>(np), 0, 64, s));
    KVF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, static_cast<uint64_t*>(nullptr),
                                           static_cast<uint64_t*>(nullptr), static_cast<int>(np), s));
    const size_t in_bytes = 256 + static_cast<size_t>(np) * (8 * 5 + 4 * 2 + 2 + 2) + 16 * 256;
    const size_t out_bytes = 256 + static_cast<size_t>(np) * 5 + 2 * 256;
    const size_t work_bytes = static_cast<size_t>(np) * (1 + 4 + 4 + 4 + 8 * 2 + 4 * 2 + 8 * 2) + sort_tmp +
                              scan_tmp + 64 * 256;
    const void* old_dev = e->ws_big.dev;
    const void* old_host = e->ws_big.host;
    int rc = e->ws_big.ensure(in_bytes + work_bytes, in_bytes + out_bytes);
    if (rc) return rc;
    if (e->ws_big.dev != old_dev || e->ws_big.host != old_host) {  // graphs bake the old pointers
        for (auto& kv : e->big_graphs) cudaGraphExecDestroy(kv.second.exec);
        e->big_graphs.clear();
    }
    // ---- pack the SoA (+ padding nodes that are never candidates) and the request ----
    char* h = static_cast<char*>(e->ws_big.host);
    char* hp = h;
    BigReq* hreq = take<BigReq>(hp, 1);
    *hreq = BigReq{q->needed,       q->floor,        q->cpu_used,  q->cpu_capacity, q->workflow_aware,
                   q->offload_mode, q->has_floor, t->bytes_per_token};
    auto put = [&](auto* src, size_t elem, int fill) {
        char* dst = hp;
        std::memcpy(dst, src, n * elem);
        std::memset(dst + n * elem, fill, (np - n) * elem);
        hp += (np * elem + 255) & ~size_t(255);
    };
    put(t->rank, 8, 0);
    put(t->time, 8, 0);
    put(t->seq, 8, 0);
    put(t->id, 8, 0);
    put(t->tokens, 8, 0);
    put(t->parent, 4, 0xFF);  // parent -1: walks stop at once
    put(t->lock, 4, 0);
    put(t->depth, 2, 0);
    put(t->status, 1, 2);     // not IN_GPU: never a candidate, never R
    put(t->backed, 1, 0);
    const size_t used = static_cast<size_t>(hp - h);
    char* hout = h + ((used + 255) & ~size_t(255));
    unsigned long long* hhdr = reinterpret_cast<unsigned long long*>(hout);
    char* hout_dev = static_cast<char*>(e->ws_big.host_dev) + (hout - h);
    int32_t* o_idx = reinterpret_cast<int32_t*>(hout_dev + 256);
    uint8_t* o_act = reinterpret_cast<uint8_t*>(hout_dev + 256 + ((np * 4ull + 255) & ~255ull));

    // node ids and access sequence numbers are counters: their LSD passes only need the bytes
    // the largest one uses (8 CUB passes per 64-bit word otherwise; padding nodes hold 0)
    uint64_t max_id = 0, max_seq = 0;
    for (uint32_t i = 0; i < n; ++i) {
        max_id = std::max(max_id, t->id[i]);
        max_seq = std::max(max_seq, t->seq[i]);
    }
    auto live_bytes = [](uint64_t x) {
        uint32_t b = 1;
        while (b < 8 && (x >> (8 * b))) ++b;
        return b;
    };
    const uint32_t id_bytes = live_bytes(max_id), seq_bytes = live_bytes(max_seq);
    // WA: ranks are SUFFIX, UNREACHABLE or small step ranks (radix_cache.hpp:30-38) -> a compact
    // order-preserving code (rank_key); anything else keeps the full 64-bit word
    uint32_t rank_bytes = 8;
    if (wa) {
        int64_t rmax = 0;
        bool small = true;
        for (uint32_t i = 0; i < n && small; ++i) {
            const int64_t r = t->rank[i];
            if (r == kSuffix || r == kUnreach) continue;
            if (r < 0 || r > (int64_t{1} << 40)) small = false;
            else rmax = std::max(rmax, r);
        }
        if (small) {
            rank_bytes = live_bytes(static_cast<uint64_t>(rmax) + 2);
            hreq->rank_max = rmax;
        }
    }
    const uint64_t key = (static_cast<uint64_t>(np) << 13) | (rank_bytes << 9) | (id_bytes << 5) | (seq_bytes << 1) |
                         (wa ? 1u : 0u);
    auto git = e->big_graphs.find(key);
    if (git == e->big_graphs.end()) {
        // ---- capture the whole device-wide sequence once per (bucket, policy, key widths) ----
        char* d = static_cast<char*>(e->ws_big.dev);
        char* dp = d;
        const BigReq* dreq = take<BigReq>(dp, 1);
        BigTree bt;
        bt.rank = take<int64_t>(dp, np);
        bt.time = take<double>(dp, np);
        bt.seq = take<uint64_t>(dp, np);
        bt.id = take<uint64_t>(dp, np);
        bt.tokens = take<uint64_t>(dp, np);
        bt.parent = take<int32_t>(dp, np);
        bt.lock = take<int32_t>(dp, np);
        bt.depth = take<uint16_t>(dp, np);
        bt.status = take<uint8_t>(dp, np);
        bt.backed = take<uint8_t>(dp, np);
        bt.n = np;
        uint8_t* flags = take<uint8_t>(dp, np);
        uint32_t* blocked = take<uint32_t>(dp, np);
        int32_t* ord = take<int32_t>(dp, np);
        int32_t* eff = take<int32_t>(dp, np);
        uint64_t* keys_a = take<uint64_t>(dp, np);
        uint64_t* keys_b = take<uint64_t>(dp, np);
        uint32_t* vals_a = take<uint32_t>(dp, np);
        uint32_t* vals_b = take<uint32_t>(dp, np);
        uint64_t* bytes = take<uint64_t>(dp, np);
        uint64_t* before = take<uint64_t>(dp, np);
        unsigned long long* d_hdr = take<unsigned long long>(dp, 4);
        void* sort_scratch = take<uint8_t>(dp, sort_tmp);
        void* scan_scratch = take<uint8_t>(dp, scan_tmp);
        const uint32_t threads = 256;
        const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>((np + threads - 1) / threads, e->sm_count * 8ull));
        cudaGraph_t g = nullptr;
        KVF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        cudaMemcpyAsync(d, h, used, cudaMemcpyHostToDevice, s);
        cudaMemsetAsync(d_hdr, 0, 32, s);
        big_stage<<<grid, threads, 0, s>>>(bt, dreq, flags, blocked, vals_a);
        for (int w = 0; w < (wa ? 4 : 3); ++w) {  // stable LSD: id, seq, time, [rank desc]
            big_gather_key<<<grid, threads, 0, s>>>(bt, dreq, vals_a, keys_a, w, rank_bytes < 8);
            const int end_bit = w == 0   ? static_cast<int>(8 * id_bytes)
                                : w == 1 ? static_cast<int>(8 * seq_bytes)
                                : w == 3 ? static_cast<int>(8 * rank_bytes)
                                         : 64;
            cub::DeviceRadixSort::SortPairs(sort_scratch, sort_tmp, keys_a, keys_b, vals_a, vals_b,
                                            static_cast<int>(np), 0, end_bit, s);
            std::swap(vals_a, vals_b);
        }
        big_ord<<<grid, threads, 0, s>>>(np, vals_a, ord);
        big_blocked<<<grid, threads, 0, s>>>(bt, flags, blocked);
        big_r_init<<<grid, threads, 0, s>>>(np, flags, blocked, ord, eff);
        big_eff<<<grid, threads, 0, s>>>(bt, flags, ord, eff);
        big_victim_keys<<<grid, threads, 0, s>>>(bt, flags, eff, keys_a, vals_a);
        cub::DeviceRadixSort::SortPairs(sort_scratch, sort_tmp, keys_a, keys_b, vals_a, vals_b, static_cast<int>(np),
                                        0, static_cast<int>(17 + bits_for(np)), s);
        big_bytes<<<grid, threads, 0, s>>>(bt, dreq, keys_b, vals_b, bytes);
        cub::DeviceScan::ExclusiveSum(scan_scratch, scan_tmp, bytes, before, static_cast<int>(np), s);
        big_cut<<<grid, threads, 0, s>>>(bt, dreq, keys_b, vals_b, before, o_idx, o_act, d_hdr);
        cudaMemcpyAsync(hhdr, d_hdr, 32, cudaMemcpyDeviceToHost, s);
        const cudaError_t cap = cudaStreamEndCapture(s, &g);
        if (cap != cudaSuccess) return cuda_error(cap, "K5 graph capture");
        BigGraph bg;
        const cudaError_t inst = cudaGraphInstantiate(&bg.exec, g, 0);
        size_t nn = 0;
        cudaGraphGetNodes(g, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        cudaGraphGetNodes(g, nodes.data(), &nn);
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType ty;
            if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++bg.kernels;
        }
        cudaGraphDestroy(g);
        if (inst != cudaSuccess) return cuda_error(inst, "K5 graph instantiate");
        git = e->big_graphs.emplace(key, bg).first;
    }
    KVF_CUDA(cudaEventRecord(e->dec_start, s));
    KVF_CUDA(cudaGraphLaunch(git->second.exec, s));
    KVF_CUDA(cudaEventRecord(e->dec_stop, s));
    e->stats.kernel_launches += git->second.kernels;
    e->stats.decisions++;
    KVF_CUDA(cudaStreamSynchronize(s));
    const uint32_t cnt = static_cast<uint32_t>(hhdr[0]);
    if (cnt > n) return set_error(KVF_E_INTERNAL, "device-wide K5: victim count beyond the tree");
    std::memcpy(out_idx, hout + 256, cnt * 4ull);
    std::memcpy(out_action, hout + 256 + ((np * 4ull + 255) & ~255ull), cnt);
    *out_count = cnt;
    *out_imm = hhdr[1];
    *out_pend = hhdr[2];
    return KVF_OK;
}

}  // namespace kvf_impl
