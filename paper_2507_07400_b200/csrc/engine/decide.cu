// Decision kernels of libkvflow.so.
//
//  K4 kvf_priority_propagate -- RadixCache::set_agent_priorities (proj/src/radix_cache.cpp:266-285):
//     rank = SUFFIX everywhere, then each boundary's candidate is min-reduced along its
//     root path (64-bit atomicMin root walks, one thread per boundary agent).
//  K5 kvf_victim_select -- RadixCache::evict selection (proj/src/radix_cache.cpp:302-372).
//     The reference pops a greedy min-heap on `before` (316-321) and re-pushes a parent
//     once its last device child is gone (365-368).  Its pop order has a closed form
//     (checked against 402 reference vectors in tests/):
//        selfok(n)   = !root && lock==0 && IN_GPU && rank > floor
//        releases(c) = Discard || cpu_backed(c) || !cpu_has_room(bytes(c))
//        R(n)        = selfok(n) && every device child c (status != BACKUP) has R(c) && releases(c)
//        eff(n)      = max(ord(n), eff(device children))   ord = position in `before` order
//        victims     = R sorted by (eff asc, depth desc), cut at the first prefix whose
//                      byte sum reaches `needed`.
//     One CTA: bitonic sort of the candidates by the 4-word key, a bottom-up level sweep
//     (shared-memory atomics) for R/eff, a bitonic sort of 64-bit (eff, depth, idx) keys,
//     and a block scan for the byte cut.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "engine_internal.hpp"

using namespace kvf_impl;

namespace {

constexpr int64_t kRankSuffix = INT64_MAX / 2;
constexpr uint32_t kMaxNodesSingleCta = 4096;
constexpr int kThreads = 1024;
constexpr int32_t kBlocked = INT32_MAX;

__global__ void __launch_bounds__(kThreads) kvf_priority_kernel(const int32_t* __restrict__ parent, uint32_t n,
                                                                const int32_t* __restrict__ bidx,
                                                                const int64_t* __restrict__ cand, uint32_t m,
                                                                long long* out) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = kRankSuffix;
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < m; b += blockDim.x) {
        const long long c = cand[b];
        for (int32_t v = bidx[b]; v > 0; v = parent[v]) atomicMin(out + v, c);
    }
}

struct TreeDev {
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
    uint64_t bpt;
};

struct ReqDev {
    uint64_t needed;
    int64_t floor;
    uint64_t cpu_used, cpu_cap;
    int32_t wa, offload, has_floor;
};

struct OutDev {
    int32_t* idx;
    uint8_t* action;
    unsigned long long* header;  // [count, immediate, pending]
};

// Strict total order of radix_cache.cpp:316-321 (`before`); 0xFFFF pads sort last.
__device__ __forceinline__ bool before(const TreeDev& t, bool wa, uint32_t a, uint32_t b) {
    if (b == 0xFFFFu) return a != 0xFFFFu;
    if (a == 0xFFFFu) return false;
    if (wa) {
        const int64_t ra = __ldg(t.rank + a), rb = __ldg(t.rank + b);
        if (ra != rb) return ra > rb;
    }
    const double ta = __ldg(t.time + a), tb = __ldg(t.time + b);
    if (ta != tb) return ta < tb;
    const uint64_t sa = __ldg(t.seq + a), sb = __ldg(t.seq + b);
    if (sa != sb) return sa < sb;
    return __ldg(t.id + a) < __ldg(t.id + b);
}

__device__ __forceinline__ void bitonic_idx(uint16_t* a, uint32_t P, const TreeDev& t, bool wa) {
    for (uint32_t k = 2; k <= P; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                const uint32_t l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const uint16_t x = a[i], y = a[l];
                    if (before(t, wa, y, x) == up) {
                        a[i] = y;
                        a[l] = x;
                    }
                }
            }
            __syncthreads();
        }
}

__device__ __forceinline__ void bitonic_u64(uint64_t* a, uint32_t P) {
    for (uint32_t k = 2; k <= P; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                const uint32_t l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const uint64_t x = a[i], y = a[l];
                    if ((y < x) == up) {
                        a[i] = y;
                        a[l] = x;
                    }
                }
            }
            __syncthreads();
        }
}

__host__ __device__ inline uint32_t pow2_ceil(uint32_t x) {
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

// dynamic smem layout for n <= 4096 (P = 4096):
//   keys u64[P] | pref u64[P] | ord i32[n] | cmax i32[n] | sel u16[P] | flags u8[n]
__global__ void __launch_bounds__(kThreads) kvf_victim_kernel(const TreeDev t, const ReqDev q, OutDev o) {
    extern __shared__ __align__(16) uint8_t sm[];
    const uint32_t n = t.n;
    const uint32_t PN = pow2_ceil(n > 1 ? n : 2);
    uint64_t* keys = reinterpret_cast<uint64_t*>(sm);
    uint64_t* pref = keys + PN;
    int32_t* ord = reinterpret_cast<int32_t*>(pref + PN);
    int32_t* cmax = ord + n;
    uint16_t* sel = reinterpret_cast<uint16_t*>(cmax + n);
    uint8_t* flags = reinterpret_cast<uint8_t*>(sel + PN);  // bit0 selfok, bit2 R (owner-written only)
    __shared__ uint32_t s_cnt, s_rcnt, s_maxd;
    __shared__ unsigned long long s_imm, s_pend, s_warp[kThreads / 32];
    if (threadIdx.x == 0) {
        s_cnt = 0;
        s_rcnt = 0;
        s_maxd = 0;
        s_imm = 0;
        s_pend = 0;
    }
    __syncthreads();
    // 1. self-eligibility (radix_cache.cpp:305-312 minus the device-child test) + compaction
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        uint8_t f = 0;
        if (i > 0 && t.lock[i] == 0 && t.status[i] == 0 && (!q.has_floor || t.rank[i] > q.floor)) f = 1;
        flags[i] = f;
        cmax[i] = -1;
        ord[i] = -1;
        if (f) sel[atomicAdd(&s_cnt, 1u)] = static_cast<uint16_t>(i);
        if (i > 0) atomicMax(&s_maxd, static_cast<uint32_t>(t.depth[i]));
    }
    __syncthreads();
    const uint32_t c = s_cnt;
    const uint32_t P = pow2_ceil(c > 1 ? c : 2);
    for (uint32_t i = c + threadIdx.x; i < P; i += blockDim.x) sel[i] = 0xFFFFu;
    __syncthreads();
    // 2. candidates in `before` order -> ord
    bitonic_idx(sel, P, t, q.wa != 0);
    for (uint32_t k = threadIdx.x; k < c; k += blockDim.x) ord[sel[k]] = static_cast<int32_t>(k);
    __syncthreads();
    // 3. bottom-up level sweep: R(n) and eff(n); a blocked or non-releasing device child
    //    pins its parent (has_device_child, radix_cache.cpp:40-45) by raising the parent's
    //    child-max to kBlocked.
    for (int d = static_cast<int>(s_maxd); d >= 1; --d) {
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            if (t.depth[i] != d) continue;
            const uint8_t f = flags[i];
            const bool r = (f & 1) && cmax[i] != kBlocked;
            const int32_t e = r ? max(ord[i], cmax[i]) : -1;
            if (r) {
                flags[i] = f | 4;
                cmax[i] = e;  // cmax now holds eff(i)
            }
            if (t.status[i] != 1) {
                const uint64_t bytes = t.tokens[i] * t.bpt;
                const bool cpu_room = q.cpu_cap == 0 || q.cpu_used + bytes <= q.cpu_cap;
                const bool releases = !q.offload || t.backed[i] || !cpu_room;
                const int32_t p = t.parent[i];
                atomicMax(&cmax[p], (r && releases) ? e : kBlocked);
            }
        }
        __syncthreads();
    }
    // 4. R nodes keyed by (eff asc, depth desc, idx) -- unique per node
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        if (flags[i] & 4) {
            const uint64_t key = (static_cast<uint64_t>(cmax[i]) << 32) |
                                 (static_cast<uint64_t>(0xFFFFu - t.depth[i]) << 16) | i;
            keys[atomicAdd(&s_rcnt, 1u)] = key;
        }
    }
    __syncthreads();
    const uint32_t r = s_rcnt;
    const uint32_t PR = pow2_ceil(r > 1 ? r : 2);
    for (uint32_t i = r + threadIdx.x; i < PR; i += blockDim.x) keys[i] = ~0ull;
    __syncthreads();
    bitonic_u64(keys, PR);
    // 5. exclusive byte prefix in victim order (block scan, 4 items/thread max)
    const uint32_t per = (r + blockDim.x - 1) / blockDim.x;
    uint64_t local = 0;
    for (uint32_t k = threadIdx.x * per; k < min(r, (threadIdx.x + 1) * per); ++k) {
        const uint32_t v = static_cast<uint32_t>(keys[k] & 0xFFFFu);
        local += t.tokens[v] * t.bpt;
    }
    uint64_t inc = local;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint64_t w = lane < blockDim.x / 32 ? s_warp[lane] : 0;
        for (int off = 1; off < 32; off <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= off) w += y;
        }
        if (lane < blockDim.x / 32) s_warp[lane] = w;
    }
    __syncthreads();
    uint64_t run = inc - local + (warp ? s_warp[warp - 1] : 0);
    // 6. cut: victim k is popped iff the bytes freed before it are < needed
    //    (the loop condition of radix_cache.cpp:335)
    for (uint32_t k = threadIdx.x * per; k < min(r, (threadIdx.x + 1) * per); ++k) {
        const uint32_t v = static_cast<uint32_t>(keys[k] & 0xFFFFu);
        const uint64_t bytes = t.tokens[v] * t.bpt;
        if (run < q.needed) {
            uint8_t act;
            if (!q.offload) act = KVF_ACT_REMOVE;
            else if (t.backed[v]) act = KVF_ACT_DISCARD_TO_BACKUP;
            else if (!(q.cpu_cap == 0 || q.cpu_used + bytes <= q.cpu_cap)) act = KVF_ACT_REMOVE;
            else act = KVF_ACT_OFFLOAD;
            o.idx[k] = static_cast<int32_t>(v);
            o.action[k] = act;
            if (act == KVF_ACT_OFFLOAD) atomicAdd(&s_pend, static_cast<unsigned long long>(bytes));
            else atomicAdd(&s_imm, static_cast<unsigned long long>(bytes));
            pref[k] = 1;
        } else {
            pref[k] = 0;
        }
        run += bytes;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t cnt = 0;
        // taken victims form a prefix; count them
        uint32_t lo = 0, hi = r;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) / 2;
            if (pref[mid]) lo = mid + 1; else hi = mid;
        }
        cnt = lo;
        o.header[0] = cnt;
        o.header[1] = s_imm;
        o.header[2] = s_pend;
    }
}

size_t victim_smem(uint32_t n) {
    const uint32_t PN = pow2_ceil(n > 1 ? n : 2);
    return PN * 8 * 2 + static_cast<size_t>(n) * 4 * 2 + PN * 2 + ((n + 3) & ~3u) + 16;
}

template <typename T>
T* carve(char*& p, size_t count) {
    T* r = reinterpret_cast<T*>(p);
    p += (count * sizeof(T) + 15) & ~size_t(15);
    return r;
}

}  // namespace

extern "C" {

int kvf_priority_propagate(kvf_engine* e, const int32_t* parent, uint32_t n, const int32_t* bidx,
                           const int64_t* cand, uint32_t m, int64_t* out_rank) {
    if (!e || !parent || !out_rank || (m && (!bidx || !cand))) return set_error(KVF_E_INVALID_ARG, "null argument");
    std::lock_guard<std::mutex> lk(e->mu);
    if (cudaSetDevice(e->device) != cudaSuccess) return set_error(KVF_E_CUDA, "cudaSetDevice failed");
    if (n == 0) return KVF_OK;
    for (uint32_t b = 0; b < m; ++b)
        if (bidx[b] < 0 || static_cast<uint32_t>(bidx[b]) >= n) return set_error(KVF_E_UNKNOWN_BOUNDARY_NODE, "boundary index out of range");
    const size_t in_bytes = ((n * 4 + 15) & ~15ull) + ((m * 4 + 15) & ~15ull) + m * 8 + 16;
    const size_t out_bytes = n * 8;
    int rc = e->ws_dec.ensure(in_bytes + out_bytes + 1024, in_bytes + 1024);
    if (rc) return rc;
    char* h = static_cast<char*>(e->ws_dec.host);
    char* hp = h;
    std::memcpy(carve<int32_t>(hp, n), parent, n * 4);
    std::memcpy(carve<int32_t>(hp, m), bidx, m * 4);
    std::memcpy(carve<int64_t>(hp, m), cand, m * 8);
    const size_t used = static_cast<size_t>(hp - h);
    char* d = static_cast<char*>(e->ws_dec.dev);
    char* dp = d;
    int32_t* d_parent = carve<int32_t>(dp, n);
    int32_t* d_bidx = carve<int32_t>(dp, m);
    int64_t* d_cand = carve<int64_t>(dp, m);
    long long* d_out = reinterpret_cast<long long*>(d + ((used + 255) & ~size_t(255)));
    KVF_CUDA(cudaMemcpyAsync(d, h, used, cudaMemcpyHostToDevice, e->s_dec));
    kvf_priority_kernel<<<1, kThreads, 0, e->s_dec>>>(d_parent, n, d_bidx, d_cand, m, d_out);
    KVF_CUDA(cudaGetLastError());
    e->stats.kernel_launches++;
    e->stats.decisions++;
    KVF_CUDA(cudaMemcpyAsync(out_rank, d_out, n * 8, cudaMemcpyDeviceToHost, e->s_dec));
    KVF_CUDA(cudaStreamSynchronize(e->s_dec));
    return KVF_OK;
}

int kvf_victim_select(kvf_engine* e, const kvf_tree_view* t, const kvf_evict_request* q, int32_t* out_idx,
                      uint8_t* out_action, uint32_t* out_count, uint64_t* out_imm, uint64_t* out_pend) {
    if (!e || !t || !q || !out_idx || !out_action || !out_count || !out_imm || !out_pend)
        return set_error(KVF_E_INVALID_ARG, "null argument");
    std::lock_guard<std::mutex> lk(e->mu);
    if (cudaSetDevice(e->device) != cudaSuccess) return set_error(KVF_E_CUDA, "cudaSetDevice failed");
    const uint32_t n = t->n;
    *out_count = 0;
    *out_imm = *out_pend = 0;
    if (n <= 1 || q->needed == 0) return KVF_OK;
    if (n > kMaxNodesSingleCta)
        return set_error(KVF_E_TOO_LARGE, "victim selection above 4096 nodes needs the multi-CTA path");
    // pack the SoA snapshot into one pinned buffer -> one H2D copy
    const size_t in_bytes = 5 * ((n * 8 + 15) & ~15ull) + 2 * ((n * 4 + 15) & ~15ull) + ((n * 2 + 15) & ~15ull) +
                            2 * ((n + 15) & ~15ull);
    const size_t out_bytes = 64 + ((n * 4 + 15) & ~15ull) + ((n + 15) & ~15ull);
    int rc = e->ws_dec.ensure(in_bytes + out_bytes + 512, in_bytes + out_bytes + 512);
    if (rc) return rc;
    char* h = static_cast<char*>(e->ws_dec.host);
    char* hp = h;
    std::memcpy(carve<int64_t>(hp, n), t->rank, n * 8);
    std::memcpy(carve<double>(hp, n), t->time, n * 8);
    std::memcpy(carve<uint64_t>(hp, n), t->seq, n * 8);
    std::memcpy(carve<uint64_t>(hp, n), t->id, n * 8);
    std::memcpy(carve<uint64_t>(hp, n), t->tokens, n * 8);
    std::memcpy(carve<int32_t>(hp, n), t->parent, n * 4);
    std::memcpy(carve<int32_t>(hp, n), t->lock, n * 4);
    std::memcpy(carve<uint16_t>(hp, n), t->depth, n * 2);
    std::memcpy(carve<uint8_t>(hp, n), t->status, n);
    std::memcpy(carve<uint8_t>(hp, n), t->backed, n);
    const size_t used = static_cast<size_t>(hp - h);
    char* d = static_cast<char*>(e->ws_dec.dev);
    char* dp = d;
    TreeDev td;
    td.rank = carve<int64_t>(dp, n);
    td.time = carve<double>(dp, n);
    td.seq = carve<uint64_t>(dp, n);
    td.id = carve<uint64_t>(dp, n);
    td.tokens = carve<uint64_t>(dp, n);
    td.parent = carve<int32_t>(dp, n);
    td.lock = carve<int32_t>(dp, n);
    td.depth = carve<uint16_t>(dp, n);
    td.status = carve<uint8_t>(dp, n);
    td.backed = carve<uint8_t>(dp, n);
    td.n = n;
    td.bpt = t->bytes_per_token;
    char* dout = d + ((used + 255) & ~size_t(255));
    OutDev od;
    od.header = reinterpret_cast<unsigned long long*>(dout);
    od.idx = reinterpret_cast<int32_t*>(dout + 64);
    od.action = reinterpret_cast<uint8_t*>(dout + 64 + ((n * 4 + 15) & ~15ull));
    ReqDev rq{q->needed, q->floor, q->cpu_used, q->cpu_capacity, q->workflow_aware, q->offload_mode, q->has_floor};
    KVF_CUDA(cudaMemcpyAsync(d, h, used, cudaMemcpyHostToDevice, e->s_dec));
    const size_t smem = victim_smem(n);
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        KVF_CUDA(cudaFuncSetAttribute(kvf_victim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(victim_smem(kMaxNodesSingleCta))));
        attr = victim_smem(kMaxNodesSingleCta);
    }
    kvf_victim_kernel<<<1, kThreads, smem, e->s_dec>>>(td, rq, od);
    KVF_CUDA(cudaGetLastError());
    e->stats.kernel_launches++;
    e->stats.decisions++;
    char* hout = h + ((used + 255) & ~size_t(255));
    KVF_CUDA(cudaMemcpyAsync(hout, dout, out_bytes, cudaMemcpyDeviceToHost, e->s_dec));
    KVF_CUDA(cudaStreamSynchronize(e->s_dec));
    const uint64_t* hdr = reinterpret_cast<const uint64_t*>(hout);
    const uint32_t cnt = static_cast<uint32_t>(hdr[0]);
    std::memcpy(out_idx, hout + 64, cnt * 4);
    std::memcpy(out_action, hout + 64 + ((n * 4 + 15) & ~15ull), cnt);
    *out_count = cnt;
    *out_imm = hdr[1];
    *out_pend = hdr[2];
    return KVF_OK;
}

}  // extern "C"
