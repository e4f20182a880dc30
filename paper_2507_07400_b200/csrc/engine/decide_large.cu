// K5, device-wide path for trees above the single-CTA limit (4096 slots).  Hand-written
// grid kernels, no library sort.
//
// Same closed form as the single-CTA kernel (decide_body.cuh), reorganised so
// only ONE sort is needed:
//   1. flags per node (self-eligible, releases-parent); candidates compacted      -- 1 kernel
//   2. blocked root walks -> R                                                    -- 1 kernel
//   3. `before` order of the candidates (radix_cache.cpp:316-321) by a stable LSD radix
//      sort, 8-bit digits, least significant word first: id, seq, [time], [rank desc] --
//      each word only over the bytes its largest value uses; time is skipped when access
//      times follow access sequence numbers (the cache says so)                    -- 3 kernels/digit
//   4. ord[x] = sorted position; eff(n) = max ord over n's R-subtree by root walks -- 2 kernels
//   5. victims WITHOUT a second sort: R sorted by (eff asc, depth desc) is a sequence of
//      chains -- each R node y with eff(y) = ord(y) heads the chain y, parent(y), ... of the
//      ancestors whose eff is ord(y), deepest first -- and the chain heads come in sorted
//      position order.  So: chain bytes per sorted position, an exclusive scan, and every chain
//      member whose bytes-before is < needed is a victim (radix_cache.cpp:335)      -- 3 kernels
// Everything is captured once per (padded size, key widths, policy) as a CUDA graph; the
// request lives in device memory, so a call = request upload + graph launch + one sync.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "engine_internal.hpp"

using namespace kvf_impl;

namespace {

constexpr int64_t kSuffix = INT64_MAX / 2;
constexpr int64_t kUnreach = INT64_MAX / 4;
constexpr uint32_t kTile = 2048;  // radix tile: 256 threads x 8 elements
constexpr uint32_t kThr = 256;

struct BigReq {  // device memory, uploaded per call
    uint64_t needed;
    int64_t floor;
    uint64_t cpu_used, cpu_cap;
    int32_t wa, offload, has_floor, pad;
    uint64_t bpt;
    int64_t rank_max;  // compact WA rank code: SUFFIX -> 0, UNREACHABLE -> 1, r -> 2 + rank_max - r
};

struct Hdr {  // device memory, zeroed per call
    unsigned long long count, imm, pend, cands;
};

__device__ __forceinline__ uint64_t time_order(double t) {
    const uint64_t b = t == 0.0 ? 0ull : static_cast<uint64_t>(__double_as_longlong(t));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// 1. flags (bit0 selfok, bit1 releases), blocked = 0, ord = -1; candidates -> vals (any order:
//    the sort key is total, ids are unique)
__global__ void __launch_bounds__(kThr) big_stage(LargeArrays a, uint32_t np, const BigReq* __restrict__ q,
                                                  uint8_t* flags, uint32_t* blocked, int32_t* ord, uint32_t* vals,
                                                  Hdr* hdr) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
        const uint64_t bytes = a.tokens[i] * q->bpt;
        const bool cpu_room = q->cpu_cap == 0 || q->cpu_used + bytes <= q->cpu_cap;
        const bool selfok = i > 0 && a.status[i] == 0 && a.lock[i] == 0 && (!q->has_floor || a.rank[i] > q->floor);
        const bool releases = !q->offload || a.backed[i] || !cpu_room;
        flags[i] = (selfok ? 1 : 0) | (releases ? 2 : 0);
        blocked[i] = 0;
        ord[i] = -1;
        // warp-aggregated slot in the candidate list
        const unsigned act = __activemask();
        const unsigned mask = __ballot_sync(act, selfok);
        const int leader = __ffs(act) - 1;
        const int lane = threadIdx.x & 31;
        unsigned long long base = 0;
        if (lane == leader && mask) base = atomicAdd(&hdr->cands, static_cast<unsigned long long>(__popc(mask)));
        base = __shfl_sync(act, base, leader);
        if (selfok) vals[base + __popc(mask & ((1u << lane) - 1u))] = i;
    }
}

// 2. blocked(p): some device node below p is not self-eligible or would not release it
//    (has_device_child, radix_cache.cpp:40-45); walkers stop where another already passed
__global__ void __launch_bounds__(kThr) big_blocked(LargeArrays a, uint32_t np, const uint8_t* flags, uint32_t* blocked) {
    for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x + 1; m < np; m += gridDim.x * blockDim.x) {
        const uint8_t f = flags[m];
        const uint8_t s = a.status[m];
        if (s == 1 || s == KVF_SLOT_DEAD || ((f & 1) && (f & 2))) continue;
        for (int32_t cur = static_cast<int32_t>(m);;) {
            const int32_t p = a.parent[cur];
            if (p <= 0) break;
            if (atomicOr(&blocked[p], 1u)) break;
            if (a.status[p] == 1) break;
            cur = p;
        }
    }
}

// 3. one 8-bit digit of the `before` key; word w: 0 id, 1 seq, 2 time, 3 rank (descending)
__device__ __forceinline__ uint32_t digit(const LargeArrays& a, const BigReq* q, uint32_t node, int w, int byte,
                                          bool compact_rank) {
    uint64_t k;
    switch (w) {
        case 0: k = a.id[node]; break;
        case 1: k = a.seq[node]; break;
        case 2: k = time_order(a.time[node]); break;
        default: {
            const int64_t r = a.rank[node];
            if (!compact_rank) k = ~(static_cast<uint64_t>(r) ^ 0x8000000000000000ull);
            else if (r == kSuffix) k = 0;
            else if (r == kUnreach) k = 1;
            else k = 2 + static_cast<uint64_t>(q->rank_max - r);
        }
    }
    return static_cast<uint32_t>(k >> (8 * byte)) & 0xFFu;
}

__global__ void __launch_bounds__(kThr) big_hist(LargeArrays a, const BigReq* q, const uint32_t* vals, const Hdr* hdr,
                                                 uint32_t* hist, int w, int byte, bool compact) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t c = static_cast<uint32_t>(hdr->cands);
    const uint32_t base = blockIdx.x * kTile;
    if (base < c) {
        for (uint32_t k = base + threadIdx.x; k < min(c, base + kTile); k += kThr)
            atomicAdd(&h[digit(a, q, vals[k], w, byte, compact)], 1u);
    }
    __syncthreads();
    hist[blockIdx.x * 256 + threadIdx.x] = h[threadIdx.x];
}

// offsets[t][d] = (elements with digit < d) + (digit-d elements of tiles < t); in place
__global__ void __launch_bounds__(kThr) big_offsets(uint32_t* hist, uint32_t tiles) {
    __shared__ uint32_t tot[256];
    const uint32_t d = threadIdx.x;
    uint32_t run = 0;
    for (uint32_t t = 0; t < tiles; ++t) {
        const uint32_t v = hist[t * 256 + d];
        hist[t * 256 + d] = run;
        run += v;
    }
    tot[d] = run;
    __syncthreads();
    for (uint32_t off = 1; off < 256; off <<= 1) {  // inclusive scan over digits
        const uint32_t y = d >= off ? tot[d - off] : 0;
        __syncthreads();
        tot[d] += y;
        __syncthreads();
    }
    const uint32_t base = tot[d] - run;
    for (uint32_t t = 0; t < tiles; ++t) hist[t * 256 + d] += base;
}

// stable scatter: a tile in 8 rounds of 256 elements in index order; within a round, equal
// digits are ranked by warp (match) and lane
__global__ void __launch_bounds__(kThr) big_scatter(LargeArrays a, const BigReq* q, const uint32_t* vin, uint32_t* vout,
                                                    const Hdr* hdr, const uint32_t* offsets, int w, int byte,
                                                    bool compact) {
    __shared__ uint32_t run[256];
    __shared__ uint16_t cnt[kThr / 32][256];
    const uint32_t c = static_cast<uint32_t>(hdr->cands);
    const uint32_t base = blockIdx.x * kTile;
    if (base >= c) return;  // uniform per CTA
    run[threadIdx.x] = offsets[blockIdx.x * 256 + threadIdx.x];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t r = 0; r < kTile / kThr; ++r) {
        for (uint32_t w8 = 0; w8 < kThr / 32; ++w8) cnt[w8][threadIdx.x] = 0;
        __syncthreads();
        const uint32_t k = base + r * kThr + threadIdx.x;
        const bool live = k < c;
        uint32_t v = 0, d = 256;
        if (live) {
            v = vin[k];
            d = digit(a, q, v, w, byte, compact);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t rk = __popc(peers & ((1u << lane) - 1u));
        if (live && rk == 0) cnt[warp][d] = static_cast<uint16_t>(__popc(peers));
        __syncthreads();
        if (live) {
            uint32_t pre = 0;
            for (uint32_t w8 = 0; w8 < warp; ++w8) pre += cnt[w8][d];
            vout[run[d] + pre + rk] = v;
        }
        __syncthreads();
        uint32_t add = 0;
        for (uint32_t w8 = 0; w8 < kThr / 32; ++w8) add += cnt[w8][threadIdx.x];
        run[threadIdx.x] += add;
        __syncthreads();
    }
}

// 4. ord, R, eff
__global__ void __launch_bounds__(kThr) big_ord(const uint32_t* vals, const Hdr* hdr, int32_t* ord) {
    const uint32_t c = static_cast<uint32_t>(hdr->cands);
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < c; k += gridDim.x * blockDim.x)
        ord[vals[k]] = static_cast<int32_t>(k);
}

__global__ void __launch_bounds__(kThr) big_r_init(uint32_t np, uint8_t* flags, const uint32_t* blocked,
                                                   const int32_t* ord, int32_t* eff) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
        const bool r = (flags[i] & 1) && !blocked[i];
        if (r) flags[i] |= 4;
        eff[i] = r ? ord[i] : -1;
    }
}

__global__ void __launch_bounds__(kThr) big_eff(LargeArrays a, uint32_t np, const uint8_t* flags, const int32_t* ord,
                                                int32_t* eff) {
    for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x + 1; m < np; m += gridDim.x * blockDim.x) {
        if (!(flags[m] & 4)) continue;
        const int32_t v = ord[m];
        for (int32_t cur = static_cast<int32_t>(m);;) {
            const int32_t p = a.parent[cur];
            if (p <= 0 || !(flags[p] & 4)) break;
            if (atomicMax(&eff[p], v) >= v) break;
            cur = p;
        }
    }
}

// 5. chains.  Sorted position k heads a chain iff its node y is in R and eff(y) == k.
__device__ __forceinline__ bool chain_head(const uint32_t* vals, const uint8_t* flags, const int32_t* eff, uint32_t k,
                                           uint32_t c, uint32_t* y) {
    if (k >= c) return false;
    *y = vals[k];
    return (flags[*y] & 4) && eff[*y] == static_cast<int32_t>(k);
}

template <typename F>
__device__ __forceinline__ void walk_chain(const LargeArrays& a, const uint8_t* flags, const int32_t* eff, uint32_t y,
                                           int32_t k, F f) {
    for (int32_t cur = static_cast<int32_t>(y);;) {
        f(static_cast<uint32_t>(cur));
        const int32_t p = a.parent[cur];
        if (p <= 0 || !(flags[p] & 4) || eff[p] != k) break;
        cur = p;
    }
}

// Block-wide exclusive scan of (bytes, count) pairs, kTile per block (8 per thread, in order).
struct Pair {
    unsigned long long b;
    uint32_t n;
};
__device__ __forceinline__ Pair block_excl(Pair mine, Pair* total) {
    __shared__ unsigned long long sb[kThr / 32];
    __shared__ uint32_t sn[kThr / 32];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Pair inc = mine;
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned long long yb = __shfl_up_sync(0xffffffffu, inc.b, off);
        const uint32_t yn = __shfl_up_sync(0xffffffffu, inc.n, off);
        if (lane >= static_cast<uint32_t>(off)) {
            inc.b += yb;
            inc.n += yn;
        }
    }
    if (lane == 31) {
        sb[warp] = inc.b;
        sn[warp] = inc.n;
    }
    __syncthreads();
    Pair before{0, 0}, all{0, 0};
    for (uint32_t w8 = 0; w8 < kThr / 32; ++w8) {
        if (w8 < warp) {
            before.b += sb[w8];
            before.n += sn[w8];
        }
        all.b += sb[w8];
        all.n += sn[w8];
    }
    __syncthreads();
    if (total) *total = all;
    return Pair{before.b + inc.b - mine.b, before.n + inc.n - mine.n};
}

__device__ __forceinline__ Pair thread_chunk(const LargeArrays& a, const BigReq* q, const uint32_t* vals,
                                             const uint8_t* flags, const int32_t* eff, uint32_t c, uint32_t k0,
                                             Pair* per /* [8] or null */) {
    Pair s{0, 0};
    for (uint32_t j = 0; j < kTile / kThr; ++j) {
        uint32_t y;
        Pair p{0, 0};
        if (chain_head(vals, flags, eff, k0 + j, c, &y))
            walk_chain(a, flags, eff, y, static_cast<int32_t>(k0 + j), [&](uint32_t v) {
                p.b += a.tokens[v] * q->bpt;
                p.n += 1;
            });
        if (per) per[j] = p;
        s.b += p.b;
        s.n += p.n;
    }
    return s;
}

__global__ void __launch_bounds__(kThr) big_tile_sums(LargeArrays a, const BigReq* q, const uint32_t* vals,
                                                      const uint8_t* flags, const int32_t* eff, const Hdr* hdr,
                                                      Pair* tsum) {
    const uint32_t c = static_cast<uint32_t>(hdr->cands);
    const uint32_t k0 = blockIdx.x * kTile + threadIdx.x * (kTile / kThr);
    Pair tot;
    block_excl(thread_chunk(a, q, vals, flags, eff, c, k0, nullptr), &tot);
    if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kThr) big_tile_scan(Pair* tsum, uint32_t tiles) {
    if (threadIdx.x == 0) {  // tiles <= ~100: serial is shorter than a block scan's barriers
        Pair run{0, 0};
        for (uint32_t t = 0; t < tiles; ++t) {
            const Pair v = tsum[t];
            tsum[t] = run;
            run.b += v.b;
            run.n += v.n;
        }
    }
}

// every chain member whose bytes-before is still < needed is popped (radix_cache.cpp:335);
// slots and actions go straight to mapped pinned memory
__global__ void __launch_bounds__(kThr) big_emit(LargeArrays a, const BigReq* q, const uint32_t* vals,
                                                 const uint8_t* flags, const int32_t* eff, Hdr* hdr, const Pair* tsum,
                                                 uint32_t* out_idx, uint8_t* out_act) {
    // a tile whose bytes-before already reach `needed` pops nothing: skip its chain walks
    if (tsum[blockIdx.x].b >= q->needed) return;  // uniform per CTA
    const uint32_t c = static_cast<uint32_t>(hdr->cands);
    const uint32_t k0 = blockIdx.x * kTile + threadIdx.x * (kTile / kThr);
    Pair per[kTile / kThr];
    const Pair mine = thread_chunk(a, q, vals, flags, eff, c, k0, per);
    Pair pre = block_excl(mine, nullptr);
    pre.b += tsum[blockIdx.x].b;
    pre.n += tsum[blockIdx.x].n;
    if (pre.b >= q->needed) return;
    unsigned long long imm = 0, pend = 0, cnt = 0;
    for (uint32_t j = 0; j < kTile / kThr && pre.b < q->needed; ++j) {
        uint32_t y;
        if (per[j].n && chain_head(vals, flags, eff, k0 + j, c, &y)) {
            walk_chain(a, flags, eff, y, static_cast<int32_t>(k0 + j), [&](uint32_t v) {
                const uint64_t bytes = a.tokens[v] * q->bpt;
                if (pre.b < q->needed) {
                    uint8_t act;
                    if (!q->offload) act = KVF_ACT_REMOVE;
                    else if (a.backed[v]) act = KVF_ACT_DISCARD_TO_BACKUP;
                    else if (!(q->cpu_cap == 0 || q->cpu_used + bytes <= q->cpu_cap)) act = KVF_ACT_REMOVE;
                    else act = KVF_ACT_OFFLOAD;
                    out_idx[pre.n] = v;
                    out_act[pre.n] = act;
                    (act == KVF_ACT_OFFLOAD ? pend : imm) += bytes;
                    cnt = max(cnt, static_cast<unsigned long long>(pre.n) + 1);
                }
                pre.b += bytes;
                pre.n += 1;
            });
        }
    }
    if (cnt) atomicMax(&hdr->count, cnt);
    if (imm) atomicAdd(&hdr->imm, imm);
    if (pend) atomicAdd(&hdr->pend, pend);
}

template <typename T>
T* take(char*& p, size_t count) {
    T* r = reinterpret_cast<T*>(p);
    p += (count * sizeof(T) + 255) & ~size_t(255);
    return r;
}

uint32_t live_bytes(uint64_t x) {
    uint32_t b = 1;
    while (b < 8 && (x >> (8 * b))) ++b;
    return b;
}

}  // namespace

namespace kvf_impl {

// Padded size: n rounded up to a quarter of its octave (<= 25 % padding), so one captured
// graph serves every tree size in the bucket; a multiple of the radix tile.
uint32_t large_capacity(uint32_t n) {
    uint32_t p = 1;
    while (p * 2 <= n) p *= 2;
    const uint32_t step = std::max<uint32_t>(kTile, p / 4);
    return (n + step - 1) / step * step;
}

void large_invalidate(LargeState& st) {
    for (auto& kv : st.graphs) cudaGraphExecDestroy(kv.second.exec);
    st.graphs.clear();
    st.baked = nullptr;
}

void large_release(LargeState& st) {
    large_invalidate(st);
    st.ws.release();
}

int victim_large(kvf_engine* e, LargeState& st, const LargeArrays& a, const kvf_evict_request* q, uint64_t bpt,
                 const LargeKeyInfo& keys, uint32_t* out_idx, uint8_t* out_action, uint32_t cap, uint32_t* out_count,
                 uint64_t* out_imm, uint64_t* out_pend) {
    const uint32_t np = large_capacity(a.n);
    const uint32_t tiles = np / kTile;
    const bool wa = q->workflow_aware != 0;
    cudaStream_t s = e->s_dec;
    const size_t work = 256 * 8 + static_cast<size_t>(np) * (1 + 4 + 4 + 4 + 4 + 4) + static_cast<size_t>(tiles) * (256 * 4 + 16) +
                        16 * 256;
    const size_t host = 512 + static_cast<size_t>(np) * 5 + 2 * 256;
    const void* old_dev = st.ws.dev;
    const void* old_host = st.ws.host;
    if (int rc = st.ws.ensure(work, host)) return rc;
    if (st.ws.dev != old_dev || st.ws.host != old_host || st.baked != a.parent) large_invalidate(st);
    st.baked = a.parent;
    // key widths (padding slots hold 0s)
    const uint32_t id_bytes = live_bytes(keys.max_id), seq_bytes = live_bytes(keys.max_seq);
    const bool compact = keys.rank_small;
    const uint32_t rank_bytes = compact ? live_bytes(static_cast<uint64_t>(keys.rank_max) + 2) : 8;
    const bool skip_time = keys.time_follows_seq;
    const uint64_t key = (static_cast<uint64_t>(np) << 16) | (rank_bytes << 12) | (id_bytes << 8) | (seq_bytes << 4) |
                         (skip_time ? 2u : 0u) | (wa ? 1u : 0u);
    char* h = static_cast<char*>(st.ws.host);
    BigReq* hreq = reinterpret_cast<BigReq*>(h);
    *hreq = BigReq{q->needed, q->floor, q->cpu_used, q->cpu_capacity, q->workflow_aware, q->offload_mode,
                   q->has_floor, 0, bpt, keys.rank_max};
    char* hout = h + 512;
    uint32_t* h_idx = reinterpret_cast<uint32_t*>(hout);
    uint8_t* h_act = reinterpret_cast<uint8_t*>(hout + ((np * 4ull + 255) & ~255ull));
    Hdr* h_hdr = reinterpret_cast<Hdr*>(h + 256);
    char* hdev = static_cast<char*>(st.ws.host_dev);
    uint32_t* o_idx = reinterpret_cast<uint32_t*>(hdev + 512);
    uint8_t* o_act = reinterpret_cast<uint8_t*>(hdev + 512 + ((np * 4ull + 255) & ~255ull));
    char* d = static_cast<char*>(st.ws.dev);
    auto git = st.graphs.find(key);
    if (git == st.graphs.end()) {
        char* dp = d;
        BigReq* dreq = take<BigReq>(dp, 1);
        Hdr* dhdr = take<Hdr>(dp, 1);
        uint8_t* flags = take<uint8_t>(dp, np);
        uint32_t* blocked = take<uint32_t>(dp, np);
        int32_t* ord = take<int32_t>(dp, np);
        int32_t* eff = take<int32_t>(dp, np);
        uint32_t* va = take<uint32_t>(dp, np);
        uint32_t* vb = take<uint32_t>(dp, np);
        uint32_t* hist = take<uint32_t>(dp, static_cast<size_t>(tiles) * 256);
        Pair* tsum = take<Pair>(dp, tiles);
        LargeArrays ga = a;
        const uint32_t grid = std::min<uint32_t>((np + kThr - 1) / kThr, static_cast<uint32_t>(e->sm_count) * 8);
        cudaGraph_t g = nullptr;
        KVF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        cudaMemsetAsync(dhdr, 0, sizeof(Hdr), s);
        big_stage<<<grid, kThr, 0, s>>>(ga, np, dreq, flags, blocked, ord, va, dhdr);
        big_blocked<<<grid, kThr, 0, s>>>(ga, np, flags, blocked);
        // stable LSD: id, seq, [time], [rank desc], least significant byte first
        struct W {
            int w;
            uint32_t bytes;
        };
        W words[4] = {{0, id_bytes}, {1, seq_bytes}, {2, skip_time ? 0u : 8u}, {3, wa ? rank_bytes : 0u}};
        for (const W& wd : words)
            for (uint32_t b = 0; b < wd.bytes; ++b) {
                big_hist<<<tiles, kThr, 0, s>>>(ga, dreq, va, dhdr, hist, wd.w, static_cast<int>(b), compact);
                big_offsets<<<1, kThr, 0, s>>>(hist, tiles);
                big_scatter<<<tiles, kThr, 0, s>>>(ga, dreq, va, vb, dhdr, hist, wd.w, static_cast<int>(b), compact);
                std::swap(va, vb);
            }
        big_ord<<<grid, kThr, 0, s>>>(va, dhdr, ord);
        big_r_init<<<grid, kThr, 0, s>>>(np, flags, blocked, ord, eff);
        big_eff<<<grid, kThr, 0, s>>>(ga, np, flags, ord, eff);
        big_tile_sums<<<tiles, kThr, 0, s>>>(ga, dreq, va, flags, eff, dhdr, tsum);
        big_tile_scan<<<1, 32, 0, s>>>(tsum, tiles);
        big_emit<<<tiles, kThr, 0, s>>>(ga, dreq, va, flags, eff, dhdr, tsum, o_idx, o_act);
        cudaMemcpyAsync(h_hdr, dhdr, sizeof(Hdr), cudaMemcpyDeviceToHost, s);
        const cudaError_t cap_rc = cudaStreamEndCapture(s, &g);
        if (cap_rc != cudaSuccess) return cuda_error(cap_rc, "K5 graph capture");
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
        git = st.graphs.emplace(key, bg).first;
    }
    KVF_CUDA(cudaMemcpyAsync(d, hreq, sizeof(BigReq), cudaMemcpyHostToDevice, s));
    KVF_CUDA(cudaEventRecord(e->dec_start, s));
    KVF_CUDA(cudaGraphLaunch(git->second.exec, s));
    KVF_CUDA(cudaEventRecord(e->dec_stop, s));
    e->stats.kernel_launches += git->second.kernels;
    KVF_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    if (cudaEventElapsedTime(&ms, e->dec_start, e->dec_stop) == cudaSuccess) e->stats.decision_kernel_ms += ms;
    const uint32_t cnt = static_cast<uint32_t>(h_hdr->count);
    if (cnt > a.n) return set_error(KVF_E_INTERNAL, "device-wide K5: victim count beyond the tree");
    if (cnt > cap) return set_error(KVF_E_INVALID_ARG, "victim buffer too small");
    std::memcpy(out_idx, h_idx, cnt * 4ull);
    std::memcpy(out_action, h_act, cnt);
    *out_count = cnt;
    *out_imm = h_hdr->imm;
    *out_pend = h_hdr->pend;
    return KVF_OK;
}

// kvf_victim_select above the single-CTA limit: the snapshot goes to HBM once (padding slots
// dead) and runs the same device-wide path.
int victim_select_large(kvf_engine* e, const kvf_tree_view* t, const kvf_evict_request* q, int32_t* out_idx,
                        uint8_t* out_action, uint32_t* out_count, uint64_t* out_imm, uint64_t* out_pend) {
    const uint32_t n = t->n;
    const uint32_t np = large_capacity(n);
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t bytes = al(np * 8ull) * 5 + al(np * 4ull) * 2 + al(np) * 2;
    const void* old = e->ws_big.dev;
    if (int rc = e->ws_big.ensure(bytes, bytes)) return rc;
    if (e->ws_big.dev != old) large_invalidate(e->large_snap);
    char* h = static_cast<char*>(e->ws_big.host);
    char* hp = h;
    auto put = [&](const void* src, size_t elem, int fill) {
        std::memcpy(hp, src, n * elem);
        std::memset(hp + n * elem, fill, (np - n) * elem);
        char* at = hp;
        hp += al(np * elem);
        return static_cast<size_t>(at - h);
    };
    const size_t o_rank = put(t->rank, 8, 0), o_time = put(t->time, 8, 0), o_seq = put(t->seq, 8, 0),
                 o_id = put(t->id, 8, 0), o_tok = put(t->tokens, 8, 0), o_par = put(t->parent, 4, 0xFF),
                 o_lock = put(t->lock, 4, 0), o_st = put(t->status, 1, KVF_SLOT_DEAD), o_bk = put(t->backed, 1, 0);
    char* d = static_cast<char*>(e->ws_big.dev);
    KVF_CUDA(cudaMemcpyAsync(d, h, static_cast<size_t>(hp - h), cudaMemcpyHostToDevice, e->s_dec));
    LargeArrays a{reinterpret_cast<const int32_t*>(d + o_par), reinterpret_cast<const uint8_t*>(d + o_st),
                  reinterpret_cast<const int32_t*>(d + o_lock), reinterpret_cast<const int64_t*>(d + o_rank),
                  reinterpret_cast<const double*>(d + o_time), reinterpret_cast<const uint64_t*>(d + o_seq),
                  reinterpret_cast<const uint64_t*>(d + o_id),  reinterpret_cast<const uint64_t*>(d + o_tok),
                  reinterpret_cast<const uint8_t*>(d + o_bk),   n};
    LargeKeyInfo ki;  // an arbitrary snapshot: widths from its values, time passes kept
    for (uint32_t i = 0; i < n; ++i) {
        ki.max_id = std::max(ki.max_id, t->id[i]);
        ki.max_seq = std::max(ki.max_seq, t->seq[i]);
        ki.note_rank(t->rank[i]);
    }
    static_assert(sizeof(uint32_t) == sizeof(int32_t), "index width");
    return victim_large(e, e->large_snap, a, q, t->bytes_per_token, ki, reinterpret_cast<uint32_t*>(out_idx),
                        out_action, n, out_count, out_imm, out_pend);
}

}  // namespace kvf_impl
