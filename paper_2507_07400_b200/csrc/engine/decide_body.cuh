// Device bodies of the decision kernels, shared by decide.cu (K4 / K5 over host-packed SoA
// snapshots, the kvf_priority_propagate / kvf_victim_select C-ABI) and mirror.cu (the same
// decisions over a tree mirrored in HBM, served by a resident decider CTA or one-shot
// launches).  Header-only on purpose: each translation unit gets its own copy (no -rdc).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "kvflow.h"

namespace kvf_dec {

constexpr int64_t kRankSuffix = INT64_MAX / 2;        // radix_cache.hpp:30-38
constexpr int64_t kRankUnreachable = INT64_MAX / 4;
constexpr uint32_t kMaxNodesSingleCta = 4096;
constexpr int kThreads = 1024;
// K5 result header: [count, immediate, pending, 6 globaltimer stamps, 6 clock64 stamps, done seq]
constexpr size_t kHeaderBytes = 128;
constexpr int kDoneWord = 15;  // the host spins on header[15] == call sequence number
// decision inputs up to this size are read by the kernel straight from mapped pinned memory
constexpr size_t kZeroCopyBytes = 64 << 10;

// Copy a packed input blob (16-B multiple) into shared memory with all of a thread's loads
// in flight before its stores: when the blob sits in mapped pinned host memory this costs
// one PCIe round trip instead of one per input array and phase.
__device__ __forceinline__ void stage_blob(uint8_t* dst, const uint8_t* src, uint32_t bytes) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    const uint32_t nv = bytes / 16;
    for (uint32_t base = threadIdx.x; base < nv; base += blockDim.x * 4) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (base + u * blockDim.x < nv) v[u] = s4[base + u * blockDim.x];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (base + u * blockDim.x < nv) d4[base + u * blockDim.x] = v[u];
    }
}

template <typename T>
__device__ __forceinline__ const T* rebase(const T* p, const uint8_t* from, const uint8_t* to) {
    return reinterpret_cast<const T*>(to + (reinterpret_cast<const uint8_t*>(p) - from));
}

// The ranks live in shared memory when they fit (n <= kPrioSmemNodes); small inputs are
// staged there too (stage_blob), so the root walks never touch PCIe-mapped host memory.
constexpr uint32_t kPrioSmemNodes = 4096;

// Publish a decision kernel's result to a host spinning on mapped memory: every thread fences
// its own output stores system-wide, then one thread writes the call's sequence number.
__device__ __forceinline__ void publish_done(unsigned long long* flag, unsigned long long seq) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && flag) {
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(seq) : "memory");
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
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
    const uint8_t* blob;  // packed inputs to stage into shared memory first (nullptr: read in place)
    uint32_t blob_bytes;
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
    unsigned long long* header;  // [count, immediate, pending, 6 phase stamps] (kHeaderBytes)
    bool spin;                   // header is mapped host memory the caller spins on
};

// Warp-aggregated slot claim on a shared counter: one atomic per warp instead of per lane.
__device__ __forceinline__ uint32_t claim(uint32_t* counter, bool take) {
    const unsigned act = __activemask();
    const unsigned mask = __ballot_sync(act, take);
    const uint32_t lane = threadIdx.x & 31;
    const int leader = __ffs(act) - 1;
    uint32_t base = 0;
    if (static_cast<int>(lane) == leader && mask) base = atomicAdd(counter, static_cast<uint32_t>(__popc(mask)));
    base = __shfl_sync(act, base, leader);
    return base + __popc(mask & ((1u << lane) - 1u));
}

__host__ __device__ inline uint32_t pow2_ceil(uint32_t x) {
#ifdef __CUDA_ARCH__
    return x <= 1 ? 1u : 1u << (32 - __clz(x - 1));
#else
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
#endif
}

// Bitonic sort with the elements in registers: thread t holds positions t*E .. t*E+E-1
// (x[]), P / E threads take part (a multiple of 32: P >= 128, E <= 4).  Per merge level k,
// stages with j >= 32E run as compare-exchanges in shared memory (ld/st: position ->
// element), stages E <= j < 32E exchange with lane t ^ (j/E) through shuffles, and j < E
// inside the thread -- at P = 512 35 of 45 stages never touch shared memory or a barrier
// (an all-shared-memory network spent ~870 cycles per stage there).
// after(a, b): a must come after b (a total order, or identical elements).
template <int E, typename V, typename After, typename Ld, typename St, typename Shfl>
__device__ __forceinline__ void bitonic_reg(uint32_t P, V (&x)[E], After after, Ld ld, St st, Shfl shfl) {
    const uint32_t t = threadIdx.x;
    const bool act = t * E < P;  // warp-uniform
    for (uint32_t k = 2; k <= P; k <<= 1) {
        uint32_t j = k >> 1;
        if (j >= 32u * E) {
            if (act) {
#pragma unroll
                for (int e = 0; e < E; ++e) st(t * E + e, x[e]);
            }
            __syncthreads();
            for (; j >= 32u * E; j >>= 1) {
                for (uint32_t pr = t; pr < P / 2; pr += blockDim.x) {
                    const uint32_t i = ((pr & ~(j - 1)) << 1) | (pr & (j - 1));
                    const uint32_t l = i | j;
                    const V a = ld(i), b = ld(l);
                    if ((i & k) == 0 ? after(a, b) : after(b, a)) {
                        st(i, b);
                        st(l, a);
                    }
                }
                __syncthreads();
            }
            // own positions only: the next round's stores (own positions again) and its
            // shared stages (after a barrier) cannot race these loads
            if (act) {
#pragma unroll
                for (int e = 0; e < E; ++e) x[e] = ld(t * E + e);
            }
        }
        if (act) {
            for (; j >= static_cast<uint32_t>(E); j >>= 1) {  // across lanes
                const uint32_t m = j / E;
                const bool lower = (t & m) == 0;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const V y = shfl(x[e], m);
                    const bool up = ((t * E + e) & k) == 0;
                    const bool x_after_y = after(x[e], y);
                    // the lower position of an ascending pair keeps the smaller element
                    if ((lower == up) == x_after_y) x[e] = y;
                }
            }
            // inside the thread: j = min(k/2, E/2) .. 1, unrolled so x[] stays in registers
#pragma unroll
            for (int jj = E / 2; jj > 0; jj >>= 1) {
                if (static_cast<uint32_t>(jj) > (k >> 1)) continue;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    if (e & jj) continue;
                    const int l = e | jj;
                    const bool up = ((t * E + e) & k) == 0;
                    if (up ? after(x[e], x[l]) : after(x[l], x[e])) {
                        const V tmp = x[e];
                        x[e] = x[l];
                        x[l] = tmp;
                    }
                }
            }
        }
    }
}

// Sort positions [0, P) of (ld, st) with bitonic_reg; out(position, element) receives the
// sorted sequence (from registers).  The caller fills [c, P) with pads that sort last.
template <typename V, typename After, typename Ld, typename St, typename Shfl, typename Out>
__device__ __forceinline__ void sort_reg(uint32_t P, After after, Ld ld, St st, Shfl shfl, Out out) {
    auto run = [&](auto tag) {
        constexpr int E = decltype(tag)::value;
        const uint32_t t = threadIdx.x;
        V x[E];
        __syncthreads();  // the pads / inputs are in place
        if (t * E < P) {
#pragma unroll
            for (int e = 0; e < E; ++e) x[e] = ld(t * E + e);
        }
        bitonic_reg<E>(P, x, after, ld, st, shfl);
        __syncthreads();  // every shared stage has been read before out() may reuse the arrays
        if (t * E < P) {
#pragma unroll
            for (int e = 0; e < E; ++e) out(t * E + e, x[e]);
        }
        __syncthreads();
    };
    if (P <= blockDim.x) run(std::integral_constant<int, 1>{});
    else if (P == 2 * blockDim.x) run(std::integral_constant<int, 2>{});
    else run(std::integral_constant<int, 4>{});
}

struct Cand {  // phase-2 element: primary key words and the node index (0xFFFF = pad)
    uint64_t a, b;
    uint32_t s;
};

// Rank sort for <= 64 elements: element i's output position is the number of elements that
// sort before it.  G = blockDim.x / 64 consecutive lanes share element i and split the j range,
// so each thread runs c / G independent comparisons (ILP instead of the 21 dependent stages a
// 64-wide bitonic network needs) and a G-lane shuffle reduction finishes the count.
template <typename Before>
__device__ __forceinline__ uint32_t rank64(uint32_t c, Before before, uint32_t& i_out) {
    const uint32_t G = blockDim.x >> 6;  // >= 2: small trees launch >= 128 threads
    const uint32_t i = threadIdx.x / G, q = threadIdx.x % G;
    uint32_t cnt = 0;
    if (i < c) {
#pragma unroll 4
        for (uint32_t j = q; j < c; j += G) cnt += (j != i && before(j, i)) ? 1u : 0u;
    }
    for (uint32_t off = G >> 1; off; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    i_out = (q == 0 && i < c) ? i : 0xFFFFFFFFu;
    return cnt;
}

// Order-preserving u64 image of a double (-0.0 == +0.0 as in the reference's `!=`).
__device__ __forceinline__ uint64_t time_order(double t) {
    const uint64_t b = t == 0.0 ? 0ull : static_cast<uint64_t>(__double_as_longlong(t));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Shared-memory layout for n <= 4096 nodes (PN = pow2 >= n):
//   pk0 u64[PN] | pk1 u64[PN]   phase-1 primary keys by candidate
//   parent i32[n] | ord i32[n] | eff i32[n] | blocked u32[n] | bytes u64[n] | id u64[n]
//   | sel u16[PN] | posn u16[PN] (node at each `before` position) | status u8[n] | flags u8[n]
//   | backed u8[n]
// Everything the later phases touch is staged here once, so inputs may live in mapped host
// memory (small trees) without per-phase PCIe round trips.
// flags: bit0 selfok, bit1 releases, bit2 R
__device__ __forceinline__ void victim_body(const TreeDev& t_in, const ReqDev& q, const OutDev& o,
                                            unsigned long long seq) {
    extern __shared__ __align__(16) uint8_t sm[];
    TreeDev t = t_in;
    const uint32_t n = t.n;
    const uint32_t PN = pow2_ceil(n > 1 ? n : 2);
    uint64_t* pk0 = reinterpret_cast<uint64_t*>(sm);
    uint64_t* pk1 = pk0 + PN;
    int32_t* parent = reinterpret_cast<int32_t*>(pk1 + PN);
    int32_t* ord = parent + n;
    int32_t* eff = ord + n;
    uint32_t* blocked = reinterpret_cast<uint32_t*>(eff + n);
    uint64_t* nbytes = reinterpret_cast<uint64_t*>(blocked + n);  // offset 16*PN + 16*n: 8-aligned
    uint64_t* nid = nbytes + n;  // node ids: exact-key ties resolve here, not in global memory
    uint16_t* sel = reinterpret_cast<uint16_t*>(nid + n);
    uint16_t* posn = sel + PN;  // node at each `before` position (phase 2 -> phase 5)
    uint8_t* st = reinterpret_cast<uint8_t*>(posn + PN);
    uint8_t* flags = st + n;
    uint8_t* bk = flags + n;
    __shared__ uint32_t s_cnt, s_slow, s_taken, s_warpn[32];
    __shared__ unsigned long long s_imm, s_pend, s_warp[32], s_stamp[12];
    // per-phase timestamps (globaltimer ns, SM cycles) -> header[3..14] at the end (read by
    // kvf_get_stats); kept in shared memory meanwhile: a store to mapped host memory per phase
    // would put the PCIe write path inside every phase
    auto stamp = [&](int k) {
        if (threadIdx.x == 0) {
            unsigned long long t_ns;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ns));
            s_stamp[k] = t_ns;
            s_stamp[6 + k] = clock64();  // SM cycles: finer than globaltimer for short phases
        }
    };
    stamp(0);
    if (t.blob_bytes) {  // small trees: the whole snapshot -> shared memory in one round trip
        uint8_t* sb = bk + ((n + 15) & ~15u);
        sb = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sb) + 15) & ~uintptr_t(15));
        stage_blob(sb, t.blob, t.blob_bytes);
        t.parent = rebase(t.parent, t.blob, sb);
        t.depth = rebase(t.depth, t.blob, sb);
        t.status = rebase(t.status, t.blob, sb);
        t.lock = rebase(t.lock, t.blob, sb);
        t.rank = rebase(t.rank, t.blob, sb);
        t.time = rebase(t.time, t.blob, sb);
        t.seq = rebase(t.seq, t.blob, sb);
        t.id = rebase(t.id, t.blob, sb);
        t.tokens = rebase(t.tokens, t.blob, sb);
        t.backed = rebase(t.backed, t.blob, sb);
    }
    if (threadIdx.x == 0) {
        s_cnt = s_slow = s_taken = 0;
        s_imm = s_pend = 0;
    }
    __syncthreads();
    const bool wa = q.wa != 0;
    // 1. stage the snapshot; self-eligibility (radix_cache.cpp:305-312 minus the device-child
    //    test); whether evicting a node frees its parent (Discard / backed / CPU full)
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint8_t s = t.status[i];
        const uint64_t bytes = t.tokens[i] * t.bpt;
        const bool cpu_room = q.cpu_cap == 0 || q.cpu_used + bytes <= q.cpu_cap;
        const int64_t rank = t.rank[i];
        const bool selfok = i > 0 && t.lock[i] == 0 && s == 0 && (!q.has_floor || rank > q.floor);
        const bool releases = !q.offload || t.backed[i] || !cpu_room;
        parent[i] = t.parent[i];
        st[i] = s;
        nbytes[i] = bytes;
        nid[i] = t.id[i];
        bk[i] = t.backed[i];
        flags[i] = (selfok ? 1 : 0) | (releases ? 2 : 0);
        blocked[i] = 0;
        ord[i] = -1;
        const uint32_t k = claim(&s_cnt, selfok);
        if (selfok) {
            sel[k] = static_cast<uint16_t>(i);
            // primary key: an exact coarsening of `before` (radix_cache.cpp:316-321) when ranks fit
            // 16 bits and seq fits 48; ties fall back to the full comparison
            const uint64_t tord = time_order(t.time[i]);
            const uint64_t seq = t.seq[i];
            if (wa) {
                uint64_t code;
                if (rank == kRankSuffix) code = 0;
                else if (rank == kRankUnreachable) code = 1;
                else if (rank >= 0 && rank <= 0xFFFD) code = 0xFFFFull - static_cast<uint64_t>(rank);
                else { code = 0xFFFF; atomicOr(&s_slow, 1u); }
                if (seq >> 48) atomicOr(&s_slow, 1u);
                pk0[k] = (code << 48) | (tord >> 16);
                pk1[k] = (tord << 48) | (seq & 0xFFFFFFFFFFFFull);
            } else {
                pk0[k] = tord;
                pk1[k] = seq;
            }
        }
    }
    __syncthreads();
    const uint32_t c = s_cnt;
    const uint32_t P = pow2_ceil(c > 1 ? c : 2);
    for (uint32_t i = c + threadIdx.x; i < P; i += blockDim.x) {
        sel[i] = 0xFFFFu;
        pk0[i] = pk1[i] = ~0ull;
    }
    const bool slow = s_slow != 0;
    stamp(1);
    // 2. candidates in `before` order -> ord
    auto full_after = [&](uint32_t x, uint32_t y) {  // is node x after node y?
        if (wa) {
            const int64_t rx = t.rank[x], ry = t.rank[y];
            if (rx != ry) return rx < ry;
        }
        const double tx = t.time[x], ty = t.time[y];
        if (tx != ty) return tx > ty;
        const uint64_t sx = t.seq[x], sy = t.seq[y];
        if (sx != sy) return sx > sy;
        return t.id[x] > t.id[y];
    };
    if (P <= 64 && !slow) {  // small trees: rank sort straight into ord, branch-free compares
        __syncthreads();
        // element i's key in registers; G lanes split the others and add up how many precede
        // it.  The words are exact: a tie is equal (rank, time, seq) and the id decides.  G is
        // as wide as the candidate count allows (<= 32 lanes: the reduction stays in a warp)
        const uint32_t G = min(32u, blockDim.x / P);
        const uint32_t i = threadIdx.x / G, q = threadIdx.x % G;
        uint32_t cnt = 0;
        if (i < c) {
            const uint64_t a0 = pk0[i], a1 = pk1[i], ad = nid[sel[i]];
#pragma unroll 8
            for (uint32_t j = q; j < c; j += G) {
                const uint64_t b0 = pk0[j], b1 = pk1[j], bd = nid[sel[j]];
                cnt += static_cast<uint32_t>((b0 < a0) | ((b0 == a0) & ((b1 < a1) | ((b1 == a1) & (bd < ad)))));
            }
        }
        for (uint32_t off = G >> 1; off; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
        if (q == 0 && i < c) {
            ord[sel[i]] = static_cast<int32_t>(cnt);
            posn[cnt] = sel[i];
        }
        __syncthreads();
    } else if (P <= 64) {  // keys beyond the exact coarsening: the full comparison
        __syncthreads();
        uint32_t i;
        const uint32_t rk = rank64(
            c, [&](uint32_t a, uint32_t b) { return full_after(sel[b], sel[a]); }, i);
        if (i != 0xFFFFFFFFu) {
            ord[sel[i]] = static_cast<int32_t>(rk);
            posn[rk] = sel[i];
        }
        __syncthreads();
    } else {
        sort_reg<Cand>(
            P,
            [&](const Cand& x, const Cand& y) {  // x must come after y
                if (x.s == 0xFFFFu || y.s == 0xFFFFu) return x.s == 0xFFFFu && y.s != 0xFFFFu;
                if (!slow) {
                    if (x.a != y.a) return x.a > y.a;
                    if (x.b != y.b) return x.b > y.b;
                    return nid[x.s] > nid[y.s];
                }
                return full_after(x.s, y.s);
            },
            [&](uint32_t i) { return Cand{pk0[i], pk1[i], sel[i]}; },
            [&](uint32_t i, const Cand& v) {
                pk0[i] = v.a;
                pk1[i] = v.b;
                sel[i] = static_cast<uint16_t>(v.s);
            },
            [](const Cand& v, uint32_t m) {
                return Cand{__shfl_xor_sync(0xffffffffu, v.a, m), __shfl_xor_sync(0xffffffffu, v.b, m),
                            __shfl_xor_sync(0xffffffffu, v.s, m)};
            },
            [&](uint32_t pos, const Cand& v) {
                if (v.s != 0xFFFFu) {
                    ord[v.s] = static_cast<int32_t>(pos);
                    posn[pos] = static_cast<uint16_t>(v.s);
                }
            });
    }
    stamp(2);
    // 3. blocked(n): some node of n's device subtree (below n) is not self-eligible or would
    //    not release it (has_device_child, radix_cache.cpp:40-45).  Every such node walks up
    //    through device-child links; a walker stops where another already passed.
    for (uint32_t m = threadIdx.x + 1; m < n; m += blockDim.x) {
        const uint8_t f = flags[m];
        if (st[m] == 1 || ((f & 1) && (f & 2))) continue;  // BACKUP children never block
        for (int32_t cur = static_cast<int32_t>(m);;) {
            const int32_t p = parent[cur];
            if (p <= 0) break;
            if (atomicOr(&blocked[p], 1u)) break;
            if (st[p] == 1) break;
            cur = p;
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const bool r = (flags[i] & 1) && !blocked[i];
        if (r) flags[i] |= 4;
        eff[i] = r ? ord[i] : -1;
    }
    __syncthreads();
    // 4. eff(n) = max ord over n's device subtree (all of it is in R when n is): R nodes push
    //    their ord up while the ancestor is in R; stop when an ancestor already holds more.
    for (uint32_t m = threadIdx.x + 1; m < n; m += blockDim.x) {
        if (!(flags[m] & 4)) continue;
        const int32_t v = ord[m];
        for (int32_t cur = static_cast<int32_t>(m);;) {
            const int32_t p = parent[cur];
            if (p <= 0 || !(flags[p] & 4)) break;
            if (atomicMax(&eff[p], v) >= v) break;
            cur = p;
        }
    }
    __syncthreads();
    stamp(3);
    // 5. victims = R sorted by (eff asc, depth desc) WITHOUT a second sort: that order is a
    //    sequence of chains -- a node y in R with eff(y) = ord(y) heads the chain y, parent(y),
    //    ... of the ancestors whose eff is ord(y), deepest first -- and the chain heads come in
    //    `before` position order.  Each thread takes a run of positions: chain bytes and member
    //    counts, a block scan, then every member whose bytes-before is < needed is popped
    //    (radix_cache.cpp:335) at its place in the order.
    auto head = [&](uint32_t k, uint32_t* y) {
        *y = posn[k];
        return (flags[*y] & 4) && eff[*y] == static_cast<int32_t>(k);
    };
    const uint32_t per = (c + blockDim.x - 1) / blockDim.x;
    const uint32_t lo_k = threadIdx.x * per, hi_k = min(c, (threadIdx.x + 1) * per);
    uint64_t lb = 0;
    uint32_t ln = 0;
    for (uint32_t k = lo_k; k < hi_k; ++k) {
        uint32_t y;
        if (!head(k, &y)) continue;
        for (int32_t cur = static_cast<int32_t>(y);;) {
            lb += nbytes[cur];
            ++ln;
            const int32_t pp = parent[cur];
            if (pp <= 0 || !(flags[pp] & 4) || eff[pp] != static_cast<int32_t>(k)) break;
            cur = pp;
        }
    }
    // 6. exclusive (bytes, members) prefix over the threads' position runs (block scan)
    uint64_t inc = lb;
    uint32_t incn = ln;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, inc, off);
        const uint32_t yn = __shfl_up_sync(0xffffffffu, incn, off);
        if (lane >= off) {
            inc += y;
            incn += yn;
        }
    }
    if (lane == 31) {
        s_warp[warp] = inc;
        s_warpn[warp] = incn;
    }
    __syncthreads();
    if (warp == 0) {
        uint64_t w = lane < nwarps ? s_warp[lane] : 0;
        uint32_t wn = lane < nwarps ? s_warpn[lane] : 0;
        for (int off = 1; off < 32; off <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, w, off);
            const uint32_t yn = __shfl_up_sync(0xffffffffu, wn, off);
            if (lane >= off) {
                w += y;
                wn += yn;
            }
        }
        if (lane < nwarps) {
            s_warp[lane] = w;
            s_warpn[lane] = wn;
        }
    }
    __syncthreads();
    uint64_t run = inc - lb + (warp ? s_warp[warp - 1] : 0);
    uint32_t idx = incn - ln + (warp ? s_warpn[warp - 1] : 0);
    // 7. pop: members in order while the bytes freed before them are still < needed
    uint64_t my_imm = 0, my_pend = 0;
    uint32_t taken = 0;
    for (uint32_t k = lo_k; k < hi_k && run < q.needed; ++k) {
        uint32_t y;
        if (!head(k, &y)) continue;
        for (int32_t cur = static_cast<int32_t>(y);;) {
            const uint32_t v = static_cast<uint32_t>(cur);
            const uint64_t bytes = nbytes[v];
            if (run < q.needed) {
                uint8_t act;
                if (!q.offload) act = KVF_ACT_REMOVE;
                else if (bk[v]) act = KVF_ACT_DISCARD_TO_BACKUP;
                else if (!(q.cpu_cap == 0 || q.cpu_used + bytes <= q.cpu_cap)) act = KVF_ACT_REMOVE;
                else act = KVF_ACT_OFFLOAD;
                o.idx[idx] = static_cast<int32_t>(v);
                o.action[idx] = act;
                (act == KVF_ACT_OFFLOAD ? my_pend : my_imm) += bytes;
                taken = idx + 1;
            }
            run += bytes;
            ++idx;
            const int32_t pp = parent[cur];
            if (pp <= 0 || !(flags[pp] & 4) || eff[pp] != static_cast<int32_t>(k)) break;
            cur = pp;
        }
    }
    for (int off = 16; off; off >>= 1) {  // one shared atomic per warp
        my_imm += __shfl_xor_sync(0xffffffffu, my_imm, off);
        my_pend += __shfl_xor_sync(0xffffffffu, my_pend, off);
        taken = max(taken, __shfl_xor_sync(0xffffffffu, taken, off));
    }
    if (lane == 0) {
        if (my_imm) atomicAdd(&s_imm, static_cast<unsigned long long>(my_imm));
        if (my_pend) atomicAdd(&s_pend, static_cast<unsigned long long>(my_pend));
        if (taken) atomicMax(&s_taken, taken);
    }
    stamp(4);
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t lo = s_taken;  // taken victims form a prefix of the order
        o.header[0] = lo;
        o.header[1] = s_imm;
        o.header[2] = s_pend;
    }
    stamp(5);
    __syncthreads();  // thread 0's last stamps before warp 0 copies them out
    if (threadIdx.x < 12) o.header[threadIdx.x < 6 ? 3 + threadIdx.x : 9 + (threadIdx.x - 6)] = s_stamp[threadIdx.x];
    if (o.spin) publish_done(o.header + kDoneWord, seq);  // else the caller publishes (mirror.cu)
}


inline size_t victim_smem(uint32_t n, size_t blob = 0) {
    const size_t PN = pow2_ceil(n > 1 ? n : 2);
    return PN * 16 + static_cast<size_t>(n) * 16 + 8 + static_cast<size_t>(n) * 16 + PN * 2 + PN * 2 +
           3 * ((n + 15) & ~15u) + 64 + (blob ? blob + 32 : 0);
}

inline uint32_t victim_threads(uint32_t n) {  // one sort element per thread up to 1024 (sort_reg: E <= 4)
    const uint32_t pn = pow2_ceil(n > 1 ? n : 2);
    return pn < 128 ? 128 : (pn > static_cast<uint32_t>(kThreads) ? kThreads : pn);
}

}  // namespace kvf_dec
