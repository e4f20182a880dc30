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
//     One CTA, everything in shared memory: a sort of the candidates by the 4-word key
//     (register bitonic, or a rank count up to 64 candidates) -> ord, R and eff by parallel
//     root walks (shared-memory atomics with early exit, no per-level barriers), and then no
//     second sort: R by (eff asc, depth desc) is a sequence of chains in ord order (a node y
//     with eff(y) = ord(y) heads the chain of its ancestors whose eff is ord(y), deepest
//     first), so a block scan of the chains' bytes places every victim (decide_body.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "decide_body.cuh"
#include "engine_internal.hpp"

using namespace kvf_impl;

namespace {

using namespace kvf_dec;

__global__ void __launch_bounds__(kThreads) kvf_priority_kernel(const int32_t* parent, uint32_t n, const int32_t* bidx,
                                                                const int64_t* cand, uint32_t m, long long* out,
                                                                const uint8_t* blob, uint32_t blob_bytes,
                                                                unsigned long long* hdr, unsigned long long seq,
                                                                long long* scratch) {
    extern __shared__ __align__(16) uint8_t psm[];
    const unsigned long long t_begin = gtimer();
    const bool staged = n <= kPrioSmemNodes;
    long long* rank = reinterpret_cast<long long*>(psm);
    if (blob_bytes) {  // inputs -> shared memory in one round trip
        uint8_t* sb = psm + (staged ? (n * 8ull + 15) & ~15ull : 0ull);
        stage_blob(sb, blob, blob_bytes);
        parent = rebase(parent, blob, sb);
        bidx = rebase(bidx, blob, sb);
        cand = rebase(cand, blob, sb);
    }
    // ranks beyond shared memory accumulate in device scratch when `out` is mapped host memory
    // (atomics there would cross PCIe one by one), else in `out` itself
    long long* r = staged ? rank : (scratch ? scratch : out);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) r[i] = kRankSuffix;
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < m; b += blockDim.x) {
        const long long c = cand[b];
        for (int32_t v = bidx[b]; v > 0; v = parent[v]) atomicMin(r + v, c);
    }
    if (r != out) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = r[i];
    }
    if (hdr && threadIdx.x == 0) {
        hdr[3] = t_begin;
        hdr[8] = gtimer();
    }
    publish_done(hdr ? hdr + kDoneWord : nullptr, seq);
}

__global__ void __launch_bounds__(kThreads) kvf_victim_kernel(const TreeDev t_in, const ReqDev q, OutDev o,
                                                              unsigned long long seq) {
    victim_body(t_in, q, o, seq);
}

int finish_decision(kvf_engine* e, std::chrono::steady_clock::time_point t0) {
    float ms = 0;
    KVF_CUDA(cudaEventElapsedTime(&ms, e->dec_start, e->dec_stop));
    e->stats.decision_kernel_ms += ms;
    e->stats.decision_call_us +=
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    return KVF_OK;
}

// Fast-path completion: the kernel publishes `seq` into mapped pinned memory after its
// outputs (publish_done); the host spins on it instead of cudaStreamSynchronize -- the
// result is usable one posted PCIe write after the kernel's last store.  A fault surfaces
// through the periodic cudaStreamQuery.  Kernel time comes from its own globaltimer stamps.
// KVF_DECISION_TRACE=<file>: one line per fast-path call -- host phases (entry -> launch
// call -> launch returned -> done word seen) and the kernel's globaltimer start / end
// against the host's CLOCK_REALTIME at the launch call (globaltimer counts Unix-epoch ns on
// this driver; the idle rows check that).  Diagnostics only.
struct DecisionTrace {
    std::chrono::steady_clock::time_point t_launch, t_launched;
    long long rt_launch_ns = 0;
};
const char* decision_trace_path() {
    static const char* p = std::getenv("KVF_DECISION_TRACE");
    return p;
}
long long realtime_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::system_clock::now().time_since_epoch())
        .count();
}

int spin_decision(kvf_engine* e, const unsigned long long* hdr, unsigned long long seq,
                  std::chrono::steady_clock::time_point t0, const DecisionTrace* tr = nullptr, const char* kind = "",
                  uint32_t n = 0) {
    const volatile unsigned long long* flag = hdr + kDoneWord;
    // a faulted kernel never publishes: look at the stream only after 200 us, then every 100 us
    // (a driver call inside the normal ~10-30 us wait would only delay seeing the done word)
    auto next_check = t0 + std::chrono::microseconds(200);
    for (uint32_t it = 1;; ++it) {
        if (__atomic_load_n(const_cast<const unsigned long long*>(flag), __ATOMIC_ACQUIRE) == seq) break;
        if ((it & 63) == 0 && std::chrono::steady_clock::now() >= next_check) {
            next_check = std::chrono::steady_clock::now() + std::chrono::microseconds(100);
            const cudaError_t st = cudaStreamQuery(e->s_dec);
            if (st != cudaSuccess && st != cudaErrorNotReady) return cuda_error(st, "decision kernel");
            if (st == cudaSuccess && __atomic_load_n(const_cast<const unsigned long long*>(flag), __ATOMIC_ACQUIRE) != seq)
                return set_error(KVF_E_INTERNAL, "decision kernel finished without publishing its result");
        }
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    e->stats.decision_kernel_ms += static_cast<double>(hdr[8] - hdr[3]) * 1e-6;
    const auto t_done = std::chrono::steady_clock::now();
    e->stats.decision_call_us += std::chrono::duration<double, std::micro>(t_done - t0).count();
    if (tr && decision_trace_path()) {
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        if (FILE* f = std::fopen(decision_trace_path(), "a")) {
            // host phases on the host clock, kernel_us on the GPU's %globaltimer: the two clocks
            // are never subtracted from each other (they are not synchronised)
            std::fprintf(f,
                         "{\"kind\": \"%s\", \"n\": %u, \"pack_us\": %.2f, \"launch_call_us\": %.2f, \"spin_us\": %.2f, "
                         "\"kernel_us\": %.2f}\n",
                         kind, n, us(t0, tr->t_launch), us(tr->t_launch, tr->t_launched), us(tr->t_launched, t_done),
                         (hdr[8] - hdr[3]) * 1e-3);
            std::fclose(f);
        }
    }
    return KVF_OK;
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
    clear_stale_error(e, __func__);
    if (n == 0) return KVF_OK;
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t b = 0; b < m; ++b)
        if (bidx[b] < 0 || static_cast<uint32_t>(bidx[b]) >= n) return set_error(KVF_E_UNKNOWN_BOUNDARY_NODE, "boundary index out of range");
    const size_t in_bytes = ((n * 4 + 15) & ~15ull) + ((m * 4 + 15) & ~15ull) + ((m * 8 + 15) & ~15ull);
    const size_t out_bytes = n * 8;
    int rc = e->ws_dec.ensure(in_bytes + out_bytes + 1024 + 512, in_bytes + out_bytes + 1024 + 512);
    if (rc) return rc;
    char* h = static_cast<char*>(e->ws_dec.host);
    char* hp = h;
    std::memcpy(carve<int32_t>(hp, n), parent, n * 4);
    std::memcpy(carve<int32_t>(hp, m), bidx, m * 4);
    std::memcpy(carve<int64_t>(hp, m), cand, m * 8);
    const size_t used = static_cast<size_t>(hp - h);
    const size_t out_off = (used + 255) & ~size_t(255);
    // The result (ranks, stamps, done word) always goes to mapped pinned memory -- coalesced
    // posted writes, the host spins on the done word: no D2H copy, no stream sync.  Inputs up
    // to kZeroCopyBytes are read in place from mapped memory too (one launch in all); larger
    // ones take one H2D copy ahead of the kernel on the same stream.
    const bool zero_in = in_bytes <= kZeroCopyBytes;
    char* hdev = static_cast<char*>(e->ws_dec.host_dev);
    char* ddev = static_cast<char*>(e->ws_dec.dev);
    char* base = zero_in ? hdev : ddev;
    char* dp = base;
    int32_t* d_parent = carve<int32_t>(dp, n);
    int32_t* d_bidx = carve<int32_t>(dp, m);
    int64_t* d_cand = carve<int64_t>(dp, m);
    long long* d_out = reinterpret_cast<long long*>(hdev + out_off);
    // ranks beyond shared memory accumulate in device scratch (never atomics on mapped memory)
    long long* scratch = n > kPrioSmemNodes ? reinterpret_cast<long long*>(ddev + out_off) : nullptr;
    const size_t hdr_off = (out_off + n * 8 + 255) & ~size_t(255);
    unsigned long long* h_hdr = reinterpret_cast<unsigned long long*>(h + hdr_off);
    unsigned long long* d_hdr = reinterpret_cast<unsigned long long*>(hdev + hdr_off);
    const unsigned long long seq = ++e->dec_seq;
    // the done word sits wherever this call's n puts it -- possibly on bytes an earlier call
    // left there (victim indices can equal a sequence number): clear it before the launch
    __atomic_store_n(h_hdr + kDoneWord, 0ull, __ATOMIC_RELEASE);
    if (!zero_in) KVF_CUDA(cudaMemcpyAsync(ddev, h, used, cudaMemcpyHostToDevice, e->s_dec));
    const size_t smem = (n <= kPrioSmemNodes ? (n * 8ull + 15) & ~15ull : 0) + (zero_in ? used : 0);
    if (!e->prio_attr_set) {
        KVF_CUDA(cudaFuncSetAttribute(kvf_priority_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kPrioSmemNodes * 8 + kZeroCopyBytes + 64)));
        e->prio_attr_set = true;
    }
    DecisionTrace tr;
    if (decision_trace_path()) {
        tr.t_launch = std::chrono::steady_clock::now();
        tr.rt_launch_ns = realtime_ns();
    }
    // sized to the tree (128..1024 threads): a small CTA also fits beside a K6 CTA on a busy SM
    const uint32_t prio_threads = std::min<uint32_t>(kThreads, std::max<uint32_t>(128, pow2_ceil(std::max(n, m))));
    kvf_priority_kernel<<<1, prio_threads, smem, e->s_dec>>>(d_parent, n, d_bidx, d_cand, m, d_out,
                                                         zero_in ? reinterpret_cast<const uint8_t*>(base) : nullptr,
                                                         zero_in ? static_cast<uint32_t>(used) : 0u, d_hdr, seq,
                                                         scratch);
    KVF_CUDA(cudaGetLastError());
    if (decision_trace_path()) tr.t_launched = std::chrono::steady_clock::now();
    e->stats.kernel_launches++;
    e->stats.decisions++;
    if (int src = spin_decision(e, h_hdr, seq, t0, &tr, "k4", n)) return src;
    std::memcpy(out_rank, h + out_off, n * 8);
    return KVF_OK;
}

int kvf_victim_select(kvf_engine* e, const kvf_tree_view* t, const kvf_evict_request* q, int32_t* out_idx,
                      uint8_t* out_action, uint32_t* out_count, uint64_t* out_imm, uint64_t* out_pend) {
    if (!e || !t || !q || !out_idx || !out_action || !out_count || !out_imm || !out_pend)
        return set_error(KVF_E_INVALID_ARG, "null argument");
    std::lock_guard<std::mutex> lk(e->mu);
    if (cudaSetDevice(e->device) != cudaSuccess) return set_error(KVF_E_CUDA, "cudaSetDevice failed");
    clear_stale_error(e, __func__);
    const uint32_t n = t->n;
    *out_count = 0;
    *out_imm = *out_pend = 0;
    if (n <= 1 || q->needed == 0) return KVF_OK;
    const auto t0 = std::chrono::steady_clock::now();
    if (n > kMaxNodesSingleCta) {  // device-wide path (decide_large.cu)
        int rc = victim_select_large(e, t, q, out_idx, out_action, out_count, out_imm, out_pend);
        return rc ? rc : finish_decision(e, t0);
    }
    // pack the SoA snapshot into one pinned buffer -> one H2D copy
    const size_t in_bytes = 5 * ((n * 8 + 15) & ~15ull) + 2 * ((n * 4 + 15) & ~15ull) + ((n * 2 + 15) & ~15ull) +
                            2 * ((n + 15) & ~15ull);
    const size_t out_bytes = kHeaderBytes + ((n * 4 + 15) & ~15ull) + ((n + 15) & ~15ull);
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
    // inputs up to kZeroCopyBytes are read in place from mapped pinned memory, larger ones take
    // one H2D copy ahead of the kernel; the result always goes to mapped memory (posted
    // writes) and the host spins on its done word -- no D2H copy, no stream sync
    const bool zero_copy = used <= kZeroCopyBytes;
    char* d = zero_copy ? static_cast<char*>(e->ws_dec.host_dev) : static_cast<char*>(e->ws_dec.dev);
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
    td.blob = zero_copy ? reinterpret_cast<const uint8_t*>(d) : nullptr;
    td.blob_bytes = zero_copy ? static_cast<uint32_t>(used) : 0u;
    char* dout = static_cast<char*>(e->ws_dec.host_dev) + ((used + 255) & ~size_t(255));
    OutDev od;
    od.header = reinterpret_cast<unsigned long long*>(dout);
    od.idx = reinterpret_cast<int32_t*>(dout + kHeaderBytes);
    od.action = reinterpret_cast<uint8_t*>(dout + kHeaderBytes + ((n * 4 + 15) & ~15ull));
    ReqDev rq{q->needed, q->floor, q->cpu_used, q->cpu_capacity, q->workflow_aware, q->offload_mode, q->has_floor};
    if (!zero_copy) KVF_CUDA(cudaMemcpyAsync(d, h, used, cudaMemcpyHostToDevice, e->s_dec));
    const size_t smem = victim_smem(n, zero_copy ? used : 0);
    if (!e->victim_attr_set) {  // once per engine (attributes are per device); unconditional:
                                 // the 48 KB default also counts the kernel's static shared memory
        KVF_CUDA(cudaFuncSetAttribute(kvf_victim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(victim_smem(kMaxNodesSingleCta))));
        e->victim_attr_set = true;
    }
    od.spin = true;
    const unsigned long long seq = ++e->dec_seq;
    // see kvf_priority_propagate: never spin on a stale word
    __atomic_store_n(reinterpret_cast<unsigned long long*>(h + ((used + 255) & ~size_t(255))) + kDoneWord, 0ull,
                     __ATOMIC_RELEASE);
    DecisionTrace tr;
    if (decision_trace_path()) {
        tr.t_launch = std::chrono::steady_clock::now();
        tr.rt_launch_ns = realtime_ns();
    }
    kvf_victim_kernel<<<1, victim_threads(n), smem, e->s_dec>>>(td, rq, od, seq);
    if (const cudaError_t le = cudaGetLastError(); le != cudaSuccess)
        return cuda_error(le, ("K5 launch (n=" + std::to_string(n) + " threads=" + std::to_string(victim_threads(n)) +
                               " smem=" + std::to_string(smem) + " zero_copy=" + std::to_string(zero_copy) + ")")
                                  .c_str());
    if (decision_trace_path()) tr.t_launched = std::chrono::steady_clock::now();
    e->stats.kernel_launches++;
    e->stats.decisions++;
    char* hout = h + ((used + 255) & ~size_t(255));
    if (int src = spin_decision(e, reinterpret_cast<const unsigned long long*>(hout), seq, t0, &tr, "k5", n))
        return src;
    const uint64_t* hdr = reinterpret_cast<const uint64_t*>(hout);
    const uint32_t cnt = static_cast<uint32_t>(hdr[0]);
    for (int k = 0; k < 5; ++k) {
        e->stats.k5_phase_ns[k] += static_cast<double>(hdr[4 + k] - hdr[3 + k]);
        e->stats.k5_phase_cycles[k] += static_cast<double>(hdr[10 + k] - hdr[9 + k]);
    }
    std::memcpy(out_idx, hout + kHeaderBytes, cnt * 4);
    std::memcpy(out_action, hout + kHeaderBytes + ((n * 4 + 15) & ~15ull), cnt);
    *out_count = cnt;
    *out_imm = hdr[1];
    *out_pend = hdr[2];
    return KVF_OK;
}

}  // extern "C"

namespace kvf_impl {
void set_carveout_decide() {
    cudaFuncSetAttribute(kvf_priority_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(kvf_victim_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
}
}  // namespace kvf_impl
