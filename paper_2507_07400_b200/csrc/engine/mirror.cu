// Decisions over a radix tree mirrored in HBM (include/kvflow.h, "decisions over a tree
// mirrored in HBM").
//
// The reference walks its live pointer tree on every decision (set_agent_priorities,
// proj/src/radix_cache.cpp:266-285; evict, :302-372).  A GPU decision that re-packs and
// re-ships the whole tree per call pays a host walk + a PCIe copy proportional to the tree,
// so here the tree's SoA lives in HBM (one slot per node, slot 0 = root) and the host ships
// only the records of nodes that changed since the previous decision.
//
// Requests (K4 priorities, K5 victims, apply-only) go through a ring in mapped pinned memory
// and are executed strictly in order by one of two executors:
//   * the RESIDENT decider: one 256-thread CTA that polls the ring (no kernel launch per
//     decision; the request's first byte is seen ~1 PCIe read after the host writes it), for
//     trees up to KVF_RESIDENT_MAX_SLOTS slots.  It idles out after idle_ns without a request
//     (so a device-wide synchronize elsewhere waits at most that long) or when asked to stop;
//     on exit it publishes the first request it did not serve, and the host hands those on.
//   * one launch per request on the decision stream (larger trees, KVF_DECIDER=0).
// Every executor acknowledges request s by a posted write of s into ack[s % kRing] after its
// results; the host spins on that word.  Requests on one tree are ordered by the ring, so a
// K4 can be queued without waiting and the K5 behind it sees its ranks.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <vector>

#include "decide_body.cuh"
#include "engine_internal.hpp"

using namespace kvf_impl;
using namespace kvf_dec;

namespace kvf_mir {  // named: kernels take these types as parameters

constexpr uint32_t kRing = 16;
constexpr uint32_t kResThreads = 128;  // 128 x <= 128 registers + <= 25 KB: fits beside a K6 CTA
constexpr size_t kSlotBytes = 512;     // one warp reads a slot in one round: 32 lanes x 16 B
constexpr size_t kHdrBytes = 128;
constexpr size_t kInlineBytes = kSlotBytes - kHdrBytes;  // records + boundaries travel in the slot
constexpr size_t kPaySlotBytes = 256u << 10;  // per ring slot, for batches that do not fit inline
enum : uint32_t { REQ_PRIO = 1, REQ_VICTIMS = 2, REQ_APPLY = 3, REQ_PRIO_VICTIMS = 4 };  // 4: K4 then K5, one slot

struct MirrorDev {
    int32_t* parent;
    uint8_t* status;
    uint8_t* backed;
    int32_t* lock;
    int64_t* rank;
    double* time;
    uint64_t* seq;
    uint64_t* id;
    uint64_t* tokens;
};

struct TreeDesc {  // device memory, per tree (rewritten only when its mirror is reallocated)
    MirrorDev mir;
    long long* scratch;           // K4 ranks above the shared-memory limit
    unsigned long long* out_k4;   // K4 result buffer 0 (mapped pinned); results from + 128 B
    unsigned long long* out_k5;
    uint64_t bpt;
    uint64_t k4_stride;           // bytes from K4 result buffer 0 to buffer 1
};

// A ring slot.  The host writes the body, then `hash` (over seq and bytes 16..511), then `seq`
// last; the decider reads all 512 B in ONE round of loads (one PCIe round trip) and takes the
// request when seq is the one it waits for and the hash matches what it read -- a read that
// raced the host's stores fails the hash and is simply repeated.
struct DecReq {
    unsigned long long seq, hash;
    uint32_t type, n, n_recs, m;
    const TreeDesc* tree;
    const kvf_node_rec* recs;  // nullptr: inline at slot + 128
    const uint32_t* bslot;     // nullptr: inline after the inline records
    const int64_t* cand;
    uint64_t needed;
    int64_t floor;
    uint64_t cpu_used, cpu_cap;
    int32_t wa, offload, has_floor;
    uint32_t k4_buf;  // K4: which of the tree's two result buffers it writes
};
static_assert(sizeof(DecReq) <= kHdrBytes, "request header");
union alignas(16) ReqSlot {
    DecReq r;
    uint4 raw[kSlotBytes / 16];
    unsigned char bytes[kSlotBytes];
};

struct Ctl {  // after the ring slots
    unsigned long long exit_epoch, exit_next, stop_epoch, pad;
    unsigned long long ack[kRing];
    unsigned long long t_seen[kRing], t_done[kRing], polls[kRing];  // diagnostics (globaltimer ns)
};

ReqSlot* ring_slot(char* base, uint64_t seq) { return reinterpret_cast<ReqSlot*>(base) + (seq % kRing); }
Ctl* ring_ctl(char* base) { return reinterpret_cast<Ctl*>(base + kRing * sizeof(ReqSlot)); }

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}
// hash term of 16-B chunk c (1..31) of a slot; the slot hash XORs them with mix64(seq)
__host__ __device__ __forceinline__ uint64_t chunk_hash(uint64_t lo, uint64_t hi, uint32_t c) {
    return mix64(lo ^ (0x9e3779b97f4a7c15ULL * (c + 1))) + mix64(hi + c);
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Warp 0: one round of uncached 16-B loads of the whole slot (+ lane 0: the stop word).  True
// (and the slot in `dst`) when it holds request `want` intact.
__device__ __forceinline__ bool read_slot(ReqSlot& dst, const ReqSlot* src, unsigned long long want,
                                          const unsigned long long* stop_word, unsigned long long* stop_seen) {
    const uint32_t lane = threadIdx.x & 31;
    const uint4 v = __ldcv(&src->raw[lane]);
    unsigned long long stop = 0;
    if (stop_word && lane == 0) stop = ld_acquire_sys(stop_word);
    if (stop_seen) *stop_seen = __shfl_sync(0xffffffffu, stop, 0);
    const uint64_t lo = (static_cast<uint64_t>(v.y) << 32) | v.x, hi = (static_cast<uint64_t>(v.w) << 32) | v.z;
    const uint64_t seq = __shfl_sync(0xffffffffu, lo, 0), hash = __shfl_sync(0xffffffffu, hi, 0);
    if (seq != want) return false;
    uint64_t h = lane ? chunk_hash(lo, hi, lane) : mix64(seq);
    for (int off = 16; off; off >>= 1) h ^= __shfl_xor_sync(0xffffffffu, h, off);
    if (h != hash) return false;
    dst.raw[lane] = v;
    return true;
}

// Node records -> mirror (last record of a slot wins: the host sends one per slot per batch);
// inline records come from the slot copy in shared memory, others from host / device memory
__device__ __forceinline__ void put_rec(const MirrorDev& mir, uint32_t s, const uint4& a, const uint4& b, const uint4& c,
                                        const uint4& d) {
    mir.parent[s] = static_cast<int32_t>(a.y);
    mir.lock[s] = static_cast<int32_t>(a.z);
    mir.status[s] = static_cast<uint8_t>(a.w & 0xFF);
    mir.backed[s] = static_cast<uint8_t>((a.w >> 8) & 0xFF);
    if (!((a.w >> 16) & KVF_REC_KEEP_RANK)) mir.rank[s] = static_cast<int64_t>((static_cast<uint64_t>(b.y) << 32) | b.x);
    mir.time[s] = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(b.w) << 32) | b.z));
    mir.seq[s] = (static_cast<uint64_t>(c.y) << 32) | c.x;
    mir.id[s] = (static_cast<uint64_t>(c.w) << 32) | c.z;
    mir.tokens[s] = (static_cast<uint64_t>(d.y) << 32) | d.x;
}

// cm (nullable): the resident CTA's shared-memory copy of the tree, updated alongside HBM
__device__ __forceinline__ void apply_records(const DecReq& q, const MirrorDev& mir, const MirrorDev* cm,
                                              const ReqSlot& slot) {
    const bool inl = q.recs == nullptr;
    for (uint32_t i = threadIdx.x; i < q.n_recs; i += blockDim.x) {
        uint4 a, b, c, d;
        if (inl) {
            const uint4* p = reinterpret_cast<const uint4*>(slot.bytes + kHdrBytes) + 4 * i;
            a = p[0];
            b = p[1];
            c = p[2];
            d = p[3];
        } else {
            const uint4* p = reinterpret_cast<const uint4*>(q.recs + i);
            a = __ldcv(p);
            b = __ldcv(p + 1);
            c = __ldcv(p + 2);
            d = __ldcv(p + 3);
        }
        put_rec(mir, a.x, a, b, c, d);
        if (cm) put_rec(*cm, a.x, a, b, c, d);
    }
    __syncthreads();
}

// Slots [from, to) of the HBM mirror -> the shared-memory copy.
__device__ __forceinline__ void load_cache(const MirrorDev& mir, const MirrorDev& cm, uint32_t from, uint32_t to) {
    for (uint32_t i = from + threadIdx.x; i < to; i += blockDim.x) {
        cm.parent[i] = mir.parent[i];
        cm.lock[i] = mir.lock[i];
        cm.status[i] = mir.status[i];
        cm.backed[i] = mir.backed[i];
        cm.rank[i] = mir.rank[i];
        cm.time[i] = mir.time[i];
        cm.seq[i] = mir.seq[i];
        cm.id[i] = mir.id[i];
        cm.tokens[i] = mir.tokens[i];
    }
}

// The shared-memory copy of a tree of up to `cap` slots, placed at `base`: 50 B per slot.
__device__ __forceinline__ MirrorDev cache_view(uint8_t* base, uint32_t cap) {
    MirrorDev m;
    m.rank = reinterpret_cast<int64_t*>(base);
    m.time = reinterpret_cast<double*>(m.rank + cap);
    m.seq = reinterpret_cast<uint64_t*>(m.time + cap);
    m.id = m.seq + cap;
    m.tokens = m.id + cap;
    m.parent = reinterpret_cast<int32_t*>(m.tokens + cap);
    m.lock = m.parent + cap;
    m.status = reinterpret_cast<uint8_t*>(m.lock + cap);
    m.backed = m.status + cap;
    return m;
}

// K4 over the mirror (radix_cache.cpp:266-285): SUFFIX everywhere, then each boundary's
// candidate min-reduced along its root path; ranks that differ from the mirror's are written
// back to it and reported as (slot, rank) changes.
// rd: where the tree is read (the resident CTA's shared-memory copy, or HBM); changed ranks are
// written to HBM and to rd.
__device__ __forceinline__ void prio_body(const DecReq& q, const TreeDesc& td, const MirrorDev& rd, const ReqSlot& slot) {
    extern __shared__ __align__(16) uint8_t sm[];
    __shared__ uint32_t s_cnt;
    const MirrorDev& mir = td.mir;
    const uint32_t n = q.n;
    const bool staged = n <= kPrioSmemNodes;
    long long* r = staged ? reinterpret_cast<long long*>(sm) : td.scratch;
    const int32_t* par = rd.parent;
    if (staged && rd.parent == mir.parent) {
        int32_t* ps = reinterpret_cast<int32_t*>(sm + n * 8ull);
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) ps[i] = mir.parent[i];
        par = ps;
    }
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) r[i] = kRankSuffix;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    // boundaries: inline after the inline records, or in the payload area
    const bool inl = q.bslot == nullptr;
    const unsigned char* ib = slot.bytes + kHdrBytes + q.n_recs * sizeof(kvf_node_rec);
    for (uint32_t b = threadIdx.x; b < q.m; b += blockDim.x) {
        long long c;
        int32_t v;
        if (inl) {
            v = static_cast<int32_t>(reinterpret_cast<const uint32_t*>(ib)[b]);
            c = reinterpret_cast<const long long*>(ib + ((q.m * 4 + 15) & ~15u))[b];
        } else {
            v = static_cast<int32_t>(__ldcv(q.bslot + b));
            c = static_cast<long long>(__ldcv(reinterpret_cast<const unsigned long long*>(q.cand) + b));
        }
        for (; v > 0; v = par[v]) atomicMin(r + v, c);
    }
    __syncthreads();
    unsigned long long* out =
        reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(td.out_k4) + q.k4_buf * td.k4_stride);
    uint32_t* o_slot = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(out) + kHeaderBytes);
    int64_t* o_rank = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(out) + kHeaderBytes + ((n * 4ull + 15) & ~15ull));
    for (uint32_t i = threadIdx.x + 1; i < n; i += blockDim.x) {
        const long long v = r[i];
        const bool ch = rd.status[i] != KVF_SLOT_DEAD && v != rd.rank[i];
        const uint32_t k = claim(&s_cnt, ch);
        if (ch) {
            mir.rank[i] = v;
            rd.rank[i] = v;
            o_slot[k] = i;
            o_rank[k] = v;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[0] = s_cnt;
}

// K5 over the mirror: the snapshot kernel's body (decide_body.cuh) reading the HBM arrays in
// place, depth recomputed from the parents.
__device__ __forceinline__ void victims_body(const DecReq& q, const TreeDesc& td, const MirrorDev& rd) {
    TreeDev t;
    t.parent = rd.parent;
    t.depth = nullptr;
    t.status = rd.status;
    t.lock = rd.lock;
    t.rank = rd.rank;
    t.time = rd.time;
    t.seq = rd.seq;
    t.id = rd.id;
    t.tokens = rd.tokens;
    t.backed = rd.backed;
    t.n = q.n;
    t.bpt = td.bpt;
    t.blob = nullptr;
    t.blob_bytes = 0;
    ReqDev rq{q.needed, q.floor, q.cpu_used, q.cpu_cap, q.wa, q.offload, q.has_floor};
    OutDev o;
    o.header = td.out_k5;
    o.idx = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(td.out_k5) + kHeaderBytes);
    o.action = reinterpret_cast<uint8_t*>(reinterpret_cast<char*>(td.out_k5) + kHeaderBytes + ((q.n * 4ull + 15) & ~15ull));
    o.spin = false;
    victim_body(t, rq, o, 0);
}

// The CTA's state across requests: the descriptor of the tree it served last and, for the
// resident CTA, how many of that tree's slots its shared-memory copy holds.  While a resident
// CTA lives it is the only writer of the small trees' mirrors (a request for any other
// executor stops it first; a mirror reallocation drains it), so the copy stays equal to HBM.
struct ServeState {
    TreeDesc td;
    const TreeDesc* tree;  // nullptr: nothing cached
    uint32_t cached_n;
};

__device__ __forceinline__ void serve(const ReqSlot& slot, Ctl* ctl, unsigned long long seq, unsigned long long polls,
                                      ServeState& ss, const MirrorDev* cm) {
    __shared__ unsigned long long s_seen;
    if (threadIdx.x == 0) s_seen = gtimer();
    const DecReq& q = slot.r;
    const bool fresh = q.tree != ss.tree;  // (read by every thread before the barrier below)
    const uint32_t have = fresh ? 0u : ss.cached_n;
    if (fresh && threadIdx.x < sizeof(TreeDesc) / 8)  // a dependent HBM read: once per tree
        reinterpret_cast<uint64_t*>(&ss.td)[threadIdx.x] = reinterpret_cast<const uint64_t*>(q.tree)[threadIdx.x];
    // a batch that did not fit the slot sits in the payload area: order those reads after the
    // slot's (the host wrote it first)
    if (q.recs || q.bslot) asm volatile("fence.acq_rel.sys;" ::: "memory");
    __syncthreads();
    const TreeDesc& td = ss.td;
    if (cm && q.n > have) {  // a new tree, or slots it grew into: from HBM once
        load_cache(td.mir, *cm, have, q.n);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ss.tree = cm ? q.tree : nullptr;
        ss.cached_n = cm ? max(q.n, have) : 0u;
    }
    apply_records(q, td.mir, cm, slot);
    const MirrorDev& rd = cm ? *cm : td.mir;
    if (q.type == REQ_PRIO || q.type == REQ_PRIO_VICTIMS) prio_body(q, td, rd, slot);
    if (q.type == REQ_PRIO_VICTIMS) __syncthreads();  // the K5 reads the ranks the K4 wrote
    if (q.type == REQ_VICTIMS || q.type == REQ_PRIO_VICTIMS) victims_body(q, td, rd);
    if (threadIdx.x == 0) {  // diagnostics (KVF_MIRROR_TRACE)
        ctl->t_seen[seq % kRing] = s_seen;
        ctl->t_done[seq % kRing] = gtimer();
        ctl->polls[seq % kRing] = polls;
    }
    // every thread's results precede thread 0's release store of the acknowledgement (the
    // barrier orders them before it, the .sys release fence is cumulative): a host that sees
    // the ack sees the results
    __syncthreads();
    if (threadIdx.x == 0) st_release_sys(&ctl->ack[seq % kRing], seq);
}

// One request, one launch (trees above the resident limit, or the resident decider off).  The
// host wrote the slot before the launch, so the first read normally holds it.
__global__ void __launch_bounds__(kThreads) kvf_decide_once(const ReqSlot* slot, Ctl* ctl, unsigned long long seq) {
    __shared__ ReqSlot req;
    __shared__ unsigned long long s_polls;
    if (threadIdx.x < 32) {
        unsigned long long polls = 1;
        while (!read_slot(req, slot, seq, nullptr, nullptr)) ++polls;
        if (threadIdx.x == 0) s_polls = polls;
    }
    __shared__ ServeState ss;
    if (threadIdx.x == 0) ss.tree = nullptr;
    __syncthreads();
    serve(req, ctl, seq, s_polls, ss, nullptr);
}

// scratch of the decision bodies for trees of up to `cap` slots (16-B multiple)
inline size_t resident_scratch(uint32_t cap) {
    const size_t v = victim_smem(cap), p = static_cast<size_t>(cap) * 12 + 64;
    return ((v > p ? v : p) + 15) & ~size_t(15);
}

// The resident decider: serves ring requests first, first+1, ... until idle_ns pass without
// one or the host raises stop_epoch to this launch's epoch; then publishes where it stopped.
__global__ void __launch_bounds__(kResThreads, 4) kvf_decider_kernel(ReqSlot* ring, Ctl* ctl, unsigned long long first,
                                                                      unsigned long long epoch,
                                                                      unsigned long long idle_ns, uint32_t cap,
                                                                      uint32_t cache_off) {
    extern __shared__ __align__(16) uint8_t sm[];
    __shared__ ReqSlot req;
    __shared__ int s_go;
    __shared__ unsigned long long s_polls;
    __shared__ ServeState ss;
    // the tree copy sits after the decision bodies' scratch (cache_off = resident_scratch(cap))
    const MirrorDev cm = cache_view(sm + cache_off, cap);
    if (threadIdx.x == 0) {
        ss.tree = nullptr;
        ss.cached_n = 0;
    }
    unsigned long long next = first;
    unsigned long long last = gtimer();
    for (;;) {
        if (threadIdx.x < 32) {  // warp 0: the whole slot + the stop word, one round trip per poll
            int go = 0;
            unsigned long long polls = 0;
            for (;;) {
                unsigned long long stop = 0;
                ++polls;
                if (read_slot(req, &ring[next % kRing], next, &ctl->stop_epoch, &stop)) {
                    go = 1;
                    break;
                }
                if (stop == epoch || gtimer() - last > idle_ns) break;
            }
            if (threadIdx.x == 0) {
                s_go = go;
                s_polls = polls;
            }
        }
        __syncthreads();
        if (!s_go) break;
        serve(req, ctl, next, s_polls, ss, &cm);
        ++next;
        last = gtimer();
        __syncthreads();  // s_go / req are rewritten next round
    }
    if (threadIdx.x == 0) {
        ctl->exit_next = next;
        __threadfence_system();
        st_release_sys(&ctl->exit_epoch, epoch);
    }
}

// shared memory of a resident CTA serving trees of up to `cap` slots: the decision bodies'
// scratch, then the tree's shared-memory copy (50 B per slot)
size_t resident_smem(uint32_t cap) { return resident_scratch(cap) + static_cast<size_t>(cap) * 50; }
// a resident CTA is sized to the tree it serves (a 44-node tree needs ~3 KB, 512 slots ~25 KB)
uint32_t resident_cap(uint32_t n) {
    uint32_t c = 64;
    while (c < n) c *= 2;
    return c;
}

uint64_t env_idle_ns() {
    const char* s = std::getenv("KVF_DECIDER_IDLE_US");
    return s ? static_cast<uint64_t>(std::strtoull(s, nullptr, 10)) * 1000ull : 200000ull;
}

}  // namespace kvf_mir

using namespace kvf_mir;

// ---------------------------------------------------------------------------------------
// the tree handle
// ---------------------------------------------------------------------------------------
struct kvf_tree {
    kvf_engine* e = nullptr;
    uint64_t bpt = 0;
    uint32_t cap = 0;  // mirror capacity (slots)
    uint32_t n = 1;    // slots in use (high-water mark + 1); slot 0 = root
    void* dblock = nullptr;
    MirrorDev mir{};
    long long* scratch = nullptr;
    char* out_h = nullptr;  // mapped pinned: [K4 result | K5 result]
    char* out_d = nullptr;
    size_t k5_off = 0;
    TreeDesc* desc = nullptr;      // device copy of the mirror / output pointers
    kvf_node_rec* bulk = nullptr;  // device copy of record batches too big for a ring slot
    size_t bulk_cap = 0;
    std::vector<kvf_node_rec> staged;
    // outstanding K4 requests (at most two, oldest at k4_head): sequence number, slot count
    uint64_t k4_seq[2] = {0, 0};
    uint32_t k4_n[2] = {0, 0};
    uint32_t k4_head = 0, k4_count = 0;  // (count includes a staged K4)
    size_t k4_stride = 0;
    // the newest K4, staged on the host until the tree's next request: it travels in the same
    // ring slot as the next K5 (one poll, one serve) or goes alone before any other reader
    bool k4_staged = false;
    uint32_t k4_staged_buf = 0;
    std::vector<uint32_t> k4_bslot;
    std::vector<int64_t> k4_cand;
    kvf_impl::LargeState large;
    kvf_impl::LargeKeyInfo keys;
};

namespace kvf_impl {

namespace {

bool exited(kvf_engine* e) {
    Ctl* c = ring_ctl(e->dec.ring_h);
    return __atomic_load_n(&c->exit_epoch, __ATOMIC_ACQUIRE) == e->dec.epoch;
}

int launch_once(kvf_engine* e, uint64_t seq) {
    DeciderState& d = e->dec;
    const DecReq& q = ring_slot(d.ring_h, seq)->r;
    uint32_t threads = kThreads;
    size_t smem = 0;
    if (q.type == REQ_VICTIMS || q.type == REQ_PRIO_VICTIMS) {
        threads = victim_threads(q.n);
        smem = victim_smem(q.n);
        if (q.type == REQ_PRIO_VICTIMS) smem = std::max<size_t>(smem, q.n * 12ull + 64);
    } else if (q.type == REQ_PRIO) {
        threads = std::min<uint32_t>(kThreads, std::max<uint32_t>(128, pow2_ceil(std::max(q.n, q.m))));
        smem = q.n <= kPrioSmemNodes ? q.n * 12ull + 64 : 0;
    }
    if (!d.once_attr_set) {
        KVF_CUDA(cudaFuncSetAttribute(kvf_decide_once, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(std::max(victim_smem(kMaxNodesSingleCta),
                                                                static_cast<size_t>(kPrioSmemNodes) * 12 + 64))));
        d.once_attr_set = true;
    }
    kvf_decide_once<<<1, threads, smem, e->s_dec>>>(reinterpret_cast<const ReqSlot*>(d.ring_d) + (seq % kRing),
                                                     reinterpret_cast<Ctl*>(ring_ctl(d.ring_d)), seq);
    KVF_CUDA(cudaGetLastError());
    e->stats.kernel_launches++;
    e->stats.oneshot_served++;
    return KVF_OK;
}

int launch_resident(kvf_engine* e, uint64_t first) {
    DeciderState& d = e->dec;
    if (!d.res_attr_set) {
        KVF_CUDA(cudaFuncSetAttribute(kvf_decider_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(resident_smem(KVF_RESIDENT_MAX_SLOTS))));
        d.res_attr_set = true;
    }
    if (d.res_cap == 0) d.res_cap = 64;
    // after every request handed to one-shot launches
    KVF_CUDA(cudaEventRecord(d.ev_dec, e->s_dec));
    KVF_CUDA(cudaStreamWaitEvent(d.s_res, d.ev_dec, 0));
    ++d.epoch;
    kvf_decider_kernel<<<1, kResThreads, resident_smem(d.res_cap), d.s_res>>>(
        reinterpret_cast<ReqSlot*>(d.ring_d), reinterpret_cast<Ctl*>(ring_ctl(d.ring_d)), first, d.epoch,
        d.hold ? ~0ull : d.idle_ns, d.res_cap, static_cast<uint32_t>(resident_scratch(d.res_cap)));
    KVF_CUDA(cudaGetLastError());
    d.running = true;
    e->stats.kernel_launches++;
    e->stats.resident_launches++;
    return KVF_OK;
}

// The resident CTA left: requests handed to it but not served move on -- to a new resident
// CTA (resident = true) or to one-shot launches -- in order, after the old CTA's work.
int after_exit(kvf_engine* e, bool resident) {
    DeciderState& d = e->dec;
    d.running = false;
    const uint64_t next = __atomic_load_n(&ring_ctl(d.ring_h)->exit_next, __ATOMIC_ACQUIRE);
    KVF_CUDA(cudaEventRecord(d.ev_res, d.s_res));
    KVF_CUDA(cudaStreamWaitEvent(e->s_dec, d.ev_res, 0));
    if (next > d.last_res_post) return KVF_OK;  // everything it was given is served
    if (resident) return launch_resident(e, next);
    for (uint64_t s = next; s <= d.last_res_post; ++s)
        if (int rc = launch_once(e, s)) return rc;
    return KVF_OK;
}

int stop_resident(kvf_engine* e) {
    DeciderState& d = e->dec;
    if (!d.running) return KVF_OK;
    __atomic_store_n(&ring_ctl(d.ring_h)->stop_epoch, d.epoch, __ATOMIC_RELEASE);
    const auto t0 = std::chrono::steady_clock::now();
    while (!exited(e)) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(5)) {
            const cudaError_t st = cudaStreamQuery(d.s_res);
            if (st != cudaErrorNotReady) break;  // gone (or faulted) without its exit word
            return set_error(KVF_E_INTERNAL, "resident decider did not stop");
        }
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    return after_exit(e, false);
}

const char* mirror_trace_path() {
    static const char* p = std::getenv("KVF_MIRROR_TRACE");
    return p;
}

int wait_req(kvf_engine* e, uint64_t seq) {
    DeciderState& d = e->dec;
    if (seq <= d.acked) return KVF_OK;
    const volatile unsigned long long* ack = &ring_ctl(d.ring_h)->ack[seq % kRing];
    const auto t0 = std::chrono::steady_clock::now();
    auto next_check = t0 + std::chrono::microseconds(200);
    for (uint32_t it = 1;; ++it) {
        if (*ack >= seq) break;
        if ((it & 15) == 0 && d.running && exited(e)) {  // idled out before it saw the request
            if (int rc = after_exit(e, true)) return rc;
            continue;
        }
        if ((it & 63) == 0 && std::chrono::steady_clock::now() >= next_check) {
            next_check = std::chrono::steady_clock::now() + std::chrono::microseconds(100);
            for (cudaStream_t s : {e->s_dec, d.s_res}) {
                const cudaError_t st = cudaStreamQuery(s);
                if (st != cudaSuccess && st != cudaErrorNotReady) return cuda_error(st, "decision request");
            }
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30))
                return set_error(KVF_E_INTERNAL, "decision request not acknowledged after 30 s");
        }
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    d.acked = std::max<uint64_t>(d.acked, seq);
    if (mirror_trace_path()) {  // diagnostics: host wait, device serve time, polls before the hit
        const Ctl* c = ring_ctl(d.ring_h);
        if (FILE* f = std::fopen(mirror_trace_path(), "a")) {
            std::fprintf(f, "{\"seq\": %llu, \"wait_us\": %.2f, \"serve_us\": %.2f, \"polls\": %llu, \"running\": %d}\n",
                         static_cast<unsigned long long>(seq),
                         std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count(),
                         (c->t_done[seq % kRing] - c->t_seen[seq % kRing]) * 1e-3, c->polls[seq % kRing],
                         d.running ? 1 : 0);
            std::fclose(f);
        }
    }
    return KVF_OK;
}

// Every queued request served, no resident CTA, decision stream idle: buffers the requests
// point into may be freed.
int drain(kvf_engine* e) {
    if (e->dec.posted) {
        if (int rc = wait_req(e, e->dec.posted)) return rc;
    }
    decider_quiesce(e);
    KVF_CUDA(cudaStreamSynchronize(e->s_dec));
    return KVF_OK;
}

int ensure_pay(kvf_engine* e, size_t need) {
    DeciderState& d = e->dec;
    if (need <= d.pay_slot) return KVF_OK;
    if (int rc = drain(e)) return rc;
    if (d.pay_h) cudaFreeHost(d.pay_h);
    d.pay_h = d.pay_d = nullptr;
    size_t sz = std::max(need, d.pay_slot * 2);
    sz = (sz + 4095) & ~size_t(4095);
    void* h = nullptr;
    KVF_CUDA(cudaHostAlloc(&h, sz * kRing, cudaHostAllocMapped | cudaHostAllocPortable));
    void* dp = nullptr;
    KVF_CUDA(cudaHostGetDevicePointer(&dp, h, 0));
    d.pay_h = static_cast<char*>(h);
    d.pay_d = static_cast<char*>(dp);
    d.pay_slot = sz;
    return KVF_OK;
}

size_t k4_out_bytes(uint32_t cap) { return kHeaderBytes + ((cap * 4ull + 15) & ~15ull) + cap * 8ull; }
size_t k5_out_bytes(uint32_t cap) { return kHeaderBytes + ((cap * 4ull + 15) & ~15ull) + ((cap + 15ull) & ~15ull); }

// Mirror capacity >= need (and the large path's padded size): a new block, old slots copied,
// new slots dead.  Everything queued so far is served first (the old block is freed).
int ensure_cap(kvf_tree* t, uint32_t need) {
    if (need <= t->cap) return KVF_OK;
    kvf_engine* e = t->e;
    uint32_t cap = std::max<uint32_t>(need + need / 2, 1024);
    cap = large_capacity(cap);
    if (int rc = drain(e)) return rc;
    // unread K4 results live in the output block being replaced: carry them over
    std::vector<char> k4_keep[2];
    for (uint32_t b = 0; b < 2; ++b)
        for (uint32_t k = 0; k < t->k4_count; ++k)
            if ((t->k4_head + k) % 2 == b && t->out_h)
                k4_keep[b].assign(t->out_h + b * t->k4_stride, t->out_h + b * t->k4_stride + k4_out_bytes(t->k4_n[b]));
    const size_t n = cap;
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t bytes = al(n * 4) * 2 + al(n) * 2 + al(n * 8) * 6;
    void* blk = nullptr;
    KVF_CUDA(cudaMalloc(&blk, bytes));
    char* p = static_cast<char*>(blk);
    MirrorDev m;
    m.parent = reinterpret_cast<int32_t*>(p); p += al(n * 4);
    m.lock = reinterpret_cast<int32_t*>(p); p += al(n * 4);
    m.status = reinterpret_cast<uint8_t*>(p); p += al(n);
    m.backed = reinterpret_cast<uint8_t*>(p); p += al(n);
    m.rank = reinterpret_cast<int64_t*>(p); p += al(n * 8);
    m.time = reinterpret_cast<double*>(p); p += al(n * 8);
    m.seq = reinterpret_cast<uint64_t*>(p); p += al(n * 8);
    m.id = reinterpret_cast<uint64_t*>(p); p += al(n * 8);
    m.tokens = reinterpret_cast<uint64_t*>(p); p += al(n * 8);
    long long* scratch = reinterpret_cast<long long*>(p);
    KVF_CUDA(cudaMemset(blk, 0, bytes));
    KVF_CUDA(cudaMemset(m.parent, 0xFF, n * 4));              // -1
    KVF_CUDA(cudaMemset(m.status, KVF_SLOT_DEAD, n));
    if (t->dblock) {
        const size_t o = t->cap;
        KVF_CUDA(cudaMemcpy(m.parent, t->mir.parent, o * 4, cudaMemcpyDeviceToDevice));
        KVF_CUDA(cudaMemcpy(m.lock, t->mir.lock, o * 4, cudaMemcpyDeviceToDevice));
        KVF_CUDA(cudaMemcpy(m.status, t->mir.status, o, cudaMemcpyDeviceToDevice));
        KVF_CUDA(cudaMemcpy(m.backed, t->mir.backed, o, cudaMemcpyDeviceToDevice));
        KVF_CUDA(cudaMemcpy(m.rank, t->mir.rank, o * 8, cudaMemcpyDeviceToDevice));
        KVF_CUDA(cudaMemcpy(m.time, t->mir.time, o * 8, cudaMemcpyDeviceToDevice));
        KVF_CUDA(cudaMemcpy(m.seq, t->mir.seq, o * 8, cudaMemcpyDeviceToDevice));
        KVF_CUDA(cudaMemcpy(m.id, t->mir.id, o * 8, cudaMemcpyDeviceToDevice));
        KVF_CUDA(cudaMemcpy(m.tokens, t->mir.tokens, o * 8, cudaMemcpyDeviceToDevice));
        cudaFree(t->dblock);
        large_invalidate(t->large);
    }
    t->dblock = blk;
    t->mir = m;
    t->scratch = scratch;
    // results: posted writes into mapped pinned memory
    if (t->out_h) cudaFreeHost(t->out_h);
    t->out_h = t->out_d = nullptr;
    t->k4_stride = (k4_out_bytes(cap) + 255) & ~size_t(255);
    t->k5_off = 2 * t->k4_stride;
    void* h = nullptr;
    KVF_CUDA(cudaHostAlloc(&h, t->k5_off + k5_out_bytes(cap), cudaHostAllocMapped | cudaHostAllocPortable));
    void* dp = nullptr;
    KVF_CUDA(cudaHostGetDevicePointer(&dp, h, 0));
    t->out_h = static_cast<char*>(h);
    t->out_d = static_cast<char*>(dp);
    for (uint32_t b = 0; b < 2; ++b)
        if (!k4_keep[b].empty()) std::memcpy(t->out_h + b * t->k4_stride, k4_keep[b].data(), k4_keep[b].size());
    t->cap = cap;
    if (!t->desc) KVF_CUDA(cudaMalloc(reinterpret_cast<void**>(&t->desc), sizeof(TreeDesc)));
    TreeDesc td{t->mir, t->scratch, reinterpret_cast<unsigned long long*>(t->out_d),
                reinterpret_cast<unsigned long long*>(t->out_d + t->k5_off), t->bpt, t->k4_stride};
    KVF_CUDA(cudaMemcpy(t->desc, &td, sizeof(td), cudaMemcpyHostToDevice));
    return KVF_OK;
}

// Queue one request on t's ring (records staged so far travel with it).  *seq_out = its number.
int post(kvf_tree* t, uint32_t type, const uint32_t* bslot, const int64_t* cand, uint32_t m,
         const kvf_evict_request* q, uint64_t* seq_out, uint32_t k4_buf = 0) {
    kvf_engine* e = t->e;
    DeciderState& d = e->dec;
    if (int rc = ensure_cap(t, t->n > kMaxNodesSingleCta ? large_capacity(t->n) : t->n)) return rc;
    const size_t rec_bytes = t->staged.size() * sizeof(kvf_node_rec);
    const size_t pay = rec_bytes + ((m * 4ull + 15) & ~15ull) + m * 8ull;
    const bool inl = pay <= kInlineBytes;   // the common case: everything in the polled slot
    const bool bulk = pay > kPaySlotBytes;  // one-time large syncs go through a device copy
    if (int rc = ensure_pay(e, bulk ? ((m * 12ull + 64 + 15) & ~15ull) : pay)) return rc;
    if (bulk && rec_bytes > t->bulk_cap) {  // (before this request takes a number: drain waits for all)
        if (int rc = drain(e)) return rc;
        if (t->bulk) cudaFree(t->bulk);
        t->bulk = nullptr;
        const size_t sz = std::max(rec_bytes, t->bulk_cap * 2);
        KVF_CUDA(cudaMalloc(reinterpret_cast<void**>(&t->bulk), sz));
        t->bulk_cap = sz;
    }
    const bool resident = !d.disabled && !bulk && t->n <= KVF_RESIDENT_MAX_SLOTS && type != REQ_APPLY;
    // a resident CTA too small for this tree makes way for a bigger one
    if (d.running && (!resident || resident_cap(t->n) > d.res_cap)) {
        if (int rc = stop_resident(e)) return rc;
    }
    if (resident && !d.running) d.res_cap = std::max(d.res_cap, resident_cap(t->n));
    const uint64_t seq = ++d.posted;
    if (seq > kRing) {  // the slot's previous request must be done
        if (int rc = wait_req(e, seq - kRing)) return rc;
    }
    ReqSlot* slot = ring_slot(d.ring_h, seq);
    char* ph = inl ? reinterpret_cast<char*>(slot->bytes + kHdrBytes) : d.pay_h + (seq % kRing) * d.pay_slot;
    char* pd = d.pay_d + (seq % kRing) * d.pay_slot;
    const kvf_node_rec* recs_dev = inl ? nullptr : reinterpret_cast<const kvf_node_rec*>(pd);
    size_t off = 0;
    if (bulk) {
        KVF_CUDA(cudaMemcpyAsync(t->bulk, t->staged.data(), rec_bytes, cudaMemcpyHostToDevice, e->s_dec));
        recs_dev = t->bulk;
    } else {
        if (rec_bytes) std::memcpy(ph, t->staged.data(), rec_bytes);
        off = rec_bytes;
    }
    if (m) {
        std::memcpy(ph + off, bslot, m * 4ull);
        std::memcpy(ph + off + ((m * 4ull + 15) & ~15ull), cand, m * 8ull);
    }
    DecReq r{};
    r.type = type;
    r.n = t->n;
    r.n_recs = static_cast<uint32_t>(t->staged.size());
    r.m = m;
    r.k4_buf = k4_buf;
    r.tree = t->desc;
    r.recs = recs_dev;
    r.bslot = inl ? nullptr : reinterpret_cast<const uint32_t*>(pd + off);
    r.cand = inl ? nullptr : reinterpret_cast<const int64_t*>(pd + off + ((m * 4ull + 15) & ~15ull));
    if (q) {
        r.needed = q->needed;
        r.floor = q->floor;
        r.cpu_used = q->cpu_used;
        r.cpu_cap = q->cpu_capacity;
        r.wa = q->workflow_aware;
        r.offload = q->offload_mode;
        r.has_floor = q->has_floor;
    }
    std::memcpy(reinterpret_cast<char*>(slot) + 16, reinterpret_cast<const char*>(&r) + 16, sizeof(r) - 16);
    // the hash over what the slot now holds (seq and bytes 16..511), then seq last
    uint64_t h = mix64(seq);
    for (uint32_t c = 1; c < kSlotBytes / 16; ++c) {
        uint64_t w[2];
        std::memcpy(w, slot->bytes + 16 * c, 16);
        h ^= chunk_hash(w[0], w[1], c);
    }
    __atomic_store_n(&slot->r.hash, static_cast<unsigned long long>(h), __ATOMIC_RELEASE);
    e->stats.mirror_records += t->staged.size();
    t->staged.clear();
    if (resident) {
        if (d.running && exited(e)) {
            if (int rc = after_exit(e, true)) return rc;
        }
        d.last_res_post = seq;
        __atomic_store_n(&slot->r.seq, static_cast<unsigned long long>(seq), __ATOMIC_RELEASE);
        if (!d.running) {
            if (int rc = launch_resident(e, seq)) return rc;
        }
        e->stats.resident_served++;
    } else {
        __atomic_store_n(&slot->r.seq, static_cast<unsigned long long>(seq), __ATOMIC_RELEASE);
        if (int rc = launch_once(e, seq)) return rc;
    }
    e->stats.decisions++;
    *seq_out = seq;
    return KVF_OK;
}

// The staged K4 on the ring by itself (a reader needs its result, or the next request cannot
// carry it).
int post_staged_k4(kvf_tree* t) {
    if (!t->k4_staged) return KVF_OK;
    t->k4_staged = false;
    const uint32_t b = t->k4_staged_buf;
    uint64_t seq = 0;
    if (int rc = post(t, REQ_PRIO, t->k4_bslot.data(), t->k4_cand.data(), static_cast<uint32_t>(t->k4_bslot.size()),
                      nullptr, &seq, b))
        return rc;
    t->k4_seq[b] = seq;
    t->k4_n[b] = t->n;
    return KVF_OK;
}

}  // namespace

void decider_quiesce(kvf_engine* e) {
    if (!e || !e->dec.ring_h) return;
    stop_resident(e);
}

namespace {
// Engines whose resident CTA may be alive.  At process exit (before the CUDA runtime's own
// teardown, registered earlier) every one is stopped: a CTA still polling the ring while its
// mapped memory is torn down would fault.
std::mutex g_live_mu;
std::set<kvf_engine*>* g_live = nullptr;
void stop_all_at_exit() {
    std::lock_guard<std::mutex> g(g_live_mu);
    if (!g_live) return;
    for (kvf_engine* e : *g_live) {
        std::lock_guard<std::mutex> lk(e->mu);
        cudaSetDevice(e->device);
        stop_resident(e);
        cudaStreamSynchronize(e->dec.s_res);
    }
}
void register_live(kvf_engine* e, bool live) {
    std::lock_guard<std::mutex> g(g_live_mu);
    if (!g_live) {
        g_live = new std::set<kvf_engine*>();
        std::atexit(stop_all_at_exit);
    }
    if (live) g_live->insert(e);
    else g_live->erase(e);
}
}  // namespace

int decider_init(kvf_engine* e) {
    DeciderState& d = e->dec;
    const char* env = std::getenv("KVF_DECIDER");
    d.disabled = env && env[0] == '0';
    d.idle_ns = env_idle_ns();
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    KVF_CUDA(cudaStreamCreateWithPriority(&d.s_res, cudaStreamNonBlocking, hi));
    KVF_CUDA(cudaEventCreateWithFlags(&d.ev_res, cudaEventDisableTiming));
    KVF_CUDA(cudaEventCreateWithFlags(&d.ev_dec, cudaEventDisableTiming));
    void* h = nullptr;
    const size_t ring_bytes = kRing * sizeof(ReqSlot) + sizeof(Ctl);
    KVF_CUDA(cudaHostAlloc(&h, ring_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(h, 0, ring_bytes);
    void* dp = nullptr;
    KVF_CUDA(cudaHostGetDevicePointer(&dp, h, 0));
    d.ring_h = static_cast<char*>(h);
    d.ring_d = static_cast<char*>(dp);
    register_live(e, true);
    return ensure_pay(e, kPaySlotBytes);
}

void decider_release(kvf_engine* e) {
    register_live(e, false);
    DeciderState& d = e->dec;
    if (d.ring_h) stop_resident(e);
    if (d.s_res) cudaStreamSynchronize(d.s_res);
    if (d.ring_h) cudaFreeHost(d.ring_h);
    if (d.pay_h) cudaFreeHost(d.pay_h);
    if (d.s_res) cudaStreamDestroy(d.s_res);
    for (cudaEvent_t ev : {d.ev_res, d.ev_dec})
        if (ev) cudaEventDestroy(ev);
    d = DeciderState{};
}

void set_carveout_mirror() {
    cudaFuncSetAttribute(kvf_decide_once, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(kvf_decider_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
}

}  // namespace kvf_impl

// ---------------------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------------------
extern "C" {

int kvf_tree_create(kvf_engine* e, uint64_t bytes_per_token, uint32_t capacity_hint, kvf_tree** out) {
    if (!out) return set_error(KVF_E_INVALID_ARG, "null argument");
    *out = nullptr;
    KVF_GUARD(e);
    if (bytes_per_token == 0) return set_error(KVF_E_INVALID_ARG, "bytes_per_token must be > 0");
    auto* t = new kvf_tree();
    t->e = e;
    t->bpt = bytes_per_token;
    t->large.ws.owner = e;
    if (int rc = ensure_cap(t, std::max<uint32_t>(capacity_hint, 1024))) {
        delete t;
        return rc;
    }
    *out = t;
    return KVF_OK;
}

int kvf_tree_destroy(kvf_tree* t) {
    if (!t) return KVF_OK;
    kvf_engine* e = t->e;
    {
        std::lock_guard<std::mutex> lk(e->mu);
        cudaSetDevice(e->device);
        drain(e);
        large_release(t->large);
        if (t->dblock) cudaFree(t->dblock);
        if (t->bulk) cudaFree(t->bulk);
        if (t->desc) cudaFree(t->desc);
        if (t->out_h) cudaFreeHost(t->out_h);
    }
    delete t;
    return KVF_OK;
}

int kvf_tree_set_hints(kvf_tree* t, uint32_t hints) {
    if (!t) return set_error(KVF_E_INVALID_ARG, "null tree");
    KVF_GUARD(t->e);
    t->keys.time_follows_seq = (hints & KVF_TREE_TIME_FOLLOWS_SEQ) != 0;
    return KVF_OK;
}

int kvf_tree_update(kvf_tree* t, const kvf_node_rec* recs, uint32_t n) {
    if (!t || (n && !recs)) return set_error(KVF_E_INVALID_ARG, "null argument");
    KVF_GUARD(t->e);
    for (uint32_t i = 0; i < n; ++i) {
        const kvf_node_rec& r = recs[i];
        if (r.slot >= (1u << 24)) return set_error(KVF_E_INVALID_ARG, "slot beyond 2^24");
        if (r.parent >= static_cast<int32_t>(1u << 24) || r.parent < -1)
            return set_error(KVF_E_INVALID_ARG, "parent slot outside [-1, 2^24)");
        // a parent named before its own record arrives still lies inside the mirror
        t->n = std::max<uint32_t>(t->n, std::max<uint32_t>(r.slot + 1, static_cast<uint32_t>(r.parent + 1)));
        t->keys.note(r);
    }
    t->staged.insert(t->staged.end(), recs, recs + n);
    return KVF_OK;
}

int kvf_tree_stage_priorities(kvf_tree* t, const uint32_t* boundary_slot, const int64_t* cand_rank, uint32_t m) {
    if (!t || (m && (!boundary_slot || !cand_rank))) return set_error(KVF_E_INVALID_ARG, "null argument");
    KVF_GUARD(t->e);
    for (uint32_t b = 0; b < m; ++b) {
        if (boundary_slot[b] >= t->n) return set_error(KVF_E_UNKNOWN_BOUNDARY_NODE, "boundary slot out of range");
        t->keys.note_rank(cand_rank[b]);
    }
    if (t->k4_count == 2) {  // both result buffers hold unread changes: the host reads the oldest first
        return set_error(KVF_E_INVALID_ARG, "two K4 results unread: call kvf_tree_rank_changes first");
    }
    if (int rc = post_staged_k4(t)) return rc;  // the previous one, in order
    t->k4_staged_buf = (t->k4_head + t->k4_count) % 2;
    t->k4_bslot.assign(boundary_slot, boundary_slot + m);
    t->k4_cand.assign(cand_rank, cand_rank + m);
    t->k4_staged = true;
    t->k4_count++;
    return KVF_OK;
}

int kvf_tree_priorities(kvf_tree* t, const uint32_t* boundary_slot, const int64_t* cand_rank, uint32_t m) {
    if (int rc = kvf_tree_stage_priorities(t, boundary_slot, cand_rank, m)) return rc;
    KVF_GUARD(t->e);
    return post_staged_k4(t);  // on the ring now: it runs while the caller goes on
}

int kvf_tree_rank_changes(kvf_tree* t, uint32_t* slots, int64_t* ranks, uint32_t cap, uint32_t* n_changed) {
    if (!t || !n_changed) return set_error(KVF_E_INVALID_ARG, "null argument");
    KVF_GUARD(t->e);
    *n_changed = 0;
    if (!t->k4_count) return KVF_OK;
    const auto t0 = std::chrono::steady_clock::now();
    const uint32_t b = t->k4_head;
    if (t->k4_staged && t->k4_staged_buf == b) {
        if (int rc = post_staged_k4(t)) return rc;
    }
    if (int rc = wait_req(t->e, t->k4_seq[b])) return rc;
    const char* o = t->out_h + b * t->k4_stride;
    const uint64_t* hdr = reinterpret_cast<const uint64_t*>(o);
    const uint32_t cnt = static_cast<uint32_t>(hdr[0]);
    if (cnt > cap || (cnt && (!slots || !ranks))) return set_error(KVF_E_INVALID_ARG, "rank-change buffer too small");
    std::memcpy(slots, o + kHeaderBytes, cnt * 4ull);
    std::memcpy(ranks, o + kHeaderBytes + ((t->k4_n[b] * 4ull + 15) & ~15ull), cnt * 8ull);
    *n_changed = cnt;
    t->k4_seq[b] = 0;
    t->k4_head = (b + 1) % 2;
    t->k4_count--;
    t->e->stats.decision_call_us +=
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    return KVF_OK;
}

int kvf_tree_victims(kvf_tree* t, const kvf_evict_request* req, uint32_t* out_slot, uint8_t* out_action, uint32_t cap,
                     uint32_t* out_count, uint64_t* out_imm, uint64_t* out_pend) {
    if (!t || !req || !out_count || !out_imm || !out_pend) return set_error(KVF_E_INVALID_ARG, "null argument");
    KVF_GUARD(t->e);
    kvf_engine* e = t->e;
    *out_count = 0;
    *out_imm = *out_pend = 0;
    const auto t0 = std::chrono::steady_clock::now();
    uint32_t cnt = 0;
    if (t->n > kMaxNodesSingleCta) {  // device-wide path: records first, then the grid kernels
        uint64_t seq = 0;
        if (int rc = post_staged_k4(t)) return rc;  // its ranks first (a one-shot launch)
        if (int rc = post(t, REQ_APPLY, nullptr, nullptr, 0, nullptr, &seq)) return rc;
        LargeArrays a{t->mir.parent, t->mir.status, t->mir.lock, t->mir.rank, t->mir.time,
                      t->mir.seq,    t->mir.id,     t->mir.tokens, t->mir.backed, t->n};
        if (int rc = victim_large(e, t->large, a, req, t->bpt, t->keys, out_slot, out_action, cap, &cnt, out_imm, out_pend))
            return rc;
        e->stats.decisions++;
        *out_count = cnt;
    } else if (t->n > 1 && req->needed) {
        uint64_t seq = 0;
        if (t->k4_staged) {  // the queued K4 and this K5 in one ring slot
            t->k4_staged = false;
            const uint32_t b = t->k4_staged_buf;
            if (int rc = post(t, REQ_PRIO_VICTIMS, t->k4_bslot.data(), t->k4_cand.data(),
                              static_cast<uint32_t>(t->k4_bslot.size()), req, &seq, b))
                return rc;
            t->k4_seq[b] = seq;
            t->k4_n[b] = t->n;
        } else if (int rc = post(t, REQ_VICTIMS, nullptr, nullptr, 0, req, &seq)) {
            return rc;
        }
        if (int rc = wait_req(e, seq)) return rc;
        const char* o = t->out_h + t->k5_off;
        const uint64_t* hdr = reinterpret_cast<const uint64_t*>(o);
        cnt = static_cast<uint32_t>(hdr[0]);
        if (cnt > t->n) return set_error(KVF_E_INTERNAL, "K5 returned more victims than slots");
        if (cnt > cap || (cnt && (!out_slot || !out_action))) return set_error(KVF_E_INVALID_ARG, "victim buffer too small");
        std::memcpy(out_slot, o + kHeaderBytes, cnt * 4ull);
        std::memcpy(out_action, o + kHeaderBytes + ((t->n * 4ull + 15) & ~15ull), cnt);
        for (int k = 0; k < 5; ++k) {
            e->stats.k5_phase_ns[k] += static_cast<double>(hdr[4 + k] - hdr[3 + k]);
            e->stats.k5_phase_cycles[k] += static_cast<double>(hdr[10 + k] - hdr[9 + k]);
        }
        e->stats.decision_kernel_ms += static_cast<double>(hdr[8] - hdr[3]) * 1e-6;
        *out_count = cnt;
        *out_imm = hdr[1];
        *out_pend = hdr[2];
    }
    e->stats.decision_call_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    return KVF_OK;
}

int kvf_decider_hold(kvf_engine* e, int32_t hold) {
    KVF_GUARD(e);
    e->dec.hold = hold != 0;
    if (!hold) decider_quiesce(e);          // leave now (its queue is served first)
    else if (e->dec.running && !e->dec.disabled) decider_quiesce(e);  // relaunched without an idle limit
    // a held decider starts now, ahead of the run's first request: launched later it would
    // queue for an SM behind whatever bulk grid (a prompt's payload fill, a K1) is running
    if (hold && !e->dec.disabled && !e->dec.running) return launch_resident(e, e->dec.posted + 1);
    return KVF_OK;
}

int kvf_decider_running(kvf_engine* e, int32_t* running) {
    if (!running) return set_error(KVF_E_INVALID_ARG, "null argument");
    KVF_GUARD(e);
    if (e->dec.running && exited(e)) after_exit(e, false);
    *running = e->dec.running ? 1 : 0;
    return KVF_OK;
}

}  // extern "C"
