// libkvflow.so -- B200-native KV-movement engine (pools, jobs, K1/K2/K3 copy kernels,
// payload fill + checksum).  Decisions (K4/K5) live in decide.cu.
//
// Replaces the modelled transfers of the reference tier engine
// (proj/src/tier_manager.cpp:35-124): there a TransferJob's completion time is
// bytes/(bw*eff)+latency; here a job is a real sm_100a kernel on a dedicated copy stream
// bracketed by CUDA events, and "completion" is the stop event.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "engine_internal.hpp"

using namespace kvf_impl;

// =====================================================================================
// errors
// =====================================================================================
namespace kvf_impl {
constexpr size_t kMaxPiecesPublic = 48;  // = kMaxPieces below: pieces one copy launch carries
static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_error(cudaError_t e, const char* what) {
    return set_error(KVF_E_CUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

// =====================================================================================
// slot allocator
// =====================================================================================
void SlotAllocator::reset(uint64_t slots) {
    by_start_.clear();
    by_len_.clear();
    capacity_ = slots;
    free_tokens_ = 0;
    if (slots) insert_free(0, slots);
}

void SlotAllocator::insert_free(uint64_t start, uint64_t len) {
    by_start_.emplace(start, len);
    by_len_.emplace(len, start);
    free_tokens_ += len;
}

void SlotAllocator::erase_free(std::map<uint64_t, uint64_t>::iterator it) {
    auto range = by_len_.equal_range(it->second);
    for (auto j = range.first; j != range.second; ++j)
        if (j->second == it->first) {
            by_len_.erase(j);
            break;
        }
    free_tokens_ -= it->second;
    by_start_.erase(it);
}

bool SlotAllocator::alloc(uint64_t tokens, std::vector<kvf_run>& out) {
    out.clear();
    if (tokens == 0) return true;
    if (tokens > free_tokens_) return false;
    // best fit: smallest free run that holds everything -> one run, no fragmentation
    auto fit = by_len_.lower_bound(tokens);
    if (fit != by_len_.end()) {
        uint64_t start = fit->second, len = fit->first;
        erase_free(by_start_.find(start));
        out.push_back({start, tokens});
        if (len > tokens) insert_free(start + tokens, len - tokens);
        return true;
    }
    // otherwise take the largest runs first (fewest pieces for the copy kernels)
    uint64_t need = tokens;
    while (need > 0) {
        auto big = std::prev(by_len_.end());
        uint64_t start = big->second, len = big->first;
        erase_free(by_start_.find(start));
        uint64_t take = std::min(len, need);
        out.push_back({start, take});
        if (len > take) insert_free(start + take, len - take);
        need -= take;
    }
    return true;
}

bool SlotAllocator::release(const kvf_run& r) {
    if (r.len == 0) return true;
    if (r.start + r.len > capacity_ || r.start + r.len < r.start) return false;
    uint64_t start = r.start, len = r.len;
    auto next = by_start_.lower_bound(start);
    if (next != by_start_.end() && next->first < start + len) return false;  // overlaps a free run
    if (next != by_start_.begin()) {
        auto prev = std::prev(next);
        if (prev->first + prev->second > start) return false;
        if (prev->first + prev->second == start) {  // coalesce left
            start = prev->first;
            len += prev->second;
            erase_free(prev);
        }
    }
    next = by_start_.lower_bound(start + len);
    if (next != by_start_.end() && next->first == start + len) {  // coalesce right
        len += next->second;
        erase_free(next);
    }
    insert_free(start, len);
    return true;
}

void merge_runs(const kvf_run* a, uint32_t na, const kvf_run* b, uint32_t nb, std::vector<Piece>& out) {
    out.clear();
    uint32_t i = 0, j = 0;
    uint64_t ao = 0, bo = 0;
    while (i < na && j < nb) {
        uint64_t l = std::min(a[i].len - ao, b[j].len - bo);
        if (l) {
            if (!out.empty() && out.back().src_slot + out.back().ntok == a[i].start + ao &&
                out.back().dst_slot + out.back().ntok == b[j].start + bo)
                out.back().ntok += l;  // adjacent on both sides: one piece
            else
                out.push_back({a[i].start + ao, b[j].start + bo, l});
        }
        ao += l;
        bo += l;
        if (ao == a[i].len) { ++i; ao = 0; }
        if (bo == b[j].len) { ++j; bo = 0; }
    }
}

int Workspace::ensure(size_t dn, size_t hn) {
    if (owner && ((dn > dev_bytes && dev) || (hn > host_bytes && host))) decider_quiesce(owner);
    if (dn > dev_bytes) {
        if (dev) cudaFree(dev);
        dev = nullptr;
        size_t sz = std::max(dn, dev_bytes * 2);
        KVF_CUDA(cudaMalloc(&dev, sz));
        dev_bytes = sz;
    }
    if (hn > host_bytes) {
        if (host) cudaFreeHost(host);
        host = nullptr;
        size_t sz = std::max(hn, host_bytes * 2);
        KVF_CUDA(cudaHostAlloc(&host, sz, cudaHostAllocMapped | cudaHostAllocPortable));
        KVF_CUDA(cudaHostGetDevicePointer(&host_dev, host, 0));
        host_bytes = sz;
    }
    return KVF_OK;
}

void Workspace::release() {
    if (dev) cudaFree(dev);
    if (host) cudaFreeHost(host);
    dev = host = host_dev = nullptr;
    dev_bytes = host_bytes = 0;
}

// A non-sticky error left in the runtime's per-thread slot by an unchecked call elsewhere
// (another engine's teardown, a caller's own CUDA use) must not be reported by the next
// launch check of this call: take it out at entry, count it, optionally trace it
// (KVF_TRACE_STALE=1).  Sticky errors (a faulted context) resurface at the next sync anyway.
void clear_stale_error(kvf_engine* e, const char* fn) {
    const cudaError_t stale = cudaGetLastError();
    if (stale == cudaSuccess) return;
    e->stats.stale_errors++;
    static const bool trace = std::getenv("KVF_TRACE_STALE") != nullptr;
    if (trace) std::fprintf(stderr, "kvflow: stale %s before %s\n", cudaGetErrorName(stale), fn);
}

int acquire_event(kvf_engine* e, cudaEvent_t* ev, bool timing) {
    std::vector<cudaEvent_t>& pool = timing ? e->event_pool : e->event_pool_nt;
    if (!pool.empty()) {
        *ev = pool.back();
        pool.pop_back();
        return KVF_OK;
    }
    KVF_CUDA(cudaEventCreateWithFlags(ev, timing ? cudaEventDefault : cudaEventDisableTiming));
    return KVF_OK;
}

void recycle_event(kvf_engine* e, cudaEvent_t ev, bool timing) {
    if (ev) (timing ? e->event_pool : e->event_pool_nt).push_back(ev);
}

int begin_job(kvf_engine* e, uint64_t job_id, cudaStream_t stream, Job& j, int32_t stamp_slot) {
    if (e->jobs.count(job_id)) return set_error(KVF_E_INVALID_ARG, "job id " + std::to_string(job_id) + " already in use");
    j.stream = stream;
    if (stamp_slot >= 0) {  // a timing event record costs ~1.3 us of host time, a plain one ~0.1
        j.stamp_slot = stamp_slot;
        e->stamp_refs[stamp_slot]++;
        return acquire_event(e, &j.stop, false);
    }
    int rc = acquire_event(e, &j.start, true);
    if (rc) return rc;
    rc = acquire_event(e, &j.stop, true);
    if (rc) return rc;
    KVF_CUDA(cudaEventRecord(j.start, stream));
    return KVF_OK;
}

// A stamp slot for the next copy launch, or -1 (event timing: the engine's mode, no free slot,
// or a copy that takes more than one launch).
int32_t take_stamp_slot(kvf_engine* e, size_t npieces, uint32_t mode) {
    if (!e->stamp_timing || mode != KVF_COPY_SM_VEC || npieces > kMaxPiecesPublic || e->stamp_free.empty()) return -1;
    const int32_t s = e->stamp_free.back();
    e->stamp_free.pop_back();
    e->stamp_refs[s] = 0;
    std::memset(e->stamps_h + static_cast<size_t>(s) * kStampCtas * 2, 0, kStampCtas * 2 * sizeof(unsigned long long));
    return s;
}

void drop_stamp_ref(kvf_engine* e, int32_t s) {
    if (s >= 0 && --e->stamp_refs[s] == 0) e->stamp_free.push_back(s);
}


int end_job(kvf_engine* e, uint64_t job_id, Job& j) {
    KVF_CUDA(cudaEventRecord(j.stop, j.stream));
    e->jobs.emplace(job_id, j);
    return KVF_OK;
}

}  // namespace kvf_impl

// =====================================================================================
// kernels
// =====================================================================================
namespace {

constexpr uint32_t kMaxPieces = 48;

// One launch copies up to kMaxPieces pieces x all planes.  The work is cut into
// fixed-size tiles (a tile never spans two plane segments) that CTAs take grid-stride.
struct CopyParams {
    const char* src;
    char* dst;
    uint64_t src_stride;  // bytes between planes in the source pool
    uint64_t dst_stride;
    uint64_t total_tiles;
    uint32_t planes;
    uint32_t npieces;
    uint32_t tile_bytes;
    uint32_t layer_major;  // tiles ordered plane-outermost (layer-pipelined K1)
    uint64_t plane_tiles;  // layer_major: tiles of one plane (sum over pieces)
    uint32_t* layer_ready; // layer_major: per-layer finished-tile counters (nullable)
    unsigned long long* stamps;  // nullable: CTA b < kStampCtas writes [2b] = start, [2b+1] = end (ns)
    uint64_t src_off[kMaxPieces];
    uint64_t dst_off[kMaxPieces];
    uint64_t seg[kMaxPieces];             // bytes of the piece in one plane
    uint64_t tile_begin[kMaxPieces + 1];  // prefix over pieces of planes*ceil(seg/tile)
                                          // (layer_major: of ceil(seg/tile), one plane)
};

struct TileRef {
    const char* s;
    char* d;
    uint32_t len;
};

__device__ __forceinline__ TileRef locate(const CopyParams& p, uint64_t t, uint32_t* plane_out = nullptr) {
    // piece-major: t -> (piece, plane, tile);  layer-major: t -> (plane, piece, tile)
    uint64_t plane = 0;
    if (p.layer_major) {
        plane = t / p.plane_tiles;
        t -= plane * p.plane_tiles;
    }
    uint32_t lo = 0, hi = p.npieces - 1;
    while (lo < hi) {
        uint32_t mid = (lo + hi + 1) >> 1;
        if (p.tile_begin[mid] <= t) lo = mid; else hi = mid - 1;
    }
    const uint64_t local = t - p.tile_begin[lo];
    const uint64_t seg = p.seg[lo];
    const uint64_t tps = (seg + p.tile_bytes - 1) / p.tile_bytes;
    if (!p.layer_major) plane = local / tps;
    const uint64_t off = (local - (p.layer_major ? 0 : plane * tps)) * p.tile_bytes;
    if (plane_out) *plane_out = static_cast<uint32_t>(plane);
    TileRef r;
    r.s = p.src + plane * p.src_stride + p.src_off[lo] + off;
    r.d = p.dst + plane * p.dst_stride + p.dst_off[lo] + off;
    r.len = static_cast<uint32_t>((seg - off < p.tile_bytes ? seg - off : (uint64_t)p.tile_bytes));
    return r;
}

__device__ __forceinline__ uint4 ld_stream(const uint4* ptr) {
    uint4 v;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(ptr));
    return v;
}
__device__ __forceinline__ void st_stream(uint4* ptr, const uint4& v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(ptr), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint2 ld_stream(const uint2* ptr) {
    uint2 v;
    asm volatile("ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(ptr));
    return v;
}
__device__ __forceinline__ void st_stream(uint2* ptr, const uint2& v) {
    asm volatile("st.global.L1::no_allocate.v2.u32 [%0], {%1,%2};" ::"l"(ptr), "r"(v.x), "r"(v.y) : "memory");
}

// K1/K2/K3, SM vector path: every thread keeps UNROLL independent 16-B loads in flight
// before its stores (PCIe latency hiding for K1; HBM streaming for K3).
__device__ __forceinline__ unsigned long long gnow() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <typename V, int UNROLL>
__global__ void __launch_bounds__(512) kvf_copy_vec_kernel(const __grid_constant__ CopyParams p) {
    const bool stamp = p.stamps && threadIdx.x == 0 && blockIdx.x < kvf_impl::kStampCtas;
    if (stamp) p.stamps[2 * blockIdx.x] = gnow();
    for (uint64_t t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        uint32_t plane = 0;
        const TileRef r = locate(p, t, &plane);
        const V* s = reinterpret_cast<const V*>(r.s);
        V* d = reinterpret_cast<V*>(r.d);
        const uint32_t nvec = r.len / sizeof(V);
        for (uint32_t base = threadIdx.x; base < nvec; base += blockDim.x * UNROLL) {
            V v[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint32_t i = base + u * blockDim.x;
                if (i < nvec) v[u] = ld_stream(s + i);
            }
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint32_t i = base + u * blockDim.x;
                if (i < nvec) st_stream(d + i, v[u]);
            }
        }
        if (p.layer_ready) {  // publish: this tile of layer plane/2 has landed
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) atomicAdd(p.layer_ready + plane / 2, 1u);
        }
    }
    if (p.stamps && blockIdx.x < kvf_impl::kStampCtas) {
        // a store to mapped host memory is posted: the CTA's last store instruction is not the
        // bytes' arrival.  Every thread fences its own stores system-wide first, so the end
        // stamp means "landed" for D2H as the stop event does (free for H2D: HBM stores)
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) p.stamps[2 * blockIdx.x + 1] = gnow();
    }
}

// Consumer side of the layer-pipelined load: hold the compute stream until layer `l` has
// all its tiles (cf. the reference's overlap_fraction gate, proj/src/scheduler.cpp:281).
__global__ void kvf_wait_layer_kernel(const uint32_t* ready, uint32_t l, uint32_t target) {
    if (threadIdx.x != 0) return;
    while (atomicAdd(const_cast<uint32_t*>(ready) + l, 0u) < target) __nanosleep(256);
    __threadfence();
}

// Prefill emulation for measurements: occupy `ctas` SMs for `ns` nanoseconds.
__global__ void kvf_spin_kernel(uint64_t ns) {
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        __nanosleep(100);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}

// ---- K1/K2 bulk path: the TMA bulk-copy engine moves CHUNK-byte pieces global->smem
// (mbarrier complete_tx) and smem->global (bulk_group), one elected thread per CTA driving
// a STAGES-deep ring, so the SM issues a handful of instructions per 16 KiB.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct ChunkIter {
    uint64_t t;
    uint32_t off;
    TileRef cur;
    bool valid;
};

__device__ __forceinline__ void iter_begin(const CopyParams& p, ChunkIter& it) {
    it.t = blockIdx.x;
    it.off = 0;
    it.valid = it.t < p.total_tiles;
    if (it.valid) it.cur = locate(p, it.t);
}
__device__ __forceinline__ void iter_next(const CopyParams& p, ChunkIter& it, uint32_t chunk) {
    it.off += chunk;
    if (it.off >= it.cur.len) {
        it.t += gridDim.x;
        it.off = 0;
        it.valid = it.t < p.total_tiles;
        if (it.valid) it.cur = locate(p, it.t);
    }
}

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(32) kvf_copy_bulk_kernel(const __grid_constant__ CopyParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar[STAGES];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < STAGES; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");

    ChunkIter ld, st;
    iter_begin(p, ld);
    iter_begin(p, st);
    uint32_t issued = 0;
    auto issue_load = [&](uint32_t k) {
        const uint32_t s = k % STAGES;
        const uint32_t bytes = (ld.cur.len - ld.off < (uint32_t)CHUNK ? ld.cur.len - ld.off : (uint32_t)CHUNK);
        const uint32_t b = smem_u32(&bar[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(smem + s * CHUNK)),
            "l"(ld.cur.s + ld.off), "r"(bytes), "r"(b)
            : "memory");
        iter_next(p, ld, CHUNK);
    };
    while (ld.valid && issued < STAGES) issue_load(issued++);
    for (uint32_t k = 0; st.valid; ++k) {
        const uint32_t s = k % STAGES;
        const uint32_t parity = (k / STAGES) & 1;
        const uint32_t b = smem_u32(&bar[s]);
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                : "=r"(done)
                : "r"(b), "r"(parity)
                : "memory");
        }
        const uint32_t bytes = (st.cur.len - st.off < (uint32_t)CHUNK ? st.cur.len - st.off : (uint32_t)CHUNK);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(st.cur.d + st.off),
                     "r"(smem_u32(smem + s * CHUNK)), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        iter_next(p, st, CHUNK);
        if (ld.valid) {
            // stage s is reused by the next load: its store must have finished reading smem
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            issue_load(issued++);
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

constexpr int kBulkStages = 8;
constexpr int kBulkChunk = 16384;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

// Prefill emulation: the bf16 payload of token k is a pure function of its content id
// (prefix hash), plane and global head.  One thread per 8-B word.
__global__ void kvf_fill_kernel(char* pool, uint64_t plane_stride, uint32_t tpb, uint32_t planes, uint32_t wph,
                                uint32_t head_offset, const uint64_t* __restrict__ slots,
                                const uint64_t* __restrict__ cids, uint64_t ntok) {
    const uint32_t wpt = tpb / 8;
    const uint64_t total = static_cast<uint64_t>(planes) * ntok * wpt;
    for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < total;
         w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t per_plane = ntok * wpt;
        const uint32_t plane = static_cast<uint32_t>(w / per_plane);
        const uint64_t r = w - plane * per_plane;
        const uint64_t k = r / wpt;
        const uint32_t j = static_cast<uint32_t>(r - k * wpt);
        const uint32_t h = j / wph, wi = j - h * wph;
        const uint64_t base =
            mix64(cids[k] ^ (static_cast<uint64_t>(plane) * 0x100000001b3ULL) ^ (static_cast<uint64_t>(head_offset + h) << 48));
        const uint64_t val = mix64(base + wi) & 0xBFFFBFFFBFFFBFFFULL;
        *reinterpret_cast<uint64_t*>(pool + plane * plane_stride + slots[k] * tpb + j * 8ull) = val;
    }
}

__global__ void kvf_checksum_kernel(const char* pool, uint64_t plane_stride, uint32_t tpb, uint32_t planes,
                                    const uint64_t* __restrict__ slots, uint64_t ntok, unsigned long long* out) {
    const uint32_t wpt = tpb / 8;
    const uint64_t total = static_cast<uint64_t>(planes) * ntok * wpt;
    uint64_t acc = 0;
    for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < total;
         w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t per_plane = ntok * wpt;
        const uint32_t plane = static_cast<uint32_t>(w / per_plane);
        const uint64_t r = w - plane * per_plane;
        const uint64_t k = r / wpt;
        const uint32_t j = static_cast<uint32_t>(r - k * wpt);
        const uint64_t word = *reinterpret_cast<const uint64_t*>(pool + plane * plane_stride + slots[k] * tpb + j * 8ull);
        acc += mix64(word ^ (w * 0x9e3779b97f4a7c15ULL));
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, static_cast<unsigned long long>(acc));
}

__global__ void kvf_payload_checksum_kernel(uint32_t tpb, uint32_t planes, uint32_t wph, uint32_t head_offset,
                                            const uint64_t* __restrict__ cids, uint64_t ntok,
                                            unsigned long long* out) {
    const uint32_t wpt = tpb / 8;
    const uint64_t total = static_cast<uint64_t>(planes) * ntok * wpt;
    uint64_t acc = 0;
    for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < total;
         w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t per_plane = ntok * wpt;
        const uint32_t plane = static_cast<uint32_t>(w / per_plane);
        const uint64_t r = w - plane * per_plane;
        const uint64_t k = r / wpt;
        const uint32_t j = static_cast<uint32_t>(r - k * wpt);
        const uint32_t h = j / wph, wi = j - h * wph;
        const uint64_t base =
            mix64(cids[k] ^ (static_cast<uint64_t>(plane) * 0x100000001b3ULL) ^ (static_cast<uint64_t>(head_offset + h) << 48));
        const uint64_t word = mix64(base + wi) & 0xBFFFBFFFBFFFBFFFULL;
        acc += mix64(word ^ (w * 0x9e3779b97f4a7c15ULL));
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, static_cast<unsigned long long>(acc));
}

}  // namespace

// =====================================================================================
// engine internals
// =====================================================================================
namespace {

char* tier_base(kvf_engine* e, int tier) { return tier == KVF_TIER_DEVICE ? e->dev_pool : e->host_pool_dev; }
uint64_t tier_slots(const kvf_engine* e, int tier) { return tier == KVF_TIER_DEVICE ? e->dev_slots : e->host_slots; }

bool runs_valid(const kvf_engine* e, int tier, const kvf_run* runs, uint32_t n, uint64_t* total) {
    uint64_t cap = tier_slots(e, tier), t = 0;
    for (uint32_t i = 0; i < n; ++i) {
        if (runs[i].start + runs[i].len > cap || runs[i].start + runs[i].len < runs[i].start) return false;
        t += runs[i].len;
    }
    *total = t;
    return true;
}

struct Endpoint {
    const char* base;
    uint64_t stride;  // bytes between planes
    bool host;
};

// Launch the copy of `pieces` (all planes) between two pools on `stream`.
int launch_copy(kvf_engine* e, cudaStream_t stream, const Endpoint& src, const Endpoint& dst,
                const std::vector<Piece>& pieces, uint32_t mode, uint32_t ctas, uint32_t* layer_ready = nullptr,
                uint64_t* tiles_per_layer = nullptr, uint32_t planes = 0, Job* stamped = nullptr) {
    if (planes == 0) planes = e->planes;  // default: every plane of the token (a whole node)
    if (layer_ready) mode = KVF_COPY_SM_VEC;  // only the vector kernel publishes per-layer progress
    const uint64_t tpb = e->tpb;
    for (size_t first = 0; first < pieces.size(); first += kMaxPieces) {
        const uint32_t np = static_cast<uint32_t>(std::min<size_t>(kMaxPieces, pieces.size() - first));
        if (mode == KVF_COPY_CE) {
            for (uint32_t i = 0; i < np; ++i) {
                const Piece& pc = pieces[first + i];
                KVF_CUDA(cudaMemcpy2DAsync(const_cast<char*>(dst.base) + pc.dst_slot * tpb, dst.stride,
                                           src.base + pc.src_slot * tpb, src.stride, pc.ntok * tpb, planes,
                                           cudaMemcpyDefault, stream));
            }
            continue;
        }
        CopyParams p;
        std::memset(&p, 0, sizeof(p));
        p.src = src.base;
        p.dst = const_cast<char*>(dst.base);
        p.src_stride = src.stride;
        p.dst_stride = dst.stride;
        p.planes = planes;
        p.npieces = np;
        const bool vec16 = (tpb % 16) == 0;
        // PCIe jobs keep ~the link's bandwidth-delay product in flight (8 CTAs x 256 thr x 4 x
        // 16 B = 128 KiB): full H2D rate, and 7x lower queueing for concurrent small H2D
        // traffic such as decision inputs (profiles/r01_probe_inflight.txt).  HBM jobs go wide.
        const bool pcie = src.host || dst.host;
        const uint32_t threads = pcie ? 256 : 512, unroll = pcie ? 4 : 8;
        // a tile is several unrolled batches so the per-tile lookup is amortised: PCIe tiles
        // 64 KiB (4 batches of 256 x 4 x 16 B), HBM tiles 64 KiB (one batch of 512 x 8 x 16 B)
        p.tile_bytes = threads * unroll * (vec16 ? 16 : 8) * (pcie ? 4 : 1);
        uint64_t tiles = 0;
        const uint64_t per_piece_planes = layer_ready ? 1 : planes;
        for (uint32_t i = 0; i < np; ++i) {
            const Piece& pc = pieces[first + i];
            p.src_off[i] = pc.src_slot * tpb;
            p.dst_off[i] = pc.dst_slot * tpb;
            p.seg[i] = pc.ntok * tpb;
            p.tile_begin[i] = tiles;
            tiles += per_piece_planes * ((p.seg[i] + p.tile_bytes - 1) / p.tile_bytes);
        }
        p.tile_begin[np] = tiles;
        if (layer_ready) {  // plane-outermost order + per-layer counters
            p.layer_major = 1;
            p.plane_tiles = tiles;
            p.layer_ready = layer_ready;
            if (tiles_per_layer) *tiles_per_layer += 2 * tiles;
            tiles *= planes;
        }
        p.total_tiles = tiles;
        if (tiles == 0) continue;
        uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(ctas, tiles));
        if (stamped && stamped->stamp_slot >= 0) {
            p.stamps = e->stamps_d + static_cast<size_t>(stamped->stamp_slot) * kStampCtas * 2;
            stamped->stamp_ctas = std::min<uint32_t>(grid, kStampCtas);
        }
        if (mode == KVF_COPY_SM_BULK && vec16) {
            const size_t smem = static_cast<size_t>(kBulkStages) * kBulkChunk;
            if (!e->bulk_attr_set) {  // per engine: attributes are per device
                KVF_CUDA(cudaFuncSetAttribute(kvf_copy_bulk_kernel<kBulkStages, kBulkChunk>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                e->bulk_attr_set = true;
            }
            kvf_copy_bulk_kernel<kBulkStages, kBulkChunk><<<grid, 32, smem, stream>>>(p);
        } else if (vec16) {
            if (pcie) kvf_copy_vec_kernel<uint4, 4><<<grid, threads, 0, stream>>>(p);
            else kvf_copy_vec_kernel<uint4, 8><<<grid, threads, 0, stream>>>(p);
        } else {
            kvf_copy_vec_kernel<uint2, 8><<<grid, threads, 0, stream>>>(p);
        }
        KVF_CUDA(cudaGetLastError());
        e->stats.kernel_launches++;
    }
    return KVF_OK;
}

int transfer(kvf_engine* e, uint64_t job_id, int src_tier, const kvf_run* src_runs, uint32_t n_src, int dst_tier,
             const kvf_run* dst_runs, uint32_t n_dst) {
    uint64_t ts = 0, td = 0;
    if ((n_src && !src_runs) || (n_dst && !dst_runs)) return set_error(KVF_E_INVALID_ARG, "null run list");
    if (!runs_valid(e, src_tier, src_runs, n_src, &ts) || !runs_valid(e, dst_tier, dst_runs, n_dst, &td))
        return set_error(KVF_E_INVALID_ARG, "run out of pool range");
    if (ts != td) return set_error(KVF_E_INVALID_ARG, "source and destination token counts differ");
    std::vector<Piece> pieces;
    merge_runs(src_runs, n_src, dst_runs, n_dst, pieces);
    const bool h2d = src_tier == KVF_TIER_HOST && dst_tier == KVF_TIER_DEVICE;
    const bool d2h = src_tier == KVF_TIER_DEVICE && dst_tier == KVF_TIER_HOST;
    cudaStream_t st = h2d ? e->s_h2d : (d2h ? e->s_d2h : e->s_dev);
    const bool pcie_job = h2d || d2h;
    const int32_t slot = pcie_job ? take_stamp_slot(e, pieces.size(), e->cfg.pcie_mode) : -1;
    Job j;
    int rc = begin_job(e, job_id, st, j, slot);
    if (rc) {
        if (slot >= 0 && e->stamp_refs[slot] == 0) e->stamp_free.push_back(slot);
        return rc;
    }
    // Order against the compute stream's last payload write (fill / K3 scatter): a D2H may
    // read those slots, an H2D may land in slots a just-discarded node's fill still targets.
    if ((d2h || h2d) && e->dev_write_pending) KVF_CUDA(cudaStreamWaitEvent(st, e->dev_write_done, 0));
    const uint64_t stride_s = tier_slots(e, src_tier) * e->tpb, stride_d = tier_slots(e, dst_tier) * e->tpb;
    Endpoint src{tier_base(e, src_tier), stride_s, src_tier == KVF_TIER_HOST};
    Endpoint dst{tier_base(e, dst_tier), stride_d, dst_tier == KVF_TIER_HOST};
    const bool pcie = h2d || d2h;
    const uint32_t mode = pcie ? e->cfg.pcie_mode : KVF_COPY_SM_VEC;
    const uint32_t ctas = pcie ? e->cfg.pcie_ctas : e->cfg.hbm_ctas;
    rc = launch_copy(e, st, src, dst, pieces, mode, ctas, nullptr, nullptr, 0, &j);
    if (rc) return rc;
    j.bytes = ts * e->token_bytes;
    if (h2d) { e->stats.h2d_bytes += j.bytes; e->stats.h2d_jobs++; }
    else if (d2h) { e->stats.d2h_bytes += j.bytes; e->stats.d2h_jobs++; }
    else { e->stats.dev_bytes += j.bytes; e->stats.dev_jobs++; }
    return end_job(e, job_id, j);
}

// K3 between the pool and a contiguous staging buffer (a 1-run pool of ntok slots).
int dev_staging_copy(kvf_engine* e, uint64_t job_id, const kvf_run* runs, uint32_t n, char* staging, bool gather) {
    uint64_t ntok = 0;
    if (!staging) return set_error(KVF_E_INVALID_ARG, "null staging buffer");
    if (!runs_valid(e, KVF_TIER_DEVICE, runs, n, &ntok)) return set_error(KVF_E_INVALID_ARG, "run out of pool range");
    kvf_run whole{0, ntok};
    std::vector<Piece> pieces;
    if (gather) merge_runs(runs, n, &whole, 1, pieces);
    else merge_runs(&whole, 1, runs, n, pieces);
    Job j;
    int rc = begin_job(e, job_id, e->s_dev, j);
    if (rc) return rc;
    Endpoint pool{e->dev_pool, e->dev_slots * e->tpb, false};
    Endpoint stage{staging, ntok * e->tpb, false};
    rc = gather ? launch_copy(e, e->s_dev, pool, stage, pieces, KVF_COPY_SM_VEC, e->cfg.hbm_ctas)
                : launch_copy(e, e->s_dev, stage, pool, pieces, KVF_COPY_SM_VEC, e->cfg.hbm_ctas);
    if (rc) return rc;
    if (!gather) {
        KVF_CUDA(cudaEventRecord(e->dev_write_done, e->s_dev));
        e->dev_write_pending = true;
    }
    j.bytes = ntok * e->token_bytes;
    e->stats.dev_bytes += j.bytes;
    e->stats.dev_jobs++;
    return end_job(e, job_id, j);
}

// Upload (slot, cid) per token into the dev workspace; returns device pointers.
int stage_slots(kvf_engine* e, const kvf_run* runs, uint32_t n, const uint64_t* cids, uint64_t ntok,
                uint64_t** d_slots, uint64_t** d_cids) {
    const size_t bytes = ntok * sizeof(uint64_t) * (cids ? 2 : 1);
    // the dev workspace may still be read by an in-flight fill: drain s_dev first
    KVF_CUDA(cudaStreamSynchronize(e->s_dev));
    int rc = e->ws_dev.ensure(bytes + 64, bytes + 64);
    if (rc) return rc;
    uint64_t* h = static_cast<uint64_t*>(e->ws_dev.host);
    uint64_t k = 0;
    for (uint32_t r = 0; r < n; ++r)
        for (uint64_t t = 0; t < runs[r].len; ++t) h[k++] = runs[r].start + t;
    if (cids) std::memcpy(h + ntok, cids, ntok * sizeof(uint64_t));
    KVF_CUDA(cudaMemcpyAsync(e->ws_dev.dev, h, bytes, cudaMemcpyHostToDevice, e->s_dev));
    *d_slots = static_cast<uint64_t*>(e->ws_dev.dev);
    if (d_cids) *d_cids = cids ? static_cast<uint64_t*>(e->ws_dev.dev) + ntok : nullptr;
    return KVF_OK;
}

uint32_t grid_for(const kvf_engine* e, uint64_t work, uint32_t threads) {
    uint64_t g = (work + threads - 1) / threads;
    return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(g, static_cast<uint64_t>(e->sm_count) * 8)));
}

// Short-lived CTAs (~per_thread items each) for bulk work that runs while decisions must
// start promptly: a grid-stride grid of sm_count x 8 resident CTAs holds every SM's thread
// slots for the whole kernel (a 1 GiB prompt fill: ~0.65 ms), so a K4/K5 CTA on the
// high-priority decision stream waited for the fill to END (measured: 665 us late starts,
// scripts/decision_trace.py).  With CTAs of a few us the block scheduler hands the next free
// slot to the decision CTA.
uint32_t grid_short(uint64_t work, uint32_t threads, uint32_t per_thread) {
    const uint64_t g = (work + static_cast<uint64_t>(threads) * per_thread - 1) / (static_cast<uint64_t>(threads) * per_thread);
    return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(g, 0x7fffffffull)));
}

void set_carveout_engine() {
    const int v = cudaSharedmemCarveoutMaxShared;
    const cudaFuncAttribute a = cudaFuncAttributePreferredSharedMemoryCarveout;
    cudaFuncSetAttribute(kvf_copy_vec_kernel<uint4, 4>, a, v);
    cudaFuncSetAttribute(kvf_copy_vec_kernel<uint4, 8>, a, v);
    cudaFuncSetAttribute(kvf_copy_vec_kernel<uint2, 8>, a, v);
    cudaFuncSetAttribute(kvf_copy_bulk_kernel<kBulkStages, kBulkChunk>, a, v);
    cudaFuncSetAttribute(kvf_wait_layer_kernel, a, v);
    cudaFuncSetAttribute(kvf_spin_kernel, a, v);
    cudaFuncSetAttribute(kvf_fill_kernel, a, v);
    cudaFuncSetAttribute(kvf_checksum_kernel, a, v);
    cudaFuncSetAttribute(kvf_payload_checksum_kernel, a, v);
}

}  // namespace

// =====================================================================================
// C-ABI
// =====================================================================================
extern "C" {

const char* kvf_last_error(void) { return g_last_error.c_str(); }
const char* kvf_version(void) { return "kvflow-b200 0.1 (sm_100a)"; }

int kvf_device_count(int32_t* out) {
    int n = 0;
    cudaError_t err = cudaGetDeviceCount(&n);
    if (err != cudaSuccess) n = 0;
    if (out) *out = n;
    return KVF_OK;
}

int kvf_device_numa_node(int32_t device, int32_t* node) {
    if (!node) return set_error(KVF_E_INVALID_ARG, "null node");
    *node = -1;
    char bus[32] = {0};
    const cudaError_t err = cudaDeviceGetPCIBusId(bus, sizeof(bus), device);
    if (err != cudaSuccess) return err == cudaErrorNoDevice || err == cudaErrorInvalidDevice
                                       ? set_error(KVF_E_NO_DEVICE, "no CUDA device")
                                       : cuda_error(err, "cudaDeviceGetPCIBusId");
    for (char* c = bus; *c; ++c) *c = static_cast<char>(std::tolower(static_cast<unsigned char>(*c)));
    const std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
    FILE* f = std::fopen(path.c_str(), "r");
    if (!f) return KVF_OK;  // unknown: -1
    int v = -1;
    if (std::fscanf(f, "%d", &v) != 1) v = -1;
    std::fclose(f);
    *node = v;
    return KVF_OK;
}

int kvf_engine_create(const kvf_geometry* g, const kvf_engine_config* cfg, kvf_engine** out) {
    if (!g || !cfg || !out) return set_error(KVF_E_INVALID_ARG, "null argument");
    *out = nullptr;
    if (g->layers == 0 || g->kv_heads_local == 0 || g->head_dim == 0 || g->dtype_bytes != 2 ||
        g->head_offset + g->kv_heads_local > g->kv_heads_total)
        return set_error(KVF_E_CONFIG, "invalid geometry (bf16 only; heads within total)");
    if ((static_cast<uint64_t>(g->kv_heads_local) * g->head_dim * g->dtype_bytes) % 8 != 0)
        return set_error(KVF_E_CONFIG, "bytes per token per plane must be a multiple of 8");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return set_error(KVF_E_NO_DEVICE, "no CUDA device: kvflow has no CPU fallback");
    if (cfg->device < 0 || cfg->device >= ndev) return set_error(KVF_E_INVALID_ARG, "device ordinal out of range");
    auto* e = new kvf_engine();
    e->geom = *g;
    e->cfg = *cfg;
    e->device = cfg->device;
    e->tpb = static_cast<uint64_t>(g->kv_heads_local) * g->head_dim * g->dtype_bytes;
    e->planes = g->layers * 2;
    e->token_bytes = e->tpb * e->planes;
    auto fail = [&](int rc) {
        kvf_engine_destroy(e);
        return rc;
    };
    if (cudaSetDevice(e->device) != cudaSuccess) return fail(set_error(KVF_E_CUDA, "cudaSetDevice"));
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, e->device) == cudaSuccess) e->sm_count = prop.multiProcessorCount;
    if (e->cfg.pcie_ctas == 0) e->cfg.pcie_ctas = 8;
    if (e->cfg.hbm_ctas == 0) e->cfg.hbm_ctas = static_cast<uint32_t>(e->sm_count) * 4;
    cudaError_t err;
    e->dev_slots = cfg->gpu_slots;
    e->host_slots = cfg->host_slots;
    if (e->dev_slots) {
        err = cudaMalloc(reinterpret_cast<void**>(&e->dev_pool), e->dev_slots * e->token_bytes);
        if (err != cudaSuccess) return fail(cuda_error(err, "cudaMalloc(device KV pool)"));
    }
    if (e->host_slots) {
        const size_t bytes = e->host_slots * e->token_bytes;
        int32_t numa = cfg->host_numa_node;
        if (numa == KVF_NUMA_AUTO && kvf_device_numa_node(e->device, &numa) != KVF_OK) numa = -1;
        if (numa >= 0) {
            // NUMA-local pinned shard: mmap, bind to the GPU's node, then pin + map.
            void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
            if (p == MAP_FAILED) return fail(set_error(KVF_E_OUT_OF_HOST_SLOTS, "mmap host pool"));
            unsigned long mask[16] = {0};
            const int node = numa;
            e->host_numa = numa;
            if (node < 1024) mask[node / 64] |= 1ul << (node % 64);
            syscall(SYS_mbind, p, bytes, 2 /*MPOL_BIND*/, mask, 1024ul, 0u);  // best effort
            e->host_pool = static_cast<char*>(p);
            e->host_map_bytes = bytes;
            err = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
            if (err != cudaSuccess) return fail(cuda_error(err, "cudaHostRegister(host KV pool)"));
            e->host_registered = true;
        } else {
            err = cudaHostAlloc(reinterpret_cast<void**>(&e->host_pool), bytes, cudaHostAllocMapped | cudaHostAllocPortable);
            if (err != cudaSuccess) return fail(cuda_error(err, "cudaHostAlloc(host KV pool)"));
        }
        void* dp = nullptr;
        err = cudaHostGetDevicePointer(&dp, e->host_pool, 0);
        if (err != cudaSuccess) return fail(cuda_error(err, "cudaHostGetDevicePointer"));
        e->host_pool_dev = static_cast<char*>(dp);
    }
    e->alloc[KVF_TIER_DEVICE].reset(e->dev_slots);
    e->alloc[KVF_TIER_HOST].reset(e->host_slots);
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if ((err = cudaStreamCreateWithFlags(&e->s_h2d, cudaStreamNonBlocking)) != cudaSuccess ||
        (err = cudaStreamCreateWithFlags(&e->s_d2h, cudaStreamNonBlocking)) != cudaSuccess ||
        (err = cudaStreamCreateWithFlags(&e->s_dev, cudaStreamNonBlocking)) != cudaSuccess ||
        (err = cudaStreamCreateWithFlags(&e->s_cmp, cudaStreamNonBlocking)) != cudaSuccess ||
        (err = cudaStreamCreateWithPriority(&e->s_dec, cudaStreamNonBlocking, hi)) != cudaSuccess)
        return fail(cuda_error(err, "cudaStreamCreate"));
    if ((err = cudaEventCreateWithFlags(&e->dev_write_done, cudaEventDisableTiming)) != cudaSuccess ||
        (err = cudaEventCreate(&e->dec_start)) != cudaSuccess || (err = cudaEventCreate(&e->dec_stop)) != cudaSuccess ||
        (err = cudaEventCreateWithFlags(&e->att_upload_done, cudaEventDisableTiming)) != cudaSuccess)
        return fail(cuda_error(err, "cudaEventCreate"));
    if ((err = cudaMalloc(reinterpret_cast<void**>(&e->d_checksum), sizeof(uint64_t))) != cudaSuccess)
        return fail(cuda_error(err, "cudaMalloc(checksum)"));
    const size_t ctr_bytes = static_cast<size_t>(kvf_impl::kLayerSlots) * e->geom.layers * sizeof(uint32_t);
    if ((err = cudaMalloc(reinterpret_cast<void**>(&e->d_layer_ctr), ctr_bytes)) != cudaSuccess ||
        (err = cudaMemset(e->d_layer_ctr, 0, ctr_bytes)) != cudaSuccess)
        return fail(cuda_error(err, "cudaMalloc(layer counters)"));
    e->lr_total.assign(kvf_impl::kLayerSlots, 0);
    for (int32_t k = static_cast<int32_t>(kvf_impl::kLayerSlots) - 1; k >= 0; --k) e->lr_free.push_back(k);
    // Size the staging workspaces once: growing them later means cudaFree (a device-wide
    // sync) and cudaHostAlloc inside a decision call -- milliseconds on the hot path.
    static std::once_flag carveout_once;  // attributes are per function (all devices alike here)
    std::call_once(carveout_once, [] {
        set_carveout_engine();
        kvf_impl::set_carveout_decide();
        kvf_impl::set_carveout_attend();
        kvf_impl::set_carveout_mirror();
    });
    cudaGetLastError();  // an attribute a driver rejects is a hint, not an error
    for (kvf_impl::Workspace* w : {&e->ws_dev, &e->ws_dec, &e->ws_att, &e->ws_big, &e->large_snap.ws}) w->owner = e;
    if (int rc = kvf_impl::decider_init(e)) return fail(rc);
    {
        void* h = nullptr;
        const size_t sb = static_cast<size_t>(kvf_impl::kStampSlots) * kvf_impl::kStampCtas * 2 * sizeof(unsigned long long);
        if ((err = cudaHostAlloc(&h, sb, cudaHostAllocMapped | cudaHostAllocPortable)) != cudaSuccess)
            return fail(cuda_error(err, "cudaHostAlloc(stamps)"));
        void* dp = nullptr;
        if ((err = cudaHostGetDevicePointer(&dp, h, 0)) != cudaSuccess) return fail(cuda_error(err, "stamps device pointer"));
        e->stamps_h = static_cast<unsigned long long*>(h);
        e->stamps_d = static_cast<unsigned long long*>(dp);
        e->stamp_refs.assign(kvf_impl::kStampSlots, 0);
        for (int32_t k = static_cast<int32_t>(kvf_impl::kStampSlots) - 1; k >= 0; --k) e->stamp_free.push_back(k);
        const char* st = std::getenv("KVF_JOB_TIMING");
        e->stamp_timing = st && std::string(st) == "stamps";
    }
    if (int rc = e->ws_dec.ensure(1u << 20, 1u << 20)) return fail(rc);
    if (int rc = e->ws_dev.ensure(4u << 20, 4u << 20)) return fail(rc);
    *out = e;
    return KVF_OK;
}

int kvf_engine_destroy(kvf_engine* e) {
    if (!e) return KVF_OK;
    cudaSetDevice(e->device);
    kvf_impl::decider_release(e);  // stops the resident CTA (else the sync below waits for its idle-out)
    cudaDeviceSynchronize();
    for (auto& [id, j] : e->jobs) {
        cudaEventDestroy(j.start);
        cudaEventDestroy(j.stop);
    }
    for (cudaEvent_t ev : e->event_pool) cudaEventDestroy(ev);
    for (cudaEvent_t ev : e->event_pool_nt) cudaEventDestroy(ev);
    if (e->stamps_h) cudaFreeHost(e->stamps_h);
    for (cudaEvent_t ev : {e->dev_write_done, e->dec_start, e->dec_stop, e->att_upload_done})
        if (ev) cudaEventDestroy(ev);
    for (cudaStream_t s : {e->s_h2d, e->s_d2h, e->s_dev, e->s_dec, e->s_cmp})
        if (s) cudaStreamDestroy(s);
    e->ws_dev.release();
    e->ws_dec.release();
    e->ws_att.release();
    kvf_impl::large_release(e->large_snap);
    e->ws_big.release();
    if (e->d_checksum) cudaFree(e->d_checksum);
    if (e->d_layer_ctr) cudaFree(e->d_layer_ctr);
    if (e->dev_pool) cudaFree(e->dev_pool);
    if (e->host_pool) {
        if (e->host_registered) {
            cudaHostUnregister(e->host_pool);
            munmap(e->host_pool, e->host_map_bytes);
        } else {
            cudaFreeHost(e->host_pool);
        }
    }
    delete e;
    return KVF_OK;
}

int kvf_engine_token_bytes(const kvf_engine* e, uint64_t* tpb, uint64_t* token_bytes) {
    if (!e) return set_error(KVF_E_INVALID_ARG, "null engine");
    if (tpb) *tpb = e->tpb;
    if (token_bytes) *token_bytes = e->token_bytes;
    return KVF_OK;
}

int kvf_engine_set_job_timing(kvf_engine* e, uint32_t mode) {
    KVF_GUARD(e);
    if (mode > KVF_JOB_TIMING_STAMPS) return set_error(KVF_E_INVALID_ARG, "unknown job timing mode");
    e->stamp_timing = mode == KVF_JOB_TIMING_STAMPS;
    return KVF_OK;
}

int kvf_engine_set_copy_mode(kvf_engine* e, uint32_t mode, uint32_t pcie_ctas, uint32_t hbm_ctas) {
    KVF_GUARD(e);
    if (mode > KVF_COPY_CE) return set_error(KVF_E_INVALID_ARG, "unknown copy mode");
    e->cfg.pcie_mode = mode;
    if (pcie_ctas) e->cfg.pcie_ctas = pcie_ctas;
    if (hbm_ctas) e->cfg.hbm_ctas = hbm_ctas;
    return KVF_OK;
}

int kvf_slots_alloc(kvf_engine* e, int32_t tier, uint64_t tokens, kvf_run* out, uint32_t max_runs, uint32_t* n_runs) {
    if (!e || !out || !n_runs || (tier != 0 && tier != 1)) return set_error(KVF_E_INVALID_ARG, "bad argument");
    std::lock_guard<std::mutex> lk(e->mu);
    std::vector<kvf_run> runs;
    if (!e->alloc[tier].alloc(tokens, runs))
        return set_error(tier == KVF_TIER_DEVICE ? KVF_E_OUT_OF_GPU_MEMORY : KVF_E_OUT_OF_HOST_SLOTS,
                         "slot pool exhausted: want " + std::to_string(tokens) + " tokens, free " +
                             std::to_string(e->alloc[tier].free_tokens()));
    if (runs.size() > max_runs) {
        for (const kvf_run& r : runs) e->alloc[tier].release(r);
        return set_error(KVF_E_TOO_LARGE, "allocation needs " + std::to_string(runs.size()) + " runs > max_runs");
    }
    std::copy(runs.begin(), runs.end(), out);
    *n_runs = static_cast<uint32_t>(runs.size());
    return KVF_OK;
}

int kvf_slots_free(kvf_engine* e, int32_t tier, const kvf_run* runs, uint32_t n) {
    if (!e || (n && !runs) || (tier != 0 && tier != 1)) return set_error(KVF_E_INVALID_ARG, "bad argument");
    std::lock_guard<std::mutex> lk(e->mu);
    for (uint32_t i = 0; i < n; ++i)
        if (!e->alloc[tier].release(runs[i]))
            return set_error(KVF_E_INTERNAL, "slot free of an unallocated or out-of-range run");
    return KVF_OK;
}

int kvf_slots_free_count(const kvf_engine* e, int32_t tier, uint64_t* free_tokens, uint64_t* free_runs) {
    if (!e || (tier != 0 && tier != 1)) return set_error(KVF_E_INVALID_ARG, "bad argument");
    if (free_tokens) *free_tokens = e->alloc[tier].free_tokens();
    if (free_runs) *free_runs = e->alloc[tier].free_runs();
    return KVF_OK;
}

int kvf_pool_ptr(const kvf_engine* e, int32_t tier, void** base, uint64_t* slots) {
    if (!e || (tier != 0 && tier != 1)) return set_error(KVF_E_INVALID_ARG, "bad argument");
    if (base) *base = tier == KVF_TIER_DEVICE ? static_cast<void*>(e->dev_pool) : static_cast<void*>(e->host_pool);
    if (slots) *slots = tier == KVF_TIER_DEVICE ? e->dev_slots : e->host_slots;
    return KVF_OK;
}

int kvf_h2d_gather(kvf_engine* e, uint64_t job_id, const kvf_run* host_runs, uint32_t n_host, const kvf_run* dev_runs,
                   uint32_t n_dev) {
    KVF_GUARD(e);
    return transfer(e, job_id, KVF_TIER_HOST, host_runs, n_host, KVF_TIER_DEVICE, dev_runs, n_dev);
}

int kvf_d2h_scatter(kvf_engine* e, uint64_t job_id, const kvf_run* dev_runs, uint32_t n_dev, const kvf_run* host_runs,
                    uint32_t n_host) {
    KVF_GUARD(e);
    return transfer(e, job_id, KVF_TIER_DEVICE, dev_runs, n_dev, KVF_TIER_HOST, host_runs, n_host);
}

int kvf_d2h_scatter_batch(kvf_engine* e, uint32_t n_jobs, const uint64_t* job_ids, const kvf_run* dev_runs,
                          const uint32_t* dev_counts, const kvf_run* host_runs, const uint32_t* host_counts) {
    KVF_GUARD(e);
    if (n_jobs == 0) return KVF_OK;
    if (!job_ids || !dev_counts || !host_counts) return set_error(KVF_E_INVALID_ARG, "null batch array");
    // validate everything before any job exists: a bad entry leaves no half-issued batch
    std::vector<Piece> pieces;
    std::vector<uint64_t> bytes(n_jobs);
    size_t od = 0, oh = 0;
    for (uint32_t k = 0; k < n_jobs; ++k) {
        if (e->jobs.count(job_ids[k])) return set_error(KVF_E_INVALID_ARG, "job id " + std::to_string(job_ids[k]) + " already in use");
        for (uint32_t q = 0; q < k; ++q)
            if (job_ids[q] == job_ids[k]) return set_error(KVF_E_INVALID_ARG, "duplicate job id in batch");
        const kvf_run* dr = dev_runs + od;
        const kvf_run* hr = host_runs + oh;
        if ((dev_counts[k] && !dev_runs) || (host_counts[k] && !host_runs)) return set_error(KVF_E_INVALID_ARG, "null run list");
        uint64_t td = 0, th = 0;
        if (!runs_valid(e, KVF_TIER_DEVICE, dr, dev_counts[k], &td) || !runs_valid(e, KVF_TIER_HOST, hr, host_counts[k], &th))
            return set_error(KVF_E_INVALID_ARG, "run out of pool range");
        if (td != th) return set_error(KVF_E_INVALID_ARG, "source and destination token counts differ");
        std::vector<Piece> mine;
        merge_runs(dr, dev_counts[k], hr, host_counts[k], mine);
        pieces.insert(pieces.end(), mine.begin(), mine.end());
        bytes[k] = td * e->token_bytes;
        od += dev_counts[k];
        oh += host_counts[k];
    }
    std::vector<Job> js(n_jobs);
    const int32_t slot = take_stamp_slot(e, pieces.size(), e->cfg.pcie_mode);  // shared by the batch
    for (uint32_t k = 0; k < n_jobs; ++k) {
        int rc = begin_job(e, job_ids[k], e->s_d2h, js[k], slot);
        if (rc) return rc;
    }
    if (e->dev_write_pending) KVF_CUDA(cudaStreamWaitEvent(e->s_d2h, e->dev_write_done, 0));
    Endpoint src{e->dev_pool, e->dev_slots * e->tpb, false};
    Endpoint dst{e->host_pool_dev, e->host_slots * e->tpb, true};
    int rc = launch_copy(e, e->s_d2h, src, dst, pieces, e->cfg.pcie_mode, e->cfg.pcie_ctas, nullptr, nullptr, 0,
                         &js[0]);  // one K2 for all
    if (rc) return rc;
    for (uint32_t k = 0; k < n_jobs; ++k) {
        js[k].stamp_ctas = js[0].stamp_ctas;
        js[k].bytes = bytes[k];
        e->stats.d2h_bytes += bytes[k];
        e->stats.d2h_jobs++;
        rc = end_job(e, job_ids[k], js[k]);
        if (rc) return rc;
    }
    return KVF_OK;
}

int kvf_h2d_gather_layered(kvf_engine* e, uint64_t job_id, const kvf_run* host_runs, uint32_t n_host,
                           const kvf_run* dev_runs, uint32_t n_dev, uint32_t* layer_ready, uint32_t* tiles_per_layer) {
    KVF_GUARD(e);
    const bool owned = layer_ready == nullptr;  // engine-owned counters (kvf_compute_wait_job_layer)
    if (owned && e->lr_free.empty()) return set_error(KVF_E_TOO_LARGE, "all layered-load counter slots in flight");
    uint64_t ts = 0, td = 0;
    if (!runs_valid(e, KVF_TIER_HOST, host_runs, n_host, &ts) || !runs_valid(e, KVF_TIER_DEVICE, dev_runs, n_dev, &td))
        return set_error(KVF_E_INVALID_ARG, "run out of pool range");
    if (ts != td) return set_error(KVF_E_INVALID_ARG, "source and destination token counts differ");
    std::vector<Piece> pieces;
    merge_runs(host_runs, n_host, dev_runs, n_dev, pieces);
    Job j;
    const int32_t slot = take_stamp_slot(e, pieces.size(), KVF_COPY_SM_VEC);
    int rc = begin_job(e, job_id, e->s_h2d, j, slot);
    if (rc) return rc;
    if (e->dev_write_pending) KVF_CUDA(cudaStreamWaitEvent(e->s_h2d, e->dev_write_done, 0));
    if (owned) {  // counters only grow: no reset, so a late waiter on a recycled slot never hangs
        j.lr_slot = e->lr_free.back();
        e->lr_free.pop_back();
        layer_ready = e->d_layer_ctr + static_cast<size_t>(j.lr_slot) * e->geom.layers;
    } else {
        KVF_CUDA(cudaMemsetAsync(layer_ready, 0, e->geom.layers * sizeof(uint32_t), e->s_h2d));
    }
    Endpoint src{e->host_pool_dev, e->host_slots * e->tpb, true};
    Endpoint dst{e->dev_pool, e->dev_slots * e->tpb, false};
    uint64_t per_layer = 0;
    rc = launch_copy(e, e->s_h2d, src, dst, pieces, KVF_COPY_SM_VEC, e->cfg.pcie_ctas, layer_ready, &per_layer, 0, &j);
    if (rc) {
        if (owned) e->lr_free.push_back(j.lr_slot);
        return rc;
    }
    if (tiles_per_layer) *tiles_per_layer = static_cast<uint32_t>(per_layer);
    if (owned) {
        j.lr_base = e->lr_total[j.lr_slot];
        j.lr_tpl = static_cast<uint32_t>(per_layer);
        e->lr_total[j.lr_slot] += j.lr_tpl;
    }
    j.bytes = ts * e->token_bytes;
    e->stats.h2d_bytes += j.bytes;
    e->stats.h2d_jobs++;
    return end_job(e, job_id, j);
}

int kvf_compute_wait_layer(kvf_engine* e, const uint32_t* layer_ready, uint32_t layer, uint32_t target) {
    KVF_GUARD(e);
    if (!layer_ready || layer >= e->geom.layers) return set_error(KVF_E_INVALID_ARG, "bad layer");
    kvf_wait_layer_kernel<<<1, 32, 0, e->s_cmp>>>(layer_ready, layer, target);
    KVF_CUDA(cudaGetLastError());
    e->stats.kernel_launches++;
    return KVF_OK;
}

int kvf_compute_spin(kvf_engine* e, uint64_t ns, uint32_t ctas) {
    KVF_GUARD(e);
    kvf_spin_kernel<<<ctas ? ctas : 1, 32, 0, e->s_cmp>>>(ns);
    KVF_CUDA(cudaGetLastError());
    e->stats.kernel_launches++;
    return KVF_OK;
}

int kvf_compute_wait_job_layer(kvf_engine* e, uint64_t job_id, uint32_t layer) {
    KVF_GUARD(e);
    auto it = e->jobs.find(job_id);
    if (it == e->jobs.end()) return set_error(KVF_E_UNKNOWN_JOB, "unknown job " + std::to_string(job_id));
    if (layer >= e->geom.layers) return set_error(KVF_E_INVALID_ARG, "bad layer");
    const kvf_impl::Job& j = it->second;
    if (j.lr_slot < 0) {  // not a layered job: the whole transfer is the dependency
        KVF_CUDA(cudaStreamWaitEvent(e->s_cmp, j.stop, 0));
        return KVF_OK;
    }
    kvf_wait_layer_kernel<<<1, 32, 0, e->s_cmp>>>(e->d_layer_ctr + static_cast<size_t>(j.lr_slot) * e->geom.layers,
                                                 layer, j.lr_base + j.lr_tpl);
    KVF_CUDA(cudaGetLastError());
    e->stats.kernel_launches++;
    return KVF_OK;
}

int kvf_compute_wait_job(kvf_engine* e, uint64_t job_id) {
    KVF_GUARD(e);
    auto it = e->jobs.find(job_id);
    if (it == e->jobs.end()) return set_error(KVF_E_UNKNOWN_JOB, "unknown job " + std::to_string(job_id));
    KVF_CUDA(cudaStreamWaitEvent(e->s_cmp, it->second.stop, 0));
    return KVF_OK;
}

int kvf_compute_job_begin(kvf_engine* e, uint64_t job_id) {
    KVF_GUARD(e);
    Job j;
    int rc = begin_job(e, job_id, e->s_cmp, j);
    if (rc) return rc;
    e->jobs.emplace(job_id, j);  // stop event recorded by kvf_compute_job_end
    return KVF_OK;
}

int kvf_compute_job_end(kvf_engine* e, uint64_t job_id) {
    KVF_GUARD(e);
    auto it = e->jobs.find(job_id);
    if (it == e->jobs.end()) return set_error(KVF_E_UNKNOWN_JOB, "unknown job " + std::to_string(job_id));
    KVF_CUDA(cudaEventRecord(it->second.stop, it->second.stream));
    return KVF_OK;
}

int kvf_dev_gather(kvf_engine* e, uint64_t job_id, const kvf_run* runs, uint32_t n, void* staging) {
    KVF_GUARD(e);
    return dev_staging_copy(e, job_id, runs, n, static_cast<char*>(staging), true);
}

int kvf_dev_scatter(kvf_engine* e, uint64_t job_id, const void* staging, const kvf_run* runs, uint32_t n) {
    KVF_GUARD(e);
    return dev_staging_copy(e, job_id, runs, n, static_cast<char*>(const_cast<void*>(staging)), false);
}

int kvf_kv_append(kvf_engine* e, uint64_t job_id, uint32_t layer, const kvf_run* runs, uint32_t n_runs, const void* k,
                  const void* v, uint64_t ntok) {
    KVF_GUARD(e);
    if (layer >= e->geom.layers) return set_error(KVF_E_INVALID_ARG, "layer out of range");
    if (ntok && (!k || !v)) return set_error(KVF_E_INVALID_ARG, "null k / v");
    uint64_t td = 0;
    if (n_runs && !runs) return set_error(KVF_E_INVALID_ARG, "null run list");
    if (!runs_valid(e, KVF_TIER_DEVICE, runs, n_runs, &td)) return set_error(KVF_E_INVALID_ARG, "run out of pool range");
    if (td != ntok) return set_error(KVF_E_INVALID_ARG, "runs and ntok disagree");
    const kvf_run whole{0, ntok};
    std::vector<Piece> pieces;
    merge_runs(&whole, 1, runs, n_runs, pieces);
    Job j;
    int rc = begin_job(e, job_id, e->s_dev, j);  // the payload-write stream: later K2 / K6 order after it
    if (rc) return rc;
    const uint64_t plane = e->dev_slots * e->tpb;
    char* kplane = e->dev_pool + static_cast<uint64_t>(2 * layer) * plane;
    for (int kv = 0; kv < 2; ++kv) {  // [ntok][heads][dim] rows -> the layer's K / V plane rows
        Endpoint from{static_cast<const char*>(kv ? v : k), ntok * e->tpb, false};
        Endpoint to{kplane + kv * plane, plane, false};
        rc = launch_copy(e, e->s_dev, from, to, pieces, KVF_COPY_SM_VEC, e->cfg.hbm_ctas, nullptr, nullptr, 1);
        if (rc) return rc;
    }
    KVF_CUDA(cudaEventRecord(e->dev_write_done, e->s_dev));
    e->dev_write_pending = true;
    j.bytes = 2 * ntok * e->tpb;
    e->stats.dev_bytes += j.bytes;
    e->stats.dev_jobs++;
    return end_job(e, job_id, j);
}

int kvf_peer_gather(kvf_engine* e, uint64_t job_id, kvf_engine* src, const kvf_run* src_runs, uint32_t n_src,
                    const kvf_run* dst_runs, uint32_t n_dst) {
    if (!e || !src) return set_error(KVF_E_INVALID_ARG, "null engine");
    // both pools are touched: hold both engines (std::lock takes the pair deadlock-free)
    std::unique_lock<std::mutex> l1(e->mu, std::defer_lock), l2(src->mu, std::defer_lock);
    if (src == e) l1.lock();
    else std::lock(l1, l2);
    if (cudaSetDevice(e->device) != cudaSuccess) return set_error(KVF_E_CUDA, "cudaSetDevice failed");
    kvf_impl::clear_stale_error(e, __func__);
    if (e->tpb != src->tpb || e->planes != src->planes || e->geom.head_offset != src->geom.head_offset)
        return set_error(KVF_E_INVALID_ARG, "peer engine holds a different KV shard geometry");
    uint64_t ts = 0, td = 0;
    if ((n_src && !src_runs) || (n_dst && !dst_runs)) return set_error(KVF_E_INVALID_ARG, "null run list");
    if (!runs_valid(src, KVF_TIER_DEVICE, src_runs, n_src, &ts) || !runs_valid(e, KVF_TIER_DEVICE, dst_runs, n_dst, &td))
        return set_error(KVF_E_INVALID_ARG, "run out of pool range");
    if (ts != td) return set_error(KVF_E_INVALID_ARG, "source and destination token counts differ");
    if (src->device != e->device) {  // NVLink / NVSwitch: the kernel on this GPU loads the peer's HBM
        int can = 0;
        KVF_CUDA(cudaDeviceCanAccessPeer(&can, e->device, src->device));
        if (!can) return set_error(KVF_E_INVALID_ARG, "no peer access between the two GPUs");
        const cudaError_t pe = cudaDeviceEnablePeerAccess(src->device, 0);
        if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (pe != cudaSuccess) return cuda_error(pe, "cudaDeviceEnablePeerAccess");
    }
    std::vector<Piece> pieces;
    merge_runs(src_runs, n_src, dst_runs, n_dst, pieces);
    Job j;
    int rc = begin_job(e, job_id, e->s_dev, j);
    if (rc) return rc;
    // the source's own payload writes (fills, K3 scatters) must have landed
    if (src != e && src->dev_write_pending) KVF_CUDA(cudaStreamWaitEvent(e->s_dev, src->dev_write_done, 0));
    Endpoint from{src->dev_pool, src->dev_slots * src->tpb, false};
    Endpoint to{e->dev_pool, e->dev_slots * e->tpb, false};
    rc = launch_copy(e, e->s_dev, from, to, pieces, KVF_COPY_SM_VEC, e->cfg.hbm_ctas);
    if (rc) return rc;
    KVF_CUDA(cudaEventRecord(e->dev_write_done, e->s_dev));  // new bytes in this pool
    e->dev_write_pending = true;
    j.bytes = ts * e->token_bytes;
    e->stats.dev_bytes += j.bytes;
    e->stats.dev_jobs++;
    return end_job(e, job_id, j);
}

int kvf_job_query(kvf_engine* e, uint64_t job_id, int32_t* done) {
    KVF_GUARD(e);
    auto it = e->jobs.find(job_id);
    if (it == e->jobs.end() || it->second.released)
        return set_error(KVF_E_UNKNOWN_JOB, "unknown job " + std::to_string(job_id));
    cudaError_t err = cudaEventQuery(it->second.stop);
    if (err == cudaErrorNotReady) {
        *done = 0;
        return KVF_OK;
    }
    if (err != cudaSuccess) return cuda_error(err, "cudaEventQuery(job)");
    *done = 1;
    return KVF_OK;
}

namespace {
// The blocking fences (wait / elapsed / release / span) take the engine lock only to look the
// job up and to drop their reference: a 20 ms K1 fence must not hold up a decision call or a
// launch from another thread on the same engine (cudaEventSynchronize itself is thread-safe).
void drop_job_ref(kvf_engine* e, uint64_t job_id) {
    auto it = e->jobs.find(job_id);
    if (it == e->jobs.end()) return;
    kvf_impl::Job& j = it->second;
    if (j.waiters) --j.waiters;
    if (j.released && j.waiters == 0) {
        recycle_event(e, j.start, true);
        recycle_event(e, j.stop, j.stamp_slot < 0);
        drop_stamp_ref(e, j.stamp_slot);
        if (j.lr_slot >= 0) e->lr_free.push_back(j.lr_slot);
        e->jobs.erase(it);
    }
}

// Look up `job_id` and take a reference (under the lock); `release` also marks it released.
int ref_job(kvf_engine* e, uint64_t job_id, bool release, cudaEvent_t* start, cudaEvent_t* stop,
            kvf_impl::Job* copy = nullptr) {
    std::lock_guard<std::mutex> lk(e->mu);
    if (cudaSetDevice(e->device) != cudaSuccess) return set_error(KVF_E_CUDA, "cudaSetDevice failed");
    kvf_impl::clear_stale_error(e, __func__);
    auto it = e->jobs.find(job_id);
    if (it == e->jobs.end() || it->second.released)
        return set_error(KVF_E_UNKNOWN_JOB, "unknown job " + std::to_string(job_id));
    ++it->second.waiters;
    if (release) it->second.released = true;
    if (start) *start = it->second.start;
    *stop = it->second.stop;
    if (copy) *copy = it->second;
    return KVF_OK;
}

// first start / last end of a job in ns on the GPU's clock (stamp-timed jobs only)
void stamp_bounds(const kvf_engine* e, const kvf_impl::Job& j, unsigned long long* lo, unsigned long long* hi) {
    const unsigned long long* st = e->stamps_h + static_cast<size_t>(j.stamp_slot) * kvf_impl::kStampCtas * 2;
    *lo = ~0ull;
    *hi = 0;
    for (uint32_t b = 0; b < j.stamp_ctas; ++b) {
        const unsigned long long a = st[2 * b], z = st[2 * b + 1];
        if (a && a < *lo) *lo = a;
        if (z > *hi) *hi = z;
    }
}

void unref_job(kvf_engine* e, uint64_t job_id) {
    std::lock_guard<std::mutex> lk(e->mu);
    drop_job_ref(e, job_id);
}
}  // namespace

int kvf_job_wait(kvf_engine* e, uint64_t job_id) {
    if (!e) return set_error(KVF_E_INVALID_ARG, "null engine");
    cudaEvent_t stop = nullptr;
    if (int rc = ref_job(e, job_id, false, nullptr, &stop)) return rc;
    const cudaError_t err = cudaEventSynchronize(stop);  // unlocked
    unref_job(e, job_id);
    return err == cudaSuccess ? KVF_OK : cuda_error(err, "cudaEventSynchronize(job)");
}

int kvf_job_elapsed_ms(kvf_engine* e, uint64_t job_id, float* ms) {
    if (!e || !ms) return set_error(KVF_E_INVALID_ARG, "null argument");
    cudaEvent_t start = nullptr, stop = nullptr;
    kvf_impl::Job j;
    if (int rc = ref_job(e, job_id, false, &start, &stop, &j)) return rc;
    cudaError_t err = cudaEventSynchronize(stop);
    if (err == cudaSuccess) {
        if (start) {
            err = cudaEventElapsedTime(ms, start, stop);
        } else {  // stamp-timed: the copy kernel's own globaltimer stamps
            unsigned long long lo, hi;
            stamp_bounds(e, j, &lo, &hi);
            *ms = hi > lo ? static_cast<float>((hi - lo) * 1e-6) : 0.f;
        }
    }
    unref_job(e, job_id);
    return err == cudaSuccess ? KVF_OK : cuda_error(err, "cudaEventElapsedTime(job)");
}

int kvf_job_release(kvf_engine* e, uint64_t job_id) {
    if (!e) return set_error(KVF_E_INVALID_ARG, "null engine");
    cudaEvent_t stop = nullptr;
    if (int rc = ref_job(e, job_id, true, nullptr, &stop)) return rc;
    // the events go back to the pool only once they have fired (and no one else waits on them)
    const cudaError_t err = cudaEventSynchronize(stop);
    unref_job(e, job_id);
    return err == cudaSuccess ? KVF_OK : cuda_error(err, "cudaEventSynchronize(release)");
}

int kvf_job_span_ms(kvf_engine* e, uint64_t first_job, uint64_t last_job, float* ms) {
    if (!e || !ms) return set_error(KVF_E_INVALID_ARG, "null argument");
    cudaEvent_t a_start = nullptr, a_stop = nullptr, b_stop = nullptr;
    kvf_impl::Job ja, jb;
    if (int rc = ref_job(e, first_job, false, &a_start, &a_stop, &ja)) return rc;
    if (int rc = ref_job(e, last_job, false, nullptr, &b_stop, &jb)) {
        unref_job(e, first_job);
        return rc;
    }
    cudaError_t err = cudaEventSynchronize(b_stop);
    if (err == cudaSuccess) err = cudaEventSynchronize(a_stop);
    if (err == cudaSuccess) {
        if (a_start && jb.start) {
            err = cudaEventElapsedTime(ms, a_start, b_stop);
        } else if (!a_start && !jb.start) {
            unsigned long long lo, hi, lo2, hi2;
            stamp_bounds(e, ja, &lo, &hi);
            stamp_bounds(e, jb, &lo2, &hi2);
            *ms = hi2 > lo ? static_cast<float>((hi2 - lo) * 1e-6) : 0.f;
        } else {
            err = cudaErrorInvalidResourceHandle;  // one event-timed, one stamp-timed: no common clock
        }
    }
    unref_job(e, last_job);
    unref_job(e, first_job);
    return err == cudaSuccess ? KVF_OK : cuda_error(err, "cudaEventElapsedTime(span)");
}

int kvf_sync_all(kvf_engine* e) {
    if (!e) return set_error(KVF_E_INVALID_ARG, "null engine");
    cudaStream_t ss[5];
    {
        KVF_GUARD(e);
        cudaStream_t s[5] = {e->s_h2d, e->s_d2h, e->s_dev, e->s_dec, e->s_cmp};
        std::copy(s, s + 5, ss);
    }
    for (cudaStream_t s : ss) KVF_CUDA(cudaStreamSynchronize(s));  // unlocked
    return KVF_OK;
}

int kvf_fill_payload(kvf_engine* e, int32_t tier, const kvf_run* runs, uint32_t n, const uint64_t* cids, uint64_t ntok) {
    KVF_GUARD(e);
    if (tier != 0 && tier != 1) return set_error(KVF_E_INVALID_ARG, "bad tier");
    uint64_t total = 0;
    if (!runs_valid(e, tier, runs, n, &total) || total != ntok || (ntok && !cids))
        return set_error(KVF_E_INVALID_ARG, "fill: runs/cids mismatch");
    if (ntok == 0) return KVF_OK;
    uint64_t *d_slots = nullptr, *d_cids = nullptr;
    int rc = stage_slots(e, runs, n, cids, ntok, &d_slots, &d_cids);
    if (rc) return rc;
    const uint64_t words = static_cast<uint64_t>(e->planes) * ntok * (e->tpb / 8);
    kvf_fill_kernel<<<grid_short(words, 256, 16), 256, 0, e->s_dev>>>(
        tier_base(e, tier), tier_slots(e, tier) * e->tpb, static_cast<uint32_t>(e->tpb), e->planes,
        e->geom.head_dim / 4, e->geom.head_offset, d_slots, d_cids, ntok);
    KVF_CUDA(cudaGetLastError());
    e->stats.kernel_launches++;
    KVF_CUDA(cudaEventRecord(e->dev_write_done, e->s_dev));
    e->dev_write_pending = true;
    return KVF_OK;
}

int kvf_checksum(kvf_engine* e, int32_t tier, const kvf_run* runs, uint32_t n, uint64_t* out) {
    KVF_GUARD(e);
    if (!out || (tier != 0 && tier != 1)) return set_error(KVF_E_INVALID_ARG, "bad argument");
    uint64_t ntok = 0;
    if (!runs_valid(e, tier, runs, n, &ntok)) return set_error(KVF_E_INVALID_ARG, "run out of pool range");
    // make every outstanding transfer visible first (a checksum is a verification read)
    for (cudaStream_t s : {e->s_h2d, e->s_d2h}) KVF_CUDA(cudaStreamSynchronize(s));
    *out = 0;
    if (ntok == 0) return KVF_OK;
    uint64_t* d_slots = nullptr;
    int rc = stage_slots(e, runs, n, nullptr, ntok, &d_slots, nullptr);
    if (rc) return rc;
    KVF_CUDA(cudaMemsetAsync(e->d_checksum, 0, sizeof(uint64_t), e->s_dev));
    const uint64_t words = static_cast<uint64_t>(e->planes) * ntok * (e->tpb / 8);
    kvf_checksum_kernel<<<grid_for(e, words, 256), 256, 0, e->s_dev>>>(
        tier_base(e, tier), tier_slots(e, tier) * e->tpb, static_cast<uint32_t>(e->tpb), e->planes, d_slots, ntok,
        reinterpret_cast<unsigned long long*>(e->d_checksum));
    KVF_CUDA(cudaGetLastError());
    e->stats.kernel_launches++;
    KVF_CUDA(cudaMemcpyAsync(out, e->d_checksum, sizeof(uint64_t), cudaMemcpyDeviceToHost, e->s_dev));
    KVF_CUDA(cudaStreamSynchronize(e->s_dev));
    return KVF_OK;
}

int kvf_payload_checksum(kvf_engine* e, const uint64_t* cids, uint64_t ntok, uint64_t* out) {
    KVF_GUARD(e);
    if (!out || (ntok && !cids)) return set_error(KVF_E_INVALID_ARG, "bad argument");
    *out = 0;
    if (ntok == 0) return KVF_OK;
    KVF_CUDA(cudaStreamSynchronize(e->s_dev));
    int rc = e->ws_dev.ensure(ntok * 8 + 64, ntok * 8 + 64);
    if (rc) return rc;
    std::memcpy(e->ws_dev.host, cids, ntok * 8);
    KVF_CUDA(cudaMemcpyAsync(e->ws_dev.dev, e->ws_dev.host, ntok * 8, cudaMemcpyHostToDevice, e->s_dev));
    KVF_CUDA(cudaMemsetAsync(e->d_checksum, 0, sizeof(uint64_t), e->s_dev));
    const uint64_t words = static_cast<uint64_t>(e->planes) * ntok * (e->tpb / 8);
    kvf_payload_checksum_kernel<<<grid_for(e, words, 256), 256, 0, e->s_dev>>>(
        static_cast<uint32_t>(e->tpb), e->planes, e->geom.head_dim / 4, e->geom.head_offset,
        static_cast<const uint64_t*>(e->ws_dev.dev), ntok, reinterpret_cast<unsigned long long*>(e->d_checksum));
    KVF_CUDA(cudaGetLastError());
    e->stats.kernel_launches++;
    KVF_CUDA(cudaMemcpyAsync(out, e->d_checksum, sizeof(uint64_t), cudaMemcpyDeviceToHost, e->s_dev));
    KVF_CUDA(cudaStreamSynchronize(e->s_dev));
    return KVF_OK;
}

int kvf_read_runs(kvf_engine* e, int32_t tier, const kvf_run* runs, uint32_t n, void* dst, uint64_t dst_bytes) {
    KVF_GUARD(e);
    if (!dst || (tier != 0 && tier != 1)) return set_error(KVF_E_INVALID_ARG, "bad argument");
    uint64_t ntok = 0;
    if (!runs_valid(e, tier, runs, n, &ntok)) return set_error(KVF_E_INVALID_ARG, "run out of pool range");
    if (dst_bytes < ntok * e->token_bytes) return set_error(KVF_E_INVALID_ARG, "destination too small");
    for (cudaStream_t s : {e->s_h2d, e->s_d2h}) KVF_CUDA(cudaStreamSynchronize(s));
    if (ntok == 0) return KVF_OK;
    KVF_CUDA(cudaStreamSynchronize(e->s_dev));
    const size_t bytes = ntok * e->token_bytes;
    int rc = e->ws_dev.ensure(bytes, 64);
    if (rc) return rc;
    kvf_run whole{0, ntok};
    std::vector<Piece> pieces;
    merge_runs(runs, n, &whole, 1, pieces);
    Endpoint src{tier_base(e, tier), tier_slots(e, tier) * e->tpb, tier == KVF_TIER_HOST};
    Endpoint dstp{static_cast<char*>(e->ws_dev.dev), ntok * e->tpb, false};
    rc = launch_copy(e, e->s_dev, src, dstp, pieces, KVF_COPY_SM_VEC, e->cfg.hbm_ctas);
    if (rc) return rc;
    KVF_CUDA(cudaMemcpyAsync(dst, e->ws_dev.dev, bytes, cudaMemcpyDeviceToHost, e->s_dev));
    KVF_CUDA(cudaStreamSynchronize(e->s_dev));
    return KVF_OK;
}

int kvf_get_stats(const kvf_engine* e, kvf_stats* out) {
    if (!e || !out) return set_error(KVF_E_INVALID_ARG, "bad argument");
    *out = e->stats;
    return KVF_OK;
}

}  // extern "C"
