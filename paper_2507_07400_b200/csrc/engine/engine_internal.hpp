// Internal declarations shared by the translation units of libkvflow.so.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "kvflow.h"

namespace kvf_impl {

// ---- error plumbing: thread-local last error, int status everywhere -------------------
int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* what);

#define KVF_CUDA(call)                                       \
    do {                                                     \
        cudaError_t _e = (call);                             \
        if (_e != cudaSuccess) return cuda_error(_e, #call); \
    } while (0)

// ---- token-slot allocator: free intervals with a size index ----------------------------
class SlotAllocator {
public:
    void reset(uint64_t slots);
    // best-fit single run, else largest-first multi-run; false if not enough free slots
    bool alloc(uint64_t tokens, std::vector<kvf_run>& out);
    // returns false on double free / out of range
    bool release(const kvf_run& r);
    uint64_t free_tokens() const { return free_tokens_; }
    uint64_t free_runs() const { return by_start_.size(); }
    uint64_t capacity() const { return capacity_; }

private:
    void insert_free(uint64_t start, uint64_t len);
    void erase_free(std::map<uint64_t, uint64_t>::iterator it);
    std::map<uint64_t, uint64_t> by_start_;           // start -> len
    std::multimap<uint64_t, uint64_t> by_len_;        // len -> start
    uint64_t capacity_ = 0;
    uint64_t free_tokens_ = 0;
};

// ---- copy descriptors ---------------------------------------------------------------
// A piece is a token range contiguous in both source and destination pools.
struct Piece {
    uint64_t src_slot, dst_slot, ntok;
};
void merge_runs(const kvf_run* a, uint32_t na, const kvf_run* b, uint32_t nb, std::vector<Piece>& out);

struct Job {
    cudaEvent_t start = nullptr, stop = nullptr;
    cudaStream_t stream = nullptr;
    uint64_t bytes = 0;
    // layered H2D with engine-owned counters: slot, and layer l has landed once
    // counters[slot][l] >= lr_base + lr_tpl (counters only grow; never reset)
    int32_t lr_slot = -1;
    uint32_t lr_base = 0, lr_tpl = 0;
    // blocking fences run outside the engine lock: threads inside one hold a reference, and a
    // release that finds waiters leaves the recycling of the events to the last of them
    uint32_t waiters = 0;
    bool released = false;
    // stamp-timed job (kvf_engine_set_job_timing STAMPS): no start event, a non-timing stop
    // event, device time from the copy kernel's per-CTA globaltimer stamps in a mapped slot
    int32_t stamp_slot = -1;
    uint32_t stamp_ctas = 0;
};

constexpr uint32_t kStampSlots = 256;  // stamp-timed transfers in flight
constexpr uint32_t kStampCtas = 64;    // CTAs stamped per slot (K1/K2 run 8)

constexpr uint32_t kLayerSlots = 64;

struct BigGraph {  // device-wide K5 captured once per (bucketed size, policy)
    cudaGraphExec_t exec = nullptr;
    uint32_t kernels = 0;
};  // concurrent layered loads with engine-owned counters

// ---- device-wide K5 (decide_large.cu) over device arrays of n entries (pads: dead) -------
struct LargeArrays {
    const int32_t* parent;
    const uint8_t* status;
    const int32_t* lock;
    const int64_t* rank;
    const double* time;
    const uint64_t* seq;
    const uint64_t* id;
    const uint64_t* tokens;
    const uint8_t* backed;
    uint32_t n;  // live slots; the arrays hold large_capacity(n) entries
};
// What bounds the sort key of `before` (radix_cache.cpp:316-321): largest id / access seq,
// whether every step rank fits the compact code, and whether access times follow access
// sequence numbers (every touch takes (now, ++counter) with a non-decreasing now: then
// (time, seq, id) orders like (seq, id) and the 8 time passes can go).
struct LargeKeyInfo {
    uint64_t max_id = 0, max_seq = 0;
    int64_t rank_max = 0;
    bool rank_small = true;
    bool time_follows_seq = false;
    void note_rank(int64_t r) {
        if (r == INT64_MAX / 2 || r == INT64_MAX / 4) return;
        if (r < 0 || r > (int64_t{1} << 40)) rank_small = false;
        else if (r > rank_max) rank_max = r;
    }
    void note(const kvf_node_rec& r) {
        if (r.status == KVF_SLOT_DEAD) return;
        if (r.id > max_id) max_id = r.id;
        if (r.seq > max_seq) max_seq = r.seq;
        note_rank(r.rank);
    }
};

struct Workspace {  // grow-only device + pinned staging buffers
    kvf_engine* owner = nullptr;  // growing frees (a device-wide sync): the resident decider stops first
    void* dev = nullptr;
    size_t dev_bytes = 0;
    void* host = nullptr;
    void* host_dev = nullptr;  // device-side alias of `host` (mapped pinned memory)
    size_t host_bytes = 0;
    int ensure(size_t dev_need, size_t host_need);
    void release();
};

struct LargeState {  // per caller of the device-wide path: scratch + captured graphs
    Workspace ws;
    std::map<uint64_t, BigGraph> graphs;
    const void* baked = nullptr;  // the input arrays the graphs were captured against
};
uint32_t large_capacity(uint32_t n);  // padded size the device-wide path runs over
void large_invalidate(LargeState& st);
void large_release(LargeState& st);

// Resident decider + request ring of the tree mirrors (mirror.cu).
struct DeciderState {
    char* ring_h = nullptr;  // mapped pinned: kRing request slots + control block
    char* ring_d = nullptr;
    char* pay_h = nullptr;   // mapped pinned: one payload area per ring slot
    char* pay_d = nullptr;
    size_t pay_slot = 0;
    uint64_t posted = 0;     // last request sequence number handed out
    uint64_t acked = 0;      // every request <= this one is known to be served
    cudaStream_t s_res = nullptr;
    cudaEvent_t ev_res = nullptr, ev_dec = nullptr;
    bool running = false;    // the resident CTA is (believed) alive
    bool hold = false;       // never idle out (kvf_decider_hold)
    bool disabled = false;   // KVF_DECIDER=0: one launch per request
    bool res_attr_set = false, once_attr_set = false;
    uint64_t epoch = 0;      // launch count of the resident CTA (its exit word carries it)
    uint64_t last_res_post = 0;  // last request handed to the resident CTA
    uint64_t idle_ns = 200000;
    uint32_t res_cap = 0;    // slots the resident CTA's shared memory is sized for
};

}  // namespace kvf_impl

struct kvf_engine {
    kvf_geometry geom{};
    kvf_engine_config cfg{};
    int device = 0;
    int sm_count = 148;
    uint64_t tpb = 0;          // bytes per token per plane on this shard
    uint32_t planes = 0;       // layers * 2
    uint64_t token_bytes = 0;  // tpb * planes

    char* dev_pool = nullptr;
    uint64_t dev_slots = 0;
    char* host_pool = nullptr;      // host address
    char* host_pool_dev = nullptr;  // device-side address of the same memory
    uint64_t host_slots = 0;
    bool host_registered = false;
    int32_t host_numa = -1;         // node the host pool is bound to (-1: none)   // mmap+cudaHostRegister (NUMA-bound) vs cudaHostAlloc
    size_t host_map_bytes = 0;

    kvf_impl::SlotAllocator alloc[2];

    cudaStream_t s_h2d = nullptr, s_d2h = nullptr, s_dev = nullptr, s_dec = nullptr;
    cudaStream_t s_cmp = nullptr;  // emulated model compute (kvf_compute_*): never behind a fill
    cudaEvent_t dev_write_done = nullptr;  // last fill / K3 scatter on s_dev
    cudaEvent_t dec_start = nullptr, dec_stop = nullptr;  // decision kernel timing (copy path)
    unsigned long long dec_seq = 0;  // decision calls: the done word the fast path spins on
    bool dev_write_pending = false;

    std::unordered_map<uint64_t, kvf_impl::Job> jobs;
    std::vector<cudaEvent_t> event_pool;
    std::vector<cudaEvent_t> event_pool_nt;  // non-timing events (stamp-timed jobs' stop events)
    bool stamp_timing = false;               // PCIe transfer jobs timed by kernel stamps
    unsigned long long* stamps_h = nullptr;  // mapped: [kStampSlots][kStampCtas][2] globaltimer ns
    unsigned long long* stamps_d = nullptr;
    std::vector<int32_t> stamp_free;
    std::vector<uint32_t> stamp_refs;        // jobs sharing a slot (one K2 batch launch)

    kvf_impl::Workspace ws_dev;  // fill / checksum / read staging (s_dev)
    kvf_impl::Workspace ws_dec;  // decision kernels (s_dec)
    kvf_impl::Workspace ws_att;  // K6 decode attention: descriptors + partials (s_cmp)
    cudaEvent_t att_upload_done = nullptr;  // last K6 descriptor upload out of ws_att.host
    bool att_upload_pending = false, attend_attr_set = false;
    int attend_occ = 0;  // resident K6 CTAs per SM
    std::vector<uint64_t> att_sig;  // K6 descriptor cache: inputs of the blob now in ws_att.dev
    std::vector<uint8_t> att_items;  // K6 work items of that blob (host copy for the launch parameters)
    uint64_t att_meta[10] = {};     //   and its sizes (a decode step calls K6 once per layer)
    kvf_impl::Workspace ws_big;  // snapshot upload for the device-wide K5 (grown on demand)
    kvf_impl::LargeState large_snap;  // device-wide K5 state of kvf_victim_select

    uint64_t* d_checksum = nullptr;
    uint32_t* d_layer_ctr = nullptr;       // [kLayerSlots][layers] landed-tile counters
    std::vector<uint32_t> lr_total;         // host mirror: tiles ever published per layer, per slot
    std::vector<int32_t> lr_free;           // free counter slots
    bool victim_attr_set = false, prio_attr_set = false, bulk_attr_set = false;
    kvf_impl::DeciderState dec;
    kvf_stats stats{};
    std::mutex mu;  // engine calls are serialised per engine
};

// Entry of every engine C-ABI call: null check, the engine's mutex, its device, and any
// non-sticky error another caller left pending taken out of the way.
#define KVF_GUARD(e)                                                                                     \
    if (!(e)) return kvf_impl::set_error(KVF_E_INVALID_ARG, "null engine");                              \
    std::lock_guard<std::mutex> _lk((e)->mu);                                                            \
    if (cudaSetDevice((e)->device) != cudaSuccess) return kvf_impl::set_error(KVF_E_CUDA, "cudaSetDevice failed"); \
    kvf_impl::clear_stale_error(e, __func__)

namespace kvf_impl {
int acquire_event(kvf_engine* e, cudaEvent_t* ev, bool timing = true);
// a job = start event on `stream` ... kernels ... stop event (end_job registers it)
int begin_job(kvf_engine* e, uint64_t job_id, cudaStream_t stream, Job& j, int32_t stamp_slot = -1);
int end_job(kvf_engine* e, uint64_t job_id, Job& j);
void clear_stale_error(kvf_engine* e, const char* fn);
// Every engine kernel prefers the max-shared-memory carveout, so SMs never switch their L1 /
// shared split between kernels: a switch needs a drained SM, and a streaming grid (a prompt
// fill) keeps every SM busy until it ends -- a decision CTA needing a different split waited
// ~0.6 ms for that (scripts/decision_trace.py, KVF_ARRIVAL_TRACE).  Once per process.
void set_carveout_decide();
void set_carveout_attend();
int victim_select_large(kvf_engine* e, const kvf_tree_view* t, const kvf_evict_request* q, int32_t* out_idx,
                        uint8_t* out_action, uint32_t* out_count, uint64_t* out_imm, uint64_t* out_pend);
// victims (as array indices) of `a` in pop order; synchronous on the decision stream
int victim_large(kvf_engine* e, LargeState& st, const LargeArrays& a, const kvf_evict_request* q, uint64_t bpt,
                 const LargeKeyInfo& keys, uint32_t* out_idx, uint8_t* out_action, uint32_t cap, uint32_t* out_count,
                 uint64_t* out_imm, uint64_t* out_pend);
void recycle_event(kvf_engine* e, cudaEvent_t ev, bool timing = true);
// mirror.cu: stop the resident decider CTA and wait for it to leave (before any call that
// synchronises the whole device: cudaFree, cudaFreeHost, cudaDeviceSynchronize)
void decider_quiesce(kvf_engine* e);
int decider_init(kvf_engine* e);
void decider_release(kvf_engine* e);
void set_carveout_mirror();
}  // namespace kvf_impl
