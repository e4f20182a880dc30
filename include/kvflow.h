/* kvflow.h -- C-ABI of the B200-native KVFlow KV-movement engine (libkvflow.so).
 *
 * This is the drop-in boundary.  The reference (kvsim, C++) models the
 * tier engine's transfers with a cost model and never moves bytes; every entry point
 * below replaces one modelled step of that engine with real sm_100a work:
 *
 *   kvf_h2d_gather        <- TierManager::begin_load     proj/src/tier_manager.cpp:61-77
 *                            (+ enqueue_job, tier_manager.cpp:35-46)           [K1]
 *   kvf_d2h_scatter       <- TierManager::begin_offload  proj/src/tier_manager.cpp:48-59 [K2]
 *   kvf_dev_gather/
 *   kvf_dev_scatter       <- (new) staged path / compaction, SURVEY §8a row A13      [K3]
 *   kvf_job_query/wait    <- TierManager::complete        proj/src/tier_manager.cpp:95-124
 *                            (the TransferDone event, scheduler.cpp:94-97)
 *   kvf_priority_propagate<- RadixCache::set_agent_priorities proj/src/radix_cache.cpp:266-285 [K4]
 *   kvf_victim_select     <- RadixCache::evict (selection) proj/src/radix_cache.cpp:302-372 [K5]
 *   kvf_decode_attend     <- (new) decode-side consumer of the slot-run table, SURVEY §8f-3 [K6]
 *   kvf_decode_attend_layers <- the same for a decode step's layers as one chained job [K6]
 *   kvf_kv_append         <- (new) its write side: a layer's new K/V rows into slot runs
 *   kvf_peer_gather       <- (new) NVLink fetch from a replica's HBM, SURVEY §8f-4
 *   kvf_slots_alloc/free  <- (new) token-slot pools; the reference keeps only a byte ledger
 *                            (GpuPool, proj/include/kvsim/tier_manager.hpp:38-46)
 *
 * Conventions: every function is extern "C", never throws, and returns an int status:
 * KVF_OK (0) or a code that maps 1:1 onto kvsim::ErrorCode (errors.hpp:8-28) as
 * (ErrorCode + 1), plus engine-specific codes >= 100.  kvf_last_error() gives the text of
 * the last failure on the calling thread.  No torch types cross this boundary.
 *
 * KV layout (both tiers, per engine = per GPU shard):
 *   pool[plane = layer*2 + (0:K|1:V)][token_slot][local kv head][head_dim]  (bf16)
 * so one token of one plane is  tpb = kv_heads_local * head_dim * dtype_bytes  contiguous
 * bytes, and a node is a list of token-slot runs.  Splitting a radix node at any token
 * offset (radix_cache.cpp:142-177, 226-259) splits its run list; no bytes move.
 */
#ifndef KVFLOW_H
#define KVFLOW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------------- */
enum {
    KVF_OK = 0,
    /* kvsim::ErrorCode + 1 (proj/include/kvsim/errors.hpp:8-28) */
    KVF_E_UNKNOWN_AGENT = 1,
    KVF_E_SELF_LOOP = 2,
    KVF_E_DUPLICATE_AGENT = 3,
    KVF_E_EMPTY_ACTIVE_SET = 4,
    KVF_E_UNDERFLOW_UNLOCK = 5,
    KVF_E_UNKNOWN_BOUNDARY_NODE = 6,
    KVF_E_BOUNDARY_BEYOND_CACHE = 7,
    KVF_E_INSUFFICIENT_HISTORY = 8,
    KVF_E_ILLEGAL_STATE = 9,
    KVF_E_OUT_OF_GPU_MEMORY = 10,
    KVF_E_CONFIG = 11,
    KVF_E_UNKNOWN_AXIS = 12,
    KVF_E_IO = 13,
    KVF_E_INTERNAL = 14,
    /* engine-specific */
    KVF_E_CUDA = 100,          /* a CUDA runtime call failed (text in kvf_last_error) */
    KVF_E_INVALID_ARG = 101,
    KVF_E_OUT_OF_HOST_SLOTS = 102,
    KVF_E_NO_DEVICE = 103,     /* no CUDA device: the engine never falls back to the CPU */
    KVF_E_UNKNOWN_JOB = 104,
    KVF_E_TOO_LARGE = 105
};

enum { KVF_TIER_DEVICE = 0, KVF_TIER_HOST = 1 };

/* copy back-ends for K1/K2 (PCIe).  K3 always uses the SM path. */
enum {
    KVF_COPY_SM_VEC = 0,  /* LDG.128 / STG.128 SM-driven zero-copy (host pool is mapped pinned) */
    KVF_COPY_SM_BULK = 1, /* cp.async.bulk (TMA bulk engine) staging through shared memory      */
    KVF_COPY_CE = 2       /* copy engine (cudaMemcpy2DAsync per piece) -- comparator only      */
};

typedef struct kvf_engine kvf_engine; /* opaque */

typedef struct {
    uint32_t layers;         /* L                                   */
    uint32_t kv_heads_total; /* Hkv of the model                    */
    uint32_t kv_heads_local; /* heads this shard holds (Hkv / G)    */
    uint32_t head_offset;    /* first global head of this shard     */
    uint32_t head_dim;       /* D                                   */
    uint32_t dtype_bytes;    /* 2 (bf16)                            */
} kvf_geometry;

typedef struct {
    int32_t device;           /* CUDA ordinal                                          */
    uint64_t gpu_slots;       /* HBM pool capacity in tokens                           */
    uint64_t host_slots;      /* pinned host pool capacity in tokens                   */
    uint32_t pcie_ctas;       /* grid for K1/K2 (0 = default)                          */
    uint32_t pcie_mode;       /* KVF_COPY_* for K1/K2                                  */
    uint32_t hbm_ctas;        /* grid for K3 (0 = default: 4 per SM)                   */
    int32_t host_numa_node;   /* -1: no binding; KVF_NUMA_AUTO (-2): the GPU's own node
                                 (sysfs of its PCI device); else mbind the host pool there */
} kvf_engine_config;

typedef struct {
    uint64_t start; /* first token slot */
    uint64_t len;   /* tokens           */
} kvf_run;

/* ---- lifecycle -------------------------------------------------------------------- */
const char* kvf_last_error(void);
const char* kvf_version(void);
int kvf_device_count(int32_t* out);
#define KVF_NUMA_AUTO (-2)
/* NUMA node of a GPU's PCI device (-1 when the platform does not say). */
int kvf_device_numa_node(int32_t device, int32_t* node);
int kvf_engine_create(const kvf_geometry* geom, const kvf_engine_config* cfg, kvf_engine** out);
int kvf_engine_destroy(kvf_engine* e);
/* bytes one token occupies in one plane on this shard, and across all planes */
int kvf_engine_token_bytes(const kvf_engine* e, uint64_t* tpb, uint64_t* token_bytes);
int kvf_engine_set_copy_mode(kvf_engine* e, uint32_t pcie_mode, uint32_t pcie_ctas, uint32_t hbm_ctas);
/* How K1 / K2 jobs are timed (kvf_job_elapsed_ms / kvf_job_span_ms):
 *   EVENTS (default): a timing CUDA event before and after the job on its stream;
 *   STAMPS: only a non-timing stop event (the fence), device time from the copy kernel's own
 *   per-CTA %globaltimer stamps -- a timing event record costs ~1.3 us of host time per call,
 *   a plain one ~0.1 us, so a control loop issuing many transfers uses STAMPS.  Other jobs
 *   (K3, K6, compute) keep events.  Env KVF_JOB_TIMING=stamps sets STAMPS at creation. */
enum { KVF_JOB_TIMING_EVENTS = 0, KVF_JOB_TIMING_STAMPS = 1 };
int kvf_engine_set_job_timing(kvf_engine* e, uint32_t mode);

/* ---- token-slot pools ---------------------------------------------------------------- */
/* Allocates `tokens` slots as <= max_runs runs (best-fit single run when possible). */
int kvf_slots_alloc(kvf_engine* e, int32_t tier, uint64_t tokens, kvf_run* out_runs, uint32_t max_runs,
                    uint32_t* n_runs);
int kvf_slots_free(kvf_engine* e, int32_t tier, const kvf_run* runs, uint32_t n_runs);
int kvf_slots_free_count(const kvf_engine* e, int32_t tier, uint64_t* free_tokens, uint64_t* free_runs);
/* Raw pool base (device pointer for DEVICE; host pointer -- also device-addressable -- for HOST). */
int kvf_pool_ptr(const kvf_engine* e, int32_t tier, void** base, uint64_t* slots);

/* ---- data movement (async; one job = one node transfer) ------------------------------- */
/* job_id is chosen by the caller (TierManager job ids, tier_manager.cpp:470-481) and must be
 * unique among unreleased jobs.  Token k of the node (in run order) moves from the k-th slot
 * of src_runs to the k-th slot of dst_runs, all planes; total src and dst tokens must match. */
int kvf_h2d_gather(kvf_engine* e, uint64_t job_id, const kvf_run* host_runs, uint32_t n_host,
                   const kvf_run* dev_runs, uint32_t n_dev); /* K1 */
int kvf_d2h_scatter(kvf_engine* e, uint64_t job_id, const kvf_run* dev_runs, uint32_t n_dev,
                    const kvf_run* host_runs, uint32_t n_host); /* K2 */
/* K3: paged HBM pool <-> contiguous HBM staging laid out [plane][token][head][dim]
 * (a 1-run pool of `tokens` slots).  staging is a device pointer. */
int kvf_dev_gather(kvf_engine* e, uint64_t job_id, const kvf_run* dev_runs, uint32_t n_dev, void* staging);
int kvf_dev_scatter(kvf_engine* e, uint64_t job_id, const void* staging, const kvf_run* dev_runs,
                    uint32_t n_dev);

/* Peer fetch (SURVEY §8f-4 follow-on): copy a node's KV from ANOTHER engine's HBM pool --
 * typically a data-parallel replica on another GPU of the box, read over NVLink / NVSwitch by
 * a K3-style kernel on this GPU -- instead of reloading it from host memory over PCIe.
 * Both engines must hold the same shard geometry; src == e copies within one pool.  The
 * caller guarantees the source node is resident (its load, if any, has completed) and not
 * released while the job runs; the source engine's own payload writes are waited for.
 * Async on this engine's HBM stream as job `job_id`. */
int kvf_peer_gather(kvf_engine* e, uint64_t job_id, kvf_engine* src, const kvf_run* src_runs, uint32_t n_src,
                    const kvf_run* dst_runs, uint32_t n_dst);

/* K2 for several nodes in ONE launch (small-node write-back batching):
 * job k moves dev_runs[off_k .. off_k + dev_counts[k]) -> host_runs[...host_counts[k]), the
 * run lists concatenated in job order.  Every job keeps its own id and events (all complete
 * when the shared launch does); the batch is validated before any job is created.
 * Reference: one tier_manager.cpp:48-59 begin_offload per node of an evict call. */
int kvf_d2h_scatter_batch(kvf_engine* e, uint32_t n_jobs, const uint64_t* job_ids, const kvf_run* dev_runs,
                          const uint32_t* dev_counts, const kvf_run* host_runs, const uint32_t* host_counts);
/* K1, layer-pipelined: tiles go plane-outermost, and each finished tile bumps
 * layer_ready[layer] (caller's device array of `layers` uint32, zeroed by the call); layer l
 * has landed when layer_ready[l] == *tiles_per_layer.  A consumer can start on layer l while
 * later layers are still on the wire -- the real mechanism behind the reference's
 * overlap_fraction gate model (proj/src/scheduler.cpp:252-284, :281). */
int kvf_h2d_gather_layered(kvf_engine* e, uint64_t job_id, const kvf_run* host_runs, uint32_t n_host,
                           const kvf_run* dev_runs, uint32_t n_dev, uint32_t* layer_ready,
                           uint32_t* tiles_per_layer);
/* layer_ready == NULL: the engine owns the counters (64 concurrent layered jobs); the compute
 * stream then waits for layer `layer` of the job with kvf_compute_wait_job_layer.  Jobs that
 * are not layered degrade to a whole-job wait.  tiles_per_layer may be NULL in this mode. */
int kvf_compute_wait_job_layer(kvf_engine* e, uint64_t job_id, uint32_t layer);
/* compute-stream helpers (model compute emulation for measurements and the wall-clock
 * driver, on the engine's own compute stream): wait for a layer of a layered load, wait for a
 * whole transfer job (its stop event), spin for ns nanoseconds on `ctas` SMs, and bracket
 * compute work as a job (kvf_job_query / kvf_job_elapsed_ms / kvf_job_release apply). */
int kvf_compute_wait_layer(kvf_engine* e, const uint32_t* layer_ready, uint32_t layer, uint32_t target);
int kvf_compute_wait_job(kvf_engine* e, uint64_t job_id);
int kvf_compute_spin(kvf_engine* e, uint64_t ns, uint32_t ctas);
int kvf_compute_job_begin(kvf_engine* e, uint64_t job_id);
int kvf_compute_job_end(kvf_engine* e, uint64_t job_id);
/* device time from first_job's start event to last_job's stop event (any streams) */
int kvf_job_span_ms(kvf_engine* e, uint64_t first_job, uint64_t last_job, float* ms);

/* fences (TierManager::complete): 1 in *done when the job's bytes have landed */
int kvf_job_query(kvf_engine* e, uint64_t job_id, int32_t* done);
int kvf_job_wait(kvf_engine* e, uint64_t job_id);
/* device duration of the job's kernel(s), CUDA events on the job's own stream */
int kvf_job_elapsed_ms(kvf_engine* e, uint64_t job_id, float* ms);
int kvf_job_release(kvf_engine* e, uint64_t job_id);
int kvf_sync_all(kvf_engine* e);

/* ---- decisions (synchronous; small SoA in, ordered actions out) ------------------------- */
/* SoA view of the radix tree, index 0 = root (parent -1), parent[i] < i (preorder). */
typedef struct {
    uint32_t n;
    const int32_t* parent;
    const uint16_t* depth;   /* root = 0 */
    const uint8_t* status;   /* 0 IN_GPU 1 BACKUP_IN_CPU 2 LOADING 3 OFFLOADING (radix_cache.hpp:21-28) */
    const int32_t* lock;
    const int64_t* rank;
    const double* time;      /* LastAccess.time (radix_cache.hpp:44-47) */
    const uint64_t* seq;     /* LastAccess.seq */
    const uint64_t* id;
    const uint64_t* tokens;
    const uint8_t* backed;   /* cpu_backed */
    uint64_t bytes_per_token;
} kvf_tree_view;

typedef struct {
    uint64_t needed;
    int32_t workflow_aware; /* EvictionPolicy::WorkflowAware */
    int32_t offload_mode;   /* TierMode::Offload */
    int32_t has_floor;      /* EvictRequest::rank_floor_exclusive engaged */
    int64_t floor;
    uint64_t cpu_used;      /* TierManager::cpu_used()      */
    uint64_t cpu_capacity;  /* 0 = unbounded                */
} kvf_evict_request;

enum { KVF_ACT_OFFLOAD = 0, KVF_ACT_DISCARD_TO_BACKUP = 1, KVF_ACT_REMOVE = 2 };

/* K4: out_rank[i] for i >= 1 = min(SUFFIX, min over boundaries b whose root path contains i
 * of cand_rank[b]).  out_rank[0] = SUFFIX. */
int kvf_priority_propagate(kvf_engine* e, const int32_t* parent, uint32_t n, const int32_t* boundary_idx,
                           const int64_t* cand_rank, uint32_t m, int64_t* out_rank);
/* K5: the ordered victims the reference's greedy heap would pop, with their actions. */
int kvf_victim_select(kvf_engine* e, const kvf_tree_view* tree, const kvf_evict_request* req, int32_t* out_idx,
                      uint8_t* out_action, uint32_t* out_count, uint64_t* out_immediate, uint64_t* out_pending);

/* ---- decisions over a tree mirrored in HBM --------------------------------------------- */
/* The calls above take a whole SoA snapshot per call.  A kvf_tree keeps the radix tree's SoA
 * resident in HBM instead, indexed by a stable per-node slot the host assigns (slot 0 = root;
 * freed slots are reused), and the host sends only the nodes that changed since the last
 * decision (insert / split / touch / lock / status / backup / removal).  Replaces the
 * pack-per-call of RadixCache::set_agent_priorities / evict
 * (proj/src/radix_cache.cpp:266-285, :302-372 walk the live tree on every call).
 *
 * Decisions are requests in a ring in mapped pinned memory, executed in order either by a
 * RESIDENT decider (one 128-thread CTA polling the ring: no launch per decision; trees up to
 * KVF_RESIDENT_MAX_SLOTS slots: its 128 threads lose to a launch sized to the tree beyond that)
 * or by one launch per request (larger trees, or the resident
 * decider disabled).  The resident CTA exits after KVF_DECIDER_IDLE_US (default 200) of idle,
 * so a device-wide synchronize elsewhere waits at most that long; kvf_decider_hold(e, 1) keeps
 * it alive across idle gaps (a driver's run), kvf_decider_hold(e, 0) lets it go at once. */
typedef struct kvf_tree kvf_tree;

#define KVF_SLOT_DEAD 0xFF        /* status of a freed slot */
#define KVF_RESIDENT_MAX_SLOTS 128u
/* Record flag: the host has not read back a queued K4 yet, so its copy of this node's rank may
 * be stale -- the record updates every other field and keeps the rank the mirror holds. */
#define KVF_REC_KEEP_RANK 1u

typedef struct {
    uint32_t slot;    /* mirror slot of this node */
    int32_t parent;   /* parent's slot; -1 for the root and for a dead slot */
    int32_t lock;     /* lock_count (radix_cache.hpp:57) */
    uint8_t status;   /* NodeStatus 0..3, or KVF_SLOT_DEAD */
    uint8_t backed;   /* cpu_backed */
    uint16_t flags;   /* KVF_REC_KEEP_RANK: leave the mirror's rank as it is (see below) */
    int64_t rank;     /* host-authored ranks (new nodes SUFFIX, split halves); K4 rewrites them */
    double time;      /* LastAccess.time */
    uint64_t seq;     /* LastAccess.seq */
    uint64_t id;
    uint64_t tokens;  /* key length */
    uint64_t pad1;
} kvf_node_rec;       /* 64 bytes */

int kvf_tree_create(kvf_engine* e, uint64_t bytes_per_token, uint32_t capacity_hint, kvf_tree** out);
int kvf_tree_destroy(kvf_tree* t);
/* Stage node records; they reach the mirror ahead of the tree's next decision (last record
 * of a slot wins).  Slots must be < 2^24. */
int kvf_tree_update(kvf_tree* t, const kvf_node_rec* recs, uint32_t n);
/* KVF_TREE_TIME_FOLLOWS_SEQ: every access stamp (time, seq) was taken with a non-decreasing
 * time and an increasing seq (a cache whose clock never runs backwards) -- then `before`
 * orders like (seq, id) and the device-wide K5 drops the 8 radix passes over the time word. */
#define KVF_TREE_TIME_FOLLOWS_SEQ 1u
int kvf_tree_set_hints(kvf_tree* t, uint32_t hints);
/* K4 over the mirror (set_agent_priorities): boundary_slot[b] / cand_rank[b] as for
 * kvf_priority_propagate.  Asynchronous: returns once the request is queued; the mirror's
 * ranks are updated before any later decision on this tree.  Up to two K4 requests may be
 * outstanding (KVF_E_INVALID_ARG for a third); kvf_tree_rank_changes waits for the OLDEST and
 * returns the slots whose rank it changed (at most the tree's slot count entries), relative
 * to the ranks the K4 before it left -- applying each result in order gives the latest ranks. */
int kvf_tree_priorities(kvf_tree* t, const uint32_t* boundary_slot, const int64_t* cand_rank, uint32_t m);
/* The same K4, staged instead of posted: it travels in the ring slot of the tree's next request
 * -- with the next kvf_tree_victims in ONE slot (records, K4, K5: one poll, one serve) -- or
 * alone when kvf_tree_rank_changes / another K4 needs it first.  For a caller that always
 * decides next (RadixCache::evict after set_agent_priorities_async). */
int kvf_tree_stage_priorities(kvf_tree* t, const uint32_t* boundary_slot, const int64_t* cand_rank, uint32_t m);
int kvf_tree_rank_changes(kvf_tree* t, uint32_t* slots, int64_t* ranks, uint32_t cap, uint32_t* n_changed);
/* K5 over the mirror (evict's victim order and actions); victims as slots.  Synchronous. */
int kvf_tree_victims(kvf_tree* t, const kvf_evict_request* req, uint32_t* out_slot, uint8_t* out_action,
                     uint32_t cap, uint32_t* out_count, uint64_t* out_immediate, uint64_t* out_pending);
/* Resident decider control (see above).  hold = 1: never idle out; 0: exit now if idle. */
int kvf_decider_hold(kvf_engine* e, int32_t hold);
/* 1 in *running while the resident decider CTA is alive. */
int kvf_decider_running(kvf_engine* e, int32_t* running);

/* ---- decode-side consumer of the slot-run table ------------------------ */
/* KV write side of the same layout: store freshly computed K and V of `ntok` tokens for one
 * layer (a prefill chunk, or one decode token per sequence) into HBM slot runs.
 *   k, v: device bf16 [ntok][kv_heads_local][head_dim] -- the model's projection layout;
 *   runs: the tokens' slots in order (sum of lengths == ntok).
 * Async on the engine's payload-write stream as job `job_id`; write-backs (K2) and K6 calls
 * issued later are ordered after it.  k / v must be ready when the call is made. */
int kvf_kv_append(kvf_engine* e, uint64_t job_id, uint32_t layer, const kvf_run* runs, uint32_t n_runs, const void* k,
                  const void* v, uint64_t ntok);

/* K6: one decode step of GQA attention, reading layer `layer`'s K and V IN PLACE from the
 * HBM pool through each sequence's slot-run list (what RadixCache::match_prefix hands out,
 * proj/src/radix_cache.cpp:88-140, plus the request's suffix) -- no compaction copy.
 *   q, out:  device bf16 [batch][kv_heads_local * group][128]  (head_dim must be 128)
 *   runs:    the sequences' run lists concatenated, run_counts[b] runs for sequence b (token
 *            order); a sequence with no runs gets out = 0.
 *   out[b][h] = softmax(scale * q[b][h] . K_b^T) V_b  over kv head h / group, fp32 softmax,
 *            P rounded to bf16 before P.V (flash-decoding).
 *   chunk_tokens: tokens per work item (multiple of 16 in [16, 2048]; 0 = one wave of CTAs).
 * Async on the engine's compute stream as job `job_id` (kvf_job_wait / elapsed / release);
 * ordered after the engine's own payload writes.  A caller consuming a prefetched node
 * fences first with kvf_compute_wait_job(prefetch job); q must be ready and out unused
 * until the job completes. */
int kvf_decode_attend(kvf_engine* e, uint64_t job_id, uint32_t layer, uint32_t batch, uint32_t group,
                      const void* q, const kvf_run* runs, const uint32_t* run_counts, float scale, void* out,
                      uint32_t chunk_tokens);
/* A decode step's layers layer0 .. layer0+nlayers-1 as ONE job over the same run tables.
 * PRECONDITION: every layer's q is ready when the call is made.  In a real decoder layer
 * l+1's q depends on layer l's output, so a decode step cannot use this chain -- it calls
 * kvf_decode_attend once per layer; this entry point is for workloads whose queries are known
 * up front (speculative / re-scoring passes) and is an upper bound for the per-layer path. */
/* Layout:
 * q[l] / out[l] are layer (layer0 + l)'s buffers, laid out as for kvf_decode_attend.  The
 * layers' kernels are chained with programmatic dependent launch, so layer l+1 starts on the
 * SMs layer l has finished with; results are bit-identical to nlayers kvf_decode_attend
 * calls.  The q / out pointer arrays are read during the call only. */
int kvf_decode_attend_layers(kvf_engine* e, uint64_t job_id, uint32_t layer0, uint32_t nlayers, uint32_t batch,
                             uint32_t group, const void* const* q, const kvf_run* runs, const uint32_t* run_counts,
                             float scale, void* const* out, uint32_t chunk_tokens);

/* ---- payload (prefill emulation) and verification ----------------------------------- */
/* Writes the deterministic payload of tokens with content ids cids[0..ntok) into the runs
 * (emulates prefill writing KV).  Async on the engine's compute stream. */
int kvf_fill_payload(kvf_engine* e, int32_t tier, const kvf_run* runs, uint32_t n_runs, const uint64_t* cids,
                     uint64_t ntok);
/* Order-independent checksum of a node's bytes in logical (plane, token, byte) order.  Sync. */
int kvf_checksum(kvf_engine* e, int32_t tier, const kvf_run* runs, uint32_t n_runs, uint64_t* out);
/* The checksum a node with content ids cids[0..ntok) must have (no buffer; computed on the
 * GPU from the payload definition).  Sync. */
int kvf_payload_checksum(kvf_engine* e, const uint64_t* cids, uint64_t ntok, uint64_t* out);
/* Copies a node's bytes in logical order into a host buffer of ntok*token_bytes bytes.  Sync. */
int kvf_read_runs(kvf_engine* e, int32_t tier, const kvf_run* runs, uint32_t n_runs, void* dst, uint64_t dst_bytes);

/* ---- stats ---------------------------------------------------------------------------- */
typedef struct {
    uint64_t kernel_launches; /* every kernel this engine launched */
    uint64_t h2d_bytes, d2h_bytes, dev_bytes;
    uint64_t h2d_jobs, d2h_jobs, dev_jobs, decisions;
    double decision_kernel_ms; /* K4+K5 kernel time, CUDA events on the decision stream */
    double decision_call_us;   /* K4+K5 host round trip (pack, H2D, kernel, D2H, sync)  */
    double k5_phase_ns[5];     /* K5 in-kernel phases: stage, sort, walks, victim sort, scan+out */
    double k5_phase_cycles[5]; /* the same phases in SM cycles (clock64)                       */
    uint64_t stale_errors;     /* non-sticky CUDA errors found pending at API entry (cleared) */
    uint64_t attend_calls, attend_bytes; /* K6 calls, KV bytes they read */
    uint64_t resident_served;  /* mirror decisions served by the resident decider CTA */
    uint64_t oneshot_served;   /* mirror decisions served by a launch of their own */
    uint64_t resident_launches;/* resident decider (re)launches */
    uint64_t mirror_records;   /* node records shipped to tree mirrors */
} kvf_stats;
int kvf_get_stats(const kvf_engine* e, kvf_stats* out);

#ifdef __cplusplus
}
#endif
#endif /* KVFLOW_H */
