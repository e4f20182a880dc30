/* kvf_oracle: CPU restatement of the KVFlow KV-movement hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the CHECKER
 * (or the timed CPU baseline).  The product path (paper_2507_07400_b200/, libkvflow.so)
 * never links or calls it.
 *
 * Pinning (see oracle/README.md and DESIGN.md §Parity):
 *   - kvfo_evict / kvfo_priority are checked against golden vectors produced by the
 *     UNMODIFIED reference (oracle/_ref/ref_trace evict|prio -> the tests/golden fixtures).
 *   - The byte oracle (payload, copy, checksum) has no reference counterpart: the reference
 *     moves no bytes.  Byte parity is therefore "unpinned by the reference";
 *     it is pinned by construction (plain memcpy over the same slot-run tables) and by
 *     round-trip properties in tests/.
 */
#ifndef KVF_ORACLE_H
#define KVF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- payload identity ------------------------------------ */
uint64_t kvfo_mix64(uint64_t x);
/* content id of token i given the content id of the token before it (prefix hash). */
uint64_t kvfo_next_cid(uint64_t prev_cid, int32_t token);
/* The bf16 bit pattern of element (plane, global head, dim) of the token with content cid. */
uint16_t kvfo_payload_elem(uint64_t cid, uint32_t plane, uint32_t head, uint32_t dim);

typedef struct {
    uint32_t layers, kv_heads, head_dim, head_offset; /* kv_heads = heads held locally */
} kvfo_geom;

/* Write the expected payload of `n` tokens (cids) into pool slots given by runs.
 * pool layout: [plane = layer*2+kv][slot][local head][dim] bf16. */
typedef struct { uint64_t start, len; } kvfo_run;
void kvfo_fill(const kvfo_geom* g, void* pool, uint64_t pool_slots, const kvfo_run* runs, uint32_t n_runs,
               const uint64_t* cids);

/* Plain memcpy restatement of a gather/scatter between two pools (K1/K2/K3 semantics):
 * token k of the logical node (in run order) moves from src slot to dst slot, all planes.
 * threads >= 1 splits the byte segments across pthreads. Returns bytes copied. */
uint64_t kvfo_copy_runs(const kvfo_geom* g, const void* src, uint64_t src_slots, const kvfo_run* src_runs,
                        uint32_t n_src, void* dst, uint64_t dst_slots, const kvfo_run* dst_runs, uint32_t n_dst,
                        int threads);

/* Order-independent 64-bit checksum of a node's bytes in logical order (plane, token, byte). */
uint64_t kvfo_checksum_runs(const kvfo_geom* g, const void* pool, uint64_t pool_slots, const kvfo_run* runs,
                            uint32_t n_runs);
/* Same checksum computed directly from content ids (no buffer): the expected value. */
uint64_t kvfo_checksum_expected(const kvfo_geom* g, const uint64_t* cids, uint64_t n_tokens);

/* ---- decisions ------------------------------------------------------------------ */
/* SoA tree, preorder, index 0 = root (parent -1).  status: 0 IN_GPU 1 BACKUP_IN_CPU
 * 2 LOADING 3 OFFLOADING (radix_cache.hpp:21-28). */
typedef struct {
    uint32_t n;
    const int32_t* parent;
    const uint8_t* status;
    const int32_t* lock;
    const int64_t* rank;
    const double* time;
    const uint64_t* seq;
    const uint64_t* id;
    const uint64_t* tokens;
    const uint8_t* backed;
    uint64_t bytes_per_token;
} kvfo_tree;

/* set_agent_priorities restatement (radix_cache.cpp:266-285): every non-root node SUFFIX,
 * then min(candidate) along each boundary's root path.  out_rank[0] (root) untouched. */
void kvfo_priority(const kvfo_tree* t, const int32_t* boundary_idx, const int64_t* cand, uint32_t m,
                   int64_t* out_rank);

enum { KVFO_ACT_OFFLOAD = 0, KVFO_ACT_DISCARD_TO_BACKUP = 1, KVFO_ACT_REMOVE = 2 };

/* evict restatement (radix_cache.cpp:302-372): greedy min-heap on `before`, parent
 * re-push, per-victim action.  Returns 0, or 13 (ErrorCode::InternalError, errors.hpp:27) when the
 * reference's remove_node would throw ("removing node with children"). */
int kvfo_evict(const kvfo_tree* t, uint64_t needed, int workflow_aware, int offload_mode, int has_floor,
               int64_t floor, uint64_t cpu_used, uint64_t cpu_cap, int32_t* out_idx, uint8_t* out_action,
               uint32_t* out_count, uint64_t* immediate, uint64_t* pending);

/* Wall-clock helper for baselines. */
double kvfo_now(void);

#ifdef __cplusplus
}
#endif
#endif
