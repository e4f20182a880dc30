// kvflow host API -- token-segment radix cache (reference: proj/include/kvsim/radix_cache.hpp:1-196).
//
// Same public surface as the reference RadixCache (match_prefix, peek_prefix, insert,
// lock/unlock_root_path, mark_fixed_boundary, boundary_node, set_agent_priorities, evict,
// dump, for_each_node, node_count, gpu_resident_bytes), plus the B200 data plane:
//   * every node carries the token-slot runs of its KV on each tier (dev_runs, host_runs);
//     splits at any token offset split the run lists (no bytes move);
//   * insert() gives new nodes HBM slots and writes their payload (prefill emulation);
//   * set_agent_priorities() runs on the GPU (K4) and evict() takes its victim order from
//     the GPU (K5) over a mirror of the tree kept in HBM (kvf_tree, include/kvflow.h): each
//     node owns a mirror slot, every mutation marks it, and a decision ships only the
//     records of the nodes that changed since the previous one.
// Without an attached Engine the tree still works as a host structure, but priorities and
// eviction throw ErrorCode::NoDevice (there is no CPU decision path).
#pragma once

#include <cstdint>
#include <limits>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "kvflow/engine.hpp"
#include "kvflow/errors.hpp"
#include "kvflow/types.hpp"

namespace kvf {

class TierManager;
class RadixCache;

enum class NodeStatus : uint8_t { InGpu = 0, BackupInCpu = 1, Loading = 2, Offloading = 3 };
const char* status_name(NodeStatus s);
bool is_legal_transition(NodeStatus from, NodeStatus to);

// Eviction rank: larger = more evictable (radix_cache.hpp:30-38 of the reference).
inline constexpr int64_t kRankUnreachable = std::numeric_limits<int64_t>::max() / 4;
inline constexpr int64_t kRankSuffix = std::numeric_limits<int64_t>::max() / 2;
inline int64_t rank_for_step(StepValue s) { return s == kStepUnreachable ? kRankUnreachable : s; }
std::string rank_label(int64_t rank);

enum class EvictionPolicy { Lru, WorkflowAware };
enum class TierMode { Discard, Offload };

struct LastAccess {
    VirtualTime time = 0;
    uint64_t seq = 0;
};

struct CacheNode {
    uint64_t id = 0;
    CacheNode* parent = nullptr;
    std::map<TokenId, std::unique_ptr<CacheNode>> children;  // by first token of the child key
    TokenSeq key;
    NodeStatus status = NodeStatus::InGpu;
    int64_t rank = kRankSuffix;
    LastAccess last_access;
    int lock_count = 0;
    bool cpu_backed = false;
    bool prefetched_unused = false;
    std::set<AgentId> fixed_boundary_for;

    // ---- data plane ----
    RunList dev_runs;       // HBM token slots (InGpu / Offloading; Loading = destination)
    RunList host_runs;      // pinned host token slots (cpu_backed, or Offloading destination)
    uint64_t prefix_cid = 0;  // content id of the token before key[0] (payload identity)
    uint64_t end_cid = 0;     // content id of key.back()

    // ---- HBM mirror bookkeeping (RadixCache) ----
    RadixCache* owner = nullptr;  // the cache whose mirror holds this node
    uint32_t slot = 0;            // its mirror slot (root: 0)
    bool mirror_dirty = false;    // changed since the mirror last heard of it
    uint64_t k4_born = 0;         // K4 requests posted before this node took its slot

    size_t token_count() const { return key.size(); }
    bool is_root() const { return parent == nullptr; }
    bool has_device_child() const;
};

struct MatchResult {
    size_t matched_tokens = 0;
    std::vector<CacheNode*> path;
    CacheNode* partial = nullptr;
    size_t partial_len = 0;
    std::vector<CacheNode*> needed_nodes() const;
};

struct InsertResult {
    std::vector<CacheNode*> path;
    Bytes new_bytes = 0;
    size_t new_nodes = 0;
};

struct EvictedVictim {
    uint64_t node_id = 0;
    Bytes bytes = 0;
    bool immediate = false;
};

struct EvictOutcome {
    std::vector<EvictedVictim> victims;
    Bytes immediate_freed = 0;
    Bytes pending_freed = 0;
    bool sufficient = false;
};

struct EvictRequest {
    Bytes needed = 0;
    EvictionPolicy policy = EvictionPolicy::Lru;
    TierMode mode = TierMode::Discard;
    std::optional<int64_t> rank_floor_exclusive;
};

// Content id chain: cid(token i) = mix(cid(token i-1), token i).  Root seed below.
inline constexpr uint64_t kRootCid = 0x6b766600ULL;
uint64_t next_cid(uint64_t prev, TokenId token);

class RadixCache {
public:
    explicit RadixCache(Bytes bytes_per_token, Engine* engine = nullptr);
    ~RadixCache();

    Bytes bytes_per_token() const { return bpt_; }
    CacheNode& root() { return *root_; }
    const CacheNode& root() const { return *root_; }
    Bytes node_bytes(const CacheNode& n) const { return n.token_count() * bpt_; }
    Engine* engine() const { return engine_; }
    void attach_engine(Engine* e);
    // Prefill emulation (harness / lockstep driver): with no model producing KV, every new
    // segment gets the deterministic synthetic payload in its fresh HBM slots.
    // Off by default: in serving, insert only allocates the slots and the model writes the
    // segment's K/V through kvf_kv_append (include/kvflow.h).
    void set_prefill_emulation(bool on) { emulate_prefill_ = on; }
    bool prefill_emulation() const { return emulate_prefill_; }

    MatchResult match_prefix(const TokenSeq& tokens, VirtualTime now);
    MatchResult peek_prefix(const TokenSeq& tokens) const;
    InsertResult insert(const TokenSeq& tokens, VirtualTime now);
    void lock_root_path(CacheNode* deepest);
    void unlock_root_path(CacheNode* deepest);
    CacheNode* mark_fixed_boundary(const AgentId& agent, const TokenSeq& tokens, size_t fixed_len);
    CacheNode* boundary_node(const AgentId& agent) const;

    // K4 on the GPU: every node SUFFIX, then min(rank_for_step) along boundary root paths.
    void set_agent_priorities(const StepMap& steps);
    // The same, deferred: the boundaries and candidates are captured now and the K4 runs on
    // the GPU ahead of the tree's next K5 (in the same ring slot), or when join_priorities()
    // needs the ranks (observers, dump, the end of a run); a newer call replaces a captured one
    // no reader needed (every K4 recomputes all ranks from scratch).  The host nodes get the
    // ranks from join_priorities(); insert / mark_fixed_boundary read back issued ones first
    // (a split copies the rank).  Until then node.rank is the old one, and the records shipped
    // for nodes that existed when a K4 was issued keep the mirror's rank (KVF_REC_KEEP_RANK).
    void set_agent_priorities_async(const StepMap& steps);
    void join_priorities();
    bool priorities_pending() const { return k4_deferred_ || k4_posts_ > k4_joined_; }
    // A node's mirrored fields changed outside the cache (TierManager: status, cpu_backed).
    void note_changed(CacheNode& n);
    // K5 on the GPU picks the ordered victims; the host applies each action through `tier`.
    EvictOutcome evict(const EvictRequest& req, TierManager& tier, VirtualTime now);

    std::string dump() const;
    template <typename F>
    void for_each_node(F&& f) const {
        // preorder, children in first-token order (same walk as the reference's for_each_impl)
        std::vector<const CacheNode*> stack;
        for (auto it = root_->children.rbegin(); it != root_->children.rend(); ++it) stack.push_back(it->second.get());
        while (!stack.empty()) {
            const CacheNode* n = stack.back();
            stack.pop_back();
            f(*n);
            for (auto it = n->children.rbegin(); it != n->children.rend(); ++it) stack.push_back(it->second.get());
        }
    }
    size_t node_count() const;
    Bytes gpu_resident_bytes() const;

    // Content ids of every token of n (walks the prefix chain of its key).
    std::vector<uint64_t> node_cids(const CacheNode& n) const;
    // Decision-call statistics (host wall time of K4/K5 calls; pack = building the change
    // records; records = node records shipped to the mirror).
    struct DecisionStats {
        uint64_t priority_calls = 0, evict_calls = 0, records = 0;
        uint64_t priority_issued = 0;  // K4s that ran on the GPU (the rest were replaced unread)
        double priority_us = 0, evict_us = 0, pack_us = 0;
        double k4_join_us = 0;  // waiting for queued K4 results (its post is priority_us - this)
        double k5_us = 0;       // inside kvf_tree_victims (post + wait + copy-out)
        double apply_us = 0;    // applying the victims' actions (ledger, tier calls, K2 issue)
    };
    const DecisionStats& decision_stats() const { return dstats_; }

private:
    friend class TierManager;
    CacheNode* new_node(CacheNode* parent, TokenSeq key, VirtualTime now);
    void touch(CacheNode& n, VirtualTime now);
    CacheNode* split_node(CacheNode* node, size_t offset);
    void remove_node(CacheNode* node);
    void drop_boundary_markers(CacheNode* node);
    void require_engine(const char* what) const;
    // mirror slots and change records
    void adopt(CacheNode* n);        // new node: a slot, marked changed
    void release_slot(CacheNode* n);  // removed node: its slot dead (reused after the next decision)
    void mark(CacheNode& n);
    void stamp(CacheNode& n, VirtualTime now);
    kvf_tree* tree();                 // created on first use (the engine may be attached late)
    void flush_records();

    Bytes bpt_;
    Engine* engine_ = nullptr;
    bool emulate_prefill_ = false;
    std::unique_ptr<CacheNode> root_;
    uint64_t next_id_ = 1;
    uint64_t touch_counter_ = 0;
    std::unordered_map<AgentId, CacheNode*, AgentIdHash> boundaries_;

    // the HBM mirror
    kvf_tree* tree_ = nullptr;
    Engine* tree_engine_ = nullptr;
    std::vector<CacheNode*> slot_node_;   // slot -> node (nullptr: dead)
    std::vector<uint32_t> free_slots_;     // min-heap: slots stay dense
    std::vector<uint32_t> freed_pending_;  // freed since the last decision: reusable after it
    std::vector<uint32_t> dirty_;          // slots to ship with the next decision
    std::vector<uint32_t> bslot_;          // K4 request staging (boundary slots, candidate ranks)
    std::vector<int64_t> cand_;
    std::vector<kvf_node_rec> recs_;
    std::vector<uint32_t> chg_slot_, vic_slot_;
    std::vector<int64_t> chg_rank_;
    std::vector<uint8_t> vic_act_;
    // K4 requests issued to the engine / read back so far; the ones in between are queued (at
    // most two, the engine's result buffers), numbered k4_joined_ + 1 .. k4_posts_
    uint64_t k4_posts_ = 0, k4_joined_ = 0;
    bool k4_deferred_ = false;  // a captured K4 (bslot_ / cand_) not issued yet
    void issue_priorities();
    void join_oldest_priorities();
    void join_issued_priorities();
    bool time_follows_seq_ = true;          // every stamp so far had a non-decreasing time
    uint32_t hints_sent_ = ~0u;
    VirtualTime last_stamp_ = -std::numeric_limits<double>::infinity();
    DecisionStats dstats_;
};

size_t update_fixed_heuristic(const std::vector<size_t>& hit_lengths, size_t window = 4);

}  // namespace kvf
