// K6 -- decode-side consumer of the slot-run table.
//
// One decode step of GQA attention for a batch of sequences whose KV lives in the engine's
// HBM pool as token-slot runs: the kernel reads K and V of layer `layer` IN PLACE through
// each sequence's run list -- exactly the lists the radix cache hands out after
// match_prefix (proj/src/radix_cache.cpp:88-140) plus the request's own suffix -- so a
// prefetched prefix (K1) feeds attention with no compaction copy (K3) in between.
//
// Why this shape on B200.  Decode attention with GQA group G (4 for Llama-3-8B, 8 for 70B)
// does 4 flop per KV byte: HBM-bound by ~50x on the tensor cores.  tcgen05 needs M >= 64
// rows and only G of them would be live, so the kernel uses the warp-level HMMA path
// (mma.sync m16n8k16 bf16 -> fp32) whose 16-row tile wastes less, and spends its design
// on the bytes: every (token, head) row of K and V is a 256-B line fetched once with
// 16-B cp.async (LDGSTS) straight into a 128-B-XOR-swizzled shared-memory tile (so the
// ldmatrix reads are conflict-free), three 64-token stages in flight per CTA, two CTAs
// per SM.  The slot of every token is resolved once per CTA from the run table
// (binary search in shared memory), which is what makes arbitrary split points
// (radix_cache.cpp:142-177) free for the consumer too.
//
// Work split (flash-decoding): a work item = (sequence, <= chunk tokens, <= kMaxRuns runs);
// grid = items x local KV heads.  Each CTA keeps an online softmax per warp, merges its 4
// warps in shared memory and writes an unnormalised partial (m, l, o[G][128]); a second
// kernel merges a sequence's partials per query head.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "engine_internal.hpp"

using namespace kvf_impl;

namespace {

constexpr int kD = 128;                     // head_dim (Llama-3 8B / 70B)
constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kTokWarp = 16;                // tokens per warp per stage (one m16n8k16 K step)
constexpr int kStageTok = kWarps * kTokWarp;  // 64
constexpr int kStages = 3;
constexpr int kRowBytes = kD * 2;           // one (token, head) row of K or V: 256 B
constexpr int kStageBytes = kStageTok * kRowBytes * 2;  // K + V: 32 KiB
constexpr int kMaxRuns = 64;                // runs one work item may span
constexpr int kMaxChunk = 1024;             // tokens per work item
constexpr int kMaxGroup = 16;               // q heads per kv head (m16 tile rows)
constexpr size_t kSmemBytes = static_cast<size_t>(kStages) * kStageBytes + kMaxChunk * 4 + kMaxRuns * 8;

struct AttnItem {
    uint32_t seq, t0, ntok, r0, nr, pad0, pad1, pad2;  // 32 B
};

struct AttnParams {
    const char* pool;        // HBM pool base
    uint64_t plane_stride;   // bytes between planes
    uint32_t tpb;            // bytes per token per plane (kv_heads_local * 256)
    uint32_t layer;
    uint32_t group, hq;      // q heads per kv head, q heads per sequence (local)
    float scale_log2;        // softmax scale * log2(e)
    const __nv_bfloat16* q;  // [batch][hq][128]
    const AttnItem* items;
    const uint32_t* run_tok;   // token offset of each run within its sequence
    const uint32_t* run_slot;  // first slot of each run
    float* part_o;             // [items][kv_heads_local][group][128]
    float* part_ml;            // [items][kv_heads_local][group][2]
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    const int n = valid ? 16 : 0;  // zero-fill rows past the item's tokens
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
// byte offset of 16-B chunk c of row r inside a [rows][256 B] tile (XOR swizzle on the low 3 bits)
__device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t c) { return r * kRowBytes + ((c ^ (r & 7)) << 4); }

__global__ void __launch_bounds__(kThreads, 2) kvf_attend_kernel(const __grid_constant__ AttnParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* stage_base = smem;
    uint32_t* slot_s = reinterpret_cast<uint32_t*>(smem + kStages * kStageBytes);
    uint32_t* rtok_s = slot_s + kMaxChunk;
    uint32_t* rslot_s = rtok_s + kMaxRuns;

    const AttnItem it = p.items[blockIdx.x];
    const uint32_t head = blockIdx.y;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // ---- resolve the item's token -> slot map once (runs cached in smem, binary search)
    for (uint32_t r = tid; r < it.nr; r += kThreads) {
        rtok_s[r] = p.run_tok[it.r0 + r];
        rslot_s[r] = p.run_slot[it.r0 + r];
    }
    __syncthreads();
    for (uint32_t j = tid; j < it.ntok; j += kThreads) {
        const uint32_t t = it.t0 + j;
        uint32_t lo = 0, hi = it.nr - 1;
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (rtok_s[mid] <= t) lo = mid; else hi = mid - 1;
        }
        slot_s[j] = rslot_s[lo] + (t - rtok_s[lo]);
    }
    __syncthreads();

    const char* kplane = p.pool + static_cast<uint64_t>(2 * p.layer) * p.plane_stride + head * kRowBytes;
    const char* vplane = kplane + p.plane_stride;
    const uint32_t nst = (it.ntok + kStageTok - 1) / kStageTok;
    const uint32_t lc = tid & 15, lr = tid >> 4;  // this thread's 16-B column, first row (8 rows apart)

    auto issue = [&](uint32_t s) {
        uint8_t* kb = stage_base + (s % kStages) * kStageBytes;
        uint8_t* vb = kb + kStageTok * kRowBytes;
#pragma unroll
        for (int i = 0; i < kStageTok / 8; ++i) {
            const uint32_t r = lr + 8 * i, j = s * kStageTok + r;
            const bool ok = j < it.ntok;
            const uint64_t off = static_cast<uint64_t>(ok ? slot_s[j] : slot_s[0]) * p.tpb + lc * 16;
            cp_async16(smem_u32(kb + swz(r, lc)), kplane + off, ok);
            cp_async16(smem_u32(vb + swz(r, lc)), vplane + off, ok);
        }
    };

    // ---- Q fragments (A operand, rows = the group's q heads, zero beyond G), loaded once
    const uint32_t g = lane >> 2, cq = 2 * (lane & 3);
    const __nv_bfloat16* qb = p.q + (static_cast<uint64_t>(it.seq) * p.hq + head * p.group) * kD;
    uint32_t qa[8][4];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const uint32_t d0 = kk * 16 + cq;
        qa[kk][0] = g < p.group ? *reinterpret_cast<const uint32_t*>(qb + g * kD + d0) : 0u;
        qa[kk][1] = g + 8 < p.group ? *reinterpret_cast<const uint32_t*>(qb + (g + 8) * kD + d0) : 0u;
        qa[kk][2] = g < p.group ? *reinterpret_cast<const uint32_t*>(qb + g * kD + d0 + 8) : 0u;
        qa[kk][3] = g + 8 < p.group ? *reinterpret_cast<const uint32_t*>(qb + (g + 8) * kD + d0 + 8) : 0u;
    }

    float acc[16][4];
#pragma unroll
    for (int n = 0; n < 16; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // rows g and g+8

#pragma unroll
    for (uint32_t s = 0; s < kStages - 1; ++s) {
        if (s < nst) issue(s);
        cp_async_commit();
    }
    for (uint32_t s = 0; s < nst; ++s) {
        if (s + kStages - 1 < nst) issue(s + kStages - 1);
        cp_async_commit();
        cp_async_wait<kStages - 1>();
        __syncthreads();
        const uint32_t tbase = s * kStageTok + warp * kTokWarp;  // first token of this warp's slice
        if (tbase < it.ntok) {
            const uint8_t* kb = stage_base + (s % kStages) * kStageBytes;
            const uint8_t* vb = kb + kStageTok * kRowBytes;
            const uint32_t row0 = warp * kTokWarp;
            // S^T tile: 16 q rows x 16 tokens (two n8 tiles), K = 128 dims
            float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
            const uint32_t krow = row0 + (lane & 7) + ((lane >> 4) << 3), kcol = (lane >> 3) & 1;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4(smem_u32(kb + swz(krow, 2 * kk + kcol)), b0, b1, b2, b3);
                mma16816(s0, qa[kk], b0, b1);
                mma16816(s1, qa[kk], b2, b3);
            }
            // online softmax over this 16-token slice (masked tokens -> -inf)
            const uint32_t tA = tbase + cq, tB = tbase + 8 + cq;
            float x[8] = {s0[0], s0[1], s0[2], s0[3], s1[0], s1[1], s1[2], s1[3]};
            const bool v[8] = {tA < it.ntok, tA + 1 < it.ntok, tA < it.ntok, tA + 1 < it.ntok,
                               tB < it.ntok, tB + 1 < it.ntok, tB < it.ntok, tB + 1 < it.ntok};
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = v[i] ? x[i] * p.scale_log2 : -INFINITY;
            float mx0 = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[4], x[5]));
            float mx1 = fmaxf(fmaxf(x[2], x[3]), fmaxf(x[6], x[7]));
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
            }
            const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);  // finite: every slice has a valid token
            const float a0 = exp2f(m0 - n0), a1 = exp2f(m1 - n1);
            m0 = n0;
            m1 = n1;
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = exp2f(x[i] - ((i & 2) ? n1 : n0));
            l0 = l0 * a0 + x[0] + x[1] + x[4] + x[5];
            l1 = l1 * a1 + x[2] + x[3] + x[6] + x[7];
#pragma unroll
            for (int n = 0; n < 16; ++n) {
                acc[n][0] *= a0;
                acc[n][1] *= a0;
                acc[n][2] *= a1;
                acc[n][3] *= a1;
            }
            // P (bf16) as the A operand of P.V: the S accumulator layout maps onto it directly
            const uint32_t pa[4] = {pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]),
                                    pack_bf16(x[6], x[7])};
            const uint32_t vrow = row0 + (lane & 7) + (((lane >> 3) & 1) << 3), vcol = lane >> 4;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(smem_u32(vb + swz(vrow, 2 * j + vcol)), b0, b1, b2, b3);
                mma16816(acc[2 * j], pa, b0, b1);
                mma16816(acc[2 * j + 1], pa, b2, b3);
            }
        }
        __syncthreads();  // the stage buffer is refilled next iteration
    }
    cp_async_wait<0>();
    __syncthreads();

    // ---- merge the 4 warps' partials in shared memory (reusing the stage buffers)
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    float* red_o = reinterpret_cast<float*>(stage_base);              // [warp][16 rows][128]
    float* red_m = red_o + kWarps * 16 * kD;                           // [warp][16]
    float* red_l = red_m + kWarps * 16;
#pragma unroll
    for (int n = 0; n < 16; ++n) {
        const uint32_t d = n * 8 + cq;
        red_o[(warp * 16 + g) * kD + d] = acc[n][0];
        red_o[(warp * 16 + g) * kD + d + 1] = acc[n][1];
        red_o[(warp * 16 + g + 8) * kD + d] = acc[n][2];
        red_o[(warp * 16 + g + 8) * kD + d + 1] = acc[n][3];
    }
    if ((lane & 3) == 0) {
        red_m[warp * 16 + g] = m0;
        red_m[warp * 16 + g + 8] = m1;
        red_l[warp * 16 + g] = l0;
        red_l[warp * 16 + g + 8] = l1;
    }
    __syncthreads();
    const uint64_t pbase = static_cast<uint64_t>(blockIdx.x) * gridDim.y + head;
    for (uint32_t e = tid; e < p.group * kD; e += kThreads) {
        const uint32_t row = e / kD, d = e % kD;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, red_m[w * 16 + row]);
        float o = 0.f, l = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const float mw = red_m[w * 16 + row];
            const float sc = mw == -INFINITY ? 0.f : exp2f(mw - M);
            o += sc * red_o[(w * 16 + row) * kD + d];
            l += sc * red_l[w * 16 + row];
        }
        p.part_o[(pbase * p.group + row) * kD + d] = o;
        if (d == 0) {
            p.part_ml[(pbase * p.group + row) * 2] = M;
            p.part_ml[(pbase * p.group + row) * 2 + 1] = l;
        }
    }
}

// out[b][hq][d] = sum_i e_i o_i / sum_i e_i l_i over the sequence's items, e_i = 2^(m_i - M)
__global__ void __launch_bounds__(kD) kvf_attend_combine_kernel(const float* part_o, const float* part_ml,
                                                                const uint32_t* seq_item0, uint32_t hkv,
                                                                uint32_t group, __nv_bfloat16* out) {
    const uint32_t b = blockIdx.x, hq = blockIdx.y, d = threadIdx.x;
    const uint32_t head = hq / group, row = hq % group;
    const uint32_t i0 = seq_item0[b], i1 = seq_item0[b + 1];
    float M = -INFINITY;
    for (uint32_t i = i0; i < i1; ++i) M = fmaxf(M, part_ml[((static_cast<uint64_t>(i) * hkv + head) * group + row) * 2]);
    float o = 0.f, l = 0.f;
    for (uint32_t i = i0; i < i1; ++i) {
        const uint64_t k = (static_cast<uint64_t>(i) * hkv + head) * group + row;
        const float mi = part_ml[k * 2];
        const float sc = mi == -INFINITY ? 0.f : exp2f(mi - M);
        o += sc * part_o[k * kD + d];
        l += sc * part_ml[k * 2 + 1];
    }
    out[(static_cast<uint64_t>(b) * gridDim.y + hq) * kD + d] = __float2bfloat16_rn(l > 0.f ? o / l : 0.f);
}

}  // namespace

#define KVF_GUARD(e)                                                                               \
    if (!(e)) return set_error(KVF_E_INVALID_ARG, "null engine");                                  \
    std::lock_guard<std::mutex> _lk((e)->mu);                                                      \
    if (cudaSetDevice((e)->device) != cudaSuccess) return set_error(KVF_E_CUDA, "cudaSetDevice failed"); \
    kvf_impl::clear_stale_error(e, __func__)

extern "C" int kvf_decode_attend(kvf_engine* e, uint64_t job_id, uint32_t layer, uint32_t batch, uint32_t group,
                                 const void* q, const kvf_run* runs, const uint32_t* run_counts, float scale,
                                 void* out, uint32_t chunk_tokens) {
    KVF_GUARD(e);
    if (e->geom.head_dim != kD || e->geom.dtype_bytes != 2)
        return set_error(KVF_E_INVALID_ARG, "kvf_decode_attend: head_dim 128, bf16 only");
    if (layer >= e->geom.layers) return set_error(KVF_E_INVALID_ARG, "layer out of range");
    if (group == 0 || group > kMaxGroup) return set_error(KVF_E_INVALID_ARG, "group must be 1..16");
    if (batch == 0) return KVF_OK;
    if (!q || !out || !run_counts) return set_error(KVF_E_INVALID_ARG, "null q / out / run_counts");
    if (e->jobs.count(job_id)) return set_error(KVF_E_INVALID_ARG, "job id " + std::to_string(job_id) + " already in use");
    const uint32_t hkv = e->geom.kv_heads_local, hq = hkv * group;

    // ---- flatten the run tables: per-run (token offset, slot), validated against the pool
    uint64_t nruns = 0, total_tok = 0;
    for (uint32_t b = 0; b < batch; ++b) nruns += run_counts[b];
    if (nruns && !runs) return set_error(KVF_E_INVALID_ARG, "null run list");
    std::vector<uint32_t> rtok(nruns), rslot(nruns);
    std::vector<uint32_t> seq_r0(batch + 1, 0);
    std::vector<uint64_t> seq_len(batch, 0);
    {
        uint64_t k = 0;
        for (uint32_t b = 0; b < batch; ++b) {
            seq_r0[b] = static_cast<uint32_t>(k);
            uint64_t t = 0;
            for (uint32_t r = 0; r < run_counts[b]; ++r, ++k) {
                const kvf_run& x = runs[k];
                if (x.len == 0 || x.start + x.len > e->dev_slots || x.start + x.len < x.start)
                    return set_error(KVF_E_INVALID_ARG, "run out of pool range (or empty)");
                rtok[k] = static_cast<uint32_t>(t);
                rslot[k] = static_cast<uint32_t>(x.start);
                t += x.len;
            }
            if (t >= (1ull << 31)) return set_error(KVF_E_TOO_LARGE, "sequence longer than 2^31 tokens");
            seq_len[b] = t;
            total_tok += t;
        }
        seq_r0[batch] = static_cast<uint32_t>(k);
    }
    if (e->dev_slots >= (1ull << 32)) return set_error(KVF_E_TOO_LARGE, "pool beyond 2^32 slots");
    // ---- work items: <= chunk tokens and <= kMaxRuns runs each (chunk from the SM count)
    uint32_t chunk = chunk_tokens;
    if (chunk == 0) {
        chunk = kMaxChunk;
        const uint64_t want = static_cast<uint64_t>(e->sm_count) * 4;  // 2 CTAs/SM, 2 waves
        while (chunk > kStageTok && ((total_tok + chunk - 1) / chunk) * hkv < want) chunk >>= 1;
    }
    if (chunk < kStageTok || chunk > kMaxChunk || chunk % kStageTok)
        return set_error(KVF_E_INVALID_ARG, "chunk_tokens must be a multiple of 64 in [64, 1024] (0 = auto)");
    std::vector<AttnItem> items;
    std::vector<uint32_t> seq_item0(batch + 1, 0);
    for (uint32_t b = 0; b < batch; ++b) {
        seq_item0[b] = static_cast<uint32_t>(items.size());
        uint32_t r = seq_r0[b];
        const uint32_t rend = seq_r0[b + 1];
        uint64_t t = 0;
        while (t < seq_len[b]) {
            while (r + 1 < rend && rtok[r + 1] <= t) ++r;  // run holding token t
            uint64_t end = std::min<uint64_t>(seq_len[b], t + chunk);
            const uint32_t rlast = std::min<uint32_t>(rend, r + kMaxRuns);  // runs [r, rlast) usable
            if (rlast < rend) end = std::min<uint64_t>(end, rtok[rlast]);
            uint32_t nr = 0;
            while (r + nr < rend && rtok[r + nr] < end) ++nr;
            items.push_back(AttnItem{b, static_cast<uint32_t>(t), static_cast<uint32_t>(end - t), r, nr, 0, 0, 0});
            t = end;
        }
    }
    seq_item0[batch] = static_cast<uint32_t>(items.size());
    const uint64_t nitems = items.size();
    if (nitems > 0x7fffffffull) return set_error(KVF_E_TOO_LARGE, "too many work items");

    // ---- device blob: items | run_tok | run_slot | seq_item0 | partials (o, ml)
    auto al = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
    const size_t b_items = al(nitems * sizeof(AttnItem)), b_rt = al(nruns * 4), b_rs = al(nruns * 4),
                 b_si = al((batch + 1) * 4);
    const size_t b_po = al(nitems * hkv * group * kD * 4), b_pm = al(nitems * hkv * group * 2 * 4);
    const size_t in_bytes = b_items + b_rt + b_rs + b_si;
    Job j;
    // grow the workspace only between calls: cudaFree must not race an in-flight reader
    if (in_bytes + b_po + b_pm > e->ws_att.dev_bytes || in_bytes > e->ws_att.host_bytes) {
        KVF_CUDA(cudaStreamSynchronize(e->s_cmp));
        e->att_upload_pending = false;
        if (int rc = e->ws_att.ensure(in_bytes + b_po + b_pm, in_bytes)) return rc;
    }
    // the pinned staging may still feed the previous call's upload: wait for that copy only
    if (e->att_upload_pending) KVF_CUDA(cudaEventSynchronize(e->att_upload_done));
    char* hs = static_cast<char*>(e->ws_att.host);
    std::memcpy(hs, items.data(), nitems * sizeof(AttnItem));
    std::memcpy(hs + b_items, rtok.data(), nruns * 4);
    std::memcpy(hs + b_items + b_rt, rslot.data(), nruns * 4);
    std::memcpy(hs + b_items + b_rt + b_rs, seq_item0.data(), (batch + 1) * 4);
    char* ds = static_cast<char*>(e->ws_att.dev);
    int rc = begin_job(e, job_id, e->s_cmp, j);
    if (rc) return rc;
    // KV written by fills / K3 scatters on the dev stream must be visible to the reads
    if (e->dev_write_pending) KVF_CUDA(cudaStreamWaitEvent(e->s_cmp, e->dev_write_done, 0));
    KVF_CUDA(cudaMemcpyAsync(ds, hs, in_bytes, cudaMemcpyHostToDevice, e->s_cmp));
    KVF_CUDA(cudaEventRecord(e->att_upload_done, e->s_cmp));
    e->att_upload_pending = true;

    AttnParams prm{};
    prm.pool = e->dev_pool;
    prm.plane_stride = e->dev_slots * e->tpb;
    prm.tpb = static_cast<uint32_t>(e->tpb);
    prm.layer = layer;
    prm.group = group;
    prm.hq = hq;
    prm.scale_log2 = scale * 1.4426950408889634f;
    prm.q = static_cast<const __nv_bfloat16*>(q);
    prm.items = reinterpret_cast<const AttnItem*>(ds);
    prm.run_tok = reinterpret_cast<const uint32_t*>(ds + b_items);
    prm.run_slot = reinterpret_cast<const uint32_t*>(ds + b_items + b_rt);
    const uint32_t* d_seq_item0 = reinterpret_cast<const uint32_t*>(ds + b_items + b_rt + b_rs);
    prm.part_o = reinterpret_cast<float*>(ds + in_bytes);
    prm.part_ml = reinterpret_cast<float*>(ds + in_bytes + b_po);
    if (!e->attend_attr_set) {
        KVF_CUDA(cudaFuncSetAttribute(kvf_attend_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kSmemBytes)));
        e->attend_attr_set = true;
    }
    if (nitems) {
        kvf_attend_kernel<<<dim3(static_cast<uint32_t>(nitems), hkv), kThreads, kSmemBytes, e->s_cmp>>>(prm);
        KVF_CUDA(cudaGetLastError());
        e->stats.kernel_launches++;
    }
    kvf_attend_combine_kernel<<<dim3(batch, hq), kD, 0, e->s_cmp>>>(prm.part_o, prm.part_ml, d_seq_item0, hkv, group,
                                                                   static_cast<__nv_bfloat16*>(out));
    KVF_CUDA(cudaGetLastError());
    e->stats.kernel_launches++;
    j.bytes = total_tok * 2 * e->tpb;  // K + V of one layer, read once
    e->stats.attend_bytes += j.bytes;
    e->stats.attend_calls++;
    return end_job(e, job_id, j);
}
