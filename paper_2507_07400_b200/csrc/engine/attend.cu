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
// on the bytes:
//  * one CTA (8 warps, one per SM) covers ALL local KV heads of a token range, so the
//    rows it has in flight are whole contiguous token rows of the pool (2 KiB per token
//    per plane for 8 heads) -- DRAM pages are read densely, not in scattered 256-B pieces;
//  * every (token, head) row of K and V is fetched once with 16-B cp.async (LDGSTS, L1
//    bypass) straight into an XOR-swizzled shared-memory tile, so ldmatrix is
//    bank-conflict free; each warp streams its own 16-token tiles through a private
//    3-stage ring (no CTA barrier in the loop): 8 warps x 2-3 tiles x 8 KiB in flight;
//  * work is sized to ONE wave of CTAs: a decode layer is ~20 us of HBM time, so a second
//    partial wave costs as much as the layer;
//  * the slot of every token is resolved once per CTA from the run table (binary search
//    in shared memory) -- arbitrary radix split points (radix_cache.cpp:142-177) are free
//    for the consumer too;
//  * flash-decoding split: a sequence cut into k > 1 work items writes k unnormalised
//    partials (m, l, o) and a combine kernel, launched with programmatic dependent launch
//    so its launch overlaps the main kernel's tail, merges them; k = 1 writes out directly;
//  * a decode step's layers chain (kvf_decode_attend_layers): every grid releases its
//    dependents as soon as all its CTAs are resident and waits (griddepcontrol.wait) only
//    before its first global write, so layer l+1's CTAs take the SMs layer l's fast CTAs
//    free while its slow ones finish -- the per-SM bandwidth spread of one layer is hidden
//    by the next instead of ending every layer.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <queue>
#include <string>
#include <vector>

#include "engine_internal.hpp"

using namespace kvf_impl;

namespace {

constexpr int kD = 128;                       // head_dim (Llama-3 8B / 70B)
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kTok = 16;                      // tokens per tile (one m16n8k16 K step of P.V)
constexpr int kRowBytes = kD * 2;             // one (token, head) row of K or V: 256 B
constexpr int kTileBytes = kTok * kRowBytes;  // 4 KiB of K (and 4 KiB of V)
constexpr int kStages = 3;                    // per-warp ring depth
constexpr int kWarpRing = kStages * 2 * kTileBytes;  // 24 KiB
constexpr int kMaxRuns = 64;                  // runs one work item may span
constexpr int kMaxChunk = 2048;               // tokens per work item
constexpr int kMaxGroup = 16;                 // q heads per kv head (m16 tile rows)
constexpr int kMaxHeadsCta = 8;               // KV heads one CTA covers
constexpr size_t kSmemBytes = static_cast<size_t>(kWarps) * kWarpRing + kMaxChunk * 4 + kMaxRuns * 8;
constexpr int kRedStride = kD + 8;            // floats per row of the warp-merge buffer
static_assert(kWarps * kWarpRing >= kWarps * 16 * kRedStride * 4 + 2 * kWarps * 16 * 4, "merge buffers reuse the rings");

struct AttnItem {
    uint32_t seq, t0, ntok, r0, nr;
    uint32_t nsib;   // items of this sequence (1: the CTA writes the output itself)
    uint32_t slot0;  // nr == 1: slot of the item's first token (its slots are slot0, slot0 + 1, ...)
    uint32_t pad;    // 32 B
};
constexpr uint32_t kParamItems = 160;  // items that ride in the launch parameters (5 KiB: one wave)

struct AttnParams {
    const char* pool;        // HBM pool base
    uint64_t plane_stride;   // bytes between planes
    uint32_t tpb;            // bytes per token per plane (kv_heads_local * 256)
    uint32_t layer;
    uint32_t group, hq;      // q heads per kv head, q heads per sequence (local)
    uint32_t hkv, hpc;       // local kv heads, kv heads per CTA (divides 8 and hkv)
    float scale_log2;        // softmax scale * log2(e)
    const __nv_bfloat16* q;  // [batch][hq][128]
    __nv_bfloat16* out;      // [batch][hq][128]
    const AttnItem* items;
    const uint32_t* run_tok;   // token offset of each run within its sequence
    const uint32_t* run_slot;  // first slot of each run
    float* part_o;             // [items][hkv][group][128]
    float* part_ml;            // [items][hkv][group][2]
    unsigned long long* trace; // diagnostics (KVF_ATTEND_TRACE): per CTA start, prologue, loop, end, smid
    uint32_t inline_items;     // 1: items[] below (grid <= kParamItems), else p.items in global memory
    AttnItem items_p[kParamItems];
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

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
// byte offset of 16-B chunk c of row r inside a [16 rows][256 B] tile (XOR swizzle, low 3 bits)
__device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t c) { return r * kRowBytes + ((c ^ (r & 7)) << 4); }

__global__ void __launch_bounds__(kThreads, 1) kvf_attend_kernel(const __grid_constant__ AttnParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* slot_s = reinterpret_cast<uint32_t*>(smem + kWarps * kWarpRing);
    uint32_t* rtok_s = slot_s + kMaxChunk;
    uint32_t* rslot_s = rtok_s + kMaxRuns;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned long long t_start = p.trace ? gtime() : 0;
    // the dependent grid (this layer's combine, or the next layer) may be scheduled once every
    // CTA of this one is resident; it waits before it writes anything (see the chain note)
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    // the item comes with the launch (parameter space) unless the grid is very large
    const AttnItem it = p.inline_items ? p.items_p[blockIdx.x] : p.items[blockIdx.x];
    // warp -> (head, sub-stream): the CTA's hpc heads x (8 / hpc) interleaved tile streams
    const uint32_t hl = warp % p.hpc, sub = warp / p.hpc, nsub = kWarps / p.hpc;
    const uint32_t head = blockIdx.y * p.hpc + hl;

    // ---- Q fragments (A operand: rows = the group's q heads, zero beyond G); issued first,
    // they land while the slot map is being resolved
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

    // ---- token -> slot map.  An item inside one run (the common case: runs are long) addresses
    // slot0 + j directly and its first loads leave at once; otherwise the runs are cached in smem
    // and every token's slot is found by binary search
    const bool one_run = it.nr == 1;
    if (!one_run) {
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
    }

    const unsigned long long t_pro = p.trace ? gtime() : 0;
    // ---- per-warp pipeline over tiles sub, sub + nsub, ... of the item, for its head
    const char* kplane = p.pool + static_cast<uint64_t>(2 * p.layer) * p.plane_stride + head * kRowBytes;
    const char* vplane = kplane + p.plane_stride;
    uint8_t* ring = smem + warp * kWarpRing;
    const uint32_t ntiles = (it.ntok + kTok - 1) / kTok;
    const uint32_t mine = sub < ntiles ? (ntiles - sub + nsub - 1) / nsub : 0;
    const uint32_t lc = lane & 15, lr = lane >> 4;  // 16-B column; rows lr, lr+2, ..., lr+14

    auto issue = [&](uint32_t i) {
        uint8_t* kb = ring + (i % kStages) * 2 * kTileBytes;
        uint8_t* vb = kb + kTileBytes;
        const uint32_t tb = (sub + i * nsub) * kTok;
#pragma unroll
        for (int k = 0; k < kTok / 2; ++k) {
            const uint32_t r = lr + 2 * k, j = tb + r;
            const bool ok = j < it.ntok;
            const uint32_t slot = one_run ? it.slot0 + (ok ? j : 0) : slot_s[ok ? j : 0];
            const uint64_t off = static_cast<uint64_t>(slot) * p.tpb + lc * 16;
            cp_async16(smem_u32(kb + swz(r, lc)), kplane + off, ok);
            cp_async16(smem_u32(vb + swz(r, lc)), vplane + off, ok);
        }
    };

    float acc[16][4];
#pragma unroll
    for (int n = 0; n < 16; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // rows g and g+8

#pragma unroll
    for (uint32_t i = 0; i < kStages - 1; ++i) {
        if (i < mine) issue(i);
        cp_async_commit();
    }
    const uint32_t krow = (lane & 7) + ((lane >> 4) << 3), kcol = (lane >> 3) & 1;
    const uint32_t vrow = (lane & 7) + (((lane >> 3) & 1) << 3), vcol = lane >> 4;
    for (uint32_t i = 0; i < mine; ++i) {
        if (i + kStages - 1 < mine) issue(i + kStages - 1);
        cp_async_commit();
        cp_async_wait<kStages - 1>();
        __syncwarp();
        const uint8_t* kb = ring + (i % kStages) * 2 * kTileBytes;
        const uint8_t* vb = kb + kTileBytes;
        const uint32_t tb = (sub + i * nsub) * kTok;
        // S^T tile: 16 q rows x 16 tokens (two n8 tiles), K = 128 dims
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4(smem_u32(kb + swz(krow, 2 * kk + kcol)), b0, b1, b2, b3);
            mma16816(s0, qa[kk], b0, b1);
            mma16816(s1, qa[kk], b2, b3);
        }
        // online softmax over the tile (masked tokens -> -inf; token tb is always valid)
        const uint32_t tA = tb + cq, tB = tb + 8 + cq;
        float x[8] = {s0[0], s0[1], s0[2], s0[3], s1[0], s1[1], s1[2], s1[3]};
        const bool v[8] = {tA < it.ntok, tA + 1 < it.ntok, tA < it.ntok, tA + 1 < it.ntok,
                           tB < it.ntok, tB + 1 < it.ntok, tB < it.ntok, tB + 1 < it.ntok};
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = v[k] ? x[k] * p.scale_log2 : -INFINITY;
        float mx0 = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[4], x[5]));
        float mx1 = fmaxf(fmaxf(x[2], x[3]), fmaxf(x[6], x[7]));
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
        }
        const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
        const float a0 = exp2f(m0 - n0), a1 = exp2f(m1 - n1);
        m0 = n0;
        m1 = n1;
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = exp2f(x[k] - ((k & 2) ? n1 : n0));
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
#pragma unroll
        for (int jn = 0; jn < 8; ++jn) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(smem_u32(vb + swz(vrow, 2 * jn + vcol)), b0, b1, b2, b3);
            mma16816(acc[2 * jn], pa, b0, b1);
            mma16816(acc[2 * jn + 1], pa, b2, b3);
        }
        __syncwarp();  // this ring slot is refilled next iteration
    }
    cp_async_wait<0>();
    // everything above only read (q, the pool, the run tables); before the first write, the
    // grid this one depends on (the previous layer's combine: it still reads the shared
    // partials buffer) must be complete -- a no-op when launched without PDL
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (p.trace) {
        __syncthreads();
        if (tid == 0) {
            unsigned long long* tr = p.trace + (static_cast<uint64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 5;
            uint32_t smid;
            asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
            tr[0] = t_start;
            tr[1] = t_pro;
            tr[2] = gtime();
            tr[4] = smid;
        }
    }

#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    if (nsub == 1) {  // one warp per head (8 local heads): write straight from the accumulators
        const uint64_t rowbase = static_cast<uint64_t>(it.seq) * p.hq + head * p.group;
        const uint64_t pk = (static_cast<uint64_t>(blockIdx.x) * p.hkv + head) * p.group;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const uint32_t row = g + 8 * half;
            if (row >= p.group) continue;
            const float l = half ? l1 : l0, m = half ? m1 : m0;
            const float r = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
            for (int n = 0; n < 16; ++n) {
                const uint32_t d = n * 8 + cq;
                const float a = acc[n][2 * half], b = acc[n][2 * half + 1];
                if (it.nsib == 1)
                    *reinterpret_cast<__nv_bfloat162*>(p.out + (rowbase + row) * kD + d) = __floats2bfloat162_rn(a * r, b * r);
                else
                    *reinterpret_cast<float2*>(&p.part_o[(pk + row) * kD + d]) = make_float2(a, b);
            }
            if (it.nsib != 1 && (lane & 3) == 0) {
                p.part_ml[(pk + row) * 2] = m;
                p.part_ml[(pk + row) * 2 + 1] = l;
            }
        }
        if (p.trace) {
            __syncthreads();
            if (tid == 0) p.trace[(static_cast<uint64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 5 + 3] = gtime();
        }
        return;
    }
    // ---- merge the warps of each head in shared memory (the rings are free once all are here)
    __syncthreads();
    // [warp][16 rows][kRedStride]: the 8-float pad puts the 8 row groups of a float2 store in
    // distinct banks (2 wavefronts per store instead of 8); rows >= group are never stored
    float* red_o = reinterpret_cast<float*>(smem);
    float* red_m = red_o + kWarps * 16 * kRedStride;  // [warp][16]
    float* red_l = red_m + kWarps * 16;
#pragma unroll
    for (int n = 0; n < 16; ++n) {
        const uint32_t d = n * 8 + cq;
        if (g < p.group)
            *reinterpret_cast<float2*>(&red_o[(warp * 16 + g) * kRedStride + d]) = make_float2(acc[n][0], acc[n][1]);
        if (g + 8 < p.group)
            *reinterpret_cast<float2*>(&red_o[(warp * 16 + g + 8) * kRedStride + d]) = make_float2(acc[n][2], acc[n][3]);
    }
    if ((lane & 3) == 0) {
        red_m[warp * 16 + g] = m0;
        red_m[warp * 16 + g + 8] = m1;
        red_l[warp * 16 + g] = l0;
        red_l[warp * 16 + g + 8] = l1;
    }
    __syncthreads();
    // outputs of this CTA: hpc heads x group rows x 128 dims, 4 dims per thread step
    for (uint32_t e = tid; e < p.hpc * p.group * (kD / 4); e += kThreads) {
        const uint32_t h = e / (p.group * (kD / 4)), row = (e / (kD / 4)) % p.group, d = (e % (kD / 4)) * 4;
        float M = -INFINITY;
        for (uint32_t s = 0; s < nsub; ++s) M = fmaxf(M, red_m[(s * p.hpc + h) * 16 + row]);
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        float l = 0.f;
        for (uint32_t s = 0; s < nsub; ++s) {
            const uint32_t w = s * p.hpc + h;
            const float mw = red_m[w * 16 + row];
            const float sc = mw == -INFINITY ? 0.f : exp2f(mw - M);
            const float4 v = *reinterpret_cast<const float4*>(&red_o[(w * 16 + row) * kRedStride + d]);
            o.x += sc * v.x;
            o.y += sc * v.y;
            o.z += sc * v.z;
            o.w += sc * v.w;
            l += sc * red_l[w * 16 + row];
        }
        const uint32_t hg = blockIdx.y * p.hpc + h;
        if (it.nsib == 1) {
            const float r = l > 0.f ? 1.f / l : 0.f;
            __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(
                p.out + ((static_cast<uint64_t>(it.seq) * p.hq + hg * p.group + row) * kD + d));
            ob[0] = __floats2bfloat162_rn(o.x * r, o.y * r);
            ob[1] = __floats2bfloat162_rn(o.z * r, o.w * r);
        } else {
            const uint64_t k = (static_cast<uint64_t>(blockIdx.x) * p.hkv + hg) * p.group + row;
            *reinterpret_cast<float4*>(&p.part_o[k * kD + d]) = o;
            if (d == 0) {
                p.part_ml[k * 2] = M;
                p.part_ml[k * 2 + 1] = l;
            }
        }
    }
    if (p.trace) {
        __syncthreads();
        if (tid == 0) p.trace[(static_cast<uint64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 5 + 3] = gtime();
    }
}

// Merge a sequence's partials per (q head): out = sum_i e_i o_i / sum_i e_i l_i, e_i = 2^(m_i - M).
// Launched as a programmatic dependent of the main kernel: its CTAs become resident next to
// the main kernel's (<= 64 registers: 8 warps x 2 KiB + the main CTA's 48 K registers fill
// one SM's 64 K) and griddepcontrol.wait releases them once the main kernel has completed.
// One CTA per (sequence, q head); its 8 warps split the partials (lane = 4 of the 128 dims),
// so a sequence cut into ~150 items still merges in a few load round trips.
constexpr int kCombWarps = 8;
__global__ void __launch_bounds__(kCombWarps * 32, 4) kvf_attend_combine_kernel(const float* part_o, const float* part_ml,
                                                                            const uint32_t* seq_item0, uint32_t hkv,
                                                                            uint32_t group, __nv_bfloat16* out) {
    __shared__ float4 red_o[kCombWarps][32];
    __shared__ float red_x[kCombWarps], red_l[kCombWarps];
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // next layer: see the chain note
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const uint32_t b = blockIdx.x, hq = blockIdx.y;
    const uint32_t i0 = seq_item0[b], n = seq_item0[b + 1] - i0;
    if (n <= 1) return;  // written by the main kernel (or an empty sequence)
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, head = hq / group, row = hq % group;
    auto key = [&](uint32_t i) { return (static_cast<uint64_t>(i0 + i) * hkv + head) * group + row; };
    // every warp pulls its first kRegs partials into registers at once (independent loads),
    // one block-wide max, then rescales from registers; partials beyond 8 x kRegs (a very long
    // sequence) take a second, load-then-scale pass
    constexpr int kRegs = 6;
    float2 ml[kRegs];
    float4 ov[kRegs];
    float mloc = -INFINITY;
#pragma unroll
    for (int k = 0; k < kRegs; ++k) {
        const uint32_t i = warp + k * kCombWarps;
        ml[k] = make_float2(-INFINITY, 0.f);
        ov[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < n) {
            const uint64_t kk = key(i);
            ml[k] = *reinterpret_cast<const float2*>(part_ml + kk * 2);
            ov[k] = reinterpret_cast<const float4*>(part_o + kk * kD)[lane];
        }
        mloc = fmaxf(mloc, ml[k].x);
    }
    for (uint32_t i = warp + kRegs * kCombWarps; i < n; i += kCombWarps)
        mloc = fmaxf(mloc, part_ml[key(i) * 2]);
    if (lane == 0) red_x[warp] = mloc;
    __syncthreads();
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kCombWarps; ++w) M = fmaxf(M, red_x[w]);
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    float l = 0.f;
#pragma unroll
    for (int k = 0; k < kRegs; ++k) {
        const float sc = ml[k].x == -INFINITY ? 0.f : exp2f(ml[k].x - M);
        o.x += sc * ov[k].x;
        o.y += sc * ov[k].y;
        o.z += sc * ov[k].z;
        o.w += sc * ov[k].w;
        l += sc * ml[k].y;
    }
#pragma unroll 4
    for (uint32_t i = warp + kRegs * kCombWarps; i < n; i += kCombWarps) {
        const uint64_t k = key(i);
        const float2 m2 = *reinterpret_cast<const float2*>(part_ml + k * 2);
        const float sc = m2.x == -INFINITY ? 0.f : exp2f(m2.x - M);
        const float4 v = reinterpret_cast<const float4*>(part_o + k * kD)[lane];
        o.x += sc * v.x;
        o.y += sc * v.y;
        o.z += sc * v.z;
        o.w += sc * v.w;
        l += sc * m2.y;
    }
    red_o[warp][lane] = o;
    if (lane == 0) red_l[warp] = l;
    __syncthreads();
    if (warp) return;
    o = red_o[0][lane];
    l = red_l[0];
#pragma unroll
    for (int w = 1; w < kCombWarps; ++w) {
        const float4 v = red_o[w][lane];
        o.x += v.x;
        o.y += v.y;
        o.z += v.z;
        o.w += v.w;
        l += red_l[w];
    }
    const float r = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat162* ob =
        reinterpret_cast<__nv_bfloat162*>(out + (static_cast<uint64_t>(b) * hkv * group + hq) * kD + lane * 4);
    ob[0] = __floats2bfloat162_rn(o.x * r, o.y * r);
    ob[1] = __floats2bfloat162_rn(o.z * r, o.w * r);
}

// sequences with no tokens: out = 0 (softmax over an empty set has no value)
__global__ void kvf_attend_zero_kernel(const uint32_t* empty, uint32_t n, uint32_t hq, __nv_bfloat16* out) {
    const uint64_t per = static_cast<uint64_t>(hq) * kD;
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n * per;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[empty[k / per] * per + k % per] = __float2bfloat16_rn(0.f);
}

// One job: layers layer0 .. layer0 + nlayers - 1 of a decode step over the same run tables
// (q[l] / out[l] per layer).  Called with the engine lock held (KVF_GUARD).
int attend_impl(kvf_engine* e, uint64_t job_id, uint32_t layer0, uint32_t nlayers, uint32_t batch, uint32_t group,
                const void* const* qs, const kvf_run* runs, const uint32_t* run_counts, float scale, void* const* outs,
                uint32_t chunk_tokens) {
    if (e->geom.head_dim != kD || e->geom.dtype_bytes != 2)
        return set_error(KVF_E_INVALID_ARG, "kvf_decode_attend: head_dim 128, bf16 only");
    if (nlayers == 0 || layer0 >= e->geom.layers || nlayers > e->geom.layers - layer0)
        return set_error(KVF_E_INVALID_ARG, "layer out of range");
    if (group == 0 || group > kMaxGroup) return set_error(KVF_E_INVALID_ARG, "group must be 1..16");
    if (chunk_tokens && (chunk_tokens % kTok || chunk_tokens > kMaxChunk))
        return set_error(KVF_E_INVALID_ARG, "chunk_tokens must be a multiple of 16 in [16, 2048] (0 = auto)");
    if (batch == 0) return KVF_OK;
    if (!qs || !outs || !run_counts) return set_error(KVF_E_INVALID_ARG, "null q / out / run_counts");
    for (uint32_t l = 0; l < nlayers; ++l) {
        if (!qs[l] || !outs[l]) return set_error(KVF_E_INVALID_ARG, "null q / out / run_counts");
        if ((reinterpret_cast<uintptr_t>(qs[l]) | reinterpret_cast<uintptr_t>(outs[l])) & 3)
            return set_error(KVF_E_INVALID_ARG, "q and out must be 4-byte aligned");
    }
    if (e->jobs.count(job_id)) return set_error(KVF_E_INVALID_ARG, "job id " + std::to_string(job_id) + " already in use");
    const uint32_t hkv = e->geom.kv_heads_local, hq = hkv * group;
    // KV heads per CTA.  A single-layer call takes 2 (more, shorter items per sequence: the
    // wave ends more evenly -- C2 2 x 8320 23.0 -> 21.2 us, C4 64 x 1792 88.7 -> 78.3 us per call);
    // a PDL-chained step keeps all of the shard's heads (dense 2 KiB token rows; the chain
    // already hides the wave's end: C2 13.1 us per layer vs 13.6 with 2).
    // scripts/attend_hpc_sweep.py, profiles/r02_attend_hpc_sweep.json
    uint32_t hpc = std::gcd(hkv, static_cast<uint32_t>(nlayers == 1 ? 2 : kMaxHeadsCta));
    if (const char* f = std::getenv("KVF_ATTEND_HPC")) {  // sweep knob
        const uint32_t want = static_cast<uint32_t>(std::atoi(f));
        if (want && std::gcd(hkv, static_cast<uint32_t>(kMaxHeadsCta)) % want == 0) hpc = want;
    }
    const uint32_t ygrid = hkv / hpc;
    if (ygrid > 65535 || batch >= (1u << 31) || hq > 65535)
        return set_error(KVF_E_TOO_LARGE, "batch or head count too large");

    uint64_t nruns = 0;
    for (uint32_t b = 0; b < batch; ++b) nruns += run_counts[b];
    if (nruns && !runs) return set_error(KVF_E_INVALID_ARG, "null run list");
    // ---- descriptor cache: a decode step calls K6 once per layer with the same run tables
    std::vector<uint64_t> sig;
    sig.reserve(4 + batch + 2 * nruns);
    sig.push_back(batch);
    sig.push_back(group);
    sig.push_back(chunk_tokens);
    sig.push_back(hpc);
    for (uint32_t b = 0; b < batch; ++b) sig.push_back(run_counts[b]);
    for (uint64_t k = 0; k < nruns; ++k) {
        sig.push_back(runs[k].start);
        sig.push_back(runs[k].len);
    }
    const bool hit = sig == e->att_sig;
    uint64_t* meta = e->att_meta;  // nitems, total_tok, in_bytes, b_items, b_rt, b_rs, b_si, b_po, nempty, multi
    Job j;
    if (!hit) {
        if (e->dev_slots >= (1ull << 32)) return set_error(KVF_E_TOO_LARGE, "pool beyond 2^32 slots");
        // ---- flatten the run tables: per-run (token offset, slot), validated against the pool
        uint64_t total_tok = 0;
        std::vector<uint32_t> rtok(nruns), rslot(nruns), seq_r0(batch + 1, 0), empty;
        std::vector<uint64_t> seq_len(batch, 0);
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
            if (t == 0) empty.push_back(b);
        }
        seq_r0[batch] = static_cast<uint32_t>(k);
        // ---- work items: one wave of resident CTAs, balanced -- a decode layer is ~20 us of
        // HBM time, so a second partial wave costs as much as the whole layer
        if (!e->attend_occ) {
            int occ = 0;
            KVF_CUDA(cudaFuncSetAttribute(kvf_attend_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(kSmemBytes)));
            KVF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kvf_attend_kernel, kThreads, kSmemBytes));
            e->attend_occ = std::max(1, occ);
            e->attend_attr_set = true;
        }
        std::vector<uint64_t> kseq(batch, 0);  // items per sequence
        if (chunk_tokens) {
            for (uint32_t b = 0; b < batch; ++b) kseq[b] = (seq_len[b] + chunk_tokens - 1) / chunk_tokens;
        } else if (total_tok) {
            const uint64_t slots = static_cast<uint64_t>(e->sm_count) * e->attend_occ;
            // >= 64 tokens per item: below that the CTA prologue outweighs its bytes
            const double T = std::max(64.0, static_cast<double>(total_tok) * ygrid / static_cast<double>(slots));
            uint64_t used = 0;
            for (uint32_t b = 0; b < batch; ++b) {
                if (!seq_len[b]) continue;
                kseq[b] = std::max<uint64_t>({1, static_cast<uint64_t>(seq_len[b] / T),
                                              (seq_len[b] + kMaxChunk - 1) / kMaxChunk});
                used += kseq[b] * ygrid;
            }
            // spend what is left of the wave on the sequences with the largest items
            std::priority_queue<std::pair<double, uint32_t>> pq;
            for (uint32_t b = 0; b < batch; ++b)
                if (seq_len[b] >= 64 * (kseq[b] + 1)) pq.push({static_cast<double>(seq_len[b]) / kseq[b], b});
            while (used + ygrid <= slots && !pq.empty()) {
                const uint32_t b = pq.top().second;
                pq.pop();
                ++kseq[b];
                used += ygrid;
                if (seq_len[b] >= 64 * (kseq[b] + 1)) pq.push({static_cast<double>(seq_len[b]) / kseq[b], b});
            }
        }
        std::vector<AttnItem> items;
        std::vector<uint32_t> seq_item0(batch + 1, 0);
        bool multi = false;
        for (uint32_t b = 0; b < batch; ++b) {
            seq_item0[b] = static_cast<uint32_t>(items.size());
            if (!seq_len[b]) continue;
            const uint64_t kb = kseq[b];
            const uint64_t per = std::min<uint64_t>(kMaxChunk, ((seq_len[b] + kb - 1) / kb + kTok - 1) / kTok * kTok);
            const size_t first = items.size();
            uint32_t r = seq_r0[b];
            const uint32_t rend = seq_r0[b + 1];
            uint64_t t = 0;
            while (t < seq_len[b]) {
                while (r + 1 < rend && rtok[r + 1] <= t) ++r;  // run holding token t
                uint64_t end = std::min<uint64_t>(seq_len[b], t + per);
                if (r + kMaxRuns < rend) end = std::min<uint64_t>(end, rtok[r + kMaxRuns]);
                uint32_t nr = 0;
                while (r + nr < rend && rtok[r + nr] < end) ++nr;
                items.push_back(AttnItem{b, static_cast<uint32_t>(t), static_cast<uint32_t>(end - t), r, nr, 0,
                                         rslot[r] + static_cast<uint32_t>(t - rtok[r]), 0});
                t = end;
            }
            for (size_t i = first; i < items.size(); ++i) items[i].nsib = static_cast<uint32_t>(items.size() - first);
            multi |= items.size() - first > 1;
        }
        seq_item0[batch] = static_cast<uint32_t>(items.size());
        const uint64_t nitems = items.size();
        if (nitems > 0x7fffffffull) return set_error(KVF_E_TOO_LARGE, "too many work items");

        // ---- device blob: items | run_tok | run_slot | seq_item0 | empty seqs | partials (o, ml)
        auto al = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
        const size_t b_items = al(nitems * sizeof(AttnItem)), b_rt = al(nruns * 4), b_rs = al(nruns * 4),
                     b_si = al((batch + 1) * 4), b_em = al(empty.size() * 4);
        const size_t b_po = multi ? al(nitems * hkv * group * kD * 4) : 0;
        const size_t b_pm = multi ? al(nitems * hkv * group * 2 * 4) : 0;
        const size_t in_bytes = b_items + b_rt + b_rs + b_si + b_em;
        const size_t dev_need = in_bytes + b_po + b_pm;
        // grow the workspace only between calls: cudaFree must not race an in-flight reader
        if (dev_need > e->ws_att.dev_bytes || in_bytes > e->ws_att.host_bytes) {
            KVF_CUDA(cudaStreamSynchronize(e->s_cmp));
            e->att_upload_pending = false;
            if (int rc = e->ws_att.ensure(dev_need, in_bytes)) return rc;
        }
        // the pinned staging may still feed the previous call's upload: wait for that copy only
        if (e->att_upload_pending) KVF_CUDA(cudaEventSynchronize(e->att_upload_done));
        char* hs = static_cast<char*>(e->ws_att.host);
        std::memcpy(hs, items.data(), nitems * sizeof(AttnItem));
        e->att_items.assign(reinterpret_cast<const uint8_t*>(items.data()),
                            reinterpret_cast<const uint8_t*>(items.data() + nitems));
        std::memcpy(hs + b_items, rtok.data(), nruns * 4);
        std::memcpy(hs + b_items + b_rt, rslot.data(), nruns * 4);
        std::memcpy(hs + b_items + b_rt + b_rs, seq_item0.data(), (batch + 1) * 4);
        std::memcpy(hs + b_items + b_rt + b_rs + b_si, empty.data(), empty.size() * 4);
        e->att_sig.clear();  // invalid until the upload below is enqueued
        int rc = begin_job(e, job_id, e->s_cmp, j);
        if (rc) return rc;
        KVF_CUDA(cudaMemcpyAsync(e->ws_att.dev, hs, in_bytes, cudaMemcpyHostToDevice, e->s_cmp));
        KVF_CUDA(cudaEventRecord(e->att_upload_done, e->s_cmp));
        e->att_upload_pending = true;
        e->att_sig.swap(sig);
        const uint64_t m[10] = {nitems, total_tok, in_bytes, b_items, b_rt, b_rs, b_si, b_po, empty.size(), multi};
        std::copy(m, m + 10, meta);
    } else {
        int rc = begin_job(e, job_id, e->s_cmp, j);
        if (rc) return rc;
    }
    // KV written by fills / K3 scatters on the dev stream must be visible to the reads
    if (e->dev_write_pending) KVF_CUDA(cudaStreamWaitEvent(e->s_cmp, e->dev_write_done, 0));
    const uint64_t nitems = meta[0], total_tok = meta[1], in_bytes = meta[2], b_items = meta[3], b_rt = meta[4],
                   b_rs = meta[5], b_si = meta[6], b_po = meta[7], nempty = meta[8], multi = meta[9];
    char* ds = static_cast<char*>(e->ws_att.dev);

    AttnParams prm{};
    prm.pool = e->dev_pool;
    prm.plane_stride = e->dev_slots * e->tpb;
    prm.tpb = static_cast<uint32_t>(e->tpb);
    prm.group = group;
    prm.hq = hq;
    prm.hkv = hkv;
    prm.hpc = hpc;
    prm.scale_log2 = scale * 1.4426950408889634f;
    prm.items = reinterpret_cast<const AttnItem*>(ds);
    if (nitems <= kParamItems) {  // one wave: the items travel with the launch
        prm.inline_items = 1;
        std::memcpy(prm.items_p, e->att_items.data(), nitems * sizeof(AttnItem));
    }
    prm.run_tok = reinterpret_cast<const uint32_t*>(ds + b_items);
    prm.run_slot = reinterpret_cast<const uint32_t*>(ds + b_items + b_rt);
    const uint32_t* d_seq_item0 = reinterpret_cast<const uint32_t*>(ds + b_items + b_rt + b_rs);
    const uint32_t* d_empty = reinterpret_cast<const uint32_t*>(ds + b_items + b_rt + b_rs + b_si);
    prm.part_o = reinterpret_cast<float*>(ds + in_bytes);
    prm.part_ml = reinterpret_cast<float*>(ds + in_bytes + b_po);
    if (!e->attend_attr_set) {
        KVF_CUDA(cudaFuncSetAttribute(kvf_attend_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kSmemBytes)));
        e->attend_attr_set = true;
    }
    static const char* trace_path = std::getenv("KVF_ATTEND_TRACE");
    unsigned long long* d_trace = nullptr;
    if (trace_path && nitems && nlayers == 1) {
        KVF_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_trace), nitems * ygrid * 5 * 8, e->s_cmp));
        prm.trace = d_trace;
    }
    // the layer chain: attend(l) -> combine(l) -> attend(l + 1) -> ..., every launch after the
    // first a programmatic dependent of the one before it (kernel-side protocol: see the top)
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    for (uint32_t l = 0; l < nlayers; ++l) {
        prm.layer = layer0 + l;
        prm.q = static_cast<const __nv_bfloat16*>(qs[l]);
        prm.out = static_cast<__nv_bfloat16*>(outs[l]);
        if (nitems) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(static_cast<uint32_t>(nitems), ygrid);
            cfg.blockDim = dim3(kThreads);
            cfg.dynamicSmemBytes = kSmemBytes;
            cfg.stream = e->s_cmp;
            cfg.attrs = pdl;
            cfg.numAttrs = l ? 1 : 0;
            KVF_CUDA(cudaLaunchKernelEx(&cfg, kvf_attend_kernel, prm));
            e->stats.kernel_launches++;
        }
        if (multi) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(batch, hq);
            cfg.blockDim = dim3(kCombWarps * 32);
            cfg.stream = e->s_cmp;
            cfg.attrs = pdl;
            cfg.numAttrs = 1;
            KVF_CUDA(cudaLaunchKernelEx(&cfg, kvf_attend_combine_kernel, static_cast<const float*>(prm.part_o),
                                        static_cast<const float*>(prm.part_ml), d_seq_item0, hkv, group, prm.out));
            e->stats.kernel_launches++;
        }
    }
    // empty sequences (rows no other kernel writes): after the chain
    for (uint32_t l = 0; nempty && l < nlayers; ++l) {
        kvf_attend_zero_kernel<<<static_cast<uint32_t>(std::min<uint64_t>(1024, (nempty * hq * kD + 255) / 256)), 256, 0,
                                 e->s_cmp>>>(d_empty, static_cast<uint32_t>(nempty), hq,
                                             static_cast<__nv_bfloat16*>(outs[l]));
        KVF_CUDA(cudaGetLastError());
        e->stats.kernel_launches++;
    }
    if (d_trace) {  // diagnostics only: synchronous dump, one line per call
        std::vector<unsigned long long> tr(nitems * ygrid * 5);
        KVF_CUDA(cudaMemcpyAsync(tr.data(), d_trace, tr.size() * 8, cudaMemcpyDeviceToHost, e->s_cmp));
        KVF_CUDA(cudaStreamSynchronize(e->s_cmp));
        KVF_CUDA(cudaFree(d_trace));
        if (FILE* f = std::fopen(trace_path, "a")) {
            std::fprintf(f, "[");
            for (size_t i = 0; i < tr.size(); i += 5)
                std::fprintf(f, "%s[%llu,%llu,%llu,%llu,%llu]", i ? "," : "", tr[i], tr[i + 1], tr[i + 2], tr[i + 3],
                             tr[i + 4]);
            std::fprintf(f, "]\n");
            std::fclose(f);
        }
    }
    j.bytes = total_tok * 2 * e->tpb * nlayers;  // K + V of each layer, read once
    e->stats.attend_bytes += j.bytes;
    e->stats.attend_calls += nlayers;
    return end_job(e, job_id, j);
}

}  // namespace

extern "C" int kvf_decode_attend(kvf_engine* e, uint64_t job_id, uint32_t layer, uint32_t batch, uint32_t group,
                                 const void* q, const kvf_run* runs, const uint32_t* run_counts, float scale,
                                 void* out, uint32_t chunk_tokens) {
    KVF_GUARD(e);
    return attend_impl(e, job_id, layer, 1, batch, group, &q, runs, run_counts, scale, &out, chunk_tokens);
}

extern "C" int kvf_decode_attend_layers(kvf_engine* e, uint64_t job_id, uint32_t layer0, uint32_t nlayers,
                                        uint32_t batch, uint32_t group, const void* const* q, const kvf_run* runs,
                                        const uint32_t* run_counts, float scale, void* const* out,
                                        uint32_t chunk_tokens) {
    KVF_GUARD(e);
    return attend_impl(e, job_id, layer0, nlayers, batch, group, q, runs, run_counts, scale, out, chunk_tokens);
}

namespace kvf_impl {
void set_carveout_attend() {
    cudaFuncSetAttribute(kvf_attend_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(kvf_attend_combine_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(kvf_attend_zero_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
}
}  // namespace kvf_impl
