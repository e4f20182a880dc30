/* kvf_oracle.c -- CPU restatement of the KVFlow KV-movement hot path.
 * TEST INFRASTRUCTURE ONLY (see kvf_oracle.h).  Plain C, single-threaded except the
 * memcpy restatement used as the CPU baseline. */
#define _GNU_SOURCE
#include "kvf_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------ payload --------- */
/* splitmix64 finaliser (public-domain constants). */
uint64_t kvfo_mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

uint64_t kvfo_next_cid(uint64_t prev, int32_t token) {
    return kvfo_mix64(prev + 0x9e3779b97f4a7c15ULL * ((uint64_t)(uint32_t)token + 1ULL));
}

static uint64_t head_base(uint64_t cid, uint32_t plane, uint32_t head) {
    return kvfo_mix64(cid ^ ((uint64_t)plane * 0x100000001b3ULL) ^ ((uint64_t)head << 48));
}

/* One 64-bit payload word = 4 consecutive bf16 elements (dims 4w..4w+3), exponent MSB
 * cleared so every element is a finite bf16. */
static uint64_t payload_word(uint64_t base, uint32_t w) {
    return kvfo_mix64(base + (uint64_t)w) & 0xBFFFBFFFBFFFBFFFULL;
}

uint16_t kvfo_payload_elem(uint64_t cid, uint32_t plane, uint32_t head, uint32_t dim) {
    uint64_t w = payload_word(head_base(cid, plane, head), dim / 4);
    return (uint16_t)(w >> (16 * (dim % 4)));
}

static uint64_t tpb_of(const kvfo_geom* g) { return (uint64_t)g->kv_heads * g->head_dim * 2; }

void kvfo_fill(const kvfo_geom* g, void* pool, uint64_t pool_slots, const kvfo_run* runs, uint32_t n_runs,
               const uint64_t* cids) {
    const uint64_t tpb = tpb_of(g);
    const uint32_t planes = g->layers * 2;
    uint64_t k = 0;
    for (uint32_t r = 0; r < n_runs; ++r) {
        for (uint64_t t = 0; t < runs[r].len; ++t, ++k) {
            uint64_t slot = runs[r].start + t;
            for (uint32_t p = 0; p < planes; ++p) {
                uint64_t* dst = (uint64_t*)((char*)pool + ((uint64_t)p * pool_slots + slot) * tpb);
                for (uint32_t h = 0; h < g->kv_heads; ++h) {
                    uint64_t base = head_base(cids[k], p, g->head_offset + h);
                    for (uint32_t w = 0; w < g->head_dim / 4; ++w) dst[h * (g->head_dim / 4) + w] = payload_word(base, w);
                }
            }
        }
    }
}

/* ------------------------------------------------------------- copies --------- */
typedef struct {
    uint64_t src_slot, dst_slot, len;
} piece_t;

/* Merge-walk two run lists into pieces contiguous on both sides. */
static piece_t* make_pieces(const kvfo_run* a, uint32_t na, const kvfo_run* b, uint32_t nb, uint32_t* np) {
    piece_t* out = (piece_t*)malloc(sizeof(piece_t) * (na + nb + 1));
    uint32_t i = 0, j = 0, n = 0;
    uint64_t ao = 0, bo = 0;
    while (i < na && j < nb) {
        uint64_t ar = a[i].len - ao, br = b[j].len - bo;
        uint64_t l = ar < br ? ar : br;
        if (l) out[n++] = (piece_t){a[i].start + ao, b[j].start + bo, l};
        ao += l;
        bo += l;
        if (ao == a[i].len) { ++i; ao = 0; }
        if (bo == b[j].len) { ++j; bo = 0; }
    }
    *np = n;
    return out;
}

typedef struct {
    const char* src;
    char* dst;
    uint64_t src_slots, dst_slots, tpb;
    uint32_t planes;
    const piece_t* pieces;
    uint32_t np;
    uint64_t first, last; /* segment range [first, last) in (piece-major, plane) order */
} copy_job_t;

static void* copy_worker(void* arg) {
    copy_job_t* j = (copy_job_t*)arg;
    for (uint64_t s = j->first; s < j->last; ++s) {
        const piece_t* pc = &j->pieces[s / j->planes];
        uint32_t p = (uint32_t)(s % j->planes);
        memcpy(j->dst + ((uint64_t)p * j->dst_slots + pc->dst_slot) * j->tpb,
               j->src + ((uint64_t)p * j->src_slots + pc->src_slot) * j->tpb, pc->len * j->tpb);
    }
    return NULL;
}

uint64_t kvfo_copy_runs(const kvfo_geom* g, const void* src, uint64_t src_slots, const kvfo_run* src_runs,
                        uint32_t n_src, void* dst, uint64_t dst_slots, const kvfo_run* dst_runs, uint32_t n_dst,
                        int threads) {
    uint32_t np = 0;
    piece_t* pcs = make_pieces(src_runs, n_src, dst_runs, n_dst, &np);
    const uint32_t planes = g->layers * 2;
    const uint64_t tpb = tpb_of(g);
    uint64_t segs = (uint64_t)np * planes, bytes = 0;
    for (uint32_t i = 0; i < np; ++i) bytes += pcs[i].len * tpb * planes;
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > segs) threads = (int)(segs ? segs : 1);
    copy_job_t* jobs = (copy_job_t*)calloc((size_t)threads, sizeof(copy_job_t));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (copy_job_t){(const char*)src, (char*)dst, src_slots, dst_slots, tpb, planes, pcs, np,
                               segs * (uint64_t)t / (uint64_t)threads, segs * (uint64_t)(t + 1) / (uint64_t)threads};
        if (threads > 1) pthread_create(&th[t], NULL, copy_worker, &jobs[t]);
    }
    if (threads > 1)
        for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    else
        copy_worker(&jobs[0]);
    free(th);
    free(jobs);
    free(pcs);
    return bytes;
}

static uint64_t ck_term(uint64_t word, uint64_t idx) { return kvfo_mix64(word ^ (idx * 0x9e3779b97f4a7c15ULL)); }

uint64_t kvfo_checksum_runs(const kvfo_geom* g, const void* pool, uint64_t pool_slots, const kvfo_run* runs,
                            uint32_t n_runs) {
    const uint64_t tpb = tpb_of(g), wpt = tpb / 8;
    const uint32_t planes = g->layers * 2;
    uint64_t ntok = 0;
    for (uint32_t r = 0; r < n_runs; ++r) ntok += runs[r].len;
    uint64_t sum = 0;
    for (uint32_t p = 0; p < planes; ++p) {
        uint64_t t = 0;
        for (uint32_t r = 0; r < n_runs; ++r)
            for (uint64_t i = 0; i < runs[r].len; ++i, ++t) {
                const uint64_t* w = (const uint64_t*)((const char*)pool + ((uint64_t)p * pool_slots + runs[r].start + i) * tpb);
                for (uint64_t k = 0; k < wpt; ++k) sum += ck_term(w[k], ((uint64_t)p * ntok + t) * wpt + k);
            }
    }
    return sum;
}

uint64_t kvfo_checksum_expected(const kvfo_geom* g, const uint64_t* cids, uint64_t ntok) {
    const uint32_t planes = g->layers * 2, wph = g->head_dim / 4;
    const uint64_t wpt = (uint64_t)g->kv_heads * wph;
    uint64_t sum = 0;
    for (uint32_t p = 0; p < planes; ++p)
        for (uint64_t t = 0; t < ntok; ++t)
            for (uint32_t h = 0; h < g->kv_heads; ++h) {
                uint64_t base = head_base(cids[t], p, g->head_offset + h);
                for (uint32_t w = 0; w < wph; ++w)
                    sum += ck_term(payload_word(base, w), ((uint64_t)p * ntok + t) * wpt + (uint64_t)h * wph + w);
            }
    return sum;
}

/* ----------------------------------------------------------- decisions -------- */
#define RANK_SUFFIX ((int64_t)(INT64_MAX / 2))

void kvfo_priority(const kvfo_tree* t, const int32_t* bidx, const int64_t* cand, uint32_t m, int64_t* out) {
    /* radix_cache.cpp:268-275: pass 1, every non-root node is a suffix */
    for (uint32_t i = 1; i < t->n; ++i) out[i] = RANK_SUFFIX;
    /* radix_cache.cpp:278-284: pass 2, min along each boundary's root path */
    for (uint32_t b = 0; b < m; ++b)
        for (int32_t v = bidx[b]; v > 0; v = t->parent[v])
            if (cand[b] < out[v]) out[v] = cand[b];
}

typedef struct {
    const kvfo_tree* t;
    int wa;
} ord_ctx;

/* radix_cache.cpp:316-321 `before` */
static int before(const ord_ctx* c, int32_t a, int32_t b) {
    const kvfo_tree* t = c->t;
    if (c->wa && t->rank[a] != t->rank[b]) return t->rank[a] > t->rank[b];
    if (t->time[a] != t->time[b]) return t->time[a] < t->time[b];
    if (t->seq[a] != t->seq[b]) return t->seq[a] < t->seq[b];
    return t->id[a] < t->id[b];
}

static void heap_push(const ord_ctx* c, int32_t* h, uint32_t* n, int32_t v) {
    uint32_t i = (*n)++;
    h[i] = v;
    while (i > 0) {
        uint32_t p = (i - 1) / 2;
        if (!before(c, h[i], h[p])) break;
        int32_t x = h[i]; h[i] = h[p]; h[p] = x;
        i = p;
    }
}

static int32_t heap_pop(const ord_ctx* c, int32_t* h, uint32_t* n) {
    int32_t top = h[0];
    h[0] = h[--(*n)];
    uint32_t i = 0;
    for (;;) {
        uint32_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && before(c, h[l], h[m])) m = l;
        if (r < *n && before(c, h[r], h[m])) m = r;
        if (m == i) break;
        int32_t x = h[i]; h[i] = h[m]; h[m] = x;
        i = m;
    }
    return top;
}

int kvfo_evict(const kvfo_tree* t, uint64_t needed, int wa, int offload, int has_floor, int64_t floor,
               uint64_t cpu_used, uint64_t cpu_cap, int32_t* out_idx, uint8_t* out_action, uint32_t* out_count,
               uint64_t* immediate, uint64_t* pending) {
    const uint32_t n = t->n;
    uint8_t* st = (uint8_t*)malloc(n);
    uint8_t* removed = (uint8_t*)calloc(n, 1);
    uint32_t* devkids = (uint32_t*)calloc(n, sizeof(uint32_t)); /* children with status != BACKUP */
    uint32_t* kids = (uint32_t*)calloc(n, sizeof(uint32_t));    /* live children (remove_node check) */
    int32_t* heap = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
    memcpy(st, t->status, n);
    for (uint32_t i = 1; i < n; ++i) {
        kids[t->parent[i]]++;
        if (st[i] != 1) devkids[t->parent[i]]++;
    }
    ord_ctx c = {t, wa};
    /* radix_cache.cpp:305-312 evictable */
#define EVICTABLE(v) ((v) > 0 && !removed[v] && t->lock[v] == 0 && st[v] == 0 && devkids[v] == 0 && \
                      (!has_floor || t->rank[v] > floor))
    uint32_t hn = 0;
    for (uint32_t i = 1; i < n; ++i)
        if (EVICTABLE((int32_t)i)) heap_push(&c, heap, &hn, (int32_t)i);
    uint64_t imm = 0, pend = 0;
    uint32_t cnt = 0;
    int rc = 0;
    while (imm + pend < needed && hn > 0) {
        int32_t v = heap_pop(&c, heap, &hn);
        if (!EVICTABLE(v)) continue;
        uint64_t bytes = t->tokens[v] * t->bytes_per_token;
        int32_t par = t->parent[v];
        uint8_t act;
        if (!offload) {
            act = KVFO_ACT_REMOVE;
        } else if (t->backed[v]) {
            act = KVFO_ACT_DISCARD_TO_BACKUP;
        } else if (!(cpu_cap == 0 || cpu_used + bytes <= cpu_cap)) {
            act = KVFO_ACT_REMOVE; /* CPU store full (radix_cache.cpp:353-358) */
        } else {
            act = KVFO_ACT_OFFLOAD;
        }
        if (act == KVFO_ACT_REMOVE) {
            if (kids[v] != 0) { rc = 13; break; } /* remove_node throws (radix_cache.cpp:297) */
            removed[v] = 1;
            kids[par]--;
            devkids[par]--;
            imm += bytes;
        } else if (act == KVFO_ACT_DISCARD_TO_BACKUP) {
            st[v] = 1;
            devkids[par]--;
            imm += bytes;
        } else {
            st[v] = 3; /* OFFLOADING: still a device child of its parent */
            pend += bytes;
        }
        out_idx[cnt] = v;
        out_action[cnt] = act;
        ++cnt;
        if (par >= 0 && EVICTABLE(par)) heap_push(&c, heap, &hn, par); /* radix_cache.cpp:365-368 */
    }
#undef EVICTABLE
    *out_count = cnt;
    *immediate = imm;
    *pending = pend;
    free(st);
    free(removed);
    free(devkids);
    free(kids);
    free(heap);
    return rc;
}

double kvfo_now(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}
