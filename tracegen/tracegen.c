/*
 * tracegen.c — seeded synthetic malloc/free traces.
 *
 * This module is shared by the oracle side (tests, bench cpu_baseline) and the
 * CUDA side (bench, GPU tests).  It holds NONE of the allocator's arithmetic:
 * it only draws request sizes and which live ids to free.  Ids are abstract
 * ("the j-th successful-or-not alloc of the trace"); mapping an id to an offset
 * is the caller's job, so the trace is allocator-independent.
 *
 * PRNG: SplitMix64 seeds xoshiro256**; bounded(n) = (next() * (u128)n) >> 64.
 *
 * Workload shapes ("randomly allocates and frees blocks ... several
 * thousand times"; sizes per BASELINE.json configs):
 *   size kind 0  LU8[2^a, 2^b): octave-uniform, e = a + bounded(b-a), s = 2^e + bounded(2^e)
 *   size kind 1  buddy orders k in [a, b], weight 2^floor((b-k)/2), s = 2^k
 *   model 0      batch model: nf = min(round(rho*B), |live|), na = B - nf; frees are
 *                uniform live ids without replacement (swap-remove) from the batch-start live set
 *   model 1      slot model (SPEC.md:497-505 shape): pick a uniform slot; if occupied free its
 *                id then alloc a new id into it, else alloc.  Batches are cut only where a free
 *                would reference an id allocated in the current batch (reading C24).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    uint64_t s[4];
    int model;
    int size_kind;
    uint64_t a, b;          /* size parameters */
    uint64_t batch;         /* B (batch model) */
    uint64_t rho_num, rho_den;
    uint64_t total_ops, ops_done;
    uint64_t next_id;
    /* batch model: live id set */
    uint64_t *live; uint64_t n_live, cap_live;
    /* slot model */
    uint64_t n_slots; uint64_t *slot_id; uint8_t *slot_used; uint64_t *slot_batch;
    uint64_t batch_idx;
    /* buddy weights */
    uint64_t wsum; uint64_t wtab[64];
    /* slot model carry-over step */
    int have_pending; uint64_t pend_slot;
} tg_t;

static uint64_t splitmix64(uint64_t *x) {
    uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static uint64_t next_u64(tg_t *t) {
    uint64_t *s = t->s;
    uint64_t result = rotl(s[1] * 5, 7) * 9;
    uint64_t u = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
    s[2] ^= u; s[3] = rotl(s[3], 45);
    return result;
}
static uint64_t bounded(tg_t *t, uint64_t n) {
    return (uint64_t)(((unsigned __int128)next_u64(t) * n) >> 64);
}

static uint64_t draw_size(tg_t *t) {
    if (t->size_kind == 0) {
        uint64_t e = t->a + bounded(t, t->b - t->a);
        return (1ull << e) + bounded(t, 1ull << e);
    } else {
        uint64_t x = bounded(t, t->wsum);
        for (uint64_t k = t->a; k <= t->b; k++) {
            if (x < t->wtab[k]) return 1ull << k;
            x -= t->wtab[k];
        }
        return 1ull << t->b; /* unreachable */
    }
}

uint64_t tg_seed(uint64_t config, uint64_t rank) { return 2405070790ull + 1000ull * config + rank; }

tg_t *tg_create(int model, uint64_t seed, uint64_t batch, uint64_t rho_num, uint64_t rho_den,
                uint64_t total_ops, int size_kind, uint64_t a, uint64_t b, uint64_t n_slots) {
    tg_t *t = (tg_t *)calloc(1, sizeof(tg_t));
    if (!t) return NULL;
    uint64_t x = seed;
    for (int i = 0; i < 4; i++) t->s[i] = splitmix64(&x);
    t->model = model; t->size_kind = size_kind; t->a = a; t->b = b;
    t->batch = batch; t->rho_num = rho_num; t->rho_den = rho_den ? rho_den : 1;
    t->total_ops = total_ops;
    if (size_kind == 1) {
        t->wsum = 0;
        for (uint64_t k = a; k <= b && k < 64; k++) { t->wtab[k] = 1ull << ((b - k) / 2); t->wsum += t->wtab[k]; }
    }
    if (model == 1) {
        t->n_slots = n_slots;
        t->slot_id = (uint64_t *)calloc(n_slots, sizeof(uint64_t));
        t->slot_used = (uint8_t *)calloc(n_slots, 1);
        t->slot_batch = (uint64_t *)calloc(n_slots, sizeof(uint64_t));
    }
    return t;
}

void tg_destroy(tg_t *t) {
    if (!t) return;
    free(t->live); free(t->slot_id); free(t->slot_used); free(t->slot_batch); free(t);
}

static void live_push(tg_t *t, uint64_t id) {
    if (t->n_live == t->cap_live) {
        t->cap_live = t->cap_live ? 2 * t->cap_live : 1024;
        t->live = (uint64_t *)realloc(t->live, t->cap_live * sizeof(uint64_t));
    }
    t->live[t->n_live++] = id;
}

uint64_t tg_n_live(const tg_t *t) { return t->n_live; }
uint64_t tg_ops_done(const tg_t *t) { return t->ops_done; }
uint64_t tg_next_id(const tg_t *t) { return t->next_id; }

/* Fill free_ids[0..nf) and sizes[0..na).  Alloc ids of this batch are next_id..next_id+na-1
 * in request order (returned through *first_alloc_id).  Buffers must hold max_n entries.
 * Returns 1 if a batch was produced, 0 when the op budget is exhausted. */
int tg_next_batch(tg_t *t, uint64_t max_n, uint64_t *free_ids, uint64_t *nf_out,
                  uint64_t *sizes, uint64_t *na_out, uint64_t *first_alloc_id) {
    uint64_t nf = 0, na = 0;
    *first_alloc_id = t->next_id;
    if (t->ops_done >= t->total_ops) { *nf_out = 0; *na_out = 0; return 0; }
    if (t->model == 0) {
        uint64_t B = t->batch;
        uint64_t left = t->total_ops - t->ops_done;
        if (B > left) B = left;
        if (B > max_n) B = max_n;
        nf = (t->rho_num * B + t->rho_den / 2) / t->rho_den;
        if (nf > t->n_live) nf = t->n_live;
        na = B - nf;
        for (uint64_t j = 0; j < nf; j++) {
            uint64_t idx = bounded(t, t->n_live);
            free_ids[j] = t->live[idx];
            t->live[idx] = t->live[--t->n_live];
        }
        for (uint64_t j = 0; j < na; j++) {
            sizes[j] = draw_size(t);
            live_push(t, t->next_id++);
        }
    } else {
        /* slot model */
        t->batch_idx++;
        for (;;) {
            if (t->ops_done + nf + na >= t->total_ops) break;
            uint64_t s;
            if (t->have_pending) { s = t->pend_slot; }
            else { s = bounded(t, t->n_slots); }
            int need_free = t->slot_used[s];
            if (need_free && t->slot_batch[s] == t->batch_idx) {
                /* cut rule: this free references an id allocated in the current batch */
                t->have_pending = 1; t->pend_slot = s;
                if (nf + na == 0) { /* cannot happen: a fresh batch has no ids yet */ }
                break;
            }
            t->have_pending = 0;
            if (nf + na + (uint64_t)need_free + 1 > max_n) { t->have_pending = 1; t->pend_slot = s; break; }
            if (need_free) {
                free_ids[nf++] = t->slot_id[s];
                t->slot_used[s] = 0;
                if (t->ops_done + nf + na >= t->total_ops) break;   /* budget ends after the free */
            }
            sizes[na++] = draw_size(t);
            t->slot_id[s] = t->next_id++;
            t->slot_used[s] = 1;
            t->slot_batch[s] = t->batch_idx;
        }
    }
    t->ops_done += nf + na;
    *nf_out = nf; *na_out = na;
    return 1;
}
