/*
 * gids_oracle.c -- CPU restatement of the reference GIDS dataloader hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker the CUDA path is held
 * to; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  The product path never links it.
 *
 * Parity pinning: every function below is checked against golden fixtures
 * produced by running the reference itself (tests/golden/make_golden.py ->
 * the .npz files under tests/golden; see tests/test_oracle.py).
 *
 * What it restates (file:line relative to /root/reference/pkg/src/tierloader):
 *   pcg64_*            numpy's PCG64 bit generator (XSL-RR 128/64) as the
 *                      reference consumes it: Generator.random()  (sampler.py:75)
 *                      and Generator.integers(n) (cache.py:165; buffered
 *                      uint32 Lemire).  numpy is a third-party dependency
 *                      (pyproject.toml: numpy>=1.24; pinned here: 2.3.5).
 *   or_sample_subgraph sampler.py:50-112 (sample_layer + sample_subgraph)
 *   or_cache_*         cache.py:94-187 (CacheState) + cache.py:190-218
 *                      (window_update), and the set-associative policy
 *                      family of DESIGN.md section 4 (a new policy; its
 *                      contract mirrors tests/refcache.py:19-90).
 *   or_gather          dataloader.py:252-290 (tier chain + gather order)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- PCG64 */
/* state words (ABI shared with the fixtures and the CUDA library):
 *   w[0]=state_hi w[1]=state_lo w[2]=inc_hi w[3]=inc_lo w[4]=has_uint32 w[5]=uinteger */
typedef struct {
    u128 state, inc;
    int has32;
    uint32_t buf32;
} pcg64_t;

static const u128 PCG_MULT =
    ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;

static void pcg_load(pcg64_t* g, const uint64_t* w) {
    g->state = ((u128)w[0] << 64) | w[1];
    g->inc = ((u128)w[2] << 64) | w[3];
    g->has32 = (int)w[4];
    g->buf32 = (uint32_t)w[5];
}
static void pcg_store(const pcg64_t* g, uint64_t* w) {
    w[0] = (uint64_t)(g->state >> 64);
    w[1] = (uint64_t)g->state;
    w[2] = (uint64_t)(g->inc >> 64);
    w[3] = (uint64_t)g->inc;
    w[4] = (uint64_t)g->has32;
    w[5] = (uint64_t)g->buf32;
}
/* step the LCG first, then permute the new state (XSL-RR) */
static inline uint64_t pcg_next64(pcg64_t* g) {
    g->state = g->state * PCG_MULT + g->inc;
    uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
    unsigned rot = (unsigned)(hi >> 58);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
}
static inline double pcg_next_double(pcg64_t* g) {
    return (double)(pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}
/* 32-bit draws come in pairs: low half now, high half buffered */
static inline uint32_t pcg_next32(pcg64_t* g) {
    if (g->has32) {
        g->has32 = 0;
        return g->buf32;
    }
    uint64_t v = pcg_next64(g);
    g->has32 = 1;
    g->buf32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
}
/* Generator.integers(n) for 1 <= n <= 2^32: Lemire's nearly-divisionless
 * method with rejection; n == 1 returns 0 without consuming a draw. */
static uint64_t pcg_bounded(pcg64_t* g, uint64_t n) {
    uint64_t rng = n - 1;
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFULL) return pcg_next32(g);
    if (rng < 0xFFFFFFFFULL) {
        uint32_t excl = (uint32_t)rng + 1u;
        uint64_t m = (uint64_t)pcg_next32(g) * excl;
        uint32_t left = (uint32_t)m;
        if (left < excl) {
            uint32_t thresh = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % excl;
            while (left < thresh) {
                m = (uint64_t)pcg_next32(g) * excl;
                left = (uint32_t)m;
            }
        }
        return m >> 32;
    }
    /* 64-bit Lemire (bounds above 2^32; not reached by cache sizes) */
    uint64_t excl = rng + 1;
    u128 m = (u128)pcg_next64(g) * excl;
    uint64_t left = (uint64_t)m;
    if (left < excl) {
        uint64_t thresh = (0xFFFFFFFFFFFFFFFFULL - rng) % excl;
        while (left < thresh) {
            m = (u128)pcg_next64(g) * excl;
            left = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}
/* bit_generator.advance(delta): LCG jump by repeated squaring; clears the
 * buffered uint32 like numpy does. */
static void pcg_advance(pcg64_t* g, u128 delta) {
    u128 am = 1, ap = 0, cm = PCG_MULT, cp = g->inc;
    while (delta) {
        if (delta & 1) {
            am *= cm;
            ap = ap * cm + cp;
        }
        cp = (cm + 1) * cp;
        cm *= cm;
        delta >>= 1;
    }
    g->state = am * g->state + ap;
    g->has32 = 0;
    g->buf32 = 0;
}

void or_pcg_raw(uint64_t* w, uint64_t* out, int64_t n) {
    pcg64_t g;
    pcg_load(&g, w);
    for (int64_t i = 0; i < n; i++) out[i] = pcg_next64(&g);
    pcg_store(&g, w);
}
void or_pcg_doubles(uint64_t* w, double* out, int64_t n) {
    pcg64_t g;
    pcg_load(&g, w);
    for (int64_t i = 0; i < n; i++) out[i] = pcg_next_double(&g);
    pcg_store(&g, w);
}
void or_pcg_bounded(uint64_t* w, const uint64_t* ns, uint64_t* out, int64_t n) {
    pcg64_t g;
    pcg_load(&g, w);
    for (int64_t i = 0; i < n; i++) out[i] = pcg_bounded(&g, ns[i]);
    pcg_store(&g, w);
}
void or_pcg_advance(uint64_t* w, uint64_t delta_hi, uint64_t delta_lo) {
    pcg64_t g;
    pcg_load(&g, w);
    pcg_advance(&g, ((u128)delta_hi << 64) | delta_lo);
    pcg_store(&g, w);
}

/* ------------------------------------------------------------- sampler */
static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}
/* sort + dedup in place; returns the new length (np.unique) */
static int64_t uniq_i64(int64_t* a, int64_t n) {
    if (n == 0) return 0;
    qsort(a, (size_t)n, sizeof(int64_t), cmp_i64);
    int64_t k = 1;
    for (int64_t i = 1; i < n; i++)
        if (a[i] != a[k - 1]) a[k++] = a[i];
    return k;
}

/*
 * sample_subgraph (sampler.py:87-112) with sample_layer (sampler.py:50-84).
 * edges_out holds the layers back to back as (E_l, 2) int64 [src, dst];
 * edge_cap bounds the total.  Returns 0, or -1 on capacity overflow.
 * draws_out receives how many doubles were consumed (for advance()).
 */
int or_sample_subgraph(const uint64_t* indptr, const uint64_t* indices, int64_t num_nodes,
                       const int64_t* seeds, int64_t n_seeds, const int64_t* fanouts, int n_layers,
                       uint64_t* rng_words, int64_t* edges_out, int64_t edge_cap,
                       int64_t* layer_len, int64_t* unique_out, int64_t* n_unique,
                       int64_t* draws_out) {
    (void)num_nodes;
    pcg64_t g;
    pcg_load(&g, rng_words);
    int64_t* frontier = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_seeds > 0 ? n_seeds : 1));
    memcpy(frontier, seeds, sizeof(int64_t) * (size_t)n_seeds);
    int64_t nf = uniq_i64(frontier, n_seeds);
    int64_t total = 0, draws = 0;
    int64_t* pool = NULL;
    int64_t pool_cap = 0;
    int rc = 0;
    int l = 0;
    for (; l < n_layers; l++) {
        int64_t f = fanouts[l];
        int64_t base = total;
        for (int64_t t = 0; t < nf; t++) {
            int64_t v = frontier[t];
            int64_t lo = (int64_t)indptr[v], hi = (int64_t)indptr[v + 1];
            int64_t deg = hi - lo;
            if (deg == 0) continue;
            int64_t take = deg <= f ? deg : f;
            if (total + take > edge_cap) { rc = -1; goto done; }
            if (deg <= f) {
                for (int64_t i = 0; i < deg; i++) {
                    edges_out[2 * (total + i)] = (int64_t)indices[lo + i];
                    edges_out[2 * (total + i) + 1] = v;
                }
            } else {
                if (deg > pool_cap) {
                    pool_cap = deg;
                    pool = (int64_t*)realloc(pool, sizeof(int64_t) * (size_t)pool_cap);
                }
                for (int64_t i = 0; i < deg; i++) pool[i] = (int64_t)indices[lo + i];
                /* partial Fisher-Yates settling the first f positions */
                for (int64_t i = 0; i < f; i++) {
                    double u = pcg_next_double(&g);
                    int64_t j = i + (int64_t)(u * (double)(deg - i));
                    int64_t tmp = pool[i];
                    pool[i] = pool[j];
                    pool[j] = tmp;
                }
                draws += f;
                for (int64_t i = 0; i < f; i++) {
                    edges_out[2 * (total + i)] = pool[i];
                    edges_out[2 * (total + i) + 1] = v;
                }
            }
            total += take;
        }
        layer_len[l] = total - base;
        /* next frontier = np.unique(src column) */
        int64_t ne = total - base;
        int64_t* nxt = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ne > 0 ? ne : 1));
        for (int64_t i = 0; i < ne; i++) nxt[i] = edges_out[2 * (base + i)];
        free(frontier);
        frontier = nxt;
        nf = uniq_i64(frontier, ne);
        if (nf == 0) {
            for (int l2 = l + 1; l2 < n_layers; l2++) layer_len[l2] = 0;
            l = n_layers;
            break;
        }
    }
    {
        /* unique_nodes = np.unique(seeds ++ every endpoint) */
        int64_t n_all = n_seeds + 2 * total;
        int64_t* all = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_all > 0 ? n_all : 1));
        memcpy(all, seeds, sizeof(int64_t) * (size_t)n_seeds);
        memcpy(all + n_seeds, edges_out, sizeof(int64_t) * (size_t)(2 * total));
        int64_t nu = uniq_i64(all, n_all);
        memcpy(unique_out, all, sizeof(int64_t) * (size_t)nu);
        *n_unique = nu;
        free(all);
    }
done:
    free(frontier);
    free(pool);
    *draws_out = draws;
    pcg_store(&g, rng_words);
    return rc;
}

/* --------------------------------------------------------------- cache */
enum { LS_EMPTY = 0, LS_SAFE = 1, LS_INUSE = 2 };
enum { K_HIT = 0, K_MISS = 1, K_BYPASS = 2 };
enum { POL_EXACT = 0, POL_SETASSOC = 1 };
#define BLK 1024

typedef struct {
    int64_t num_nodes, lines;
    int policy, ways;
    int64_t sets;
    uint64_t evict_key; /* set-associative draws */
    pcg64_t rng;        /* exact policy draws (cache.py:108) */
    int32_t* slot_of;   /* node -> line, -1 */
    int64_t* line_node; /* line -> node, -1 */
    int8_t* state;      /* LS_* */
    uint32_t* reuse;    /* per-node predicted reuse (dict in cache.py:107) */
    int64_t* blk_safe;  /* safe lines per BLK-line block (select index) */
    int64_t fill, safe_count;
    int64_t hits, misses, bypasses, evictions, inc, dec;
} or_cache_t;

static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
/* set-associative policy: set index and per-eviction draw */
static inline int64_t sa_set_of(int64_t node, int64_t sets) {
    return (int64_t)(((u128)mix64((uint64_t)node) * (uint64_t)sets) >> 64);
}
static inline uint32_t sa_draw(uint64_t key, uint64_t epoch, int64_t node, uint32_t n) {
    uint64_t h = mix64(key ^ mix64(epoch * 0xD1B54A32D192ED03ULL + (uint64_t)node));
    return (uint32_t)(((uint64_t)(uint32_t)(h >> 32) * n) >> 32);
}

void* or_cache_new(int64_t num_nodes, int64_t lines, int policy, int ways,
                   const uint64_t* rng_words, uint64_t evict_key) {
    or_cache_t* c = (or_cache_t*)calloc(1, sizeof(or_cache_t));
    c->num_nodes = num_nodes;
    c->policy = policy;
    c->ways = ways > 0 ? ways : 1;
    if (policy == POL_SETASSOC) {
        c->sets = lines / c->ways;
        lines = c->sets * c->ways;
    }
    c->lines = lines;
    c->evict_key = evict_key;
    if (rng_words) pcg_load(&c->rng, rng_words);
    c->slot_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)(num_nodes > 0 ? num_nodes : 1));
    for (int64_t i = 0; i < num_nodes; i++) c->slot_of[i] = -1;
    c->line_node = (int64_t*)malloc(sizeof(int64_t) * (size_t)(lines > 0 ? lines : 1));
    for (int64_t i = 0; i < lines; i++) c->line_node[i] = -1;
    c->state = (int8_t*)calloc((size_t)(lines > 0 ? lines : 1), 1);
    c->reuse = (uint32_t*)calloc((size_t)(num_nodes > 0 ? num_nodes : 1), sizeof(uint32_t));
    c->blk_safe = (int64_t*)calloc((size_t)(lines / BLK + 1), sizeof(int64_t));
    return c;
}
void or_cache_free(void* h) {
    or_cache_t* c = (or_cache_t*)h;
    if (!c) return;
    free(c->slot_of);
    free(c->line_node);
    free(c->state);
    free(c->reuse);
    free(c->blk_safe);
    free(c);
}
static inline void set_safe(or_cache_t* c, int64_t s) {
    c->state[s] = LS_SAFE;
    c->blk_safe[s / BLK]++;
    c->safe_count++;
}
static inline void clear_safe(or_cache_t* c, int64_t s, int8_t to) {
    c->state[s] = to;
    c->blk_safe[s / BLK]--;
    c->safe_count--;
}
/* k-th SafeToEvict line in ascending slot order (np.flatnonzero(mask)[k]) */
static int64_t select_safe(or_cache_t* c, int64_t k) {
    int64_t b = 0;
    while (k >= c->blk_safe[b]) k -= c->blk_safe[b++];
    for (int64_t s = b * BLK;; s++)
        if (c->state[s] == LS_SAFE && k-- == 0) return s;
}

/*
 * window_update (cache.py:190-218): for each current node, count the future
 * lists containing it (binary search in each ascending list), raise the
 * reuse counter, and flip a resident SafeToEvict line to InUse when the
 * counter leaves zero.  counts_out receives the per-node counts.
 */
void or_cache_window_update(void* h, const int64_t* cur, int64_t n_cur, const int64_t* fut,
                            const int64_t* fut_off, int n_fut, int64_t* counts_out) {
    or_cache_t* c = (or_cache_t*)h;
    for (int64_t i = 0; i < n_cur; i++) {
        int64_t x = cur[i], cnt = 0;
        for (int w = 0; w < n_fut; w++) {
            int64_t lo = fut_off[w], hi = fut_off[w + 1];
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                if (fut[mid] < x) lo = mid + 1; else hi = mid;
            }
            if (lo < fut_off[w + 1] && fut[lo] == x) cnt++;
        }
        counts_out[i] = cnt;
        if (cnt == 0) continue;
        uint32_t before = c->reuse[x];
        c->reuse[x] = before + (uint32_t)cnt;
        c->inc += cnt;
        if (before == 0) {
            int32_t s = c->slot_of[x];
            if (s >= 0 && c->state[s] == LS_SAFE) clear_safe(c, s, LS_INUSE);
        }
    }
}

static inline uint32_t consume(or_cache_t* c, int64_t x) {
    uint32_t r = c->reuse[x];
    if (r > 0) {
        r--;
        c->dec++;
        c->reuse[x] = r;
    }
    return r;
}
static inline void place(or_cache_t* c, int64_t x, int64_t s, uint32_t cnt) {
    c->slot_of[x] = (int32_t)s;
    c->line_node[s] = x;
    if (cnt > 0) c->state[s] = LS_INUSE;
    else set_safe(c, s);
}

/* CacheState.access (cache.py:144-180) */
static int access_exact(or_cache_t* c, int64_t x, int64_t* slot) {
    int32_t s = c->slot_of[x];
    if (s >= 0) {
        c->hits++;
        uint32_t cnt = consume(c, x);
        if (cnt == 0 && c->state[s] == LS_INUSE) set_safe(c, s);
        *slot = s;
        return K_HIT;
    }
    uint32_t cnt = consume(c, x);
    if (c->fill < c->lines) {
        int64_t t = c->fill++;
        c->misses++;
        place(c, x, t, cnt);
        *slot = t;
        return K_MISS;
    }
    if (c->safe_count > 0) {
        int64_t k = (int64_t)pcg_bounded(&c->rng, (uint64_t)c->safe_count);
        int64_t t = select_safe(c, k);
        int64_t victim = c->line_node[t];
        c->slot_of[victim] = -1;
        clear_safe(c, t, LS_EMPTY);
        c->evictions++;
        c->misses++;
        place(c, x, t, cnt);
        *slot = t;
        return K_MISS;
    }
    c->bypasses++;
    *slot = -1;
    return K_BYPASS;
}

/* set-associative access: same contract restricted to the node's set */
static int access_setassoc(or_cache_t* c, int64_t x, uint64_t epoch, int64_t* slot) {
    int32_t s = c->slot_of[x];
    if (s >= 0) {
        c->hits++;
        uint32_t cnt = consume(c, x);
        if (cnt == 0 && c->state[s] == LS_INUSE) set_safe(c, s);
        *slot = s;
        return K_HIT;
    }
    uint32_t cnt = consume(c, x);
    if (c->sets == 0) {
        c->bypasses++;
        *slot = -1;
        return K_BYPASS;
    }
    int64_t set = sa_set_of(x, c->sets), base = set * c->ways;
    int64_t t = -1;
    uint32_t n_safe = 0;
    for (int w = 0; w < c->ways; w++) {
        if (c->state[base + w] == LS_EMPTY) { t = base + w; break; }
        if (c->state[base + w] == LS_SAFE) n_safe++;
    }
    if (t < 0 && n_safe > 0) {
        uint32_t k = sa_draw(c->evict_key, epoch, x, n_safe);
        for (int w = 0; w < c->ways; w++)
            if (c->state[base + w] == LS_SAFE && k-- == 0) { t = base + w; break; }
        int64_t victim = c->line_node[t];
        c->slot_of[victim] = -1;
        clear_safe(c, t, LS_EMPTY);
        c->evictions++;
    }
    if (t < 0) {
        c->bypasses++;
        *slot = -1;
        return K_BYPASS;
    }
    c->misses++;
    place(c, x, t, cnt);
    *slot = t;
    return K_MISS;
}

/* serve one batch's ascending unique list through the cache */
void or_cache_access_batch(void* h, const int64_t* nodes, int64_t n, uint64_t epoch,
                           int8_t* kind_out, int64_t* slot_out) {
    or_cache_t* c = (or_cache_t*)h;
    for (int64_t i = 0; i < n; i++) {
        int64_t s;
        int k = c->policy == POL_EXACT ? access_exact(c, nodes[i], &s)
                                       : access_setassoc(c, nodes[i], epoch, &s);
        kind_out[i] = (int8_t)k;
        slot_out[i] = s;
    }
}

/* stats: hits, misses, bypasses, evictions, total_increments, total_decrements,
 * safe_count, fill */
void or_cache_stats(void* h, int64_t* out) {
    or_cache_t* c = (or_cache_t*)h;
    out[0] = c->hits; out[1] = c->misses; out[2] = c->bypasses; out[3] = c->evictions;
    out[4] = c->inc; out[5] = c->dec; out[6] = c->safe_count; out[7] = c->fill;
}
void or_cache_rng(void* h, uint64_t* w) { pcg_store(&((or_cache_t*)h)->rng, w); }
int64_t or_cache_lines(void* h) { return ((or_cache_t*)h)->lines; }

/* run-ahead contribution (dataloader.py:188-192): unpinned and not resident */
int64_t or_contribution(void* h, const int64_t* nodes, int64_t n, const int32_t* pinned_off) {
    or_cache_t* c = (or_cache_t*)h;
    int64_t k = 0;
    for (int64_t i = 0; i < n; i++)
        if (pinned_off[nodes[i]] < 0 && c->slot_of[nodes[i]] < 0) k++;
    return k;
}
/* full line table snapshot: line_node[L], state[L] */
void or_cache_lines_snapshot(void* h, int64_t* node_out, int8_t* state_out) {
    or_cache_t* c = (or_cache_t*)h;
    memcpy(node_out, c->line_node, sizeof(int64_t) * (size_t)c->lines);
    memcpy(state_out, c->state, (size_t)c->lines);
}

/*
 * Tier chain + gather (dataloader.py:252-290): hits read cache rows before
 * any insertion of this batch lands; the rest come from the constant buffer
 * when pinned, else from the backing table; then each inserted slot takes
 * its row (a later insertion into the same slot wins, as the dict does).
 * tiers_out: hits, buffer, storage, bypasses.
 */
void or_gather(const int64_t* nodes, int64_t n, const int8_t* kind, const int64_t* slot,
               const int32_t* pinned_off, const float* buffer_rows, const float* table,
               float* cache_rows, float* out, int64_t dim, int64_t* tiers_out) {
    size_t rb = sizeof(float) * (size_t)dim;
    int64_t t[4] = {0, 0, 0, 0};
    for (int64_t i = 0; i < n; i++) {
        int64_t x = nodes[i];
        if (kind[i] == K_HIT) {
            memcpy(out + i * dim, cache_rows + slot[i] * dim, rb);
            t[0]++;
            continue;
        }
        if (kind[i] == K_BYPASS) t[3]++;
        if (pinned_off[x] >= 0) {
            memcpy(out + i * dim, buffer_rows + (int64_t)pinned_off[x] * dim, rb);
            t[1]++;
        } else {
            memcpy(out + i * dim, table + x * dim, rb);
            t[2]++;
        }
    }
    for (int64_t i = 0; i < n; i++)
        if (kind[i] == K_MISS) memcpy(cache_rows + slot[i] * dim, out + i * dim, rb);
    for (int k = 0; k < 4; k++) tiers_out[k] = t[k];
}

/* synthetic feature cell (graph.py:256-275), for on-the-fly verification */
void or_feature_rows(uint64_t seed, const int64_t* nodes, int64_t n, int64_t dim, float* out) {
    uint64_t seed_mix = seed * 0xD6E8FEB86659FD93ULL;
    for (int64_t i = 0; i < n; i++)
        for (int64_t col = 0; col < dim; col++) {
            uint64_t z = ((uint64_t)nodes[i] * 0x9E3779B97F4A7C15ULL) ^
                         ((uint64_t)col * 0xC2B2AE3D27D4EB4FULL) ^ seed_mix;
            z += 0x9E3779B97F4A7C15ULL;
            z ^= z >> 30;
            z *= 0xBF58476D1CE4E5B9ULL;
            z ^= z >> 27;
            z *= 0x94D049BB133111EBULL;
            z ^= z >> 31;
            out[i * dim + col] = (float)(z >> 40) / 16777216.0f;
        }
}

/* ------------------------------------------------------------------------
 * Setup-time restatements used by the C4/C5-scale checks and the CPU
 * baseline at those shapes (still TEST INFRASTRUCTURE ONLY).
 * ---------------------------------------------------------------------- */
#include <pthread.h>

typedef struct {
    void (*fn)(void* arg, int64_t lo, int64_t hi);
    void* arg;
    int64_t n;
    int nthreads, t;
} par_job_t;

static void* par_entry(void* p) {
    par_job_t* j = (par_job_t*)p;
    int64_t per = (j->n + j->nthreads - 1) / j->nthreads;
    int64_t lo = per * j->t, hi = lo + per < j->n ? lo + per : j->n;
    if (lo < hi) j->fn(j->arg, lo, hi);
    return NULL;
}
static void par_for(int64_t n, int nthreads, void (*fn)(void*, int64_t, int64_t), void* arg) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    par_job_t jobs[256];
    for (int t = 0; t < nthreads; t++) {
        jobs[t] = (par_job_t){fn, arg, n, nthreads, t};
        pthread_create(&th[t], NULL, par_entry, &jobs[t]);
    }
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
}

/* synthetic_feature_rows (graph.py:256-275) for rows [row0, row0+n), threaded */
typedef struct { uint64_t seed; int64_t row0, dim; float* out; } feat_job_t;
static void feat_part(void* a, int64_t lo, int64_t hi) {
    feat_job_t* j = (feat_job_t*)a;
    for (int64_t i = lo; i < hi; i++) {
        int64_t node = j->row0 + i;
        or_feature_rows(j->seed, &node, 1, j->dim, j->out + i * j->dim);
    }
}
void or_feature_table(uint64_t seed, int64_t row0, int64_t n, int64_t dim, float* out,
                      int nthreads) {
    feat_job_t j = {seed, row0, dim, out};
    par_for(n, nthreads, feat_part, &j);
}

/*
 * Uniform graph generator of csrc/graph_setup.cu (its header states the
 * definition): dst(e) = hi64(mix64(s_dst + e) * N); segment of v drawn as
 * src(v,k,a) = hi64(mix64(mix64(s_src ^ v) + (a<<32) + k) * N), sorted, and
 * repeats at sorted position r redrawn with src(v, r, a) for a = 1, 2, ...
 * Output in the reference's GraphCsc dtypes (u64).
 */
static inline uint64_t hi64(uint64_t a, uint64_t b) { return (uint64_t)(((u128)a * b) >> 64); }

typedef struct { uint64_t s; int64_t n; uint32_t* cnt; } hist_job_t;
static void hist_part(void* a, int64_t lo, int64_t hi) {
    hist_job_t* j = (hist_job_t*)a;
    for (int64_t e = lo; e < hi; e++)
        __atomic_fetch_add(&j->cnt[hi64(mix64(j->s + (uint64_t)e), (uint64_t)j->n)], 1u,
                           __ATOMIC_RELAXED);
}
typedef struct { uint64_t s; int64_t n; const uint64_t* indptr; uint64_t* indices; int bad; } fill_job_t;
static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}
static void fill_part(void* a, int64_t lo, int64_t hi) {
    fill_job_t* j = (fill_job_t*)a;
    const uint64_t n = (uint64_t)j->n;
    for (int64_t v = lo; v < hi; v++) {
        uint64_t* seg = j->indices + j->indptr[v];
        int64_t deg = (int64_t)(j->indptr[v + 1] - j->indptr[v]);
        if (deg == 0) continue;
        if (deg > 1024) { j->bad = 1; continue; }
        uint64_t zv = mix64(j->s ^ (uint64_t)v);
        for (int64_t k = 0; k < deg; k++) seg[k] = hi64(mix64(zv + (uint64_t)k), n);
        for (uint64_t att = 1;; att++) {
            qsort(seg, (size_t)deg, sizeof(uint64_t), cmp_u64);
            int rep = 0;
            /* decide every repeat against the sorted array before rewriting */
            uint64_t prev = seg[0];
            for (int64_t r = 1; r < deg; r++) {
                uint64_t cur = seg[r];
                if (cur == prev) {
                    seg[r] = hi64(mix64(zv + (att << 32) + (uint64_t)r), n);
                    rep = 1;
                }
                prev = cur;
            }
            if (!rep) break;
        }
    }
}
int or_generate_uniform(int64_t n, int64_t e, uint64_t seed, uint64_t* indptr, uint64_t* indices,
                        int nthreads) {
    uint32_t* cnt = (uint32_t*)calloc((size_t)n, sizeof(uint32_t));
    if (!cnt) return -1;
    hist_job_t hj = {mix64(seed ^ 0x243F6A8885A308D3ULL), n, cnt};
    par_for(e, nthreads, hist_part, &hj);
    indptr[0] = 0;
    for (int64_t v = 0; v < n; v++) indptr[v + 1] = indptr[v] + cnt[v];
    free(cnt);
    fill_job_t fj = {mix64(seed ^ 0x13198A2E03707344ULL), n, indptr, indices, 0};
    par_for(n, nthreads, fill_part, &fj);
    return fj.bad ? -2 : 0;
}

/*
 * reverse_pagerank (cpu_buffer.py:26-74, unit weights), float64-identical to
 * the reference: np.bincount accumulates each node's shares in edge order,
 * i.e. by ascending destination, so the pull over per-source lists sorted by
 * destination reproduces it term for term; sums of x[sink] and |nxt - x|
 * follow numpy's pairwise summation (loops_utils.h: 8 accumulators over
 * blocks of <= 128, split at n/2 rounded down to a multiple of 8).
 */
static double pw_sum_gen(const double* a, const int64_t* idx, int64_t n) {
#define PW_AT(i) (idx ? a[idx[(i)]] : a[(i)])
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; i++) r += PW_AT(i);
        return r;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = PW_AT(j);
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += PW_AT(i + j);
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += PW_AT(i);
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pw_sum_gen(a, idx, n2) + pw_sum_gen(idx ? a : a + n2, idx ? idx + n2 : NULL, n - n2);
    }
#undef PW_AT
}
/* numpy-order pairwise sum of a[0..n) (exported for the tests) */
double or_pairwise_sum(const double* a, int64_t n) { return pw_sum_gen(a, NULL, n); }

typedef struct {
    const uint64_t* indptr; const uint64_t* indices;
    uint64_t* tptr; uint32_t* cur; uint32_t* towner; uint32_t* cnt;
    const double* y; double* nxt; const double* x; double* diff; double damping, c;
} pr_job_t;
static void pr_count(void* a, int64_t lo, int64_t hi) {
    pr_job_t* j = (pr_job_t*)a;
    for (int64_t e = lo; e < hi; e++) __atomic_fetch_add(&j->cnt[j->indices[e]], 1u, __ATOMIC_RELAXED);
}
static void pr_scatter(void* a, int64_t lo, int64_t hi) {
    pr_job_t* j = (pr_job_t*)a;
    for (int64_t v = lo; v < hi; v++)
        for (uint64_t e = j->indptr[v]; e < j->indptr[v + 1]; e++) {
            uint64_t u = j->indices[e];
            uint32_t at = __atomic_fetch_add(&j->cur[u], 1u, __ATOMIC_RELAXED);
            j->towner[j->tptr[u] + at] = (uint32_t)v;
        }
}
static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}
static void pr_sortlists(void* a, int64_t lo, int64_t hi) {
    pr_job_t* j = (pr_job_t*)a;
    for (int64_t u = lo; u < hi; u++)
        qsort(j->towner + j->tptr[u], (size_t)(j->tptr[u + 1] - j->tptr[u]), sizeof(uint32_t),
              cmp_u32);
}
static void pr_pull(void* a, int64_t lo, int64_t hi) {
    pr_job_t* j = (pr_job_t*)a;
    for (int64_t u = lo; u < hi; u++) {
        double acc = 0.0;
        for (uint64_t k = j->tptr[u]; k < j->tptr[u + 1]; k++) acc += j->y[j->towner[k]];
        double v = acc * j->damping;
        v = v + j->c;
        j->nxt[u] = v;
        double d = v - j->x[u];
        j->diff[u] = d < 0 ? -d : d;
    }
}
int or_reverse_pagerank(const uint64_t* indptr, const uint64_t* indices, int64_t n, double damping,
                        double tol, int max_iter, double* scores, int* iters, int* conv,
                        int nthreads) {
    int64_t e = (int64_t)indptr[n];
    pr_job_t j;
    memset(&j, 0, sizeof(j));
    j.indptr = indptr;
    j.indices = indices;
    j.cnt = (uint32_t*)calloc((size_t)n, sizeof(uint32_t));
    j.cur = (uint32_t*)calloc((size_t)n, sizeof(uint32_t));
    j.tptr = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n + 1));
    j.towner = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(e > 0 ? e : 1));
    double* denom = (double*)malloc(sizeof(double) * (size_t)n);
    double* x = (double*)malloc(sizeof(double) * (size_t)n);
    double* nxt = (double*)malloc(sizeof(double) * (size_t)n);
    double* y = (double*)malloc(sizeof(double) * (size_t)n);
    double* diff = (double*)malloc(sizeof(double) * (size_t)n);
    int64_t* sinks = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    par_for(e, nthreads, pr_count, &j);
    j.tptr[0] = 0;
    for (int64_t u = 0; u < n; u++) j.tptr[u + 1] = j.tptr[u] + j.cnt[u];
    par_for(n, nthreads, pr_scatter, &j);
    par_for(n, nthreads, pr_sortlists, &j);
    int64_t ns = 0;
    for (int64_t v = 0; v < n; v++) {
        uint64_t d = indptr[v + 1] - indptr[v];
        denom[v] = d == 0 ? 1.0 : (double)d;
        if (d == 0) sinks[ns++] = v;
        x[v] = 1.0 / (double)n;
    }
    double teleport = (1.0 - damping) / (double)n;
    int it = 0, converged = 0;
    while (it < max_iter) {
        it++;
        for (int64_t v = 0; v < n; v++) y[v] = x[v] / denom[v];
        double s = pw_sum_gen(x, sinks, ns);
        j.c = teleport + damping * s / (double)n;
        j.damping = damping;
        j.y = y;
        j.x = x;
        j.nxt = nxt;
        j.diff = diff;
        par_for(n, nthreads, pr_pull, &j);
        double delta = pw_sum_gen(diff, NULL, n);
        double* t = x;
        x = nxt;
        nxt = t;
        if (delta < tol) {
            converged = 1;
            break;
        }
    }
    memcpy(scores, x, sizeof(double) * (size_t)n);
    *iters = it;
    *conv = converged;
    free(j.cnt); free(j.cur); free(j.tptr); free(j.towner);
    free(denom); free(x); free(nxt); free(y); free(diff); free(sinks);
    return 0;
}
