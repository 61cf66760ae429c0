// gids_internal.cuh -- shared state, device helpers and launcher prototypes
// for libgids.so (B200 / sm_100a).  See DESIGN.md for the data layout.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/gids.h"

#define GIDS_WARP 32

// ---------------------------------------------------------------- errors
void gids_set_error(const std::string& msg);

#define GIDS_CUDA_TRY(expr)                                                      \
    do {                                                                         \
        cudaError_t _e = (expr);                                                 \
        if (_e != cudaSuccess) {                                                 \
            gids_set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));  \
            return GIDS_E_CUDA;                                                  \
        }                                                                        \
    } while (0)

#define GIDS_LAUNCH_CHECK(h)                                                      \
    do {                                                                          \
        cudaError_t _e = cudaGetLastError();                                      \
        if (_e != cudaSuccess) {                                                  \
            gids_set_error(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
            return GIDS_E_CUDA;                                                   \
        }                                                                         \
        (h)->launches++;                                                          \
    } while (0)

// ------------------------------------------------------------ 128-bit math
struct u128 {
    uint64_t lo, hi;
};

__host__ __device__ __forceinline__ u128 mul128(u128 a, u128 b) {
    u128 r;
#ifdef __CUDA_ARCH__
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
#else
    unsigned __int128 p = (unsigned __int128)a.lo * b.lo;
    r.lo = (uint64_t)p;
    r.hi = (uint64_t)(p >> 64) + a.lo * b.hi + a.hi * b.lo;
#endif
    return r;
}
__host__ __device__ __forceinline__ u128 add128(u128 a, u128 b) {
    u128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
    return r;
}

// numpy PCG64 (XSL-RR 128/64): multiplier of the 128-bit LCG
static constexpr uint64_t PCG_MULT_HI = 0x2360ED051FC65DA4ULL;
static constexpr uint64_t PCG_MULT_LO = 0x4385DF649FCCF645ULL;

struct Pcg64 {
    u128 state, inc;
    uint32_t has32, buf32;
};

__host__ __device__ __forceinline__ uint64_t pcg_output(u128 s) {
    uint64_t x = s.hi ^ s.lo;
    unsigned rot = (unsigned)(s.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}
__host__ __device__ __forceinline__ uint64_t pcg_next64(Pcg64& g) {
    g.state = add128(mul128(g.state, u128{PCG_MULT_LO, PCG_MULT_HI}), g.inc);
    return pcg_output(g.state);
}
__host__ __device__ __forceinline__ uint32_t pcg_next32(Pcg64& g) {
    if (g.has32) {
        g.has32 = 0;
        return g.buf32;
    }
    uint64_t v = pcg_next64(g);
    g.has32 = 1;
    g.buf32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
}
// Generator.integers(n), 1 <= n < 2^32 (buffered-uint32 Lemire, numpy)
__host__ __device__ __forceinline__ uint32_t pcg_bounded32(Pcg64& g, uint32_t n) {
    if (n <= 1) return 0;
    uint64_t m = (uint64_t)pcg_next32(g) * n;
    uint32_t left = (uint32_t)m;
    if (left < n) {
        uint32_t thresh = (uint32_t)(0u - n) % n;
        while (left < thresh) {
            m = (uint64_t)pcg_next32(g) * n;
            left = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

inline Pcg64 pcg_from_words(const uint64_t* w) {
    Pcg64 g;
    g.state = u128{w[1], w[0]};
    g.inc = u128{w[3], w[2]};
    g.has32 = (uint32_t)w[4];
    g.buf32 = (uint32_t)w[5];
    return g;
}
inline void pcg_to_words(const Pcg64& g, uint64_t* w) {
    w[0] = g.state.hi;
    w[1] = g.state.lo;
    w[2] = g.inc.hi;
    w[3] = g.inc.lo;
    w[4] = g.has32;
    w[5] = g.buf32;
}

// splitmix64 finaliser (set hashing and set-associative eviction draws)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// ------------------------------------------------------------- the handle
// Per-batch device counters (one struct, zeroed per sample / serve).
struct SampleCounters {
    int64_t n_front;                      // current frontier size
    int64_t layer_len[GIDS_MAX_LAYERS];   // edges per layer
    int64_t layer_draw_base[GIDS_MAX_LAYERS + 1];  // doubles consumed before layer l
    int64_t n_unique;
    int64_t contribution;
    int64_t overflow;                     // workspace bound exceeded
    // the batch's sizes as exported ([layer_len[0..L), n_unique, draws,
    // contribution, overflow]), written by the last compaction
    int64_t exp[GIDS_MAX_LAYERS + 4];
    uint32_t tile_ctr[GIDS_MAX_LAYERS + 2];  // single-pass compactions: next tile
};

// decoupled look-back state of one 8192-node bitmap tile (sampler.cu):
// the tile's own sums, then the inclusive prefix through it
struct LbTile {
    unsigned long long agg;  // take | count << 24 | draws-nodes << 38
    unsigned long long inc_take;
    uint32_t inc_cnt, inc_nd;
    uint32_t flag;           // 0 nothing, 1 agg, 2 inclusive
    uint32_t pad;
};

// per-call arguments of a serve replayed as a CUDA graph (the kernels read
// them from device memory; NULL = the launch's own arguments)
struct ServeArgs {
    const int64_t* uniq;
    int64_t n;
    uint64_t epoch;
    float* out;
    const int64_t* pop;  // window shift applied before the decisions
    int64_t n_pop;
    const int64_t* push;
    int64_t n_push;
};

// a window pop / push folded into the next serve (gids_serve_shift)
struct WindowShift {
    const int64_t* pop;
    int64_t n_pop;
    const int64_t* push;
    int64_t n_push;
};

struct ServeCounters {
    int64_t tiers[4];      // hits, buffer, storage, bypasses (this batch)
    int64_t n_log;         // insertions logged by the exact policy this batch
    int64_t n_miss0;       // nodes not resident when the batch's decisions start
    int64_t shard_local, shard_remote;  // sharded-table mode: rows from own / peer HBM
    int64_t n_cand;        // resident SafeToEvict nodes of the batch (exact_par.cu)
    int64_t xp_done;       // the batch was decided by k_exact_par
    int64_t xp_stats[4];   // its rounds; rounds ended by a rejection / full change list / lost line
    int64_t bad_order;     // the served list was not strictly ascending (k_window_consume)
    int64_t xp_prof[12];   // SM cycles per phase (see exact_par.cu) and fixed-point passes
};

struct CacheMeta {  // persistent cache counters (CacheState)
    int64_t hits, misses, bypasses, evictions, inc, dec;
    int64_t safe_count, fill;
    uint64_t rng[6];       // exact-policy eviction PCG64 words
};

struct FileTier;

// one instantiated sampling graph per distinct seed count (sampler.cu)
struct SampleGraph {
    int64_t n_seeds;
    int64_t kernels;  // kernel nodes, for the launch counter
    cudaGraphExec_t exec;
};
constexpr int GIDS_MAX_SGRAPHS = 4;

struct gids_handle {
    gids_config cfg;
    int device;
    int64_t N, E, L;       // nodes, edges, cache lines (effective)
    int64_t sets;          // set-associative sets (L / 32)
    int64_t row_floats;
    int64_t launches;
    cudaStream_t last_stream;
    cudaEvent_t counted = nullptr;  // the last serve's tier counts are in svc_host
    bool counted_valid = false;
    cudaEvent_t contributed = nullptr;  // the last gids_contribution_async's reads done
    bool contributed_valid = false;

    // graph (HBM)
    int64_t* indptr;       // [N+1]
    int32_t* indices;      // [E]

    // tiers
    const float* backing;  // host table (zero-copy), N x dim
    bool backing_registered;
    const float* buffer_rows;  // host constant buffer rows, k x dim
    bool buffer_registered;
    int64_t buffer_k;
    int32_t* pinned_off;   // [N] node -> constant-buffer row, -1

    // cache state (HBM)
    float* cache_rows;     // [L x dim]
    int32_t* slot_of;      // [N] node -> line, -1
    int32_t* line_node;    // [L] line -> node, -1
    uint32_t* safe_bits;   // [ceil(L/32)] SafeToEvict bitmap
    uint32_t* blk_cnt;     // [ceil(L/1024)] safe lines per 1024-line block
    uint32_t* sup_cnt;     // [ceil(L/32768)] safe lines per 32768-line superblock
    uint32_t* evict_bits;  // [ceil(L/32)] lines evicted during the current batch
    uint32_t* reuse;       // [N] predicted-reuse counters
    uint8_t* future;       // [N] lookahead-window occurrence counts
    CacheMeta* meta;       // device
    int32_t* last_ins;     // [L] scratch: last log index per line (-1)
    // CTA-parallel exact policy for a full cache (exact_par.cu)
    uint32_t* xcls;        // [serve_cap] access class | candidate index << 3
    int32_t* cand_of_slot; // [L] candidate index of the line's batch-start node, -1
    int32_t* cand_slot;    // [GIDS_XP_CAND_CAP] line of each candidate
    uint32_t* xp_halves;   // [xp_hcap] the batch's eviction draw halves
    int64_t xp_hcap;
    bool xp_enabled;       // GIDS_EXACT_PAR=0 keeps every batch on k_exact_seq
    int64_t xp_safe_div;   // k_exact_par needs safe_count * div >= misses (0: any; GIDS_EXACT_PAR=2)
    int64_t xp_batches;    // served batches k_exact_par decided
    int64_t xp_stats[16];  // their ServeCounters.xp_stats, xp_prof, summed
    bool counts_read;      // the last serve's counts were read once already

    // sampler workspace (HBM)
    int64_t max_seeds;
    int window_lists = 0;  // lists pushed and not popped (future[] is 8-bit)
    bool host_timing = false;  // GIDS_SERVE_TIMING=1: host ns per serve section
    double host_ns[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t host_calls = 0;
    unsigned long long* line_mark = nullptr;  // shared cache (owner role): (batch, pos) of each line's last insert
    uint64_t* shared_rows = nullptr; // shared cache (requester role): owners' cache_rows pointers
    int32_t shared_rows_g = 0;
    int64_t edge_cap;      // total edges over all layers
    int64_t front_cap;     // max frontier size
    uint32_t* bm_front;    // [ceil(N/32)]
    uint32_t* bm_all;      // [ceil(N/32)]
    int32_t* frontier;     // [front_cap]
    int64_t* seeds_dev;    // [max_seeds]
    int64_t lb_tiles;      // bitmap tiles of 8192 nodes; LbTile[(n_layers+1) * lb_tiles] follow *sc
    int64_t* take_off;     // [front_cap+1] exclusive scan of min(deg, f)
    int64_t* draw_off;     // [front_cap+1] exclusive scan of draws
    int64_t* edges;        // [2*edge_cap]
    int32_t* unique32;     // [front_cap_all]
    int64_t unique_cap;
    u128* jump_tab;        // [GIDS_JUMP_TAB] jumps {A_i, H_i} of 2^i, then steps of k <= 1024
    u128* jump_host;       // pinned staging of the table
    u128* rng_dev;         // [2] device-resident sampler stream: state, inc
    u128* rng_host;        // pinned staging
    uint64_t jump_inc_hi, jump_inc_lo;
    bool jump_valid;
    SampleCounters* sc;    // device
    int64_t* contrib_dev;  // [2] scratch of gids_contribution_async (sum, blocks done; left 0)
    SampleCounters* sc_host;  // pinned mirror
    int64_t scan_parts_cap;
    int64_t* scan_parts;   // [scan_parts_cap * 2]
    uint32_t* word_parts;  // [scan_parts_cap]
    // the serving path's own scan partials: sampling runs on another stream,
    // concurrently with the decisions and the file-tier page planning
    int64_t* serve_parts;       // [scan_parts_cap * 2]
    uint32_t* serve_word_parts;  // [scan_parts_cap]

    // serve workspace
    int64_t serve_cap;     // max unique per batch
    uint32_t* ev;          // [serve_cap] packed (line+1)<<1 | inuse_after
    // decisions are double-buffered: the gather of batch b reads set b&1
    // while the decide phase of batch b+1 writes the other one
    int8_t* kind_buf[2];   // [serve_cap] GIDS_KIND_*
    int32_t* line_buf[2];  // [serve_cap] line read (hit) or taken (miss), -1
    int32_t* ins_buf[2];   // [serve_cap] line this node's row must be written to, -1
    // compacted work lists of the gather, per decision set: positions of the
    // cache hits, and (position, source row) of the host-tier rows where the
    // source is a constant-buffer row (>= 0) or backing row x (encoded -(x+1))
    int32_t* hit_list_buf[2];   // [serve_cap]
    int2* host_list_buf[2];     // [serve_cap]
    int64_t* list_cnt_buf[2];   // [2] hits, host rows
    int8_t* kind;          // current set (alias)
    int32_t* line;
    int32_t* ins;
    int32_t* hit_list;
    int2* host_list;
    int64_t* list_cnt;
    int parity;
    cudaEvent_t gathered[2];  // gather of the last batch that used each set
    bool gathered_valid[2];
    cudaEvent_t decided;      // decide phase of the last served batch
    int32_t* log_line;     // [serve_cap] exact-policy insertion log
    int32_t* log_pos;      // [serve_cap]
    int32_t* set_cnt;      // [sets]
    int64_t* set_off;      // [sets+1]
    int32_t* set_cur;      // [sets]
    int32_t* bucket;       // [serve_cap]
    ServeCounters* svc;    // device
    ServeCounters* svc_host;  // pinned mirror
    int64_t last_serve_n;
    bool exact_smem;       // exact-policy tables fit in shared memory
    int gather_blocks;     // gather grid (resident blocks of 8 warps)
    int gather_unroll;     // 16-B loads in flight per lane in the host gather (1,2,4,8)
    int hit_blocks;        // hit-gather grid (GIDS_HIT_BPS blocks of 8 warps per SM)
    int hit_unroll;        // 16-B loads in flight per lane in the hit gather (4, 8)

    // HBM-sharded feature table: node v lives in
    // shard v % n_shards at row v / n_shards; shard pointers may be peer
    // (NVLink) addresses opened from CUDA IPC handles
    int32_t n_shards;      // 0 = tiered mode (cache + host tiers)
    int32_t my_shard;
    const float** shard_ptrs;  // device array [n_shards]

    // CUDA graphs of the sampling sequence and of the serve (GIDS_NO_GRAPHS=1
    // disables): per decision-buffer parity, decisions and rows
    ServeArgs* sargs;  // device [2]
    WindowShift shift;  // of the serve being launched (zero: none)
    cudaGraphExec_t dgraph[2], ggraph[2];
    int64_t dgraph_kernels[2], ggraph_kernels[2];
    int64_t serves;
    int64_t serve_replays;
    bool graphs_failed;
    bool use_graphs;
    int n_sgraphs;
    SampleGraph sgraphs[GIDS_MAX_SGRAPHS];

    // file-backed storage tier (storage_file.cu); null = pinned-host tier
    struct FileTier* ft;

    // phase timing (gids_set_profiling)
    bool profiling;
    cudaEvent_t tev[8];    // 2,3 decide phase
    // sampling time: a ring of (start, end) event pairs harvested without
    // blocking (cudaEventQuery), so profiling does not serialise run-ahead
    static constexpr int SRING = 64;
    cudaEvent_t sev[SRING][2];
    int sev_head, sev_count;
    cudaEvent_t gev[2][3]; // per decision set: gather start, hits done, host rows done
    bool gather_pending[2];
    bool serve_timed;
    double phase_ms[5];
};

// fold the finished gather timing of decision set `par` into phase_ms
// (profiling only; timing failures are dropped and must not leave a sticky
// error for the next launch check)
inline void gids_harvest_gather(gids_handle* h, int par) {
    if (!h->gather_pending[par]) return;
    h->gather_pending[par] = false;
    float b = 0.f, c = 0.f;
    if (cudaEventSynchronize(h->gev[par][2]) == cudaSuccess &&
        cudaEventElapsedTime(&b, h->gev[par][0], h->gev[par][1]) == cudaSuccess &&
        cudaEventElapsedTime(&c, h->gev[par][1], h->gev[par][2]) == cudaSuccess) {
        h->phase_ms[2] += b;
        h->phase_ms[3] += c;
    }
    cudaGetLastError();
}
// fold finished sampling intervals into phase_ms[0]: oldest first, stopping
// at the first unfinished one unless `wait` (then the oldest is awaited)
inline void gids_harvest_sample(gids_handle* h, bool wait) {
    while (h->sev_count > 0) {
        int i = (h->sev_head - h->sev_count + gids_handle::SRING) % gids_handle::SRING;
        if (wait) {
            cudaEventSynchronize(h->sev[i][1]);
        } else if (cudaEventQuery(h->sev[i][1]) != cudaSuccess) {
            break;
        }
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, h->sev[i][0], h->sev[i][1]) == cudaSuccess)
            h->phase_ms[0] += ms;
        h->sev_count--;
    }
    cudaGetLastError();
}
// open a sampling interval on `st` (profiling only); the ring never waits
// unless it is full
inline void gids_sample_begin(gids_handle* h, cudaStream_t st) {
    if (!h->profiling) return;
    gids_harvest_sample(h, false);
    if (h->sev_count == gids_handle::SRING) {
        int i = (h->sev_head - h->sev_count + gids_handle::SRING) % gids_handle::SRING;
        cudaEventSynchronize(h->sev[i][1]);
        gids_harvest_sample(h, false);
    }
    cudaEventRecord(h->sev[h->sev_head][0], st);
}
inline void gids_sample_end(gids_handle* h, cudaStream_t st) {
    if (!h->profiling) return;
    cudaEventRecord(h->sev[h->sev_head][1], st);
    h->sev_head = (h->sev_head + 1) % gids_handle::SRING;
    h->sev_count++;
}

inline void gids_mark(gids_handle* h, int i, cudaStream_t st) {
    if (h->profiling) cudaEventRecord(h->tev[i], st);
}

// ------------------------------------------------------------- launchers
// scan.cu
int gids_scan_take_draw(gids_handle* h, int fanout, int layer, cudaStream_t st);
int gids_bitmap_compact(gids_handle* h, uint32_t* bm, int32_t* out, int64_t* count_out,
                        int64_t cap, bool clear, cudaStream_t st);
int gids_bitmap_compact_n(gids_handle* h, uint32_t* bm, int64_t nbits, int32_t* out,
                          int64_t* count_out, int64_t cap, bool clear, int64_t* overflow,
                          uint32_t* parts, cudaStream_t st);
int gids_scan_i32_to_i64(gids_handle* h, const int32_t* in, int64_t n, int64_t* out,
                         cudaStream_t st);
// sampler.cu
int gids_launch_sample(gids_handle* h, int64_t n_seeds, const uint64_t* rng_words, bool raw,
                       cudaStream_t st);
int gids_launch_export_unique(gids_handle* h, int64_t* unique_dev, cudaStream_t st);
int gids_launch_export(gids_handle* h, int64_t* edges_dev, int64_t* unique_dev, cudaStream_t st,
                       int64_t* sizes_host = nullptr);
// exact_par.cu
constexpr int64_t GIDS_XP_CAND_CAP = 1 << 17;
// access classes of a batch against a full cache (k_window_consume -> k_exact_par)
enum { GIDS_XC_STAY = 0, GIDS_XC_ADD = 1, GIDS_XC_CAND = 2, GIDS_XC_M0 = 3, GIDS_XC_MU = 4 };
int gids_launch_exact_par(gids_handle* h, int64_t n, cudaStream_t st,
                          const ServeArgs* sa = nullptr);
int gids_launch_xp_reset(gids_handle* h, cudaStream_t st);
size_t gids_xp_smem_bytes(int64_t L);
// cache.cu
// the serve graphs bake the handle's table pointers in: dropped (and captured
// again) whenever a setter changes one
void gids_drop_serve_graphs(gids_handle* h);
int gids_launch_serve(gids_handle* h, const int64_t* unique, int64_t n, uint64_t epoch,
                      float* out, cudaStream_t st, cudaStream_t gst);
int gids_launch_window(gids_handle* h, const int64_t* nodes, int64_t n, int delta,
                       cudaStream_t st);
int gids_launch_contribution(gids_handle* h, cudaStream_t st);
// shard.cu
int gids_launch_shard_serve(gids_handle* h, const int64_t* uniq, int64_t n, float* out,
                            cudaStream_t st, cudaStream_t gst, int par);
// storage_file.cu
int gids_file_plan(gids_handle* h, int par, cudaStream_t st);
int gids_file_fetch_and_gather(gids_handle* h, int par, float* out, cudaStream_t gst);
void gids_file_free(gids_handle* h);
// gather.cu
int gids_launch_gather(gids_handle* h, const int64_t* unique, int64_t n, float* out,
                       cudaStream_t st, const ServeArgs* sa = nullptr);

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
static inline int gids_grid(int64_t work, int block, int max_blocks) {
    int64_t g = ceil_div(work, block);
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (int)g;
}
constexpr int GIDS_SMS = 148;
constexpr int GIDS_JUMP_TAB = 128 + 2 * 1025;  // sampler LCG tables (sampler.cu)
