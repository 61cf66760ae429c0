/*
 * gids.h -- C ABI of the B200 GIDS dataloader hot path (libgids.so).
 *
 * Plain pointers and sizes only; no torch types.  Device pointers are raw
 * CUDA device addresses (e.g. torch.Tensor.data_ptr() of a cuda tensor);
 * streams are cudaStream_t passed as void* (0 = legacy default stream).
 * Every entry point returns 0 on success and a negative GIDS_E_* code on
 * failure; gids_last_error() then holds a message.  A handle is bound to
 * one device and is not thread-safe (the reference is single-writer,
 * SPEC.md:386,468).
 *
 * Each entry point names the reference interface it replaces, relative to
 * /root/reference/pkg/src/tierloader/.  The Python side that calls this ABI
 * (paper_2306_16384_b200/) keeps those interfaces' names, argument meaning
 * and exceptions; see INTEGRATION.md for the binding.
 */
#ifndef GIDS_H_
#define GIDS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GIDS_ABI_VERSION 1

#if defined(__GNUC__)
#define GIDS_API __attribute__((visibility("default")))
#else
#define GIDS_API
#endif

enum {
    GIDS_OK = 0,
    GIDS_E_INVALID = -1,   /* bad argument (maps to ValueError) */
    GIDS_E_CUDA = -2,      /* CUDA runtime failure */
    GIDS_E_CAPACITY = -3,  /* a workspace bound was exceeded */
    GIDS_E_STATE = -4      /* call out of protocol order (CacheProtocolError) */
};

enum { GIDS_POLICY_EXACT = 0, GIDS_POLICY_SETASSOC = 1 };
enum { GIDS_KIND_HIT = 0, GIDS_KIND_MISS = 1, GIDS_KIND_BYPASS = 2 };

#define GIDS_MAX_LAYERS 8

typedef struct gids_handle gids_handle;

typedef struct {
    int64_t num_nodes;        /* N (< 2^31) */
    int64_t num_edges;        /* E */
    int32_t feature_dim;      /* fp32 columns per row */
    int32_t device;           /* CUDA ordinal */
    int64_t cache_lines;      /* capacity in rows: PipelineConfig.resolved_cache_lines() */
    int32_t policy;           /* GIDS_POLICY_* */
    int32_t ways;             /* set-associative ways (32) */
    uint64_t evict_key;       /* set-associative eviction draw key */
    int32_t window_depth;     /* W (<= 255) */
    int32_t n_layers;         /* len(fanouts) */
    int32_t fanouts[GIDS_MAX_LAYERS];
    int64_t max_seeds;        /* largest batch the workspace must hold */
} gids_config;

/* per-batch tier split, as IterationStats counts it (dataloader.py:48-63) */
typedef struct {
    int64_t sampled, cache_hits, cpu_buffer_hits, storage, bypasses;
} gids_tier_counts;

/* CacheState counters (cache.py:104-113,182-187) */
typedef struct {
    int64_t hits, misses, bypasses, evictions, total_increments, total_decrements;
    int64_t safe_count, filled;
} gids_cache_counters;

GIDS_API int gids_abi_version(void);
GIDS_API const char* gids_last_error(void);

/* Dataloader.__init__ device-side setup (dataloader.py:98-159).
 * Allocates the HBM cache (cache.py:94-113: CacheState + _cache_rows) and
 * the per-node metadata.  eviction_rng: the 6-word PCG64 state of
 * default_rng(evict_seed) (cache.py:108), word order
 * [state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger]. */
GIDS_API int gids_create(const gids_config* cfg, const uint64_t eviction_rng[6], gids_handle** out);
GIDS_API int gids_destroy(gids_handle* h);

/* GraphCsc (graph.py:46-71): host indptr u64[N+1] / indices u64[E] are
 * copied into HBM (indices narrowed to int32; N < 2^31 is checked). */
GIDS_API int gids_load_graph(gids_handle* h, const uint64_t* indptr, const uint64_t* indices);

/* FeatureStore rows (graph.py:278-301) as the storage tier: a pinned or
 * registrable host table of n_rows x feature_dim fp32, read zero-copy. */
GIDS_API int gids_set_backing(gids_handle* h, const float* table_host, int64_t n_rows);

/* ConstantBuffer (cpu_buffer.py:77-138): node_ids in pin order and their
 * rows (host, pinned or registrable); rows are read zero-copy. */
GIDS_API int gids_set_constant_buffer(gids_handle* h, const int64_t* node_ids, int64_t k,
                             const float* rows_host);

/* sample_subgraph (sampler.py:87-112) into the handle's workspace.
 * seeds: host int64[n_seeds] (validated by the caller as sampler.py:91-96
 * does).  The sampler stream lives on the device: rng (6-word PCG64 state
 * of the sampler Generator) seeds it; NULL continues from where the previous
 * batch left it (the device advances its state by the batch's draws, so
 * consecutive batches need no host round trip).  The caller advances its
 * own Generator by the `draws` reported for each batch
 * (rng.bit_generator.advance(draws)) to stay in step with the reference. */
GIDS_API int gids_sample(gids_handle* h, const int64_t* seeds, int64_t n_seeds,
                const uint64_t* rng, void* stream);

/* sample_layer (sampler.py:50-84) for an explicit frontier: host int64[n]
 * visited in the given order, repeats included (each occurrence draws its
 * own `fanout` doubles), on a handle configured with one fanout.  Same
 * stream semantics, sizes and export as gids_sample; layer 0's edges are
 * grouped by frontier position.  Replaces sampler.py:59-84 for callers that
 * pass a frontier the reference's sample_subgraph would not (unsorted,
 * duplicated). */
GIDS_API int gids_sample_frontier(gids_handle* h, const int64_t* frontier, int64_t n,
                                  const uint64_t* rng, void* stream);

/* Sizes of the last gids_sample (synchronises the stream):
 * layer_len[n_layers], n_unique, draws (doubles consumed), and the run-ahead
 * contribution of the batch (dataloader.py:188-192), counted by this call on
 * the sampling stream against the cache as that stream sees it. */
GIDS_API int gids_sample_sizes(gids_handle* h, int64_t* layer_len, int64_t* n_unique,
                      int64_t* draws, int64_t* contribution);

/* Copy the last sample out: edges as the layers' (E_l,2) int64 [src,dst]
 * arrays back to back; unique_nodes int64[U] ascending.  Device pointers. */
GIDS_API int gids_sample_export(gids_handle* h, int64_t* edges_dev, int64_t* unique_dev, void* stream);

/* Asynchronous export of the last gids_sample, enqueued on `stream` without
 * a host round trip: edges_dev / unique_dev must hold the workspace bounds
 * (gids_sample_capacity); sizes_host (pinned, int64[n_layers + 5]) receives
 * [layer_len..., n_unique, draws, contribution, overflow] when the stream
 * gets there; the contribution slot is 0 -- count it with
 * gids_contribution_async, ordered against the serving stream. */
GIDS_API int gids_sample_export_async(gids_handle* h, int64_t* edges_dev, int64_t* unique_dev,
                                      int64_t* sizes_host, void* stream);
/* gids_sample + gids_sample_export_async in one call (the serving loop's
 * per-batch sampling launch); seeds from pinned host memory copy without a
 * host stall. */
GIDS_API int gids_sample_async(gids_handle* h, const int64_t* seeds, int64_t n_seeds,
                               const uint64_t* rng, void* stream, int64_t* edges_dev,
                               int64_t* unique_dev, int64_t* sizes_host);
GIDS_API int gids_sample_capacity(gids_handle* h, int64_t* edge_cap, int64_t* unique_cap);
/* Run-ahead contribution (dataloader.py:188-192) of an exported batch --
 * its unpinned, non-resident nodes -- against the cache as `stream` reaches
 * the call: n is read through n_ptr (device-visible, e.g. the pinned sizes
 * row of gids_sample_export_async), the count lands in out_host (pinned).
 * Lets a caller sample ahead of the point where the reference samples.
 * Ordered on the device after the last gids_serve's decisions, and the next
 * gids_serve waits for it.  Calls on one handle are serialised on one stream
 * (they share a scratch). */
GIDS_API int gids_contribution_async(gids_handle* h, const int64_t* unique_dev,
                                     const int64_t* n_ptr, int64_t* out_host, void* stream);
/* Device-resident sampler stream state (synchronises; for tests). */
GIDS_API int gids_sampler_rng(gids_handle* h, uint64_t words_out[6]);

/* WindowBuffer.push_iteration / pop_iteration (cache.py:66-91) for an
 * ascending unique device list.  The per-node lookahead count is 8-bit: a
 * push beyond 255 lists in flight returns GIDS_E_CAPACITY (the reference
 * has no bound; the configs use W <= 255), a pop of an empty window
 * GIDS_E_STATE. */
GIDS_API int gids_window_push(gids_handle* h, const int64_t* nodes_dev, int64_t n, void* stream);
GIDS_API int gids_window_pop(gids_handle* h, const int64_t* nodes_dev, int64_t n, void* stream);

/* One served batch (dataloader.py:248-290): window_update (cache.py:190-218),
 * per-node CacheState.access in ascending order (cache.py:144-180) or the
 * set-associative policy, tier chain, gather into out_dev (U x dim fp32,
 * ascending unique order) and cache insertion.  epoch keys the
 * set-associative eviction draws.  The decisions run on `stream`; the row
 * movement runs on `gather_stream` (NULL = same stream) after them, so the
 * next batch's decisions can overlap this batch's gather.  out_dev is
 * complete when gather_stream reaches this point.  Precondition: unique_dev
 * strictly ascending (MiniBatch.unique_nodes is); a violation is detected on
 * the device and reported by the next gids_serve_counts (GIDS_E_INVALID). */
GIDS_API int gids_serve(gids_handle* h, const int64_t* unique_dev, int64_t n, uint64_t epoch,
               float* out_dev, void* stream, void* gather_stream);

/* gids_window_pop(pop_dev), gids_window_push(push_dev), gids_serve(...) as
 * one call (either list may be NULL): the window shift of next_batch
 * (dataloader.py:232-299 -- the served batch leaves the window, the batch W
 * ahead joins) runs on `stream` right before the decisions, inside the
 * serve's launch sequence. */
GIDS_API int gids_serve_shift(gids_handle* h, const int64_t* unique_dev, int64_t n,
                              uint64_t epoch, float* out_dev, void* stream, void* gather_stream,
                              const int64_t* pop_dev, int64_t n_pop, const int64_t* push_dev,
                              int64_t n_push);

/* Tier counts of the last gids_serve: waits for that call's decisions only
 * (an event recorded on its `stream`), not for work queued after it -- the
 * caller may launch the next batches' sampling before asking. */
GIDS_API int gids_serve_counts(gids_handle* h, gids_tier_counts* out);

/* Hand the last gids_serve's batch to `stream` without blocking the host:
 * `stream` waits (device-side) for that call's decisions and its gather.
 * The host-side counterpart of next_batch returning rows the caller's stream
 * may read (dataloader.py:232-299 returns host arrays instead). */
GIDS_API int gids_wait_served(gids_handle* h, void* stream);

/* Per-node decisions of the last gids_serve: kind int8[U] (GIDS_KIND_*) and
 * line int64[U] (-1 on bypass).  Device pointers. */
GIDS_API int gids_serve_decisions(gids_handle* h, int8_t* kind_dev, int64_t* line_dev, void* stream);

/* The cache driven directly (the reference exports CacheState and
 * window_update besides the loader).  gids_cache_window_update: window_update
 * (cache.py:190-218) of `nodes` against the handle's window (gids_window_push
 * / pop); counts_dev int32[n] (optional) receives each node's lookahead count.
 * gids_cache_access: CacheState.access (cache.py:144-180) for n distinct
 * nodes in list order, exact policy; kind_dev int8[n] (GIDS_KIND_*), line_dev
 * int32[n] (-1 on bypass), victim_dev int64[n] (optional: the node each
 * miss evicted -- the previous inserter of that line within this call, else
 * the line's occupant at the call's start; -1 when none).  Device pointers. */
GIDS_API int gids_cache_window_update(gids_handle* h, const int64_t* nodes_dev, int64_t n,
                                      int32_t* counts_dev, void* stream);
GIDS_API int gids_cache_access(gids_handle* h, const int64_t* nodes_dev, int64_t n,
                               int8_t* kind_dev, int32_t* line_dev, int64_t* victim_dev,
                               void* stream);
/* reuse_counter (cache.py:104-113) of every node: uint32[num_nodes], host */
GIDS_API int gids_cache_reuse(gids_handle* h, uint32_t* reuse_host);

GIDS_API int gids_cache_stats(gids_handle* h, gids_cache_counters* out);       /* synchronises */
GIDS_API int gids_cache_rng(gids_handle* h, uint64_t words_out[6]);          /* exact-policy RNG */
/* line table snapshot: node int64[L] (-1 empty), state int8[L] (0 empty,
 * 1 SafeToEvict, 2 InUse) -- LineState (cache.py:38-41).  Host pointers. */
GIDS_API int gids_cache_lines(gids_handle* h, int64_t* node_host, int8_t* state_host);
GIDS_API int64_t gids_cache_capacity(gids_handle* h);

/* Synthetic feature rows (graph.py:256-275) written by the GPU straight into
 * a host (pinned) or device table: rows [row0, row0+n) of an N x dim table. */
GIDS_API int gids_synthesize_rows(int device, uint64_t seed, int64_t row0, int64_t n, int32_t dim,
                         float* dst, void* stream);

/* Verify gathered rows against the synthetic formula (verify_gather,
 * dataloader.py:291-294); returns the mismatching row count in *bad. */
GIDS_API int gids_verify_rows(int device, uint64_t seed, const int64_t* nodes_dev, int64_t n, int32_t dim,
                     const float* rows_dev, int64_t* bad, void* stream);

/* ---- setup-time graph work on the GPU ---- */

/* Uniform random graph with exactly num_edges distinct (src,dst) pairs, in
 * CSC form in HBM (indptr int64[N+1], indices int32[E], sources ascending per
 * destination) -- the reference's "uniform" degree model (graph.py:164-180)
 * made counter-based so it runs at 1.6B edges; definition in
 * csrc/graph_setup.cu.  Fails with GIDS_E_INVALID if an in-degree exceeds 1024. */
GIDS_API int gids_generate_uniform_graph(int device, int64_t num_nodes, int64_t num_edges,
                                         uint64_t seed, int64_t* indptr_dev, int32_t* indices_dev,
                                         void* stream);

/* reverse_pagerank (cpu_buffer.py:26-74, unit edge weights) over a device
 * CSC; scores_dev double[N] receives the same float64 values the reference
 * computes (bit-identical), *iterations / *converged as PageRankResult. */
GIDS_API int gids_reverse_pagerank(int device, int64_t num_nodes, int64_t num_edges,
                                   const int64_t* indptr_dev, const int32_t* indices_dev,
                                   double damping, double tol, int32_t max_iter,
                                   double* scores_dev, int32_t* iterations, int32_t* converged,
                                   void* stream);

/* GraphCsc already in HBM (indptr int64[N+1], indices int32[E], device
 * pointers): copied into the handle like gids_load_graph. */
GIDS_API int gids_load_graph_device(gids_handle* h, const int64_t* indptr_dev,
                                    const int32_t* indices_dev);

/* ---- HBM-sharded feature table across data-parallel ranks ----
 * SURVEY.md section 8(e), config C5 (a 409.6 GB table over 8 GPUs): node v
 * lives in shard v % n_shards at row v / n_shards; every rank samples its own
 * batches and gathers rows from the owners' HBM -- its own shard over HBM,
 * the others as peer loads over NVLink (no collective on the data path).
 * Replaces, for tables larger than one GPU, the FeatureStore lookups of the
 * tier chain (dataloader.py:279-290): with the whole table resident every
 * access is a cache hit. */

/* A shard's own device allocation (IPC handles name whole allocations). */
GIDS_API int gids_device_alloc(int device, int64_t bytes, void** dev_ptr_out);
GIDS_API int gids_device_free(int device, void* dev_ptr);
/* CUDA IPC: export a gids_device_alloc'd shard / open a peer's (64-byte handles). */
GIDS_API int gids_ipc_handle(int device, const void* dev_ptr, uint8_t handle_out[64]);
GIDS_API int gids_ipc_open(int device, const uint8_t handle[64], void** dev_ptr_out);
GIDS_API int gids_ipc_close(int device, void* dev_ptr);

/* shard_ptrs: n_shards device addresses (own or IPC-opened peer memory),
 * each a dense fp32 [rows x feature_dim] shard; switches the handle to the
 * sharded mode (gids_serve then reads rows from the shards). */
GIDS_API int gids_set_sharded_table(gids_handle* h, const uint64_t* shard_ptrs, int32_t n_shards,
                                    int32_t my_shard);
/* rows of the last gids_serve read from this rank's shard / from peers
 * (waits like gids_serve_counts) */
GIDS_API int gids_shard_counts(gids_handle* h, int64_t* local, int64_t* remote);

/* synthetic_feature_rows (graph.py:256-275) for rows row0 + i*stride,
 * i < n, written densely to dst (a shard) */
GIDS_API int gids_synthesize_rows_strided(int device, uint64_t seed, int64_t row0, int64_t stride,
                                          int64_t n, int32_t dim, float* dst, void* stream);

/* ---- file-backed storage tier ----
 * The storage tier read from a file instead of pinned memory: the reference's
 * .gfea layout (graph.py:304-327) -- `offset` header bytes, then fp32 rows --
 * read in pages of `page_bytes` (the GIDS init parameters).
 * Each served batch's storage rows become an ascending, de-duplicated page
 * list (the access accumulator), read as runs of consecutive pages by
 * `io_threads` pread() threads into pinned staging (O_DIRECT when `direct`
 * and page_bytes % 4096 == 0), copied to HBM by one DMA, then gathered.
 * Replaces gids_set_backing; max_pages bounds the staging (0 = automatic). */
GIDS_API int gids_set_storage_file(gids_handle* h, const char* path, int64_t offset,
                                   int32_t page_bytes, int64_t max_pages, int32_t io_threads,
                                   int32_t direct);
/* cumulative pages / bytes read, read calls (runs), host I/O time, O_DIRECT in use */
GIDS_API int gids_storage_file_stats(gids_handle* h, int64_t* pages, int64_t* bytes, int64_t* runs,
                                     double* io_ms, int32_t* direct);

/* Page-lock (and map for zero-copy reads) host memory the caller allocated,
 * e.g. a 2 MiB-page (THP) region for a multi-GB storage tier. */
GIDS_API int gids_host_register(void* ptr, int64_t bytes);
GIDS_API int gids_host_unregister(void* ptr);

/* Per-phase device time (CUDA events on the launching stream), accumulated
 * while profiling is on: out_ms[0] sampling, [1] window + cache policy,
 * [2] hit gather (HBM), [3] host-tier gather (zero-copy), [4] batches
 * served.  gids_set_profiling(h, 1) resets the accumulators. */
GIDS_API int gids_set_profiling(gids_handle* h, int on);
GIDS_API int gids_phase_times(gids_handle* h, double out_ms[5]);

/* Kernel launches issued by this handle since creation (evidence counter). */
GIDS_API int64_t gids_launch_count(gids_handle* h);
/* Serves replayed as CUDA graphs (decisions + rows) since creation (evidence
 * counter; GIDS_NO_GRAPHS=1 launches every kernel directly instead). */
GIDS_API int64_t gids_serve_graph_replays(gids_handle* h);

/* Served batches whose exact-policy decisions were made by the CTA-parallel
 * kernel for a full cache (csrc/exact_par.cu) rather than the sequential warp,
 * counted as gids_serve_counts reads them (evidence counter). */
GIDS_API int64_t gids_exact_par_batches(gids_handle* h);
/* Over those batches: rounds of accesses, rounds ended early by a Lemire
 * rejection / a full change list / a candidate losing its line, then the
 * kernel's SM cycles per phase (draws, T tables, first selects, sort, masks,
 * resolve, candidates, fixed-point passes, verify, commit, ring, spare). */
GIDS_API int gids_exact_par_stats(gids_handle* h, int64_t out[16]);

/* ---- Owner-sharded cache of data-parallel ranks (SURVEY 8(e) exchange step;
 * csrc/shared_cache.cu).  Node v lives only in the cache of rank v % G; the
 * owner decides every rank's accesses of its nodes with the reference policy
 * (gids_cache_window_update + gids_cache_access, cache.py:144-218) in global
 * batch order; requesters peer-load hits from the owner's lines.
 *
 * gids_owner_split: a batch's ascending unique nodes grouped by owner (stable:
 * each group ascending) into out_dev, perm_dev[i] = input position of
 * out_dev[i]; counts_host[G] per-owner sizes (synchronises the stream). */
GIDS_API int gids_owner_split(gids_handle* h, const int64_t* unique_dev, int64_t n, int32_t G,
                              int64_t* out_dev, int32_t* perm_dev, int64_t* counts_host,
                              void* stream);
/* Owner, after gids_cache_access of global batch `batch` (step's first batch
 * step0): flags_dev[i] bit 0 = a hit on a line inserted earlier in this step
 * ("fresh": its row may not have landed); the batch's inserts are stamped. */
GIDS_API int gids_shared_marks(gids_handle* h, const int8_t* kind_dev, const int32_t* line_dev,
                               int64_t n, int32_t batch, int32_t step0, uint8_t* flags_dev,
                               void* stream);
/* Owner, after the step's last batch: bit 1 = this miss is its line's final
 * inserter in the step; packed_dev[i] = line | kind << 32 | flags << 40. */
GIDS_API int gids_shared_final(gids_handle* h, const int8_t* kind_dev, const int32_t* line_dev,
                               const uint8_t* flags_dev, int64_t n, int32_t batch,
                               int64_t* packed_dev, void* stream);
/* Requester: packed decisions (owner-grouped, as split) back in unique order. */
GIDS_API int gids_shared_unsplit(gids_handle* h, const int64_t* packed_dev, const int32_t* perm_dev,
                                 int64_t n, int64_t* dec_dev, void* stream);
/* Requester: hits / constant buffer / storage / bypasses of the batch
 * (dataloader.py:262-277; synchronises). */
GIDS_API int gids_shared_tiers(gids_handle* h, const int64_t* unique_dev, const int64_t* dec_dev,
                               int64_t n, int64_t tiers_out[4], void* stream);
/* Requester: phase 0 gathers every row into out_dev (U x dim) -- non-fresh
 * hits from owner_rows_host[v % G] (device pointers: this rank's cache rows or
 * peers' opened by CUDA IPC), the rest from this handle's host tiers; phase 1
 * (after every rank finished phase 0) writes the final inserters' rows into
 * the owners' lines. */
GIDS_API int gids_shared_gather(gids_handle* h, const int64_t* unique_dev, const int64_t* dec_dev,
                                int64_t n, int32_t G, const uint64_t* owner_rows_host,
                                float* out_dev, int32_t phase, void* stream);
/* The handle's cache rows (device pointer; a whole cudaMalloc allocation, so
 * it can be exported with gids_ipc_handle). */
GIDS_API float* gids_cache_rows_ptr(gids_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* GIDS_H_ */
