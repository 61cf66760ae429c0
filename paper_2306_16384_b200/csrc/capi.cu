// capi.cu -- the extern "C" surface declared in include/gids.h.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "gids_internal.cuh"

static thread_local std::string g_err;
void gids_set_error(const std::string& msg) { g_err = msg; }

size_t gids_exact_smem_bytes(int64_t L, bool with_bits);

namespace {

template <typename T>
int dalloc(T** p, int64_t count, cudaStream_t st = 0) {
    (void)st;
    size_t bytes = sizeof(T) * (size_t)(count > 0 ? count : 1);
    cudaError_t e = cudaMalloc((void**)p, bytes);
    if (e != cudaSuccess) {
        gids_set_error(std::string("cudaMalloc(") + std::to_string(bytes) + "): " +
                       cudaGetErrorString(e));
        return GIDS_E_CUDA;
    }
    return GIDS_OK;
}

#define TRY(x)                \
    do {                      \
        int _rc = (x);        \
        if (_rc) return _rc;  \
    } while (0)

#define CHECK_H(h)                                            \
    do {                                                      \
        if (!(h)) {                                           \
            gids_set_error("null gids handle");               \
            return GIDS_E_INVALID;                            \
        }                                                     \
        cudaError_t _e = cudaSetDevice((h)->device);          \
        if (_e != cudaSuccess) {                              \
            gids_set_error(cudaGetErrorString(_e));           \
            return GIDS_E_CUDA;                               \
        }                                                     \
    } while (0)

// host memory the kernels read zero-copy: pinned already, or register it
int map_host(const void* p, size_t bytes, bool* registered) {
    *registered = false;
    if (!p || bytes == 0) return GIDS_OK;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e == cudaSuccess && (a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice ||
                             a.type == cudaMemoryTypeManaged))
        return GIDS_OK;
    cudaGetLastError();
    GIDS_CUDA_TRY(cudaHostRegister(const_cast<void*>(p), bytes,
                                   cudaHostRegisterMapped | cudaHostRegisterReadOnly));
    *registered = true;
    return GIDS_OK;
}

}  // namespace

// everything after the device allocations: pinned mirrors, initial state,
// events, launch geometry (gids_create destroys the handle if this fails)
static int init_handle(gids_handle* h, const uint64_t* eviction_rng) {
    const int64_t N = h->N, L = h->L;
    GIDS_CUDA_TRY(cudaMallocHost((void**)&h->sc_host, sizeof(SampleCounters)));
    GIDS_CUDA_TRY(cudaMallocHost((void**)&h->svc_host, sizeof(ServeCounters)));
    GIDS_CUDA_TRY(cudaMallocHost((void**)&h->jump_host, sizeof(u128) * GIDS_JUMP_TAB));
    GIDS_CUDA_TRY(cudaMallocHost((void**)&h->rng_host, sizeof(u128) * 2));
    GIDS_CUDA_TRY(cudaMemset(h->pinned_off, 0xff, sizeof(int32_t) * N));
    GIDS_CUDA_TRY(cudaMemset(h->slot_of, 0xff, sizeof(int32_t) * N));
    GIDS_CUDA_TRY(cudaMemset(h->line_node, 0xff, sizeof(int32_t) * (L > 0 ? L : 1)));
    GIDS_CUDA_TRY(cudaMemset(h->last_ins, 0xff, sizeof(int32_t) * (L > 0 ? L : 1)));
    GIDS_CUDA_TRY(cudaMemset(h->safe_bits, 0, sizeof(uint32_t) * 32 * ceil_div(L > 0 ? L : 1, 1024)));
    GIDS_CUDA_TRY(cudaMemset(h->cand_of_slot, 0xff, sizeof(int32_t) * (L > 0 ? L : 1)));
    GIDS_CUDA_TRY(cudaMemset(h->evict_bits, 0, sizeof(uint32_t) * ceil_div(L > 0 ? L : 1, 32)));
    GIDS_CUDA_TRY(cudaMemset(h->blk_cnt, 0, sizeof(uint32_t) * ceil_div(L > 0 ? L : 1, 1024)));
    GIDS_CUDA_TRY(cudaMemset(h->sup_cnt, 0, sizeof(uint32_t) * ceil_div(L > 0 ? L : 1, 32768)));
    GIDS_CUDA_TRY(cudaMemset(h->reuse, 0, sizeof(uint32_t) * N));
    GIDS_CUDA_TRY(cudaMemset(h->future, 0, N));
    GIDS_CUDA_TRY(cudaMemset(h->bm_front, 0, sizeof(uint32_t) * ceil_div(N, 32)));
    GIDS_CUDA_TRY(cudaMemset(h->bm_all, 0, sizeof(uint32_t) * ceil_div(N, 32)));
    CacheMeta m;
    memset(&m, 0, sizeof(m));
    if (eviction_rng)
        for (int i = 0; i < 6; i++) m.rng[i] = eviction_rng[i];
    GIDS_CUDA_TRY(cudaMemcpy(h->meta, &m, sizeof(m), cudaMemcpyHostToDevice));

    // exact policy: keep the safe/evicted bitmaps in shared memory when they fit
    int dev_smem = 0;
    GIDS_CUDA_TRY(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                         h->device));
    size_t with_bits = gids_exact_smem_bytes(L, true), without = gids_exact_smem_bytes(L, false);
    const size_t static_smem = 4096;  // k_exact_seq's event ring
    h->exact_smem = with_bits + static_smem <= (size_t)dev_smem;
    {
        h->host_timing = getenv("GIDS_SERVE_TIMING") && getenv("GIDS_SERVE_TIMING")[0] == '1';
        const char* e = getenv("GIDS_EXACT_PAR");
        // (a cache with a line for every node never fills: the CTA kernel
        // and its launches are skipped)
        h->xp_enabled = !(e && e[0] == '0') && gids_xp_smem_bytes(L) <= (size_t)dev_smem &&
                        h->cfg.policy == GIDS_POLICY_EXACT && L > 0 && L < h->N;
        h->xp_safe_div = (e && e[0] == '2') ? 0 : 16;  // 2: every full-cache batch (tests)
    }
    if (!h->exact_smem && without + static_smem > (size_t)dev_smem) {
        gids_set_error("cache_lines too large for the exact policy (use the set-associative one)");
        gids_destroy(h);
        return GIDS_E_INVALID;
    }
    for (int i = 0; i < 8; i++) GIDS_CUDA_TRY(cudaEventCreate(&h->tev[i]));
    for (int i = 0; i < gids_handle::SRING; i++)
        for (int j = 0; j < 2; j++) GIDS_CUDA_TRY(cudaEventCreate(&h->sev[i][j]));
    // gather residency in warps per SM (GIDS_GATHER_WPS).  2 keeps ~0.6 MB of
    // 16-B loads in flight -- several times the host link's bandwidth-delay
    // product -- and leaves the SMs to sampling and decisions: measured on
    // B200 (profiles/r01_bench_wps_b7_*.json) 1/2/4 warps per SM give the same
    // link rate, while 4 slows the overlapped exact-policy decisions by 30%
    {
        int wps = 2;  // with gather_unroll 2: ~300 KB of loads in flight (profiles/r01_gather_wps_unroll_sweep_c2.txt)
        if (const char* e = getenv("GIDS_GATHER_WPS")) wps = atoi(e);
        if (wps < 1) wps = 1;
        int blocks = (wps * GIDS_SMS + 7) / 8;
        h->gather_blocks = blocks;
        h->gather_unroll = 2;
        // hit gather: 2 blocks per SM with 8 loads in flight per lane keep HBM
        // saturated while leaving each SM room for the other streams' kernels
        // (4 blocks of 256 threads filled every SM for the whole gather, so the
        // next batch's contribution / sampling / decisions waited behind it)
        int hbps = 2;
        if (const char* e = getenv("GIDS_HIT_BPS")) hbps = atoi(e);
        h->hit_blocks = (hbps < 1 ? 1 : hbps > 8 ? 8 : hbps) * GIDS_SMS;
        h->hit_unroll = 8;
        if (const char* e = getenv("GIDS_HIT_UNROLL")) h->hit_unroll = atoi(e) >= 8 ? 8 : 4;
        const char* ng = getenv("GIDS_NO_GRAPHS");
        h->use_graphs = !(ng && ng[0] == '1');
        if (const char* e = getenv("GIDS_GATHER_UNROLL")) {
            int u = atoi(e);
            h->gather_unroll = u >= 8 ? 8 : u >= 4 ? 4 : u >= 2 ? 2 : 1;
        }
    }
    for (int i = 0; i < 2; i++) {
        GIDS_CUDA_TRY(cudaEventCreateWithFlags(&h->gathered[i], cudaEventDisableTiming));
        for (int j = 0; j < 3; j++) GIDS_CUDA_TRY(cudaEventCreate(&h->gev[i][j]));
    }
    GIDS_CUDA_TRY(cudaEventCreateWithFlags(&h->decided, cudaEventDisableTiming));
    GIDS_CUDA_TRY(cudaEventCreateWithFlags(&h->contributed, cudaEventDisableTiming));
    GIDS_CUDA_TRY(cudaEventCreateWithFlags(&h->counted, cudaEventDisableTiming));
    h->kind = h->kind_buf[0];
    h->line = h->line_buf[0];
    h->ins = h->ins_buf[0];
    h->hit_list = h->hit_list_buf[0];
    h->host_list = h->host_list_buf[0];
    h->list_cnt = h->list_cnt_buf[0];
    return GIDS_OK;
}

extern "C" {

int gids_abi_version(void) { return GIDS_ABI_VERSION; }
const char* gids_last_error(void) { return g_err.c_str(); }

int gids_create(const gids_config* cfg, const uint64_t eviction_rng[6], gids_handle** out) {
    if (!cfg || !out) {
        gids_set_error("null argument");
        return GIDS_E_INVALID;
    }
    if (cfg->num_nodes <= 0 || cfg->num_nodes >= (int64_t)1 << 31) {
        gids_set_error("num_nodes must be in [1, 2^31)");
        return GIDS_E_INVALID;
    }
    if (cfg->feature_dim <= 0 || cfg->n_layers < 1 || cfg->n_layers > GIDS_MAX_LAYERS ||
        cfg->cache_lines < 0 || cfg->cache_lines >= (int64_t)1 << 30 || cfg->max_seeds < 1 ||
        cfg->window_depth < 0 || cfg->window_depth > 255) {
        gids_set_error("invalid gids_config (dim, layers 1..8, lines < 2^30, W <= 255)");
        return GIDS_E_INVALID;
    }
    for (int l = 0; l < cfg->n_layers; l++)
        if (cfg->fanouts[l] < 1) {
            gids_set_error("every fanout must be >= 1");
            return GIDS_E_INVALID;
        }
    if (cfg->policy == GIDS_POLICY_SETASSOC && cfg->ways != 32) {
        gids_set_error("set-associative policy supports 32 ways");
        return GIDS_E_INVALID;
    }
    GIDS_CUDA_TRY(cudaSetDevice(cfg->device));
    gids_handle* h = new gids_handle();
    memset((void*)h, 0, sizeof(gids_handle));
    h->cfg = *cfg;
    h->device = cfg->device;
    h->N = cfg->num_nodes;
    h->E = cfg->num_edges;
    h->row_floats = cfg->feature_dim;
    if (cfg->policy == GIDS_POLICY_SETASSOC) {
        h->sets = cfg->cache_lines / 32;
        h->L = h->sets * 32;
        if (h->L == 0) h->cfg.policy = GIDS_POLICY_EXACT;  // no sets: bypass-only cache
    } else {
        h->L = cfg->cache_lines;
    }
    const int64_t N = h->N, L = h->L;

    // workspace bounds (sampler.py: every layer edge <= frontier * fanout)
    h->max_seeds = cfg->max_seeds;
    // (layer 0 may be an explicit frontier with repeats: gids_sample_frontier)
    int64_t front = cfg->max_seeds, ecap = 0, fcap = front;
    for (int l = 0; l < cfg->n_layers; l++) {
        int64_t e = front * cfg->fanouts[l];
        ecap += e;
        front = e < N ? e : N;
        fcap = front > fcap ? front : fcap;
    }
    h->edge_cap = ecap > 0 ? ecap : 1;
    h->front_cap = fcap;
    h->unique_cap = (cfg->max_seeds + ecap) < N ? (cfg->max_seeds + ecap) : N;
    h->serve_cap = h->unique_cap;

    int rc = GIDS_OK;
#define A(ptr, cnt) \
    if (!rc) rc = dalloc(&(ptr), (cnt))
    A(h->indptr, N + 1);
    A(h->indices, h->E > 0 ? h->E : 1);
    A(h->pinned_off, N);
    A(h->cache_rows, L * h->row_floats);
    A(h->slot_of, N);
    A(h->line_node, L);
    A(h->safe_bits, 32 * ceil_div(L > 0 ? L : 1, 1024));  // whole 1024-line blocks (exact_par.cu)
    A(h->cand_of_slot, L);
    A(h->cand_slot, GIDS_XP_CAND_CAP);
    A(h->xcls, h->serve_cap);
    h->xp_hcap = h->serve_cap + h->serve_cap / 32 + 4096;
    A(h->xp_halves, h->xp_hcap);
    A(h->evict_bits, ceil_div(L, 32));
    A(h->blk_cnt, ceil_div(L, 1024));
    A(h->sup_cnt, ceil_div(L, 32768));
    A(h->reuse, N);
    A(h->future, ceil_div(N, 4) * 4);  // (k_window_shift: 32-bit atomics on byte lanes)
    A(h->meta, 1);
    A(h->last_ins, L);
    A(h->bm_front, ceil_div(N, 32));
    A(h->bm_all, ceil_div(N, 32));
    A(h->frontier, h->front_cap);
    A(h->seeds_dev, h->max_seeds);
    A(h->take_off, h->front_cap + 1);
    A(h->draw_off, h->front_cap + 1);
    A(h->edges, 2 * h->edge_cap);
    A(h->unique32, h->unique_cap);
    A(h->jump_tab, GIDS_JUMP_TAB);
    A(h->rng_dev, 2);
    h->lb_tiles = ceil_div(ceil_div(N, 32), 256);
    A(h->sc, 1 + ceil_div((int64_t)sizeof(LbTile) * (cfg->n_layers + 1) * h->lb_tiles,
                          (int64_t)sizeof(SampleCounters)));
    A(h->contrib_dev, 2);
    if (!rc) rc = cudaMemset(h->contrib_dev, 0, 2 * sizeof(int64_t)) == cudaSuccess ? GIDS_OK
                                                                                 : GIDS_E_CUDA;
    h->scan_parts_cap = 1024;
    A(h->scan_parts, 2 * h->scan_parts_cap);
    A(h->word_parts, h->scan_parts_cap);
    A(h->serve_parts, 2 * h->scan_parts_cap);
    A(h->serve_word_parts, h->scan_parts_cap);
    A(h->ev, h->serve_cap);
    for (int b = 0; b < 2; b++) {
        A(h->kind_buf[b], h->serve_cap);
        A(h->line_buf[b], h->serve_cap);
        A(h->ins_buf[b], h->serve_cap);
        A(h->hit_list_buf[b], h->serve_cap);
        A(h->host_list_buf[b], h->serve_cap);
        A(h->list_cnt_buf[b], 2);
    }
    A(h->sargs, 2);
    A(h->log_line, h->serve_cap);
    A(h->log_pos, h->serve_cap);
    A(h->set_cnt, h->sets);
    A(h->set_off, h->sets + 1);
    A(h->set_cur, h->sets);
    A(h->bucket, h->serve_cap);
    A(h->svc, 1);
#undef A
    if (rc) {
        gids_destroy(h);
        return rc;
    }
    rc = init_handle(h, eviction_rng);
    if (rc) {  // no partially built handle escapes
        gids_destroy(h);
        return rc;
    }
    *out = h;
    return GIDS_OK;
}

int gids_destroy(gids_handle* h) {
    if (!h) return GIDS_OK;
    if (h->host_timing && h->host_calls)
        fprintf(stderr, "gids serve host us/call: wait %.1f memset %.1f consume %.1f policy %.1f "
                "tiers %.1f select %.1f counts %.1f gather %.1f (%lld calls)\n",
                h->host_ns[0] / h->host_calls / 1e3, h->host_ns[1] / h->host_calls / 1e3,
                h->host_ns[2] / h->host_calls / 1e3, h->host_ns[3] / h->host_calls / 1e3,
                h->host_ns[4] / h->host_calls / 1e3, h->host_ns[5] / h->host_calls / 1e3,
                h->host_ns[6] / h->host_calls / 1e3, h->host_ns[7] / h->host_calls / 1e3,
                (long long)h->host_calls);
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    gids_file_free(h);
    for (int i = 0; i < h->n_sgraphs; i++)
        if (h->sgraphs[i].exec) cudaGraphExecDestroy(h->sgraphs[i].exec);
    for (int i = 0; i < 2; i++) {
        if (h->dgraph[i]) cudaGraphExecDestroy(h->dgraph[i]);
        if (h->ggraph[i]) cudaGraphExecDestroy(h->ggraph[i]);
    }
    void* ptrs[] = {h->indptr,    h->indices,  h->pinned_off, h->cache_rows, h->slot_of,
                    h->line_node, h->safe_bits, h->evict_bits, h->blk_cnt,   h->sup_cnt,
                    h->reuse,     h->future,   h->meta,       h->last_ins,   h->bm_front,
                    h->bm_all,    h->frontier, h->seeds_dev,  h->take_off,   h->draw_off,
                    h->edges,     h->unique32, h->jump_tab,   h->rng_dev,    h->sc,
                    h->scan_parts,
                    h->word_parts, h->ev,      h->kind_buf[0], h->line_buf[0], h->ins_buf[0],
                    h->kind_buf[1], h->line_buf[1], h->ins_buf[1],            h->log_line,
                    h->log_pos,   h->set_cnt,  h->set_off,    h->set_cur,    h->bucket,
                    h->svc,       h->hit_list_buf[0], h->hit_list_buf[1], h->host_list_buf[0],
                    h->host_list_buf[1], h->list_cnt_buf[0], h->list_cnt_buf[1],
                    (void*)h->shard_ptrs, h->contrib_dev,
                    h->serve_parts, h->serve_word_parts, h->cand_of_slot, h->cand_slot,
                    h->xcls,      h->xp_halves, h->line_mark, h->shared_rows, h->sargs};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (int i = 0; i < 8; i++)
        if (h->tev[i]) cudaEventDestroy(h->tev[i]);
    for (int i = 0; i < gids_handle::SRING; i++)
        for (int j = 0; j < 2; j++)
            if (h->sev[i][j]) cudaEventDestroy(h->sev[i][j]);
    for (int i = 0; i < 2; i++) {
        if (h->gathered[i]) cudaEventDestroy(h->gathered[i]);
        for (int j = 0; j < 3; j++)
            if (h->gev[i][j]) cudaEventDestroy(h->gev[i][j]);
    }
    if (h->decided) cudaEventDestroy(h->decided);
    if (h->counted) cudaEventDestroy(h->counted);
    if (h->contributed) cudaEventDestroy(h->contributed);
    if (h->sc_host) cudaFreeHost(h->sc_host);
    if (h->jump_host) cudaFreeHost(h->jump_host);
    if (h->rng_host) cudaFreeHost(h->rng_host);
    if (h->svc_host) cudaFreeHost(h->svc_host);
    if (h->backing_registered) cudaHostUnregister(const_cast<float*>(h->backing));
    if (h->buffer_registered) cudaHostUnregister(const_cast<float*>(h->buffer_rows));
    delete h;
    return GIDS_OK;
}

int gids_load_graph(gids_handle* h, const uint64_t* indptr, const uint64_t* indices) {
    CHECK_H(h);
    const int64_t N = h->N, E = h->E;
    if (!indptr || (E > 0 && !indices)) {
        gids_set_error("null graph array");
        return GIDS_E_INVALID;
    }
    if (indptr[0] != 0 || (int64_t)indptr[N] != E) {
        gids_set_error("indptr must start at 0 and end at num_edges");
        return GIDS_E_INVALID;
    }
    GIDS_CUDA_TRY(cudaMemcpy(h->indptr, indptr, sizeof(int64_t) * (N + 1), cudaMemcpyHostToDevice));
    // narrow indices to int32 in bounded chunks through a pinned staging buffer
    const int64_t chunk = (int64_t)1 << 24;
    int32_t* stage = nullptr;
    GIDS_CUDA_TRY(cudaMallocHost((void**)&stage, sizeof(int32_t) * chunk));
    for (int64_t b = 0; b < E; b += chunk) {
        int64_t n = E - b < chunk ? E - b : chunk;
        for (int64_t i = 0; i < n; i++) {
            uint64_t v = indices[b + i];
            if (v >= (uint64_t)N) {
                cudaFreeHost(stage);
                gids_set_error("node " + std::to_string(v) + " out of range (num_nodes=" +
                               std::to_string(N) + ")");
                return GIDS_E_INVALID;
            }
            stage[i] = (int32_t)v;
        }
        cudaError_t e = cudaMemcpy(h->indices + b, stage, sizeof(int32_t) * n,
                                   cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFreeHost(stage);
            gids_set_error(cudaGetErrorString(e));
            return GIDS_E_CUDA;
        }
    }
    cudaFreeHost(stage);
    return GIDS_OK;
}

int gids_load_graph_device(gids_handle* h, const int64_t* indptr, const int32_t* indices) {
    CHECK_H(h);
    if (!indptr || (h->E > 0 && !indices)) {
        gids_set_error("null graph array");
        return GIDS_E_INVALID;
    }
    int64_t ends[2] = {0, 0};
    GIDS_CUDA_TRY(cudaMemcpy(&ends[0], indptr, sizeof(int64_t), cudaMemcpyDeviceToHost));
    GIDS_CUDA_TRY(cudaMemcpy(&ends[1], indptr + h->N, sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (ends[0] != 0 || ends[1] != h->E) {
        gids_set_error("indptr must start at 0 and end at num_edges");
        return GIDS_E_INVALID;
    }
    GIDS_CUDA_TRY(cudaMemcpy(h->indptr, indptr, sizeof(int64_t) * (h->N + 1),
                             cudaMemcpyDeviceToDevice));
    if (h->E > 0)
        GIDS_CUDA_TRY(cudaMemcpy(h->indices, indices, sizeof(int32_t) * h->E,
                                 cudaMemcpyDeviceToDevice));
    return GIDS_OK;
}

int gids_set_backing(gids_handle* h, const float* table, int64_t n_rows) {
    CHECK_H(h);
    gids_drop_serve_graphs(h);
    if (n_rows != h->N) {
        gids_set_error("feature table and graph disagree on node count");
        return GIDS_E_INVALID;
    }
    if (h->backing_registered) cudaHostUnregister(const_cast<float*>(h->backing));
    TRY(map_host(table, sizeof(float) * (size_t)n_rows * h->row_floats, &h->backing_registered));
    h->backing = table;
    return GIDS_OK;
}

int gids_set_constant_buffer(gids_handle* h, const int64_t* node_ids, int64_t k,
                             const float* rows) {
    CHECK_H(h);
    gids_drop_serve_graphs(h);
    if (h->buffer_registered) cudaHostUnregister(const_cast<float*>(h->buffer_rows));
    h->buffer_registered = false;
    std::vector<int32_t> off((size_t)h->N, -1);
    for (int64_t i = 0; i < k; i++) {
        int64_t x = node_ids[i];
        if (x < 0 || x >= h->N) {
            gids_set_error("pinned list names nodes outside the feature table");
            return GIDS_E_INVALID;
        }
        off[(size_t)x] = (int32_t)i;
    }
    GIDS_CUDA_TRY(cudaMemcpy(h->pinned_off, off.data(), sizeof(int32_t) * h->N,
                             cudaMemcpyHostToDevice));
    if (k > 0) TRY(map_host(rows, sizeof(float) * (size_t)k * h->row_floats, &h->buffer_registered));
    h->buffer_rows = k > 0 ? rows : nullptr;
    h->buffer_k = k;
    return GIDS_OK;
}

int gids_sample(gids_handle* h, const int64_t* seeds, int64_t n_seeds, const uint64_t* rng,
                void* stream) {
    CHECK_H(h);
    if (n_seeds < 1 || n_seeds > h->max_seeds) {
        gids_set_error("seed count must be in [1, max_seeds]");
        return GIDS_E_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    GIDS_CUDA_TRY(cudaMemcpyAsync(h->seeds_dev, seeds, sizeof(int64_t) * n_seeds,
                                  cudaMemcpyHostToDevice, st));
    h->last_stream = st;
    return gids_launch_sample(h, n_seeds, rng, false, st);
}

int gids_sample_frontier(gids_handle* h, const int64_t* frontier, int64_t n, const uint64_t* rng,
                         void* stream) {
    CHECK_H(h);
    if (n < 1 || n > h->max_seeds) {
        gids_set_error("frontier length must be in [1, max_seeds]");
        return GIDS_E_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    GIDS_CUDA_TRY(cudaMemcpyAsync(h->seeds_dev, frontier, sizeof(int64_t) * n,
                                  cudaMemcpyHostToDevice, st));
    h->last_stream = st;
    return gids_launch_sample(h, n, rng, true, st);
}

int gids_sample_sizes(gids_handle* h, int64_t* layer_len, int64_t* n_unique, int64_t* draws,
                      int64_t* contribution) {
    CHECK_H(h);
    // the contribution is counted here, on the sampling stream after the
    // batch, against the cache as that stream sees it (the serving path
    // counts its admissions with gids_contribution_async instead)
    TRY(gids_launch_contribution(h, h->last_stream));
    GIDS_CUDA_TRY(cudaMemcpyAsync(&h->sc_host->contribution, &h->sc->contribution, sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, h->last_stream));
    GIDS_CUDA_TRY(cudaStreamSynchronize(h->last_stream));
    gids_harvest_sample(h, false);
    const SampleCounters& c = *h->sc_host;
    if (c.overflow) {
        gids_set_error("sampler workspace bound exceeded");
        return GIDS_E_CAPACITY;
    }
    for (int l = 0; l < h->cfg.n_layers; l++) layer_len[l] = c.layer_len[l];
    *n_unique = c.n_unique;
    *draws = c.layer_draw_base[h->cfg.n_layers];
    *contribution = c.contribution;
    return GIDS_OK;
}

int gids_sample_export(gids_handle* h, int64_t* edges_dev, int64_t* unique_dev, void* stream) {
    CHECK_H(h);
    cudaStream_t st = (cudaStream_t)stream;
    const SampleCounters& c = *h->sc_host;
    int64_t e = 0;
    for (int l = 0; l < h->cfg.n_layers; l++) e += c.layer_len[l];
    if (e > 0 && edges_dev)
        GIDS_CUDA_TRY(cudaMemcpyAsync(edges_dev, h->edges, sizeof(int64_t) * 2 * e,
                                      cudaMemcpyDeviceToDevice, st));
    if (unique_dev && c.n_unique > 0) TRY(gids_launch_export_unique(h, unique_dev, st));
    return GIDS_OK;
}

int gids_sample_export_async(gids_handle* h, int64_t* edges_dev, int64_t* unique_dev,
                             int64_t* sizes_host, void* stream) {
    CHECK_H(h);
    cudaStream_t st = (cudaStream_t)stream;
    // sizes: [layer_len[0..L), n_unique, draws, contribution, overflow] (sc->exp),
    // stored into the pinned row by the export kernel itself
    if (edges_dev || unique_dev || sizes_host)
        TRY(gids_launch_export(h, edges_dev, unique_dev, st, sizes_host));
    return GIDS_OK;
}

int gids_sample_async(gids_handle* h, const int64_t* seeds, int64_t n_seeds, const uint64_t* rng,
                      void* stream, int64_t* edges_dev, int64_t* unique_dev, int64_t* sizes_host) {
    TRY(gids_sample(h, seeds, n_seeds, rng, stream));
    return gids_sample_export_async(h, edges_dev, unique_dev, sizes_host, stream);
}

int gids_sample_capacity(gids_handle* h, int64_t* edge_cap, int64_t* unique_cap) {
    CHECK_H(h);
    *edge_cap = h->edge_cap;
    *unique_cap = h->unique_cap;
    return GIDS_OK;
}

int gids_sampler_rng(gids_handle* h, uint64_t words_out[6]) {
    CHECK_H(h);
    GIDS_CUDA_TRY(cudaDeviceSynchronize());
    u128 st[2];
    GIDS_CUDA_TRY(cudaMemcpy(st, h->rng_dev, sizeof(st), cudaMemcpyDeviceToHost));
    words_out[0] = st[0].hi;
    words_out[1] = st[0].lo;
    words_out[2] = st[1].hi;
    words_out[3] = st[1].lo;
    words_out[4] = 0;
    words_out[5] = 0;
    return GIDS_OK;
}

// future[] holds one byte per node: at most 255 lists may be in the window
int gids_window_push(gids_handle* h, const int64_t* nodes, int64_t n, void* stream) {
    CHECK_H(h);
    if (h->window_lists >= 255) {
        gids_set_error("window holds 255 lists (the per-node lookahead count is 8-bit)");
        return GIDS_E_CAPACITY;
    }
    TRY(gids_launch_window(h, nodes, n, +1, (cudaStream_t)stream));
    h->window_lists++;
    return GIDS_OK;
}
int gids_window_pop(gids_handle* h, const int64_t* nodes, int64_t n, void* stream) {
    CHECK_H(h);
    if (h->window_lists <= 0) {
        gids_set_error("window is empty");
        return GIDS_E_STATE;
    }
    TRY(gids_launch_window(h, nodes, n, -1, (cudaStream_t)stream));
    h->window_lists--;
    return GIDS_OK;
}

int gids_serve(gids_handle* h, const int64_t* unique_dev, int64_t n, uint64_t epoch,
               float* out_dev, void* stream, void* gather_stream) {
    CHECK_H(h);
    if (n < 0 || n > h->serve_cap) {
        gids_set_error("batch larger than the serving workspace");
        return GIDS_E_CAPACITY;
    }
    if (n > 0 && !h->backing && h->n_shards == 0 && !h->ft) {
        gids_set_error("no backing store attached (gids_set_backing)");
        return GIDS_E_STATE;
    }
    h->last_stream = (cudaStream_t)stream;
    h->counts_read = false;
    return gids_launch_serve(h, unique_dev, n, epoch, out_dev, (cudaStream_t)stream,
                             gather_stream ? (cudaStream_t)gather_stream : (cudaStream_t)stream);
}

int gids_serve_shift(gids_handle* h, const int64_t* unique_dev, int64_t n, uint64_t epoch,
                     float* out_dev, void* stream, void* gather_stream, const int64_t* pop_dev,
                     int64_t n_pop, const int64_t* push_dev, int64_t n_push) {
    CHECK_H(h);
    if (n_pop < 0 || n_push < 0 || n_pop > h->serve_cap || n_push > h->serve_cap ||
        (n_pop > 0 && !pop_dev) || (n_push > 0 && !push_dev)) {
        gids_set_error("serve_shift: bad window lists");
        return GIDS_E_INVALID;
    }
    const int32_t lists = h->window_lists - (pop_dev ? 1 : 0);
    if (pop_dev && h->window_lists <= 0) {
        gids_set_error("window is empty");
        return GIDS_E_STATE;
    }
    if (push_dev && lists >= 255) {
        gids_set_error("window holds 255 lists (the per-node lookahead count is 8-bit)");
        return GIDS_E_CAPACITY;
    }
    h->shift = WindowShift{pop_dev, pop_dev ? n_pop : 0, push_dev, push_dev ? n_push : 0};
    const int rc = gids_serve(h, unique_dev, n, epoch, out_dev, stream, gather_stream);
    h->shift = WindowShift{nullptr, 0, nullptr, 0};
    if (rc == GIDS_OK) h->window_lists = lists + (push_dev ? 1 : 0);
    return rc;
}

int gids_wait_served(gids_handle* h, void* stream) {
    CHECK_H(h);
    cudaStream_t st = (cudaStream_t)stream;
    if (h->counted_valid) GIDS_CUDA_TRY(cudaStreamWaitEvent(st, h->counted, 0));
    if (h->last_serve_n > 0 && h->gathered_valid[h->parity])
        GIDS_CUDA_TRY(cudaStreamWaitEvent(st, h->gathered[h->parity], 0));
    return GIDS_OK;
}

int gids_serve_counts(gids_handle* h, gids_tier_counts* out) {
    CHECK_H(h);
    // waits for the decisions' counts only: work queued on the control stream
    // after the serve (the next batches' sampling) keeps running
    if (h->counted_valid)
        GIDS_CUDA_TRY(cudaEventSynchronize(h->counted));
    else
        GIDS_CUDA_TRY(cudaStreamSynchronize(h->last_stream));
    if (h->serve_timed) {
        float a = 0.f;
        if (cudaEventElapsedTime(&a, h->tev[2], h->tev[3]) == cudaSuccess) h->phase_ms[1] += a;
        cudaGetLastError();
        h->phase_ms[4] += 1.0;
        h->serve_timed = false;
    }
    const ServeCounters& c = *h->svc_host;
    if (c.bad_order) {
        gids_set_error("gids_serve: unique_dev was not strictly ascending (cache state is "
                       "undefined from this batch on)");
        return GIDS_E_INVALID;
    }
    if (!h->counts_read && c.xp_done) {
        h->xp_batches++;
        for (int i = 0; i < 4; i++) h->xp_stats[i] += c.xp_stats[i];
        for (int i = 0; i < 12; i++) h->xp_stats[4 + i] += c.xp_prof[i];
    }
    h->counts_read = true;
    out->sampled = h->last_serve_n;
    out->cache_hits = c.tiers[0];
    out->cpu_buffer_hits = c.tiers[1];
    out->storage = c.tiers[2];
    out->bypasses = c.tiers[3];
    return GIDS_OK;
}

int gids_serve_decisions(gids_handle* h, int8_t* kind_dev, int64_t* line_dev, void* stream) {
    CHECK_H(h);
    cudaStream_t st = (cudaStream_t)stream;
    int64_t n = h->last_serve_n;
    if (n == 0) return GIDS_OK;
    GIDS_CUDA_TRY(cudaMemcpyAsync(kind_dev, h->kind, n, cudaMemcpyDeviceToDevice, st));
    std::vector<int32_t> l32((size_t)n);
    GIDS_CUDA_TRY(cudaMemcpyAsync(l32.data(), h->line, sizeof(int32_t) * n,
                                  cudaMemcpyDeviceToHost, st));
    GIDS_CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<int64_t> l64(l32.begin(), l32.end());
    GIDS_CUDA_TRY(cudaMemcpy(line_dev, l64.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice));
    return GIDS_OK;
}

int gids_cache_stats(gids_handle* h, gids_cache_counters* out) {
    CHECK_H(h);
    GIDS_CUDA_TRY(cudaDeviceSynchronize());
    CacheMeta m;
    GIDS_CUDA_TRY(cudaMemcpy(&m, h->meta, sizeof(m), cudaMemcpyDeviceToHost));
    out->hits = m.hits;
    out->misses = m.misses;
    out->bypasses = m.bypasses;
    out->evictions = m.evictions;
    out->total_increments = m.inc;
    out->total_decrements = m.dec;
    if (h->cfg.policy == GIDS_POLICY_EXACT) {
        out->safe_count = m.safe_count;
        out->filled = m.fill;
    } else {  // derived from the line table
        std::vector<uint32_t> bits((size_t)ceil_div(h->L, 32));
        std::vector<int32_t> nodes((size_t)h->L);
        if (h->L > 0) {
            GIDS_CUDA_TRY(cudaMemcpy(bits.data(), h->safe_bits, 4 * bits.size(),
                                     cudaMemcpyDeviceToHost));
            GIDS_CUDA_TRY(cudaMemcpy(nodes.data(), h->line_node, 4 * nodes.size(),
                                     cudaMemcpyDeviceToHost));
        }
        int64_t sc = 0, fill = 0;
        for (uint32_t b : bits) sc += __builtin_popcount(b);
        for (int32_t x : nodes) fill += x >= 0;
        out->safe_count = sc;
        out->filled = fill;
    }
    return GIDS_OK;
}

int gids_cache_rng(gids_handle* h, uint64_t words_out[6]) {
    CHECK_H(h);
    GIDS_CUDA_TRY(cudaDeviceSynchronize());
    CacheMeta m;
    GIDS_CUDA_TRY(cudaMemcpy(&m, h->meta, sizeof(m), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 6; i++) words_out[i] = m.rng[i];
    return GIDS_OK;
}

int gids_cache_lines(gids_handle* h, int64_t* node_host, int8_t* state_host) {
    CHECK_H(h);
    GIDS_CUDA_TRY(cudaDeviceSynchronize());
    const int64_t L = h->L;
    if (L == 0) return GIDS_OK;
    std::vector<int32_t> nodes((size_t)L);
    std::vector<uint32_t> bits((size_t)ceil_div(L, 32));
    GIDS_CUDA_TRY(cudaMemcpy(nodes.data(), h->line_node, 4 * L, cudaMemcpyDeviceToHost));
    GIDS_CUDA_TRY(cudaMemcpy(bits.data(), h->safe_bits, 4 * bits.size(), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < L; i++) {
        node_host[i] = nodes[(size_t)i];
        bool safe = (bits[(size_t)(i >> 5)] >> (i & 31)) & 1u;
        state_host[i] = nodes[(size_t)i] < 0 ? 0 : (safe ? 1 : 2);
    }
    return GIDS_OK;
}

int gids_set_profiling(gids_handle* h, int on) {
    CHECK_H(h);
    h->profiling = on != 0;
    gids_harvest_sample(h, true);  // drop intervals of the previous session
    h->serve_timed = false;
    h->gather_pending[0] = h->gather_pending[1] = false;
    for (int i = 0; i < 5; i++) h->phase_ms[i] = 0.0;
    return GIDS_OK;
}

int gids_phase_times(gids_handle* h, double out_ms[5]) {
    CHECK_H(h);
    gids_harvest_sample(h, true);
    gids_harvest_gather(h, 0);
    gids_harvest_gather(h, 1);
    for (int i = 0; i < 5; i++) out_ms[i] = h->phase_ms[i];
    return GIDS_OK;
}

int gids_host_register(void* ptr, int64_t bytes) {
    if (!ptr || bytes <= 0) {
        gids_set_error("host_register: bad arguments");
        return GIDS_E_INVALID;
    }
    GIDS_CUDA_TRY(cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterMapped));
    return GIDS_OK;
}

int gids_host_unregister(void* ptr) {
    GIDS_CUDA_TRY(cudaHostUnregister(ptr));
    return GIDS_OK;
}

int64_t gids_cache_capacity(gids_handle* h) { return h ? h->L : -1; }
int64_t gids_serve_graph_replays(gids_handle* h) { return h ? h->serve_replays : 0; }

int64_t gids_launch_count(gids_handle* h) { return h ? h->launches : -1; }
int64_t gids_exact_par_batches(gids_handle* h) { return h ? h->xp_batches : -1; }
int gids_exact_par_stats(gids_handle* h, int64_t out[12]) {
    CHECK_H(h);
    for (int i = 0; i < 16; i++) out[i] = h->xp_stats[i];
    return GIDS_OK;
}

}  // extern "C"
