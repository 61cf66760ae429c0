// shared_cache.cu -- the owner-sharded cache of data-parallel ranks
// ("one exchange step per global step").
//
// G ranks each serve their own batches; node v is owned by rank v % G, whose
// HBM cache lines are the only cache v can live in.  Per global step (G
// batches, global batch id b = step * G + rank):
//   requester  splits its batch's ascending unique nodes by owner
//              (gids_owner_split) and sends each owner its list
//   owner      runs the reference policy (window_update + CacheState.access,
//              cache.py:144-218, the standalone entry points in cache.cu) over
//              the G lists it received, in global batch order, and marks each
//              access: a hit on a line inserted earlier in this step is
//              "fresh" (its row may not have landed yet), a miss whose line
//              no later batch of the step re-inserts is the line's "final"
//              inserter (gids_shared_marks / gids_shared_final)
//   requester  gets its decisions back (packed, gids_shared_unsplit), gathers:
//              hits from the owner's cache line (its own HBM or a peer's over
//              NVLink, CUDA IPC pointers), everything else -- misses,
//              bypasses, fresh hits -- from its host tiers (constant buffer or
//              backing store over its own link); after a cross-rank barrier
//              the final inserters write their rows into the owners' lines
//              (peer stores), so every hit of a step reads lines as they were
//              when the step began
// The multi-rank oracle is one reference CacheState per owner driven by its
// owned nodes of every batch in global batch order (tests/test_gpu_shared_cache.py).
#include <vector>

#include "gids_internal.cuh"

#define CHECK_H(h)                                   \
    do {                                             \
        if (!(h)) {                                  \
            gids_set_error("null gids handle");      \
            return GIDS_E_INVALID;                   \
        }                                            \
        GIDS_CUDA_TRY(cudaSetDevice((h)->device));   \
    } while (0)

namespace {

constexpr int SB = 256;  // owner-split block: one element per thread
constexpr int SW = SB / 32;
constexpr int MAXG = 64;

// per block, per owner counts (owner-major: cnt[o * nblk + blk])
__global__ void k_own_count(const int64_t* __restrict__ u, int64_t n, int32_t G, int32_t* cnt,
                            int32_t nblk) {
    __shared__ int32_t c[MAXG];
    for (int i = threadIdx.x; i < G; i += SB) c[i] = 0;
    __syncthreads();
    const int64_t p = (int64_t)blockIdx.x * SB + threadIdx.x;
    if (p < n) atomicAdd(&c[(int32_t)(u[p] % G)], 1);
    __syncthreads();
    for (int i = threadIdx.x; i < G; i += SB) cnt[(int64_t)i * nblk + blockIdx.x] = c[i];
}

// stable scatter: out[off] = u[p], perm[off] = p, off = owner's exclusive offset
// over (owner, block) + rank among the block's earlier elements of that owner
__global__ void k_own_scatter(const int64_t* __restrict__ u, int64_t n, int32_t G,
                              const int64_t* __restrict__ off, int32_t nblk, int64_t* out,
                              int32_t* perm) {
    __shared__ int32_t wc[SW][MAXG];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t p = (int64_t)blockIdx.x * SB + threadIdx.x;
    const int32_t o = p < n ? (int32_t)(u[p] % G) : -1;
    int32_t rk = 0;
    for (int g = 0; g < G; g++) {
        const unsigned m = __ballot_sync(0xffffffffu, o == g);
        if (o == g) rk = __popc(m & ((1u << lane) - 1u));
        if (lane == 0) wc[w][g] = __popc(m);
    }
    __syncthreads();
    if (p < n) {
        int64_t at = off[(int64_t)o * nblk + blockIdx.x] + rk;
        for (int ww = 0; ww < w; ww++) at += wc[ww][o];
        out[at] = u[p];
        perm[at] = (int32_t)p;
    }
}

// owner side: fresh hits (their line was inserted earlier in this step), then
// this batch's inserts are stamped (batch id, position) -- the stamp of a line
// is its last insert: later batch, or later position in the same batch (a line
// filled and evicted again within one batch)
__device__ __forceinline__ unsigned long long stamp_of(int32_t batch, int64_t pos) {
    return ((unsigned long long)(uint32_t)batch << 32) | (unsigned long long)(uint32_t)pos;
}
__global__ void k_marks(const int8_t* __restrict__ kind, const int32_t* __restrict__ line,
                        int64_t n, int32_t batch, int32_t step0,
                        const unsigned long long* __restrict__ line_mark, uint8_t* flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint8_t f = 0;
        if (kind[i] == GIDS_KIND_HIT) {
            const unsigned long long m = line_mark[line[i]];
            if (m != ~0ull && (int64_t)(m >> 32) >= step0) f = 1;
        }
        flags[i] = f;
    }
}
__global__ void k_stamp(const int8_t* __restrict__ kind, const int32_t* __restrict__ line,
                        int64_t n, int32_t batch, unsigned long long* line_mark) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (kind[i] == GIDS_KIND_MISS) {
            unsigned long long* m = &line_mark[line[i]];
            if (*m == ~0ull) atomicCAS(m, ~0ull, 0ull);  // (unstamped: below any stamp)
            atomicMax(m, stamp_of(batch, i));
        }
}
// after the step: a miss is its line's final inserter when no later insert of
// the step stamped the line; pack (line, kind, flags) for the return trip
__global__ void k_final_pack(const int8_t* __restrict__ kind, const int32_t* __restrict__ line,
                             const uint8_t* __restrict__ flags, int64_t n, int32_t batch,
                             const unsigned long long* __restrict__ line_mark, int64_t* packed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int k = kind[i];
        uint32_t f = flags[i];
        if (k == GIDS_KIND_MISS && line_mark[line[i]] == stamp_of(batch, i)) f |= 2u;
        packed[i] = (int64_t)(uint32_t)line[i] | ((int64_t)(k & 0xff) << 32) | ((int64_t)f << 40);
    }
}

// requester: decisions back in unique order
__global__ void k_unsplit(const int64_t* __restrict__ packed, const int32_t* __restrict__ perm,
                          int64_t n, int64_t* dec) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dec[perm[i]] = packed[i];
}

__device__ __forceinline__ int dec_kind(int64_t d) { return (int)((d >> 32) & 0xff); }
__device__ __forceinline__ int dec_flags(int64_t d) { return (int)((d >> 40) & 0xff); }
__device__ __forceinline__ int32_t dec_line(int64_t d) { return (int32_t)(uint32_t)d; }

// tier split of a batch (dataloader.py:262-277): hits, buffer, storage, bypasses
__global__ void k_shared_tiers(const int64_t* __restrict__ u, const int64_t* __restrict__ dec,
                               int64_t n, const int32_t* __restrict__ pinned_off,
                               unsigned long long* t) {
    unsigned long long a = 0, b = 0, c = 0, d = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int k = dec_kind(dec[i]);
        if (k == GIDS_KIND_HIT) {
            a++;
        } else {
            if (pinned_off[u[i]] >= 0) b++;
            else c++;
            if (k == GIDS_KIND_BYPASS) d++;
        }
    }
    atomicAdd(&t[0], a);
    atomicAdd(&t[1], b);
    atomicAdd(&t[2], c);
    atomicAdd(&t[3], d);
}

// phase 0: every row of the batch -- non-fresh hits from the owner's line,
// the rest from this rank's host tiers; phase 1: final inserters' rows into
// the owners' lines.  One warp per row, 16-B or 4-B elements.
template <typename T>
__global__ void __launch_bounds__(256)
k_shared_gather(const int64_t* __restrict__ u, const int64_t* __restrict__ dec, int64_t n,
                int32_t G, T* const* __restrict__ owner_rows, const int32_t* __restrict__ pinned_off,
                const T* __restrict__ buffer_rows, const T* __restrict__ backing, T* __restrict__ out,
                int64_t cpr, int phase) {
    const int lane = threadIdx.x & 31;
    for (int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; p < n;
         p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t d = dec[p], x = u[p];
        const int k = dec_kind(d), f = dec_flags(d);
        T* dst = out + p * cpr;
        if (phase == 0) {
            const T* src;
            if (k == GIDS_KIND_HIT && !(f & 1)) {
                src = owner_rows[x % G] + (int64_t)dec_line(d) * cpr;
            } else {
                const int32_t b = pinned_off[x];
                src = b >= 0 ? buffer_rows + (int64_t)b * cpr : backing + x * cpr;
            }
            for (int64_t c = lane; c < cpr; c += 32) dst[c] = src[c];
        } else if (k == GIDS_KIND_MISS && (f & 2)) {
            T* line = owner_rows[x % G] + (int64_t)dec_line(d) * cpr;
            for (int64_t c = lane; c < cpr; c += 32) line[c] = dst[c];
        }
    }
}

}  // namespace

extern "C" {

int gids_owner_split(gids_handle* h, const int64_t* unique_dev, int64_t n, int32_t G,
                     int64_t* out_dev, int32_t* perm_dev, int64_t* counts_host, void* stream) {
    if (!h || n < 0 || G < 1 || G > MAXG || (n > 0 && (!unique_dev || !out_dev || !perm_dev)) ||
        !counts_host) {
        gids_set_error("owner_split: bad arguments (1 <= G <= 64)");
        return GIDS_E_INVALID;
    }
    GIDS_CUDA_TRY(cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)stream;
    for (int g = 0; g < G; g++) counts_host[g] = 0;
    if (n == 0) return GIDS_OK;
    const int32_t nblk = (int32_t)ceil_div(n, SB);
    const int64_t m = (int64_t)nblk * G;
    int32_t* cnt = nullptr;
    int64_t* off = nullptr;
    GIDS_CUDA_TRY(cudaMallocAsync((void**)&cnt, sizeof(int32_t) * m, st));
    GIDS_CUDA_TRY(cudaMallocAsync((void**)&off, sizeof(int64_t) * (m + 1), st));
    k_own_count<<<nblk, SB, 0, st>>>(unique_dev, n, G, cnt, nblk);
    GIDS_LAUNCH_CHECK(h);
    int rc = gids_scan_i32_to_i64(h, cnt, m, off, st);
    if (rc) return rc;
    k_own_scatter<<<nblk, SB, 0, st>>>(unique_dev, n, G, off, nblk, out_dev, perm_dev);
    GIDS_LAUNCH_CHECK(h);
    // per-owner counts: differences of the owners' first offsets
    std::vector<int64_t> first(G + 1);
    for (int g = 0; g < G; g++)
        GIDS_CUDA_TRY(cudaMemcpyAsync(&first[g], off + (int64_t)g * nblk, sizeof(int64_t),
                                      cudaMemcpyDeviceToHost, st));
    GIDS_CUDA_TRY(cudaStreamSynchronize(st));
    first[G] = n;
    for (int g = 0; g < G; g++) counts_host[g] = first[g + 1] - first[g];
    cudaFreeAsync(cnt, st);
    cudaFreeAsync(off, st);
    return GIDS_OK;
}

// owner side, after gids_cache_access of one batch's owned list
int gids_shared_marks(gids_handle* h, const int8_t* kind_dev, const int32_t* line_dev, int64_t n,
                      int32_t batch, int32_t step0, uint8_t* flags_dev, void* stream) {
    CHECK_H(h);
    if (n < 0 || batch < 0 || step0 < 0 || step0 > batch) {
        gids_set_error("shared_marks: bad arguments");
        return GIDS_E_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (!h->line_mark) {  // ~0: never inserted through the shared path
        const size_t b = sizeof(unsigned long long) * (h->L > 0 ? h->L : 1);
        GIDS_CUDA_TRY(cudaMalloc((void**)&h->line_mark, b));
        GIDS_CUDA_TRY(cudaMemset(h->line_mark, 0xff, b));
    }
    if (n == 0) return GIDS_OK;
    const int g = gids_grid(n, 256, 8 * GIDS_SMS);
    k_marks<<<g, 256, 0, st>>>(kind_dev, line_dev, n, batch, step0, h->line_mark, flags_dev);
    GIDS_LAUNCH_CHECK(h);
    k_stamp<<<g, 256, 0, st>>>(kind_dev, line_dev, n, batch, h->line_mark);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

int gids_shared_final(gids_handle* h, const int8_t* kind_dev, const int32_t* line_dev,
                      const uint8_t* flags_dev, int64_t n, int32_t batch, int64_t* packed_dev,
                      void* stream) {
    CHECK_H(h);
    if (n == 0) return GIDS_OK;
    if (!h->line_mark) {
        gids_set_error("shared_final: no marks (call gids_shared_marks first)");
        return GIDS_E_STATE;
    }
    k_final_pack<<<gids_grid(n, 256, 8 * GIDS_SMS), 256, 0, (cudaStream_t)stream>>>(
        kind_dev, line_dev, flags_dev, n, batch, h->line_mark, packed_dev);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

int gids_shared_unsplit(gids_handle* h, const int64_t* packed_dev, const int32_t* perm_dev,
                        int64_t n, int64_t* dec_dev, void* stream) {
    CHECK_H(h);
    if (n == 0) return GIDS_OK;
    k_unsplit<<<gids_grid(n, 256, 8 * GIDS_SMS), 256, 0, (cudaStream_t)stream>>>(packed_dev,
                                                                                 perm_dev, n,
                                                                                 dec_dev);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

int gids_shared_tiers(gids_handle* h, const int64_t* unique_dev, const int64_t* dec_dev,
                      int64_t n, int64_t tiers_out[4], void* stream) {
    CHECK_H(h);
    cudaStream_t st = (cudaStream_t)stream;
    for (int i = 0; i < 4; i++) tiers_out[i] = 0;
    if (n == 0) return GIDS_OK;
    unsigned long long* t = nullptr;
    GIDS_CUDA_TRY(cudaMallocAsync((void**)&t, sizeof(unsigned long long) * 4, st));
    GIDS_CUDA_TRY(cudaMemsetAsync(t, 0, sizeof(unsigned long long) * 4, st));
    k_shared_tiers<<<gids_grid(n, 256, 4 * GIDS_SMS), 256, 0, st>>>(unique_dev, dec_dev, n,
                                                                   h->pinned_off, t);
    GIDS_LAUNCH_CHECK(h);
    unsigned long long host[4];
    GIDS_CUDA_TRY(cudaMemcpyAsync(host, t, sizeof(host), cudaMemcpyDeviceToHost, st));
    GIDS_CUDA_TRY(cudaStreamSynchronize(st));
    cudaFreeAsync(t, st);
    for (int i = 0; i < 4; i++) tiers_out[i] = (int64_t)host[i];
    return GIDS_OK;
}

int gids_shared_gather(gids_handle* h, const int64_t* unique_dev, const int64_t* dec_dev,
                       int64_t n, int32_t G, const uint64_t* owner_rows_host, float* out_dev,
                       int32_t phase, void* stream) {
    CHECK_H(h);
    if (n < 0 || G < 1 || G > MAXG || !owner_rows_host || (phase != 0 && phase != 1)) {
        gids_set_error("shared_gather: bad arguments");
        return GIDS_E_INVALID;
    }
    if (n == 0) return GIDS_OK;
    if (!h->backing) {
        gids_set_error("shared_gather: no storage tier (gids_set_backing)");
        return GIDS_E_STATE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (!h->shared_rows || h->shared_rows_g != G) {
        if (h->shared_rows) cudaFree(h->shared_rows);
        GIDS_CUDA_TRY(cudaMalloc((void**)&h->shared_rows, sizeof(uint64_t) * G));
        h->shared_rows_g = G;
    }
    GIDS_CUDA_TRY(cudaMemcpyAsync(h->shared_rows, owner_rows_host, sizeof(uint64_t) * G,
                                  cudaMemcpyHostToDevice, st));
    const int64_t dim = h->row_floats;
    const int grid = gids_grid(n * 32, 256, 16 * GIDS_SMS);
    if ((dim & 3) == 0) {
        k_shared_gather<int4><<<grid, 256, 0, st>>>(
            unique_dev, dec_dev, n, G, reinterpret_cast<int4* const*>(h->shared_rows),
            h->pinned_off, reinterpret_cast<const int4*>(h->buffer_rows),
            reinterpret_cast<const int4*>(h->backing), reinterpret_cast<int4*>(out_dev), dim >> 2,
            phase);
    } else {
        k_shared_gather<float><<<grid, 256, 0, st>>>(
            unique_dev, dec_dev, n, G, reinterpret_cast<float* const*>(h->shared_rows),
            h->pinned_off, h->buffer_rows, h->backing, out_dev, dim, phase);
    }
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

float* gids_cache_rows_ptr(gids_handle* h) { return h ? h->cache_rows : nullptr; }

}  // extern "C"
