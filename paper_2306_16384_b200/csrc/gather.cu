// gather.cu -- K5 tier chain + feature gather, K7 on-device verification.
//
// dataloader.py:279-290 gathers cache hits first (before any insertion of the
// batch lands), then constant-buffer rows, then backing-store rows, then
// writes inserted rows into their lines.  Two kernels keep that order:
//   k_gather_hits   HBM cache line -> out row          (HBM -> HBM)
//   k_gather_host   pinned host row -> out row (+ cache line when this node
//                   is the line's final occupant)       (host link -> HBM)
// Rows move warp-per-row with 16-byte vector loads (ld.global.nc, no L1
// allocation) and streaming stores; host rows are read zero-copy over the
// host link, so the copy engines are not involved.
#include "gids_internal.cuh"

namespace {

constexpr int BLOCK = 256;
constexpr int WARPS = BLOCK / 32;

__device__ __forceinline__ int4 ld_stream(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream(int4* p, int4 v) {
    asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// Work is a flat range of 16-byte chunks over the compacted row list: chunk
// i is chunk (i % cpr) of list row (i / cpr), cpr = chunks per row.  Every
// lane keeps UNROLL loads in flight before it stores, so a warp has
// UNROLL x 512 B outstanding whatever the row width (a 128-d row is exactly
// one warp-wide load; a 1024-d row is eight).
template <typename T>
__device__ __forceinline__ T ld_nc(const T* p) { return __ldg(p); }
template <>
__device__ __forceinline__ int4 ld_nc<int4>(const int4* p) { return ld_stream(p); }
template <typename T>
__device__ __forceinline__ void st_cs(T* p, T v) { *p = v; }
template <>
__device__ __forceinline__ void st_cs<int4>(int4* p, int4 v) { st_stream(p, v); }

struct ChunkIdx {
    uint32_t shift, mask, cpr;  // shift/mask when cpr is a power of two
    __device__ __forceinline__ void split(uint32_t i, uint32_t& r, uint32_t& c) const {
        if (mask) {
            r = i >> shift;
            c = i & mask;
        } else if (cpr == 1) {
            r = i;
            c = 0;
        } else {
            r = i / cpr;
            c = i - r * cpr;
        }
    }
};

// cache hits: out[p] = cache_rows[line[p]]   (HBM -> HBM, before any insert)
template <typename T, int UNROLL>
__global__ void __launch_bounds__(BLOCK)
k_gather_hits(const int32_t* __restrict__ hit_list, const int64_t* __restrict__ list_cnt,
              const int32_t* __restrict__ line, const T* __restrict__ cache_rows,
              T* __restrict__ out, ChunkIdx ci, const ServeArgs* sa = nullptr) {
    if (sa) out = reinterpret_cast<T*>(sa->out);
    const uint32_t total = (uint32_t)list_cnt[0] * ci.cpr;
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * BLOCK + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * BLOCK) >> 5;
    for (uint32_t base = warp * UNROLL * 32; base < total; base += nwarps * UNROLL * 32) {
        T v[UNROLL];
        int64_t dst[UNROLL];
#pragma unroll
        for (int k = 0; k < UNROLL; k++) {
            const uint32_t i = base + k * 32 + lane;
            dst[k] = -1;
            if (i < total) {
                uint32_t r, c;
                ci.split(i, r, c);
                const int32_t p = hit_list[r];
                v[k] = ld_nc(cache_rows + (int64_t)line[p] * ci.cpr + c);
                dst[k] = (int64_t)p * ci.cpr + c;
            }
        }
#pragma unroll
        for (int k = 0; k < UNROLL; k++)
            if (dst[k] >= 0) st_cs(out + dst[k], v[k]);
    }
}

// host tiers: out[p] = constant-buffer or backing row (zero-copy over the
// host link); the row also lands in its cache line when p inserts (ins[p])
template <typename T, int UNROLL>
__global__ void __launch_bounds__(BLOCK)
k_gather_host(const int2* __restrict__ host_list, const int64_t* __restrict__ list_cnt,
              const int32_t* __restrict__ ins, const T* __restrict__ buffer_rows,
              const T* __restrict__ backing, T* __restrict__ cache_rows, T* __restrict__ out,
              ChunkIdx ci, const ServeArgs* sa = nullptr) {
    if (sa) out = reinterpret_cast<T*>(sa->out);
    const uint32_t total = (uint32_t)list_cnt[1] * ci.cpr;
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * BLOCK + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * BLOCK) >> 5;
    for (uint32_t base = warp * UNROLL * 32; base < total; base += nwarps * UNROLL * 32) {
        T v[UNROLL];
        int64_t dst[UNROLL], dst2[UNROLL];
#pragma unroll
        for (int k = 0; k < UNROLL; k++) {
            const uint32_t i = base + k * 32 + lane;
            dst[k] = -1;
            if (i < total) {
                uint32_t r, c;
                ci.split(i, r, c);
                const int2 it = host_list[r];
                const T* src = it.y >= 0 ? buffer_rows + (int64_t)it.y * ci.cpr
                                         : backing + (int64_t)(-(it.y + 1)) * ci.cpr;
                v[k] = ld_nc(src + c);
                dst[k] = (int64_t)it.x * ci.cpr + c;
                const int32_t t = ins[it.x];
                dst2[k] = t >= 0 ? (int64_t)t * ci.cpr + c : -1;
            }
        }
#pragma unroll
        for (int k = 0; k < UNROLL; k++) {
            if (dst[k] >= 0) {
                st_cs(out + dst[k], v[k]);
                if (dst2[k] >= 0) cache_rows[dst2[k]] = v[k];
            }
        }
    }
}

// synthetic_feature_rows (graph.py:256-275), one thread per cell
__device__ __forceinline__ float feature_cell(uint64_t node, uint64_t col, uint64_t seed_mix) {
    uint64_t z = (node * 0x9E3779B97F4A7C15ULL) ^ (col * 0xC2B2AE3D27D4EB4FULL) ^ seed_mix;
    z += 0x9E3779B97F4A7C15ULL;
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return (float)(z >> 40) / 16777216.0f;
}

__global__ void k_synth(uint64_t seed_mix, int64_t row0, int64_t n, int64_t dim, float* dst) {
    int64_t total = n * dim;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / dim, c = i - r * dim;
        dst[i] = feature_cell((uint64_t)(row0 + r), (uint64_t)c, seed_mix);
    }
}

__global__ void k_verify(uint64_t seed_mix, const int64_t* __restrict__ nodes, int64_t n,
                         int64_t dim, const float* __restrict__ rows,
                         unsigned long long* bad) {
    const int lane = threadIdx.x & 31;
    int64_t nbad = 0;
    for (int64_t p = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5); p < n;
         p += (int64_t)gridDim.x * WARPS) {
        uint64_t x = (uint64_t)nodes[p];
        bool ok = true;
        for (int64_t c = lane; c < dim; c += 32)
            ok &= __float_as_uint(rows[p * dim + c]) ==
                  __float_as_uint(feature_cell(x, (uint64_t)c, seed_mix));
        nbad += __all_sync(0xffffffffu, ok) ? 0 : (lane == 0);
    }
    if (nbad) atomicAdd(bad, (unsigned long long)nbad);
}

}  // namespace

static ChunkIdx chunk_idx(int64_t cpr) {
    ChunkIdx ci{0, 0, (uint32_t)cpr};
    if (cpr > 1 && (cpr & (cpr - 1)) == 0) {
        while (((int64_t)1 << ci.shift) < cpr) ci.shift++;
        ci.mask = (uint32_t)(cpr - 1);
    }
    return ci;
}

int gids_launch_gather(gids_handle* h, const int64_t* uniq, int64_t n, float* out,
                       cudaStream_t st, const ServeArgs* sa) {
    (void)uniq;  // (sa: a graph capture; n is the bound, out and the counts are read on the device)
    const int64_t dim = h->row_floats;
    if ((dim & 3) == 0 ? (n * (dim >> 2) >= ((int64_t)1 << 32)) : (n * dim >= ((int64_t)1 << 32))) {
        gids_set_error("batch too large for the gather's 32-bit chunk index");
        return GIDS_E_CAPACITY;
    }
    // hits: HBM -> HBM, the whole GPU for the few microseconds it takes;
    // host rows: grid sized by GIDS_GATHER_WPS (capi.cu) -- a few warps per SM
    // with 8 loads in flight per lane saturate the host link and leave the
    // rest of the GPU to the next batch's sampling and cache decisions
    const int hit_grid = gids_grid(n, WARPS, h->hit_blocks);
    const int host_grid = gids_grid(n, WARPS, h->gather_blocks);
    if (h->ft) {  // file-backed storage tier: hits, then pages -> HBM staging -> rows
        if ((dim & 3) == 0) {
            (h->hit_unroll == 8 ? k_gather_hits<int4, 8> : k_gather_hits<int4, 4>)<<<hit_grid, BLOCK, 0, st>>>(
                h->hit_list, h->list_cnt, h->line, reinterpret_cast<const int4*>(h->cache_rows),
                reinterpret_cast<int4*>(out), chunk_idx(dim >> 2), sa);
        } else {
            k_gather_hits<float, 4><<<hit_grid, BLOCK, 0, st>>>(h->hit_list, h->list_cnt, h->line,
                                                                h->cache_rows, out, chunk_idx(dim), sa);
        }
        GIDS_LAUNCH_CHECK(h);
        if (h->profiling) cudaEventRecord(h->gev[h->parity][1], st);
        int rc = gids_file_fetch_and_gather(h, h->parity, out, st);
        if (rc) return rc;
        if (h->profiling) cudaEventRecord(h->gev[h->parity][2], st);
        return GIDS_OK;
    }
    if ((dim & 3) == 0) {
        ChunkIdx ci = chunk_idx(dim >> 2);
        (h->hit_unroll == 8 ? k_gather_hits<int4, 8> : k_gather_hits<int4, 4>)<<<hit_grid, BLOCK, 0, st>>>(
            h->hit_list, h->list_cnt, h->line, reinterpret_cast<const int4*>(h->cache_rows),
            reinterpret_cast<int4*>(out), ci, sa);
        GIDS_LAUNCH_CHECK(h);
        if (h->profiling) cudaEventRecord(h->gev[h->parity][1], st);
        auto kh = h->gather_unroll == 1   ? k_gather_host<int4, 1>
                  : h->gather_unroll == 2 ? k_gather_host<int4, 2>
                  : h->gather_unroll == 4 ? k_gather_host<int4, 4>
                                          : k_gather_host<int4, 8>;
        kh<<<host_grid, BLOCK, 0, st>>>(
            h->host_list, h->list_cnt, h->ins, reinterpret_cast<const int4*>(h->buffer_rows),
            reinterpret_cast<const int4*>(h->backing), reinterpret_cast<int4*>(h->cache_rows),
            reinterpret_cast<int4*>(out), ci, sa);
        GIDS_LAUNCH_CHECK(h);
    } else {
        ChunkIdx ci = chunk_idx(dim);
        k_gather_hits<float, 4><<<hit_grid, BLOCK, 0, st>>>(h->hit_list, h->list_cnt, h->line,
                                                            h->cache_rows, out, ci, sa);
        GIDS_LAUNCH_CHECK(h);
        if (h->profiling) cudaEventRecord(h->gev[h->parity][1], st);
        k_gather_host<float, 8><<<host_grid, BLOCK, 0, st>>>(h->host_list, h->list_cnt, h->ins,
                                                             h->buffer_rows, h->backing,
                                                             h->cache_rows, out, ci, sa);
        GIDS_LAUNCH_CHECK(h);
    }
    if (h->profiling) cudaEventRecord(h->gev[h->parity][2], st);
    return GIDS_OK;
}

extern "C" int gids_synthesize_rows(int device, uint64_t seed, int64_t row0, int64_t n,
                                    int32_t dim, float* dst, void* stream) {
    GIDS_CUDA_TRY(cudaSetDevice(device));
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return GIDS_OK;
    uint64_t seed_mix = seed * 0xD6E8FEB86659FD93ULL;
    k_synth<<<gids_grid(n * dim, 256, 32 * GIDS_SMS), 256, 0, st>>>(seed_mix, row0, n, dim, dst);
    GIDS_CUDA_TRY(cudaGetLastError());
    return GIDS_OK;
}

extern "C" int gids_verify_rows(int device, uint64_t seed, const int64_t* nodes_dev, int64_t n,
                                int32_t dim, const float* rows_dev, int64_t* bad, void* stream) {
    GIDS_CUDA_TRY(cudaSetDevice(device));
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long* d_bad = nullptr;
    GIDS_CUDA_TRY(cudaMallocAsync((void**)&d_bad, sizeof(unsigned long long), st));
    GIDS_CUDA_TRY(cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), st));
    if (n > 0) {
        k_verify<<<gids_grid(n, WARPS, 16 * GIDS_SMS), BLOCK, 0, st>>>(
            seed * 0xD6E8FEB86659FD93ULL, nodes_dev, n, dim, rows_dev, d_bad);
        GIDS_CUDA_TRY(cudaGetLastError());
    }
    unsigned long long hb = 0;
    GIDS_CUDA_TRY(cudaMemcpyAsync(&hb, d_bad, sizeof(hb), cudaMemcpyDeviceToHost, st));
    GIDS_CUDA_TRY(cudaFreeAsync(d_bad, st));
    GIDS_CUDA_TRY(cudaStreamSynchronize(st));
    *bad = (int64_t)hb;
    return GIDS_OK;
}
