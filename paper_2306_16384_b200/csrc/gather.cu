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

// copy one row with the warp; dst2 (may be null) receives a second copy
__device__ __forceinline__ void copy_row(const float* __restrict__ src, float* __restrict__ dst,
                                         float* __restrict__ dst2, int64_t dim, int lane) {
    if ((dim & 3) == 0) {
        const int4* s = reinterpret_cast<const int4*>(src);
        int4* d = reinterpret_cast<int4*>(dst);
        int4* d2 = reinterpret_cast<int4*>(dst2);
        const int64_t nv = dim >> 2;
        int64_t c = lane;
        for (; c + 96 < nv; c += 128) {  // four 16-B loads in flight per lane
            int4 a = ld_stream(s + c), b = ld_stream(s + c + 32), e = ld_stream(s + c + 64),
                 f = ld_stream(s + c + 96);
            st_stream(d + c, a);
            st_stream(d + c + 32, b);
            st_stream(d + c + 64, e);
            st_stream(d + c + 96, f);
            if (d2) {
                d2[c] = a;
                d2[c + 32] = b;
                d2[c + 64] = e;
                d2[c + 96] = f;
            }
        }
        for (; c < nv; c += 32) {
            int4 a = ld_stream(s + c);
            st_stream(d + c, a);
            if (d2) d2[c] = a;
        }
    } else {
        for (int64_t c = lane; c < dim; c += 32) {
            float v = src[c];
            dst[c] = v;
            if (dst2) dst2[c] = v;
        }
    }
}

__global__ void __launch_bounds__(BLOCK)
k_gather_hits(int64_t n, const int8_t* __restrict__ kind, const int32_t* __restrict__ line,
              const float* __restrict__ cache_rows, float* __restrict__ out, int64_t dim) {
    const int lane = threadIdx.x & 31;
    for (int64_t p = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5); p < n;
         p += (int64_t)gridDim.x * WARPS) {
        if (kind[p] != GIDS_KIND_HIT) continue;
        copy_row(cache_rows + (int64_t)line[p] * dim, out + p * dim, nullptr, dim, lane);
    }
}

__global__ void __launch_bounds__(BLOCK)
k_gather_host(const int64_t* __restrict__ uniq, int64_t n, const int8_t* __restrict__ kind,
              const int32_t* __restrict__ ins_line, const int32_t* __restrict__ pinned_off,
              const float* __restrict__ buffer_rows, const float* __restrict__ backing,
              float* __restrict__ cache_rows, float* __restrict__ out, int64_t dim) {
    const int lane = threadIdx.x & 31;
    for (int64_t p = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5); p < n;
         p += (int64_t)gridDim.x * WARPS) {
        if (kind[p] == GIDS_KIND_HIT) continue;
        const int32_t x = (int32_t)uniq[p];
        const int32_t off = pinned_off[x];
        const float* src = off >= 0 ? buffer_rows + (int64_t)off * dim : backing + (int64_t)x * dim;
        const int32_t t = ins_line[p];
        copy_row(src, out + p * dim, t >= 0 ? cache_rows + (int64_t)t * dim : nullptr, dim, lane);
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

int gids_launch_gather(gids_handle* h, const int64_t* uniq, int64_t n, float* out,
                       cudaStream_t st) {
    const int64_t dim = h->row_floats;
    // grid sized by GIDS_GATHER_WPS (capi.cu): a few warps per SM already
    // saturate the host link; the rest of the GPU stays free for the next
    // batch's sampling and cache decisions on the control stream
    int grid = gids_grid(n, WARPS, h->gather_blocks);
    k_gather_hits<<<grid, BLOCK, 0, st>>>(n, h->kind, h->line, h->cache_rows, out, dim);
    GIDS_LAUNCH_CHECK(h);
    if (h->profiling) cudaEventRecord(h->gev[h->parity][1], st);
    k_gather_host<<<grid, BLOCK, 0, st>>>(uniq, n, h->kind, h->ins, h->pinned_off,
                                          h->buffer_rows, h->backing, h->cache_rows, out, dim);
    GIDS_LAUNCH_CHECK(h);
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
