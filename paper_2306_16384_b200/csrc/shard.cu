// shard.cu -- the HBM-sharded feature table for tables larger than one GPU
// (409.6 GB over 8 x B200).
//
// Data-parallel ranks each sample their own batches; the feature table is
// split by owner(v) = v mod G, shard s holding the rows of nodes s, s+G, ...
// in its HBM.  A rank gathers its batch's rows straight from the owners'
// HBM: local rows over HBM, remote rows as peer loads over NVLink 5 /
// NVSwitch (CUDA IPC mappings), 16-byte loads with many in flight -- one
// kernel, no staging copy, no collective on the data path.  The whole table
// is resident, so every access is a hit (no cache policy, no host tier).
#include <cstdlib>
#include <cstring>
#include <vector>

#include "gids_internal.cuh"

namespace {

constexpr int BLOCK = 256;

__global__ void k_shard_count(const int64_t* __restrict__ uniq, int64_t n, int32_t G, int32_t me,
                              ServeCounters* svc) {
    int64_t loc = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x)
        loc += (uniq[p] % G) == me;
    for (int o = 16; o > 0; o >>= 1) loc += __shfl_xor_sync(0xffffffffu, loc, o);
    if ((threadIdx.x & 31) == 0 && loc)
        atomicAdd((unsigned long long*)&svc->shard_local, (unsigned long long)loc);
}

__global__ void k_shard_finish(int64_t n, ServeCounters* svc) {
    svc->tiers[0] = n;
    svc->shard_remote = n - svc->shard_local;
}

// out[p] = row of uniq[p] from its owner's shard; flat 16-byte chunks,
// U loads in flight per lane (peer latency over NVLink is ~2 us, so the
// whole GPU keeps several MB outstanding).  Index math is 32-bit (the chunk
// count and node ids fit: checked on the host) and, when the row's chunk
// count / the shard count are powers of two (every config here), shifts and
// masks -- round 1's 64-bit i / cpr, x % G, x / G per chunk held the kernel
// at 0.61 of HBM.
template <int U, bool POW2>
__global__ void __launch_bounds__(BLOCK)
k_gather_shards(const int64_t* __restrict__ uniq, uint32_t n, const int4* const* __restrict__ shards,
                uint32_t G, uint32_t g_shift, uint32_t cpr, uint32_t cpr_shift,
                int4* __restrict__ out) {
    const uint32_t total = n * cpr;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * (uint32_t)BLOCK + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * (uint32_t)BLOCK) >> 5;
    for (uint32_t base = warp * U * 32; base < total; base += nwarps * U * 32) {
        int4 v[U];
#pragma unroll
        for (int k = 0; k < U; k++) {
            const uint32_t i = base + k * 32 + lane;
            if (i < total) {
                uint32_t r, c, o, q;
                if (POW2) {
                    r = i >> cpr_shift;
                    c = i & (cpr - 1);
                } else {
                    r = i / cpr;
                    c = i - r * cpr;
                }
                const uint32_t x = (uint32_t)__ldg(uniq + r);
                if (POW2) {
                    o = x & (G - 1);
                    q = x >> g_shift;
                } else {
                    q = x / G;
                    o = x - q * G;
                }
                const int4* src = shards[o] + (size_t)q * cpr + c;
                asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                             : "l"(src));
            }
        }
#pragma unroll
        for (int k = 0; k < U; k++) {
            const uint32_t i = base + k * 32 + lane;
            if (i < total)
                asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(out + i),
                             "r"(v[k].x), "r"(v[k].y), "r"(v[k].z), "r"(v[k].w)
                             : "memory");
        }
    }
}

__global__ void __launch_bounds__(BLOCK)
k_gather_shards_f32(const int64_t* __restrict__ uniq, int64_t n, const float* const* shards,
                    int32_t G, int64_t dim, float* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * dim;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / dim, c = i - r * dim, x = uniq[r];
        out[i] = shards[x % G][(x / G) * dim + c];
    }
}

// synthetic rows for a shard: rows (row0 + i*stride), i < n, written densely
__global__ void k_synth_strided(uint64_t seed_mix, int64_t row0, int64_t stride, int64_t n,
                                int64_t dim, float* dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * dim;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / dim, c = i - r * dim;
        uint64_t z = ((uint64_t)(row0 + r * stride) * 0x9E3779B97F4A7C15ULL) ^
                     ((uint64_t)c * 0xC2B2AE3D27D4EB4FULL) ^ seed_mix;
        z += 0x9E3779B97F4A7C15ULL;
        z ^= z >> 30;
        z *= 0xBF58476D1CE4E5B9ULL;
        z ^= z >> 27;
        z *= 0x94D049BB133111EBULL;
        z ^= z >> 31;
        dst[i] = (float)(z >> 40) / 16777216.0f;
    }
}

}  // namespace

int gids_launch_shard_serve(gids_handle* h, const int64_t* uniq, int64_t n, float* out,
                            cudaStream_t st, cudaStream_t gst, int par) {
    GIDS_CUDA_TRY(cudaMemsetAsync(h->svc, 0, sizeof(ServeCounters), st));
    if (n > 0) {
        k_shard_count<<<gids_grid(n, BLOCK, 4 * GIDS_SMS), BLOCK, 0, st>>>(uniq, n, h->n_shards,
                                                                        h->my_shard, h->svc);
        GIDS_LAUNCH_CHECK(h);
    }
    k_shard_finish<<<1, 1, 0, st>>>(n, h->svc);
    GIDS_LAUNCH_CHECK(h);
    GIDS_CUDA_TRY(cudaMemcpyAsync(h->svc_host, h->svc, sizeof(ServeCounters),
                                  cudaMemcpyDeviceToHost, st));
    gids_mark(h, 3, st);  // (before `counted`: serve_counts reads this mark's time)
    GIDS_CUDA_TRY(cudaEventRecord(h->counted, st));
    h->counted_valid = true;
    h->last_serve_n = n;
    if (n == 0) return GIDS_OK;
    if (gst != st) {
        GIDS_CUDA_TRY(cudaEventRecord(h->decided, st));
        GIDS_CUDA_TRY(cudaStreamWaitEvent(gst, h->decided, 0));
    }
    if (h->profiling) cudaEventRecord(h->gev[par][0], gst);
    if (h->profiling) cudaEventRecord(h->gev[par][1], gst);  // no separate hit phase
    const int64_t dim = h->row_floats;
    const int64_t cpr = dim >> 2;
    if ((dim & 3) == 0 && n * cpr < (int64_t)UINT32_MAX && h->N < (int64_t)INT32_MAX) {
        auto pow2 = [](int64_t v) { return v > 0 && (v & (v - 1)) == 0; };
        auto lg = [](int64_t v) { uint32_t s = 0; while ((int64_t(1) << s) < v) s++; return s; };
        const uint32_t G = (uint32_t)h->n_shards;
        const auto* sp = reinterpret_cast<const int4* const*>(h->shard_ptrs);
        // blocks per SM and 16-B loads in flight per lane (GIDS_SHARD_BPS /
        // GIDS_SHARD_U: experiments; defaults measured best)
        static int bps = getenv("GIDS_SHARD_BPS") ? atoi(getenv("GIDS_SHARD_BPS")) : 4;
        static int un = getenv("GIDS_SHARD_U") ? atoi(getenv("GIDS_SHARD_U")) : 4;
        const int grid = bps * GIDS_SMS;
        auto* o4 = reinterpret_cast<int4*>(out);
        if (pow2(cpr) && pow2(G)) {
            if (un >= 8)
                k_gather_shards<8, true><<<grid, BLOCK, 0, gst>>>(uniq, (uint32_t)n, sp, G, lg(G),
                                                                 (uint32_t)cpr, lg(cpr), o4);
            else
                k_gather_shards<4, true><<<grid, BLOCK, 0, gst>>>(uniq, (uint32_t)n, sp, G, lg(G),
                                                                 (uint32_t)cpr, lg(cpr), o4);
        } else {
            k_gather_shards<4, false><<<grid, BLOCK, 0, gst>>>(uniq, (uint32_t)n, sp, G, 0,
                                                              (uint32_t)cpr, 0, o4);
        }
    } else {
        k_gather_shards_f32<<<gids_grid(n * dim, BLOCK, 8 * GIDS_SMS), BLOCK, 0, gst>>>(
            uniq, n, h->shard_ptrs, h->n_shards, dim, out);
    }
    GIDS_LAUNCH_CHECK(h);
    if (h->profiling) cudaEventRecord(h->gev[par][2], gst);
    GIDS_CUDA_TRY(cudaEventRecord(h->gathered[par], gst));
    h->gathered_valid[par] = true;
    h->gather_pending[par] = h->profiling;
    h->serve_timed = h->profiling;
    return GIDS_OK;
}

extern "C" {

// shards are their own cudaMalloc allocations: an IPC handle names a whole
// allocation, so a shard must start at one (a caching allocator's
// sub-block would open at the wrong base in the peer)
int gids_device_alloc(int device, int64_t bytes, void** dev_ptr_out) {
    GIDS_CUDA_TRY(cudaSetDevice(device));
    GIDS_CUDA_TRY(cudaMalloc(dev_ptr_out, (size_t)(bytes > 0 ? bytes : 1)));
    return GIDS_OK;
}

int gids_device_free(int device, void* dev_ptr) {
    GIDS_CUDA_TRY(cudaSetDevice(device));
    GIDS_CUDA_TRY(cudaFree(dev_ptr));
    return GIDS_OK;
}

int gids_ipc_handle(int device, const void* dev_ptr, uint8_t handle_out[64]) {
    GIDS_CUDA_TRY(cudaSetDevice(device));
    cudaIpcMemHandle_t hd;
    GIDS_CUDA_TRY(cudaIpcGetMemHandle(&hd, const_cast<void*>(dev_ptr)));
    static_assert(sizeof(hd) == 64, "CUDA IPC handle is 64 bytes");
    memcpy(handle_out, &hd, 64);
    return GIDS_OK;
}

int gids_ipc_open(int device, const uint8_t handle[64], void** dev_ptr_out) {
    GIDS_CUDA_TRY(cudaSetDevice(device));
    cudaIpcMemHandle_t hd;
    memcpy(&hd, handle, 64);
    GIDS_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr_out, hd, cudaIpcMemLazyEnablePeerAccess));
    return GIDS_OK;
}

int gids_ipc_close(int device, void* dev_ptr) {
    GIDS_CUDA_TRY(cudaSetDevice(device));
    GIDS_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
    return GIDS_OK;
}

int gids_set_sharded_table(gids_handle* h, const uint64_t* shard_ptrs, int32_t n_shards,
                           int32_t my_shard) {
    if (h) gids_drop_serve_graphs(h);
    if (!h || !shard_ptrs || n_shards < 1 || my_shard < 0 || my_shard >= n_shards) {
        gids_set_error("set_sharded_table: need 1 <= n_shards and 0 <= my_shard < n_shards");
        return GIDS_E_INVALID;
    }
    GIDS_CUDA_TRY(cudaSetDevice(h->device));
    for (int s = 0; s < n_shards; s++)
        if (!shard_ptrs[s]) {
            gids_set_error("set_sharded_table: null shard pointer");
            return GIDS_E_INVALID;
        }
    if (h->shard_ptrs) cudaFree((void*)h->shard_ptrs);
    GIDS_CUDA_TRY(cudaMalloc((void**)&h->shard_ptrs, sizeof(void*) * n_shards));
    GIDS_CUDA_TRY(cudaMemcpy((void*)h->shard_ptrs, shard_ptrs, sizeof(void*) * n_shards,
                             cudaMemcpyHostToDevice));
    h->n_shards = n_shards;
    h->my_shard = my_shard;
    return GIDS_OK;
}

int gids_shard_counts(gids_handle* h, int64_t* local, int64_t* remote) {
    if (!h) {
        gids_set_error("null gids handle");
        return GIDS_E_INVALID;
    }
    GIDS_CUDA_TRY(cudaSetDevice(h->device));
    if (h->counted_valid)
        GIDS_CUDA_TRY(cudaEventSynchronize(h->counted));
    else
        GIDS_CUDA_TRY(cudaStreamSynchronize(h->last_stream));
    *local = h->svc_host->shard_local;
    *remote = h->svc_host->shard_remote;
    return GIDS_OK;
}

int gids_synthesize_rows_strided(int device, uint64_t seed, int64_t row0, int64_t stride,
                                 int64_t n, int32_t dim, float* dst, void* stream) {
    GIDS_CUDA_TRY(cudaSetDevice(device));
    if (n <= 0) return GIDS_OK;
    if (stride < 1 || dim < 1) {
        gids_set_error("synthesize_rows_strided: stride and dim must be >= 1");
        return GIDS_E_INVALID;
    }
    k_synth_strided<<<gids_grid(n * dim, 256, 32 * GIDS_SMS), 256, 0, (cudaStream_t)stream>>>(
        seed * 0xD6E8FEB86659FD93ULL, row0, stride, n, dim, dst);
    GIDS_CUDA_TRY(cudaGetLastError());
    return GIDS_OK;
}

}  // extern "C"
