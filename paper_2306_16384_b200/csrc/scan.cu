// scan.cu -- device-wide exclusive scans and bitmap compaction.
//
// All scans are reduce-then-scan over a fixed number of chunks so that the
// element count can live in device memory (no host round trip between the
// sampler's layers).  Bitmap compaction turns an N-bit membership bitmap into
// the ascending id list -- the B200 replacement of np.unique at
// sampler.py:99,103,111 (sorted output falls out of the word order).
#include "gids_internal.cuh"

namespace {

constexpr int SCAN_BLOCK = 256;
constexpr int MAX_PARTS = 1024;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += u;
    }
    return v;
}

// exclusive block scan of one value per thread; *total receives the sum
template <typename T, int BLOCK>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
    __shared__ T warp_sums[BLOCK / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T inc = warp_incl_scan(v);
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        T s = lane < BLOCK / 32 ? warp_sums[lane] : T(0);
        s = warp_incl_scan(s);
        if (lane < BLOCK / 32) warp_sums[lane] = s;
    }
    __syncthreads();
    T prefix = wid > 0 ? warp_sums[wid - 1] : T(0);
    *total = warp_sums[BLOCK / 32 - 1];
    __syncthreads();
    return prefix + inc - v;
}

template <typename T, int BLOCK>
__device__ __forceinline__ T block_sum(T v) {
    T total;
    block_excl_scan<T, BLOCK>(v, &total);
    return total;
}

__device__ __forceinline__ void chunk_of(int64_t n, int64_t* lo, int64_t* hi) {
    int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    *lo = (int64_t)blockIdx.x * chunk;
    *hi = *lo + chunk < n ? *lo + chunk : n;
}

// ---------------------------------------------------------------------------
// take_i = min(deg, f), draws_i = deg > f ? f : 0 over the current frontier
// (sample_layer, sampler.py:64-79).

__device__ __forceinline__ void take_draw(const int64_t* indptr, const int32_t* front, int64_t i,
                                          int fanout, int64_t* take, int64_t* draw) {
    int32_t v = front[i];
    int64_t deg = indptr[v + 1] - indptr[v];
    *take = deg < fanout ? deg : fanout;
    *draw = deg > fanout ? fanout : 0;
}

__global__ void k_td_reduce(const int64_t* __restrict__ indptr, const int32_t* __restrict__ front,
                            const SampleCounters* sc, int fanout, int64_t* parts) {
    int64_t n = sc->n_front, lo, hi;
    chunk_of(n, &lo, &hi);
    int64_t st = 0, sd = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += SCAN_BLOCK) {
        int64_t t, d;
        take_draw(indptr, front, i, fanout, &t, &d);
        st += t;
        sd += d;
    }
    st = block_sum<int64_t, SCAN_BLOCK>(st);
    sd = block_sum<int64_t, SCAN_BLOCK>(sd);
    if (threadIdx.x == 0) {
        parts[2 * blockIdx.x] = st;
        parts[2 * blockIdx.x + 1] = sd;
    }
}

// single block: exclusive scan of the per-chunk partials
__global__ void k_td_parts(int64_t* parts, int nparts, SampleCounters* sc, int layer,
                           int64_t edge_cap) {
    int i = threadIdx.x;
    int64_t t = i < nparts ? parts[2 * i] : 0, d = i < nparts ? parts[2 * i + 1] : 0;
    int64_t tt, dt;
    int64_t te = block_excl_scan<int64_t, MAX_PARTS>(t, &tt);
    int64_t de = block_excl_scan<int64_t, MAX_PARTS>(d, &dt);
    if (i < nparts) {
        parts[2 * i] = te;
        parts[2 * i + 1] = de;
    }
    if (i == 0) {
        int64_t base = 0;
        for (int l = 0; l < layer; l++) base += sc->layer_len[l];
        sc->layer_len[layer] = tt;
        sc->layer_draw_base[layer + 1] = sc->layer_draw_base[layer] + dt;
        if (base + tt > edge_cap) sc->overflow = 1;
    }
}

__global__ void k_td_apply(const int64_t* __restrict__ indptr, const int32_t* __restrict__ front,
                           const SampleCounters* sc, int fanout, const int64_t* parts,
                           int64_t* take_off, int64_t* draw_off) {
    int64_t n = sc->n_front, lo, hi;
    chunk_of(n, &lo, &hi);
    int64_t ct = parts[2 * blockIdx.x], cd = parts[2 * blockIdx.x + 1];
    for (int64_t b = lo; b < hi; b += SCAN_BLOCK) {
        int64_t i = b + threadIdx.x, t = 0, d = 0;
        if (i < hi) take_draw(indptr, front, i, fanout, &t, &d);
        int64_t tt, dt;
        int64_t te = block_excl_scan<int64_t, SCAN_BLOCK>(t, &tt);
        int64_t de = block_excl_scan<int64_t, SCAN_BLOCK>(d, &dt);
        if (i < hi) {
            take_off[i] = ct + te;
            draw_off[i] = cd + de;
        }
        ct += tt;
        cd += dt;
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        take_off[n] = ct;  // grand totals land after the last element
        draw_off[n] = cd;
    }
}

// ---------------------------------------------------------------------------
// bitmap -> ascending id list

__global__ void k_bm_reduce(const uint32_t* __restrict__ bm, int64_t nwords, uint32_t* parts) {
    int64_t lo, hi;
    chunk_of(nwords, &lo, &hi);
    uint32_t s = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += SCAN_BLOCK) s += __popc(bm[i]);
    s = block_sum<uint32_t, SCAN_BLOCK>(s);
    if (threadIdx.x == 0) parts[blockIdx.x] = s;
}

__global__ void k_bm_parts(uint32_t* parts, int nparts, int64_t* count_out, int64_t cap,
                           int64_t* overflow) {
    int i = threadIdx.x;
    int64_t v = i < nparts ? parts[i] : 0, tot;
    int64_t e = block_excl_scan<int64_t, MAX_PARTS>(v, &tot);
    if (i < nparts) parts[i] = (uint32_t)e;
    if (i == 0) {
        *count_out = tot;
        if (tot > cap) *overflow = 1;
    }
}

__global__ void k_bm_apply(uint32_t* __restrict__ bm, int64_t nwords, const uint32_t* parts,
                           int32_t* __restrict__ out, int64_t cap, int clear) {
    int64_t lo, hi;
    chunk_of(nwords, &lo, &hi);
    int64_t base = parts[blockIdx.x];
    for (int64_t b = lo; b < hi; b += SCAN_BLOCK) {
        int64_t i = b + threadIdx.x;
        uint32_t w = i < hi ? bm[i] : 0u;
        int64_t tot;
        int64_t pos = base + block_excl_scan<int64_t, SCAN_BLOCK>((int64_t)__popc(w), &tot);
        if (w) {
            if (clear) bm[i] = 0u;
            while (w) {
                int bit = __ffs(w) - 1;
                w &= w - 1;
                if (pos < cap) out[pos] = (int32_t)(i * 32 + bit);
                pos++;
            }
        }
        base += tot;
    }
}

// ---------------------------------------------------------------------------
__global__ void k_i32_reduce(const int32_t* __restrict__ in, int64_t n, int64_t* parts) {
    int64_t lo, hi;
    chunk_of(n, &lo, &hi);
    int64_t s = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += SCAN_BLOCK) s += in[i];
    s = block_sum<int64_t, SCAN_BLOCK>(s);
    if (threadIdx.x == 0) parts[blockIdx.x] = s;
}
__global__ void k_i64_parts(int64_t* parts, int nparts) {
    int i = threadIdx.x;
    int64_t v = i < nparts ? parts[i] : 0, tot;
    int64_t e = block_excl_scan<int64_t, MAX_PARTS>(v, &tot);
    if (i < nparts) parts[i] = e;
}
__global__ void k_i32_apply(const int32_t* __restrict__ in, int64_t n, const int64_t* parts,
                            int64_t* out) {
    int64_t lo, hi;
    chunk_of(n, &lo, &hi);
    int64_t c = parts[blockIdx.x];
    for (int64_t b = lo; b < hi; b += SCAN_BLOCK) {
        int64_t i = b + threadIdx.x;
        int64_t v = i < hi ? in[i] : 0, tot;
        int64_t e = block_excl_scan<int64_t, SCAN_BLOCK>(v, &tot);
        if (i < hi) out[i] = c + e;
        c += tot;
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = c;
}

int parts_for(int64_t n) {
    int64_t p = ceil_div(n, SCAN_BLOCK * 8);
    if (p < 1) p = 1;
    if (p > MAX_PARTS) p = MAX_PARTS;
    return (int)p;
}

}  // namespace

int gids_scan_take_draw(gids_handle* h, int fanout, int layer, cudaStream_t st) {
    // the frontier size lives on the device; size the grid by its bound
    int np = parts_for(h->front_cap);
    k_td_reduce<<<np, SCAN_BLOCK, 0, st>>>(h->indptr, h->frontier, h->sc, fanout, h->scan_parts);
    GIDS_LAUNCH_CHECK(h);
    k_td_parts<<<1, MAX_PARTS, 0, st>>>(h->scan_parts, np, h->sc, layer, h->edge_cap);
    GIDS_LAUNCH_CHECK(h);
    k_td_apply<<<np, SCAN_BLOCK, 0, st>>>(h->indptr, h->frontier, h->sc, fanout, h->scan_parts,
                                          h->take_off, h->draw_off);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

int gids_bitmap_compact(gids_handle* h, uint32_t* bm, int32_t* out, int64_t* count_out,
                        int64_t cap, bool clear, cudaStream_t st) {
    return gids_bitmap_compact_n(h, bm, h->N, out, count_out, cap, clear, &h->sc->overflow,
                                 h->word_parts, st);
}

int gids_bitmap_compact_n(gids_handle* h, uint32_t* bm, int64_t nbits, int32_t* out,
                          int64_t* count_out, int64_t cap, bool clear, int64_t* overflow,
                          uint32_t* parts, cudaStream_t st) {
    int64_t nwords = ceil_div(nbits, 32);
    int np = parts_for(nwords);
    k_bm_reduce<<<np, SCAN_BLOCK, 0, st>>>(bm, nwords, parts);
    GIDS_LAUNCH_CHECK(h);
    k_bm_parts<<<1, MAX_PARTS, 0, st>>>(parts, np, count_out, cap, overflow);
    GIDS_LAUNCH_CHECK(h);
    k_bm_apply<<<np, SCAN_BLOCK, 0, st>>>(bm, nwords, parts, out, cap, clear ? 1 : 0);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

int gids_scan_i32_to_i64(gids_handle* h, const int32_t* in, int64_t n, int64_t* out,
                         cudaStream_t st) {
    int np = parts_for(n);
    // serving path only (set-associative bucketing): its own partials
    k_i32_reduce<<<np, SCAN_BLOCK, 0, st>>>(in, n, h->serve_parts);
    GIDS_LAUNCH_CHECK(h);
    k_i64_parts<<<1, MAX_PARTS, 0, st>>>(h->serve_parts, np);
    GIDS_LAUNCH_CHECK(h);
    k_i32_apply<<<np, SCAN_BLOCK, 0, st>>>(in, n, h->serve_parts, out);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}
