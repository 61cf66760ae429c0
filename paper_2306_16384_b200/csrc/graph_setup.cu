// graph_setup.cu -- setup-time graph work on the GPU.
//
//  * gids_generate_uniform_graph: a uniform random graph with exactly E distinct
//    (src, dst) pairs, built in HBM in CSC form.  Same distribution as the
//    reference's "uniform" generator (graph.py:164-180: uniform endpoints,
//    parallel edges redrawn, exactly round(N * avg_degree) edges), but
//    counter-based so that it runs in parallel at 1.6B edges; the reference
//    needs 128 s at 3M nodes.  Definition (restated
//    bit-exactly by tests/graphgen_ref.py and oracle/gids_oracle.c):
//        dst(e)      = hi64(mix64(s_dst + e) * N)              e in [0, E)
//        deg(v)      = #{e : dst(e) == v}, indptr = cumsum(deg)
//        src(v,k,a)  = hi64(mix64(mix64(s_src ^ v) + (a << 32) + k) * N)
//    segment v starts as src(v, k, 0) for k < deg(v); then, repeatedly for
//    a = 1, 2, ...: sort ascending, and every sorted position r >= 1 that
//    repeats position r-1 is replaced by src(v, r, a); until no repeats.
//    s_dst = mix64(seed ^ 0x243F6A8885A308D3), s_src = mix64(seed ^ 0x13198A2E03707344).
//
//  * gids_reverse_pagerank: cpu_buffer.py:26-74 on the GPU, bit-identical to
//    the reference's float64 numpy arithmetic:
//      share/bincount  -> pull over the edge-reversed CSR (built by a stable
//                         radix sort, so each node's terms are summed in edge
//                         order exactly as np.bincount accumulates them)
//      x[sink].sum(), np.abs(nxt - x).sum()
//                      -> numpy's pairwise summation tree (8-way unrolled
//                         leaves of <= 128 terms, splits at n/2 rounded down
//                         to a multiple of 8), evaluated level by level
//      nxt *= d; nxt += c  -> two separately rounded operations (no FMA)
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <vector>

#include "gids_internal.cuh"

namespace {

constexpr uint64_t GEN_DST_SALT = 0x243F6A8885A308D3ULL;
constexpr uint64_t GEN_SRC_SALT = 0x13198A2E03707344ULL;
constexpr int GEN_WARPS = 4;
constexpr int GEN_MAX_DEG = 1024;

__device__ __forceinline__ int32_t gen_src(uint64_t zv, int64_t k, uint64_t a, uint64_t n) {
    return (int32_t)__umul64hi(mix64(zv + (a << 32) + (uint64_t)k), n);
}

__global__ void k_gen_hist(uint64_t s_dst, int64_t E, uint64_t n, unsigned long long* cnt) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        uint64_t d = __umul64hi(mix64(s_dst + (uint64_t)e), n);
        atomicAdd(cnt + d, 1ull);
    }
}

// one warp per destination: draw, sort (rank sort in shared memory), redraw repeats
__global__ void __launch_bounds__(GEN_WARPS * 32)
k_gen_fill(uint64_t s_src, int64_t N, const int64_t* __restrict__ indptr, int32_t* indices,
           int* too_big) {
    __shared__ int32_t sbuf[GEN_WARPS][GEN_MAX_DEG];
    __shared__ int32_t stmp[GEN_WARPS][GEN_MAX_DEG];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t* buf = sbuf[w];
    int32_t* tmp = stmp[w];
    for (int64_t v = (int64_t)blockIdx.x * GEN_WARPS + w; v < N;
         v += (int64_t)gridDim.x * GEN_WARPS) {
        const int64_t lo = indptr[v];
        const int deg = (int)(indptr[v + 1] - lo);
        if (deg == 0) continue;
        if (deg > GEN_MAX_DEG) {
            if (lane == 0) atomicExch(too_big, 1);
            continue;
        }
        const uint64_t zv = mix64(s_src ^ (uint64_t)v);
        for (int k = lane; k < deg; k += 32) buf[k] = gen_src(zv, k, 0, (uint64_t)N);
        __syncwarp();
        for (uint64_t a = 1;; a++) {
            for (int i = lane; i < deg; i += 32) {  // stable rank sort buf -> tmp
                const int32_t x = buf[i];
                int r = 0;
                for (int j = 0; j < deg; j++) {
                    const int32_t y = buf[j];
                    r += (y < x) | ((y == x) & (j < i));
                }
                tmp[r] = x;
            }
            __syncwarp();
            bool rep = false;
            for (int r = lane; r < deg; r += 32) {
                const bool dup = r > 0 && tmp[r] == tmp[r - 1];
                buf[r] = dup ? gen_src(zv, r, a, (uint64_t)N) : tmp[r];
                rep |= dup;
            }
            if (!__any_sync(0xffffffffu, rep)) break;
            __syncwarp();
        }
        for (int k = lane; k < deg; k += 32) indices[lo + k] = tmp[k];
        __syncwarp();
    }
}

__global__ void k_zero_i64(int64_t* p) { *p = 0; }

// --------------------------------------------------------------- pagerank
// owner (destination) of every edge, warp per node
__global__ void k_owner(const int64_t* __restrict__ indptr, int64_t N, int32_t* owner) {
    const int lane = threadIdx.x & 31;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < N;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t lo = indptr[v], hi = indptr[v + 1];
        for (int64_t e = lo + lane; e < hi; e += 32) owner[e] = (int32_t)v;
    }
}

__global__ void k_src_hist(const int32_t* __restrict__ src, int64_t E, unsigned long long* cnt) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + src[e], 1ull);
}

// denom = max-free out weight (unweighted: the in-degree in CSC), sink flags, x0
__global__ void k_pr_init(const int64_t* __restrict__ indptr, int64_t N, double x0,
                          double* denom, uint8_t* sink, double* x) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = indptr[v + 1] - indptr[v];
        denom[v] = d == 0 ? 1.0 : (double)d;
        sink[v] = d == 0;
        x[v] = x0;
    }
}

__global__ void k_pr_share(const double* __restrict__ x, const double* __restrict__ denom,
                           int64_t N, double* y) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N;
         v += (int64_t)gridDim.x * blockDim.x)
        y[v] = __ddiv_rn(x[v], denom[v]);
}

// c = teleport + damping * S / n, evaluated in Python's order
__global__ void k_pr_const(const double* S, double teleport, double damping, double n,
                           double* c) {
    *c = __dadd_rn(teleport, __ddiv_rn(__dmul_rn(damping, *S), n));
}

// nxt[u] = (sum_{edges u->v, edge order} y[v]) * damping + c
__global__ void k_pr_pull(const int64_t* __restrict__ tptr, const int32_t* __restrict__ towner,
                          const double* __restrict__ y, const double* __restrict__ c, int64_t N,
                          double damping, double* nxt) {
    const double cc = *c;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < N;
         u += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        const int64_t lo = tptr[u], hi = tptr[u + 1];
        for (int64_t k = lo; k < hi; k++) acc = __dadd_rn(acc, y[towner[k]]);
        nxt[u] = __dadd_rn(__dmul_rn(acc, damping), cc);
    }
}

// ---------------------------------------------------- numpy pairwise sum
struct AccGather {  // x[idx[i]]
    const double* x;
    const int32_t* idx;
    __device__ __forceinline__ double operator()(int64_t i) const { return x[idx[i]]; }
};
struct AccAbsDiff {  // |a[i] - b[i]|
    const double* a;
    const double* b;
    __device__ __forceinline__ double operator()(int64_t i) const {
        return fabs(__dsub_rn(a[i], b[i]));
    }
};

template <typename Acc>
__global__ void k_pw_leaf(Acc acc, const int64_t* __restrict__ off, const int64_t* __restrict__ len,
                          const int32_t* __restrict__ node, int64_t nleaves, double* val) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nleaves;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = off[t], n = len[t];
        double res;
        if (n < 8) {
            res = 0.0;
            for (int64_t i = 0; i < n; i++) res = __dadd_rn(res, acc(o + i));
        } else {
            double r[8];
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = acc(o + j);
            int64_t i = 8;
            for (; i < n - (n % 8); i += 8) {
#pragma unroll
                for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], acc(o + i + j));
            }
            res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                            __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
            for (; i < n; i++) res = __dadd_rn(res, acc(o + i));
        }
        val[node[t]] = res;
    }
}

__global__ void k_pw_combine(const int32_t* __restrict__ trip, int64_t count, double* val) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = trip[3 * t], l = trip[3 * t + 1], r = trip[3 * t + 2];
        val[p] = __dadd_rn(val[l], val[r]);
    }
}

}  // namespace

// The summation tree numpy's DOUBLE_pairwise_sum walks for n terms, laid out
// for level-by-level evaluation: leaves (offset, length, node id), then the
// internal nodes of each depth as (node, left, right) triples, deepest first.
struct PairwiseTree {
    int64_t n = 0;
    int64_t nodes = 0;
    int64_t nleaves = 0;
    int64_t *d_off = nullptr, *d_len = nullptr;
    int32_t* d_leafnode = nullptr;
    int32_t* d_trip = nullptr;
    std::vector<int64_t> level_start, level_count;  // into d_trip, deepest first
    double* d_val = nullptr;

    int build(int64_t n_, cudaStream_t st) {
        n = n_;
        std::vector<int64_t> off, len;
        std::vector<int32_t> leafnode;
        std::vector<std::vector<int32_t>> levels;  // by depth: node, left, right
        // iterative pre-order walk of the recursion
        struct Item { int64_t o, l; int depth; int32_t id; };
        std::vector<Item> stack;
        int32_t next_id = 0;
        stack.push_back({0, n, 0, next_id++});
        while (!stack.empty()) {
            Item it = stack.back();
            stack.pop_back();
            if (it.l <= 128) {
                off.push_back(it.o);
                len.push_back(it.l);
                leafnode.push_back(it.id);
                continue;
            }
            int64_t n2 = it.l / 2;
            n2 -= n2 % 8;
            int32_t lid = next_id++, rid = next_id++;
            if ((int)levels.size() <= it.depth) levels.resize(it.depth + 1);
            levels[it.depth].insert(levels[it.depth].end(), {it.id, lid, rid});
            stack.push_back({it.o + n2, it.l - n2, it.depth + 1, rid});
            stack.push_back({it.o, n2, it.depth + 1, lid});
        }
        nodes = next_id;
        nleaves = (int64_t)off.size();
        std::vector<int32_t> trip;
        for (int d = (int)levels.size() - 1; d >= 0; d--) {
            level_start.push_back((int64_t)trip.size() / 3);
            level_count.push_back((int64_t)levels[d].size() / 3);
            trip.insert(trip.end(), levels[d].begin(), levels[d].end());
        }
        GIDS_CUDA_TRY(cudaMallocAsync((void**)&d_off, sizeof(int64_t) * (nleaves + 1), st));
        GIDS_CUDA_TRY(cudaMallocAsync((void**)&d_len, sizeof(int64_t) * (nleaves + 1), st));
        GIDS_CUDA_TRY(cudaMallocAsync((void**)&d_leafnode, sizeof(int32_t) * (nleaves + 1), st));
        GIDS_CUDA_TRY(cudaMallocAsync((void**)&d_trip, sizeof(int32_t) * (trip.size() + 3), st));
        GIDS_CUDA_TRY(cudaMallocAsync((void**)&d_val, sizeof(double) * (nodes + 1), st));
        GIDS_CUDA_TRY(cudaMemcpyAsync(d_off, off.data(), sizeof(int64_t) * nleaves,
                                      cudaMemcpyHostToDevice, st));
        GIDS_CUDA_TRY(cudaMemcpyAsync(d_len, len.data(), sizeof(int64_t) * nleaves,
                                      cudaMemcpyHostToDevice, st));
        GIDS_CUDA_TRY(cudaMemcpyAsync(d_leafnode, leafnode.data(), sizeof(int32_t) * nleaves,
                                      cudaMemcpyHostToDevice, st));
        if (!trip.empty())
            GIDS_CUDA_TRY(cudaMemcpyAsync(d_trip, trip.data(), sizeof(int32_t) * trip.size(),
                                          cudaMemcpyHostToDevice, st));
        // host vectors die with this scope: the copies must land first
        GIDS_CUDA_TRY(cudaStreamSynchronize(st));
        return GIDS_OK;
    }

    // sum of acc(0..n) into d_val[0] (the root)
    template <typename Acc>
    int sum(Acc acc, cudaStream_t st) {
        if (n == 0) {
            GIDS_CUDA_TRY(cudaMemsetAsync(d_val, 0, sizeof(double), st));
            return GIDS_OK;
        }
        k_pw_leaf<<<gids_grid(nleaves, 256, 16 * GIDS_SMS), 256, 0, st>>>(acc, d_off, d_len,
                                                                       d_leafnode, nleaves, d_val);
        GIDS_CUDA_TRY(cudaGetLastError());
        for (size_t l = 0; l < level_start.size(); l++) {
            k_pw_combine<<<gids_grid(level_count[l], 256, 16 * GIDS_SMS), 256, 0, st>>>(
                d_trip + 3 * level_start[l], level_count[l], d_val);
            GIDS_CUDA_TRY(cudaGetLastError());
        }
        return GIDS_OK;
    }

    void release(cudaStream_t st) {
        void* ps[] = {d_off, d_len, d_leafnode, d_trip, d_val};
        for (void* p : ps)
            if (p) cudaFreeAsync(p, st);
    }
};

namespace {

// counts (u64, N) -> indptr (i64, N+1) = [0, inclusive_scan(counts)]
int counts_to_indptr(unsigned long long* cnt, int64_t N, int64_t* indptr, cudaStream_t st) {
    size_t tb = 0;
    GIDS_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tb, (int64_t*)cnt, indptr + 1, N, st));
    void* tmp = nullptr;
    GIDS_CUDA_TRY(cudaMallocAsync(&tmp, tb, st));
    GIDS_CUDA_TRY(cub::DeviceScan::InclusiveSum(tmp, tb, (int64_t*)cnt, indptr + 1, N, st));
    GIDS_CUDA_TRY(cudaFreeAsync(tmp, st));
    k_zero_i64<<<1, 1, 0, st>>>(indptr);
    GIDS_CUDA_TRY(cudaGetLastError());
    return GIDS_OK;
}

struct DevFree {  // frees stream-ordered allocations on scope exit
    cudaStream_t st;
    std::vector<void*> ps;
    ~DevFree() {
        for (void* p : ps)
            if (p) cudaFreeAsync(p, st);
    }
    template <typename T>
    int alloc(T** p, size_t count) {
        cudaError_t e = cudaMallocAsync((void**)p, sizeof(T) * (count ? count : 1), st);
        if (e != cudaSuccess) {
            gids_set_error(std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
            return GIDS_E_CUDA;
        }
        ps.push_back(*p);
        return GIDS_OK;
    }
};

#define TRY_RC(x)             \
    do {                      \
        int _rc = (x);        \
        if (_rc) return _rc;  \
    } while (0)

}  // namespace

extern "C" int gids_generate_uniform_graph(int device, int64_t N, int64_t E, uint64_t seed,
                                           int64_t* indptr, int32_t* indices, void* stream) {
    if (N <= 0 || N >= ((int64_t)1 << 31) || E < 0 || !indptr || (E > 0 && !indices)) {
        gids_set_error("generate_uniform_graph: need 0 < N < 2^31, E >= 0 and output buffers");
        return GIDS_E_INVALID;
    }
    if ((double)E > 0.5 * (double)N * (double)N) {
        gids_set_error("generate_uniform_graph: more edges than half of all node pairs");
        return GIDS_E_INVALID;
    }
    GIDS_CUDA_TRY(cudaSetDevice(device));
    cudaStream_t st = (cudaStream_t)stream;
    DevFree f{st, {}};
    unsigned long long* cnt = nullptr;
    int* flag = nullptr;
    TRY_RC(f.alloc(&cnt, (size_t)N));
    TRY_RC(f.alloc(&flag, 1));
    GIDS_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * N, st));
    GIDS_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), st));
    const uint64_t s_dst = mix64(seed ^ GEN_DST_SALT), s_src = mix64(seed ^ GEN_SRC_SALT);
    if (E > 0) {
        k_gen_hist<<<gids_grid(E, 256, 64 * GIDS_SMS), 256, 0, st>>>(s_dst, E, (uint64_t)N, cnt);
        GIDS_CUDA_TRY(cudaGetLastError());
    }
    TRY_RC(counts_to_indptr(cnt, N, indptr, st));
    if (E > 0) {
        k_gen_fill<<<gids_grid(N, GEN_WARPS, 32 * GIDS_SMS), GEN_WARPS * 32, 0, st>>>(
            s_src, N, indptr, indices, flag);
        GIDS_CUDA_TRY(cudaGetLastError());
    }
    int hflag = 0;
    GIDS_CUDA_TRY(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    GIDS_CUDA_TRY(cudaStreamSynchronize(st));
    if (hflag) {
        gids_set_error("generate_uniform_graph: a node's in-degree exceeds 1024");
        return GIDS_E_INVALID;
    }
    return GIDS_OK;
}

extern "C" int gids_reverse_pagerank(int device, int64_t N, int64_t E, const int64_t* indptr,
                                     const int32_t* indices, double damping, double tol,
                                     int32_t max_iter, double* scores, int32_t* iterations,
                                     int32_t* converged, void* stream) {
    if (N <= 0 || E < 0 || !indptr || (E > 0 && !indices) || !scores || !iterations ||
        !converged) {
        gids_set_error("reverse_pagerank: bad arguments");
        return GIDS_E_INVALID;
    }
    if (!(damping > 0.0 && damping < 1.0)) {
        gids_set_error("damping must be in (0, 1)");
        return GIDS_E_INVALID;
    }
    if (!(tol > 0.0)) {
        gids_set_error("tol must be positive");
        return GIDS_E_INVALID;
    }
    GIDS_CUDA_TRY(cudaSetDevice(device));
    cudaStream_t st = (cudaStream_t)stream;
    DevFree f{st, {}};

    // edge-reversed CSR: (src, owner) pairs stably sorted by src
    int32_t *owner = nullptr, *ksort = nullptr, *towner = nullptr;
    int64_t* tptr = nullptr;
    unsigned long long* cnt = nullptr;
    TRY_RC(f.alloc(&owner, (size_t)E));
    TRY_RC(f.alloc(&ksort, (size_t)E));
    TRY_RC(f.alloc(&towner, (size_t)E));
    TRY_RC(f.alloc(&tptr, (size_t)N + 1));
    TRY_RC(f.alloc(&cnt, (size_t)N));
    if (E > 0) {
        k_owner<<<gids_grid(N * 32, 256, 64 * GIDS_SMS), 256, 0, st>>>(indptr, N, owner);
        GIDS_CUDA_TRY(cudaGetLastError());
        int bits = 1;
        while (bits < 31 && ((int64_t)1 << bits) < N) bits++;
        size_t tb = 0;
        GIDS_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, indices, ksort, owner, towner,
                                                      E, 0, bits, st));
        void* tmp = nullptr;
        GIDS_CUDA_TRY(cudaMallocAsync(&tmp, tb, st));
        GIDS_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, indices, ksort, owner, towner, E, 0,
                                                      bits, st));
        GIDS_CUDA_TRY(cudaFreeAsync(tmp, st));
    }
    GIDS_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * N, st));
    if (E > 0) {
        k_src_hist<<<gids_grid(E, 256, 64 * GIDS_SMS), 256, 0, st>>>(ksort, E, cnt);
        GIDS_CUDA_TRY(cudaGetLastError());
    }
    TRY_RC(counts_to_indptr(cnt, N, tptr, st));

    // per-node state; sinks (no in-neighbours in CSC) compacted in ascending order
    double *denom = nullptr, *x = nullptr, *nxt = nullptr, *y = nullptr, *c = nullptr;
    uint8_t* sink = nullptr;
    int32_t* sinks = nullptr;
    int64_t* nsink_d = nullptr;
    TRY_RC(f.alloc(&denom, (size_t)N));
    TRY_RC(f.alloc(&x, (size_t)N));
    TRY_RC(f.alloc(&nxt, (size_t)N));
    TRY_RC(f.alloc(&y, (size_t)N));
    TRY_RC(f.alloc(&c, 1));
    TRY_RC(f.alloc(&sink, (size_t)N));
    TRY_RC(f.alloc(&sinks, (size_t)N));
    TRY_RC(f.alloc(&nsink_d, 1));
    const int g = gids_grid(N, 256, 64 * GIDS_SMS);
    k_pr_init<<<g, 256, 0, st>>>(indptr, N, 1.0 / (double)N, denom, sink, x);
    GIDS_CUDA_TRY(cudaGetLastError());
    {
        size_t tb = 0;
        thrust::counting_iterator<int32_t> ids(0);
        GIDS_CUDA_TRY(cub::DeviceSelect::Flagged(nullptr, tb, ids, sink, sinks, nsink_d, N, st));
        void* tmp = nullptr;
        GIDS_CUDA_TRY(cudaMallocAsync(&tmp, tb, st));
        GIDS_CUDA_TRY(cub::DeviceSelect::Flagged(tmp, tb, ids, sink, sinks, nsink_d, N, st));
        GIDS_CUDA_TRY(cudaFreeAsync(tmp, st));
    }
    int64_t nsink = 0;
    GIDS_CUDA_TRY(cudaMemcpyAsync(&nsink, nsink_d, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GIDS_CUDA_TRY(cudaStreamSynchronize(st));

    PairwiseTree tsink, tall;
    int rc = tsink.build(nsink, st);
    if (!rc) rc = tall.build(N, st);
    double* delta_h = nullptr;
    if (!rc && cudaMallocHost((void**)&delta_h, sizeof(double)) != cudaSuccess) {
        gids_set_error("cudaMallocHost");
        rc = GIDS_E_CUDA;
    }
    const double teleport = (1.0 - damping) / (double)N;
    int it = 0;
    bool conv = false;
    while (!rc && it < max_iter) {
        it++;
        k_pr_share<<<g, 256, 0, st>>>(x, denom, N, y);
        if ((rc = tsink.sum(AccGather{x, sinks}, st))) break;
        k_pr_const<<<1, 1, 0, st>>>(tsink.d_val, teleport, damping, (double)N, c);
        k_pr_pull<<<g, 256, 0, st>>>(tptr, towner, y, c, N, damping, nxt);
        if (cudaGetLastError() != cudaSuccess) {
            gids_set_error("reverse_pagerank: kernel launch failed");
            rc = GIDS_E_CUDA;
            break;
        }
        if ((rc = tall.sum(AccAbsDiff{nxt, x}, st))) break;
        if (cudaMemcpyAsync(delta_h, tall.d_val, sizeof(double), cudaMemcpyDeviceToHost, st) !=
                cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            gids_set_error("reverse_pagerank: stream failure");
            rc = GIDS_E_CUDA;
            break;
        }
        double* t = x;
        x = nxt;
        nxt = t;
        if (*delta_h < tol) {
            conv = true;
            break;
        }
    }
    if (!rc) {
        GIDS_CUDA_TRY(cudaMemcpyAsync(scores, x, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
        GIDS_CUDA_TRY(cudaStreamSynchronize(st));
    }
    tsink.release(st);
    tall.release(st);
    if (delta_h) cudaFreeHost(delta_h);
    *iterations = it;
    *converged = conv ? 1 : 0;
    return rc;
}
