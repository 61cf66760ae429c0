// sampler.cu -- K1/K2: layered uniform neighbour sampling over the HBM CSC.
//
// Replaces sample_layer / sample_subgraph (sampler.py:50-112) bit-exactly.
// The reference draws `fanout` doubles per frontier node with deg > fanout
// from ONE sequential numpy PCG64 stream, visiting the frontier ascending.
// Here every draw is addressed by its stream offset instead:
//   offset(node i, draw t) = draws before this layer + exclusive_scan(draws)_i + t
// and each lane jumps the LCG straight to it (x -> A_i x + H_i per set bit,
// tables for the stream's increment), so a layer is fully parallel and the
// host Generator is advanced by the total afterwards (D1 in SURVEY.md).
//
// The partial Fisher-Yates (sampler.py:76-78) is resolved without
// materialising the pool: with j_t = t + int(u_t * (deg - t)), the value
// settled at position t is indices[lo + p] where p starts at j_t and walks
// s = t-1 .. 0 taking p = s whenever j_s == p (the last earlier swap that
// moved something into position p).  One warp handles one frontier node.
#include <cuda/atomic>

#include "gids_internal.cuh"

namespace {

constexpr int SAMPLE_BLOCK = 256;
constexpr int SAMPLE_WARPS = SAMPLE_BLOCK / 32;
constexpr int MAX_FANOUT = 1024;

__device__ __forceinline__ u128 jump(u128 s, uint64_t k, const u128* __restrict__ tab) {
    while (k) {
        int i = __ffsll((long long)k) - 1;
        k &= k - 1;
        s = add128(mul128(tab[2 * i], s), tab[2 * i + 1]);
    }
    return s;
}

__device__ __forceinline__ void mark(uint32_t* bm, int32_t v) {
    atomicOr(bm + (v >> 5), 1u << (v & 31));
}

// sample_layer's frontier as given (sampler.py:59-84: any order, duplicates
// expanded again, each with its own draws): ids narrowed in place of the
// deduplicated seed frontier
__global__ void k_front_raw(const int64_t* __restrict__ seeds, int64_t n, int32_t* front,
                            SampleCounters* sc, uint32_t* bm_all) {
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->n_front = n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = (int32_t)seeds[i];
        front[i] = v;
        mark(bm_all, v);
    }
}

__global__ void k_seed_mark(const int64_t* __restrict__ seeds, int64_t n, uint32_t* bm_front,
                            uint32_t* bm_all) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = (int32_t)seeds[i];
        if (bm_front) mark(bm_front, v);
        mark(bm_all, v);
    }
}

// ---------------------------------------------------------------------------
// Single-pass bitmap compaction (np.unique of a layer's sources,
// sampler.py:99,103,111): one bitmap word per thread, a tile of 8192 nodes
// per CTA, tiles taken in launch order from a counter and chained by a
// decoupled look-back (each tile publishes its own sums at once, then its
// inclusive prefix), so the whole compaction is one launch with no
// device-wide barrier.  With TD it also produces the next layer's per-node
// take = min(deg, f) and draw offsets (scan.cu's three take/draw passes) from
// the same walk.  The words are cleared for the next use.
constexpr int LB_BLOCK = 256;

__device__ __forceinline__ void lb_take(const int64_t* __restrict__ indptr, int64_t v, int fanout,
                                        uint32_t& tk, uint32_t& nd) {
    const int64_t deg = __ldg(indptr + v + 1) - __ldg(indptr + v);
    tk += (uint32_t)(deg < fanout ? deg : fanout);
    nd += deg > fanout ? 1u : 0u;
}

template <bool TD>
__global__ void __launch_bounds__(LB_BLOCK)
k_compact_lb(uint32_t* __restrict__ bm, int64_t nwords, int32_t* __restrict__ out, int64_t cap,
             LbTile* tiles, uint32_t* tile_ctr, SampleCounters* sc, int layer, int fanout,
             const int64_t* __restrict__ indptr, int64_t* __restrict__ take_off,
             int64_t* __restrict__ draw_off, int64_t edge_cap, int n_layers, u128* rng_state,
             const u128* __restrict__ tab) {
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_warp[LB_BLOCK / 32];
    __shared__ unsigned long long s_pre[3];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    if (t == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t wi = (int64_t)tile * LB_BLOCK + t;
    const uint32_t w = wi < nwords ? bm[wi] : 0u;
    if (w) bm[wi] = 0u;
    uint32_t tk = 0, nd = 0;
    if (TD && w) {  // up to 8 nodes' degree loads in flight per step
        uint32_t ww = w;
        const int64_t* ip = indptr + wi * 32;
        while (ww) {  // (branch-free: every step issues its loads together)
            int64_t lo[8], hi[8];
            uint32_t ok = 0;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const int b = ww ? __ffs(ww) - 1 : 0;
                ok |= (ww ? 1u : 0u) << k;
                ww &= ww - 1;
                lo[k] = __ldg(ip + b);
                hi[k] = __ldg(ip + b + 1);
            }
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const int64_t d = hi[k] - lo[k];
                const bool on = (ok >> k) & 1u;
                tk += on ? (uint32_t)(d < fanout ? d : fanout) : 0u;
                nd += (on && d > fanout) ? 1u : 0u;
            }
        }
    }
    typedef unsigned long long u64;
    const u64 mine = (u64)tk | ((u64)__popc(w) << 24) | ((u64)nd << 38);
    // block exclusive scan of the packed (take, count, draw-nodes)
    u64 inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u64 u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    u64 wsum = lane < LB_BLOCK / 32 ? s_warp[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < LB_BLOCK / 32; o <<= 1) {
        const u64 u = __shfl_up_sync(0xffffffffu, wsum, o);
        if (lane >= o) wsum += u;
    }
    const u64 agg = __shfl_sync(0xffffffffu, wsum, LB_BLOCK / 32 - 1);
    const u64 ex = inc - mine + (wid > 0 ? __shfl_sync(0xffffffffu, wsum, wid > 0 ? wid - 1 : 0) : 0ull);
    if (wid == 0) {  // look-back: the prefix of every earlier tile
        u64 pc = 0, pt = 0, pn = 0;
        const u64 at = agg & 0xffffffull, ac = (agg >> 24) & 0x3fffull, an = (agg >> 38) & 0x3fffull;
        LbTile* me = tiles + tile;
        if (tile > 0) {
            if (lane == 0) {
                me->agg = agg;
                cuda::atomic_ref<uint32_t, cuda::thread_scope_device>(me->flag).store(
                    1u, cuda::memory_order_release);
            }
            int64_t j0 = (int64_t)tile - 1;
            while (true) {
                const int64_t j = j0 - lane;
                uint32_t f = 2u;  // (before tile 0: an empty inclusive prefix)
                if (j >= 0) {
                    cuda::atomic_ref<uint32_t, cuda::thread_scope_device> fl(tiles[j].flag);
                    do {
                        f = fl.load(cuda::memory_order_acquire);
                    } while (f == 0u);
                }
                const unsigned pm = __ballot_sync(0xffffffffu, f == 2u);
                const int first = pm ? __ffs(pm) - 1 : 32;
                u64 vt = 0, vc = 0, vn = 0;
                if (j >= 0 && lane < first) {
                    const u64 a = __ldcg(&tiles[j].agg);
                    vt = a & 0xffffffull;
                    vc = (a >> 24) & 0x3fffull;
                    vn = (a >> 38) & 0x3fffull;
                } else if (j >= 0 && lane == first) {
                    vt = __ldcg(&tiles[j].inc_take);
                    vc = __ldcg(&tiles[j].inc_cnt);
                    vn = __ldcg(&tiles[j].inc_nd);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    vt += __shfl_xor_sync(0xffffffffu, vt, o);
                    vc += __shfl_xor_sync(0xffffffffu, vc, o);
                    vn += __shfl_xor_sync(0xffffffffu, vn, o);
                }
                pt += vt;
                pc += vc;
                pn += vn;
                if (pm) break;
                j0 -= 32;
            }
        }
        if (lane == 0) {
            me->inc_take = pt + at;
            me->inc_cnt = (uint32_t)(pc + ac);
            me->inc_nd = (uint32_t)(pn + an);
            cuda::atomic_ref<uint32_t, cuda::thread_scope_device>(me->flag).store(
                2u, cuda::memory_order_release);
            s_pre[0] = pc;
            s_pre[1] = pt;
            s_pre[2] = pn;
        }
    }
    __syncthreads();
    // this thread's nodes at their global positions
    int64_t pos = (int64_t)(s_pre[0] + ((ex >> 24) & 0x3fffull));
    if (w) {
        int64_t take = (int64_t)(s_pre[1] + (ex & 0xffffffull));
        int64_t dn = (int64_t)(s_pre[2] + ((ex >> 38) & 0x3fffull));
        uint32_t ww = w;
        while (ww) {
            const int64_t v = wi * 32 + (__ffs(ww) - 1);
            ww &= ww - 1;
            if (pos < cap) {
                out[pos] = (int32_t)v;
                if (TD) {
                    take_off[pos] = take;
                    draw_off[pos] = dn * fanout;
                }
            }
            if (TD) {
                uint32_t a = 0, b = 0;
                lb_take(indptr, v, fanout, a, b);
                take += a;
                dn += b;
            }
            pos++;
        }
    }
    if (tile == gridDim.x - 1 && t == 0) {  // the last tile holds the totals
        const int64_t n = (int64_t)(s_pre[0] + ((agg >> 24) & 0x3fffull));
        if (n > cap) sc->overflow = 1;
        if (TD) {
            const int64_t tt = (int64_t)(s_pre[1] + (agg & 0xffffffull));
            const int64_t dd = (int64_t)(s_pre[2] + ((agg >> 38) & 0x3fffull)) * fanout;
            if (n <= cap) {
                take_off[n] = tt;
                draw_off[n] = dd;
            }
            int64_t base = 0;
            for (int l = 0; l < layer; l++) base += sc->layer_len[l];
            sc->n_front = n;
            sc->layer_len[layer] = tt;
            sc->layer_draw_base[layer + 1] = sc->layer_draw_base[layer] + dd;
            if (base + tt > edge_cap) sc->overflow = 1;
        } else {
            // the batch's unique nodes; the stream moves past its draws; the
            // sizes the host reads back
            sc->n_unique = n;
            const int64_t draws = sc->layer_draw_base[n_layers];
            rng_state[0] = jump(rng_state[0], (uint64_t)draws, tab);
            for (int l = 0; l < n_layers; l++) sc->exp[l] = sc->layer_len[l];
            sc->exp[n_layers] = n;
            sc->exp[n_layers + 1] = draws;
            sc->exp[n_layers + 2] = sc->contribution;
            sc->exp[n_layers + 3] = sc->overflow;
        }
    }
}

// Each warp takes a contiguous run of frontier nodes (ascending ids, so the
// indptr reads are near each other) and walks the draw stream along it: one
// full jump to the run's first offset, then per node every lane t reaches its
// draw with ONE LCG step of t+1 (x -> A_{t+1} x + H_{t+1}, step table) and the
// run's state moves on by the node's draw count -- instead of a full
// O(log offset) jump per draw.  fanout <= 32 keeps the swap targets in
// registers; larger fanouts stage them in shared memory.
__global__ void __launch_bounds__(SAMPLE_BLOCK)
k_sample_layer(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
               const int32_t* __restrict__ front, const int64_t* __restrict__ take_off,
               const int64_t* __restrict__ draw_off, const SampleCounters* __restrict__ sc,
               int layer, int fanout, const u128* __restrict__ rng_state,
               const u128* __restrict__ tab, int64_t* __restrict__ edges, uint32_t* bm_front,
               uint32_t* bm_all) {
    // (bm_front null: the last layer, no next frontier)
    extern __shared__ int64_t j_smem[];  // fanout > 32: swap targets per warp
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t nf = sc->n_front;
    int64_t ebase = 0;
    for (int l = 0; l < layer; l++) ebase += sc->layer_len[l];
    const uint64_t dbase = (uint64_t)sc->layer_draw_base[layer];
    const u128 s0 = rng_state[0];  // stream state at the start of this batch
    const u128* step = tab + 128;  // step[2k], step[2k+1] = A_k, H_k
    int64_t* jw = j_smem + (int64_t)wib * fanout;

    const int64_t nwarps = (int64_t)gridDim.x * SAMPLE_WARPS;
    const int64_t per = (nf + nwarps - 1) / nwarps;
    const int64_t i0 = ((int64_t)blockIdx.x * SAMPLE_WARPS + wib) * per;
    const int64_t i1 = i0 + per < nf ? i0 + per : nf;
    if (i0 >= i1) return;
    // stream state before this run's first draw
    u128 s = jump(s0, dbase + (uint64_t)draw_off[i0], tab);
    const u128 Af = step[2 * fanout], Hf = step[2 * fanout + 1];

    for (int64_t i = i0; i < i1; i++) {
        const int32_t v = front[i];
        const int64_t lo = indptr[v];
        const int64_t deg = indptr[v + 1] - lo;
        if (deg == 0) continue;
        int64_t* out = edges + 2 * (ebase + take_off[i]);
        if (deg <= fanout) {  // whole slice in stored order (sampler.py:70-71)
            for (int64_t t = lane; t < deg; t += 32) {
                int32_t src = indices[lo + t];
                out[2 * t] = src;
                out[2 * t + 1] = v;
                if (bm_front) mark(bm_front, src);
                mark(bm_all, src);
            }
            continue;
        }
        if (fanout <= 32) {
            int64_t j = 0;
            if (lane < fanout) {
                // draw t is the output of the state t+1 steps past s
                const u128 st = add128(mul128(step[2 * (lane + 1)], s), step[2 * (lane + 1) + 1]);
                double u = (double)(pcg_output(st) >> 11) * (1.0 / 9007199254740992.0);
                j = lane + (int64_t)__dmul_rn(u, (double)(deg - lane));
            }
            int64_t p = j;
            for (int q = 30; q >= 0; q--) {
                int64_t jq = __shfl_sync(0xffffffffu, j, q);
                if (q < lane && jq == p) p = q;
            }
            if (lane < fanout) {
                int32_t src = indices[lo + p];
                out[2 * lane] = src;
                out[2 * lane + 1] = v;
                if (bm_front) mark(bm_front, src);
                mark(bm_all, src);
            }
        } else {
            for (int t = lane; t < fanout; t += 32) {
                const u128 st = add128(mul128(step[2 * (t + 1)], s), step[2 * (t + 1) + 1]);
                double u = (double)(pcg_output(st) >> 11) * (1.0 / 9007199254740992.0);
                jw[t] = t + (int64_t)__dmul_rn(u, (double)(deg - t));
            }
            __syncwarp();
            for (int t = lane; t < fanout; t += 32) {
                int64_t p = jw[t];
                for (int q = t - 1; q >= 0; q--)
                    if (jw[q] == p) p = q;
                int32_t src = indices[lo + p];
                out[2 * t] = src;
                out[2 * t + 1] = v;
                if (bm_front) mark(bm_front, src);
                mark(bm_all, src);
            }
            __syncwarp();
        }
        s = add128(mul128(Af, s), Hf);  // past this node's `fanout` draws
    }
}

__global__ void k_rng_set(u128* rng_state, u128 state, u128 inc) {
    rng_state[0] = state;
    rng_state[1] = inc;
}

// the batch consumed `draws` doubles: move the device-resident stream past them
// the batch's edges (device-side count) and unique ids widened to int64 into
// caller buffers, one launch
__global__ void k_export(const int64_t* __restrict__ src, const SampleCounters* sc, int n_layers,
                         int64_t* __restrict__ dst, const int32_t* __restrict__ uniq,
                         int64_t* __restrict__ udst, int64_t* sizes) {
    if (sizes && blockIdx.x == 0 && threadIdx.x < n_layers + 4)  // (pinned host row)
        sizes[threadIdx.x] = sc->exp[threadIdx.x];
    int64_t e = 0;
    for (int l = 0; l < n_layers; l++) e += sc->layer_len[l];
    const int64_t ne = dst ? 2 * e : 0, nu = udst ? sc->n_unique : 0;
    const int64_t n = ne > nu ? ne : nu;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < ne) dst[i] = src[i];
        if (i < nu) udst[i] = uniq[i];
    }
}

}  // namespace

// LCG tables for one increment: jumps A_i = M^(2^i), H_i = inc * sum_{k<2^i} M^k
// (i < 64, entries 0..127), then single steps of k = 0..MAX_FANOUT:
// A_k = M^k, H_k = inc * sum_{j<k} M^j (entries 128 + 2k, 128 + 2k + 1)
static void build_jump_table(uint64_t inc_hi, uint64_t inc_lo, u128* tab) {
    u128 cm{PCG_MULT_LO, PCG_MULT_HI}, cp{inc_lo, inc_hi};
    for (int i = 0; i < 64; i++) {
        tab[2 * i] = cm;
        tab[2 * i + 1] = cp;
        cp = mul128(add128(cm, u128{1, 0}), cp);
        cm = mul128(cm, cm);
    }
    const u128 m{PCG_MULT_LO, PCG_MULT_HI}, inc{inc_lo, inc_hi};
    u128 a{1, 0}, hh{0, 0};
    for (int k = 0; k <= MAX_FANOUT; k++) {
        tab[128 + 2 * k] = a;
        tab[128 + 2 * k + 1] = hh;
        hh = add128(mul128(m, hh), inc);  // x_{k+1} = M x_k + inc
        a = mul128(m, a);
    }
}

// The per-batch sampling sequence (~20 kernels and copies, all sized by
// n_seeds and the handle's bounds, every count staying on the device):
// capturable as one CUDA graph.
// compaction of one bitmap (LB instance `inst`): with TD the frontier of
// layer `layer` and its take / draw offsets, else the unique nodes
static int compact_lb(gids_handle* h, bool td, int inst, int layer, cudaStream_t st) {
    const int64_t nwords = ceil_div(h->N, 32), nt = h->lb_tiles;
    LbTile* tiles = reinterpret_cast<LbTile*>(h->sc + 1) + (int64_t)inst * nt;
    uint32_t* ctr = &h->sc->tile_ctr[inst];
    if (td)
        k_compact_lb<true><<<(unsigned)nt, LB_BLOCK, 0, st>>>(
            h->bm_front, nwords, h->frontier, h->front_cap, tiles, ctr, h->sc, layer,
            h->cfg.fanouts[layer], h->indptr, h->take_off, h->draw_off, h->edge_cap,
            h->cfg.n_layers, h->rng_dev, h->jump_tab);
    else
        k_compact_lb<false><<<(unsigned)nt, LB_BLOCK, 0, st>>>(
            h->bm_all, nwords, h->unique32, h->unique_cap, tiles, ctr, h->sc, 0, 1, h->indptr,
            nullptr, nullptr, h->edge_cap, h->cfg.n_layers, h->rng_dev, h->jump_tab);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

// The per-batch sampling sequence, every count staying on the device:
// counters, seed marks, then per layer one compaction (frontier + offsets)
// and one sampling launch, and the unique-node compaction (which also moves
// the stream on and lays out the exported sizes) -- 2L + 4 graph nodes.
static int sample_body(gids_handle* h, int64_t n_seeds, bool raw, cudaStream_t st) {
    const gids_config& c = h->cfg;
    GIDS_CUDA_TRY(cudaMemsetAsync(
        h->sc, 0,
        sizeof(SampleCounters) + sizeof(LbTile) * (size_t)(c.n_layers + 1) * (size_t)h->lb_tiles,
        st));
    int rc = GIDS_OK;
    if (raw) {
        k_front_raw<<<gids_grid(n_seeds, 256, 4 * GIDS_SMS), 256, 0, st>>>(
            h->seeds_dev, n_seeds, h->frontier, h->sc, h->bm_all);
        GIDS_LAUNCH_CHECK(h);
        if (c.n_layers > 0) {
            rc = gids_scan_take_draw(h, c.fanouts[0], 0, st);
            if (rc) return rc;
        }
    } else {
        k_seed_mark<<<gids_grid(n_seeds, 256, 4 * GIDS_SMS), 256, 0, st>>>(
            h->seeds_dev, n_seeds, c.n_layers > 0 ? h->bm_front : nullptr, h->bm_all);
        GIDS_LAUNCH_CHECK(h);
    }
    for (int l = 0; l < c.n_layers; l++) {
        int f = c.fanouts[l];
        if (l > 0 || !raw) {
            rc = compact_lb(h, true, l, l, st);
            if (rc) return rc;
        }
        size_t smem = f > 32 ? (size_t)SAMPLE_WARPS * f * sizeof(int64_t) : 0;
        int64_t bound = l == 0 ? n_seeds : h->front_cap;
        int grid = gids_grid(bound, SAMPLE_WARPS, 16 * GIDS_SMS);
        k_sample_layer<<<grid, SAMPLE_BLOCK, smem, st>>>(
            h->indptr, h->indices, h->frontier, h->take_off, h->draw_off, h->sc, l, f, h->rng_dev,
            h->jump_tab, h->edges, l + 1 < c.n_layers ? h->bm_front : nullptr, h->bm_all);
        GIDS_LAUNCH_CHECK(h);
    }
    rc = compact_lb(h, false, c.n_layers, 0, st);
    if (rc) return rc;
    GIDS_CUDA_TRY(cudaMemcpyAsync(h->sc_host, h->sc, sizeof(SampleCounters),
                                  cudaMemcpyDeviceToHost, st));
    return GIDS_OK;
}

int gids_launch_sample(gids_handle* h, int64_t n_seeds, const uint64_t* w, bool raw,
                       cudaStream_t st) {
    const gids_config& c = h->cfg;
    for (int l = 0; l < c.n_layers; l++) {
        if (c.fanouts[l] > MAX_FANOUT) {
            gids_set_error("fanout above 1024 is not supported by the CUDA sampler");
            return GIDS_E_INVALID;
        }
        size_t smem = c.fanouts[l] > 32 ? (size_t)SAMPLE_WARPS * c.fanouts[l] * sizeof(int64_t) : 0;
        if (smem > 48 * 1024)  // set before any capture
            GIDS_CUDA_TRY(cudaFuncSetAttribute(k_sample_layer,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)smem));
    }
    gids_sample_begin(h, st);
    if (w) {  // (re)seed the device-resident stream from the host Generator
        if (!h->jump_valid || h->jump_inc_hi != w[2] || h->jump_inc_lo != w[3]) {
            build_jump_table(w[2], w[3], h->jump_host);
            GIDS_CUDA_TRY(cudaMemcpyAsync(h->jump_tab, h->jump_host, sizeof(u128) * GIDS_JUMP_TAB,
                                          cudaMemcpyHostToDevice, st));
            GIDS_CUDA_TRY(cudaStreamSynchronize(st));  // staging buffer is reused
            h->jump_valid = true;
            h->jump_inc_hi = w[2];
            h->jump_inc_lo = w[3];
        }
        k_rng_set<<<1, 1, 0, st>>>(h->rng_dev, u128{w[1], w[0]}, u128{w[3], w[2]});
        GIDS_LAUNCH_CHECK(h);
    } else if (!h->jump_valid) {
        gids_set_error("sampler stream not seeded (pass the Generator state once)");
        return GIDS_E_STATE;
    }
    // replay the batch's launch sequence as one CUDA graph (one per distinct
    // seed count; not on the legacy default stream, which cannot capture)
    int rc;
    if (h->use_graphs && !raw && st != 0 && st != cudaStreamLegacy) {
        SampleGraph* g = nullptr;
        for (int i = 0; i < h->n_sgraphs; i++)
            if (h->sgraphs[i].n_seeds == n_seeds) g = &h->sgraphs[i];
        if (!g && h->n_sgraphs < GIDS_MAX_SGRAPHS) {
            const int64_t l0 = h->launches;
            GIDS_CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            rc = sample_body(h, n_seeds, false, st);
            cudaGraph_t graph = nullptr;
            cudaError_t e = cudaStreamEndCapture(st, &graph);
            if (rc) {
                if (graph) cudaGraphDestroy(graph);
                return rc;
            }
            if (e != cudaSuccess) {
                gids_set_error(std::string("sampler graph capture: ") + cudaGetErrorString(e));
                return GIDS_E_CUDA;
            }
            g = &h->sgraphs[h->n_sgraphs];
            e = cudaGraphInstantiate(&g->exec, graph, 0);
            cudaGraphDestroy(graph);
            if (e != cudaSuccess) {
                gids_set_error(std::string("sampler graph instantiate: ") + cudaGetErrorString(e));
                return GIDS_E_CUDA;
            }
            g->n_seeds = n_seeds;
            g->kernels = h->launches - l0;
            h->launches = l0;
            h->n_sgraphs++;
        }
        if (g) {
            GIDS_CUDA_TRY(cudaGraphLaunch(g->exec, st));
            h->launches += g->kernels;
            gids_sample_end(h, st);
            return GIDS_OK;
        }
    }
    rc = sample_body(h, n_seeds, raw, st);
    if (rc) return rc;
    gids_sample_end(h, st);
    return GIDS_OK;
}

int gids_launch_export(gids_handle* h, int64_t* edges_dev, int64_t* unique_dev, cudaStream_t st,
                       int64_t* sizes_host) {
    const int64_t bound = 2 * h->edge_cap > h->unique_cap ? 2 * h->edge_cap : h->unique_cap;
    k_export<<<gids_grid(bound, 256, 8 * GIDS_SMS), 256, 0, st>>>(
        h->edges, h->sc, h->cfg.n_layers, edges_dev, h->unique32, unique_dev, sizes_host);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

int gids_launch_export_unique(gids_handle* h, int64_t* unique_dev, cudaStream_t st) {
    return gids_launch_export(h, nullptr, unique_dev, st);
}
