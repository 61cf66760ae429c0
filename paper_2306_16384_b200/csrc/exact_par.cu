// exact_par.cu -- the reference eviction policy for a FULL cache, decided by a
// whole CTA instead of one warp.
//
// CacheState.access (cache.py:144-180) over a batch in ascending node order
// is a sequential state machine, but once the cache is full (no fill pointer
// left) almost all of it is static per batch.  With `cb` / `ca` the node's
// reuse count before / after its own consumption (both known after
// window_update, k_window_consume) and the invariant "a resident line is
// InUse iff its node's count > 0", every access is one of:
//   STAY  resident, ca > 0          hit, line stays InUse        (no change)
//   ADD   resident, cb > 0, ca == 0 hit, line becomes SafeToEvict (safe += s)
//   CAND  resident, cb == 0         hit -- unless an earlier eviction of this
//                                   batch took its (safe) line: then a miss
//                                   that evicts, inserting SafeToEvict
//   M0    not resident, ca == 0     miss: evict, insert SafeToEvict (safe set
//                                   unchanged: the victim line stays safe)
//   MU    not resident, ca > 0      miss: evict, insert InUse     (safe -= v)
// so the safe COUNT seen by each access is a prefix over the batch (a
// saturating one: a miss with no safe line bypasses), the eviction draw of
// each miss is a fixed position in the numpy PCG64 half stream (pre-generated
// in parallel, k_xp_halves), and the safe SET only changes at ADD / MU
// events (~7% of the accesses at C3/C4).  The only truly dynamic part is a
// CAND losing its line, which inserts one more draw into the stream.
//
// The kernel walks the batch in rounds of XT accesses, one per thread:
//   A  classify, saturating prefix of the safe count, prefix of the draws
//   B  Lemire-bounded draw per miss (numpy integers(n), buffered 32-bit
//      halves); a rejection moves every later draw of the round by the
//      halves it consumed: the first is absorbed (the later accesses redraw),
//      a second ends the round after it
//   C  the round's ADD lines join the bitmap and the prefix counts at once:
//      T = start set + ADDs.  An access then sees T minus its "holes" -- the
//      ADD lines of later accesses and the lines earlier MU accesses removed
//      -- and its eviction is the least fixed point of q = r + #holes(<= line
//      of rank q in T), found from q = r by a few selects in T (interpolated
//      block search over shared-memory prefix counts, then the 32 words of
//      the 1024-line block from the L2-resident bitmap, kept in registers)
//      and popcounts of prefix masks over the line-sorted change list
//   D  the MU lines are themselves answers: Jacobi passes over the
//      triangular system until none moves (pass k fixes the first k; two in
//      practice)
//   E  every other eviction resolves once against the final change list
//   F  a CAND whose line was taken earlier (this or the previous round; older
//      rounds flag it through cand_of_slot) ends the round before itself and
//      is a miss in the next one
//   G  commit: decisions, insertion log, bitmap and prefix counts
// and is bit-exact with the sequential reference (tests/test_gpu_exact_par.py).
// Not full, too many candidates, or a cache larger than XP_MAX_L lines: the
// sequential warp (k_exact_seq) decides the batch instead.
#include "gids_internal.cuh"

// per-phase cycle counters of thread 0 (exact_par_stats): compiled in with
// -DGIDS_XP_PROF=1 -- the clock reads sit on warp 0's path through every phase
#ifndef GIDS_XP_PROF
#define GIDS_XP_PROF 0
#endif
#define XP_MARK(i)                                \
    do {                                          \
        if (GIDS_XP_PROF && t == 0) {             \
            const long long _n = clock64();       \
            prof[i] += _n - tc;                   \
            tc = _n;                              \
        }                                         \
    } while (0)

namespace {

constexpr int XT = 512;           // threads = accesses per round
constexpr int XW = XT / 32;
constexpr int XP_MAX_CHG = 64;    // set changes per round (the round ends before the 65th)
constexpr int RING = 4096;        // staged accesses (ev, class)
constexpr int HRING = 4096;       // staged draw halves
constexpr int RING_LAG = 4;       // commit groups allowed in flight when a round reads: a round
                                  // reads entries staged >= (RING - 2 XT) / XT rounds ago
constexpr int32_t NEG = -(1 << 29);
constexpr int MOVN = 2048;        // moved-line filter: buckets (lines >> movs)
constexpr int MOVSPAN = 8;        // longer moves / ranges: every earlier MU is checked
constexpr int CUMN = 256;         // change-line buckets of count_le (lines >> bsh)
constexpr int HSZ = XT;           // the round's candidates: (line, lane) list
constexpr int CHBW = 128;         // candidate-line filter: 4096 bits

enum { C_STAY = GIDS_XC_STAY, C_ADD = GIDS_XC_ADD, C_CAND = GIDS_XC_CAND, C_M0 = GIDS_XC_M0,
       C_MU = GIDS_XC_MU };

__device__ __forceinline__ u128 pcg_advance(u128 s, u128 inc, uint64_t k) {
    u128 am = {1, 0}, ap = {0, 0}, cm = {PCG_MULT_LO, PCG_MULT_HI}, cp = inc;
    while (k) {
        if (k & 1) {
            am = mul128(am, cm);
            ap = add128(mul128(ap, cm), cp);
        }
        cp = mul128(add128(cm, u128{1, 0}), cp);
        cm = mul128(cm, cm);
        k >>= 1;
    }
    return add128(mul128(am, s), ap);
}

// half j of the eviction stream from the batch-start generator: the buffered
// upper half first (if any), then lo, hi of each next64 output
__device__ __forceinline__ uint32_t half_direct(const CacheMeta* meta, int64_t j) {
    const uint32_t has = (uint32_t)meta->rng[4];
    if (has) {
        if (j == 0) return (uint32_t)meta->rng[5];
        j -= 1;
    }
    u128 s = {meta->rng[1], meta->rng[0]}, inc = {meta->rng[3], meta->rng[2]};
    uint64_t o = pcg_output(pcg_advance(s, inc, (uint64_t)(j >> 1) + 1));
    return (j & 1) ? (uint32_t)(o >> 32) : (uint32_t)o;
}

// the CTA decides a batch when the cache is full and has safe lines for a
// good share of the batch's misses (safe_div: safe_count * div >= misses;
// 0 = always).  A starved cache -- the window protecting nearly every line,
// misses mostly bypassing -- evicts little and stays on the sequential warp,
// which is cheaper there (its cost follows the evictions, this kernel's the
// accesses).
__device__ __forceinline__ bool xp_runs(const CacheMeta* meta, const ServeCounters* svc,
                                        int64_t L, int64_t cand_cap, int64_t safe_div) {
    return svc->n_miss0 != 0 && meta->fill >= L && svc->n_cand <= cand_cap &&
           (safe_div == 0 || meta->safe_count * safe_div >= svc->n_miss0);
}

// the batch's eviction half stream, 8 next64 outputs per thread
__global__ void k_xp_halves(const CacheMeta* meta, const ServeCounters* svc, int64_t L,
                            int64_t cand_cap, int64_t safe_div, uint32_t* H, int64_t hcap) {
    if (!xp_runs(meta, svc, L, cand_cap, safe_div)) return;
    const uint32_t has = (uint32_t)meta->rng[4];
    const int64_t outs = (hcap + 1) / 2;
    const int64_t t0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (t0 >= outs) return;
    if (t0 == 0 && has) H[0] = (uint32_t)meta->rng[5];
    const u128 inc = {meta->rng[3], meta->rng[2]};
    u128 s = pcg_advance(u128{meta->rng[1], meta->rng[0]}, inc, (uint64_t)t0);
    for (int q = 0; q < 8 && t0 + q < outs; q++) {
        s = add128(mul128(s, u128{PCG_MULT_LO, PCG_MULT_HI}), inc);
        const uint64_t o = pcg_output(s);
        const int64_t j = (has ? 1 : 0) + 2 * (t0 + q);
        if (j < hcap) H[j] = (uint32_t)o;
        if (j + 1 < hcap) H[j + 1] = (uint32_t)(o >> 32);
    }
}

struct XpArgs {
    const uint32_t* ev;      // (line_at_start + 1) << 1 | (ca > 0)
    const uint32_t* xcls;    // class | candidate index << 3
    int64_t n, L;
    CacheMeta* meta;
    ServeCounters* svc;
    uint32_t* safe_bits;     // padded to whole 1024-line blocks
    uint32_t* blk_cnt;
    uint32_t* sup_cnt;
    const int32_t* cand_of_slot;
    int64_t cand_cap;
    int64_t safe_div;
    const uint32_t* H;
    int64_t hcap;
    int8_t* kind;
    int32_t* line;
    int32_t* log_line;
    int32_t* log_pos;
    const ServeArgs* sa;     // (graph replay: n from here)
};

// shared-memory view of the round state.  Within a round the tables and the
// global bitmap describe T = (round-start safe set) + (the round's ADD lines);
// an access sees T minus its "holes": the ADD lines of later accesses and the
// lines removed by earlier MU accesses.
struct Xs {
    uint32_t* CNT;    // [nb] lines of T per block
    uint32_t* BLKP;   // [nb] exclusive prefix within the 32-block superblock
    uint32_t* SUPP;   // [ns+1] exclusive prefix over superblocks
    uint32_t* CONV;   // [cand_cap/32] candidates whose line was taken
    uint32_t* GCNT;   // [2*nb] lines of T per 128-line group, one byte each
    int32_t* FIN;     // [XP_MAX_CHG] MU lines found by the current pass
    unsigned long long* MOVM;  // [MOVN] per bucket: MU changes whose move crossed it (this pass)
    int32_t* CUMB;    // [CUMN+1] changes with line < (b << bsh), b = 0..CUMN
    int32_t* CHK;     // [HSZ] candidate lines of the round (MISC[7] of them)
    int32_t* CHV;     // [HSZ] their lanes
    uint32_t* CHB;    // [CHBW] filter bits of their lines (line & 4095)
    uint32_t* REV;    // [RING]
    uint32_t* RCL;    // [RING]
    uint32_t* RH;     // [HRING]
    int32_t* ANS;     // [XT] final line per evicting access of the round, -1
    int32_t* PANS;    // [XT] same, previous round
    int32_t* CSLOT;   // [XP_MAX_CHG] line of each set change, in access order
    int32_t* CTYPE;   // [XP_MAX_CHG] +1 ADD, -1 MU
    int32_t* SS;      // [XP_MAX_CHG] change lines, ascending
    int32_t* SIDX;    // [XP_MAX_CHG] their change indices
    int32_t* RANKS;   // [XP_MAX_CHG] rank of each change (by line)
    int32_t* CHT;     // [XP_MAX_CHG] the access (thread) of each change
    unsigned long long* PM;  // [XP_MAX_CHG+1] change-index mask of the k lowest lines
    int32_t* W;       // [XW * 8] warp partials
    int32_t* MISC;    // [16]
    int32_t nb, ns, L;  // (a cache of L < 2^31 lines: int32 index math throughout)
    int bsh;
    const uint32_t* gbits;
};

__device__ __forceinline__ uint32_t pb(const Xs& x, int32_t g) { return x.SUPP[g >> 5] + x.BLKP[g]; }

// block holding the r-th line of T (r < total): interpolated guess, then
// steps sized by the mean block count (float arithmetic: only a guess)
__device__ int32_t locate(const Xs& x, uint32_t r, uint32_t total) {
    const int32_t nb = x.nb;
    const float per = __fdividef((float)nb, (float)total);  // blocks per line
    int32_t g = (int32_t)((float)r * per);
    if (g >= nb) g = nb - 1;
    if (g < 0) g = 0;
    for (int it = 0; it < 6; it++) {
        const uint32_t base = pb(x, g), c = x.CNT[g];
        if (r < base) {
            const int32_t st = (int32_t)((float)(base - r) * per) + 1;
            g = g - st < 0 ? 0 : g - st;
        } else if (r >= base + c) {
            const int32_t st = (int32_t)((float)(r - base - c) * per) + 1;
            g = g + st >= nb ? nb - 1 : g + st;
        } else {
            return g;
        }
    }
    int32_t lo = 0, hi = nb - 1;  // largest g with pb(g) <= r
    while (lo < hi) {
        const int32_t mid = (lo + hi + 1) >> 1;
        if (pb(x, mid) <= r) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// position of the k-th set bit of w (k < popc(w))
__device__ __forceinline__ int bit_select(uint32_t w, uint32_t k) {
    int pos = 0;
    uint32_t c = __popc(w & 0xffffu);
    if (k >= c) { k -= c; pos = 16; }
    c = __popc((w >> pos) & 0xffu);
    if (k >= c) { k -= c; pos += 8; }
    c = __popc((w >> pos) & 0xfu);
    if (k >= c) { k -= c; pos += 4; }
    c = __popc((w >> pos) & 0x3u);
    if (k >= c) { k -= c; pos += 2; }
    if (k >= ((w >> pos) & 1u)) pos += 1;
    return pos;
}

// the 128-line group of T an access last selected in: its four bitmap words
// (one 16-B load from the L2-resident bitmap), rank base and count
struct Grp {
    int32_t gi;     // group (line >> 7), -1 none
    uint32_t base, cnt;
    uint4 w;
    uint32_t cnt2;  // the next group, prefetched with it (0: none)
    uint4 w2;
};

// the k-th set bit of the held group
__device__ __forceinline__ int32_t sel_grp(const Grp& G, uint32_t k) {
    uint32_t w = G.w.x;
    int wi = 0;
    uint32_t c = __popc(G.w.x);
    if (k >= c) {
        k -= c;
        wi = 1;
        w = G.w.y;
        c = __popc(G.w.y);
        if (k >= c) {
            k -= c;
            wi = 2;
            w = G.w.z;
            c = __popc(G.w.z);
            if (k >= c) {
                k -= c;
                wi = 3;
                w = G.w.w;
            }
        }
    }
    return G.gi * 128 + wi * 32 + bit_select(w, k);
}

// hold the 128-line group of T holding rank q (its words are loaded, not
// waited for: the first use waits)
__device__ __forceinline__ void find_grp(const Xs& x, uint32_t q, uint32_t total, Grp& G) {
    int32_t g = -1;
    uint32_t base = 0;
    if (G.gi >= 0) {
        base = pb(x, G.gi >> 3);
        if (q >= base && q < base + x.CNT[G.gi >> 3]) g = G.gi >> 3;
    }
    if (g < 0) {
        g = locate(x, q, total);
        base = pb(x, g);
    }
    const uint2 cc = *reinterpret_cast<const uint2*>(x.GCNT + 2 * g);
    // the group of in-block rank rr: a 3-step search over the byte counts
    // (dp4a sums four bytes)
    uint32_t rem = q - base;
    const uint32_t s4 = __dp4a(cc.x, 0x01010101u, 0u);
    const bool h4 = rem >= s4;
    uint32_t w = h4 ? cc.y : cc.x, accb = h4 ? s4 : 0u;
    rem -= h4 ? s4 : 0u;
    const uint32_t s2 = (w & 0xffu) + ((w >> 8) & 0xffu);
    const bool h2 = rem >= s2;
    w = h2 ? (w >> 16) : w;
    accb += h2 ? s2 : 0u;
    rem -= h2 ? s2 : 0u;
    const uint32_t c0 = w & 0xffu;
    const bool h1 = rem >= c0;
    const int grp = (h4 ? 4 : 0) + (h2 ? 2 : 0) + (h1 ? 1 : 0);
    accb += h1 ? c0 : 0u;
    G.gi = (int32_t)(g * 8 + grp);
    G.base = base + accb;
    G.cnt = h1 ? ((w >> 8) & 0xffu) : c0;
    G.w = __ldcg(reinterpret_cast<const uint4*>(x.gbits) + G.gi);
    // and the next group: a fixed point moves up by the few holes below, so
    // its answer is usually here or there
    const int32_t gn = G.gi + 1;
    G.cnt2 = 0;
    if (gn < (int32_t)(x.nb * 8)) {
        G.cnt2 = (x.GCNT[gn >> 2] >> ((gn & 3) * 8)) & 0xffu;
        G.w2 = __ldcg(reinterpret_cast<const uint4*>(x.gbits) + gn);
    }
}

// the q-th line of T (the held group is reused when it covers q)
__device__ __forceinline__ int32_t sel_T(const Xs& x, uint32_t q, uint32_t total, Grp& G) {
    if (!(G.gi >= 0 && q - G.base < G.cnt)) {
        if (G.gi >= 0 && q - G.base - G.cnt < G.cnt2 && q >= G.base + G.cnt) {  // the next group
            G.base += G.cnt;
            G.cnt = G.cnt2;
            G.w = G.w2;
            G.gi += 1;
            G.cnt2 = 0;
        } else {
            find_grp(x, q, total, G);
        }
    }
    return sel_grp(G, q - G.base);
}

// lane of the round's candidate whose line this is, -1 none (a filter bit
// first: almost every answer is no candidate's line)
__device__ __forceinline__ int32_t cand_lane(const Xs& x, int32_t line) {
    if (!((x.CHB[(line >> 5) & (CHBW - 1)] >> (line & 31)) & 1u)) return -1;
    const int nc = x.MISC[7];
    for (int k = 0; k < nc; k++)
        if (x.CHK[k] == line) return x.CHV[k];
    return -1;
}

// lines among the round's changes <= y: the bucket's start, then the few
// changes inside the bucket
__device__ __forceinline__ int count_le(const Xs& x, int m, int32_t y) {
    int j = x.CUMB[y >> x.bsh];
    while (j < m && x.SS[j] <= y) j++;
    return j;
}

// one line joins (+1) or leaves (-1) T: block / group counts and the two
// prefix levels, updated in place by one warp (a lane per prefix entry;
// the round's changes are spread over the warps)
__device__ __forceinline__ void t_update_warp(const Xs& x, int32_t s, int delta, int lane) {
    const int32_t g = s >> 10, sb = g >> 5;
    const uint32_t d = (uint32_t)delta;
    if (lane == 0) {
        atomicAdd(&x.CNT[g], d);
        atomicAdd(&x.GCNT[s >> 9], d << (((s >> 7) & 3) * 8));
    }
    const int32_t ge = (sb + 1) * 32 < x.nb ? (sb + 1) * 32 : x.nb;
    if (g + 1 + lane < ge) atomicAdd(&x.BLKP[g + 1 + lane], d);
    for (int32_t u = sb + 1 + lane; u <= x.ns; u += 32) atomicAdd(&x.SUPP[u], d);
}

// the r-th line of T minus `holes` (a mask over the change list): the least
// fixed point of q = r + #holes(<= sel_T(q)).  Every fixed point lies at or
// above r + #holes below the block holding T's r-th line (the answer is not
// below that block), so the iteration starts there -- usually already the
// answer, one bitmap load.  The hole counts it used: at line lb, and at the
// lines of [ylo, answer].
__device__ __forceinline__ int32_t resolve(const Xs& x, uint32_t r, unsigned long long holes,
                                           int m, uint32_t total, int32_t rblk, Grp& B,
                                           int32_t& lb, int32_t& ylo) {
    if (!holes) {
        const int32_t y = sel_T(x, r, total, B);
        ylo = y;
        lb = -1;
        return y;
    }
    lb = rblk * 1024 - 1;  // (rblk: the block of T's r-th line)
    uint32_t q = r + (lb >= 0 ? (uint32_t)__popcll(x.PM[count_le(x, m, lb)] & holes) : 0u);
    int32_t y = sel_T(x, q, total, B);
    ylo = y;
    for (int it = 0; it <= XP_MAX_CHG; it++) {
        const uint32_t q2 = r + (uint32_t)__popcll(x.PM[count_le(x, m, y)] & holes);
        if (q2 == q) break;
        q = q2;
        y = sel_T(x, q, total, B);
    }
    return y;
}

// the prefix tables from CNT (all threads; ends synchronised).  Once, at
// the start: rounds then update them in place (t_update).
__device__ void prefix_all(const Xs& x, int t) {
    const int lane = t & 31, wid = t >> 5;
    for (int64_t sb = wid; sb < x.ns; sb += XW) {
        const int64_t blk = sb * 32 + lane;
        const uint32_t c = blk < x.nb ? x.CNT[blk] : 0u;
        uint32_t inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (blk < x.nb) x.BLKP[blk] = inc - c;
        if (lane == 31) x.SUPP[sb + 1] = inc;  // (superblock total, summed below)
    }
    __syncthreads();
    if (t == 0) {
        uint32_t run = 0;
        x.SUPP[0] = 0;
        for (int64_t u = 1; u <= x.ns; u++) {
            run += x.SUPP[u];
            x.SUPP[u] = run;
        }
    }
    __syncthreads();
}

__device__ __forceinline__ uint32_t get_half(const Xs& x, const XpArgs& a, int32_t k,
                                             int32_t kfill) {
    if (k < kfill && k >= kfill - HRING) return x.RH[k & (HRING - 1)];
    if (k < (int32_t)a.hcap) return __ldcg(a.H + k);
    return half_direct(a.meta, k);
}

// numpy's Generator.integers(n) (Lemire, buffered 32-bit halves) from stream
// position k: r in [0, n), `extra` halves consumed beyond the first
__device__ __forceinline__ void lemire(const Xs& x, const XpArgs& a, int32_t k, int32_t kfill,
                                       uint32_t n, uint32_t& r, int& extra) {
    extra = 0;
    uint64_t m = (uint64_t)get_half(x, a, k, kfill) * n;
    uint32_t left = (uint32_t)m;
    if (left < n) {
        const uint32_t thr = (0u - n) % n;
        while (left < thr) {
            extra++;
            m = (uint64_t)get_half(x, a, k + extra, kfill) * n;
            left = (uint32_t)m;
        }
    }
    r = (uint32_t)(m >> 32);
}

// (d, c): x -> max(x + d, c); (d2, c2) becomes "(d1, c1) first, then (d2, c2)"
__device__ __forceinline__ void sat_compose(int32_t d1, int32_t c1, int32_t& d2, int32_t& c2) {
    const int32_t c = max(c1 + d2, c2);
    d2 = d1 + d2;
    c2 = c;
}

__device__ __forceinline__ void stage(uint32_t* dst, const uint32_t* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src));
}

__global__ void __launch_bounds__(XT, 1) k_exact_par(XpArgs a) {
    if (!xp_runs(a.meta, a.svc, a.L, a.cand_cap, a.safe_div)) return;
    extern __shared__ __align__(16) uint32_t smem[];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const unsigned below = (1u << lane) - 1u;
    Xs x;
    x.L = (int32_t)a.L;
    x.nb = (int32_t)((a.L + 1023) >> 10);
    x.ns = (x.nb + 31) >> 5;
    x.gbits = a.safe_bits;
    {
        uint32_t* p = smem;
        x.PM = reinterpret_cast<unsigned long long*>(p);
        p += 2 * (XP_MAX_CHG + 2);
        x.GCNT = p;
        p += 2 * x.nb;
        x.FIN = reinterpret_cast<int32_t*>(p);
        p += XP_MAX_CHG;
        x.CUMB = reinterpret_cast<int32_t*>(p);
        p += CUMN + 2;
        x.CHK = reinterpret_cast<int32_t*>(p);
        p += HSZ;
        x.CHV = reinterpret_cast<int32_t*>(p);
        p += HSZ;
        x.CHB = p;
        p += CHBW;
        x.REV = p;
        p += RING;
        x.RCL = p;
        p += RING;
        x.RH = p;
        p += HRING;
        x.CNT = p;
        p += x.nb;
        x.BLKP = p;
        p += x.nb;
        x.SUPP = p;
        p += x.ns + 1;
        x.CONV = p;
        p += (a.cand_cap + 31) / 32;
        x.ANS = reinterpret_cast<int32_t*>(p);
        p += XT;
        x.PANS = reinterpret_cast<int32_t*>(p);
        p += XT;
        x.CSLOT = reinterpret_cast<int32_t*>(p);
        p += XP_MAX_CHG;
        x.CTYPE = reinterpret_cast<int32_t*>(p);
        p += XP_MAX_CHG;
        x.SS = reinterpret_cast<int32_t*>(p);
        p += XP_MAX_CHG;
        x.SIDX = reinterpret_cast<int32_t*>(p);
        p += XP_MAX_CHG;
        x.RANKS = reinterpret_cast<int32_t*>(p);
        p += XP_MAX_CHG;
        x.CHT = reinterpret_cast<int32_t*>(p);
        p += XP_MAX_CHG;
        x.W = reinterpret_cast<int32_t*>(p);
        p += XW * 8;
        x.MISC = reinterpret_cast<int32_t*>(p);
        p += 16;
        p += (reinterpret_cast<uintptr_t>(p) & 7) ? 1 : 0;
        x.MOVM = reinterpret_cast<unsigned long long*>(p);
    }
    x.bsh = 0;
    while (((x.L - 1) >> x.bsh) >= CUMN) x.bsh++;
    const int32_t n = (int32_t)(a.sa ? a.sa->n : a.n), nb = x.nb, ns = x.ns;  // (n <= serve_cap < 2^31)
    const int32_t hcap = (int32_t)a.hcap;
    for (int64_t i = t; i < nb; i += XT) x.CNT[i] = a.blk_cnt[i];
    for (int64_t i = t; i < 2 * nb; i += XT) {  // four 128-line group counts per word
        const uint4* src = reinterpret_cast<const uint4*>(a.safe_bits + i * 16);
        uint32_t packed = 0;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const uint4 v = __ldcg(src + q);
            packed |= (uint32_t)(__popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w)) << (8 * q);
        }
        x.GCNT[i] = packed;
    }
    for (int64_t i = t; i < (a.cand_cap + 31) / 32; i += XT) x.CONV[i] = 0u;
    for (int i = t; i < CHBW; i += XT) x.CHB[i] = 0u;
    for (int i = t; i < MOVN; i += XT) x.MOVM[i] = 0ull;
    x.PANS[t] = -1;
    // stage the first accesses and halves
    int32_t efill = n < RING ? n : RING;
    int32_t kfill = hcap < HRING ? hcap : HRING;
    for (int32_t i = t; i < efill; i += XT) {
        stage(&x.REV[i & (RING - 1)], a.ev + i);
        stage(&x.RCL[i & (RING - 1)], a.xcls + i);
    }
    for (int32_t i = t; i < kfill; i += XT) stage(&x.RH[i & (HRING - 1)], a.H + i);
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 0;");
    __syncthreads();
    prefix_all(x, t);

    int movs = 0;  // moved-line filter: MOVN buckets over the lines
    while (((x.L - 1) >> movs) >= MOVN) movs++;
    int32_t pos = 0, kpos = 0, nlog = 0;
    int32_t nsafe = (int32_t)a.meta->safe_count;
    int32_t pend_cidx = -1;  // cand_of_slot of this thread's last committed eviction
    int64_t hits = 0, misses = 0, byp = 0;
    int64_t st_rounds = 0, st_rej = 0, st_chg = 0, st_conv = 0;  // round ends (thread 0)
    long long prof[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // cycles per phase, passes (thread 0)
    long long tc = GIDS_XP_PROF ? clock64() : 0;

    while (pos < n) {
        // (the ring entries this round reads were waited for before the last
        // round's closing barrier, which also ordered its commit)
        XP_MARK(10);  // (refill issue)
        // ---------------- A: classify, saturating safe-count prefix, draw prefix
        const int32_t p = pos + t;
        const bool valid = p < n;
        const uint32_t e = valid ? x.REV[p & (RING - 1)] : 0u;
        const uint32_t xc = valid ? x.RCL[p & (RING - 1)] : 0u;
        const int32_t s = (int32_t)(e >> 1) - 1;
        const int cls = (int)(xc & 7u);
        const uint32_t cidx = xc >> 3;
        const bool conv = valid && cls == C_CAND && ((x.CONV[cidx >> 5] >> (cidx & 31)) & 1u);
        const bool miss = valid && (cls == C_M0 || cls == C_MU || conv);
        int32_t d = 0, c = NEG;
        if (valid && cls == C_ADD) d = 1;
        if (miss && cls == C_MU) {
            d = -1;
            c = 0;
        }
        if (t == 0) {
            x.MISC[0] = XT;  // end of the round before conversions (min)
            x.MISC[1] = XT;  // first candidate that lost its line (min)
            x.MISC[3] = 0;   // set changes in the round
            x.MISC[7] = 0;   // unconverted candidates of the round
            x.MISC[8] = XT;  // first Lemire rejection (+1)
            x.MISC[15] = 0;  // Lemire rejections in the round
            x.MISC[11] = 0;  // ADD changes (bits by change index, 11: 0-31, 12: 32-63)
            x.MISC[12] = 0;
            x.MISC[9] = XT;  // end by a full change list
            x.MISC[14] = XT;  // first candidate whose line the previous round took (min)
        }
        int32_t ni, pdr, psel, pchg;
        bool sel, dr, chg;
        if (nsafe >= XT + 2) {
            // no access of the round can see fewer than 2 safe lines: every
            // miss evicts and draws, so one packed scan of (misses, ADDs,
            // MUs) gives the safe count, draw, log and change positions
            const uint32_t pk = (miss ? 1u : 0u) | ((valid && cls == C_ADD) ? (1u << 10) : 0u) |
                                ((miss && cls == C_MU) ? (1u << 20) : 0u);
            uint32_t inc = pk;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += u;
            }
            if (lane == 31) x.W[wid * 8 + 0] = (int32_t)inc;
            __syncthreads();
            uint32_t wv = lane < XW ? (uint32_t)x.W[lane * 8 + 0] : 0u;
#pragma unroll
            for (int o = 1; o < XW; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, wv, o);
                if (lane >= o) wv += u;
            }
            const uint32_t wp = __shfl_sync(0xffffffffu, wv, wid > 0 ? wid - 1 : 0);
            const uint32_t ex = inc - pk + (wid > 0 ? wp : 0u);
            const int32_t em = (int32_t)(ex & 1023u), ea = (int32_t)((ex >> 10) & 1023u),
                          eu = (int32_t)(ex >> 20);
            ni = nsafe + ea - eu;
            sel = miss;
            dr = miss;
            chg = valid && (cls == C_ADD || cls == C_MU);
            pdr = em;
            psel = em;
            pchg = ea + eu;
        } else {
            int32_t di = d, ci = c;  // inclusive warp scan of the saturating map
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t d2 = __shfl_up_sync(0xffffffffu, di, o);
                const int32_t c2 = __shfl_up_sync(0xffffffffu, ci, o);
                if (lane >= o) sat_compose(d2, c2, di, ci);
            }
            int32_t de = __shfl_up_sync(0xffffffffu, di, 1), ce = __shfl_up_sync(0xffffffffu, ci, 1);
            if (lane == 0) {
                de = 0;
                ce = NEG;
            }
            if (lane == 31) {
                x.W[wid * 8 + 0] = di;
                x.W[wid * 8 + 1] = ci;
            }
            __syncthreads();
            {  // earlier warps, composed: lane w holds warp w's map, scanned across lanes
                int32_t wd = lane < XW ? x.W[lane * 8 + 0] : 0,
                        wc = lane < XW ? x.W[lane * 8 + 1] : NEG;
#pragma unroll
                for (int o = 1; o < XW; o <<= 1) {
                    const int32_t d2 = __shfl_up_sync(0xffffffffu, wd, o);
                    const int32_t c2 = __shfl_up_sync(0xffffffffu, wc, o);
                    if (lane >= o) sat_compose(d2, c2, wd, wc);
                }
                int32_t dp = __shfl_sync(0xffffffffu, wd, wid > 0 ? wid - 1 : 0);
                int32_t cp = __shfl_sync(0xffffffffu, wc, wid > 0 ? wid - 1 : 0);
                if (wid == 0) {
                    dp = 0;
                    cp = NEG;
                }
                sat_compose(dp, cp, de, ce);  // exclusive prefix at this thread
            }
            ni = max(nsafe + de, ce);  // safe lines seen by this access
            sel = miss && ni >= 1;     // evicts (else bypass)
            dr = miss && ni >= 2;      // consumes a draw (integers(1) draws nothing)
            chg = valid && (cls == C_ADD || (cls == C_MU && sel));
            const unsigned bdr = __ballot_sync(0xffffffffu, dr);
            const unsigned bsel = __ballot_sync(0xffffffffu, sel);
            const unsigned bchg = __ballot_sync(0xffffffffu, chg);
            if (lane == 0) {
                x.W[wid * 8 + 2] = __popc(bdr);
                x.W[wid * 8 + 3] = __popc(bsel);
                x.W[wid * 8 + 4] = __popc(bchg);
            }
            __syncthreads();
            pdr = __popc(bdr & below);
            psel = __popc(bsel & below);
            pchg = __popc(bchg & below);
            {  // earlier warps' counts: exclusive scan across lanes
                int32_t v2 = lane < XW ? x.W[lane * 8 + 2] : 0, v3 = lane < XW ? x.W[lane * 8 + 3] : 0,
                        v4 = lane < XW ? x.W[lane * 8 + 4] : 0;
#pragma unroll
                for (int o = 1; o < XW; o <<= 1) {
                    const int32_t u2 = __shfl_up_sync(0xffffffffu, v2, o);
                    const int32_t u3 = __shfl_up_sync(0xffffffffu, v3, o);
                    const int32_t u4 = __shfl_up_sync(0xffffffffu, v4, o);
                    if (lane >= o) {
                        v2 += u2;
                        v3 += u3;
                        v4 += u4;
                    }
                }
                const int src = wid > 0 ? wid - 1 : 0;
                const int32_t e2 = __shfl_sync(0xffffffffu, v2, src),
                              e3 = __shfl_sync(0xffffffffu, v3, src),
                              e4 = __shfl_sync(0xffffffffu, v4, src);
                if (wid > 0) {
                    pdr += e2;
                    psel += e3;
                    pchg += e4;
                }
            }
        }
        // ---------------- B: draws
        uint32_t r = 0;
        int extra = 0;
        if (dr) {
            lemire(x, a, kpos + pdr, kfill, (uint32_t)ni, r, extra);
            if (extra) {  // a Lemire rejection: later draws sit `extra` halves later
                atomicMin(&x.MISC[8], t + 1);
                atomicAdd(&x.MISC[15], 1);
                x.MISC[2] = extra;  // (read only when it is the round's one rejection)
            }
        }
        if (chg && pchg == XP_MAX_CHG) {  // change list full
            atomicMin(&x.MISC[0], t);
            atomicMin(&x.MISC[9], t);
        }
        __syncthreads();
        if (x.MISC[15] == 1) {
            // the round's one rejection: the accesses after it redraw from
            // their shifted stream positions instead of ending the round; a
            // rejection among those redraws ends the round after it
            const int j = x.MISC[8] - 1, ex = x.MISC[2];
            if (t > j) {
                pdr += ex;
                if (dr) {
                    lemire(x, a, kpos + pdr, kfill, (uint32_t)ni, r, extra);
                    if (extra) atomicMin(&x.MISC[0], t + 1);
                }
            }
            __syncthreads();
        } else if (x.MISC[15] > 1) {  // several: the round ends after the first
            if (t == 0) x.MISC[0] = min(x.MISC[0], x.MISC[8]);
            __syncthreads();
        }
        XP_MARK(0);  // A + B
        const int Epre0 = x.MISC[0];
        const int Epre = (int)((n - pos) < Epre0 ? (n - pos) : Epre0);
        const bool in = t < Epre;
        // ---------------- C: T = start set + the round's ADD lines; the start-of-T answers
        if (chg && in) {
            x.CTYPE[pchg] = cls == C_ADD ? 1 : -1;
            x.CHT[pchg] = t;
            atomicMax(&x.MISC[3], pchg + 1);
            if (cls == C_ADD) {
                x.CSLOT[pchg] = s;
                atomicOr(&a.safe_bits[s >> 5], 1u << (s & 31));
                atomicOr(reinterpret_cast<unsigned*>(&x.MISC[11 + (pchg >> 5)]), 1u << (pchg & 31));
            }
        }
        if (valid && in && cls == C_CAND && !conv) {
            const int k = atomicAdd(&x.MISC[7], 1);
            x.CHK[k] = s;
            x.CHV[k] = t;
            atomicOr(&x.CHB[(s >> 5) & (CHBW - 1)], 1u << (s & 31));
        }
        __syncthreads();
        {  // the round's ADD lines join T's tables
            const int nc0 = x.MISC[3];
            for (int e = wid; e < nc0; e += XW)
                if (x.CTYPE[e] > 0) t_update_warp(x, x.CSLOT[e], +1, lane);
        }
        __syncthreads();
        XP_MARK(1);  // C: T tables
        const int nchg = x.MISC[3];
        const uint32_t total = x.SUPP[ns];
        Grp B;
        B.gi = -1;
        int32_t cur = -1, ylo = -1, lb = -1;
        int32_t rblk = 0;
        if (sel && in) {
            // the group of T's r-th line: its load overlaps the change sort;
            // an MU access's first approximation of its line is interpolated
            // inside that group (no wait: the fixed point corrects it)
            find_grp(x, r, total, B);
            rblk = B.gi >> 3;
            if (chg && cls == C_MU)
                x.CSLOT[pchg] = B.gi * 128 + (int32_t)__fdividef((float)(r - B.base) * 128.f,
                                                                  (float)(B.cnt ? B.cnt : 1u));
        }
        __syncthreads();
        XP_MARK(2);  // C selects
        // ---------------- D/E: every eviction resolves against the change list.
        // The MU lines are themselves answers, so a pass uses the previous
        // pass's MU lines (the first pass: their no-hole lines); the result is
        // exact unless, for some access, an earlier MU line moved across the
        // range of lines its fixed-point iteration looked at -- checked
        // exactly, and another pass run (rare: the moves are short)
        const unsigned long long mine = pchg >= 64 ? ~0ull : ((1ull << pchg) - 1ull);
        int32_t mlo = 0, mhi = -1;  // buckets this MU marked in MOVM (cleared after use)
        for (int pass = 0; pass <= XP_MAX_CHG + 1; pass++) {
            if (pass > 0) __syncthreads();  // (pass 0: the first selects' barrier)
            // sort the change lines (rank sort), then the prefix masks
            {  // rank of change e = t / 8 among the changes of slice t % 8
                const int e = t >> 3, part = t & 7;
                const int32_t v = e < nchg ? x.CSLOT[e] : 0;
                int rk = 0;
                if (e < nchg)
                    for (int j = part * 8; j < part * 8 + 8 && j < nchg; j++) {
                        const int32_t u = x.CSLOT[j];
                        rk += (u < v || (u == v && j < e)) ? 1 : 0;
                    }
                rk += __shfl_xor_sync(0xffffffffu, rk, 1);
                rk += __shfl_xor_sync(0xffffffffu, rk, 2);
                rk += __shfl_xor_sync(0xffffffffu, rk, 4);
                if (e < nchg && part == 0) {
                    x.SS[rk] = v;
                    x.SIDX[rk] = e;
                }
                if (e < nchg && part == 1) x.FIN[e] = v;  // (ADD lines are final)
                if (e < nchg && part == 2) x.RANKS[e] = rk;
            }
            if (t == 0) {
                x.MISC[10] = 0;
                x.MISC[13] = 0;  // an MU moved across more than MOVSPAN buckets
            }
            __syncthreads();
            XP_MARK(3);  // sort
            // PM[k] = change indices of the k lowest lines: thread (k, half)
            // builds one 32-bit half from the ranks (no serial scan)
            if (t < 2 * (nchg + 1)) {
                const int k = t >> 1, h0 = (t & 1) * 32;
                const int hn = nchg - h0 < 32 ? nchg - h0 : 32;
                uint32_t m = 0;
                for (int j = 0; j < hn; j++) m |= (x.RANKS[h0 + j] < k ? 1u : 0u) << j;
                reinterpret_cast<uint32_t*>(x.PM)[2 * k + (t & 1)] = m;
            } else if (t >= XT - (XP_MAX_CHG + 1) && t - (XT - (XP_MAX_CHG + 1)) <= nchg) {
                // CUMB[b] = changes with line < b << bsh: sorted change j fills the
                // buckets after its predecessor's up to its own (j = nchg: the rest)
                const int j = t - (XT - (XP_MAX_CHG + 1));
                const int lo = j == 0 ? 0 : (x.SS[j - 1] >> x.bsh) + 1;
                const int hi = j == nchg ? CUMN : (x.SS[j] >> x.bsh);
                for (int b = lo; b <= hi; b++) x.CUMB[b] = j;
            }
            __syncthreads();
            XP_MARK(4);  // resolve
            const unsigned long long addm =
                (unsigned long long)(uint32_t)x.MISC[11] |
                ((unsigned long long)(uint32_t)x.MISC[12] << 32);
            const unsigned long long allm = nchg >= 64 ? ~0ull : ((1ull << nchg) - 1ull);
            const unsigned long long holes = (addm & ~mine & allm) | (~addm & mine & allm);
            if (sel && in) {
                cur = resolve(x, r, holes, nchg, total, rblk, B, lb, ylo);
                if (chg && cls == C_MU) {
                    x.FIN[pchg] = cur;
                    const int32_t u0 = x.CSLOT[pchg];
                    if (u0 != cur) {  // mark the buckets the move spans (short moves)
                        mlo = min(u0, cur) >> movs;
                        mhi = max(u0, cur) >> movs;
                        if (mhi - mlo >= MOVSPAN) {
                            x.MISC[13] = 1;
                            mhi = -1;
                        }
                        for (int32_t b = mlo; b <= mhi; b++) atomicOr(&x.MOVM[b], 1ull << pchg);
                    }
                }
            }
            __syncthreads();
            XP_MARK(5);  // verify
            if (t == 0) prof[7]++;
            // the earlier MU lines this access counted, used vs found: only
            // those whose move crossed a bucket of the lines it looked at
            unsigned long long mu = 0;
            if (sel && in) {
                if (x.MISC[13] || (cur >> movs) - (ylo >> movs) >= MOVSPAN) {
                    mu = ~0ull;  // (a long move or range: all earlier MUs)
                } else {
                    for (int32_t b = ylo >> movs; b <= (cur >> movs); b++) mu |= x.MOVM[b];
                    if (lb >= 0) mu |= x.MOVM[lb >> movs];
                }
                mu &= ~addm & mine & allm;
            }
            if (mu) {
                bool moved = false;
                while (mu) {
                    const int i = __ffsll((long long)mu) - 1;
                    mu &= mu - 1;
                    const int32_t u0 = x.CSLOT[i], u1 = x.FIN[i];
                    if (u0 != u1 && ((max(u0, u1) >= ylo && min(u0, u1) <= cur) ||
                                     ((u0 <= lb) != (u1 <= lb))))
                        moved = true;
                }
                if (moved) x.MISC[10] = 1;
            }
            // ---------------- F (with the check, one barrier): a candidate whose
            // line an earlier eviction took -- each access checks its own answer
            // of this pass (MISC[1], redone by a further pass) and of the previous
            // round (MISC[14], once) against the round's few candidates
            if (sel && in) {
                const int32_t cl = cand_lane(x, cur);
                if (cl > t) atomicMin(&x.MISC[1], cl);
            }
            if (pass == 0) {
                const int32_t mine_prev = x.PANS[t];
                if (mine_prev >= 0) {
                    const int32_t cl = cand_lane(x, mine_prev);
                    if (cl >= 0) atomicMin(&x.MISC[14], cl);
                }
            }
            __syncthreads();
            for (int32_t b = mlo; b <= mhi; b++) x.MOVM[b] = 0ull;  // (read above, all done)
            mhi = -1;
            if (!x.MISC[10]) break;
            if (t == 0) x.MISC[1] = XT;  // (read only after the last pass's barrier)
            if (chg && in && cls == C_MU) x.CSLOT[pchg] = cur;  // next pass
        }
        const int32_t pans = (sel && in) ? cur : -1;  // this thread's answer, for the next round's F
        const int lost = x.MISC[1] < x.MISC[14] ? x.MISC[1] : x.MISC[14];
        const int E = Epre < lost ? Epre : lost;
        XP_MARK(8);  // check + F
        if (t == 0) {
            st_rounds++;
            if (E < n - pos && E < XT) {
                if (E == lost) st_conv++;
                else if (E == x.MISC[9]) st_chg++;
                else st_rej++;
            }
        }
        if (t == E && E < Epre)  // (atomic: other lanes OR their pend_cidx bits into the same words)
            atomicOr(&x.CONV[cidx >> 5], 1u << (cidx & 31));
        // ---------------- G: commit the accesses [pos, pos + E)
        if (pend_cidx >= 0) atomicOr(&x.CONV[pend_cidx >> 5], 1u << (pend_cidx & 31));
        pend_cidx = -1;
        if (t < E) {
            int kd, ln;
            if (!miss) {
                kd = GIDS_KIND_HIT;
                ln = s;
                hits++;
            } else if (sel) {
                kd = GIDS_KIND_MISS;
                ln = cur;
                misses++;
                const int32_t li = nlog + psel;
                a.log_line[li] = cur;
                a.log_pos[li] = (int32_t)p;
                pend_cidx = __ldcg(a.cand_of_slot + cur);
            } else {
                kd = GIDS_KIND_BYPASS;
                ln = -1;
                byp++;
            }
            a.kind[p] = (int8_t)kd;
            a.line[p] = ln;
        }
        // committed MU lines leave T; ADD lines of accesses past the end return
        {
            const int nc0 = x.MISC[3];
            for (int e = wid; e < nc0; e += XW) {
                const bool add = x.CTYPE[e] > 0, done = x.CHT[e] < E;
                if (add == done) continue;
                const int32_t off = add ? x.CSLOT[e] : x.FIN[e];
                if (lane == 0) atomicAnd(&a.safe_bits[off >> 5], ~(1u << (off & 31)));
                t_update_warp(x, off, -1, lane);
            }
        }
        for (int i = t; i < CHBW; i += XT) x.CHB[i] = 0u;  // (read in F, before the barrier above)
        // state after the last committed access
        if (t == E - 1) {
            x.MISC[4] = max(ni + d, c);              // safe count after it
            x.MISC[5] = pdr + (dr ? 1 + extra : 0);  // halves consumed through it
            x.MISC[6] = psel + (sel ? 1 : 0);        // log entries through it
        }
        // the next round's staged entries have landed (the groups issued before
        // this round's refill, RING_LAG - 1 of them still in flight: as with a
        // wait of RING_LAG after it), for every thread after the barrier
        asm volatile("cp.async.wait_group %0;" ::"n"(RING_LAG - 1));
        __syncthreads();
        XP_MARK(9);  // G commit (+ ring wait)
        if (E > 0) {
            nsafe = x.MISC[4];
            kpos += x.MISC[5];
            nlog += x.MISC[6];
        }
        x.PANS[t] = t < E ? pans : -1;
        pos += E;
        // refill the rings past the consumed prefix
        {
            const int32_t etop = (pos + RING) < n ? pos + RING : n;
            for (int32_t i = efill + t; i < etop; i += XT) {
                stage(&x.REV[i & (RING - 1)], a.ev + i);
                stage(&x.RCL[i & (RING - 1)], a.xcls + i);
            }
            efill = etop > efill ? etop : efill;
            const int32_t ktop = (kpos + HRING) < hcap ? kpos + HRING : hcap;
            for (int32_t i = kfill + t; i < ktop; i += XT) stage(&x.RH[i & (HRING - 1)], a.H + i);
            kfill = ktop > kfill ? ktop : kfill;
            asm volatile("cp.async.commit_group;");
        }
    }
    asm volatile("cp.async.wait_group 0;");
    __syncthreads();
    // write back: block / superblock counts, counters, generator state
    for (int64_t i = t; i < nb; i += XT) a.blk_cnt[i] = x.CNT[i];
    for (int64_t sb = t; sb < ns; sb += XT) a.sup_cnt[sb] = x.SUPP[sb + 1] - x.SUPP[sb];
    hits = __reduce_add_sync(0xffffffffu, (unsigned)hits);
    misses = __reduce_add_sync(0xffffffffu, (unsigned)misses);
    byp = __reduce_add_sync(0xffffffffu, (unsigned)byp);
    if (lane == 0) {
        atomicAdd((unsigned long long*)&a.meta->hits, (unsigned long long)hits);
        atomicAdd((unsigned long long*)&a.meta->misses, (unsigned long long)misses);
        atomicAdd((unsigned long long*)&a.meta->bypasses, (unsigned long long)byp);
        atomicAdd((unsigned long long*)&a.meta->evictions, (unsigned long long)misses);
    }
    if (t == 0) {
        // generator after kpos halves
        CacheMeta* m = a.meta;
        const uint32_t has = (uint32_t)m->rng[4];
        int64_t kk = kpos;
        if (kk > 0) {
            int64_t k2 = has ? kk - 1 : kk;  // halves taken from next64 outputs
            if (k2 > 0) {
                const uint64_t outs = (uint64_t)((k2 + 1) / 2);
                const u128 inc = {m->rng[3], m->rng[2]};
                const u128 sn = pcg_advance(u128{m->rng[1], m->rng[0]}, inc, outs);
                m->rng[0] = sn.hi;
                m->rng[1] = sn.lo;
                m->rng[4] = (k2 & 1) ? 1u : 0u;
                m->rng[5] = (uint32_t)(pcg_output(sn) >> 32);
            } else {
                m->rng[4] = 0u;  // only the buffered half was used
            }
        }
        m->safe_count = nsafe;
        a.svc->n_log = nlog;
        a.svc->xp_done = 1;
        a.svc->xp_stats[0] = st_rounds;
        a.svc->xp_stats[1] = st_rej;
        a.svc->xp_stats[2] = st_chg;
        a.svc->xp_stats[3] = st_conv;
        for (int i = 0; i < 12; i++) a.svc->xp_prof[i] = prof[i];
    }
}

// the batch's candidates leave cand_of_slot as they found it (-1)
__global__ void k_xp_reset(const ServeCounters* svc, const int32_t* __restrict__ cand_slot,
                           int32_t* cand_of_slot) {
    int64_t n = svc->n_cand < GIDS_XP_CAND_CAP ? svc->n_cand : GIDS_XP_CAND_CAP;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        cand_of_slot[cand_slot[i]] = -1;
}

}  // namespace

int gids_launch_xp_reset(gids_handle* h, cudaStream_t st) {
    if (!h->xp_enabled) return GIDS_OK;  // (nothing set cand_of_slot)
    k_xp_reset<<<64, 256, 0, st>>>(h->svc, h->cand_slot, h->cand_of_slot);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

// shared memory of k_exact_par for a cache of L lines
size_t gids_xp_smem_bytes(int64_t L) {
    const int64_t nb = (L + 1023) / 1024, ns = (nb + 31) / 32;
    return sizeof(uint32_t) * (size_t)(2 * (XP_MAX_CHG + 2) + 2 * nb + XP_MAX_CHG + CUMN + 2 +
                                       2 * HSZ + CHBW + 2 * RING + HRING + nb + nb + ns + 1 +
                                       (GIDS_XP_CAND_CAP + 31) / 32 + 2 * XT + 6 * XP_MAX_CHG +
                                       XW * 8 + 16 + 1) +
           sizeof(unsigned long long) * MOVN;
}

// launched before k_exact_seq; each checks on the device which of them runs
int gids_launch_exact_par(gids_handle* h, int64_t n, cudaStream_t st, const ServeArgs* sa) {
    if (!h->xp_enabled || n == 0) return GIDS_OK;
    const int64_t outs = (h->xp_hcap + 1) / 2;
    k_xp_halves<<<gids_grid(ceil_div(outs, 8), 256, 1 << 20), 256, 0, st>>>(
        h->meta, h->svc, h->L, GIDS_XP_CAND_CAP, h->xp_safe_div, h->xp_halves, h->xp_hcap);
    GIDS_LAUNCH_CHECK(h);
    XpArgs a;
    a.ev = h->ev;
    a.xcls = h->xcls;
    a.n = n;
    a.L = h->L;
    a.meta = h->meta;
    a.svc = h->svc;
    a.safe_bits = h->safe_bits;
    a.blk_cnt = h->blk_cnt;
    a.sup_cnt = h->sup_cnt;
    a.cand_of_slot = h->cand_of_slot;
    a.cand_cap = GIDS_XP_CAND_CAP;
    a.safe_div = h->xp_safe_div;
    a.H = h->xp_halves;
    a.hcap = h->xp_hcap;
    a.kind = h->kind;
    a.line = h->line;
    a.log_line = h->log_line;
    a.log_pos = h->log_pos;
    a.sa = sa;
    const size_t smem = gids_xp_smem_bytes(h->L);
    static size_t attr_smem = 0;  // (the attribute is per function: set when it grows)
    if (smem > attr_smem) {
        GIDS_CUDA_TRY(cudaFuncSetAttribute(k_exact_par, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
        attr_smem = smem;
    }
    k_exact_par<<<1, XT, smem, st>>>(a);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}
