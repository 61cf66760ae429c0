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
//      halves); a rejection ends the round after that access
//   C  every evicting access selects the r-th safe line of the round-START set
//      (interpolated block search over shared-memory prefix counts, then the
//      32 words of the 1024-line block from the L2-resident bitmap)
//   D  one warp finalises the round's set changes in order: each MU answer is
//      moved past the earlier changes (removal at or below -> next safe line,
//      addition below -> previous safe line) on a private copy of its block
//   E  every other evicting access applies the finalised changes the same way
//   F  a CAND whose line was taken earlier (this or the previous round; older
//      rounds flag it through cand_of_slot) ends the round before itself and
//      is a miss in the next one
//   G  commit: decisions, insertion log, bitmap and prefix counts
// and is bit-exact with the sequential reference (tests/test_gpu_exact_par.py).
// Not full, too many candidates, or a cache larger than XP_MAX_L lines: the
// sequential warp (k_exact_seq) decides the batch instead.
#include "gids_internal.cuh"

namespace {

constexpr int XT = 256;           // threads = accesses per round
constexpr int XW = XT / 32;
constexpr int XP_MAX_CHG = 32;    // set changes per round (the round ends before the 33rd)
constexpr int RING = 4096;        // staged accesses (ev, class)
constexpr int HRING = 4096;       // staged draw halves
constexpr int RING_LAG = 12;      // commit groups allowed in flight when a round reads
constexpr int32_t NEG = -(1 << 29);
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

__device__ __forceinline__ bool xp_runs(const CacheMeta* meta, const ServeCounters* svc,
                                        int64_t L, int64_t cand_cap) {
    return svc->n_miss0 != 0 && meta->fill >= L && svc->n_cand <= cand_cap;
}

// the batch's eviction half stream, 8 next64 outputs per thread
__global__ void k_xp_halves(const CacheMeta* meta, const ServeCounters* svc, int64_t L,
                            int64_t cand_cap, uint32_t* H, int64_t hcap) {
    if (!xp_runs(meta, svc, L, cand_cap)) return;
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
    const uint32_t* H;
    int64_t hcap;
    int8_t* kind;
    int32_t* line;
    int32_t* log_line;
    int32_t* log_pos;
};

// shared-memory view of the round state
struct Xs {
    uint32_t* CNT;    // [nb] safe lines per block
    uint32_t* BLKP;   // [nb] exclusive prefix within the 32-block superblock
    uint32_t* SUPP;   // [ns+1] exclusive prefix over superblocks
    uint32_t* CONV;   // [cand_cap/32] candidates whose line was taken
    uint32_t* ROWS;   // [XT*32] private block copies (16-B chunks swizzled)
    int32_t* ROWBLK;  // [XT] block held by each row (-1 none)
    uint32_t* REV;    // [RING]
    uint32_t* RCL;    // [RING]
    uint32_t* RH;     // [HRING]
    int32_t* ANS;     // [XT] final line per evicting access of the round, -1
    int32_t* PANS;    // [XT] same, previous round
    int32_t* CSLOT;   // [XP_MAX_CHG]
    int32_t* CTYPE;   // [XP_MAX_CHG] +1 add, -1 remove
    int32_t* CLANE;   // [XP_MAX_CHG]
    int32_t* W;       // [XW * 8] warp partials
    int32_t* MISC;    // [16]
    int64_t nb, ns, L;
    const uint32_t* gbits;
};

__device__ __forceinline__ uint32_t& rw(const Xs& x, int row, int w) {
    return x.ROWS[row * 32 + ((((w >> 2) ^ (row & 7)) << 2) | (w & 3))];
}

// block g of the round-start bitmap into `row`, then the changes [0, lim) that
// fall into it (the finalised prefix of this round's change list)
__device__ void load_row(const Xs& x, int row, int64_t g, int lim) {
    const uint4* src = reinterpret_cast<const uint4*>(x.gbits + g * 32);
#pragma unroll
    for (int q = 0; q < 8; q++) {
        const uint4 v = __ldcg(src + q);
        uint32_t* d = &x.ROWS[row * 32 + ((q ^ (row & 7)) << 2)];
        d[0] = v.x;
        d[1] = v.y;
        d[2] = v.z;
        d[3] = v.w;
    }
    for (int i = 0; i < lim; i++) {
        const int32_t u = x.CSLOT[i];
        if ((u >> 10) == g) {
            uint32_t& wd = rw(x, row, (u >> 5) & 31);
            if (x.CTYPE[i] > 0) wd |= 1u << (u & 31);
            else wd &= ~(1u << (u & 31));
        }
    }
    x.ROWBLK[row] = (int32_t)g;
}

// smallest safe line > cur in the current set (L if none)
__device__ int32_t next_safe(const Xs& x, int row, int32_t cur, int lim) {
    int64_t g = cur >> 10;
    int b = (cur & 1023) + 1;
    for (;;) {
        if (b < 1024) {
            if (x.ROWBLK[row] != g) load_row(x, row, g, lim);
            for (int w = b >> 5; w < 32; w++) {
                uint32_t m = rw(x, row, w);
                if (w == (b >> 5)) m &= 0xffffffffu << (b & 31);
                if (m) return (int32_t)(g * 1024 + w * 32 + __ffs(m) - 1);
            }
        }
        g++;
        b = 0;
        if (g >= x.nb) return (int32_t)x.L;
    }
}

// largest safe line < cur in the current set (-1 if none); cur may be L
__device__ int32_t prev_safe(const Xs& x, int row, int32_t cur, int lim) {
    int64_t g = (cur - 1) >> 10;
    if (cur <= 0) return -1;
    int b = (cur - 1) & 1023;  // last candidate bit in block g
    if ((int64_t)cur >= x.L) {
        g = x.nb - 1;
        b = 1023;
    }
    for (;;) {
        if (x.ROWBLK[row] != g) load_row(x, row, g, lim);
        for (int w = b >> 5; w >= 0; w--) {
            uint32_t m = rw(x, row, w);
            if (w == (b >> 5) && (b & 31) != 31) m &= (2u << (b & 31)) - 1u;
            if (m) return (int32_t)(g * 1024 + w * 32 + 31 - __clz(m));
        }
        if (g == 0) return -1;
        g--;
        b = 1023;
    }
}

// move an answer past one set change (u, ty) made before its access:
// removal at or below -> next safe line; addition below -> previous safe line
// (the new set holds u).  cur == L with excess ex: the rank is ex past the end.
__device__ __forceinline__ void apply_change(const Xs& x, int row, int32_t u, int ty,
                                             int32_t& cur, int32_t& ex, int lim) {
    if (x.ROWBLK[row] == (u >> 10)) {
        uint32_t& wd = rw(x, row, (u >> 5) & 31);
        if (ty > 0) wd |= 1u << (u & 31);
        else wd &= ~(1u << (u & 31));
    }
    if ((int64_t)cur >= x.L) {
        if (ty < 0) {
            ex++;
        } else if (ex > 0) {
            ex--;
        } else {
            cur = prev_safe(x, row, (int32_t)x.L, lim);
        }
        return;
    }
    if (ty < 0) {
        if (u <= cur) {
            cur = next_safe(x, row, cur, lim);
            if ((int64_t)cur >= x.L) ex = 0;
        }
    } else if (u < cur) {
        cur = prev_safe(x, row, cur, lim);
    }
}

__device__ __forceinline__ uint32_t pb(const Xs& x, int64_t g) { return x.SUPP[g >> 5] + x.BLKP[g]; }

// block holding the r-th safe line of the round-start set (r < total)
__device__ int64_t locate(const Xs& x, uint32_t r, uint32_t total) {
    const int64_t nb = x.nb;
    const uint32_t avg = total / (uint32_t)nb > 0 ? total / (uint32_t)nb : 1u;
    int64_t g = (int64_t)(((uint64_t)r * (uint64_t)nb) / total);
    if (g >= nb) g = nb - 1;
    for (int it = 0; it < 6; it++) {
        const uint32_t base = pb(x, g), c = x.CNT[g];
        if (r < base) {
            int64_t st = (base - r) / avg + 1;
            g = g - st < 0 ? 0 : g - st;
        } else if (r >= base + c) {
            int64_t st = (r - base - c) / avg + 1;
            g = g + st >= nb ? nb - 1 : g + st;
        } else {
            return g;
        }
    }
    int64_t lo = 0, hi = nb - 1;  // largest g with pb(g) <= r
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (pb(x, mid) <= r) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ uint32_t get_half(const Xs& x, const XpArgs& a, int64_t k,
                                             int64_t kfill) {
    if (k < kfill && k >= kfill - HRING) return x.RH[k % HRING];
    if (k < a.hcap) return __ldcg(a.H + k);
    return half_direct(a.meta, k);
}

// (d, c): x -> max(x + d, c); compose(first, then)
__device__ __forceinline__ void sat_compose(int32_t d1, int32_t c1, int32_t& d2, int32_t& c2) {
    const int32_t c = max(c1 + d2, c2);
    d2 = d1 + d2;
    c2 = c;
}

__global__ void __launch_bounds__(XT, 1) k_exact_par(XpArgs a) {
    if (!xp_runs(a.meta, a.svc, a.L, a.cand_cap)) return;
    extern __shared__ __align__(16) uint32_t smem[];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const unsigned below = (1u << lane) - 1u;
    Xs x;
    x.L = a.L;
    x.nb = (a.L + 1023) >> 10;
    x.ns = (x.nb + 31) >> 5;
    x.gbits = a.safe_bits;
    {
        uint32_t* p = smem;
        x.ROWS = p;
        p += XT * 32;
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
        x.ROWBLK = reinterpret_cast<int32_t*>(p);
        p += XT;
        x.ANS = reinterpret_cast<int32_t*>(p);
        p += XT;
        x.PANS = reinterpret_cast<int32_t*>(p);
        p += XT;
        x.CSLOT = reinterpret_cast<int32_t*>(p);
        p += XP_MAX_CHG;
        x.CTYPE = reinterpret_cast<int32_t*>(p);
        p += XP_MAX_CHG;
        x.CLANE = reinterpret_cast<int32_t*>(p);
        p += XP_MAX_CHG;
        x.W = reinterpret_cast<int32_t*>(p);
        p += XW * 8;
        x.MISC = reinterpret_cast<int32_t*>(p);
    }
    const int64_t n = a.n, nb = x.nb, ns = x.ns;
    // prefix tables from the block counts
    for (int64_t i = t; i < nb; i += XT) x.CNT[i] = a.blk_cnt[i];
    for (int64_t i = t; i < (a.cand_cap + 31) / 32; i += XT) x.CONV[i] = 0u;
    x.ROWBLK[t] = -1;
    x.PANS[t] = -1;
    __syncthreads();
    for (int64_t s = t; s < ns; s += XT) {
        uint32_t run = 0;
        for (int64_t b = s * 32; b < nb && b < s * 32 + 32; b++) {
            x.BLKP[b] = run;
            run += x.CNT[b];
        }
        x.SUPP[s + 1] = run;  // per-superblock totals, prefixed next
    }
    __syncthreads();
    if (t == 0) {
        uint32_t run = 0;
        x.SUPP[0] = 0;
        for (int64_t s = 0; s < ns; s++) {
            run += x.SUPP[s + 1];
            x.SUPP[s + 1] = run;
        }
    }
    // stage the first accesses and halves
    int64_t efill = n < RING ? n : RING;
    int64_t kfill = a.hcap < HRING ? a.hcap : HRING;
    for (int64_t i = t; i < efill; i += XT) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&x.REV[i % RING])),
                     "l"(a.ev + i));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&x.RCL[i % RING])),
                     "l"(a.xcls + i));
    }
    for (int64_t i = t; i < kfill; i += XT)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&x.RH[i % HRING])),
                     "l"(a.H + i));
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 0;");
    __syncthreads();

    int64_t pos = 0, kpos = 0, nlog = 0;
    int32_t nsafe = (int32_t)a.meta->safe_count;
    int prevE = 0;
    int32_t pend_cidx = -1;  // cand_of_slot of this thread's last committed eviction
    int64_t hits = 0, misses = 0, byp = 0;

    while (pos < n) {
        asm volatile("cp.async.wait_group %0;" ::"n"(RING_LAG));
        __syncthreads();
        // ---------------- A: classify, saturating safe-count prefix, draw prefix
        const int64_t p = pos + t;
        const bool valid = p < n;
        const uint32_t e = valid ? x.REV[p % RING] : 0u;
        const uint32_t xc = valid ? x.RCL[p % RING] : 0u;
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
        // inclusive warp scan of the saturating map
        int32_t di = d, ci = c;
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
        if (t == 0) {
            x.MISC[0] = XT;  // end of the round before conversions (min)
            x.MISC[1] = XT;  // first candidate that lost its line (min)
            x.MISC[3] = 0;   // set changes at accesses before that end
        }
        __syncthreads();
        int32_t dp = 0, cp = NEG;  // earlier warps, composed
        for (int w = 0; w < wid; w++) sat_compose(x.W[w * 8 + 0], x.W[w * 8 + 1], dp, cp);
        sat_compose(dp, cp, de, ce);  // exclusive prefix at this thread
        const int32_t ni = max(nsafe + de, ce);   // safe lines seen by this access
        const bool sel = miss && ni >= 1;         // evicts (else bypass)
        const bool dr = miss && ni >= 2;          // consumes a draw (integers(1) draws nothing)
        const bool chg = valid && (cls == C_ADD || (cls == C_MU && sel));
        const unsigned bdr = __ballot_sync(0xffffffffu, dr);
        const unsigned bsel = __ballot_sync(0xffffffffu, sel);
        const unsigned bchg = __ballot_sync(0xffffffffu, chg);
        if (lane == 0) {
            x.W[wid * 8 + 2] = __popc(bdr);
            x.W[wid * 8 + 3] = __popc(bsel);
            x.W[wid * 8 + 4] = __popc(bchg);
        }
        __syncthreads();
        int32_t pdr = __popc(bdr & below), psel = __popc(bsel & below), pchg = __popc(bchg & below);
        for (int w = 0; w < wid; w++) {
            pdr += x.W[w * 8 + 2];
            psel += x.W[w * 8 + 3];
            pchg += x.W[w * 8 + 4];
        }
        // ---------------- B: draws
        uint32_t r = 0;
        int extra = 0;
        if (dr) {
            const int64_t k = kpos + pdr;
            uint64_t m = (uint64_t)get_half(x, a, k, kfill) * (uint32_t)ni;
            uint32_t left = (uint32_t)m;
            if (left < (uint32_t)ni) {
                const uint32_t thr = (0u - (uint32_t)ni) % (uint32_t)ni;
                while (left < thr) {  // Lemire rejection: the round ends here
                    extra++;
                    m = (uint64_t)get_half(x, a, k + extra, kfill) * (uint32_t)ni;
                    left = (uint32_t)m;
                }
            }
            r = (uint32_t)(m >> 32);
            if (extra) atomicMin(&x.MISC[0], t + 1);
        }
        if (chg && pchg == XP_MAX_CHG) atomicMin(&x.MISC[0], t);  // change list full
        // ---------------- C: select in the round-start set
        const uint32_t total = x.SUPP[ns];
        int32_t cur = -1, ex = 0;
        if (sel) {
            if (r < total) {
                const int64_t g = locate(x, r, total);
                const uint32_t rr = r - pb(x, g);
                const uint4* src = reinterpret_cast<const uint4*>(a.safe_bits + g * 32);
                uint32_t wv[32];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const uint4 v = __ldcg(src + q);
                    wv[4 * q] = v.x;
                    wv[4 * q + 1] = v.y;
                    wv[4 * q + 2] = v.z;
                    wv[4 * q + 3] = v.w;
                    uint32_t* dst = &x.ROWS[t * 32 + ((q ^ (t & 7)) << 2)];
                    dst[0] = v.x;
                    dst[1] = v.y;
                    dst[2] = v.z;
                    dst[3] = v.w;
                }
                x.ROWBLK[t] = (int32_t)g;
                uint32_t acc = 0, accb = 0, wsel = 0;
                int found = 0;
                bool got = false;
#pragma unroll
                for (int q = 0; q < 32; q++) {
                    const uint32_t cq = __popc(wv[q]);
                    const bool h = !got && acc + cq > rr;
                    if (h) {
                        found = q;
                        accb = acc;
                        wsel = wv[q];
                        got = true;
                    }
                    acc += cq;
                }
                cur = (int32_t)(g * 1024 + found * 32 + __fns(wsel, 0, (int)(rr - accb) + 1));
            } else {
                cur = (int32_t)a.L;
                ex = (int32_t)(r - total);
            }
        }
        __syncthreads();
        const int Epre0 = x.MISC[0];
        const int Epre = (int)((n - pos) < Epre0 ? (n - pos) : Epre0);
        // ---------------- D: the round's set changes, finalised in order
        if (chg && t < Epre) {
            x.CSLOT[pchg] = cls == C_ADD ? s : cur;
            x.CTYPE[pchg] = cls == C_ADD ? 1 : -1;
            x.CLANE[pchg] = t;
            if (cls == C_MU) x.ANS[pchg] = ex;  // (scratch: the MU's excess)
            atomicMax(&x.MISC[3], pchg + 1);
        }
        __syncthreads();
        const int nchg = x.MISC[3];
        if (wid == 0) {
            int32_t ucur = -1, uex = 0, uty = 0, urow = 0;
            if (lane < nchg) {
                ucur = x.CSLOT[lane];
                uty = x.CTYPE[lane];
                urow = x.CLANE[lane];
                uex = uty < 0 ? x.ANS[lane] : 0;
            }
            for (int i = 0; i < nchg; i++) {
                const int32_t ui = __shfl_sync(0xffffffffu, ucur, i);
                const int32_t ti = __shfl_sync(0xffffffffu, uty, i);
                if (lane == i) x.CSLOT[i] = ucur;  // final
                __syncwarp();
                if (lane > i && lane < nchg && uty < 0)
                    apply_change(x, urow, ui, ti, ucur, uex, i + 1);
                __syncwarp();
            }
        }
        __syncthreads();
        // ---------------- E: every other eviction moves past the final changes
        if (sel && t < Epre) {
            if (chg) {
                cur = x.CSLOT[pchg];
            } else {
                for (int i = 0; i < nchg && x.CLANE[i] < t; i++)
                    apply_change(x, t, x.CSLOT[i], x.CTYPE[i], cur, ex, i + 1);
            }
        }
        x.ANS[t] = (sel && t < Epre) ? cur : -1;
        __syncthreads();
        // ---------------- F: a candidate whose line an earlier eviction took
        if (valid && t < Epre && cls == C_CAND && !conv) {
            bool taken = false;
            for (int j = 0; j < t && !taken; j++) taken = x.ANS[j] == s;
            for (int j = 0; j < prevE && !taken; j++) taken = x.PANS[j] == s;
            if (taken) atomicMin(&x.MISC[1], t);
        }
        __syncthreads();
        const int E = Epre < x.MISC[1] ? Epre : x.MISC[1];
        if (t == E && E < Epre) x.CONV[cidx >> 5] |= 1u << (cidx & 31);  // (only this lane writes)
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
                const int64_t li = nlog + psel;
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
        // the set changes of the committed accesses: bitmap and prefix tables
        int ncommit = 0;
        for (int i = 0; i < nchg; i++) {
            if (x.CLANE[i] >= E) break;
            ncommit++;
        }
        for (int i = 0; i < ncommit; i++) {
            const int32_t u = x.CSLOT[i];
            const int ty = x.CTYPE[i];
            const int64_t b = u >> 10, sb = b >> 5;
            if (t == 0) {
                if (ty > 0) atomicOr(&a.safe_bits[u >> 5], 1u << (u & 31));
                else atomicAnd(&a.safe_bits[u >> 5], ~(1u << (u & 31)));
                x.CNT[b] += (uint32_t)ty;
            }
            if (t < 32 && t > (int)(b & 31) && (sb << 5) + t < nb) x.BLKP[(sb << 5) + t] += (uint32_t)ty;
            for (int64_t q = t; q <= ns; q += XT)
                if (q > sb) x.SUPP[q] += (uint32_t)ty;
        }
        // state after the last committed access
        if (t == E - 1) {
            x.MISC[4] = max(ni + d, c);           // safe count after it
            x.MISC[5] = pdr + (dr ? 1 + extra : 0);  // halves consumed through it
            x.MISC[6] = psel + (sel ? 1 : 0);       // log entries through it
        }
        __syncthreads();
        if (E > 0) {
            nsafe = x.MISC[4];
            kpos += x.MISC[5];
            nlog += x.MISC[6];
        }
        x.PANS[t] = t < E ? x.ANS[t] : -1;
        x.ROWBLK[t] = -1;  // (the bitmap moved on; private copies are stale)
        prevE = E;
        pos += E;
        // refill the rings past the consumed prefix
        {
            const int64_t etop = (pos + RING) < n ? pos + RING : n;
            for (int64_t i = efill + t; i < etop; i += XT) {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                                 (uint32_t)__cvta_generic_to_shared(&x.REV[i % RING])),
                             "l"(a.ev + i));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                                 (uint32_t)__cvta_generic_to_shared(&x.RCL[i % RING])),
                             "l"(a.xcls + i));
            }
            efill = etop;
            const int64_t ktop = (kpos + HRING) < a.hcap ? kpos + HRING : a.hcap;
            for (int64_t i = kfill + t; i < ktop; i += XT)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                                 (uint32_t)__cvta_generic_to_shared(&x.RH[i % HRING])),
                             "l"(a.H + i));
            kfill = ktop > kfill ? ktop : kfill;
            asm volatile("cp.async.commit_group;");
        }
    }
    asm volatile("cp.async.wait_group 0;");
    if (pend_cidx >= 0) atomicOr(&x.CONV[pend_cidx >> 5], 1u << (pend_cidx & 31));
    __syncthreads();
    // write back: block / superblock counts, counters, generator state
    for (int64_t i = t; i < nb; i += XT) a.blk_cnt[i] = x.CNT[i];
    for (int64_t sb = t; sb < ns; sb += XT) a.sup_cnt[sb] = x.SUPP[sb + 1] - x.SUPP[sb];
    // block reduction of the counters
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
    k_xp_reset<<<64, 256, 0, st>>>(h->svc, h->cand_slot, h->cand_of_slot);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

// shared memory of k_exact_par for a cache of L lines
size_t gids_xp_smem_bytes(int64_t L) {
    const int64_t nb = (L + 1023) / 1024, ns = (nb + 31) / 32;
    return sizeof(uint32_t) * (size_t)(XT * 32 + 2 * RING + HRING + 2 * nb + ns + 1 +
                                       (GIDS_XP_CAND_CAP + 31) / 32 + 3 * XT + 3 * XP_MAX_CHG +
                                       XW * 8 + 16);
}

// launched before k_exact_seq; each checks on the device which of them runs
int gids_launch_exact_par(gids_handle* h, int64_t n, cudaStream_t st) {
    if (!h->xp_enabled || n == 0) return GIDS_OK;
    const int64_t outs = (h->xp_hcap + 1) / 2;
    k_xp_halves<<<gids_grid(ceil_div(outs, 8), 256, 1 << 20), 256, 0, st>>>(
        h->meta, h->svc, h->L, GIDS_XP_CAND_CAP, h->xp_halves, h->xp_hcap);
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
    a.H = h->xp_halves;
    a.hcap = h->xp_hcap;
    a.kind = h->kind;
    a.line = h->line;
    a.log_line = h->log_line;
    a.log_pos = h->log_pos;
    const size_t smem = gids_xp_smem_bytes(h->L);
    GIDS_CUDA_TRY(cudaFuncSetAttribute(k_exact_par, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    k_exact_par<<<1, XT, smem, st>>>(a);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}
