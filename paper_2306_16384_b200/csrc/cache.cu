// cache.cu -- K3/K4: lookahead-window counters and the HBM software cache.
//
// State (all HBM):
//   slot_of[N]   node -> line (-1)          (CacheState.resident, cache.py:106)
//   line_node[L] line -> node (-1 empty)    (CacheState.slot_node, cache.py:107)
//   safe_bits    SafeToEvict bitmap over lines; with 32 ways, word s IS set s
//   blk_cnt / sup_cnt  safe lines per 1024 / 32768 lines (exact-policy select)
//   reuse[N]     predicted-reuse counters   (CacheState.reuse_counter)
//   future[N]    how many lookahead-window lists contain the node; replaces
//                the sorted-concat + searchsorted of window_update
//                (cache.py:201-206) by +-1 on push/pop (lists are unique).
//
// Serving a batch:
//   k_window_consume  window_update (cache.py:190-218) fused with the
//                     per-access reuse consumption (cache.py:121-131): both
//                     are order-independent per node, so fully parallel.
//   exact policy      k_exact_seq: the reference CacheState.access sequence
//                     (cache.py:144-180) in ascending node order on ONE warp,
//                     tables in shared memory, uniform eviction draws from the
//                     numpy PCG64 stream; only the order-dependent decisions
//                     are sequential, the line/node bookkeeping is done after
//                     in parallel (k_post_*).
//   set-associative   32-way sets, one warp per set, lanes = ways; the same
//                     contract per set with a counter-based eviction draw.

#include <chrono>

#include "gids_internal.cuh"

namespace {

constexpr int BLOCK = 256;

__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

// ---------------------------------------------------------------- window
__global__ void k_window(const int64_t* __restrict__ nodes, int64_t n, uint8_t* future,
                         int delta) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        future[nodes[i]] += (uint8_t)delta;
}

// a window pop then push in one pass (window.py: the served batch leaves,
// the batch W ahead joins): byte counts updated with 32-bit atomics on their
// lane -- a node may be in both lists, and a count never borrows (>= 1 when
// popped) nor carries (<= 254 when pushed)
__global__ void k_window_shift(const int64_t* __restrict__ pop, int64_t n_pop,
                               const int64_t* __restrict__ push, int64_t n_push, uint8_t* future,
                               const ServeArgs* sa) {
    if (sa) {
        pop = sa->pop;
        n_pop = sa->n_pop;
        push = sa->push;
        n_push = sa->n_push;
    }
    uint32_t* words = reinterpret_cast<uint32_t*>(future);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pop + n_push;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n_pop) {
            const int64_t x = pop[i];
            atomicSub(&words[x >> 2], 1u << ((x & 3) * 8));
        } else {
            const int64_t x = push[i - n_pop];
            atomicAdd(&words[x >> 2], 1u << ((x & 3) * 8));
        }
    }
}

// run-ahead contribution: unpinned and not resident (dataloader.py:188-192)
__global__ void k_contribution(const int32_t* __restrict__ uniq, SampleCounters* sc,
                               const int32_t* __restrict__ pinned_off,
                               const int32_t* __restrict__ slot_of) {
    int64_t n = sc->n_unique, c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t x = uniq[i];
        c += (pinned_off[x] < 0 && slot_of[x] < 0) ? 1 : 0;
    }
    c = warp_sum64(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd((unsigned long long*)&sc->contribution,
                                                (unsigned long long)c);
}

// the same count for an exported batch, at the moment it joins the run-ahead
// queue: n read once per block through a device-visible pointer (pinned host
// is fine); the last block to finish stores the total into the pinned result
// and leaves the scratch zeroed -- one launch, no memset or copy around it
__global__ void k_contribution64(const int64_t* __restrict__ uniq, const int64_t* n_ptr,
                                 const int32_t* __restrict__ pinned_off,
                                 const int32_t* __restrict__ slot_of,
                                 unsigned long long* scratch, int64_t* out_host) {
    __shared__ int64_t s_n;
    if (threadIdx.x == 0) s_n = *n_ptr;
    __syncthreads();
    const int64_t n = s_n;
    int64_t c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = uniq[i];
        c += (pinned_off[x] < 0 && slot_of[x] < 0) ? 1 : 0;
    }
    c = warp_sum64(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&scratch[0], (unsigned long long)c);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&scratch[1], 1ull) == gridDim.x - 1) {  // every block's sum is in
            __threadfence();
            *out_host = (int64_t)atomicExch(&scratch[0], 0ull);
            scratch[1] = 0;
        }
    }
}

// window_update + reuse consumption; ev[p] = (line_at_start+1)<<1 | (count_after>0)
// mode bit 1: window_update (raise by the lookahead counts, Safe->InUse flip);
// mode bit 2: the accesses' reuse consumption (writes ev).  The serving path
// runs both fused (every node of a batch is accessed right after the update);
// the standalone CacheState API runs them separately.  counts (optional)
// receives each node's lookahead count.
__global__ void k_window_consume(const int64_t* __restrict__ uniq, int64_t n,
                                 const uint8_t* __restrict__ future, uint32_t* reuse,
                                 const int32_t* __restrict__ slot_of, uint32_t* safe_bits,
                                 uint32_t* blk_cnt, uint32_t* sup_cnt, int exact,
                                 CacheMeta* meta, uint32_t* ev, int mode = 3,
                                 int32_t* counts = nullptr, int64_t* nmiss0 = nullptr,
                                 uint32_t* xcls = nullptr, int32_t* cand_of_slot = nullptr,
                                 int32_t* cand_slot = nullptr, int64_t* n_cand = nullptr,
                                 int64_t* bad_order = nullptr, int64_t* zero2 = nullptr,
                                 int32_t* ins = nullptr, const ServeArgs* sa = nullptr) {
    if (sa) {
        uniq = sa->uniq;
        n = sa->n;
    }
    int64_t inc = 0, dec = 0, unsafe = 0, miss0 = 0;
    if (zero2 && blockIdx.x == 0 && threadIdx.x == 0) {  // the batch's work-list counts
        zero2[0] = 0;
        zero2[1] = 0;
    }
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        int32_t x = (int32_t)uniq[p];
        if (ins) ins[p] = -1;  // (no insertion unless a policy logs one)
        // the serving precondition (strictly ascending, hence distinct): the
        // counters below are updated without atomics
        if (bad_order && p > 0 && uniq[p - 1] >= uniq[p]) *bad_order = 1;
        uint32_t c = (mode & 1) ? future[x] : 0u;
        if (counts) counts[p] = (int32_t)c;
        uint32_t old = reuse[x];
        uint32_t now = old + c;
        int32_t s = slot_of[x];
        if (c > 0) {
            inc += c;
            if (old == 0 && s >= 0) {
                uint32_t bit = 1u << (s & 31);
                if (safe_bits[s >> 5] & bit) {  // resident SafeToEvict -> InUse
                    atomicAnd(&safe_bits[s >> 5], ~bit);
                    if (exact) {
                        atomicSub(&blk_cnt[s >> 10], 1u);
                        atomicSub(&sup_cnt[s >> 15], 1u);
                    }
                    unsafe++;
                }
            }
        }
        if ((mode & 2) && now > 0) {
            now--;
            dec++;
        }
        reuse[x] = now;
        if (mode & 2) ev[p] = ((uint32_t)(s + 1) << 1) | (now > 0 ? 1u : 0u);
        miss0 += s < 0;
        if (xcls && (mode & 2)) {
            // the access's class for k_exact_par: by the invariant "resident
            // line InUse iff count > 0", the count before this access's own
            // consumption (old + c) tells a protected line from a safe one
            const bool cb = old + c > 0, ca = now > 0;
            const bool cand = s >= 0 && !cb;
            uint32_t cls = s >= 0 ? (ca ? GIDS_XC_STAY : cb ? GIDS_XC_ADD : GIDS_XC_CAND)
                                  : (ca ? GIDS_XC_MU : GIDS_XC_M0);
            const unsigned am = __activemask();
            const unsigned cm = __ballot_sync(am, cand);
            const int leader = __ffs(am) - 1, lane = threadIdx.x & 31;
            unsigned long long b0 = 0;
            if (lane == leader && cm) b0 = atomicAdd((unsigned long long*)n_cand, (unsigned long long)__popc(cm));
            b0 = __shfl_sync(am, b0, leader);
            if (cand) {
                const int64_t idx = (int64_t)b0 + __popc(cm & ((1u << lane) - 1u));
                if (idx < GIDS_XP_CAND_CAP) {
                    cand_of_slot[s] = (int32_t)idx;
                    cand_slot[idx] = s;
                    cls |= (uint32_t)idx << 3;
                }
            }
            xcls[p] = cls;
        }
    }
    inc = warp_sum64(inc);
    dec = warp_sum64(dec);
    unsafe = warp_sum64(unsafe);
    if (nmiss0) {
        miss0 = warp_sum64(miss0);
        if ((threadIdx.x & 31) == 0 && miss0)
            atomicAdd((unsigned long long*)nmiss0, (unsigned long long)miss0);
    }
    if ((threadIdx.x & 31) == 0) {
        if (inc) atomicAdd((unsigned long long*)&meta->inc, (unsigned long long)inc);
        if (dec) atomicAdd((unsigned long long*)&meta->dec, (unsigned long long)dec);
        if (unsafe) atomicAdd((unsigned long long*)&meta->safe_count, (unsigned long long)(-unsafe));
    }
}

// ----------------------------------------------------------- exact policy
struct ExactTables {
    uint32_t* safe;   // [nw]
    uint32_t* evict;  // [nw]
    uint32_t* blk;    // [nb]
    uint32_t* sup;    // [ns]
};

// lane-cooperative search: index of the entry holding the r-th unit among
// cnt[0..m); r is reduced to the rank inside that entry
__device__ __forceinline__ int64_t warp_find(const uint32_t* cnt, int64_t m, uint32_t& r) {
    const int lane = threadIdx.x & 31;
    for (int64_t base = 0; base < m; base += 32) {
        uint32_t c = base + lane < m ? cnt[base + lane] : 0u;
        uint32_t inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t u = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += u;
        }
        uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
        if (r < total) {
            unsigned m2 = __ballot_sync(0xffffffffu, inc > r);
            int f = __ffs(m2) - 1;
            uint32_t excl = __shfl_sync(0xffffffffu, inc - c, f);
            r -= excl;
            return base + f;
        }
        r -= total;
    }
    return -1;  // unreachable when r < total safe lines
}

// r-th set bit among the 32 safe words starting at word w0 (warp-cooperative)
__device__ __forceinline__ int64_t select_in_words(const ExactTables& t, int64_t nw, int64_t w0,
                                                   uint32_t r) {
    const int lane = threadIdx.x & 31;
    uint32_t word = w0 + lane < nw ? t.safe[w0 + lane] : 0u;
    const uint32_t c = __popc(word);
    // inclusive prefix of the per-word counts (0..32, six bits) from one
    // ballot per bit plane: six independent votes instead of a five-step
    // dependent shuffle scan on the eviction's critical path
    const unsigned le = 0xffffffffu >> (31 - lane);
    uint32_t inc = 0;
#pragma unroll
    for (int k = 0; k < 6; k++)
        inc += (uint32_t)__popc(__ballot_sync(0xffffffffu, (c >> k) & 1u) & le) << k;
    unsigned m = __ballot_sync(0xffffffffu, inc > r);
    int f = __ffs(m) - 1;
    uint32_t excl = __shfl_sync(0xffffffffu, inc - c, f);
    uint32_t wsel = __shfl_sync(0xffffffffu, word, f);
    // the (r - excl)-th set bit of wsel: lane b holds bit b and its rank
    const bool at = ((wsel >> lane) & 1u) && __popc(wsel & ((1u << lane) - 1u)) == (int)(r - excl);
    int bit = __ffs(__ballot_sync(0xffffffffu, at)) - 1;
    return (w0 + f) * 32 + bit;
}

// r-th SafeToEvict line in ascending line order (np.flatnonzero(mask)[r])
__device__ __forceinline__ int64_t select_safe(const ExactTables& t, int64_t nw, int64_t nb,
                                               int64_t ns, uint32_t r) {
    int64_t sb = warp_find(t.sup, ns, r);
    int64_t b0 = sb * 32;
    int64_t bsel = b0 + warp_find(t.blk + b0, (nb - b0) < 32 ? (nb - b0) : 32, r);
    return select_in_words(t, nw, bsel * 32, r);
}

// Caches of up to 128 blocks (131072 lines) also keep the inclusive prefix of
// safe lines over the 1024-line blocks in registers, four blocks per lane,
// updated in place on every change (a predicated add per lane, no
// shuffles), so an eviction finds its block with one ballot instead of two
// warp scans over the count tables.
struct RegPrefix {
    uint32_t p[4];  // safe lines in blocks [0, 4*lane + j]
    __device__ __forceinline__ void add(int64_t b, int d) {
        const int64_t mine = 4 * (int64_t)(threadIdx.x & 31);
#pragma unroll
        for (int j = 0; j < 4; j++) p[j] += (mine + j >= b) ? d : 0;
    }
};

__device__ __forceinline__ void reg_prefix_init(RegPrefix& P, const ExactTables& t, int64_t nb) {
    const int lane = threadIdx.x & 31;
    uint32_t run = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int64_t b = 4 * (int64_t)lane + j;
        run += b < nb ? t.blk[b] : 0u;
        P.p[j] = run;
    }
    uint32_t inc = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t u = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += u;
    }
    const uint32_t before = inc - run;
#pragma unroll
    for (int j = 0; j < 4; j++) P.p[j] += before;
}

__device__ __forceinline__ int64_t select_reg(const ExactTables& t, int64_t nw,
                                              const RegPrefix& P, uint32_t r) {
    const int lane = threadIdx.x & 31;
    const unsigned bal = __ballot_sync(0xffffffffu, P.p[3] > r);
    const int f = __ffs(bal) - 1;
    const uint32_t q0 = __shfl_sync(0xffffffffu, P.p[0], f);
    const uint32_t q1 = __shfl_sync(0xffffffffu, P.p[1], f);
    const uint32_t q2 = __shfl_sync(0xffffffffu, P.p[2], f);
    const uint32_t up = __shfl_sync(0xffffffffu, P.p[3], f > 0 ? f - 1 : 0);
    int j;
    uint32_t excl;
    if (q0 > r) {
        j = 0;
        excl = f > 0 ? up : 0u;
    } else if (q1 > r) {
        j = 1;
        excl = q0;
    } else if (q2 > r) {
        j = 2;
        excl = q1;
    } else {
        j = 3;
        excl = q2;
    }
    (void)lane;
    return select_in_words(t, nw, (int64_t)(4 * f + j) * 32, r - excl);
}

// several lanes may mark different lines of one word / block at once
__device__ __forceinline__ void tab_set_safe_atomic(const ExactTables& t, int64_t s) {
    atomicOr(&t.safe[s >> 5], 1u << (s & 31));
    atomicAdd(&t.blk[s >> 10], 1u);
    atomicAdd(&t.sup[s >> 15], 1u);
}
// ascending list of SafeToEvict lines held one per lane (lane i = i-th
// smallest), valid while there are at most 32 of them: in the steady state of
// a window-protected cache almost every eviction sees 1-3 safe lines, and
// then select(r) is a single shuffle instead of a three-level table walk
constexpr int32_t NO_LINE = 0x7fffffff;
constexpr int EV_AHEAD = 16;  // chunks of the event stream in flight
constexpr int EV_RING = 32;
constexpr int EV_FAST = 4;    // all-hit chunks decided together (fast path)

__device__ __forceinline__ void list_insert(int32_t& sl, int32_t s) {
    const int lane = threadIdx.x & 31;
    const int at = __popc(__ballot_sync(0xffffffffu, sl < s));
    const int32_t up = __shfl_up_sync(0xffffffffu, sl, 1);
    sl = lane < at ? sl : (lane == at ? s : up);
}
__device__ __forceinline__ void list_remove(int32_t& sl, int r) {
    const int lane = threadIdx.x & 31;
    const int32_t down = __shfl_down_sync(0xffffffffu, sl, 1);
    sl = lane < r ? sl : (lane == 31 ? NO_LINE : down);
}

// `added` lanes just made the lines in `val` SafeToEvict: count them, keep
// the short sorted list (while it holds <= 32 lines) and the register prefix
// (a few lines update the prefix in place; more mark it stale, and it is
// rebuilt from the block counts when an eviction next needs it)
__device__ __forceinline__ void note_added(unsigned added, int32_t val, int64_t& safe_count,
                                           bool& list_ok, int32_t& sl, bool reg, RegPrefix& P,
                                           bool& stale) {
    const int na = __popc(added);
    safe_count += na;
    if (list_ok && safe_count > 32) list_ok = false;
    const bool upd = reg && !stale && na <= 2;
    if (reg && !upd && na) stale = true;
    if (!list_ok && !upd) return;
    while (added) {
        const int l = __ffs(added) - 1;
        added &= added - 1;
        const int32_t v = __shfl_sync(0xffffffffu, val, l);
        if (list_ok) list_insert(sl, v);
        if (upd) P.add(v >> 10, 1);
    }
}

// rebuild the list from the tables (<= 32 safe lines known to exist)
__device__ __forceinline__ int32_t list_rebuild(const ExactTables& t, int64_t nw, int64_t nb) {
    const int lane = threadIdx.x & 31;
    int32_t sl = NO_LINE;
    int k = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += 32) {
        uint32_t c = b0 + lane < nb ? t.blk[b0 + lane] : 0u;
        unsigned nz = __ballot_sync(0xffffffffu, c != 0u);
        while (nz) {
            const int64_t b = b0 + __ffs(nz) - 1;
            nz &= nz - 1;
            const int64_t w = b * 32 + lane;
            uint32_t word = w < nw ? t.safe[w] : 0u;
            unsigned has = __ballot_sync(0xffffffffu, word != 0u);
            while (has) {
                const int src = __ffs(has) - 1;
                has &= has - 1;
                uint32_t wv = __shfl_sync(0xffffffffu, word, src);
                while (wv) {
                    const int bit = __ffs(wv) - 1;
                    wv &= wv - 1;
                    if (lane == k) sl = (int32_t)((b * 32 + src) * 32 + bit);
                    k++;
                }
            }
        }
    }
    return sl;
}

// Sequential CacheState.access over the batch, 32 events per step.  Within a
// chunk only two things are order-dependent: a miss that fills or evicts
// (it moves the fill pointer / consumes a draw / may evict a later hit's
// line) and, when the cache is full with no SafeToEvict line, the first hit
// that makes a line safe (it ends a run of bypasses).  Everything between two
// such events is decided in parallel from ballots:
//   fill state (fill < L): hits and the misses that still find empty lines
//     are decided at once, misses taking lines in order
//   active state (safe lines exist): hits up to the next miss are HITs (their
//     InUse->Safe flips commute); that miss then evicts the r-th safe line
//   starved state (full, no safe line): misses up to the first safe-making hit
//     are BYPASSes; that hit restores one safe line.
// A lane's hit status only changes when its line is evicted, so the shared
// tables are read once per chunk.
// A batch whose nodes are all resident when its decisions start has no miss,
// hence no fill, eviction or bypass: every access hits its line and the only
// state change is InUse->Safe for the lines whose reuse count reached zero --
// independent per line.  Decided by the whole GPU instead of the sequential
// warp (k_exact_seq then returns at once); a no-op when n_miss0 > 0.
__global__ void k_exact_allhit(const uint32_t* __restrict__ ev, int64_t n, CacheMeta* meta,
                               uint32_t* safe_bits, uint32_t* blk, uint32_t* sup,
                               const ServeCounters* __restrict__ svc, int8_t* __restrict__ kind,
                               int32_t* __restrict__ line, const ServeArgs* sa = nullptr) {
    if (svc->n_miss0 != 0) return;
    if (sa) n = sa->n;
    int64_t adds = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t e = ev[p];
        const int32_t s = (int32_t)(e >> 1) - 1;
        kind[p] = (int8_t)GIDS_KIND_HIT;
        line[p] = s;
        const uint32_t bit = 1u << (s & 31);
        if (!(e & 1u) && !(safe_bits[s >> 5] & bit)) {
            atomicOr(&safe_bits[s >> 5], bit);
            atomicAdd(&blk[s >> 10], 1u);
            atomicAdd(&sup[s >> 15], 1u);
            adds++;
        }
    }
    adds = warp_sum64(adds);
    if ((threadIdx.x & 31) == 0 && adds)
        atomicAdd((unsigned long long*)&meta->safe_count, (unsigned long long)adds);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        atomicAdd((unsigned long long*)&meta->hits, (unsigned long long)n);
}

// smem_bits: the safe / evicted bitmaps fit in shared memory.  (Specialising
// the kernel on it -- shared-space loads and aggregated ATOMS -- measured 20%
// slower on all-hit batches: the generic accesses stay.)
__global__ void __launch_bounds__(32, 1)
k_exact_seq(const uint32_t* __restrict__ ev, int64_t n, int64_t L, CacheMeta* meta,
            uint32_t* g_safe, uint32_t* g_evict, uint32_t* g_blk, uint32_t* g_sup, int smem_bits,
            int8_t* __restrict__ kind, int32_t* __restrict__ line, int32_t* __restrict__ log_line,
            int32_t* __restrict__ log_pos, ServeCounters* svc, const ServeArgs* sa = nullptr) {
    extern __shared__ uint32_t sm[];
    if (svc->n_miss0 == 0) return;  // all hits: decided by k_exact_allhit
    if (svc->xp_done) return;       // full cache: decided by k_exact_par
    if (sa) n = sa->n;
    const int lane = threadIdx.x;
    const unsigned below = (1u << lane) - 1u;
    const int64_t nw = (L + 31) / 32, nb = (L + 1023) / 1024, ns = (L + 32767) / 32768;
    ExactTables t;
    uint32_t* p = sm;
    t.blk = p;
    p += nb;
    t.sup = p;
    p += ns;
    if (smem_bits) {
        t.safe = p;
        p += nw;
        t.evict = p;
    } else {
        t.safe = g_safe;
        t.evict = g_evict;
    }
    for (int64_t i = lane; i < nb; i += 32) t.blk[i] = g_blk[i];
    for (int64_t i = lane; i < ns; i += 32) t.sup[i] = g_sup[i];
    if (smem_bits)
        for (int64_t i = lane; i < nw; i += 32) {
            t.safe[i] = g_safe[i];
            t.evict[i] = 0u;
        }
    __syncwarp();

    Pcg64 g = {u128{meta->rng[1], meta->rng[0]}, u128{meta->rng[3], meta->rng[2]},
               (uint32_t)meta->rng[4], (uint32_t)meta->rng[5]};
    int64_t fill = meta->fill, safe_count = meta->safe_count;
    int64_t hits = 0, misses = 0, byp = 0, evs = 0, nlog = 0;
    bool list_ok = safe_count <= 32;
    int32_t sl = list_ok ? list_rebuild(t, nw, nb) : NO_LINE;
    const bool reg = nb <= 128;
    RegPrefix P;
    bool stale = true;  // built on the first eviction that needs it

    // the event stream is staged through a shared-memory ring by cp.async,
    // EV_AHEAD chunks ahead, so the sequential loop never waits on HBM
    __shared__ uint32_t ev_ring[EV_RING][32];
    const int64_t nchunks = (n + 31) / 32;
    for (int c = 0; c < EV_AHEAD; c++) {
        const int64_t i = (int64_t)c * 32 + lane;
        if (i < n) {
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&ev_ring[c % EV_RING][lane]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(ev + i));
        }
        asm volatile("cp.async.commit_group;");
    }
    int fast_skip = 0;
    for (int64_t base = 0, chunk = 0; base < n; base += 32, chunk++) {
        // fast path: EV_FAST consecutive full chunks in which every event is a
        // hit change nothing order-dependent (no fill, eviction or bypass; the
        // hits' InUse->Safe flips touch distinct lines and commute), so they
        // are decided together -- the common case of a warm, large cache
        if (fast_skip > 0) {
            fast_skip--;
        } else if (base + EV_FAST * 32 <= n) {
            asm volatile("cp.async.wait_group %0;" ::"n"(EV_AHEAD - EV_FAST));
            __syncwarp();
            uint32_t fe[EV_FAST];
            bool all = true;
#pragma unroll
            for (int k = 0; k < EV_FAST; k++) {
                fe[k] = ev_ring[(chunk + k) % EV_RING][lane];
                const int32_t fs = (int32_t)(fe[k] >> 1) - 1;
                all &= fs >= 0 && !((t.evict[fs >> 5] >> (fs & 31)) & 1u);
            }
            if (__all_sync(0xffffffffu, all)) {
#pragma unroll
                for (int k = 0; k < EV_FAST; k++) {
                    const int32_t fs = (int32_t)(fe[k] >> 1) - 1;
                    const bool fadd = !(fe[k] & 1u) && !((t.safe[fs >> 5] >> (fs & 31)) & 1u);
                    if (fadd) tab_set_safe_atomic(t, fs);
                    {  // note_added without the in-place prefix update: a run of
                       // hits adds many lines, so the prefix goes stale instead
                        unsigned added = __ballot_sync(0xffffffffu, fadd);
                        safe_count += __popc(added);
                        if (added) stale = true;
                        if (list_ok) {
                            if (safe_count > 32) {
                                list_ok = false;
                            } else {
                                while (added) {
                                    const int l = __ffs(added) - 1;
                                    added &= added - 1;
                                    list_insert(sl, __shfl_sync(0xffffffffu, fs, l));
                                }
                            }
                        }
                    }
                    kind[base + k * 32 + lane] = (int8_t)GIDS_KIND_HIT;
                    line[base + k * 32 + lane] = fs;
                    // refill, one commit group per consumed chunk as below
                    const int64_t nc = chunk + k + EV_AHEAD;
                    const int64_t i = nc * 32 + lane;
                    if (nc < nchunks && i < n) {
                        const uint32_t sa =
                            (uint32_t)__cvta_generic_to_shared(&ev_ring[nc % EV_RING][lane]);
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa),
                                     "l"(ev + i));
                    }
                    asm volatile("cp.async.commit_group;");
                }
                hits += 32 * EV_FAST;
                base += 32 * (EV_FAST - 1);
                chunk += EV_FAST - 1;
                continue;
            }
            fast_skip = 8;  // misses around: back off before probing again
        }
        const int cnt = n - base < 32 ? (int)(n - base) : 32;
        const unsigned valid = cnt == 32 ? 0xffffffffu : ((1u << cnt) - 1u);
        asm volatile("cp.async.wait_group %0;" ::"n"(EV_AHEAD - 1));
        __syncwarp();
        const uint32_t my_ev = lane < cnt ? ev_ring[chunk % EV_RING][lane] : 0u;
        {  // refill: chunk + EV_AHEAD goes where chunk - (EV_RING - EV_AHEAD) was
            const int64_t nc = chunk + EV_AHEAD;
            const int64_t i = nc * 32 + lane;
            if (nc < nchunks && i < n) {
                const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&ev_ring[nc % EV_RING][lane]);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(ev + i));
            }
            asm volatile("cp.async.commit_group;");
        }
        const int32_t my_s = (int32_t)(my_ev >> 1) - 1;
        const bool my_inuse = my_ev & 1u;
        const unsigned IU = __ballot_sync(0xffffffffu, my_inuse);
        bool hit = lane < cnt && my_s >= 0 && !((t.evict[my_s >> 5] >> (my_s & 31)) & 1u);
        bool adds = hit && !my_inuse && !((t.safe[my_s >> 5] >> (my_s & 31)) & 1u);
        int my_kind = GIDS_KIND_BYPASS, my_line = -1;
        int pos = 0;
        while (pos < cnt) {
            const unsigned live = valid & ~((1u << pos) - 1u);
            const unsigned H = __ballot_sync(0xffffffffu, hit) & live;
            const unsigned A = __ballot_sync(0xffffffffu, adds) & live;
            const unsigned M = live & ~H;
            unsigned span;
            if (fill < L) {
                // the first min(#misses, L - fill) misses take empty lines in order
                const int nm = __popc(M);
                const int nf = (int64_t)nm < L - fill ? nm : (int)(L - fill);
                const int stop = nf < nm ? __fns(M, 0, nf + 1) : cnt;
                span = live & (stop >= 32 ? 0xffffffffu : ((1u << stop) - 1u));
                const unsigned fm = M & span;
                const bool mine = (span >> lane) & 1u;
                if (mine && hit) {
                    my_kind = GIDS_KIND_HIT;
                    my_line = my_s;
                } else if (mine) {
                    my_kind = GIDS_KIND_MISS;
                    my_line = (int)(fill + __popc(fm & below));
                }
                const bool mk = mine && (hit ? adds : !my_inuse);
                if (mk) tab_set_safe_atomic(t, my_line);
                note_added(__ballot_sync(0xffffffffu, mk), my_line, safe_count, list_ok, sl, reg,
                           P, stale);
                hits += __popc(H & span);
                misses += __popc(fm);
                fill += __popc(fm);
                pos = stop;
            } else if (safe_count > 0 || A) {
                // hits up to the next miss (all of them when starved: then the
                // span ends at the first safe-making hit)
                int stop;
                if (safe_count > 0) {
                    const int m = M ? __ffs(M) - 1 : cnt;
                    stop = m;
                } else {
                    stop = __ffs(A);  // through the first safe-making hit
                }
                span = live & (stop >= 32 ? 0xffffffffu : ((1u << stop) - 1u));
                const bool mine = (span >> lane) & 1u;
                if (mine) {
                    my_kind = hit ? GIDS_KIND_HIT : GIDS_KIND_BYPASS;
                    my_line = hit ? my_s : -1;
                }
                const bool mk = mine && adds;
                if (mk) tab_set_safe_atomic(t, my_s);
                byp += __popc(M & span);
                hits += __popc(H & span);
                note_added(__ballot_sync(0xffffffffu, mk), my_s, safe_count, list_ok, sl, reg, P,
                           stale);
                pos = stop;
                // evictions: the miss at pos and every miss directly after it
                // (no hit span between them) while safe lines remain, without
                // re-deriving the chunk's masks in between; an eviction that
                // takes a later hit's line turns that lane into a miss
                unsigned Mr = M;
                while (safe_count > 0 && pos < cnt && ((Mr >> pos) & 1u)) {
                    const int m = pos;
                    const bool inuse_m = (IU >> m) & 1u;
                    const uint32_t r = pcg_bounded32(g, (uint32_t)safe_count);
                    int32_t v;
                    if (list_ok) {
                        v = __shfl_sync(0xffffffffu, sl, (int)r);
                        if (inuse_m) list_remove(sl, (int)r);
                    } else if (safe_count == L) {
                        v = (int32_t)r;  // every line is SafeToEvict: the r-th is line r
                    } else {
                        __syncwarp();
                        if (reg && stale) {
                            reg_prefix_init(P, t, nb);
                            stale = false;
                        }
                        v = (int32_t)(reg ? select_reg(t, nw, P, r) : select_safe(t, nw, nb, ns, r));
                    }
                    if (lane == 0) {
                        atomicOr(&t.evict[v >> 5], 1u << (v & 31));
                        if (inuse_m) {
                            atomicAnd(&t.safe[v >> 5], ~(1u << (v & 31)));
                            atomicSub(&t.blk[v >> 10], 1u);
                            atomicSub(&t.sup[v >> 15], 1u);
                        }
                    }
                    Mr |= __ballot_sync(0xffffffffu, hit && my_s == v);
                    if (my_s == v) {  // a later hit of this chunk lost its line
                        hit = false;
                        adds = false;
                    }
                    if (lane == m) {
                        my_kind = GIDS_KIND_MISS;
                        my_line = v;
                    }
                    if (inuse_m) {
                        if (reg && !stale) P.add(v >> 10, -1);
                        safe_count--;
                        if (!list_ok && safe_count <= 16) {
                            __syncwarp();
                            sl = list_rebuild(t, nw, nb);
                            list_ok = true;
                        }
                    }
                    misses++;
                    evs++;
                    pos = m + 1;
                }
            } else {
                // starved and no hit restores a line: the rest of the chunk
                span = live;
                const bool mine = (span >> lane) & 1u;
                if (mine) {
                    my_kind = hit ? GIDS_KIND_HIT : GIDS_KIND_BYPASS;
                    my_line = hit ? my_s : -1;
                }
                byp += __popc(M);
                hits += __popc(H);
                pos = cnt;
            }
        }
        __syncwarp();
        if (lane < cnt) {
            kind[base + lane] = (int8_t)my_kind;
            line[base + lane] = my_line;
        }
        const unsigned mm = __ballot_sync(0xffffffffu, lane < cnt && my_kind == GIDS_KIND_MISS);
        if (lane < cnt && my_kind == GIDS_KIND_MISS) {
            const int64_t at = nlog + __popc(mm & below);
            log_line[at] = my_line;
            log_pos[at] = (int32_t)(base + lane);
        }
        nlog += __popc(mm);
    }
    __syncwarp();
    for (int64_t i = lane; i < nb; i += 32) g_blk[i] = t.blk[i];
    for (int64_t i = lane; i < ns; i += 32) g_sup[i] = t.sup[i];
    if (smem_bits)
        for (int64_t i = lane; i < nw; i += 32) g_safe[i] = t.safe[i];
    if (lane == 0) {
        meta->rng[0] = g.state.hi;
        meta->rng[1] = g.state.lo;
        meta->rng[4] = g.has32;
        meta->rng[5] = g.buf32;
        meta->fill = fill;
        meta->safe_count = safe_count;
        meta->hits += hits;
        meta->misses += misses;
        meta->bypasses += byp;
        meta->evictions += evs;
        svc->n_log = nlog;
    }
}

// post-pass A: drop every displaced occupant and every inserted node from
// slot_of, and find each line's final inserter of this batch
__global__ void k_post_a(const int64_t* __restrict__ uniq, const ServeCounters* svc,
                         const int32_t* __restrict__ log_line, const int32_t* __restrict__ log_pos,
                         const int32_t* __restrict__ line_node, int32_t* slot_of, int32_t* last_ins,
                         uint32_t* g_evict, int clear_evict, const ServeArgs* sa = nullptr) {
    if (sa) uniq = sa->uniq;
    int64_t n = svc->n_log;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t t = log_line[i];
        int32_t o = line_node[t];
        if (o >= 0) slot_of[o] = -1;
        slot_of[uniq[log_pos[i]]] = -1;
        atomicMax(&last_ins[t], (int32_t)i);
        if (clear_evict) g_evict[t >> 5] = 0u;
    }
}
// CacheState.access's `evicted` per insertion of a multi-node call, in log
// order: the previous inserter of the same line in this call, else the
// line's occupant at the call's start (standalone API only: one thread,
// last_ins as per-line scratch, left as it was found, -1)
__global__ void k_victims(const int64_t* __restrict__ uniq, const ServeCounters* svc,
                          const int32_t* __restrict__ log_line, const int32_t* __restrict__ log_pos,
                          const int32_t* __restrict__ line_node, int32_t* last_ins,
                          int64_t* victim) {
    const int64_t n = svc->n_log;
    for (int64_t i = 0; i < n; i++) {
        const int32_t t = log_line[i];
        const int32_t prev = last_ins[t];
        victim[log_pos[i]] = prev >= 0 ? uniq[log_pos[prev]] : (int64_t)line_node[t];
        last_ins[t] = (int32_t)i;
    }
    for (int64_t i = 0; i < n; i++) last_ins[log_line[i]] = -1;
}
// post-pass B: the final inserter owns the line
__global__ void k_post_b(const int64_t* __restrict__ uniq, const ServeCounters* svc,
                         const int32_t* __restrict__ log_line, const int32_t* __restrict__ log_pos,
                         int32_t* line_node, int32_t* slot_of, const int32_t* __restrict__ last_ins,
                         int32_t* __restrict__ ins, const ServeArgs* sa = nullptr) {
    if (sa) uniq = sa->uniq;
    int64_t n = svc->n_log;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t t = log_line[i];
        if (last_ins[t] == (int32_t)i) {
            int32_t p = log_pos[i];
            int32_t x = (int32_t)uniq[p];
            slot_of[x] = t;
            line_node[t] = x;
            ins[p] = t;  // this row is the line's content after the batch
        }
    }
}

// tier split of the batch (dataloader.py:262-277), decided before the gather,
// plus the flags from which the gather's work lists are compacted (in
// position order: ascending node ids, so host-tier reads walk the backing
// table upward -- measured 10% faster over the host link than a scrambled order)
// tier counts and the gather's two work lists in one pass: hit positions,
// and (position, source row) of the host-tier rows -- constant-buffer row
// >= 0 or backing row x encoded -(x+1).  Each block tile reserves its range
// of a list with one atomic, so a list is ascending within a tile (the
// tiles' order is the blocks' arrival order; the gather does not depend on it).
__global__ void __launch_bounds__(BLOCK)
k_tier_lists(const int64_t* __restrict__ uniq, int64_t n, const int8_t* __restrict__ kind,
             const int32_t* __restrict__ pinned_off, ServeCounters* svc,
             int32_t* __restrict__ hit_list, int2* __restrict__ host_list, int64_t* list_cnt,
             const ServeArgs* sa = nullptr) {
    if (sa) {
        uniq = sa->uniq;
        n = sa->n;
    }
    __shared__ uint32_t s_w[BLOCK / 32];
    __shared__ uint32_t s_base[2];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    int64_t a = 0, b = 0, c = 0, d = 0;
    for (int64_t p0 = (int64_t)blockIdx.x * BLOCK; p0 < n; p0 += (int64_t)gridDim.x * BLOCK) {
        const int64_t p = p0 + t;
        const bool valid = p < n;
        const int k = valid ? kind[p] : GIDS_KIND_HIT;
        const bool hit = valid && k == GIDS_KIND_HIT, host = valid && k != GIDS_KIND_HIT;
        int2 item = make_int2(0, 0);
        if (hit) a++;
        if (host) {
            const int64_t x = uniq[p];
            const int32_t off = pinned_off[x];
            item = make_int2((int32_t)p, off >= 0 ? off : (int32_t)(-(x + 1)));
            d += k == GIDS_KIND_BYPASS;
            if (off >= 0) b++;
            else c++;
        }
        // block exclusive scan of (hit, host), packed in 16-bit halves
        const uint32_t mine = (hit ? 1u : 0u) | (host ? 1u << 16 : 0u);
        uint32_t inc = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) s_w[wid] = inc;
        __syncthreads();
        uint32_t ws = lane < BLOCK / 32 ? s_w[lane] : 0u;
#pragma unroll
        for (int o = 1; o < BLOCK / 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, ws, o);
            if (lane >= o) ws += u;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, ws, BLOCK / 32 - 1);
        const uint32_t ex = inc - mine + (wid > 0 ? __shfl_sync(0xffffffffu, ws, wid > 0 ? wid - 1 : 0) : 0u);
        if (t == 0) {
            s_base[0] = (uint32_t)atomicAdd((unsigned long long*)&list_cnt[0],
                                            (unsigned long long)(tot & 0xffffu));
            s_base[1] = (uint32_t)atomicAdd((unsigned long long*)&list_cnt[1],
                                            (unsigned long long)(tot >> 16));
        }
        __syncthreads();
        if (hit) hit_list[s_base[0] + (ex & 0xffffu)] = (int32_t)p;
        if (host) host_list[s_base[1] + (ex >> 16)] = item;
        __syncthreads();  // (s_w / s_base reused by the next tile)
    }
    a = warp_sum64(a);
    b = warp_sum64(b);
    c = warp_sum64(c);
    d = warp_sum64(d);
    if (lane == 0) {
        if (a) atomicAdd((unsigned long long*)&svc->tiers[0], (unsigned long long)a);
        if (b) atomicAdd((unsigned long long*)&svc->tiers[1], (unsigned long long)b);
        if (c) atomicAdd((unsigned long long*)&svc->tiers[2], (unsigned long long)c);
        if (d) atomicAdd((unsigned long long*)&svc->tiers[3], (unsigned long long)d);
    }
}

__global__ void k_post_c(const ServeCounters* svc, const int32_t* __restrict__ log_line,
                         int32_t* last_ins) {
    int64_t n = svc->n_log;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        last_ins[log_line[i]] = -1;
}

// ------------------------------------------------- set-associative policy
__device__ __forceinline__ int64_t sa_set_of(int64_t node, int64_t sets) {
    return (int64_t)__umul64hi(mix64((uint64_t)node), (uint64_t)sets);
}
__device__ __forceinline__ uint32_t sa_draw(uint64_t key, uint64_t epoch, int64_t node,
                                            uint32_t n) {
    uint64_t h = mix64(key ^ mix64(epoch * 0xD1B54A32D192ED03ULL + (uint64_t)node));
    return (uint32_t)(((uint64_t)(uint32_t)(h >> 32) * n) >> 32);
}

__global__ void k_sa_hist(const int64_t* __restrict__ uniq, int64_t n, int64_t sets,
                          int32_t* set_cnt, const ServeArgs* sa = nullptr) {
    if (sa) {
        uniq = sa->uniq;
        n = sa->n;
    }
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&set_cnt[sa_set_of(uniq[p], sets)], 1);
}
__global__ void k_sa_scatter(const int64_t* __restrict__ uniq, int64_t n, int64_t sets,
                             const int64_t* __restrict__ set_off, int32_t* set_cur,
                             int32_t* bucket, const ServeArgs* sa = nullptr) {
    if (sa) {
        uniq = sa->uniq;
        n = sa->n;
    }
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        int64_t s = sa_set_of(uniq[p], sets);
        bucket[set_off[s] + atomicAdd(&set_cur[s], 1)] = (int32_t)p;
    }
}

constexpr int SA_WARPS = BLOCK / 32;
constexpr int SA_SORT_MAX = 256;  // bucket entries sorted in registers

__global__ void __launch_bounds__(BLOCK)
k_sa_process(const int64_t* __restrict__ uniq, const uint32_t* __restrict__ ev, int64_t sets,
             const int32_t* __restrict__ set_cnt, const int64_t* __restrict__ set_off,
             int32_t* bucket, int32_t* line_node, int32_t* slot_of, uint32_t* safe_bits,
             uint64_t key, uint64_t epoch, int8_t* kind, int32_t* line, int32_t* ins,
             CacheMeta* meta, const ServeArgs* sa = nullptr) {
    if (sa) {
        uniq = sa->uniq;
        epoch = sa->epoch;
    }
    __shared__ int32_t order[SA_WARPS][SA_SORT_MAX];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int64_t hits = 0, misses = 0, byp = 0, evs = 0;
    for (int64_t s = (int64_t)blockIdx.x * SA_WARPS + wib; s < sets;
         s += (int64_t)gridDim.x * SA_WARPS) {
        const int cnt = set_cnt[s];
        if (cnt == 0) continue;
        int32_t* bk = bucket + set_off[s];
        const bool small = cnt <= SA_SORT_MAX;
        if (small) {  // rank sort of the bucket's batch positions
            int32_t e[SA_SORT_MAX / 32];
            int rank[SA_SORT_MAX / 32];
#pragma unroll
            for (int q = 0; q < SA_SORT_MAX / 32; q++) {
                int idx = lane + 32 * q;
                e[q] = idx < cnt ? bk[idx] : 0x7fffffff;
                rank[q] = 0;
            }
#pragma unroll
            for (int q2 = 0; q2 < SA_SORT_MAX / 32; q2++) {
                if (q2 * 32 >= cnt) break;
                const int lim = cnt - q2 * 32 < 32 ? cnt - q2 * 32 : 32;
                for (int jj = 0; jj < lim; jj++) {
                    int32_t vj = __shfl_sync(0xffffffffu, e[q2], jj);
#pragma unroll
                    for (int q = 0; q < SA_SORT_MAX / 32; q++) rank[q] += vj < e[q] ? 1 : 0;
                }
            }
#pragma unroll
            for (int q = 0; q < SA_SORT_MAX / 32; q++)
                if (lane + 32 * q < cnt) order[wib][rank[q]] = e[q];
            __syncwarp();
        }
        int32_t tag = line_node[s * 32 + lane];
        uint32_t safe = safe_bits[s];
        int32_t last = -1;
        int32_t my_ins = -1;  // batch position of this way's latest insertion
        for (int q = 0; q < cnt; q++) {
            int32_t p;
            if (small) {
                p = order[wib][q];
            } else {  // large bucket: next-smallest position by warp reduction
                int32_t best = 0x7fffffff;
                for (int idx = lane; idx < cnt; idx += 32) {
                    int32_t v = bk[idx];
                    if (v > last && v < best) best = v;
                }
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) {
                    int32_t o = __shfl_xor_sync(0xffffffffu, best, d);
                    best = o < best ? o : best;
                }
                p = best;
                last = best;
            }
            const int32_t x = (int32_t)uniq[p];
            const bool inuse = ev[p] & 1u;
            unsigned hm = __ballot_sync(0xffffffffu, tag == x);
            int kd, ln;
            if (hm) {
                int w = __ffs(hm) - 1;
                kd = GIDS_KIND_HIT;
                ln = (int)(s * 32 + w);
                hits++;
                if (!inuse) safe |= 1u << w;
            } else {
                unsigned em = __ballot_sync(0xffffffffu, tag < 0);
                int w = -1;
                if (em) {
                    w = __ffs(em) - 1;
                } else if (safe) {
                    uint32_t k = sa_draw(key, epoch, x, (uint32_t)__popc(safe));
                    w = __fns(safe, 0, (int)k + 1);
                    int32_t victim = __shfl_sync(0xffffffffu, tag, w);
                    if (lane == 0) slot_of[victim] = -1;
                    evs++;
                }
                if (w >= 0) {
                    kd = GIDS_KIND_MISS;
                    ln = (int)(s * 32 + w);
                    misses++;
                    if (lane == w) {
                        tag = x;
                        my_ins = p;
                    }
                    if (inuse) safe &= ~(1u << w);
                    else safe |= 1u << w;
                    if (lane == 0) slot_of[x] = ln;
                } else {
                    kd = GIDS_KIND_BYPASS;
                    ln = -1;
                    byp++;
                }
            }
            if (lane == 0) {
                kind[p] = (int8_t)kd;
                line[p] = ln;
            }
        }
        line_node[s * 32 + lane] = tag;
        if (my_ins >= 0) ins[my_ins] = (int32_t)(s * 32 + lane);
        if (lane == 0) safe_bits[s] = safe;
        __syncwarp();
    }
    if (lane == 0) {
        if (hits) atomicAdd((unsigned long long*)&meta->hits, (unsigned long long)hits);
        if (misses) atomicAdd((unsigned long long*)&meta->misses, (unsigned long long)misses);
        if (byp) atomicAdd((unsigned long long*)&meta->bypasses, (unsigned long long)byp);
        if (evs) atomicAdd((unsigned long long*)&meta->evictions, (unsigned long long)evs);
    }
}

}  // namespace

static int launch_exact_seq(gids_handle* h, int64_t n, size_t smem, cudaStream_t st,
                            const ServeArgs* sa) {
    {
        int rc = gids_launch_exact_par(h, n, st, sa);
        if (rc) return rc;
    }
    k_exact_allhit<<<gids_grid(n, BLOCK, 8 * GIDS_SMS), BLOCK, 0, st>>>(
        h->ev, n, h->meta, h->safe_bits, h->blk_cnt, h->sup_cnt, h->svc, h->kind, h->line, sa);
    GIDS_LAUNCH_CHECK(h);
    auto k = k_exact_seq;
    static size_t attr_smem = 48 * 1024;  // (per function: set when it grows)
    if (smem > attr_smem) {
        GIDS_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
        attr_smem = smem;
    }
    k<<<1, 32, smem, st>>>(h->ev, n, h->L, h->meta, h->safe_bits, h->evict_bits, h->blk_cnt,
                           h->sup_cnt, h->exact_smem ? 1 : 0, h->kind, h->line, h->log_line,
                           h->log_pos, h->svc, sa);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

int gids_launch_window(gids_handle* h, const int64_t* nodes, int64_t n, int delta,
                       cudaStream_t st) {
    if (n == 0) return GIDS_OK;
    k_window<<<gids_grid(n, BLOCK, 8 * GIDS_SMS), BLOCK, 0, st>>>(nodes, n, h->future, delta);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

int gids_launch_contribution(gids_handle* h, cudaStream_t st) {
    if (h->n_shards > 0) return GIDS_OK;  // whole table resident in HBM shards
    k_contribution<<<gids_grid(h->unique_cap, BLOCK, 4 * GIDS_SMS), BLOCK, 0, st>>>(
        h->unique32, h->sc, h->pinned_off, h->slot_of);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

size_t gids_exact_smem_bytes(int64_t L, bool with_bits) {
    int64_t nw = (L + 31) / 32, nb = (L + 1023) / 1024, ns = (L + 32767) / 32768;
    return sizeof(uint32_t) * (size_t)(nb + ns + (with_bits ? 2 * nw : 0));
}

// host time per section of the serve launch sequence (GIDS_SERVE_TIMING=1,
// printed at gids_destroy): where the API calls of a latency-bound batch go
#define HT(i)                                                                        \
    do {                                                                             \
        if (h->host_timing) {                                                        \
            const auto _n = std::chrono::steady_clock::now();                        \
            h->host_ns[i] += std::chrono::duration<double, std::nano>(_n - _ht).count(); \
            _ht = _n;                                                                \
        }                                                                            \
    } while (0)

// a serve replayed as a graph reads its per-call arguments from here
__global__ void k_serve_args(ServeArgs* sa, ServeArgs v) { *sa = v; }

// the folded window shift launched on its own (no decisions follow in this call)
static int launch_shift(gids_handle* h, cudaStream_t st) {
    const int64_t m = h->shift.n_pop + h->shift.n_push;
    if (m == 0) return GIDS_OK;
    k_window_shift<<<gids_grid(m, BLOCK, 8 * GIDS_SMS), BLOCK, 0, st>>>(
        h->shift.pop, h->shift.n_pop, h->shift.push, h->shift.n_push, h->future, nullptr);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

// the decisions of one batch on `st`: counters, window update + reuse
// consumption, the policy, tier counts and the gather's work lists, the
// counts' copy to the host.  sa != NULL: a graph capture -- n is then the
// workspace bound (grid sizes) and the kernels read the call's uniq / n /
// epoch from sa.
static int serve_decisions(gids_handle* h, const int64_t* uniq, int64_t n, uint64_t epoch,
                           cudaStream_t st, const ServeArgs* sa,
                           std::chrono::steady_clock::time_point& _ht) {
    const bool exact = h->cfg.policy == GIDS_POLICY_EXACT;
    GIDS_CUDA_TRY(cudaMemsetAsync(h->svc, 0, sizeof(ServeCounters), st));
    HT(1);
    int g = gids_grid(n, BLOCK, 8 * GIDS_SMS);
    if (sa || h->shift.n_pop + h->shift.n_push > 0) {  // the folded window shift
        const int64_t m = sa ? 2 * h->serve_cap : h->shift.n_pop + h->shift.n_push;
        k_window_shift<<<gids_grid(m, BLOCK, 8 * GIDS_SMS), BLOCK, 0, st>>>(
            h->shift.pop, h->shift.n_pop, h->shift.push, h->shift.n_push, h->future, sa);
        GIDS_LAUNCH_CHECK(h);
    }
    k_window_consume<<<g, BLOCK, 0, st>>>(uniq, n, h->future, h->reuse, h->slot_of,
                                          h->safe_bits, h->blk_cnt, h->sup_cnt, exact ? 1 : 0,
                                          h->meta, h->ev, 3, nullptr, &h->svc->n_miss0,
                                          exact ? h->xcls : nullptr, h->cand_of_slot,
                                          h->cand_slot, &h->svc->n_cand, &h->svc->bad_order,
                                          h->list_cnt, h->ins, sa);
    GIDS_LAUNCH_CHECK(h);
    HT(2);
    if (exact) {
        size_t smem = gids_exact_smem_bytes(h->L, h->exact_smem);
        int rc = launch_exact_seq(h, n, smem, st, sa);
        if (rc) return rc;
        k_post_a<<<g, BLOCK, 0, st>>>(uniq, h->svc, h->log_line, h->log_pos, h->line_node,
                                      h->slot_of, h->last_ins, h->evict_bits,
                                      h->exact_smem ? 0 : 1, sa);
        GIDS_LAUNCH_CHECK(h);
        k_post_b<<<g, BLOCK, 0, st>>>(uniq, h->svc, h->log_line, h->log_pos, h->line_node,
                                      h->slot_of, h->last_ins, h->ins, sa);
        GIDS_LAUNCH_CHECK(h);
        k_post_c<<<g, BLOCK, 0, st>>>(h->svc, h->log_line, h->last_ins);
        GIDS_LAUNCH_CHECK(h);
        int rc2 = gids_launch_xp_reset(h, st);
        if (rc2) return rc2;
    } else {
        GIDS_CUDA_TRY(cudaMemsetAsync(h->set_cnt, 0, sizeof(int32_t) * h->sets, st));
        GIDS_CUDA_TRY(cudaMemsetAsync(h->set_cur, 0, sizeof(int32_t) * h->sets, st));
        k_sa_hist<<<g, BLOCK, 0, st>>>(uniq, n, h->sets, h->set_cnt, sa);
        GIDS_LAUNCH_CHECK(h);
        int rc = gids_scan_i32_to_i64(h, h->set_cnt, h->sets, h->set_off, st);
        if (rc) return rc;
        k_sa_scatter<<<g, BLOCK, 0, st>>>(uniq, n, h->sets, h->set_off, h->set_cur, h->bucket,
                                          sa);
        GIDS_LAUNCH_CHECK(h);
        k_sa_process<<<gids_grid(h->sets, SA_WARPS, 16 * GIDS_SMS), BLOCK, 0, st>>>(
            uniq, h->ev, h->sets, h->set_cnt, h->set_off, h->bucket, h->line_node, h->slot_of,
            h->safe_bits, h->cfg.evict_key, epoch, h->kind, h->line, h->ins, h->meta, sa);
        GIDS_LAUNCH_CHECK(h);
    }
    HT(3);
    k_tier_lists<<<g, BLOCK, 0, st>>>(uniq, n, h->kind, h->pinned_off, h->svc, h->hit_list,
                                      h->host_list, h->list_cnt, sa);
    GIDS_LAUNCH_CHECK(h);
    HT(4);
    GIDS_CUDA_TRY(cudaMemcpyAsync(h->svc_host, h->svc, sizeof(ServeCounters),
                                  cudaMemcpyDeviceToHost, st));
    return GIDS_OK;
}

void gids_drop_serve_graphs(gids_handle* h) {
    if (!h->dgraph[0] && !h->dgraph[1] && !h->ggraph[0] && !h->ggraph[1]) return;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();  // (no launch of them still in flight)
    for (int i = 0; i < 2; i++) {
        if (h->dgraph[i]) cudaGraphExecDestroy(h->dgraph[i]);
        if (h->ggraph[i]) cudaGraphExecDestroy(h->ggraph[i]);
        h->dgraph[i] = h->ggraph[i] = nullptr;
    }
}

// one capture of `st`'s work into *exec (kernel count into *kernels); false
// (capture abandoned, the direct launches are used) on any failure
template <typename F>
static bool capture(gids_handle* h, cudaStream_t st, cudaGraphExec_t* exec, int64_t* kernels,
                    F&& body) {
    const int64_t l0 = h->launches;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    const int rc = body();
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(st, &graph);
    *kernels = h->launches - l0;
    h->launches = l0;
    bool ok = rc == GIDS_OK && e == cudaSuccess && graph &&
              cudaGraphInstantiate(exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    if (!ok) {
        *exec = nullptr;
        cudaGetLastError();
    }
    return ok;
}

int gids_launch_serve(gids_handle* h, const int64_t* uniq, int64_t n, uint64_t epoch, float* out,
                      cudaStream_t st, cudaStream_t gst) {
    auto _ht = std::chrono::steady_clock::now();
    // decision buffers: reuse the set of batch b-2 only after its gather finished
    h->parity ^= 1;
    const int par = h->parity;
    h->kind = h->kind_buf[par];
    h->line = h->line_buf[par];
    h->ins = h->ins_buf[par];
    h->hit_list = h->hit_list_buf[par];
    h->host_list = h->host_list_buf[par];
    h->list_cnt = h->list_cnt_buf[par];
    if (h->gathered_valid[par]) GIDS_CUDA_TRY(cudaStreamWaitEvent(st, h->gathered[par], 0));
    if (h->contributed_valid) {  // admissions counted against the cache this serve changes
        GIDS_CUDA_TRY(cudaStreamWaitEvent(st, h->contributed, 0));
        h->contributed_valid = false;
    }
    gids_harvest_gather(h, par);  // batch b-2's gather timing (profiling only)
    gids_mark(h, 2, st);
    if (h->n_shards > 0) {
        const int rc = launch_shift(h, st);
        return rc ? rc : gids_launch_shard_serve(h, uniq, n, out, st, gst, par);
    }
    HT(0);
    // replay as two graphs (decisions on st, rows on gst) once the first
    // serves have set every function attribute: the ~12 launches of a batch
    // cost more host time than a small batch's device work
    bool graphs = h->use_graphs && !h->graphs_failed && !h->ft && !h->profiling && n > 0 &&
                  h->serves >= 2 && st != 0 && st != cudaStreamLegacy && gst != 0 &&
                  gst != cudaStreamLegacy && gst != st;
    if (graphs) {
        ServeArgs* sa = h->sargs + par;
        k_serve_args<<<1, 1, 0, st>>>(sa, ServeArgs{uniq, n, epoch, out, h->shift.pop,
                                                      h->shift.n_pop, h->shift.push,
                                                      h->shift.n_push});
        GIDS_LAUNCH_CHECK(h);
        if (!h->dgraph[par] &&
            !capture(h, st, &h->dgraph[par], &h->dgraph_kernels[par], [&] {
                return serve_decisions(h, nullptr, h->serve_cap, epoch, st, sa, _ht);
            }))
            graphs = false, h->graphs_failed = true;  // (direct launches from now on)
    }
    if (graphs) {
        GIDS_CUDA_TRY(cudaGraphLaunch(h->dgraph[par], st));
        h->launches += h->dgraph_kernels[par];
        h->serve_replays++;
    } else if (n > 0) {
        int rc = serve_decisions(h, uniq, n, epoch, st, nullptr, _ht);
        if (rc) return rc;
        HT(5);
        if (h->ft) {  // file-backed storage tier: plan this batch's page reads
            int rc2 = gids_file_plan(h, par, st);
            if (rc2) return rc2;
        }
    } else {
        const int rc = launch_shift(h, st);
        if (rc) return rc;
        GIDS_CUDA_TRY(cudaMemsetAsync(h->svc, 0, sizeof(ServeCounters), st));
        GIDS_CUDA_TRY(cudaMemcpyAsync(h->svc_host, h->svc, sizeof(ServeCounters),
                                      cudaMemcpyDeviceToHost, st));
    }
    gids_mark(h, 3, st);  // (before `counted`: serve_counts reads this mark's time)
    GIDS_CUDA_TRY(cudaEventRecord(h->counted, st));
    h->counted_valid = true;
    h->last_serve_n = n;
    HT(6);
    if (n > 0) {
        if (gst != st) {
            GIDS_CUDA_TRY(cudaEventRecord(h->decided, st));
            GIDS_CUDA_TRY(cudaStreamWaitEvent(gst, h->decided, 0));
        }
        if (graphs) {
            const ServeArgs* sa = h->sargs + par;
            if (!h->ggraph[par] &&
                !capture(h, gst, &h->ggraph[par], &h->ggraph_kernels[par], [&] {
                    return gids_launch_gather(h, nullptr, h->serve_cap, nullptr, gst, sa);
                }))
                graphs = false, h->graphs_failed = true;
        }
        if (graphs) {
            GIDS_CUDA_TRY(cudaGraphLaunch(h->ggraph[par], gst));
            h->launches += h->ggraph_kernels[par];
        } else {
            if (h->profiling) cudaEventRecord(h->gev[par][0], gst);
            int rc = gids_launch_gather(h, uniq, n, out, gst);
            if (rc) return rc;
        }
        GIDS_CUDA_TRY(cudaEventRecord(h->gathered[par], gst));
        h->gathered_valid[par] = true;
        h->gather_pending[par] = h->profiling;
        h->serve_timed = h->profiling;
    }
    h->serves++;
    HT(7);
    if (h->host_timing) h->host_calls++;
    return GIDS_OK;
}

// ------------------------------------------------ standalone CacheState API
// window_update (cache.py:190-218) and CacheState.access (cache.py:144-180)
// as separate calls, for callers that drive the cache directly (the reference
// exports both); the serving path fuses them in gids_launch_serve.
extern "C" int gids_cache_window_update(gids_handle* h, const int64_t* nodes, int64_t n,
                                        int32_t* counts, void* stream) {
    if (!h || n < 0 || (n > 0 && !nodes)) {
        gids_set_error("cache_window_update: bad arguments");
        return GIDS_E_INVALID;
    }
    GIDS_CUDA_TRY(cudaSetDevice(h->device));
    if (n == 0) return GIDS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    h->last_stream = st;
    const bool exact = h->cfg.policy == GIDS_POLICY_EXACT;
    k_window_consume<<<gids_grid(n, BLOCK, 8 * GIDS_SMS), BLOCK, 0, st>>>(
        nodes, n, h->future, h->reuse, h->slot_of, h->safe_bits, h->blk_cnt, h->sup_cnt,
        exact ? 1 : 0, h->meta, h->ev, 1, counts);
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

extern "C" int gids_cache_access(gids_handle* h, const int64_t* nodes, int64_t n,
                                 int8_t* kind_out, int32_t* line_out, int64_t* victim_out,
                                 void* stream) {
    if (!h || n < 0 || (n > 0 && (!nodes || !kind_out || !line_out))) {
        gids_set_error("cache_access: bad arguments");
        return GIDS_E_INVALID;
    }
    if (h->cfg.policy != GIDS_POLICY_EXACT) {
        gids_set_error("cache_access drives the reference (exact) policy");
        return GIDS_E_INVALID;
    }
    if (n > h->serve_cap) {
        gids_set_error("cache_access: more nodes than the handle's serving workspace");
        return GIDS_E_CAPACITY;
    }
    GIDS_CUDA_TRY(cudaSetDevice(h->device));
    if (n == 0) return GIDS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    h->last_stream = st;
    for (int b = 0; b < 2; b++)  // a served batch's gather may still read the lines
        if (h->gathered_valid[b]) GIDS_CUDA_TRY(cudaStreamWaitEvent(st, h->gathered[b], 0));
    GIDS_CUDA_TRY(cudaMemsetAsync(h->svc, 0, sizeof(ServeCounters), st));
    GIDS_CUDA_TRY(cudaMemsetAsync(h->ins, 0xff, sizeof(int32_t) * n, st));
    if (victim_out) GIDS_CUDA_TRY(cudaMemsetAsync(victim_out, 0xff, sizeof(int64_t) * n, st));
    const int g = gids_grid(n, BLOCK, 8 * GIDS_SMS);
    k_window_consume<<<g, BLOCK, 0, st>>>(nodes, n, h->future, h->reuse, h->slot_of,
                                          h->safe_bits, h->blk_cnt, h->sup_cnt, 1, h->meta, h->ev,
                                          2, nullptr, &h->svc->n_miss0, h->xcls,
                                          h->cand_of_slot, h->cand_slot, &h->svc->n_cand);
    GIDS_LAUNCH_CHECK(h);
    size_t smem = gids_exact_smem_bytes(h->L, h->exact_smem);
    {
        int rc = launch_exact_seq(h, n, smem, st, nullptr);
        if (rc) return rc;
    }
    if (victim_out) {
        k_victims<<<1, 1, 0, st>>>(nodes, h->svc, h->log_line, h->log_pos, h->line_node,
                                   h->last_ins, victim_out);
        GIDS_LAUNCH_CHECK(h);
    }
    k_post_a<<<g, BLOCK, 0, st>>>(nodes, h->svc, h->log_line, h->log_pos, h->line_node,
                                  h->slot_of, h->last_ins, h->evict_bits, h->exact_smem ? 0 : 1);
    GIDS_LAUNCH_CHECK(h);
    k_post_b<<<g, BLOCK, 0, st>>>(nodes, h->svc, h->log_line, h->log_pos, h->line_node,
                                  h->slot_of, h->last_ins, h->ins);
    GIDS_LAUNCH_CHECK(h);
    k_post_c<<<g, BLOCK, 0, st>>>(h->svc, h->log_line, h->last_ins);
    GIDS_LAUNCH_CHECK(h);
    {
        int rc = gids_launch_xp_reset(h, st);
        if (rc) return rc;
    }
    GIDS_CUDA_TRY(cudaMemcpyAsync(kind_out, h->kind, n, cudaMemcpyDeviceToDevice, st));
    GIDS_CUDA_TRY(cudaMemcpyAsync(line_out, h->line, sizeof(int32_t) * n,
                                  cudaMemcpyDeviceToDevice, st));
    return GIDS_OK;
}

// per-node predicted-reuse counters (reuse_counter, cache.py:104-113), host copy
extern "C" int gids_cache_reuse(gids_handle* h, uint32_t* reuse_host) {
    if (!h || !reuse_host) {
        gids_set_error("cache_reuse: bad arguments");
        return GIDS_E_INVALID;
    }
    GIDS_CUDA_TRY(cudaSetDevice(h->device));
    GIDS_CUDA_TRY(cudaDeviceSynchronize());
    GIDS_CUDA_TRY(cudaMemcpy(reuse_host, h->reuse, sizeof(uint32_t) * h->N,
                             cudaMemcpyDeviceToHost));
    return GIDS_OK;
}

// run-ahead contribution of an already exported batch (dataloader.py:188-192)
// against the cache as the stream reaches this call: lets the loader sample
// batches ahead of the moment the reference would, and still count them
// against the reference's cache state
extern "C" int gids_contribution_async(gids_handle* h, const int64_t* unique_dev,
                                       const int64_t* n_ptr, int64_t* out_host, void* stream) {
    if (!h || !unique_dev || !n_ptr || !out_host) {
        gids_set_error("contribution_async: bad arguments");
        return GIDS_E_INVALID;
    }
    GIDS_CUDA_TRY(cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long* scratch = reinterpret_cast<unsigned long long*>(h->contrib_dev);
    if (h->n_shards > 0) {  // a sharded table keeps every row resident: 0
        GIDS_CUDA_TRY(cudaMemsetAsync(out_host, 0, sizeof(int64_t), st));
        return GIDS_OK;
    }
    // against the cache as the last serve's decisions leave it; the next serve
    // waits for these reads (both orderings on the device, no host events)
    if (h->counted_valid) GIDS_CUDA_TRY(cudaStreamWaitEvent(st, h->counted, 0));
    k_contribution64<<<gids_grid(h->unique_cap, BLOCK, 4 * GIDS_SMS), BLOCK, 0, st>>>(
        unique_dev, n_ptr, h->pinned_off, h->slot_of, scratch, out_host);
    GIDS_LAUNCH_CHECK(h);
    GIDS_CUDA_TRY(cudaEventRecord(h->contributed, st));
    h->contributed_valid = true;
    return GIDS_OK;
}
