// hostread_bench.cu -- host-link read micro-benchmark for the storage-tier
// gather (not part of the product).
//
// Gathers `nsel` random rows (ascending, like a batch's unique nodes) of a
// pinned host table into HBM three ways and prints GB/s:
//   ldg   warp-wide 16-B zero-copy loads, U loads in flight per lane
//   tma   cp.async.bulk (TMA bulk copy) host -> smem, D stages per CTA,
//         then cp.async.bulk smem -> HBM
//   dma   cudaMemcpyAsync of one contiguous block (the copy-engine ceiling)
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o hostread_bench hostread_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <sys/mman.h>

#include <algorithm>
#include <random>
#include <vector>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x,               \
                    cudaGetErrorString(e));                                         \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

template <int U>
__global__ void k_ldg(const int32_t* __restrict__ sel, int64_t nsel, int cpr,
                      const int4* __restrict__ table, int4* __restrict__ out) {
    const uint32_t total = (uint32_t)(nsel * cpr);
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t base = warp * U * 32; base < total; base += nw * U * 32) {
        int4 v[U];
        int64_t d[U];
#pragma unroll
        for (int k = 0; k < U; k++) {
            uint32_t i = base + k * 32 + lane;
            d[k] = -1;
            if (i < total) {
                uint32_t r = i / cpr, c = i - r * cpr;
                asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                             : "l"(table + (int64_t)sel[r] * cpr + c));
                d[k] = (int64_t)r * cpr + c;
            }
        }
#pragma unroll
        for (int k = 0; k < U; k++)
            if (d[k] >= 0) out[d[k]] = v[k];
    }
}

// the product's k_gather_host shape: int2 (position, source) list, per-row
// insert line; MODE bit0 = write the cache insert, bit1 = read ins[]
template <int U, int MODE>
__global__ void k_prod(const int2* __restrict__ list, int64_t n, int cpr,
                       const int32_t* __restrict__ ins, const int4* __restrict__ table,
                       int4* __restrict__ cache, int4* __restrict__ out) {
    const uint32_t total = (uint32_t)(n * cpr);
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t base = warp * U * 32; base < total; base += nw * U * 32) {
        int4 v[U];
        int64_t d[U], d2[U];
#pragma unroll
        for (int k = 0; k < U; k++) {
            uint32_t i = base + k * 32 + lane;
            d[k] = -1;
            if (i < total) {
                uint32_t r = i / cpr, c = i - r * cpr;
                int2 it = list[r];
                asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                             : "l"(table + (int64_t)(-(it.y + 1)) * cpr + c));
                d[k] = (int64_t)it.x * cpr + c;
                int32_t t = (MODE & 2) ? ins[it.x] : -1;
                d2[k] = t >= 0 ? (int64_t)t * cpr + c : -1;
            }
        }
#pragma unroll
        for (int k = 0; k < U; k++)
            if (d[k] >= 0) {
                asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(out + d[k]),
                             "r"(v[k].x), "r"(v[k].y), "r"(v[k].z), "r"(v[k].w) : "memory");
                if ((MODE & 1) && d2[k] >= 0) cache[d2[k]] = v[k];
            }
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// one warp per CTA; lane 0 drives a D-stage ring of bulk copies
template <int D>
__global__ void k_tma(const int32_t* __restrict__ sel, int64_t nsel, int row_bytes,
                      const char* __restrict__ table, char* __restrict__ out) {
    extern __shared__ __align__(128) char smem[];
    __shared__ __align__(8) uint64_t bar[D];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < D; s++)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    const int64_t first = blockIdx.x, step = gridDim.x;
    uint32_t phase[D];
    for (int s = 0; s < D; s++) phase[s] = 0;
    auto issue = [&](int64_t j, int s) {
        const char* src = table + (int64_t)sel[j] * row_bytes;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         smem_u32(&bar[s])),
                     "r"(row_bytes));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(smem + (int64_t)s * row_bytes)),
            "l"(src), "r"(row_bytes), "r"(smem_u32(&bar[s]))
            : "memory");
    };
    int64_t j = first;
    int filled = 0;
    for (int s = 0; s < D && j + (int64_t)s * step < nsel; s++, filled++) issue(j + s * step, s);
    int s = 0;
    for (int64_t k = j; k < nsel; k += step) {
        // wait for stage s
        uint32_t ok = 0;
        while (!ok) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 "
                "%0, 1, 0, p; }"
                : "=r"(ok)
                : "r"(smem_u32(&bar[s])), "r"(phase[s]));
        }
        phase[s] ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                         out + k * row_bytes),
                     "r"(smem_u32(smem + (int64_t)s * row_bytes)), "r"(row_bytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        int64_t nk = k + (int64_t)D * step;
        if (nk < nsel) issue(nk, s);
        s = (s + 1) % D;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
    int row_bytes = argc > 1 ? atoi(argv[1]) : 512;
    int64_t table_bytes = (argc > 2 ? atoll(argv[2]) : 8LL) << 30;
    double frac = argc > 3 ? atof(argv[3]) : 0.05;
    int64_t nrows = table_bytes / row_bytes;
    int64_t nsel = (int64_t)(nrows * frac);
    if ((int64_t)nsel * row_bytes > (3LL << 30)) nsel = (3LL << 30) / row_bytes;
    int mode = argc > 4 ? atoi(argv[4]) : 0;
    int quick = argc > 5 ? atoi(argv[5]) : 0;
    char* table;
    if (mode == 0) {
        CK(cudaHostAlloc(&table, table_bytes, cudaHostAllocMapped));
    } else {  // 2 MiB-aligned anonymous memory with transparent huge pages, then registered
        void* p = mmap(nullptr, table_bytes + (2 << 20), PROT_READ | PROT_WRITE,
                       MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (p == MAP_FAILED) { perror("mmap"); return 1; }
        table = (char*)(((uintptr_t)p + (2 << 20) - 1) & ~(uintptr_t)((2 << 20) - 1));
        if (madvise(table, table_bytes, MADV_HUGEPAGE)) perror("madvise");
    }
    for (int64_t i = 0; i < table_bytes; i += 4096) table[i] = (char)i;
    if (mode != 0) CK(cudaHostRegister(table, table_bytes, cudaHostRegisterMapped));
    printf("alloc mode %d\n", mode);
    std::vector<int32_t> sel(nrows);
    for (int64_t i = 0; i < nrows; i++) sel[i] = (int32_t)i;
    std::mt19937_64 rng(1);
    std::shuffle(sel.begin(), sel.end(), rng);
    sel.resize(nsel);
    std::sort(sel.begin(), sel.end());
    int32_t* dsel;
    char* out;
    CK(cudaMalloc(&dsel, sizeof(int32_t) * nsel));
    CK(cudaMemcpy(dsel, sel.data(), sizeof(int32_t) * nsel, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&out, (size_t)nsel * row_bytes));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const double bytes = (double)nsel * row_bytes;
    printf("row_bytes=%d table=%.1fGB nsel=%lld (%.2f GB)\n", row_bytes, table_bytes / 1e9,
           (long long)nsel, bytes / 1e9);
    auto timeit = [&](const char* name, auto&& launch) {
        launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a));
        for (int r = 0; r < 3; r++) launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        printf("  %-24s %7.2f GB/s\n", name, 3 * bytes / (ms * 1e-3) / 1e9);
        fflush(stdout);
    };
    const int cpr = row_bytes / 16;
    char name[64];
    for (int wps : {2, 4, 8})
        for (int u : {1, 2, 4}) {
            if (quick && !(wps == 2 && u == 2) && !(wps == 8 && u == 4)) continue;
            int blocks = wps * 148 / 8;
            snprintf(name, sizeof name, "ldg wps=%d u=%d", wps, u);
            timeit(name, [&] {
                if (u == 1) k_ldg<1><<<blocks, 256>>>(dsel, nsel, cpr, (const int4*)table, (int4*)out);
                if (u == 2) k_ldg<2><<<blocks, 256>>>(dsel, nsel, cpr, (const int4*)table, (int4*)out);
                if (u == 4) k_ldg<4><<<blocks, 256>>>(dsel, nsel, cpr, (const int4*)table, (int4*)out);
            });
        }
    for (int cps : {1, 2, 4, 8})
        for (int d : {2, 4, 8}) {
            size_t sm = (size_t)d * row_bytes;
            if (sm > 200 * 1024 || sm * cps > 220 * 1024) continue;
            if (quick && !(cps == 2 && d == 4)) continue;
            int blocks = cps * 148;
            snprintf(name, sizeof name, "tma ctas/sm=%d D=%d", cps, d);
            auto go = [&](auto kern) {
                CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                timeit(name, [&] { kern<<<blocks, 32, sm>>>(dsel, nsel, row_bytes, table, out); });
            };
            if (d == 2) go(k_tma<2>);
            if (d == 4) go(k_tma<4>);
            if (d == 8) go(k_tma<8>);
            CK(cudaGetLastError());
        }
    {
        // product-like inputs: positions interleaved with hits (every 20th
        // position is a hit and absent), ins[] = a cache line per position
        std::vector<int2> lst(nsel);
        std::vector<int32_t> insv(nsel + nsel / 19 + 2);
        int64_t lines = 2097152;
        std::mt19937_64 r2(2);
        for (int64_t i = 0; i < nsel; i++) lst[i] = make_int2((int32_t)(i + i / 19), -(sel[i] + 1));
        for (auto& x : insv) x = (int32_t)(r2() % lines);
        int2* dl;
        int32_t* di;
        int4 *dc, *dout2;
        CK(cudaMalloc(&dl, sizeof(int2) * nsel));
        CK(cudaMalloc(&di, sizeof(int32_t) * insv.size()));
        CK(cudaMalloc(&dc, (size_t)lines * row_bytes));
        CK(cudaMalloc(&dout2, (size_t)insv.size() * row_bytes));
        CK(cudaMemcpy(dl, lst.data(), sizeof(int2) * nsel, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(di, insv.data(), sizeof(int32_t) * insv.size(), cudaMemcpyHostToDevice));
        for (int wps : {2, 8})
            for (int u : {2, 8}) {
                int blocks = wps * 148 / 8;
                snprintf(name, sizeof name, "prod wps=%d u=%d full", wps, u);
                timeit(name, [&] {
                    if (u == 2) k_prod<2, 3><<<blocks, 256>>>(dl, nsel, cpr, di, (const int4*)table, dc, dout2);
                    else k_prod<8, 3><<<blocks, 256>>>(dl, nsel, cpr, di, (const int4*)table, dc, dout2);
                });
                snprintf(name, sizeof name, "prod wps=%d u=%d noins", wps, u);
                timeit(name, [&] {
                    if (u == 2) k_prod<2, 0><<<blocks, 256>>>(dl, nsel, cpr, di, (const int4*)table, dc, dout2);
                    else k_prod<8, 0><<<blocks, 256>>>(dl, nsel, cpr, di, (const int4*)table, dc, dout2);
                });
                snprintf(name, sizeof name, "prod wps=%d u=%d readins", wps, u);
                timeit(name, [&] {
                    if (u == 2) k_prod<2, 2><<<blocks, 256>>>(dl, nsel, cpr, di, (const int4*)table, dc, dout2);
                    else k_prod<8, 2><<<blocks, 256>>>(dl, nsel, cpr, di, (const int4*)table, dc, dout2);
                });
            }
    }
    // (the copy-engine per-row batch copy measured in round 1 -- 3.8 GB/s at 4 KB,
    // profiles/r01_hostread_microbench_dma_batch.txt -- is a closed API on this pool)
    timeit("dma contiguous", [&] {
        CK(cudaMemcpyAsync(out, table, (size_t)bytes, cudaMemcpyHostToDevice));
    });
    return 0;
}
