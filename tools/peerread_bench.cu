// peerread_bench.cu -- NVLink peer-read micro-benchmark for the sharded-table
// gather (not part of the product).
//
// GPU 0 gathers random 4 KiB rows that live in GPU 1's HBM (peer access over
// NVLink 5 / NVSwitch) with the same flat 16-byte-chunk loop as
// k_gather_shards, at several grid sizes, and prints GB/s next to a
// cudaMemcpyPeer of one contiguous block.  Needs >= 2 GPUs.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o peerread_bench peerread_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <random>
#include <vector>

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e = (x);                                                         \
        if (e != cudaSuccess) {                                                      \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

template <int U>
__global__ void k_peer(const int32_t* __restrict__ sel, int64_t nsel, int cpr,
                       const int4* __restrict__ src, int4* __restrict__ out) {
    const uint64_t total = (uint64_t)nsel * cpr;
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = warp * U * 32; base < total; base += nw * U * 32) {
        int4 v[U];
        int64_t d[U];
#pragma unroll
        for (int k = 0; k < U; k++) {
            const uint64_t i = base + k * 32 + lane;
            d[k] = -1;
            if (i < total) {
                const uint64_t r = i / cpr, c = i - r * cpr;
                v[k] = __ldg(src + (int64_t)sel[r] * cpr + c);
                d[k] = (int64_t)i;
            }
        }
#pragma unroll
        for (int k = 0; k < U; k++)
            if (d[k] >= 0) out[d[k]] = v[k];
    }
}

int main() {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) {
        printf("peerread_bench: needs >= 2 GPUs (found %d)\n", ndev);
        return 0;
    }
    int can = 0;
    CK(cudaDeviceCanAccessPeer(&can, 0, 1));
    if (!can) {
        printf("peerread_bench: GPU 0 cannot access GPU 1\n");
        return 0;
    }
    const int row = 4096, cpr = row / 16;
    const int64_t nrows = 4 << 20;  // 16 GiB shard on GPU 1
    const int64_t nsel = 256 << 10;  // 1 GiB gathered
    char* shard;
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&shard, (size_t)nrows * row));
    CK(cudaMemset(shard, 1, (size_t)nrows * row));
    CK(cudaSetDevice(0));
    CK(cudaDeviceEnablePeerAccess(1, 0));
    std::vector<int32_t> sel(nsel);
    std::mt19937_64 rng(1);
    for (auto& x : sel) x = (int32_t)(rng() % nrows);
    std::sort(sel.begin(), sel.end());
    int32_t* dsel;
    char* out;
    CK(cudaMalloc(&dsel, sizeof(int32_t) * nsel));
    CK(cudaMemcpy(dsel, sel.data(), sizeof(int32_t) * nsel, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&out, (size_t)nsel * row));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const double bytes = (double)nsel * row;
    auto timeit = [&](const char* name, auto&& launch) {
        launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a));
        for (int r = 0; r < 5; r++) launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        printf("  %-28s %8.1f GB/s\n", name, 5 * bytes / (ms * 1e-3) / 1e9);
    };
    char name[64];
    for (int bps : {1, 2, 4, 8})
        for (int u : {2, 4}) {
            snprintf(name, sizeof name, "peer ldg blocks/sm=%d u=%d", bps, u);
            timeit(name, [&] {
                if (u == 2)
                    k_peer<2><<<148 * bps, 256>>>(dsel, nsel, cpr, (const int4*)shard, (int4*)out);
                else
                    k_peer<4><<<148 * bps, 256>>>(dsel, nsel, cpr, (const int4*)shard, (int4*)out);
            });
        }
    timeit("cudaMemcpyPeer contiguous", [&] {
        CK(cudaMemcpyPeerAsync(out, 0, shard, 1, (size_t)bytes));
    });
    return 0;
}
