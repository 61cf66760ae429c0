// Micro-benchmark: cost of a __syncthreads round trip for one 512-thread CTA
// (the shape of k_exact_par), with and without a dependent shared-memory
// chain per phase.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bb tools/barrier_bench.cu
#include <cstdio>
__global__ void __launch_bounds__(512, 1) k(int iters, int chain, long long* out, int* sink) {
    __shared__ int buf[1024];
    const int t = threadIdx.x;
    buf[t] = t;
    buf[t + 512] = t;
    __syncthreads();
    int v = t;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        for (int c = 0; c < chain; c++) v = buf[(v + c) & 1023];
        __syncthreads();
    }
    long long t1 = clock64();
    if (t == 0) *out = t1 - t0;
    if (v == -1) *sink = v;
}
int main() {
    long long* d;
    int* s;
    cudaMalloc(&d, 8);
    cudaMalloc(&s, 4);
    for (int chain : {0, 1, 4, 8, 16}) {
        k<<<1, 512>>>(10000, chain, d, s);
        long long h;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("chain %2d: %.1f cycles per phase\n", chain, h / 10000.0);
    }
    return 0;
}
