// Microbenchmark: __match_any_sync latency/throughput vs number of distinct values,
// compared with a ballot-based equivalent (11-bit keys).  Run: ./match_bench
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_match(unsigned *out, int distinct, int iters, long long *cyc) {
    unsigned lane = threadIdx.x & 31;
    unsigned v = (lane * 2654435761u) % distinct;
    unsigned acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        unsigned m = __match_any_sync(0xffffffffu, v + acc);
        acc += __popc(m) & 1;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_ballot(unsigned *out, int distinct, int iters, long long *cyc) {
    unsigned lane = threadIdx.x & 31;
    unsigned v = (lane * 2654435761u) % distinct;
    unsigned acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        unsigned x = (v + acc) & 2047u, m = 0xffffffffu;
#pragma unroll
        for (int b = 0; b < 11; ++b) { unsigned bb = __ballot_sync(0xffffffffu, (x >> b) & 1); m &= ((x >> b) & 1) ? bb : ~bb; }
        acc += __popc(m) & 1;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    unsigned *out; long long *cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    long long h[148];
    for (int warps : {1, 16}) for (int d : {1, 4, 16, 32}) {
        int it = 2000;
        k_match<<<148, 32 * warps>>>(out, d, it, cyc); cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
        double m1 = (double)h[0] / it;
        k_ballot<<<148, 32 * warps>>>(out, d, it, cyc); cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
        double m2 = (double)h[0] / it;
        printf("warps/SM %2d distinct %2d: match %.1f cyc/iter per warp, ballot11 %.1f\n", warps, d, m1, m2);
    }
    return 0;
}
