// Microbenchmark of warp ranking primitives on B200 (16 warps/SM, 148 CTAs):
// per-SM cycles per 32-key chunk for: match_any, 11-bit ballot rank, tag-based
// (unstable) rank via smem, smem atomicAdd per lane.  Column values: 32 lanes
// drawn from `ncol` columns (random, fixed seed).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned hash32(unsigned x) { x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x; }
template <int MODE>
__global__ void k(unsigned *out, int ncol, int iters, long long *cyc) {
    __shared__ unsigned short cnt[16][1024];
    __shared__ unsigned char tag[16][1000];
    const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 16 * 1000; i += blockDim.x) { (&cnt[0][0])[i] = 0; (&tag[0][0])[i] = 0; }
    __syncthreads();
    unsigned acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const unsigned u = hash32(it * 977 + lane * 31 + blockIdx.x) % ncol;
        unsigned r;
        if (MODE == 0) {
            const unsigned peers = __match_any_sync(0xffffffffu, u);
            const unsigned leader = __ffs(peers) - 1;
            unsigned old = 0;
            if (lane == leader) { old = cnt[w][u]; cnt[w][u] = old + __popc(peers); }
            old = __shfl_sync(0xffffffffu, old, leader);
            r = old + __popc(peers & ((1u << lane) - 1));
            __syncwarp();
        } else if (MODE == 1) {
            unsigned peers = 0xffffffffu;
#pragma unroll
            for (int b = 0; b < 11; ++b) { const unsigned bb = __ballot_sync(0xffffffffu, (u >> b) & 1); peers &= ((u >> b) & 1) ? bb : ~bb; }
            const unsigned leader = __ffs(peers) - 1;
            unsigned old = 0;
            if (lane == leader) { old = cnt[w][u]; cnt[w][u] = old + __popc(peers); }
            old = __shfl_sync(0xffffffffu, old, leader);
            r = old + __popc(peers & ((1u << lane) - 1));
            __syncwarp();
        } else if (MODE == 2) {   // tag rounds (unstable)
            bool done = false;
            r = 0;
            while (__any_sync(0xffffffffu, !done)) {
                if (!done) tag[w][u] = (unsigned char)lane;
                __syncwarp();
                if (!done && tag[w][u] == lane) { r = cnt[w][u]; cnt[w][u] = r + 1; done = true; }
                __syncwarp();
            }
        } else {                  // smem atomic per lane (unstable)
            r = atomicAdd((unsigned*)&cnt[w][u & ~1u], (u & 1) ? 65536u : 1u);
        }
        acc += r;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    unsigned *out; long long *cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    long long h[148];
    const char *names[4] = {"match_any", "ballot11", "tag-rounds", "atomicAdd"};
    for (int ncol : {8, 64, 400, 1000}) {
        printf("ncol %4d:", ncol);
        for (int mode = 0; mode < 4; ++mode) {
            int it = 4000;
            if (mode == 0) k<0><<<148, 512>>>(out, ncol, it, cyc);
            if (mode == 1) k<1><<<148, 512>>>(out, ncol, it, cyc);
            if (mode == 2) k<2><<<148, 512>>>(out, ncol, it, cyc);
            if (mode == 3) k<3><<<148, 512>>>(out, ncol, it, cyc);
            cudaDeviceSynchronize();
            cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
            printf("  %s %.1f", names[mode], (double)h[0] / it / 16.0);
        }
        printf("   (SM cycles per 32-key chunk)\n");
    }
    return 0;
}
