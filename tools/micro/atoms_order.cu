// Does a warp's shared-memory atomicAdd return old values in lane order for
// lanes that hit the same address?  Random digit patterns, many trials.
#include <cstdio>
#include <cstdint>
__global__ void k(unsigned *bad, unsigned *tot, unsigned seed, int ndig) {
    __shared__ unsigned cnt[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    unsigned lane = threadIdx.x & 31;
    unsigned long long z = seed * 0x9E3779B97F4A7C15ull + blockIdx.x * 7919ull + threadIdx.x * 104729ull;
    for (int it = 0; it < 64; ++it) {
        z = z * 6364136223846793005ull + 1442695040888963407ull;
        unsigned d = (unsigned)(z >> 33) % ndig;
        unsigned old = atomicAdd(&cnt[d], 1u);
        unsigned peers = __match_any_sync(0xffffffffu, d);
        // old must be increasing in lane order among peers
        unsigned lower = peers & ((1u << lane) - 1u);
        unsigned prev_old = 0;
        bool ok = true;
        // compare with every lower peer
        for (int j = 0; j < 32; ++j) {
            unsigned o = __shfl_sync(0xffffffffu, old, j);
            if ((lower >> j) & 1u) ok &= o < old;
        }
        if (!ok) atomicAdd(bad, 1u);
        if (__popc(peers) > 1) atomicAdd(tot, 1u);
        __syncwarp();
    }
}
int main() {
    unsigned *b, *t;
    cudaMallocManaged(&b, 4); cudaMallocManaged(&t, 4);
    for (int nd : {2, 8, 64, 700}) {
        *b = 0; *t = 0;
        for (int s = 0; s < 20; ++s) k<<<296, 384>>>(b, t, s, nd);
        cudaDeviceSynchronize();
        printf("ndig %4d: keys in collision groups %u, lane-order violations %u\n", nd, *t, *b);
    }
}
