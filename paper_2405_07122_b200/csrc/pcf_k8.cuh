// pcf_k8.cuh -- K8: the GPU "Standard-Sort" for buckets too large for one
// CTA (Lemma 1 needs a worst-case O(n log n) sort,
// PAPER.md:235).  A comparison merge sort: 2048-key tiles sorted in shared
// memory (bitonic), then log2(m/2048) stable merge-path passes.  Keys are
// compared as ordered u64 (IEEE totalOrder for f64, reading R11).
#pragma once
#include "pcf_common.cuh"

namespace pcf {

constexpr int K8_THREADS = 512;
constexpr int K8_TILE = 2048;
constexpr int K8_IPT = K8_TILE / K8_THREADS;   // 4

template <class K>
__global__ void __launch_bounds__(K8_THREADS) k8_blocksort(const u64 *__restrict__ src, u64 *__restrict__ dst, u64 m) {
    __shared__ u64 a[K8_TILE];
    const u64 base = (u64)blockIdx.x * K8_TILE;
    const u32 n = (u32)min((u64)K8_TILE, m - base);
    for (u32 k = threadIdx.x; k < K8_TILE; k += K8_THREADS) a[k] = k < n ? K::to_okey(src[base + k]) : ~0ull;
    __syncthreads();
    // full bitonic sort of 2048 keys (padding = max key sorts to the end)
    for (u32 k = 2; k <= (u32)K8_TILE; k <<= 1) {
        for (u32 j = k >> 1; j > 0; j >>= 1) {
            for (u32 t = threadIdx.x; t < K8_TILE / 2; t += K8_THREADS) {
                u32 lo = ((t / j) * 2 * j) + (t % j), hi = lo + j;
                bool up = (lo & k) == 0;
                u64 x = a[lo], y = a[hi];
                if ((x > y) == up) { a[lo] = y; a[hi] = x; }
            }
            __syncthreads();
        }
    }
    for (u32 k = threadIdx.x; k < n; k += K8_THREADS) dst[base + k] = K::from_okey(a[k]);
}

template <class K>
__global__ void __launch_bounds__(K8_THREADS) k8_merge(const u64 *__restrict__ src, u64 *__restrict__ dst, u64 m, u64 width) {
    __shared__ u64 sa[K8_TILE + 8];
    __shared__ u32 split_s[2];
    const u64 o0 = (u64)blockIdx.x * K8_TILE;
    if (o0 >= m) return;
    const u64 pair0 = (o0 / (2 * width)) * (2 * width);
    const u64 a0g = pair0, a1g = min(pair0 + width, m), b1g = min(pair0 + 2 * width, m);
    const u32 na = (u32)(a1g - a0g), nb = (u32)(b1g - a1g);
    const u32 d0 = (u32)(o0 - pair0), d1 = (u32)min((u64)d0 + K8_TILE, (u64)na + nb);
    const u64 *A = src + a0g, *B = src + a1g;
    if (threadIdx.x < 2) {
        u32 d = threadIdx.x == 0 ? d0 : d1;
        auto gA = [&](u32 i) { return K::to_okey(A[i]); };
        auto gB = [&](u32 i) { return K::to_okey(B[i]); };
        u32 lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
        while (lo < hi) {
            u32 mid = (lo + hi) >> 1;
            if (gA(mid) <= gB(d - 1 - mid)) lo = mid + 1; else hi = mid;
        }
        split_s[threadIdx.x] = lo;
    }
    __syncthreads();
    const u32 ia0 = split_s[0], ia1 = split_s[1];
    const u32 ib0 = d0 - ia0, ib1 = d1 - ia1;
    const u32 la = ia1 - ia0, lb = ib1 - ib0;
    // smem: A part at [0, la), B part at [la, la+lb)
    for (u32 k = threadIdx.x; k < la; k += K8_THREADS) sa[k] = K::to_okey(A[ia0 + k]);
    for (u32 k = threadIdx.x; k < lb; k += K8_THREADS) sa[la + k] = K::to_okey(B[ib0 + k]);
    __syncthreads();
    const u32 tot = la + lb;
    const u32 dd = min(threadIdx.x * K8_IPT, tot);
    u32 lo = dd > lb ? dd - lb : 0, hi = dd < la ? dd : la;
    while (lo < hi) {
        u32 mid = (lo + hi) >> 1;
        if (sa[mid] <= sa[la + dd - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    u32 ia = lo, ib = dd - lo;
    u64 *out = dst + o0 + dd;
#pragma unroll
    for (int k = 0; k < K8_IPT; ++k) {
        if (dd + k >= tot) break;
        bool takeA;
        if (ia >= la) takeA = false;
        else if (ib >= lb) takeA = true;
        else takeA = sa[ia] <= sa[la + ib];
        u64 v = takeA ? sa[ia++] : sa[la + ib++];
        out[k] = K::from_okey(v);
    }
}

template <class K>
__global__ void k8_copy(const u64 *__restrict__ src, u64 *__restrict__ dst, u64 m) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x) dst[i] = src[i];
}

}  // namespace pcf
