// pcf_k8.cuh -- K8: the GPU "Standard-Sort" for buckets too large for one
// CTA (Lemma 1 needs a worst-case O(n log n) sort,
// PAPER.md:235).  A comparison merge sort: K8_TILE-key tiles sorted in shared
// memory (bitonic), then log2(m / K8_TILE) merge passes.  Every pass first
// places the merge-path split of each output tile (k8_partition, one thread
// per tile), then merges tile by tile through shared memory with coalesced
// loads and stores (k8_merge).  Keys are compared as ordered u64 (IEEE
// totalOrder for f64, reading R11).  A bucket whose keys are all equal
// (k8_check; e.g. the duplicate-heavy bucket of config c3) is already sorted:
// its tiles are copied straight to the output and the passes are skipped.
#pragma once
#include "pcf_common.cuh"

namespace pcf {

constexpr int K8_THREADS = 512;
constexpr int K8_TILE = 4096;
constexpr int K8_IPT = K8_TILE / K8_THREADS;   // 8
constexpr int K8_MERGE_SMEM = 2 * K8_TILE * 8;

// flag[0] = 1 if the bucket holds two different keys; flag[1] = first key
__global__ void __launch_bounds__(256) k8_check(const u64 *__restrict__ src, u64 m, u32 *__restrict__ flag) {
    const u64 first = src[0];
    bool diff = false;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x)
        diff |= src[i] != first;
    if (__syncthreads_or(diff) && threadIdx.x == 0) atomicOr(flag, 1u);
}

template <class K>
__global__ void __launch_bounds__(K8_THREADS) k8_blocksort(const u64 *__restrict__ src, u64 *__restrict__ dst,
                                                          u64 *__restrict__ out, u64 m, const u32 *__restrict__ flag) {
    __shared__ u64 a[K8_TILE];
    const u64 base = (u64)blockIdx.x * K8_TILE;
    const u32 n = (u32)min((u64)K8_TILE, m - base);
    if (*flag == 0) {   // all keys equal: already sorted, final position
        for (u32 k = threadIdx.x; k < n; k += K8_THREADS) out[base + k] = src[base + k];
        return;
    }
    for (u32 k = threadIdx.x; k < K8_TILE; k += K8_THREADS) a[k] = k < n ? K::to_okey(src[base + k]) : ~0ull;
    __syncthreads();
    // full bitonic sort (padding = max key sorts to the end)
    for (u32 k = 2; k <= (u32)K8_TILE; k <<= 1) {
        for (u32 j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (u32 t = threadIdx.x; t < K8_TILE / 2; t += K8_THREADS) {
                const u32 lo = ((t / j) * 2 * j) + (t % j), hi = lo + j;
                const bool up = (lo & k) == 0;
                const u64 x = a[lo], y = a[hi];
                if ((x > y) == up) { a[lo] = y; a[hi] = x; }
            }
            __syncthreads();
        }
    }
    for (u32 k = threadIdx.x; k < n; k += K8_THREADS) dst[base + k] = K::from_okey(a[k]);
}

// Merge-path split of output tile t (diagonal t*K8_TILE inside its run pair):
// sp[t] = number of keys taken from the first run.  One thread per tile.
template <class K>
__global__ void k8_partition(const u64 *__restrict__ src, u64 m, u64 width, u32 ntiles, u32 *__restrict__ sp,
                             const u32 *__restrict__ flag) {
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles || *flag == 0) return;
    const u64 o0 = (u64)t * K8_TILE;
    const u64 pair0 = (o0 / (2 * width)) * (2 * width);
    const u64 na = min(pair0 + width, m) - pair0, nb = min(pair0 + 2 * width, m) - min(pair0 + width, m);
    const u64 d = o0 - pair0;
    const u64 *A = src + pair0, *B = src + pair0 + na;
    u64 lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
    while (lo < hi) {   // first i with A[i] > B[d-1-i]  (A first among equal keys)
        const u64 mid = (lo + hi) >> 1;
        if (K::to_okey(A[mid]) <= K::to_okey(B[d - 1 - mid])) lo = mid + 1; else hi = mid;
    }
    sp[t] = (u32)lo;
}

template <class K>
__global__ void __launch_bounds__(K8_THREADS) k8_merge(const u64 *__restrict__ src, u64 *__restrict__ dst, u64 m, u64 width,
                                                      const u32 *__restrict__ sp, const u32 *__restrict__ flag) {
    extern __shared__ __align__(16) u64 k8_smem[];   // 2 * K8_TILE keys (dynamic: > 48 KB)
    u64 *sa = k8_smem, *so = k8_smem + K8_TILE;
    if (*flag == 0) return;
    const u32 t = blockIdx.x;
    const u64 o0 = (u64)t * K8_TILE;
    if (o0 >= m) return;
    const u64 pair0 = (o0 / (2 * width)) * (2 * width);
    const u64 na = min(pair0 + width, m) - pair0, nb = min(pair0 + 2 * width, m) - min(pair0 + width, m);
    const u64 d0 = o0 - pair0, d1 = min(d0 + K8_TILE, na + nb);
    const u32 ia0 = sp[t];
    const u32 ia1 = d1 == na + nb ? (u32)na : sp[t + 1];
    const u32 ib0 = (u32)(d0 - ia0), ib1 = (u32)(d1 - ia1);
    const u32 la = ia1 - ia0, lb = ib1 - ib0, tot = la + lb;
    const u64 *A = src + pair0, *B = src + pair0 + na;
    for (u32 k = threadIdx.x; k < la; k += K8_THREADS) sa[k] = K::to_okey(A[ia0 + k]);
    for (u32 k = threadIdx.x; k < lb; k += K8_THREADS) sa[la + k] = K::to_okey(B[ib0 + k]);
    __syncthreads();
    // per thread: K8_IPT consecutive outputs from its own merge-path split
    const u32 dd = min(threadIdx.x * K8_IPT, tot);
    u32 lo = dd > lb ? dd - lb : 0, hi = dd < la ? dd : la;
    while (lo < hi) {
        const u32 mid = (lo + hi) >> 1;
        if (sa[mid] <= sa[la + dd - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    u32 ia = lo, ib = dd - lo;
#pragma unroll
    for (int k = 0; k < K8_IPT; ++k) {
        if (dd + k < tot) {
            bool takeA;
            if (ia >= la) takeA = false;
            else if (ib >= lb) takeA = true;
            else takeA = sa[ia] <= sa[la + ib];
            so[dd + k] = takeA ? sa[ia++] : sa[la + ib++];
        }
    }
    __syncthreads();
    u64 *out = dst + o0;
    for (u32 k = threadIdx.x; k < tot; k += K8_THREADS) out[k] = K::from_okey(so[k]);
}

}  // namespace pcf
