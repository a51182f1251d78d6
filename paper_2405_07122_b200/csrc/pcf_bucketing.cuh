// One model-based bucketing step M_PCF with decoupled alpha, beta, gamma: the
// quantity measured by the paper's failure-frequency experiment (PAPER.md:516-519,
// §4.3, Fig. 4): Pr[exists j, |c_j| > delta] against Lemma 3.
// The sort itself fixes alpha = beta = gamma = delta = floor(m^{3/4}) and runs its
// own fused passes (pcf_global.cuh); this is the plain counting form of the same
// step, at the paper's experiment size (n = 10^6), with one key per thread-slot:
//   k_bk_minmax   x_min, x_max (ordered keys; NaN sorts past +-inf, R13)
//   k_bk_train    b: per-interval sample counts (i(x) of R6)
//   k_bk_scan     b_i = |{ k : i(a_k) <= i }| (inclusive prefix, one CTA)
//   k_bk_classify H[j] = |c_j|, j = floor(b_{i(x)} gamma / alpha) + 1 (R7)
//   k_bk_max      max_j |c_j|
#pragma once
#include "pcf_common.cuh"
#include "pcf_k7.cuh"

namespace pcf {

constexpr int BK_THREADS = 256;
constexpr u32 BK_SMEM_BINS = 8192;   // gamma + 1 up to this: block-private histogram in shared memory

// (warp_min_u64 / warp_max_u64 come from pcf_k7.cuh)

// mm[0] = min ordered key, mm[1] = max ordered key (pre-set to ~0 / 0 by the host)
__global__ void __launch_bounds__(BK_THREADS) k_bk_minmax(const u64 *__restrict__ x, u64 n, u64 *mm) {
    u64 lo = ~0ull, hi = 0;
    for (u64 i = (u64)blockIdx.x * BK_THREADS + threadIdx.x; i < n; i += (u64)gridDim.x * BK_THREADS) {
        const u64 k = KeyF64::to_okey(x[i]);
        lo = k < lo ? k : lo;
        hi = k > hi ? k : hi;
    }
    lo = warp_min_u64(lo);
    hi = warp_max_u64(hi);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(reinterpret_cast<unsigned long long *>(&mm[0]), lo);
        atomicMax(reinterpret_cast<unsigned long long *>(&mm[1]), hi);
    }
}

// b[i - 1] += 1 for every sample a_k = x[sample_pos(k)] with i = i(a_k)  (b pre-zeroed)
__global__ void __launch_bounds__(BK_THREADS) k_bk_train(const u64 *__restrict__ x, u64 n, u32 alpha, u32 beta,
                                                         u64 seed, const u64 *mm, u32 *b) {
    Model md;
    if (!make_model<KeyF64>(mm[0], mm[1], beta, md)) return;   // degenerate or NaN: the host reports it
    const u64 nk = node_key(seed, 1u, 0);                       // the root node's sampler stream (R3)
    for (u32 k = blockIdx.x * BK_THREADS + threadIdx.x; k < alpha; k += gridDim.x * BK_THREADS) {
        const u64 p = sample_pos(nk, k, n);
        atomicAdd(&b[interval_index<KeyF64>(KeyF64::to_okey(x[p]), md) - 1u], 1u);
    }
}

// in-place inclusive prefix sum of b[0, len) by one CTA of 1024 threads
__global__ void __launch_bounds__(1024) k_bk_scan(u32 *b, u32 len) {
    __shared__ u32 ws[32];
    const u32 t = threadIdx.x, chunk = (len + 1023u) / 1024u;
    const u32 s = min(t * chunk, len), e = min(s + chunk, len);
    u32 sum = 0;
    for (u32 i = s; i < e; ++i) sum += b[i];
    u32 inc = sum;   // block inclusive scan of the per-thread sums
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const u32 v = __shfl_up_sync(0xffffffffu, inc, o); if ((t & 31) >= (u32)o) inc += v; }
    if ((t & 31) == 31) ws[t >> 5] = inc;
    __syncthreads();
    if (t < 32) {
        u32 w = ws[t];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const u32 v = __shfl_up_sync(0xffffffffu, w, o); if (t >= (u32)o) w += v; }
        ws[t] = w;
    }
    __syncthreads();
    u32 run = inc - sum + ((t >> 5) ? ws[(t >> 5) - 1] : 0u);
    for (u32 i = s; i < e; ++i) { run += b[i]; b[i] = run; }
}

// H[j - 1] = |c_j|  (H pre-zeroed)
__global__ void __launch_bounds__(BK_THREADS) k_bk_classify(const u64 *__restrict__ x, u64 n, u32 alpha, u32 beta,
                                                            u32 gamma, const u64 *mm, const u32 *__restrict__ b, u32 *H) {
    __shared__ u32 sh[BK_SMEM_BINS];
    Model md;
    if (!make_model<KeyF64>(mm[0], mm[1], beta, md)) return;
    const u32 nbin = gamma + 1u;
    const bool local = nbin <= BK_SMEM_BINS;
    if (local) {
        for (u32 i = threadIdx.x; i < nbin; i += BK_THREADS) sh[i] = 0;
        __syncthreads();
    }
    for (u64 k = (u64)blockIdx.x * BK_THREADS + threadIdx.x; k < n; k += (u64)gridDim.x * BK_THREADS) {
        const u32 i = interval_index<KeyF64>(KeyF64::to_okey(x[k]), md);
        const u32 j = bucket_of(b[i - 1u], alpha, gamma);
        atomicAdd(local ? &sh[j - 1u] : &H[j - 1u], 1u);
    }
    if (local) {
        __syncthreads();
        for (u32 i = threadIdx.x; i < nbin; i += BK_THREADS)
            if (sh[i]) atomicAdd(&H[i], sh[i]);
    }
}

// mm[2] = max_j H[j]  (pre-zeroed)
__global__ void __launch_bounds__(BK_THREADS) k_bk_max(const u32 *__restrict__ H, u32 len, u64 *mm) {
    u64 m = 0;
    for (u32 i = blockIdx.x * BK_THREADS + threadIdx.x; i < len; i += gridDim.x * BK_THREADS) m = H[i] > m ? H[i] : m;
    m = warp_max_u64(m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(reinterpret_cast<unsigned long long *>(&mm[2]), m);
}

}  // namespace pcf
