// pcf_shard.cuh -- SURVEY.md 8(e) / 8(f) F3: the level-1 bucketing of a sort whose
// keys are sharded over R GPUs (one process per GPU, NCCL collectives between the
// calls, issued by the Python driver paper_2405_07122_b200/sharded.py).
//
// Alg. 1 is run on the WHOLE array of N keys, exactly as on one
// GPU: the level-1 node's x_min / x_max are the all-reduced shard
// extremes; its alpha sample positions (reading R3) are the single-GPU positions
// over [0, N), each drawn by the rank that holds it, and the per-bin sample counts
// are all-reduced, so b and T (R7) are the single-GPU ones; the
// bucket histogram H is the sum of the shards' histograms.
// Buckets are then dealt out to ranks as contiguous ranges [J_r, J_{r+1}) of about
// N / R keys, every rank sends its keys of range r to rank r in input (stable)
// order, and rank r sorts its range -- the rest of Alg. 1 for those buckets --
// with the single-GPU machinery (split rounds, K7, the radix Standard-Sort) at global offset
// O_r = sum_{j < J_r} H[j], so every deeper node has the single-GPU sampler key
// and record.  The concatenation of the ranks' outputs is the single-GPU output.
#pragma once
#include "pcf_common.cuh"
#include "pcf_global.cuh"

namespace pcf {

// Device state of one rank (one allocation, carved by shard_layout).
struct ShardState {
    long long mm[4];          // [0] min, [1] max (order-preserving int64 of the ordered key), [2] NaN flag
    unsigned long long range_off, range_m;   // this rank's range: global offset and key count
    unsigned long long send[64], recv[64];   // keys this rank sends to / receives from each rank
    u32 J[65];                // bucket range of rank r: [J[r], J[r+1])
    u32 degenerate;           // the global level-1 range is not in (0, inf) (R9/R10)
};
constexpr u32 SHARD_RMAX = 64;

__device__ __forceinline__ long long okey_to_i64(u64 k) { return (long long)(k ^ 0x8000000000000000ull); }
__device__ __forceinline__ u64 i64_to_okey(long long v) { return (u64)v ^ 0x8000000000000000ull; }

// Local extremes (ordered keys) and NaN flag of the shard.
template <class K>
__global__ void __launch_bounds__(256) k_shard_minmax(const u64 *__restrict__ x, u64 n, ShardState *S) {
    u64 mn = ~0ull, mx = 0;
    bool nan = false;
    for (u64 i = (u64)blockIdx.x * 256 + threadIdx.x; i < n; i += (u64)gridDim.x * 256) {
        const u64 raw = x[i];
        if (K::is_f64) nan |= (raw & 0x7fffffffffffffffull) > 0x7ff0000000000000ull;
        const u64 k = K::to_okey(raw);
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const u64 a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn; mx = b > mx ? b : mx;
    }
    const bool anynan = __syncthreads_or(nan);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&S->mm[0], okey_to_i64(mn));
        atomicMax(&S->mm[1], okey_to_i64(mx));
    }
    if (anynan && threadIdx.x == 0) atomicMax(&S->mm[2], 1ll);
}

// The level-1 model from the all-reduced extremes (every rank computes the same).
template <class K>
__device__ __forceinline__ bool shard_model(const ShardState *S, u32 beta, Model &md) {
    return make_model<K>(i64_to_okey(S->mm[0]), i64_to_okey(S->mm[1]), beta, md);
}

// Per-bin counts of the level-1 samples this rank holds: sample k sits at the
// single-GPU position p_k = sample_pos(node_key(seed, 1, 0), k, N) (R3, R4).
template <class K>
__global__ void __launch_bounds__(256) k_shard_counts(const u64 *__restrict__ x, u64 n, u64 off, u64 N, u32 alpha, u32 beta,
                                                      u64 seed, u32 flags, const ShardState *S, u32 *__restrict__ cnt) {
    Model md;
    if (!shard_model<K>(S, beta, md)) return;
    const u64 nk = node_key(seed, 1, 0);
    for (u64 k = (u64)blockIdx.x * 256 + threadIdx.x; k < alpha; k += (u64)gridDim.x * 256) {
        const u64 p = (flags & FLAG_SAMPLE_ALL) ? k : sample_pos(nk, k, N);
        if (p >= off && p < off + n) atomicAdd(&cnt[interval_index<K>(K::to_okey(x[p - off]), md)], 1u);
    }
}

// T[i] = floor(b_i * gamma / alpha) + 1 from the all-reduced counts (one CTA: the
// table is at most a few M entries; computed identically on every rank).
__global__ void __launch_bounds__(1024) k_shard_table(const u32 *__restrict__ cnt, u32 beta, u32 alpha, u32 gamma,
                                                      u32 *__restrict__ T) {
    __shared__ u32 wsum[33];
    const u64 nb = (u64)beta + 1;
    u32 carry = 0;
    for (u64 base0 = 0; base0 < nb; base0 += SCAN_CHUNK) {
        const u64 base = base0 + (u64)threadIdx.x * SCAN_ITEMS;
        u32 v[SCAN_ITEMS], sm = 0;
#pragma unroll
        for (int q = 0; q < SCAN_ITEMS; ++q) { v[q] = base + q < nb ? cnt[base + q + 1] : 0; sm += v[q]; }
        u32 total;
        u32 e = block_excl_scan_1024(sm, wsum, total) + carry;
#pragma unroll
        for (int q = 0; q < SCAN_ITEMS; ++q) {
            e += v[q];
            if (base + q < nb) T[base + q + 1] = bucket_of(e, alpha, gamma);
        }
        carry += total;
    }
}

// The shard's bucket histogram H[j], j = T[i(x)].
template <class K>
__global__ void __launch_bounds__(256) k_shard_hist(const u64 *__restrict__ x, u64 n, u32 beta, const ShardState *S,
                                                    const u32 *__restrict__ T, u32 *__restrict__ H) {
    Model md;
    if (!shard_model<K>(S, beta, md)) return;
    for (u64 i = (u64)blockIdx.x * 256 + threadIdx.x; i < n; i += (u64)gridDim.x * 256)
        atomicAdd(&H[__ldg(&T[interval_index<K>(K::to_okey(x[i]), md)])], 1u);
}

// Degenerate global range (R9/R10: not 0 < x_max - x_min < inf): every shard key
// counts in bucket 1, so the plan gives the whole array to rank 0, whose sort
// Standard-Sorts it (Alg. 1 on a degenerate node).
template <class K>
__global__ void k_shard_deg_hist(ShardState *S, u32 beta, u64 n, u32 *H) {
    Model md;
    const bool ok = shard_model<K>(S, beta, md);
    S->degenerate = ok ? 0u : 1u;
    if (!ok) H[1] = (u32)n;
}

// Plan of the exchange (one CTA, identical on every rank): global H = sum of the
// ranks' histograms; bucket ranges [J_r, J_{r+1}) cut where the running key count
// crosses r * N / R (never inside a bucket: Alg. 1 recurses per bucket); send and
// receive counts; this rank's range offset and size.  Hall: R rows of gamma + 2.
__global__ void __launch_bounds__(1024) k_shard_plan(const u32 *__restrict__ Hall, u32 R, u32 rank, u32 gamma, u64 N,
                                                     u32 *__restrict__ Hg, ShardState *S) {
    __shared__ unsigned long long wsum[33];
    __shared__ unsigned long long sendv[SHARD_RMAX], recvv[SHARD_RMAX];
    __shared__ u32 Jv[SHARD_RMAX + 1];
    __shared__ unsigned long long roff;
    const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const u64 ncol = (u64)gamma + 2;   // 1-based buckets 1..gamma+1
    if (threadIdx.x <= SHARD_RMAX) { Jv[threadIdx.x] = (u32)ncol; }
    if (threadIdx.x < SHARD_RMAX) { sendv[threadIdx.x] = 0; recvv[threadIdx.x] = 0; }
    if (threadIdx.x == 0) { Jv[0] = 1; roff = 0; }
    __syncthreads();
    // pass 1: global H and the cut points (first bucket j whose exclusive prefix >= r N / R)
    unsigned long long carry = 0;
    for (u64 base = 1; base < ncol; base += 1024) {
        const u64 j = base + threadIdx.x;
        u64 h = 0;
        if (j < ncol) {
            for (u32 r = 0; r < R; ++r) h += Hall[(u64)r * ncol + j];
            Hg[j] = (u32)h;
        }
        u64 xs = h;
        for (int o = 1; o < 32; o <<= 1) { const u64 y = __shfl_up_sync(0xffffffffu, xs, o); if (lane >= (u32)o) xs += y; }
        if (lane == 31) wsum[w] = xs;
        __syncthreads();
        if (w == 0) {
            u64 sv = wsum[lane], t2 = sv;
            for (int o = 1; o < 32; o <<= 1) { const u64 y = __shfl_up_sync(0xffffffffu, t2, o); if (lane >= (u32)o) t2 += y; }
            wsum[lane] = t2 - sv;
            if (lane == 31) wsum[32] = t2;
        }
        __syncthreads();
        const u64 ex = carry + wsum[w] + xs - h;   // keys in buckets < j
        if (j < ncol) {
            for (u32 r = 1; r < R; ++r) {          // bucket j starts range r iff ex < rN/R <= ex + h ... first j with ex + h > target
                const u64 target = (N * r) / R;
                if (ex <= target && target < ex + h) atomicMin(&Jv[r], (u32)(ex == target ? j : j + 1));
            }
        }
        carry += wsum[32];
        __syncthreads();
    }
    __syncthreads();
    if (threadIdx.x == 0)   // ranges are monotone and cover [1, ncol)
        for (u32 r = 1; r <= R; ++r) Jv[r] = r == R ? (u32)ncol : max(Jv[r], Jv[r - 1]);
    __syncthreads();
    // pass 2: send counts (this rank's keys per destination), receive counts (keys of
    // this rank's range per source rank), this rank's global offset
    unsigned long long off_part = 0;
    for (u64 j = 1 + threadIdx.x; j < ncol; j += 1024) {
        u32 dst = 0;
        while (dst + 1 < R && j >= Jv[dst + 1]) ++dst;
        const u32 mine = Hall[(u64)rank * ncol + j];
        if (mine) atomicAdd(&sendv[dst], (unsigned long long)mine);
        if (dst == rank)
            for (u32 r = 0; r < R; ++r) { const u32 v = Hall[(u64)r * ncol + j]; if (v) atomicAdd(&recvv[r], (unsigned long long)v); }
        if (j < Jv[rank]) off_part += Hg[j];
    }
    atomicAdd(&roff, off_part);
    __syncthreads();
    if (threadIdx.x < R) { S->send[threadIdx.x] = sendv[threadIdx.x]; S->recv[threadIdx.x] = recvv[threadIdx.x]; }
    if (threadIdx.x <= R) S->J[threadIdx.x] = Jv[threadIdx.x];
    if (threadIdx.x == 0) {
        S->range_off = roff;
        unsigned long long m = 0;
        for (u32 r = 0; r < R; ++r) m += recvv[r];
        S->range_m = m;
    }
}

// Stable partition of the shard's keys by destination rank (the rank whose bucket
// range holds j(x)): per tile of SH_TILE keys, per-destination counts (pass 1),
// an exclusive scan of the destination-major matrix, then the placement (pass 2)
// with ranks in input order (chunk by chunk per warp, MATCH inside a chunk).
constexpr int SH_WARPS = 8, SH_KPL = 16, SH_TILE = SH_WARPS * 32 * SH_KPL;   // 4096 keys

template <class K>
__device__ __forceinline__ u32 shard_dest(u64 okey, const Model &md, const u32 *__restrict__ T, const u32 *Jv, u32 R) {
    const u32 j = __ldg(&T[interval_index<K>(okey, md)]);
    u32 d = 0;
    while (d + 1 < R && j >= Jv[d + 1]) ++d;
    return d;
}

template <class K>
__global__ void __launch_bounds__(SH_WARPS * 32) k_shard_dcount(const u64 *__restrict__ x, u64 n, u32 beta, u32 R,
                                                                const ShardState *S, const u32 *__restrict__ T,
                                                                u32 *__restrict__ C, u32 ntiles) {
    __shared__ u32 cnt[SHARD_RMAX], Jv[SHARD_RMAX + 1];
    const u32 tile = blockIdx.x;
    if (threadIdx.x < R) cnt[threadIdx.x] = 0;
    if (threadIdx.x <= R) Jv[threadIdx.x] = S->J[threadIdx.x];
    __syncthreads();
    Model md;
    const bool ok = shard_model<K>(S, beta, md);
    const u64 k0 = (u64)tile * SH_TILE, k1 = min(n, k0 + SH_TILE);
    for (u64 i = k0 + threadIdx.x; i < k1; i += SH_WARPS * 32)
        atomicAdd(&cnt[ok ? shard_dest<K>(K::to_okey(x[i]), md, T, Jv, R) : 0u], 1u);
    __syncthreads();
    if (threadIdx.x < R) C[(u64)threadIdx.x * ntiles + tile] = cnt[threadIdx.x];
}

template <class K>
__global__ void __launch_bounds__(SH_WARPS * 32) k_shard_dscatter(const u64 *__restrict__ x, u64 n, u32 beta, u32 R,
                                                                  const ShardState *S, const u32 *__restrict__ T,
                                                                  const u32 *__restrict__ P, u32 ntiles, u64 *__restrict__ y) {
    __shared__ u32 wc[SH_WARPS][SHARD_RMAX], Jv[SHARD_RMAX + 1], base[SHARD_RMAX];
    const u32 tile = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x <= R) Jv[threadIdx.x] = S->J[threadIdx.x];
    for (u32 i = threadIdx.x; i < SH_WARPS * SHARD_RMAX; i += SH_WARPS * 32) wc[i / SHARD_RMAX][i % SHARD_RMAX] = 0;
    if (threadIdx.x < R) base[threadIdx.x] = P[(u64)threadIdx.x * ntiles + tile];
    __syncthreads();
    Model md;
    const bool ok = shard_model<K>(S, beta, md);
    const u64 k0 = (u64)tile * SH_TILE + (u64)w * 32 * SH_KPL;   // warp w: SH_KPL consecutive chunks
    u64 key[SH_KPL];
    u32 dr[SH_KPL];   // dest | in-warp rank << 8
#pragma unroll
    for (int q = 0; q < SH_KPL; ++q) {
        const u64 i = k0 + (u64)q * 32 + lane;
        const bool v = i < n;
        key[q] = v ? x[i] : 0ull;
        const u32 d = v ? (ok ? shard_dest<K>(K::to_okey(key[q]), md, T, Jv, R) : 0u) : 0xffu;
        const u32 peers = __match_any_sync(0xffffffffu, d);
        const u32 leader = __ffs(peers) - 1;
        u32 old = 0;
        if (v && lane == leader) { old = wc[w][d]; wc[w][d] = old + __popc(peers); }
        old = __shfl_sync(0xffffffffu, old, leader);
        dr[q] = d | ((old + __popc(peers & ((1u << lane) - 1u))) << 8);
        __syncwarp();
    }
    __syncthreads();
    if (threadIdx.x < R) {   // exclusive prefix over warps per destination
        u32 run = 0;
        for (u32 ww = 0; ww < SH_WARPS; ++ww) { const u32 v = wc[ww][threadIdx.x]; wc[ww][threadIdx.x] = run; run += v; }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < SH_KPL; ++q) {
        const u32 d = dr[q] & 0xffu;
        if (d != 0xffu) y[(u64)base[d] + wc[w][d] + (dr[q] >> 8)] = key[q];
    }
}

}  // namespace pcf
