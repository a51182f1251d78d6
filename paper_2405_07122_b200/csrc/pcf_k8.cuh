// pcf_k8.cuh -- K8: the GPU "Standard-Sort" for buckets too large for one
// CTA (Lemma 1 needs a worst-case O(n log n) sort,
// PAPER.md:235).  A comparison merge sort: K8_TILE-key tiles sorted in shared
// memory (bitonic), then log2(m / K8_TILE) merge passes.  Every pass first
// places the merge-path split of each output tile (k8_partition, one thread
// per tile), then merges tile by tile through shared memory with coalesced
// loads and stores (k8_merge).  Keys are compared as ordered u64 (IEEE
// totalOrder for f64, reading R11); the block sort writes ordered keys, the
// passes keep them, and the last pass writes the raw keys.  A bucket whose keys are all equal
// (k8_check; e.g. the duplicate-heavy bucket of config c3) is already sorted:
// its tiles are copied straight to the output and the passes are skipped.
#pragma once
#include "pcf_common.cuh"
#include "pcf_global.cuh"

namespace pcf {

#ifndef PCF_K8_THREADS
#define PCF_K8_THREADS 512
#endif
constexpr int K8_THREADS = PCF_K8_THREADS;
#ifndef PCF_K8_TILE
#define PCF_K8_TILE 4096
#endif
constexpr int K8_TILE = PCF_K8_TILE;
constexpr int K8_IPT = K8_TILE / K8_THREADS;   // 8
#ifndef PCF_K8_MTILE
#define PCF_K8_MTILE 1024
#endif
#ifndef PCF_K8_MTHREADS
#define PCF_K8_MTHREADS 256
#endif
constexpr int K8_MTILE = PCF_K8_MTILE;            // outputs of one merge CTA
constexpr int K8_MTHREADS = PCF_K8_MTHREADS;
constexpr int K8_MIPT = K8_MTILE / K8_MTHREADS;   // outputs per merge thread
constexpr int K8_MERGE_SMEM = K8_MTILE * 12;   // keys (+ key-value mode: u32 indices)
constexpr int K8_SORT_SMEM = 2 * K8_TILE * 8;


// Compare-exchange of two registers (ascending).
__device__ __forceinline__ void k8_cx(u64 &a, u64 &b) { const u64 x = a < b ? a : b; b = a < b ? b : a; a = x; }

// Merge-path split inside shared memory: number of keys taken from A (length
// la) among the first d outputs of merge(A, B) (A first among equal keys).
__device__ __forceinline__ u32 k8_split(const u64 *A, u32 la, const u64 *B, u32 lb, u32 d) {
    u32 lo = d > lb ? d - lb : 0, hi = d < la ? d : la;
    while (lo < hi) {
        const u32 mid = (lo + hi) >> 1;
        if (A[mid] <= B[d - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// K8_IPT consecutive outputs of merge(A, B) starting at A[ia], B[ib] into o[].
template <int NO>
__device__ __forceinline__ void k8_merge_seq(const u64 *A, u32 la, const u64 *B, u32 lb, u32 ia, u32 ib, u64 (&o)[NO]) {
    u64 xa = ia < la ? A[ia] : ~0ull, xb = ib < lb ? B[ib] : ~0ull;
#pragma unroll
    for (int k = 0; k < NO; ++k) {
        const bool ta = ib >= lb || (ia < la && xa <= xb);
        o[k] = ta ? xa : xb;
        if (ta) { ++ia; xa = ia < la ? A[ia] : ~0ull; }
        else { ++ib; xb = ib < lb ? B[ib] : ~0ull; }
    }
}

// Sorted K8_TILE-key tiles: 8 keys per thread sorted by a register network
// (Batcher odd-even merge sort, 19 comparators), then log2(K8_TILE / 8) levels
// of merge-path merges of sorted runs through shared memory (each thread
// emits 8 consecutive outputs).  Padding with the largest ordered key sorts last.
template <class K>
__device__ __forceinline__ void k8_sort_tile(u64 *k8_bs, const u64 *__restrict__ src, u64 *__restrict__ dst, u64 m, u64 base) {
    u64 *a = k8_bs, *b = k8_bs + K8_TILE;
    const u32 n = (u32)min((u64)K8_TILE, m - base);
    {
        u64 v[K8_IPT];
#pragma unroll
        for (int j = 0; j < K8_IPT; ++j) {
            const u32 k = threadIdx.x + j * K8_THREADS;
            v[j] = k < n ? src[base + k] : 0ull;
        }
#pragma unroll
        for (int j = 0; j < K8_IPT; ++j) {
            const u32 k = threadIdx.x + j * K8_THREADS;
            a[k] = k < n ? K::to_okey(v[j]) : ~0ull;
        }
    }
    __syncthreads();
    const u32 t0 = threadIdx.x * K8_IPT;
    u64 r[K8_IPT];
#pragma unroll
    for (int k = 0; k < K8_IPT; ++k) r[k] = a[t0 + ((k + threadIdx.x) & (K8_IPT - 1))];   // rotated: fewer bank conflicts
    // Batcher odd-even merge sort of each 8 registers
#define K8_BATCHER8(o)                                                                                   \
    k8_cx(r[o + 0], r[o + 1]); k8_cx(r[o + 2], r[o + 3]); k8_cx(r[o + 4], r[o + 5]); k8_cx(r[o + 6], r[o + 7]); \
    k8_cx(r[o + 0], r[o + 2]); k8_cx(r[o + 1], r[o + 3]); k8_cx(r[o + 4], r[o + 6]); k8_cx(r[o + 5], r[o + 7]); \
    k8_cx(r[o + 1], r[o + 2]); k8_cx(r[o + 5], r[o + 6]);                                                   \
    k8_cx(r[o + 0], r[o + 4]); k8_cx(r[o + 1], r[o + 5]); k8_cx(r[o + 2], r[o + 6]); k8_cx(r[o + 3], r[o + 7]); \
    k8_cx(r[o + 2], r[o + 4]); k8_cx(r[o + 3], r[o + 5]);                                                   \
    k8_cx(r[o + 1], r[o + 2]); k8_cx(r[o + 3], r[o + 4]); k8_cx(r[o + 5], r[o + 6]);
#pragma unroll
    for (int o = 0; o < K8_IPT; o += 8) { K8_BATCHER8(o) }
#undef K8_BATCHER8
    // the tested configuration: 512 threads x 8 keys (the 16-key and no-register-merge
    // variants measured slower in round 1 and were dropped rather than left untested)
    static_assert(K8_IPT == 8, "K8_IPT must be 8 (PCF_K8_TILE / PCF_K8_THREADS)");
    // 16 .. 32 * K8_IPT keys: the warp's ascending runs of 8 merged in registers by a
    // bitonic network (each stage: compare element i = K8_IPT * lane + q with its
    // mirror i ^ (k - 1), then half-cleaners i ^ j), lane shuffles, no shared memory
    {
        const u32 L = threadIdx.x & 31;
#pragma unroll
        for (u32 k = 16; k <= 32u * K8_IPT; k <<= 1) {
            if (k <= (u32)K8_IPT) {   // mirror inside the lane
#pragma unroll
                for (u32 q = 0; q < (u32)K8_IPT; ++q)
                    if (!(q & (k / 2))) k8_cx(r[q], r[q ^ (k - 1)]);
            } else {
                const bool lo = (L & (k / (2 * K8_IPT))) == 0;
                u64 p[K8_IPT];
#pragma unroll
                for (int q = 0; q < K8_IPT; ++q) p[q] = __shfl_xor_sync(0xffffffffu, r[K8_IPT - 1 - q], k / K8_IPT - 1);
#pragma unroll
                for (int q = 0; q < K8_IPT; ++q) r[q] = (lo == (p[q] < r[q])) ? p[q] : r[q];
            }
#pragma unroll
            for (u32 j = k / 4; j >= 1; j >>= 1) {
                if (j >= (u32)K8_IPT) {
                    const bool lo = (L & (j / K8_IPT)) == 0;
#pragma unroll
                    for (int q = 0; q < K8_IPT; ++q) {
                        const u64 p = __shfl_xor_sync(0xffffffffu, r[q], j / K8_IPT);
                        r[q] = (lo == (p < r[q])) ? p : r[q];
                    }
                } else {
#pragma unroll
                    for (u32 q = 0; q < (u32)K8_IPT; ++q)
                        if (!(q & j)) k8_cx(r[q], r[q | j]);
                }
            }
        }
    }
    constexpr u32 RUN0 = 32 * K8_IPT;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K8_IPT; ++k) a[t0 + k] = r[k];
    __syncthreads();
    u64 *sa = a, *sb = b;
    for (u32 run = RUN0; run < (u32)K8_TILE; run <<= 1) {
        const u32 p0 = (t0 / (2 * run)) * (2 * run), d = t0 - p0;
        const u64 *A = sa + p0, *B = sa + p0 + run;
        const u32 ia = k8_split(A, run, B, run, d);
        k8_merge_seq<K8_IPT>(A, run, B, run, ia, d - ia, r);
#pragma unroll
        for (int k = 0; k < K8_IPT; ++k) sb[t0 + k] = r[k];
        __syncthreads();
        u64 *tmp = sa; sa = sb; sb = tmp;
    }
    for (u32 k = threadIdx.x; k < n; k += K8_THREADS) dst[base + k] = m <= (u64)K8_TILE ? K::from_okey(sa[k]) : sa[k];
}

// Key-value mode: a K8_TILE tile of (ordered key, source index)
// pairs sorted by a shared-memory bitonic network on (key, index) -- equal keys in
// index order, so the block sort is stable; the merge passes (A first among equal
// keys) keep it stable.  Simpler than the keys-only register network: this mode is
// not the benchmarked path.
template <class K>
__device__ __forceinline__ void k8_sort_tile_pr(u64 *a, u32 *ai, const u64 *__restrict__ src, const u32 *__restrict__ isrc,
                                                u64 src_off, u64 *__restrict__ dst, u32 *__restrict__ idst, u64 m, u64 base) {
    const u32 n = (u32)min((u64)K8_TILE, m - base);
    for (u32 k = threadIdx.x; k < (u32)K8_TILE; k += K8_THREADS) {
        a[k] = k < n ? K::to_okey(src[base + k]) : ~0ull;
        ai[k] = k < n ? (isrc ? isrc[src_off + base + k] : (u32)(src_off + base + k)) : 0xffffffffu;
    }
    __syncthreads();
    for (u32 k = 2; k <= (u32)K8_TILE; k <<= 1) {
        for (u32 j = k >> 1; j > 0; j >>= 1) {
            for (u32 t = threadIdx.x; t < (u32)K8_TILE / 2; t += K8_THREADS) {
                const u32 lo = ((t / j) * 2 * j) + (t % j), hi = lo + j;
                const bool up = (lo & k) == 0;
                const u64 x = a[lo], y = a[hi];
                const u32 ix = ai[lo], iy = ai[hi];
                const bool gt = x > y || (x == y && ix > iy);
                if (gt == up) { a[lo] = y; a[hi] = x; ai[lo] = iy; ai[hi] = ix; }
            }
            __syncthreads();
        }
    }
    for (u32 k = threadIdx.x; k < n; k += K8_THREADS) {
        dst[base + k] = m <= (u64)K8_TILE ? K::from_okey(a[k]) : a[k];
        idst[base + k] = ai[k];
    }
}

// ------------------------------------------------------------------ segmented driver
// Every Standard-Sort bucket of > S_CAP keys (the fallback segments collected by
// k_items_to_nodes) is sorted by one chain of launches: k8_plan, k8_check,
// k8_blocksort, then a CUDA-graph WHILE loop of (k8_partition, k8_merge,
// k8_pass_end) over the merge passes of the largest segment.  Segment s has
// merges(s) = ceil(log2(ceil(m_s / K8_TILE))) passes; its block sort writes to
// out if merges(s) is even (tmp otherwise) and pass p writes to out iff
// merges(s) - 1 - p is even, so its last pass lands in out.  All kernels are
// grid-stride over the tiles of all segments and find their segment by a binary
// search over the per-segment tile prefix sums.
__device__ __forceinline__ u32 k8_merges(u64 m) {
    u32 r = 0;
    for (u64 w = K8_TILE; w < m; w *= 2) ++r;
    return r;
}
__device__ __forceinline__ u32 k8_seg_of(const u32 *__restrict__ pre, u32 nseg, u32 x) {   // last s with pre[s] <= x
    u32 lo = 0, hi = nseg - 1;
    while (lo < hi) {
        const u32 mid = (lo + hi + 1) >> 1;
        if (pre[mid] <= x) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Also sets the conditions of the tail graph: hseg (any segment: check + block
// sort), h (merge passes left: the pass loop) and hlog (pass log on: records).
__global__ void __launch_bounds__(1024) k8_plan(const DevCtx *__restrict__ c, cudaGraphConditionalHandle hseg,
                                                cudaGraphConditionalHandle h, cudaGraphConditionalHandle hlog) {
    pdl_entry();
    __shared__ u32 wsum[33];
    __shared__ u32 smax;
    __shared__ unsigned long long sbytes, skeys;
    Counters &C = *c->cnt;
    const u32 nseg = C.nan_flag ? 0u : C.fb_count;
    if (threadIdx.x == 0) { smax = 0; sbytes = 0; skeys = 0; }
    __syncthreads();
    u32 ct = 0, cm = 0, mx = 0;
    unsigned long long by = 0, ks = 0;
    for (u32 base = 0; base < nseg; base += 1024) {
        const u32 s = base + threadIdx.x;
        u32 nt = 0, nm = 0;
        if (s < nseg) {
            const u64 m = c->fb[s].m;
            nt = (u32)((m + K8_TILE - 1) / K8_TILE);
            nm = (u32)((m + K8_MTILE - 1) / K8_MTILE);
            mx = max(mx, k8_merges(m));
            by += 24ull * m;   // all-equal check (8 B/key) + block sort (16 B/key)
            ks += m;
            c->k8_flag[s] = 0;
        }
        u32 tot;
        const u32 et = block_excl_scan_1024(nt, wsum, tot);
        const u32 tt = tot;
        const u32 em = block_excl_scan_1024(nm, wsum, tot);
        if (s < nseg) { c->k8_tb[s] = ct + et; c->k8_mb[s] = cm + em; }
        ct += tt; cm += tot;
    }
    atomicMax(&smax, mx);
    atomicAdd(&sbytes, by);
    atomicAdd(&skeys, ks);
    __syncthreads();
    if (threadIdx.x == 0) {
        K8Plan pl;
        pl.nseg = nseg; pl.tiles = ct; pl.mtiles = cm; pl.max_merges = smax; pl.pass = 0; pl.pad = 0;
        C.k8 = pl;
        C.k8_bytes = sbytes;
        C.fb_keys = skeys;
        cudaGraphSetConditional(hseg, nseg > 0 ? 1u : 0u);
        (void)h;   // the pass loop's condition is set by k8_passes, after the all-equal check
        cudaGraphSetConditional(hlog, c->rec != nullptr && !C.nan_flag ? 1u : 0u);
    }
}

// "two distinct keys" flag per segment (an all-equal bucket, e.g. config c3's
// duplicate-heavy one, is already sorted: copied, no merge passes)
__global__ void __launch_bounds__(256) k8_check(const DevCtx *__restrict__ c) {
    pdl_entry();
    const K8Plan pl = c->cnt->k8;
    for (u32 t = blockIdx.x; t < pl.tiles; t += gridDim.x) {
        const u32 s = k8_seg_of(c->k8_tb, pl.nseg, t);
        const SegItem it = c->fb[s];
        const u64 *src = c->buf[it.src] + it.off;
        const u64 first = src[0];
        const u64 b0 = (u64)(t - c->k8_tb[s]) * K8_TILE, b1 = min((u64)it.m, b0 + K8_TILE);
        bool diff = false;
        for (u64 i = b0 + threadIdx.x; i < b1; i += blockDim.x) diff |= src[i] != first;
        if (__syncthreads_or(diff) && threadIdx.x == 0) atomicOr(&c->k8_flag[s], 1u);
    }
}

// Merge passes of the segments that hold two distinct keys (all-equal segments are
// copied by the block sort and need none): sets the pass loop's condition.
__global__ void __launch_bounds__(1024) k8_passes(const DevCtx *__restrict__ c, cudaGraphConditionalHandle h) {
    pdl_entry();
    __shared__ u32 smax;
    Counters &C = *c->cnt;
    if (threadIdx.x == 0) smax = 0;
    __syncthreads();
    u32 mx = 0;
    for (u32 s = threadIdx.x; s < C.k8.nseg; s += blockDim.x)
        if (c->k8_flag[s]) mx = max(mx, k8_merges(c->fb[s].m));
    atomicMax(&smax, mx);
    __syncthreads();
    if (threadIdx.x == 0) {
        C.k8.max_merges = smax;
        cudaGraphSetConditional(h, smax > 0 && !C.err_flag ? 1u : 0u);
    }
}

template <class K, bool PR>
__global__ void __launch_bounds__(K8_THREADS) k8_blocksort(const DevCtx *__restrict__ c) {
    pdl_entry();
    extern __shared__ __align__(16) u64 k8_bs[];   // 2 * K8_TILE keys (PR: K8_TILE keys + indices)
    const K8Plan pl = c->cnt->k8;
    u64 *out = c->buf[2], *tmp = c->buf[1];
    for (u32 t = blockIdx.x; t < pl.tiles; t += gridDim.x) {
        const u32 s = k8_seg_of(c->k8_tb, pl.nseg, t);
        const SegItem it = c->fb[s];
        const u64 *src = c->buf[it.src] + it.off;
        const u32 *isrc = PR ? c->ibuf[it.src] : nullptr;
        const u64 base = (u64)(t - c->k8_tb[s]) * K8_TILE;
        if (c->k8_flag[s] == 0) {   // all keys equal: already sorted, final position
            const u32 n = (u32)min((u64)K8_TILE, (u64)it.m - base);
            constexpr u32 NQ = PR ? (u32)((K8_TILE + K8_THREADS - 1) / K8_THREADS) : 1u;
            u32 g[NQ];
            if (PR) {   // indices first: ibuf[src] may be ibuf[2] itself
#pragma unroll
                for (u32 q = 0; q < NQ; ++q) {
                    const u32 k = threadIdx.x + q * K8_THREADS;
                    g[q] = k < n ? (isrc ? isrc[it.off + base + k] : (u32)(it.off + base + k)) : 0u;
                }
            }
            for (u32 k = threadIdx.x; k < n; k += K8_THREADS) out[it.off + base + k] = src[base + k];
            if (PR) {
#pragma unroll
                for (u32 q = 0; q < NQ; ++q) {
                    const u32 k = threadIdx.x + q * K8_THREADS;
                    if (k < n) c->ibuf[2][it.off + base + k] = g[q];
                }
            }
            continue;
        }
        __syncthreads();   // the previous tile's shared-memory stage is drained
        const bool to_out = (k8_merges(it.m) & 1u) == 0;
        u64 *dst0 = (to_out ? out : tmp) + it.off;
        if (PR) k8_sort_tile_pr<K>(k8_bs, reinterpret_cast<u32 *>(k8_bs + K8_TILE), src, isrc, it.off, dst0,
                                   c->ibuf[to_out ? 2 : 1] + it.off, it.m, base);
        else k8_sort_tile<K>(k8_bs, src, dst0, it.m, base);
    }
}

// Merge pass `pl.pass` (width K8_TILE << pass): the merge-path split of every
// output tile of every segment still merging (one thread per tile).
template <class K>
__global__ void k8_partition(const DevCtx *__restrict__ c) {
    pdl_entry();
    const K8Plan pl = c->cnt->k8;
    const u64 width = (u64)K8_TILE << pl.pass;
    for (u32 gt = blockIdx.x * blockDim.x + threadIdx.x; gt < pl.mtiles; gt += gridDim.x * blockDim.x) {
        const u32 s = k8_seg_of(c->k8_mb, pl.nseg, gt);
        const SegItem it = c->fb[s];
        const u32 mg = k8_merges(it.m);
        if (pl.pass >= mg || c->k8_flag[s] == 0) continue;
        const u32 t = gt - c->k8_mb[s];
        const u64 m = it.m;
        if (t == 0) atomicAdd(&c->cnt->k8_bytes, 16ull * m);
        const u64 *src = (((mg - pl.pass) & 1u) == 0 ? c->buf[2] : c->buf[1]) + it.off;   // = dst of pass - 1
        const u64 o0 = (u64)t * K8_MTILE;
        const u64 pair0 = (o0 / (2 * width)) * (2 * width);
        const u64 na = min(pair0 + width, m) - pair0, nb = min(pair0 + 2 * width, m) - min(pair0 + width, m);
        const u64 d = o0 - pair0;
        const u64 *A = src + pair0, *B = src + pair0 + na;
        u64 lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
        while (lo < hi) {   // first i with A[i] > B[d-1-i]  (A first among equal keys; ordered keys)
            const u64 mid = (lo + hi) >> 1;
            if (A[mid] <= B[d - 1 - mid]) lo = mid + 1; else hi = mid;
        }
        c->k8_sp[gt] = (u32)lo;
    }
}

template <class K, bool PR>
__global__ void __launch_bounds__(K8_MTHREADS) k8_merge(const DevCtx *__restrict__ c) {
    pdl_entry();
    extern __shared__ __align__(16) u64 k8_smem[];   // K8_MTILE input keys (+ PR: their indices)
    u64 *sa = k8_smem;
    u32 *sai = reinterpret_cast<u32 *>(k8_smem + K8_MTILE);
    const K8Plan pl = c->cnt->k8;
    const u64 width = (u64)K8_TILE << pl.pass;
    // persistent CTAs, each over a contiguous run of merge tiles: the segment record
    // is fetched once per segment, not once per 1024-output tile
    const u32 per = (pl.mtiles + gridDim.x - 1) / gridDim.x;
    const u32 g0 = blockIdx.x * per, g1 = min(pl.mtiles, g0 + per);
    u32 s = 0, s_beg = 1, s_end = 0, mg = 0;
    bool skip = true;
    // merge-path splits of the tile (sp[gt], sp[gt + 1]) are loaded one tile ahead
    u32 spa = g0 < g1 ? c->k8_sp[g0] : 0u, spb = g0 + 1 < g1 + 1 ? c->k8_sp[min(g0 + 1, pl.mtiles)] : 0u;
    SegItem it;
    it.off = 0; it.m = 0; it.level = 0; it.src = 0; it.kind = 0;
    for (u32 gt = g0; gt < g1; ++gt) {
        if (gt >= s_end || gt < s_beg) {   // entering a segment
            s = k8_seg_of(c->k8_mb, pl.nseg, gt);
            it = c->fb[s];
            mg = k8_merges(it.m);
            skip = pl.pass >= mg || c->k8_flag[s] == 0;   // uniform per CTA
            s_beg = c->k8_mb[s];
            s_end = s + 1 < pl.nseg ? c->k8_mb[s + 1] : pl.mtiles;
        }
        if (skip) {
            gt = s_end - 1;
            if (gt + 1 < g1) { spa = c->k8_sp[gt + 1]; spb = c->k8_sp[min(gt + 2, pl.mtiles)]; }
            continue;
        }
        const u32 cur_a = spa, cur_b = spb;
        if (gt + 1 < g1) { spa = cur_b; spb = c->k8_sp[min(gt + 2, pl.mtiles)]; }
        __syncthreads();   // the previous tile's stage is drained
        const u32 t = gt - s_beg;
        const u64 m = it.m;
        const bool last = pl.pass + 1 == mg;
        const u64 *src = (((mg - pl.pass) & 1u) == 0 ? c->buf[2] : c->buf[1]) + it.off;
        const bool to_out = ((mg - 1 - pl.pass) & 1u) == 0;
        u64 *dst = (to_out ? c->buf[2] : c->buf[1]) + it.off;
        const u32 *isrc = PR ? (to_out ? c->ibuf[1] : c->ibuf[2]) + it.off : nullptr;
        u32 *idst = PR ? (to_out ? c->ibuf[2] : c->ibuf[1]) + it.off : nullptr;
        const u64 o0 = (u64)t * K8_MTILE;
        const u64 pair0 = (o0 / (2 * width)) * (2 * width);
        const u64 na = min(pair0 + width, m) - pair0, nb = min(pair0 + 2 * width, m) - min(pair0 + width, m);
        const u64 d0 = o0 - pair0, d1 = min(d0 + K8_MTILE, na + nb);
        const u32 ia0 = cur_a;
        const u32 ia1 = d1 == na + nb ? (u32)na : cur_b;
        const u32 ib0 = (u32)(d0 - ia0), ib1 = (u32)(d1 - ia1);
        const u32 la = ia1 - ia0, lb = ib1 - ib0, tot = la + lb;
        const u64 *A = src + pair0, *B = src + pair0 + na;
        {   // all loads of a thread in flight at once, then the stores to shared memory
            u64 v[K8_MIPT];
#pragma unroll
            for (int j = 0; j < K8_MIPT; ++j) {
                const u32 k = threadIdx.x + j * K8_MTHREADS;
                v[j] = k < la ? A[ia0 + k] : k < tot ? B[ib0 + (k - la)] : 0ull;
            }
#pragma unroll
            for (int j = 0; j < K8_MIPT; ++j) {
                const u32 k = threadIdx.x + j * K8_MTHREADS;
                if (k < tot) sa[k] = v[j];
                if (PR && k < tot) sai[k] = k < la ? isrc[pair0 + ia0 + k] : isrc[pair0 + na + ib0 + (k - la)];
            }
        }
        __syncthreads();
        // per thread: K8_MIPT consecutive outputs from its own merge-path split, stored
        // straight from registers (a warp writes 32 x 32 contiguous bytes)
        const u32 dd = min(threadIdx.x * K8_MIPT, tot);
        const u32 ia = k8_split(sa, la, sa + la, lb, dd);
        u64 r[K8_MIPT];
        if (PR) {   // the same merge, by positions, so the indices follow their keys
            u32 ja = ia, jb = dd - ia;
#pragma unroll
            for (int k = 0; k < K8_MIPT; ++k) {
                const bool ta = jb >= lb || (ja < la && sa[ja] <= sa[la + jb]);
                const u32 sp = ta ? ja : la + jb;
                if (ta) ++ja; else ++jb;
                if (dd + k < tot) { r[k] = sa[sp]; idst[o0 + dd + k] = sai[sp]; }
            }
        } else {
            k8_merge_seq<K8_MIPT>(sa, la, sa + la, lb, ia, dd - ia, r);
        }
        u64 *outp = dst + o0 + dd;
#pragma unroll
        for (int k = 0; k < K8_MIPT; ++k) if (dd + k < tot) outp[k] = last ? K::from_okey(r[k]) : r[k];
    }
}

__global__ void k8_pass_end(const DevCtx *__restrict__ c, cudaGraphConditionalHandle h) {
    pdl_entry();
    K8Plan &pl = c->cnt->k8;
    pl.pass += 1;
    cudaGraphSetConditional(h, pl.pass < pl.max_merges && !c->cnt->err_flag ? 1u : 0u);
}

}  // namespace pcf
