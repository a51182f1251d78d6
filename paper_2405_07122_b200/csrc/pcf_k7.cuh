// pcf_k7.cuh -- K7: run the whole remaining Algorithm-1 subtree of a segment
// in shared memory, one CTA per task, persistent.
//
// A task is one of
//   K7_GROUP : buckets [jlo, jhi) of a global bucketing node whose keys lie,
//              in stable (Append) order, in one contiguous range.  The CTA
//              finishes the node's model-based bucketing for those buckets
//              (stable placement by j) and then processes
//              every bucket per Alg. 1 lines 160-167.
//   K7_NODE  : a segment that is a fresh Learned-Sort call (level L, offset o).
//   K7_SORT  : a bucket that Alg. 1 sends to Standard-Sort (|c_j| >= delta or
//              n < tau): sorted and written out.
// The task's keys are loaded once (HBM read), every deeper level runs in
// shared memory, and each finished bucket is written once to `out`.
//
// After every partition the children are classified in parallel (one thread
// or lane per bucket): buckets Alg. 1 sends to Standard-Sort with <= 64 keys
// are sorted by a key-parallel rank pass (each key counts the smaller keys of
// its own bucket -- O(|c_j|) per key); larger sorted buckets use a bitonic
// network; recursing buckets become warp items (<= WMAX keys, warp_node with an
// explicit DFS stack) or CTA items (> WMAX, cta_node).  Stable placement uses
// per-warp counters over warp-contiguous key ranges (CTA) or in-order 32-key
// chunks with __match_any_sync (warp), so every bucket keeps the Append order
// and the next level samples the same keys as the oracle (readings R4, R16).
#pragma once
#include "pcf_common.cuh"

namespace pcf {

struct WarpScratch {
    u16 cnt[WNB];    // per-bin sample counts -> b (inclusive prefix), 1-based
    u16 T[WNB];      // bucket table, 1-based; reused for the child kinds
    u16 H[WNB];      // bucket sizes, 0-based bucket index u = j-1
    u16 C[WNB];      // running cursors -> bucket ends
    u32 stack[WSTACK];
};

// Batched processing of all small recursing nodes of one level (<= BATCH_MAX_M
// keys each): flat key-, sample-, bin- and bucket-parallel steps for every node
// at once, one warp per group of whole nodes for the stable placement.
constexpr int BN_MAX = 128;          // nodes per batch
constexpr int BBINS = 3072;          // sum of (beta+2) (and of gamma+1) per batch
constexpr int BLIST_CAP = 1024;      // nodes per level list
constexpr u32 BATCH_MAX_M = 1024;
constexpr u32 BATCH_MIN_TAU = 16;    // batching needs nodes of >= 16 keys (bounds BBINS)
constexpr int LEAF_CAP = BBINS;

struct BatchSmem {
    u32 cnt[BBINS];          // per-bin sample counts; after the fit: u16 bucket cursors
    u16 T[BBINS];            // bucket table per node segment (1-based bins)
    u32 H[BBINS];            // bucket sizes per node segment
    u16 npos[BN_MAX], nm[BN_MAX], nP[BN_MAX], nal[BN_MAX];
    u32 nbin[BN_MAX + 1], nbkt[BN_MAX + 1], nsmp[BN_MAX + 1], nkey[BN_MAX + 1];
    unsigned long long nmin[BN_MAX], nmax[BN_MAX];
    double nxm[BN_MAX], nrr[BN_MAX];
    unsigned long long ndb[BN_MAX], ndh[BN_MAX];
    u32 ncnt[BN_MAX];        // pass log: nf | ns << 10 | nr << 20
    u8 ndeg[BN_MAX], nwarp[BN_MAX];
    u32 list[2][BLIST_CAP];  // level node lists: pos | m << 13
    u32 nlist[2];
    u32 nsub;                // nodes in the current sub-batch
};

struct BigItem {
    u32 pos, size, level, buf, kind;   // kind: 0 node, 1 sort
};

constexpr int BIG_CAP = 48;
constexpr int ITEM_CAP = NB_CAP + 64;
constexpr u32 RANK_MAX = 64;   // Standard-Sort buckets up to this size are rank-sorted key-parallel
enum : u32 { CK_EMPTY = 0, CK_RANK = 1, CK_RECURSE = 2, CK_BITONIC = 3, CK_NET = 4 };
constexpr u32 NET_MAX = 16;    // Standard-Sort buckets up to this size: one thread, register network

struct K7Smem {
    u64 A[S_CAP];
    u64 B[S_CAP];
    u16 U[S_CAP];            // bucket index per buffer position
    u32 Hc[NB_CAP + 1];      // CTA-level bucket sizes
    u32 Bs[NB_CAP + 1];      // CTA-level bucket starts (absolute buffer positions)
    u8 kindc[NB_CAP + 4];
    u32 items[ITEM_CAP];     // warp items: pos(13) | size(11) << 13 | kind(1) << 24 (0 node, 1 sort)
    u32 leaf[LEAF_CAP];      // network-sorted leaf buckets, class segments (<=4, <=8, <=16): pos | h << 16
    u32 nleaf[3], leafbase[3], leafcur[3];
    union {
        u16 wcnt[K7_WARPS][NB_CAP];               // CTA partition per-warp counters
        struct { u32 cnt[S_CAP / 8 + 8]; u32 T[S_CAP / 8 + 8]; } fit;   // CTA fit (beta+2 <= 863)
        WarpScratch w[K7_WARPS];
        BatchSmem b;
    } u;
    BigItem big[BIG_CAP];
    u64 red[2 * K7_WARPS];
    u32 scan_tmp[K7_WARPS + 1];
    K7Task task;
    u32 task_idx;
    u32 nbig;
    u32 nitems, nitems_lo, item_next;
    u32 gnode_delta, gnode_level;
    Model gmd;
    const u32 *gT;
    u32 *gH;
    long long prof_t;                       // PCF_FLAG_PROFILE bookkeeping (thread 0)
    unsigned long long prof[K7_PROF_SLOTS];
};

// K7 phase profiling (PCF_FLAG_PROFILE): thread 0 charges the cycles since the
// previous mark to slot `id`.  Slots: 0 claim, 1 load, 2 group classify,
// 3 group partition, 4 children: classify+lists, 5 children: networks,
// 6 children: rank, 7 children: warp items (incl. barrier wait), 8 cta_node
// fit+classify, 9 cta_node partition, 10 sort/node tasks, 11 tasks, 12 keys.
__device__ __forceinline__ void prof_mark(const DevCtx *c, K7Smem &S, int id) {
    if (c->k7_prof && threadIdx.x == 0) {
        long long t = clock64();
        S.prof[id] += (unsigned long long)(t - S.prof_t);
        S.prof_t = t;
    }
}

// ------------------------------------------------------------------ small helpers
__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ u32 warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ u32 lanemask_lt() {
    u32 r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}
__device__ __forceinline__ u32 next_pow2(u32 v) { return v <= 1 ? 1 : 1u << (32 - __clz(v - 1)); }

__device__ __forceinline__ u64 warp_min_u64(u64 v) {
    for (int o = 16; o > 0; o >>= 1) { u64 w = __shfl_xor_sync(0xffffffffu, v, o); v = w < v ? w : v; }
    return v;
}
__device__ __forceinline__ u64 warp_max_u64(u64 v) {
    for (int o = 16; o > 0; o >>= 1) { u64 w = __shfl_xor_sync(0xffffffffu, v, o); v = w > v ? w : v; }
    return v;
}
__device__ __forceinline__ u64 warp_sum_u64(u64 v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ u32 warp_sum_u32(u32 v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ u32 warp_incl_scan(u32 v) {
    u32 lane = lane_id();
    for (int o = 1; o < 32; o <<= 1) {
        u32 w = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= (u32)o) v += w;
    }
    return v;
}

// floor(m^{3/4}) for m <= S_CAP (m^3 < 2^40): float estimate + exact u64 fix-up (R5)
__device__ __forceinline__ u32 iroot34_small(u32 m) {
    u64 m3 = (u64)m * m * m;
    u32 c = (u32)sqrtf(sqrtf((float)m3));
    auto p4 = [](u64 x) { return x * x * x * x; };
    while (c > 0 && p4(c) > m3) --c;
    while (p4((u64)c + 1) <= m3) ++c;
    return c;
}

// ------------------------------------------------------------------ node record (pass log)
__device__ __forceinline__ void write_record(const DevCtx *c, u32 level, u32 alpha, u64 off, u64 m,
                                             u64 xmin_bits, u64 xmax_bits, u64 db, u64 dh, u32 nf,
                                             u32 ns, u32 nr) {
    unsigned long long slot = atomicAdd(c->rec_count, 1ull);
    if (slot < c->rec_cap) {
        NodeRec r;
        r.level = level; r.alpha = alpha; r.offset = off; r.m = m;
        r.xmin_bits = xmin_bits; r.xmax_bits = xmax_bits;
        r.digest_b = db; r.digest_h = dh;
        r.n_fallback = nf; r.n_small = ns; r.n_recurse = nr; r.reserved = 0;
        c->rec[slot] = r;
    }
}

// ------------------------------------------------------------------ sorting ("Standard-Sort", R2)
// Bitonic network over ordered keys; all merges ascending (first step of each
// stage compares i with its mirror), so virtual +inf padding never moves.
__device__ void warp_bitonic_smem(u64 *a, u32 n) {
    if (n <= 1) return;
    u32 P = next_pow2(n);
    u32 lane = lane_id();
    u32 lgP = 31 - __clz(P);
    for (u32 lk = 1; lk <= lgP; ++lk) {
        u32 k = 1u << lk, lh = lk - 1;
        for (u32 t = lane; t < (P >> 1); t += 32) {
            u32 blk = t >> lh, w = t & ((1u << lh) - 1);
            u32 lo = (blk << lk) + w, hi = (blk << lk) + k - 1 - w;
            if (hi < n) { u64 x = a[lo], y = a[hi]; if (x > y) { a[lo] = y; a[hi] = x; } }
        }
        __syncwarp();
        for (int lj = (int)lh - 1; lj >= 0; --lj) {
            u32 j = 1u << lj;
            for (u32 t = lane; t < (P >> 1); t += 32) {
                u32 lo = ((t >> lj) << (lj + 1)) + (t & (j - 1)), hi = lo + j;
                if (hi < n) { u64 x = a[lo], y = a[hi]; if (x > y) { a[lo] = y; a[hi] = x; } }
            }
            __syncwarp();
        }
    }
}

// Register bitonic for 16 < n <= 64: lane l holds elements l and l+32 (+inf padded).
template <class K>
__device__ void warp_sort64_write(const u64 *a, u32 n, u64 *gout_raw) {
    const u32 lane = lane_id();
    u64 v0 = lane < n ? a[lane] : ~0ull;
    u64 v1 = lane + 32 < n ? a[lane + 32] : ~0ull;
    const u32 kmax = n > 32 ? 64 : 32;
    for (u32 k = 2; k <= kmax; k <<= 1) {
        for (u32 j = k >> 1; j > 0; j >>= 1) {
            if (j == 32) {   // partner of element lane is lane+32 (same lane); k == 64 -> ascending
                const u64 lo = v0 < v1 ? v0 : v1, hi = v0 < v1 ? v1 : v0;
                v0 = lo; v1 = hi;
            } else {
                const u64 p0 = __shfl_xor_sync(0xffffffffu, v0, j);
                const bool low = (lane & j) == 0;
                const bool up0 = (lane & k) == 0, up1 = ((lane + 32) & k) == 0;
                v0 = (low == up0) ? (v0 < p0 ? v0 : p0) : (v0 > p0 ? v0 : p0);
                if (kmax == 64) {
                    const u64 p1 = __shfl_xor_sync(0xffffffffu, v1, j);
                    v1 = (low == up1) ? (v1 < p1 ? v1 : p1) : (v1 > p1 ? v1 : p1);
                }
            }
        }
    }
    if (lane < n) gout_raw[lane] = K::from_okey(v0);
    if (lane + 32 < n) gout_raw[lane + 32] = K::from_okey(v1);
}

// Whole segment a[0, n) sorted by one warp and written (raw keys) to gout[0, n).
template <class K>
__device__ void warp_sort_write(u64 *a, u32 n, u64 *gout_raw) {
    const u32 lane = lane_id();
    if (n <= RANK_MAX) {   // rank sort: each key counts the keys before it in sorted order
        for (u32 i = lane; i < n; i += 32) {
            u64 v = a[i];
            u32 r = 0;
            for (u32 j = 0; j < n; ++j) { u64 w = a[j]; r += (w < v) | ((w == v) & (j < i)); }
            gout_raw[r] = K::from_okey(v);
        }
    } else if (n <= 64) {
        warp_sort64_write<K>(a, n, gout_raw);
    } else {
        warp_bitonic_smem(a, n);
        for (u32 k = lane; k < n; k += 32) gout_raw[k] = K::from_okey(a[k]);
    }
    __syncwarp();
}

template <class K>
__device__ void cta_sort_write(u64 *a, u32 n, u64 *gout_raw) {
    if (n > 1) {
        u32 P = next_pow2(n);
        u32 lgP = 31 - __clz(P);
        for (u32 lk = 1; lk <= lgP; ++lk) {
            u32 k = 1u << lk, lh = lk - 1;
            for (u32 t = threadIdx.x; t < (P >> 1); t += K7_THREADS) {
                u32 blk = t >> lh, w = t & ((1u << lh) - 1);
                u32 lo = (blk << lk) + w, hi = (blk << lk) + k - 1 - w;
                if (hi < n) { u64 x = a[lo], y = a[hi]; if (x > y) { a[lo] = y; a[hi] = x; } }
            }
            __syncthreads();
            for (int lj = (int)lh - 1; lj >= 0; --lj) {
                u32 j = 1u << lj;
                for (u32 t = threadIdx.x; t < (P >> 1); t += K7_THREADS) {
                    u32 lo = ((t >> lj) << (lj + 1)) + (t & (j - 1)), hi = lo + j;
                    if (hi < n) { u64 x = a[lo], y = a[hi]; if (x > y) { a[lo] = y; a[hi] = x; } }
                }
                __syncthreads();
            }
        }
    }
    for (u32 k = threadIdx.x; k < n; k += K7_THREADS) gout_raw[k] = K::from_okey(a[k]);
    __syncthreads();
}

// One thread sorts a whole bucket of h <= N keys (Y[s, s+h)) in registers with
// a fully unrolled bitonic network (+inf padded) and writes it to gout[s, s+h).
// Predicated on `act`; the warp executes the network once for up to 32 buckets.
template <int N>
struct CeilLog2 { static constexpr int v = N <= 1 ? 0 : 1 + CeilLog2<(N + 1) / 2>::v; };
template <>
struct CeilLog2<1> { static constexpr int v = 0; };

template <class K, int N>
__device__ __forceinline__ void net_sort_write(bool act, const u64 *Y, u32 s, u32 h, u64 *gout) {
    u64 v[N];
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = (act && (u32)i < h) ? Y[s + i] : ~0ull;
    // Batcher's merge exchange (Knuth, TAOCP 5.2.2 Algorithm M); every step ascending
    constexpr int T = CeilLog2<N>::v;
#pragma unroll
    for (int pe = T - 1; pe >= 0; --pe) {
        const int p = 1 << pe;
#pragma unroll
        for (int k = 0; k <= T - 1 - pe; ++k) {
            const int d = k == 0 ? p : (1 << (T - k)) - p;
            const int r = k == 0 ? 0 : p;
#pragma unroll
            for (int i = 0; i < N; ++i) {
                if (i + d < N && (i & p) == r) {
                    const u64 a = v[i], b = v[i + d];
                    v[i] = a < b ? a : b;
                    v[i + d] = a < b ? b : a;
                }
            }
        }
    }
    if (act) {
#pragma unroll
        for (int i = 0; i < N; ++i)
            if ((u32)i < h) gout[s + i] = K::from_okey(v[i]);
    }
}

// Size class of a network-sorted leaf bucket: 0 (<= 4 keys), 1 (<= 8), 2 (<= 16).
__device__ __forceinline__ u32 net_class(u32 h) { return h <= 4 ? 0u : h <= 8 ? 1u : 2u; }

template <class K>
__device__ __forceinline__ void net_sort_class(u32 cls, bool act, const u64 *Y, u32 s, u32 h, u64 *gout) {
    if (cls == 0) net_sort_write<K, 4>(act, Y, s, h, gout);
    else if (cls == 1) net_sort_write<K, 8>(act, Y, s, h, gout);
    else net_sort_write<K, 16>(act, Y, s, h, gout);
}

// Rank-sort the key at buffer position i of a small bucket [s, e) and write it.
template <class K>
__device__ __forceinline__ void rank_place(const u64 *Y, u32 i, u32 s, u32 e, u64 *gout) {
    const u64 v = Y[i];
    u32 r = 0;
    for (u32 j = s; j < e; ++j) { u64 w = Y[j]; r += (w < v) | ((w == v) & (j < i)); }
    gout[s + r] = K::from_okey(v);
}

// ------------------------------------------------------------------ warp-level Alg. 1
// Learned-Sort of the segment X[p, p+m) (m <= WMAX) at level L, global offset
// gbase + p, and all its descendants; finished buckets go to gout[pos].
// Stack entries: pos(13) | size(11) | depth(4) | buf(1).
template <class K>
__device__ void warp_node(const DevCtx *c, K7Smem &S, u32 buf0, u32 p0, u32 m0, u32 L0, u64 gbase,
                          u64 *gout) {
    WarpScratch &ws = S.u.w[warp_id()];
    const u32 lane = lane_id();
    const u32 tau = c->tau;
    const bool sample_all = (c->flags & FLAG_SAMPLE_ALL) != 0;
    const bool logging = c->rec != nullptr;
    if (lane == 0) ws.stack[0] = p0 | (m0 << 13) | (buf0 << 28);
    u32 sp = 1;
    __syncwarp();
    while (sp > 0) {
        const u32 e = ws.stack[--sp];
        __syncwarp();
        const u32 p = e & 0x1fffu, m = (e >> 13) & 0x7ffu, d = (e >> 24) & 0xfu, bi = e >> 28;
        u64 *X = bi ? S.B : S.A;
        u64 *Y = bi ? S.A : S.B;
        const u32 L = L0 + d;
        if (m < tau) { warp_sort_write<K>(X + p, m, gout + p); continue; }
        // x_min, x_max over the segment
        u64 mn = ~0ull, mx = 0;
        for (u32 k = lane; k < m; k += 32) { u64 v = X[p + k]; mn = v < mn ? v : mn; mx = v > mx ? v : mx; }
        mn = warp_min_u64(mn);
        mx = warp_max_u64(mx);
        Model md;
        const u32 P = iroot34_small(m);
        if (!make_model<K>(mn, mx, P, md)) { warp_sort_write<K>(X + p, m, gout + p); continue; }   // R9/R10
        const u32 alpha = sample_all ? m : P, beta = P, gamma = P, delta = P;
        const u32 ng = gamma + 1;
        for (u32 i = lane; i <= beta + 1; i += 32) ws.cnt[i] = 0;
        for (u32 u = lane; u < ng; u += 32) ws.H[u] = 0;
        __syncwarp();
        // sample (R3, R4) and count per interval
        const u64 nkey = node_key(c->seed, L, gbase + p);
        for (u32 k0 = 0; k0 < alpha; k0 += 32) {
            const u32 k = k0 + lane;
            const bool act = k < alpha;
            u32 i = 0xffffffffu;
            if (act) i = interval_index<K>(X[p + (sample_all ? k : (u32)sample_pos(nkey, k, m))], md);
            const u32 peers = __match_any_sync(0xffffffffu, i);
            if (act && (peers & lanemask_lt()) == 0) ws.cnt[i] += (u16)__popc(peers);
            __syncwarp();
        }
        // b = inclusive prefix of the counts, T = floor(b*gamma/alpha)+1
        u64 db = 0;
        {
            const u32 nb = beta + 1;
            const u32 per = (nb + 31) / 32;
            const u32 s0 = 1 + lane * per, s1 = min(s0 + per, nb + 1);
            u32 loc = 0;
            for (u32 i = s0; i < s1; ++i) loc += ws.cnt[i];
            u32 run = warp_incl_scan(loc) - loc;
            for (u32 i = s0; i < s1; ++i) {
                run += ws.cnt[i];
                ws.cnt[i] = (u16)run;
                ws.T[i] = (u16)bucket_of(run, alpha, gamma);
                if (logging) db += digest_term(i, run);
            }
        }
        __syncwarp();
        // classify every key: u = T[i(x)] - 1; histogram H[u]
        for (u32 k0 = 0; k0 < m; k0 += 32) {
            const u32 k = k0 + lane;
            const bool act = k < m;
            u32 u = 0xffffffffu;
            if (act) { u = ws.T[interval_index<K>(X[p + k], md)] - 1u; S.U[p + k] = (u16)u; }
            const u32 peers = __match_any_sync(0xffffffffu, u);
            if (act && (peers & lanemask_lt()) == 0) ws.H[u] += (u16)__popc(peers);
            __syncwarp();
        }
        // exclusive prefix of H -> cursors
        {
            const u32 perg = (ng + 31) / 32;
            const u32 g0 = lane * perg, g1 = min(g0 + perg, ng);
            u32 locg = 0;
            for (u32 u = g0; u < g1; ++u) locg += ws.H[u];
            u32 rg = warp_incl_scan(locg) - locg;
            for (u32 u = g0; u < g1; ++u) { ws.C[u] = (u16)rg; rg += ws.H[u]; }
        }
        __syncwarp();
        // stable scatter (Append in index order)
        for (u32 k0 = 0; k0 < m; k0 += 32) {
            const u32 k = k0 + lane;
            const bool act = k < m;
            const u32 u = act ? (u32)S.U[p + k] : 0xffffffffu;
            const u32 peers = __match_any_sync(0xffffffffu, u);
            const u32 base = act ? ws.C[u] : 0;
            __syncwarp();
            if (act) {
                const u32 rank = __popc(peers & lanemask_lt());
                Y[p + base + rank] = X[p + k];
                if (rank == 0) ws.C[u] = (u16)(base + __popc(peers));
            }
            __syncwarp();
        }
        // ws.C[u] = end of bucket u (relative to p).  Node record (pass log).
        if (logging) {
            u32 nf = 0, ns = 0, nr = 0;
            u64 dh = 0;
            for (u32 u = lane; u < ng; u += 32) {
                const u32 h = ws.H[u];
                dh += digest_term(u + 1, h);
                if (h) { if (h >= delta) nf++; else if (h < tau) ns++; else nr++; }
            }
            db = warp_sum_u64(db);
            dh = warp_sum_u64(dh);
            nf = warp_sum_u32(nf); ns = warp_sum_u32(ns); nr = warp_sum_u32(nr);
            if (lane == 0)
                write_record(c, L, alpha, gbase + p, m, K::from_okey(mn), K::from_okey(mx), db, dh, nf, ns, nr);
            if (L == 1 && c->l1_b) {
                for (u32 i = lane; i <= beta && i < c->l1_cap; i += 32) c->l1_b[i] = ws.cnt[i + 1];
                for (u32 u = lane; u < ng && u < c->l1_cap; u += 32) c->l1_h[u] = ws.H[u];
            }
        }
        // children, one lane per bucket
        for (u32 u0 = 0; u0 < ng; u0 += 32) {
            const u32 u = u0 + lane;
            u32 kind = CK_EMPTY, h = 0, s = 0;
            if (u < ng) {
                h = ws.H[u];
                s = ws.C[u] - h;
                // small leaves: rank pass for nodes with few buckets, class networks otherwise
                if (h) kind = (h >= delta || h < tau) ? (h <= NET_MAX ? (ng < 64 ? CK_RANK : CK_NET) : CK_BITONIC)
                                                      : CK_RECURSE;
                ws.T[u] = (u16)kind;
                if (kind == CK_RANK)
                    for (u32 i = s; i < s + h; ++i) S.U[p + i] = (u16)u;
            }
            const u32 rmask = __ballot_sync(0xffffffffu, kind == CK_RECURSE);
            if (kind == CK_RECURSE) {
                const u32 slot = sp + __popc(rmask & lanemask_lt());
                if (slot < WSTACK && d + 1 < 16) ws.stack[slot] = (p + s) | (h << 13) | ((d + 1) << 24) | ((bi ^ 1u) << 28);
                else atomicOr(c->err_flag, 2u);
            }
            sp = min(sp + __popc(rmask), (u32)WSTACK);
            u32 bmask = __ballot_sync(0xffffffffu, kind == CK_BITONIC);
            while (bmask) {
                const int b = __ffs(bmask) - 1;
                bmask &= bmask - 1;
                const u32 hs = __shfl_sync(0xffffffffu, h, b), ss = __shfl_sync(0xffffffffu, s, b);
                warp_sort_write<K>(Y + p + ss, hs, gout + p + ss);
            }
        }
        __syncwarp();
        if (ng < 64) {
            // leaf buckets of <= 16 keys: key-parallel rank sort (each key scans its own bucket)
            for (u32 i = lane; i < m; i += 32) {
                const u32 u = S.U[p + i];
                if (u < ng && ws.T[u] == CK_RANK) {
                    const u32 en = ws.C[u], st = en - ws.H[u];
                    if (i >= st && i < en) rank_place<K>(Y + p, i, st, en, gout + p);
                }
            }
        } else {
            // leaf buckets of <= 16 keys: compacted per size class (list in ws.cnt),
            // one lane per bucket, register network
#pragma unroll 1
            for (u32 cls = 0; cls < 3; ++cls) {
                u32 nl = 0;
                for (u32 u0 = 0; u0 < ng; u0 += 32) {
                    const u32 u = u0 + lane;
                    const bool in = u < ng && ws.T[u] == CK_NET && net_class(ws.H[u]) == cls;
                    const u32 mk = __ballot_sync(0xffffffffu, in);
                    if (in) ws.cnt[nl + __popc(mk & lanemask_lt())] = (u16)u;
                    nl += __popc(mk);
                }
                __syncwarp();
                for (u32 i = lane; i < nl; i += 32) {
                    const u32 u = ws.cnt[i], h = ws.H[u];
                    net_sort_class<K>(cls, true, Y + p, ws.C[u] - h, h, gout + p);
                }
                __syncwarp();
            }
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ CTA-level primitives
__device__ __forceinline__ u64 cta_reduce_min(K7Smem &S, u64 v) {
    v = warp_min_u64(v);
    if (lane_id() == 0) S.red[warp_id()] = v;
    __syncthreads();
    if (warp_id() == 0) {
        u64 w = lane_id() < K7_WARPS ? S.red[lane_id()] : ~0ull;
        w = warp_min_u64(w);
        if (lane_id() == 0) S.red[K7_WARPS] = w;
    }
    __syncthreads();
    u64 r = S.red[K7_WARPS];
    __syncthreads();
    return r;
}
__device__ __forceinline__ u64 cta_reduce_max(K7Smem &S, u64 v) {
    v = warp_max_u64(v);
    if (lane_id() == 0) S.red[warp_id()] = v;
    __syncthreads();
    if (warp_id() == 0) {
        u64 w = lane_id() < K7_WARPS ? S.red[lane_id()] : 0ull;
        w = warp_max_u64(w);
        if (lane_id() == 0) S.red[K7_WARPS] = w;
    }
    __syncthreads();
    u64 r = S.red[K7_WARPS];
    __syncthreads();
    return r;
}
__device__ __forceinline__ u64 cta_reduce_sum64(K7Smem &S, u64 v) {
    v = warp_sum_u64(v);
    if (lane_id() == 0) S.red[warp_id()] = v;
    __syncthreads();
    if (warp_id() == 0) {
        u64 w = lane_id() < K7_WARPS ? S.red[lane_id()] : 0ull;
        w = warp_sum_u64(w);
        if (lane_id() == 0) S.red[K7_WARPS] = w;
    }
    __syncthreads();
    u64 r = S.red[K7_WARPS];
    __syncthreads();
    return r;
}

// exclusive scan of a[0..n) (n <= 2*K7_THREADS) in place; returns the total
__device__ u32 cta_excl_scan(K7Smem &S, u32 *a, u32 n) {
    u32 t = threadIdx.x;
    u32 i0 = 2 * t, i1 = 2 * t + 1;
    u32 v0 = i0 < n ? a[i0] : 0, v1 = i1 < n ? a[i1] : 0;
    u32 loc = v0 + v1;
    u32 incl = warp_incl_scan(loc);
    if (lane_id() == 31) S.scan_tmp[warp_id()] = incl;
    __syncthreads();
    if (warp_id() == 0) {
        u32 w = lane_id() < K7_WARPS ? S.scan_tmp[lane_id()] : 0;
        u32 wi = warp_incl_scan(w);
        if (lane_id() < K7_WARPS) S.scan_tmp[lane_id()] = wi - w;
        if (lane_id() == K7_WARPS - 1) S.scan_tmp[K7_WARPS] = wi;
    }
    __syncthreads();
    u32 base = S.scan_tmp[warp_id()] + incl - loc;
    if (i0 < n) a[i0] = base;
    if (i1 < n) a[i1] = base + v0;
    u32 total = S.scan_tmp[K7_WARPS];
    __syncthreads();
    return total;
}

// Stable partition X[p..p+m) -> Y[p..p+m) by U[p+k] in [0, nb): warp w owns a
// contiguous range of <= 512 keys; pass 1 ranks each key inside its warp
// (__match_any_sync per 32-key chunk, per-warp counters) and keeps bucket and
// rank in a register; after the cross-warp prefix every key is placed directly.
// Hc = bucket sizes, Bs = absolute bucket starts.
constexpr int PART_CH = S_CAP / K7_WARPS / 32;   // <= 16 chunks per warp
__device__ void cta_partition(K7Smem &S, const u64 *X, u64 *Y, u32 p, u32 m, u32 nb) {
    const u32 w = warp_id(), lane = lane_id();
    const u32 R = (m + K7_WARPS - 1) / K7_WARPS;
    const u32 r0 = p + min(w * R, m), r1 = p + min(w * R + R, m);
    const u32 nch = (r1 - r0 + 31) / 32;
    for (u32 u = lane; u < nb; u += 32) S.u.wcnt[w][u] = 0;
    __syncwarp();
    u32 pk[PART_CH];
#pragma unroll
    for (int q = 0; q < PART_CH; ++q) {
        pk[q] = 0xffffffffu;
        if ((u32)q < nch) {   // warp-uniform
            const u32 k = r0 + q * 32 + lane;
            const bool act = k < r1;
            const u32 u = act ? (u32)S.U[k] : 0xffffffffu;
            const u32 peers = __match_any_sync(0xffffffffu, u);
            const u32 leader = __ffs(peers) - 1;
            u32 old = 0;
            if (act && lane == leader) { old = S.u.wcnt[w][u]; S.u.wcnt[w][u] = (u16)(old + __popc(peers)); }
            old = __shfl_sync(0xffffffffu, old, leader);
            if (act) pk[q] = u | ((old + __popc(peers & lanemask_lt())) << 16);
            __syncwarp();
        }
    }
    __syncthreads();
    // bucket totals, their exclusive scan and the per-warp offsets in one step
    // (thread t owns buckets 2t and 2t+1; nb <= NB_CAP = 2 * K7_THREADS)
    {
        const u32 u0 = 2 * threadIdx.x, u1 = u0 + 1;
        u32 t0 = 0, t1 = 0;
        if (u0 < nb) for (u32 ww = 0; ww < K7_WARPS; ++ww) t0 += S.u.wcnt[ww][u0];
        if (u1 < nb) for (u32 ww = 0; ww < K7_WARPS; ++ww) t1 += S.u.wcnt[ww][u1];
        const u32 loc = t0 + t1;
        const u32 incl = warp_incl_scan(loc);
        if (lane == 31) S.scan_tmp[w] = incl;
        __syncthreads();
        u32 wbase = 0;
        for (u32 ww = 0; ww < w; ++ww) wbase += S.scan_tmp[ww];
        u32 run = p + wbase + incl - loc;
        if (u0 < nb) {
            S.Hc[u0] = t0; S.Bs[u0] = run;
            for (u32 ww = 0; ww < K7_WARPS; ++ww) { u32 cc = S.u.wcnt[ww][u0]; S.u.wcnt[ww][u0] = (u16)run; run += cc; }
        }
        if (u1 < nb) {
            S.Hc[u1] = t1; S.Bs[u1] = run;
            for (u32 ww = 0; ww < K7_WARPS; ++ww) { u32 cc = S.u.wcnt[ww][u1]; S.u.wcnt[ww][u1] = (u16)run; run += cc; }
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PART_CH; ++q) {
        if (pk[q] != 0xffffffffu) {
            const u32 k = r0 + q * 32 + lane;
            Y[S.u.wcnt[w][pk[q] & 0xffffu] + (pk[q] >> 16)] = X[k];
        }
    }
    __syncthreads();
}

// ------------------------------------------------------------------ leaf lists (class segments)
// Pass 1 counts network-sorted leaf buckets per size class, leaf_segments() lays
// the classes out in S.leaf, pass 2 appends.  Called with warp-uniform trip counts.
__device__ __forceinline__ void leaf_count(K7Smem &S, bool is_net, u32 h) {
#pragma unroll
    for (u32 cls = 0; cls < 3; ++cls) {
        const u32 mk = __ballot_sync(0xffffffffu, is_net && net_class(h) == cls);
        if (mk && lane_id() == (u32)(__ffs(mk) - 1)) atomicAdd(&S.nleaf[cls], (u32)__popc(mk));
    }
}
__device__ __forceinline__ void leaf_segments(const DevCtx *c, K7Smem &S) {
    if (threadIdx.x == 0) {
        S.leafbase[0] = 0; S.leafbase[1] = S.nleaf[0]; S.leafbase[2] = S.nleaf[0] + S.nleaf[1];
        S.leafcur[0] = S.leafcur[1] = S.leafcur[2] = 0;
        if (S.nleaf[0] + S.nleaf[1] + S.nleaf[2] > (u32)LEAF_CAP) atomicOr(c->err_flag, 2u);
    }
}
__device__ __forceinline__ void leaf_append(K7Smem &S, bool is_net, u32 s, u32 h) {
#pragma unroll
    for (u32 cls = 0; cls < 3; ++cls) {
        const bool in = is_net && net_class(h) == cls;
        const u32 mk = __ballot_sync(0xffffffffu, in);
        if (mk) {
            u32 base = 0;
            if (lane_id() == (u32)(__ffs(mk) - 1)) base = atomicAdd(&S.leafcur[cls], (u32)__popc(mk));
            base = __shfl_sync(0xffffffffu, base, __ffs(mk) - 1);
            const u32 slot = S.leafbase[cls] + base + __popc(mk & lanemask_lt());
            if (in && slot < (u32)LEAF_CAP) S.leaf[slot] = s | (h << 16);
        }
    }
}
// Networks over the leaf list (one thread per bucket), then the warp items
// (sorted buckets of 17..WMAX keys, and -- outside batch mode -- recursing ones).
template <class K>
__device__ void run_leaves_and_items(const DevCtx *c, K7Smem &S, u32 ybuf, u32 Lc, u64 gbase, u64 *gout) {
    u64 *Y = ybuf ? S.B : S.A;
    {
        const u32 n0 = S.nleaf[0], n1 = S.nleaf[1], n2 = S.nleaf[2];
        const u32 nt = min(n0 + n1 + n2, (u32)LEAF_CAP);
        for (u32 i = threadIdx.x; i < nt; i += K7_THREADS) {
            const u32 cls = i < n0 ? 0u : i < n0 + n1 ? 1u : 2u;
            const u32 e = S.leaf[i];
            net_sort_class<K>(cls, true, Y, e & 0xffffu, e >> 16, gout);
        }
    }
    prof_mark(c, S, 5);
    const u32 nhi = S.nitems, nlo = S.nitems_lo;
    const u32 nitems = min(nhi + nlo, (u32)ITEM_CAP);
    const u32 lane = lane_id();
    for (;;) {
        u32 idx = 0;
        if (lane == 0) idx = atomicAdd(&S.item_next, 1u);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx >= nitems) break;
        const u32 it = S.items[idx < nhi ? idx : ITEM_CAP - 1 - (idx - nhi)];
        const u32 pos = it & 0x1fffu, size = (it >> 13) & 0x7ffu;
        if (it >> 24) warp_sort_write<K>(Y + pos, size, gout + pos);
        else warp_node<K>(c, S, ybuf, pos, size, Lc, gbase, gout);
    }
    __syncthreads();
}

__device__ __forceinline__ void push_item(const DevCtx *c, K7Smem &S, u32 s, u32 h, bool sort) {
    // large items from the front, small ones from the back: processed largest-first
    const bool large = h >= 256;
    const u32 slot = atomicAdd(large ? &S.nitems : &S.nitems_lo, 1u);
    if (slot + (large ? S.nitems_lo : S.nitems) < ITEM_CAP)
        S.items[large ? slot : ITEM_CAP - 1 - slot] = s | (h << 13) | ((sort ? 1u : 0u) << 24);
    else atomicOr(c->err_flag, 2u);
}

__device__ __forceinline__ void reset_child_lists(K7Smem &S) {
    if (threadIdx.x == 0) {
        S.nitems = 0; S.nitems_lo = 0; S.item_next = 0;
        S.nleaf[0] = S.nleaf[1] = S.nleaf[2] = 0;
    }
}

// largest i in [0, n) with a[i] <= x (a non-decreasing, a[0] <= x)
template <class T>
__device__ __forceinline__ u32 seg_of(const T *a, u32 n, u32 x) {
    u32 lo = 0, hi = n - 1;
    while (lo < hi) { const u32 mid = (lo + hi + 1) >> 1; if (a[mid] <= x) lo = mid; else hi = mid - 1; }
    return lo;
}

template <class K>
__device__ __forceinline__ Model batch_model(const BatchSmem &B, u32 i) {
    Model md;
    md.xmin = B.nxm[i]; md.r = B.nrr[i]; md.betad = (double)B.nP[i]; md.umin = B.nmin[i];
    md.beta = B.nP[i]; md.pad = 0;
    return md;
}

// One batch: nodes list[cur][first, first+N), all at level L in buffer xbuf.
// Alg. 1 lines 152-167 for every node at once; recursing children go to list[cur^1].
template <class K>
__device__ void batch_one(const DevCtx *c, K7Smem &S, u32 xbuf, u32 cur, u32 first, u32 N, u32 L, u64 gbase,
                          u64 *gout) {
    BatchSmem &B = S.u.b;
    u64 *X = xbuf ? S.B : S.A;
    u64 *Y = xbuf ? S.A : S.B;
    const u32 tau = c->tau;
    const bool sample_all = (c->flags & FLAG_SAMPLE_ALL) != 0;
    const bool logging = c->rec != nullptr;
    const u32 tid = threadIdx.x, lane = lane_id(), w = warp_id();
    // S1: per-node parameters and four exclusive scans (bins, buckets, samples, keys)
    {
        u32 v[4] = {0, 0, 0, 0};
        u32 pos = 0, m = 0, P = 0, al = 0;
        if (tid < N) {
            const u32 e = B.list[cur][first + tid];
            pos = e & 0x1fffu; m = e >> 13;
            P = iroot34_small(m); al = sample_all ? m : P;
            v[0] = P + 2; v[1] = P + 1; v[2] = al; v[3] = m;
        }
        u32 incl[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) incl[q] = warp_incl_scan(v[q]);
        if (lane == 31 && w < BN_MAX / 32) {
#pragma unroll
            for (int q = 0; q < 4; ++q) S.red[w * 4 + q] = incl[q];   // red has 2*K7_WARPS u64 slots
        }
        __syncthreads();
        if (tid < BN_MAX) {
            u32 base[4] = {0, 0, 0, 0};
            for (u32 ww = 0; ww < w; ++ww)
#pragma unroll
                for (int q = 0; q < 4; ++q) base[q] += (u32)S.red[ww * 4 + q];
            if (tid < N) {
                B.npos[tid] = (u16)pos; B.nm[tid] = (u16)m; B.nP[tid] = (u16)P; B.nal[tid] = (u16)al;
                B.nbin[tid] = base[0] + incl[0] - v[0]; B.nbkt[tid] = base[1] + incl[1] - v[1];
                B.nsmp[tid] = base[2] + incl[2] - v[2]; B.nkey[tid] = base[3] + incl[3] - v[3];
                B.nmin[tid] = ~0ull; B.nmax[tid] = 0; B.ndb[tid] = 0; B.ndh[tid] = 0; B.ncnt[tid] = 0; B.ndeg[tid] = 0;
            }
            if (tid == N - 1) {
                B.nbin[N] = base[0] + incl[0]; B.nbkt[N] = base[1] + incl[1];
                B.nsmp[N] = base[2] + incl[2]; B.nkey[N] = base[3] + incl[3];
            }
        }
        __syncthreads();
    }
    const u32 M = B.nkey[N], Btot = B.nbin[N], Ktot = B.nbkt[N], Stot = B.nsmp[N];
    for (u32 i = tid; i < N; i += K7_THREADS) B.nwarp[i] = (u8)min((u32)(K7_WARPS - 1), B.nkey[i] * K7_WARPS / M);
    for (u32 i = tid; i < Btot; i += K7_THREADS) B.cnt[i] = 0;
    for (u32 i = tid; i < Ktot; i += K7_THREADS) B.H[i] = 0;
    // S2: node id of every key (into U) and per-node x_min / x_max;
    // warp w takes the flat keys [w*R, (w+1)*R), R a multiple of 32
    const u32 Rw = ((M + K7_WARPS * 32 - 1) / (K7_WARPS * 32)) * 32;
    const u32 fw0 = w * Rw, fw1 = min(M, fw0 + Rw);
    {
        u32 node = fw0 + lane < fw1 ? seg_of(B.nkey, N, fw0 + lane) : 0;
        u64 mn = ~0ull, mx = 0;
        for (u32 j = 0; j < Rw / 32; ++j) {
            const u32 f = fw0 + j * 32 + lane;
            if (f >= fw1) break;
            while (node + 1 < N && f >= B.nkey[node + 1]) {
                if (mn != ~0ull) { atomicMin(&B.nmin[node], mn); atomicMax(&B.nmax[node], mx); }
                mn = ~0ull; mx = 0; ++node;
            }
            const u32 pos = B.npos[node] + (f - B.nkey[node]);
            const u64 v = X[pos];
            S.U[pos] = (u16)node;
            mn = v < mn ? v : mn; mx = v > mx ? v : mx;
        }
        if (mn != ~0ull) { atomicMin(&B.nmin[node], mn); atomicMax(&B.nmax[node], mx); }
    }
    __syncthreads();
    // S3: models (R9/R10: degenerate nodes are sorted as a whole)
    for (u32 i = tid; i < N; i += K7_THREADS) {
        Model md;
        const bool ok = make_model<K>(B.nmin[i], B.nmax[i], B.nP[i], md);
        B.nxm[i] = md.xmin; B.nrr[i] = md.r; B.ndeg[i] = ok ? 0 : 1;
    }
    __syncthreads();
    // S4: samples (R3, R4) -> per-bin counts
    for (u32 sidx = tid; sidx < Stot; sidx += K7_THREADS) {
        const u32 i = seg_of(B.nsmp, N, sidx);
        const u32 k = sidx - B.nsmp[i], m = B.nm[i], p0 = B.npos[i];
        if (B.ndeg[i]) {   // keep the segment totals consistent for the scan
            if (k == 0) atomicAdd(&B.cnt[B.nbin[i] + 1], (u32)B.nal[i]);
            continue;
        }
        const Model md = batch_model<K>(B, i);
        const u32 pos = sample_all ? k : (u32)sample_pos(node_key(c->seed, L, gbase + p0), k, m);
        atomicAdd(&B.cnt[B.nbin[i] + interval_index<K>(X[p0 + pos], md)], 1u);
    }
    __syncthreads();
    // S5: b = prefix of the counts per node, T = floor(b*gamma/alpha)+1
    {
        constexpr u32 PER = (BBINS + K7_THREADS - 1) / K7_THREADS;
        const u32 e0 = tid * PER;
        u32 val[PER], loc = 0;
#pragma unroll
        for (u32 q = 0; q < PER; ++q) { val[q] = e0 + q < Btot ? B.cnt[e0 + q] : 0; loc += val[q]; }
        const u32 incl = warp_incl_scan(loc);
        if (lane == 31) S.scan_tmp[w] = incl;
        __syncthreads();
        u32 run = incl - loc;
        for (u32 ww = 0; ww < w; ++ww) run += S.scan_tmp[ww];
        u32 i = e0 < Btot ? seg_of(B.nbin, N, e0) : 0;
#pragma unroll
        for (u32 q = 0; q < PER; ++q) {
            const u32 e = e0 + q;
            run += val[q];
            if (e < Btot) {
                while (i + 1 < N && e >= B.nbin[i + 1]) ++i;
                const u32 bi = e - B.nbin[i];   // 1-based interval index within the node
                if (bi >= 1 && bi <= (u32)B.nP[i] + 1 && !B.ndeg[i]) {
                    const u32 b = run - B.nsmp[i];
                    B.T[e] = (u16)bucket_of(b, B.nal[i], B.nP[i]);
                    if (logging) atomicAdd(&B.ndb[i], digest_term(bi, b));
                }
            }
        }
    }
    __syncthreads();
    // S6: classify every key: flat bucket id (node's bucket base + T[i(x)] - 1) into U; sizes H
    {
        u32 node = fw0 + lane < fw1 ? seg_of(B.nkey, N, fw0 + lane) : 0;
        for (u32 j = 0; j < Rw / 32; ++j) {
            const u32 f = fw0 + j * 32 + lane;
            if (f >= fw1) break;
            while (node + 1 < N && f >= B.nkey[node + 1]) ++node;
            const u32 pos = B.npos[node] + (f - B.nkey[node]);
            u32 u = 0;
            if (!B.ndeg[node]) u = B.T[B.nbin[node] + interval_index<K>(X[pos], batch_model<K>(B, node))] - 1u;
            const u32 fb = B.nbkt[node] + u;
            S.U[pos] = (u16)fb;
            atomicAdd(&B.H[fb], 1u);
        }
    }
    __syncthreads();
    // S7: bucket starts (node-local exclusive prefix of H) -> cursors; pass-log sums
    u16 *CUR = reinterpret_cast<u16 *>(B.cnt);
    {
        constexpr u32 PER = (BBINS + K7_THREADS - 1) / K7_THREADS;
        const u32 e0 = tid * PER;
        u32 val[PER], loc = 0;
#pragma unroll
        for (u32 q = 0; q < PER; ++q) { val[q] = e0 + q < Ktot ? B.H[e0 + q] : 0; loc += val[q]; }
        const u32 incl = warp_incl_scan(loc);
        if (lane == 31) S.scan_tmp[w] = incl;
        __syncthreads();
        u32 run = incl - loc;
        for (u32 ww = 0; ww < w; ++ww) run += S.scan_tmp[ww];
        u32 i = e0 < Ktot ? seg_of(B.nbkt, N, e0) : 0;
#pragma unroll
        for (u32 q = 0; q < PER; ++q) {
            const u32 e = e0 + q;
            if (e < Ktot) {
                while (i + 1 < N && e >= B.nbkt[i + 1]) ++i;
                CUR[e] = (u16)(B.npos[i] + (run - B.nkey[i]));
                if (logging && !B.ndeg[i]) {
                    const u32 h = val[q], P = B.nP[i];
                    atomicAdd(&B.ndh[i], digest_term(e - B.nbkt[i] + 1, h));
                    if (h) atomicAdd(&B.ncnt[i], h >= P ? 1u : h < tau ? (1u << 10) : (1u << 20));
                }
            }
            run += val[q];
        }
    }
    __syncthreads();
    // S8: stable placement (Append order); warp w places its whole nodes
    {
        const u32 wa = (w == 0) ? 0u : (B.nwarp[N - 1] < w ? N : seg_of(B.nwarp, N, w - 1) + 1);
        u32 wb = wa;
        while (wb < N && B.nwarp[wb] == w) ++wb;
        for (u32 i = wa; i < wb; ++i) {
            const u32 p0 = B.npos[i], m = B.nm[i];
            for (u32 k0 = 0; k0 < m; k0 += 32) {
                const u32 k = k0 + lane;
                const bool act = k < m;
                const u32 fb = act ? (u32)S.U[p0 + k] : 0xffffffffu;
                const u32 peers = __match_any_sync(0xffffffffu, fb);
                const u32 base = act ? CUR[fb] : 0;
                __syncwarp();
                if (act) {
                    const u32 rank = __popc(peers & lanemask_lt());
                    Y[base + rank] = X[p0 + k];
                    if (rank == 0) CUR[fb] = (u16)(base + __popc(peers));
                }
                __syncwarp();
            }
        }
    }
    __syncthreads();
    // S9: children: leaves to the networks / warp sorts, recursions to the next list
    reset_child_lists(S);
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
        for (u32 u0 = 0; u0 < Ktot; u0 += K7_THREADS) {   // warp-uniform trip count
            const u32 fb = u0 + tid;
            const bool valid = fb < Ktot;
            const u32 h = valid ? B.H[fb] : 0;
            u32 kind = CK_EMPTY, s = 0;
            if (h) {
                const u32 i = seg_of(B.nbkt, N, fb);
                s = CUR[fb] - h;
                const bool leaf = B.ndeg[i] || h >= B.nP[i] || h < tau;
                kind = leaf ? (h <= NET_MAX ? CK_NET : CK_BITONIC) : CK_RECURSE;
            }
            if (pass == 0) {
                leaf_count(S, kind == CK_NET, h);
                if (kind == CK_BITONIC) push_item(c, S, s, h, true);
                const u32 rm = __ballot_sync(0xffffffffu, kind == CK_RECURSE);
                if (rm) {
                    u32 base = 0;
                    if (lane == (u32)(__ffs(rm) - 1)) base = atomicAdd(&B.nlist[cur ^ 1u], (u32)__popc(rm));
                    base = __shfl_sync(0xffffffffu, base, __ffs(rm) - 1);
                    const u32 slot = base + __popc(rm & lanemask_lt());
                    if (kind == CK_RECURSE) {
                        if (slot < BLIST_CAP) B.list[cur ^ 1u][slot] = s | (h << 13);
                        else atomicOr(c->err_flag, 2u);
                    }
                }
            } else {
                leaf_append(S, kind == CK_NET, s, h);
            }
        }
        __syncthreads();
        if (pass == 0) leaf_segments(c, S);
        __syncthreads();
    }
    // S10: sort the leaves; S11: node records
    run_leaves_and_items<K>(c, S, xbuf ^ 1u, L + 1, gbase, gout);
    if (logging) {
        for (u32 i = tid; i < N; i += K7_THREADS) {
            if (B.ndeg[i]) continue;
            const u32 cc = B.ncnt[i];
            write_record(c, L, B.nal[i], gbase + B.npos[i], B.nm[i], K::from_okey(B.nmin[i]), K::from_okey(B.nmax[i]),
                         B.ndb[i], B.ndh[i], cc & 1023u, (cc >> 10) & 1023u, cc >> 20);
        }
    }
    __syncthreads();
}

// All levels of batched nodes starting from list[0] (level L, buffer xbuf).
template <class K>
__device__ void batch_levels(const DevCtx *c, K7Smem &S, u32 xbuf, u32 L, u64 gbase, u64 *gout) {
    BatchSmem &B = S.u.b;
    u32 cur = 0;
    for (;;) {
        __syncthreads();
        const u32 ntot = min(B.nlist[cur], (u32)BLIST_CAP);
        if (ntot == 0) break;
        __syncthreads();
        if (threadIdx.x == 0) B.nlist[cur ^ 1u] = 0;
        __syncthreads();
        for (u32 first = 0; first < ntot;) {
            // sub-batch: <= BN_MAX nodes with sum(beta+2) <= BBINS
            if (threadIdx.x < BN_MAX) {
                const u32 i = first + threadIdx.x;
                const u32 v = i < ntot ? iroot34_small(B.list[cur][i] >> 13) + 2 : (u32)BBINS + 1;
                const u32 incl = warp_incl_scan(v);
                if (lane_id() == 31) S.scan_tmp[warp_id()] = incl;
                // count of prefixes that fit (per warp, combined below)
            }
            __syncthreads();
            if (threadIdx.x < BN_MAX) {
                const u32 i = first + threadIdx.x;
                const u32 v = i < ntot ? iroot34_small(B.list[cur][i] >> 13) + 2 : (u32)BBINS + 1;
                u32 incl = warp_incl_scan(v);
                for (u32 ww = 0; ww < warp_id(); ++ww) incl += S.scan_tmp[ww];
                const u32 fits = __ballot_sync(0xffffffffu, i < ntot && incl <= (u32)BBINS);
                if (lane_id() == 0) S.red[warp_id()] = __popc(fits);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                u32 nsub = 0;
                for (u32 ww = 0; ww < BN_MAX / 32; ++ww) nsub += (u32)S.red[ww];
                B.nsub = max(nsub, 1u);
            }
            __syncthreads();
            const u32 N = B.nsub;
            batch_one<K>(c, S, xbuf, cur, first, N, L, gbase, gout);
            first += N;
        }
        cur ^= 1u;
        xbuf ^= 1u;
        L += 1;
    }
}

// Children of a CTA-level partition into Y (Hc/Bs valid for nb buckets of the
// range [p, p+m)): leaves sorted (networks, warp sorts), recursing buckets as
// CTA items (> WMAX), batched nodes (tau >= BATCH_MIN_TAU) or warp items.
template <class K>
__device__ void cta_children(const DevCtx *c, K7Smem &S, u32 ybuf, u32 p, u32 m, u32 nb, u32 delta, u32 Lc,
                             u64 gbase, u64 *gout) {
    const u32 tau = c->tau;
    const bool batch = tau >= BATCH_MIN_TAU;
    reset_child_lists(S);
    if (threadIdx.x == 0) S.u.b.nlist[0] = 0;
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
        for (u32 u0 = 0; u0 < nb; u0 += K7_THREADS) {   // warp-uniform trip count
            const u32 u = u0 + threadIdx.x;
            const bool valid = u < nb;
            const u32 h = valid ? S.Hc[u] : 0, s = valid ? S.Bs[u] : 0;
            u32 kind = CK_EMPTY;
            if (h) kind = (h >= delta || h < tau) ? (h <= NET_MAX ? CK_NET : CK_BITONIC) : CK_RECURSE;
            if (pass == 1) { leaf_append(S, kind == CK_NET, s, h); continue; }
            leaf_count(S, kind == CK_NET, h);
            if (kind == CK_RECURSE || kind == CK_BITONIC) {
                if (h > WMAX) {
                    const u32 slot = atomicAdd(&S.nbig, 1u);
                    if (slot < BIG_CAP) {
                        BigItem it;
                        it.pos = s; it.size = h; it.level = Lc; it.buf = ybuf; it.kind = kind == CK_RECURSE ? 0u : 1u;
                        S.big[slot] = it;
                    } else {
                        atomicOr(c->err_flag, 2u);
                    }
                } else if (kind == CK_RECURSE && batch && h <= BATCH_MAX_M) {
                    const u32 slot = atomicAdd(&S.u.b.nlist[0], 1u);
                    if (slot < BLIST_CAP) S.u.b.list[0][slot] = s | (h << 13);
                    else atomicOr(c->err_flag, 2u);
                } else {
                    push_item(c, S, s, h, kind == CK_BITONIC);
                }
            }
        }
        __syncthreads();
        if (pass == 0) leaf_segments(c, S);
        __syncthreads();
    }
    prof_mark(c, S, 4);
    run_leaves_and_items<K>(c, S, ybuf, Lc, gbase, gout);
    prof_mark(c, S, 6);
    if (batch) batch_levels<K>(c, S, ybuf, Lc, gbase, gout);
    prof_mark(c, S, 7);
}

// CTA-level Alg. 1 on X[p, p+m) (WMAX < m <= S_CAP), level L, global offset
// gbase + p.  Leaves sorted or partitions into the other buffer and recurses.
template <class K>
__device__ void cta_node(const DevCtx *c, K7Smem &S, u32 xbuf, u32 p, u32 m, u32 L, u64 gbase, u64 *gout) {
    u64 *X = xbuf ? S.B : S.A;
    u64 *Y = xbuf ? S.A : S.B;
    const u32 tau = c->tau;
    const bool sample_all = (c->flags & FLAG_SAMPLE_ALL) != 0;
    const bool logging = c->rec != nullptr;
    if (m < tau) { cta_sort_write<K>(X + p, m, gout + p); return; }
    const u32 P = iroot34_small(m);
    const u32 alpha = sample_all ? m : P, beta = P, gamma = P, delta = P;
    u32 *cnt = S.u.fit.cnt, *T = S.u.fit.T;
    for (u32 i = threadIdx.x; i <= beta + 1; i += K7_THREADS) cnt[i] = 0;
    // x_min, x_max: one fused min/max reduction
    u64 mn = ~0ull, mx = 0;
    for (u32 k = threadIdx.x; k < m; k += K7_THREADS) { u64 v = X[p + k]; mn = v < mn ? v : mn; mx = v > mx ? v : mx; }
    mn = warp_min_u64(mn);
    mx = warp_max_u64(mx);
    if (lane_id() == 0) { S.red[warp_id()] = mn; S.red[K7_WARPS + warp_id()] = mx; }
    __syncthreads();
    mn = S.red[0]; mx = S.red[K7_WARPS];
    for (u32 w = 1; w < K7_WARPS; ++w) { mn = S.red[w] < mn ? S.red[w] : mn; mx = S.red[K7_WARPS + w] > mx ? S.red[K7_WARPS + w] : mx; }
    Model md;
    if (!make_model<K>(mn, mx, P, md)) { __syncthreads(); cta_sort_write<K>(X + p, m, gout + p); return; }
    const u64 nkey = node_key(c->seed, L, gbase + p);
    for (u32 k = threadIdx.x; k < alpha; k += K7_THREADS) {
        u32 pos = sample_all ? k : (u32)sample_pos(nkey, k, m);
        atomicAdd(&cnt[interval_index<K>(X[p + pos], md)], 1u);
    }
    __syncthreads();
    // b = inclusive prefix of cnt[1..beta+1] and T, in one CTA scan
    u64 db = 0;
    {
        const u32 i0 = 2 * threadIdx.x + 1, i1 = i0 + 1;
        const u32 v0 = i0 <= beta + 1 ? cnt[i0] : 0, v1 = i1 <= beta + 1 ? cnt[i1] : 0;
        const u32 loc = v0 + v1;
        const u32 incl = warp_incl_scan(loc);
        if (lane_id() == 31) S.scan_tmp[warp_id()] = incl;
        __syncthreads();
        u32 wbase = 0;
        for (u32 w = 0; w < warp_id(); ++w) wbase += S.scan_tmp[w];
        const u32 b0 = wbase + incl - loc + v0, b1 = b0 + v1;
        if (i0 <= beta + 1) {
            cnt[i0] = b0; T[i0] = bucket_of(b0, alpha, gamma);
            if (logging) db += digest_term(i0, b0);
            if (logging && L == 1 && c->l1_b && i0 - 1 < c->l1_cap) c->l1_b[i0 - 1] = b0;
        }
        if (i1 <= beta + 1) {
            cnt[i1] = b1; T[i1] = bucket_of(b1, alpha, gamma);
            if (logging) db += digest_term(i1, b1);
            if (logging && L == 1 && c->l1_b && i1 - 1 < c->l1_cap) c->l1_b[i1 - 1] = b1;
        }
    }
    __syncthreads();
    if (logging) db = cta_reduce_sum64(S, db);
    for (u32 k = threadIdx.x; k < m; k += K7_THREADS) S.U[p + k] = (u16)(T[interval_index<K>(X[p + k], md)] - 1u);
    __syncthreads();
    prof_mark(c, S, 8);
    cta_partition(S, X, Y, p, m, gamma + 1);
    prof_mark(c, S, 9);
    if (logging) {
        u64 dh = 0;
        u32 nf = 0, ns = 0, nr = 0;
        for (u32 u = threadIdx.x; u <= gamma; u += K7_THREADS) {
            u32 h = S.Hc[u];
            dh += digest_term(u + 1, h);
            if (h) { if (h >= delta) nf++; else if (h < tau) ns++; else nr++; }
        }
        dh = cta_reduce_sum64(S, dh);
        u64 cnts = cta_reduce_sum64(S, (u64)nf | ((u64)ns << 21) | ((u64)nr << 42));
        if (threadIdx.x == 0)
            write_record(c, L, alpha, gbase + p, m, K::from_okey(mn), K::from_okey(mx), db, dh,
                         (u32)(cnts & 0x1fffff), (u32)((cnts >> 21) & 0x1fffff), (u32)(cnts >> 42));
        if (L == 1 && c->l1_h)
            for (u32 u = threadIdx.x; u <= gamma && u < c->l1_cap; u += K7_THREADS) c->l1_h[u] = S.Hc[u];
    }
    cta_children<K>(c, S, xbuf ^ 1u, p, m, gamma + 1, delta, L + 1, gbase, gout);
}

// ------------------------------------------------------------------ the kernel
__device__ __forceinline__ ulonglong2 ld_stream2(const ulonglong2 *p) {
    ulonglong2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p));
    return r;
}

// Load src[0, m) into A as ordered keys; returns true if a NaN was seen (f64).
template <class K>
__device__ __forceinline__ bool load_task(K7Smem &S, const u64 *src, u32 m) {
    bool nan = false;
    auto put = [&](u32 k, u64 raw) {
        if (K::is_f64) nan |= (raw & 0x7fffffffffffffffull) > 0x7ff0000000000000ull;
        S.A[k] = K::to_okey(raw);
    };
    const u32 head = ((uintptr_t)src & 15) ? 1u : 0u;
    if (head && m && threadIdx.x == 0) put(0, src[0]);
    const u32 nv = (m - min(head, m)) / 2;
    const ulonglong2 *v = reinterpret_cast<const ulonglong2 *>(src + head);
    constexpr u32 U4 = 4;
    u32 i = threadIdx.x;
    for (; i + (U4 - 1) * K7_THREADS < nv; i += U4 * K7_THREADS) {
        ulonglong2 r[U4];
#pragma unroll
        for (u32 q = 0; q < U4; ++q) r[q] = ld_stream2(v + i + q * K7_THREADS);
#pragma unroll
        for (u32 q = 0; q < U4; ++q) { put(head + 2 * (i + q * K7_THREADS), r[q].x); put(head + 2 * (i + q * K7_THREADS) + 1, r[q].y); }
    }
    for (; i < nv; i += K7_THREADS) { ulonglong2 r = ld_stream2(v + i); put(head + 2 * i, r.x); put(head + 2 * i + 1, r.y); }
    if (m > head && ((m - head) & 1) && threadIdx.x == 0) put(m - 1, src[m - 1]);
    return nan;
}

template <class K>
__global__ void __launch_bounds__(K7_THREADS, 1) k7_kernel(const DevCtx *__restrict__ c) {
    extern __shared__ __align__(16) unsigned char k7_smem_raw[];
    K7Smem &S = *reinterpret_cast<K7Smem *>(k7_smem_raw);
    if (*c->nan_flag) return;
    const u32 ntasks = *c->k7_count;
    const u32 begin = *c->k7_begin;
    if (c->k7_prof && threadIdx.x == 0) {
        for (int i = 0; i < K7_PROF_SLOTS; ++i) S.prof[i] = 0;
        S.prof_t = clock64();
    }
    for (;;) {
        if (threadIdx.x == 0) {
            S.task_idx = begin + atomicAdd(c->k7_next, 1u);
            if (S.task_idx < ntasks) S.task = c->k7[S.task_idx];
            S.nbig = 0;
        }
        __syncthreads();
        if (S.task_idx >= ntasks) break;
        prof_mark(c, S, 0);
        const K7Task task = S.task;
        const u64 *src = c->buf[task.src] + task.off;
        u64 *gout = c->buf[2] + task.off;
        const u32 m = task.size;
        const bool nan_here = load_task<K>(S, src, m);
        if (K::is_f64 && task.level == 1 && __syncthreads_or(nan_here)) {
            if (threadIdx.x == 0) atomicOr(c->nan_flag, 1u);
            return;
        }
        __syncthreads();
        prof_mark(c, S, 1);
        if (threadIdx.x == 0 && c->k7_prof) { S.prof[11] += 1; S.prof[12] += m; }
        if (task.kind == K7_SORT) {
            cta_sort_write<K>(S.A, m, gout);
            prof_mark(c, S, 10);
        } else if (task.kind == K7_NODE) {
            if (m <= WMAX) {
                if (warp_id() == 0) warp_node<K>(c, S, 0u, 0u, m, task.level, task.off, gout);
                __syncthreads();
            } else {
                if (threadIdx.x == 0) {
                    BigItem it; it.pos = 0; it.size = m; it.level = task.level; it.buf = 0; it.kind = 0;
                    S.big[0] = it; S.nbig = 1;
                }
                __syncthreads();
            }
        } else {  // K7_GROUP: finish the global node's placement for buckets [jlo, jhi)
            if (threadIdx.x == 0) {
                const GNode &g = c->nodes[task.node];
                S.gmd = g.md; S.gT = g.T; S.gH = g.H;
                S.gnode_delta = g.delta; S.gnode_level = g.level;
            }
            __syncthreads();
            const Model md = S.gmd;
            const u32 *gT = S.gT;
            constexpr u32 G4 = 4;
            u32 k = threadIdx.x;
            for (; k + (G4 - 1) * K7_THREADS < m; k += G4 * K7_THREADS) {
                u32 ix[G4], j[G4];
#pragma unroll
                for (u32 q = 0; q < G4; ++q) ix[q] = interval_index<K>(S.A[k + q * K7_THREADS], md);
#pragma unroll
                for (u32 q = 0; q < G4; ++q) j[q] = __ldg(&gT[ix[q]]);
#pragma unroll
                for (u32 q = 0; q < G4; ++q) S.U[k + q * K7_THREADS] = (u16)(j[q] - task.jlo);
            }
            for (; k < m; k += K7_THREADS) S.U[k] = (u16)(__ldg(&gT[interval_index<K>(S.A[k], md)]) - task.jlo);
            __syncthreads();
            prof_mark(c, S, 2);
            const u32 nb = task.jhi - task.jlo;
            cta_partition(S, S.A, S.B, 0u, m, nb);
            prof_mark(c, S, 3);
            for (u32 u = threadIdx.x; u < nb; u += K7_THREADS) S.gH[task.jlo + u] = S.Hc[u];
            cta_children<K>(c, S, 1u, 0u, m, nb, S.gnode_delta, S.gnode_level + 1, task.off, gout);
        }
        // big items (> WMAX): processed by the whole CTA, LIFO
        for (;;) {
            __syncthreads();
            const u32 nb_ = S.nbig;
            if (nb_ == 0 || nb_ > BIG_CAP) break;
            const BigItem it = S.big[nb_ - 1];
            __syncthreads();
            if (threadIdx.x == 0) S.nbig = nb_ - 1;
            __syncthreads();
            u64 *X = it.buf ? S.B : S.A;
            if (it.kind == 1) cta_sort_write<K>(X + it.pos, it.size, gout + it.pos);
            else cta_node<K>(c, S, it.buf, it.pos, it.size, it.level, task.off, gout);
        }
        __syncthreads();
    }
    if (c->k7_prof && threadIdx.x == 0)
        for (int i = 0; i < K7_PROF_SLOTS; ++i) atomicAdd(&c->k7_prof[i], S.prof[i]);
}

}  // namespace pcf
