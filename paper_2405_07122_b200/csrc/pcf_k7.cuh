// pcf_k7.cuh -- K7: run the whole remaining Algorithm-1 subtree of a segment
// of <= S_CAP keys in shared memory, one CTA per task,
// persistent grid.
//
// A task is one of
//   K7_GROUP : buckets [jlo, jhi) of a global bucketing node whose keys lie,
//              in stable (Append) order, in one contiguous range.  The CTA
//              finishes the node's model-based bucketing for those buckets
//              (stable placement by j) and processes every
//              bucket per Alg. 1 lines 160-167.
//   K7_NODE  : a segment that is a fresh Learned-Sort call (level L, offset o).
//   K7_SORT  : a bucket that Alg. 1 sends to Standard-Sort.
// The task's keys are read once from HBM, every deeper level runs in shared
// memory, and the finished (sorted) task is written back once, coalesced.
//
// Level-synchronous, key-parallel design:
//  * The nodes of one recursion level form an ordered list (a ring of
//    (position, size) entries).  They are processed in sub-batches whose
//    bucket columns fit the counter matrix (MC columns): every step of
//    Alg. 1 lines 152-158 runs flat over all keys / samples / bins /
//    buckets of the sub-batch at once, so every lane has work regardless of
//    the node sizes.
//  * Stable placement (Append order; readings R4, R16): warp
//    w owns a contiguous range of the sub-batch's keys; one pass computes each
//    key's bucket, then ranks it inside its warp with __match_any_sync and a
//    per-warp counter row (no shared-memory atomics on the per-key path); a
//    column pass turns the [warp x bucket] counts into destinations.
//  * Each node's columns are preceded by a "gap" column holding the number of
//    buffer positions between it and the previous node, so one exclusive scan
//    over the columns yields absolute buffer positions, and a max-scan over
//    the gap markers tells every column its node.
//  * Buckets Alg. 1 sends to Standard-Sort (|c_j| >= delta or |c_j| < tau) are
//    placed directly into buffer A and sorted there in place (per-thread
//    register networks for <= 32 keys, compacted by size class; warp sorts up
//    to 1024; a CTA sort above); recursing buckets go to the other buffer and
//    to the next level's node list.  Every position ends in A, sorted; one
//    coalesced copy writes the task out.
#pragma once
#include "pcf_common.cuh"

namespace pcf {

constexpr int MC = 1280;                          // bucket columns (and bins) of one sub-batch
constexpr int NCAP = 256;                         // nodes of one sub-batch
constexpr int RING = S_CAP / 2;                   // level node lists: nodes hold >= 2 keys (tau >= 2)
constexpr int CH = S_CAP / (K7_WARPS * 32);       // 32-key chunks per warp (16)
constexpr int BIGM = 1024;                        // nodes above this size: CTA-wide min/max
constexpr int BIGCAP = S_CAP / BIGM;
constexpr u32 SMALL_MAX = 64;                     // leaves up to this size: key-parallel rank sort
constexpr int BLCAP = S_CAP / (SMALL_MAX + 1) + 1;  // larger leaves of one sub-batch
constexpr u32 NONE = 0xffffffffu;
// destination row entries: buffer position | target (Y: recursing bucket, A: leaf of
// one key -- final, B: larger leaf -- sorted into A by the leaf phase)
constexpr u32 DEST_A = 0x4000u, DEST_B = 0x8000u, POS_MASK = 0x3fffu;

struct K7Smem {
    u64 A[S_CAP];
    u64 B[S_CAP];
    union {
        u16 wcnt[K7_WARPS][MC];   // per-warp bucket counters -> per-warp destinations
        u32 cnt[MC];              // fit: per-bin sample counts (dead before the rank pass)
    } m;
    u16 T[MC];                    // bucket table of every node's bins (1-based within the node)
    u16 GM[MC];                   // column marker: node index + 1 at the node's gap column
    u32 leaf[MC];                 // leaves of 2..SMALL_MAX keys, in position order: pos | h << 16
    u16 lkp[MC + 1];              // exclusive key prefix over leaf[]
    u32 bleaf[BLCAP];             // leaves of > SMALL_MAX keys: pos | h << 16
    u32 ring[RING];               // node lists: pos | m << 13
    // node table of the current sub-batch
    u32 nkey[NCAP + 1];           // flat key offsets
    u16 nb0[NCAP + 1];            // first column / bin (the gap column; bins are 1-based)
    u16 nsmp[NCAP + 1];           // flat sample offsets
    u16 npos[NCAP], nm[NCAP], nP[NCAP], nal[NCAP], ngap[NCAP];
    u8 ndeg[NCAP];
    u64 nmin[NCAP], nmax[NCAP];
    u64 ndb[NCAP], ndh[NCAP];
    u32 ncnt[NCAP];               // pass log: nf | ns << 10 | nr << 20
    u16 big[BIGCAP];
    u32 nbig;
    u32 nleaf, lkeys, nbleaf;
    u32 scan_a[K7_WARPS][4], scan_b[K7_WARPS][2], scan_c[K7_WARPS][3];
    u32 N, head, tail, level_end, item_next, new_tail;
    u32 task_idx;
    K7Task task;
    Model gmd;
    const u32 *gT;
    u32 *gH;
    u32 gdelta, glevel, gjlo;
    long long prof_t;                       // PCF_FLAG_PROFILE bookkeeping (thread 0)
    unsigned long long prof[K7_PROF_SLOTS];
};

static_assert(sizeof(K7Smem) <= 232448, "K7 shared memory exceeds 227 KB");

// K7 phase profiling (PCF_FLAG_PROFILE): thread 0 charges the cycles since the
// previous mark to slot `id` (barrier waits included).  Slots: 0 claim, 1 load,
// 2 group rank, 3 group columns+place, 4 leaves, 5 setup, 6 min/max,
// 7 sample, 8 fit, 9 rank, 10 columns+place, 11 tasks, 12 keys, 13 store.
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
__device__ __forceinline__ u32 warp_incl_scan(u32 v) {
    const u32 lane = lane_id();
    for (int o = 1; o < 32; o <<= 1) {
        u32 w = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= (u32)o) v += w;
    }
    return v;
}
__device__ __forceinline__ u32 warp_incl_max(u32 v) {
    const u32 lane = lane_id();
    for (int o = 1; o < 32; o <<= 1) {
        u32 w = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= (u32)o) v = w > v ? w : v;
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

// largest i in [0, n) with a[i] <= x (a non-decreasing, a[0] <= x)
template <class T>
__device__ __forceinline__ u32 seg_of(const T *a, u32 n, u32 x) {
    u32 lo = 0, hi = n - 1;
    while (lo < hi) { const u32 mid = (lo + hi + 1) >> 1; if ((u32)a[mid] <= x) lo = mid; else hi = mid - 1; }
    return lo;
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

// ------------------------------------------------------------------ Standard-Sort (R2) on ordered keys
// Bitonic network over a[0, n) by one warp in shared memory; all merges
// ascending (first step of each stage compares i with its mirror), so the
// virtual +inf padding never moves.
__device__ void warp_bitonic_smem(u64 *a, u32 n) {
    if (n <= 1) return;
    const u32 P = next_pow2(n);
    const u32 lane = lane_id();
    const u32 lgP = 31 - __clz(P);
    for (u32 lk = 1; lk <= lgP; ++lk) {
        const u32 k = 1u << lk, lh = lk - 1;
        for (u32 t = lane; t < (P >> 1); t += 32) {
            const u32 blk = t >> lh, w = t & ((1u << lh) - 1);
            const u32 lo = (blk << lk) + w, hi = (blk << lk) + k - 1 - w;
            if (hi < n) { u64 x = a[lo], y = a[hi]; if (x > y) { a[lo] = y; a[hi] = x; } }
        }
        __syncwarp();
        for (int lj = (int)lh - 1; lj >= 0; --lj) {
            const u32 j = 1u << lj;
            for (u32 t = lane; t < (P >> 1); t += 32) {
                const u32 lo = ((t >> lj) << (lj + 1)) + (t & (j - 1)), hi = lo + j;
                if (hi < n) { u64 x = a[lo], y = a[hi]; if (x > y) { a[lo] = y; a[hi] = x; } }
            }
            __syncwarp();
        }
    }
}

// Same network by the whole CTA (leaves > 1024 keys: rare fallback buckets).
__device__ void cta_bitonic_smem(u64 *a, u32 n) {
    if (n > 1) {
        const u32 P = next_pow2(n);
        const u32 lgP = 31 - __clz(P);
        for (u32 lk = 1; lk <= lgP; ++lk) {
            const u32 k = 1u << lk, lh = lk - 1;
            for (u32 t = threadIdx.x; t < (P >> 1); t += K7_THREADS) {
                const u32 blk = t >> lh, w = t & ((1u << lh) - 1);
                const u32 lo = (blk << lk) + w, hi = (blk << lk) + k - 1 - w;
                if (hi < n) { u64 x = a[lo], y = a[hi]; if (x > y) { a[lo] = y; a[hi] = x; } }
            }
            __syncthreads();
            for (int lj = (int)lh - 1; lj >= 0; --lj) {
                const u32 j = 1u << lj;
                for (u32 t = threadIdx.x; t < (P >> 1); t += K7_THREADS) {
                    const u32 lo = ((t >> lj) << (lj + 1)) + (t & (j - 1)), hi = lo + j;
                    if (hi < n) { u64 x = a[lo], y = a[hi]; if (x > y) { a[lo] = y; a[hi] = x; } }
                }
                __syncthreads();
            }
        }
    }
    __syncthreads();
}

// Standard-Sort of every leaf of the sub-batch (keys in B) into A.
// Leaves of <= SMALL_MAX keys: one thread per key, flat over all their keys
// (every lane busy, one compact loop): the key's rank inside its leaf counts
// the smaller keys and the equal keys before it, and the key is written to
// A[leaf start + rank].  A warp handles 32 consecutive keys; it finds their
// leaves with one binary search and a bit mask of the leaf boundaries.
// Larger leaves (fallback buckets, rare): bitonic networks by a warp (<= 1024
// keys) or by the CTA, in B, then copied to A.
__device__ __noinline__ void leaf_phase(K7Smem &S) {
    const u32 lane = lane_id(), w = warp_id();
    const u32 NL = S.nleaf, K = S.lkeys;
    // warp w: keys [w*RW, (w+1)*RW); the leaf of the first key is carried from chunk to chunk
    const u32 RW = ((K + K7_THREADS - 1) / K7_THREADS) * 32;
    const u32 kw0 = w * RW, kw1 = min(kw0 + RW, K);
    u32 a = kw0 < kw1 ? seg_of(S.lkp, NL, kw0) : 0;
    for (u32 k0 = kw0; k0 < kw1; k0 += 32) {
        const u32 bi = a + 1 + lane;
        const u32 b = bi <= NL ? (u32)S.lkp[bi] : 0xffffffffu;
        const u32 bit = (b - k0 < 32u) ? (1u << (b - k0)) : 0u;      // boundaries in (k0, k0 + 31]
        const u32 mask = __reduce_or_sync(0xffffffffu, bit);
        const u32 my = a + __popc(mask & ((2u << lane) - 1u));
        const u32 k = k0 + lane;
        if (k < kw1) {
            const u32 e = S.leaf[my], st = e & 0xffffu, h = e >> 16;
            const u32 p = st + (k - S.lkp[my]);
            const u64 v = S.B[p];
            // rank = #{j : (B[j], j) < (v, p)} (keys below v, and equal keys before p):
            // one 96-bit subtract chain per key; PTX's carry flag after it is set iff
            // (B[j], j) >= (v, p) (carry = no borrow), so r counts the others and
            // rank = h - r
            u32 r = 0;
            const u32 vlo = (u32)v, vhi = (u32)(v >> 32);
            for (u32 j = st; j < st + h; ++j) {
                const u64 x = S.B[j];
                asm("{\n\t.reg .u32 t;\n\t"
                    "sub.cc.u32 t, %1, %2;\n\t"
                    "subc.cc.u32 t, %3, %4;\n\t"
                    "subc.cc.u32 t, %5, %6;\n\t"
                    "addc.u32 %0, %0, 0;\n\t}"
                    : "+r"(r) : "r"(j), "r"(p), "r"((u32)x), "r"(vlo), "r"((u32)(x >> 32)), "r"(vhi));
            }
            S.A[st + (h - r)] = v;
        }
        // leaf of key k0 + 32
        a += __popc(mask);
        if (a + 1 <= NL && (u32)S.lkp[a + 1] <= k0 + 32) ++a;
    }
    const u32 NB = S.nbleaf;
    for (;;) {
        u32 idx = 0;
        if (lane == 0) idx = atomicAdd(&S.item_next, 1u);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx >= NB) break;
        const u32 e = S.bleaf[idx], st = e & 0xffffu, h = e >> 16;
        if (h > 1024) continue;
        warp_bitonic_smem(S.B + st, h);
        for (u32 i = lane; i < h; i += 32) S.A[st + i] = S.B[st + i];
        __syncwarp();
    }
    __syncthreads();
    for (u32 idx = 0; idx < NB; ++idx) {
        const u32 e = S.bleaf[idx], st = e & 0xffffu, h = e >> 16;
        if (h <= 1024) continue;
        cta_bitonic_smem(S.B + st, h);
        for (u32 i = threadIdx.x; i < h; i += K7_THREADS) S.A[st + i] = S.B[st + i];
        __syncthreads();
    }
}

// ------------------------------------------------------------------ one sub-batch of a level
// Setup: take nodes ring[head ..) while their columns (P+2 each: gap + P+1
// buckets) fit MC and they fit NCAP; node table, flat offsets, markers.
__device__ void sub_setup(const DevCtx *c, K7Smem &S) {
    const u32 tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const bool sample_all = (c->flags & FLAG_SAMPLE_ALL) != 0;
    const u32 head = S.head, navail = S.level_end - S.head;
    for (u32 i = tid; i < MC; i += K7_THREADS) { S.m.cnt[i] = 0; S.GM[i] = 0; }
    if (tid == 0) S.nbig = 0;
    u32 pos = 0, m = 0, P = 0, al = 0, sz = 0;
    const bool valid = tid < NCAP && tid < navail;
    if (valid) {
        const u32 e = S.ring[(head + tid) & (RING - 1)];
        pos = e & 0x1fffu; m = e >> 13;
        P = iroot34_small(m); al = sample_all ? m : P; sz = P + 2;
    }
    u32 isz = 0, im = 0, ial = 0;
    if (tid < NCAP) {
        isz = warp_incl_scan(sz); im = warp_incl_scan(m); ial = warp_incl_scan(al);
        if (lane == 31) { S.scan_a[w][0] = isz; S.scan_a[w][1] = im; S.scan_a[w][2] = ial; }
    }
    __syncthreads();
    if (tid < NCAP) {
        for (u32 ww = 0; ww < w; ++ww) { isz += S.scan_a[ww][0]; im += S.scan_a[ww][1]; ial += S.scan_a[ww][2]; }
        const bool fits = valid && isz <= (u32)MC;
        if (fits) {
            const u32 i = tid;
            u32 prev_end = 0;
            if (i > 0) { const u32 pe = S.ring[(head + i - 1) & (RING - 1)]; prev_end = (pe & 0x1fffu) + (pe >> 13); }
            S.npos[i] = (u16)pos; S.nm[i] = (u16)m; S.nP[i] = (u16)P; S.nal[i] = (u16)al;
            S.ngap[i] = (u16)(pos - prev_end);
            S.nkey[i] = im - m; S.nb0[i] = (u16)(isz - sz); S.nsmp[i] = (u16)(ial - al);
            S.nmin[i] = ~0ull; S.nmax[i] = 0; S.ndb[i] = 0; S.ndh[i] = 0; S.ncnt[i] = 0;
            S.GM[isz - sz] = (u16)(i + 1);
            if (m > (u32)BIGM) { const u32 b = atomicAdd(&S.nbig, 1u); if (b < (u32)BIGCAP) S.big[b] = (u16)i; }
            // last fitting node: totals
            bool last = i + 1 >= navail || i + 1 >= (u32)NCAP;
            if (!last) {
                const u32 e2 = S.ring[(head + i + 1) & (RING - 1)];
                last = isz + iroot34_small(e2 >> 13) + 2 > (u32)MC;
            }
            if (last) { S.N = i + 1; S.nkey[i + 1] = im; S.nb0[i + 1] = (u16)isz; S.nsmp[i + 1] = (u16)ial; }
        }
    }
    __syncthreads();
}

// x_min, x_max of every node: one warp per node <= BIGM keys,
// the whole CTA for the few larger ones.
__device__ void sub_minmax(K7Smem &S, const u64 *X) {
    const u32 N = S.N, w = warp_id(), lane = lane_id();
    for (u32 i = w; i < N; i += K7_WARPS) {
        const u32 m = S.nm[i];
        if (m > (u32)BIGM) continue;
        const u64 *x = X + S.npos[i];
        u64 mn = ~0ull, mx = 0;
        for (u32 k = lane; k < m; k += 32) { const u64 v = x[k]; mn = v < mn ? v : mn; mx = v > mx ? v : mx; }
        mn = warp_min_u64(mn);
        mx = warp_max_u64(mx);
        if (lane == 0) { S.nmin[i] = mn; S.nmax[i] = mx; }
    }
    const u32 nb = min(S.nbig, (u32)BIGCAP);
    for (u32 b = 0; b < nb; ++b) {
        const u32 i = S.big[b], m = S.nm[i];
        const u64 *x = X + S.npos[i];
        u64 mn = ~0ull, mx = 0;
        for (u32 k = threadIdx.x; k < m; k += K7_THREADS) { const u64 v = x[k]; mn = v < mn ? v : mn; mx = v > mx ? v : mx; }
        mn = warp_min_u64(mn);
        mx = warp_max_u64(mx);
        if (lane == 0) { atomicMin(&S.nmin[i], mn); atomicMax(&S.nmax[i], mx); }
    }
    __syncthreads();
}

// alpha samples per node (R3, R4) -> per-bin counts.
template <class K>
__device__ void sub_sample(const DevCtx *c, K7Smem &S, const u64 *X, u32 L, u64 gbase) {
    const u32 N = S.N, Stot = S.nsmp[N];
    const bool sample_all = (c->flags & FLAG_SAMPLE_ALL) != 0;
    for (u32 i = threadIdx.x; i < N; i += K7_THREADS) {
        Model md;
        S.ndeg[i] = make_model<K>(S.nmin[i], S.nmax[i], S.nP[i], md) ? 0 : 1;
    }
    for (u32 s = threadIdx.x; s < Stot; s += K7_THREADS) {
        const u32 i = seg_of(S.nsmp, N, s);
        const u32 k = s - S.nsmp[i];
        Model md;
        if (!make_model<K>(S.nmin[i], S.nmax[i], S.nP[i], md)) {   // R9/R10: whole node to Standard-Sort
            if (k == 0) atomicAdd(&S.m.cnt[S.nb0[i]], (u32)S.nal[i]);   // keeps the flat prefix per node
            continue;
        }
        const u32 p0 = S.npos[i];
        const u32 pos = sample_all ? k : (u32)sample_pos(node_key(c->seed, L, gbase + p0), k, S.nm[i]);
        atomicAdd(&S.m.cnt[S.nb0[i] + interval_index<K>(X[p0 + pos], md)], 1u);
    }
    __syncthreads();
}

// b = inclusive prefix of the counts per node, T = floor(b*gamma/alpha)+1 (R7).
__device__ void sub_fit(const DevCtx *c, K7Smem &S, u32 L) {
    constexpr u32 PER = (MC + K7_THREADS - 1) / K7_THREADS;
    const u32 N = S.N, nbins = S.nb0[N];
    const u32 tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const bool logging = c->rec != nullptr;
    const u32 e0 = tid * PER;
    u32 v[PER], loc = 0;
#pragma unroll
    for (u32 q = 0; q < PER; ++q) { v[q] = e0 + q < nbins ? S.m.cnt[e0 + q] : 0; loc += v[q]; }
    const u32 incl = warp_incl_scan(loc);
    if (lane == 31) S.scan_b[w][0] = incl;
    __syncthreads();
    u32 run = incl - loc;
    for (u32 ww = 0; ww < w; ++ww) run += S.scan_b[ww][0];
    if (e0 < nbins) {
        u32 i = seg_of(S.nb0, N, e0);
#pragma unroll
        for (u32 q = 0; q < PER; ++q) {
            const u32 e = e0 + q;
            run += v[q];
            if (e < nbins) {
                while (e >= S.nb0[i + 1]) ++i;
                const u32 ix = e - S.nb0[i];   // 1-based interval index within the node
                if (ix >= 1 && !S.ndeg[i]) {
                    const u32 b = run - S.nsmp[i];
                    S.T[e] = (u16)bucket_of(b, S.nal[i], S.nP[i]);
                    if (logging) {
                        atomicAdd((unsigned long long *)&S.ndb[i], (unsigned long long)digest_term(ix, b));
                        if (L == 1 && c->l1_b && ix - 1 < c->l1_cap) c->l1_b[ix - 1] = b;
                    }
                }
            }
        }
    }
    __syncthreads();
}

// Classify + rank + columns + placement of one sub-batch (or of a K7 group).
// X -> Y for recursing buckets, X -> A for leaves.  Appends the children.
template <class K, bool GROUP>
__device__ void sub_place(const DevCtx *c, K7Smem &S, const u64 *X, u64 *Y, u32 L) {
    const u32 tid = threadIdx.x, w = warp_id(), lane = lane_id();
    const u32 N = S.N, Mtot = S.nkey[N], ncols = S.nb0[N];
    const u32 tau = c->tau;
    const bool logging = c->rec != nullptr;
    // ---- pass 1: bucket column of every key (flat index f over the sub-batch's keys)
    {
        u32 *row32 = reinterpret_cast<u32 *>(S.m.wcnt[w]);
        for (u32 i = lane; i < (ncols + 1) / 2; i += 32) row32[i] = 0;
    }
    const u32 R = ((Mtot + K7_WARPS * 32 - 1) / (K7_WARPS * 32)) * 32;
    const u32 f0 = w * R, f1 = min(f0 + R, Mtot);
    const u32 nch = f1 > f0 ? (f1 - f0 + 31) / 32 : 0;
    u64 key[CH];
    u32 pk[CH];
    if (GROUP) {
        const Model md = S.gmd;
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            pk[q] = NONE;
            key[q] = 0;
            const u32 f = f0 + q * 32 + lane;
            if ((u32)q < nch && f < f1) { key[q] = X[f]; pk[q] = interval_index<K>(key[q], md); }
        }
        const u32 *gT = S.gT;
        const u32 jb = S.gjlo - 1u;
#pragma unroll
        for (int q = 0; q < CH; ++q)
            if (pk[q] != NONE) pk[q] = __ldg(gT + pk[q]) - jb;   // column 1 + (j - jlo)
    } else {
        u32 node = 0, cn = NONE, base = 0;
        int pdelta = 0;
        bool deg = false;
        Model md;
        if (f0 + lane < f1) node = seg_of(S.nkey, N, f0 + lane);
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            pk[q] = NONE;
            key[q] = 0;
            const u32 f = f0 + q * 32 + lane;
            if ((u32)q < nch && f < f1) {
                while (f >= S.nkey[node + 1]) ++node;
                if (node != cn) {
                    cn = node;
                    base = S.nb0[node];
                    pdelta = (int)S.npos[node] - (int)S.nkey[node];
                    deg = S.ndeg[node] != 0;
                    if (!deg) make_model<K>(S.nmin[node], S.nmax[node], S.nP[node], md);
                }
                const u64 x = X[(int)f + pdelta];
                key[q] = x;
                pk[q] = deg ? base + 1 : base + S.T[base + interval_index<K>(x, md)];
            }
        }
    }
    __syncwarp();
    // ---- pass 2: counts per (warp, column) and a rank inside the warp.
    // Group level: stable ranks (Append order; almost every key recurses) with
    // __match_any_sync.  Deeper levels: almost every key goes to a leaf, whose
    // order is irrelevant (it is sorted next), so each key takes an unstable rank
    // from a shared-memory atomic (8 cycles/chunk on B200 vs ~60 for MATCH over
    // ~30 distinct columns); keys of recursing buckets are re-ranked stably at
    // placement time.
    if (GROUP) {
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            if ((u32)q < nch) {
                const u32 u = pk[q];
                const u32 peers = __match_any_sync(0xffffffffu, u);
                const u32 leader = __ffs(peers) - 1;
                u32 old = 0;
                if (u != NONE && lane == leader) { old = S.m.wcnt[w][u]; S.m.wcnt[w][u] = (u16)(old + __popc(peers)); }
                old = __shfl_sync(0xffffffffu, old, leader);
                if (u != NONE) pk[q] = u | ((old + __popc(peers & lanemask_lt())) << 16);
                __syncwarp();
            }
        }
    } else {
        u32 *row32 = reinterpret_cast<u32 *>(S.m.wcnt[w]);
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            if ((u32)q < nch && pk[q] != NONE) {
                const u32 u = pk[q];
                const u32 old = atomicAdd(&row32[u >> 1], (u & 1) ? 0x10000u : 1u);
                pk[q] = u | (((u & 1) ? old >> 16 : old & 0xffffu) << 16);
            }
        }
    }
    __syncthreads();
    if (GROUP) prof_mark(c, S, 2); else prof_mark(c, S, 9);
    // ---- columns: totals, positions (exclusive scan incl. gaps), node of each column (max-scan)
    constexpr u32 CPT = (MC + K7_THREADS - 1) / K7_THREADS;   // columns per thread
    const u32 c0 = tid * CPT;
    u32 h[CPT], mk[CPT];
    u32 sum = 0, mxk = 0;
#pragma unroll
    for (u32 k = 0; k < CPT; ++k) {
        const u32 col = c0 + k;
        h[k] = 0; mk[k] = 0;
        if (col < ncols) {
            mk[k] = S.GM[col];
            if (mk[k]) h[k] = S.ngap[mk[k] - 1];
            else {
                u32 t = 0;
#pragma unroll
                for (u32 ww = 0; ww < (u32)K7_WARPS; ++ww) t += S.m.wcnt[ww][col];
                h[k] = t;
            }
        }
        sum += h[k];
        mxk = mk[k] > mxk ? mk[k] : mxk;
    }
    const u32 isum = warp_incl_scan(sum), imx = warp_incl_max(mxk);
    if (lane == 31) { S.scan_b[w][0] = isum; S.scan_b[w][1] = imx; }
    __syncthreads();
    u32 run = isum - sum;
    u32 rmx = __shfl_up_sync(0xffffffffu, imx, 1);
    if (lane == 0) rmx = 0;
    for (u32 ww = 0; ww < w; ++ww) { run += S.scan_b[ww][0]; rmx = S.scan_b[ww][1] > rmx ? S.scan_b[ww][1] : rmx; }
    // kinds: 0 none/gap/empty, 1 leaf of 2..SMALL_MAX keys, 2 leaf of one key, 3 node, 4 larger leaf
    u32 st[CPT], kd[CPT];
    u32 nl = 0, kl = 0, nn = 0;
#pragma unroll
    for (u32 k = 0; k < CPT; ++k) {
        const u32 col = c0 + k;
        rmx = mk[k] > rmx ? mk[k] : rmx;
        st[k] = run;
        kd[k] = 0;
        if (col < ncols && !mk[k] && rmx) {
            const u32 i = rmx - 1;
            const u32 j = col - S.nb0[i];     // 1-based bucket index of the node
            const u32 hh = h[k];
            const bool deg = GROUP ? false : S.ndeg[i] != 0;
            const u32 delta = GROUP ? S.gdelta : (u32)S.nP[i];
            if (hh) {
                const bool leaf = deg || hh >= delta || hh < tau;   // Alg. 1
                kd[k] = !leaf ? 3u : hh == 1 ? 2u : hh <= SMALL_MAX ? 1u : 4u;
                nn += kd[k] == 3u ? 1u : 0u;
                nl += kd[k] == 1u ? 1u : 0u;
                kl += kd[k] == 1u ? hh : 0u;
                // per-warp destinations of this column
                u32 d = run | (kd[k] == 3u ? 0u : kd[k] == 2u ? DEST_A : DEST_B);
#pragma unroll
                for (u32 ww = 0; ww < (u32)K7_WARPS; ++ww) { const u32 o = S.m.wcnt[ww][col]; S.m.wcnt[ww][col] = (u16)d; d += o; }
                if (kd[k] == 4u) {
                    const u32 sl = atomicAdd(&S.nbleaf, 1u);
                    if (sl < (u32)BLCAP) S.bleaf[sl] = run | (hh << 16);
                    else atomicOr(c->err_flag, 2u);
                }
            }
            if (GROUP) {
                S.gH[S.gjlo + j - 1] = hh;
            } else if (logging && !deg) {
                atomicAdd((unsigned long long *)&S.ndh[i], (unsigned long long)digest_term(j, hh));
                if (hh) atomicAdd(&S.ncnt[i], hh >= delta ? 1u : hh < tau ? (1u << 10) : (1u << 20));
                if (L == 1 && c->l1_h && j - 1 < c->l1_cap) c->l1_h[j - 1] = hh;
            }
        }
        run += h[k];
    }
    // ordered appends: counts of small leaves, their keys, nodes per warp
    const u32 inl = warp_incl_scan(nl), ikl = warp_incl_scan(kl), inn = warp_incl_scan(nn);
    if (lane == 31) { S.scan_c[w][0] = inl; S.scan_c[w][1] = ikl; S.scan_c[w][2] = inn; }
    __syncthreads();
    {
        u32 sl = inl - nl, sk = ikl - kl, sn = S.tail + inn - nn;
        for (u32 ww = 0; ww < w; ++ww) { sl += S.scan_c[ww][0]; sk += S.scan_c[ww][1]; sn += S.scan_c[ww][2]; }
#pragma unroll
        for (u32 k = 0; k < CPT; ++k) {
            if (kd[k] == 1u) { S.leaf[sl] = st[k] | (h[k] << 16); S.lkp[sl] = (u16)sk; ++sl; sk += h[k]; }
            else if (kd[k] == 3u) { S.ring[sn & (RING - 1)] = st[k] | (h[k] << 13); ++sn; }
        }
        if (tid == K7_THREADS - 1) {
            u32 tl = 0, tk = 0, tn = 0;
            for (u32 ww = 0; ww < (u32)K7_WARPS; ++ww) { tl += S.scan_c[ww][0]; tk += S.scan_c[ww][1]; tn += S.scan_c[ww][2]; }
            S.nleaf = tl; S.lkeys = tk; S.lkp[tl] = (u16)tk;
            S.new_tail = S.tail + tn;
        }
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            if ((u32)q < nch) {
                const u32 u = pk[q] & 0xffffu;
                u32 d = 0;
                if (pk[q] != NONE) d = (u32)S.m.wcnt[w][u] + (pk[q] >> 16);
                if (!GROUP) {   // recursing bucket: stable rank (Append order), running per-warp cursor
                    const bool nd = pk[q] != NONE && (d & (DEST_A | DEST_B)) == 0;
                    if (__any_sync(0xffffffffu, nd)) {
                        const u32 peers = __match_any_sync(0xffffffffu, nd ? u : NONE);
                        const u32 leader = __ffs(peers) - 1;
                        u32 base = 0;
                        if (nd && lane == leader) { base = S.m.wcnt[w][u]; S.m.wcnt[w][u] = (u16)(base + __popc(peers)); }
                        base = __shfl_sync(0xffffffffu, base, leader);
                        if (nd) d = base + __popc(peers & lanemask_lt());
                        __syncwarp();
                    }
                }
                if (pk[q] != NONE) {
                    u64 *dst = (d & DEST_A) ? S.A : (d & DEST_B) ? S.B : Y;
                    dst[d & POS_MASK] = key[q];
                }
            }
        }
    }
    __syncthreads();
}

// Node records of the sub-batch (pass log).
template <class K>
__device__ void sub_records(const DevCtx *c, K7Smem &S, u32 L, u64 gbase) {
    for (u32 i = threadIdx.x; i < S.N; i += K7_THREADS) {
        if (S.ndeg[i]) continue;
        const u32 cc = S.ncnt[i];
        write_record(c, L, S.nal[i], gbase + S.npos[i], S.nm[i], K::from_okey(S.nmin[i]), K::from_okey(S.nmax[i]),
                     S.ndb[i], S.ndh[i], cc & 1023u, (cc >> 10) & 1023u, cc >> 20);
    }
}

__device__ __forceinline__ void reset_leaf_lists(K7Smem &S) {
    if (threadIdx.x == 0) { S.item_next = 0; S.nbleaf = 0; S.nleaf = 0; S.lkeys = 0; }
}

// ------------------------------------------------------------------ global I/O
__device__ __forceinline__ ulonglong2 ld_stream2(const ulonglong2 *p) {
    ulonglong2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p));
    return r;
}

// Load src[0, m) into dst (A or B) as ordered keys; returns true if a NaN was seen (f64).
template <class K>
__device__ __forceinline__ bool load_task(u64 *dst, const u64 *src, u32 m) {
    bool nan = false;
    auto put = [&](u32 k, u64 raw) {
        if (K::is_f64) nan |= (raw & 0x7fffffffffffffffull) > 0x7ff0000000000000ull;
        dst[k] = K::to_okey(raw);
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

// Write A[0, m) (sorted ordered keys) to dst as raw keys, 16-byte stores.
template <class K>
__device__ __forceinline__ void store_task(const K7Smem &S, u64 *dst, u32 m) {
    const u32 head = ((uintptr_t)dst & 15) ? 1u : 0u;
    if (head && m && threadIdx.x == 0) dst[0] = K::from_okey(S.A[0]);
    const u32 nv = (m - min(head, m)) / 2;
    ulonglong2 *v = reinterpret_cast<ulonglong2 *>(dst + head);
    for (u32 i = threadIdx.x; i < nv; i += K7_THREADS) {
        ulonglong2 r;
        r.x = K::from_okey(S.A[head + 2 * i]);
        r.y = K::from_okey(S.A[head + 2 * i + 1]);
        v[i] = r;
    }
    if (m > head && ((m - head) & 1) && threadIdx.x == 0) dst[m - 1] = K::from_okey(S.A[m - 1]);
}

// ------------------------------------------------------------------ the kernel
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
            S.head = 0; S.tail = 0; S.level_end = 0;
        }
        reset_leaf_lists(S);
        __syncthreads();
        if (S.task_idx >= ntasks) break;
        prof_mark(c, S, 0);
        const K7Task task = S.task;
        const u64 *src = c->buf[task.src] + task.off;
        u64 *gout = c->buf[2] + task.off;
        const u32 M = task.size;
        const bool sort_task = task.kind == K7_SORT || (task.kind == K7_NODE && M < c->tau);
        const bool nan_here = load_task<K>(sort_task ? S.B : S.A, src, M);
        if (K::is_f64 && task.level == 1 && __syncthreads_or(nan_here)) {
            if (threadIdx.x == 0) atomicOr(c->nan_flag, 1u);
            return;
        }
        __syncthreads();
        prof_mark(c, S, 1);
        if (threadIdx.x == 0 && c->k7_prof) { S.prof[11] += 1; S.prof[12] += M; }
        u32 L = task.level;
        u32 xbuf = 0;   // buffer holding the current level's nodes (0: A, 1: B)
        if (sort_task) {   // the task is one leaf (keys in B)
            if (threadIdx.x == 0) {
                if (M <= SMALL_MAX) { S.leaf[0] = 0u | (M << 16); S.lkp[0] = 0; S.lkp[1] = (u16)M; S.nleaf = 1; S.lkeys = M; }
                else { S.bleaf[0] = 0u | (M << 16); S.nbleaf = 1; }
            }
            __syncthreads();
            leaf_phase(S);
            __syncthreads();
        } else if (task.kind == K7_NODE) {
            if (threadIdx.x == 0) { S.ring[0] = 0u | (M << 13); S.tail = 1; S.level_end = 1; }
            __syncthreads();
        } else {   // K7_GROUP: finish the global node's placement for buckets [jlo, jhi)
            if (threadIdx.x == 0) {
                const GNode &g = c->nodes[task.node];
                S.gmd = g.md; S.gT = g.T; S.gH = g.H;
                S.gdelta = g.delta; S.glevel = g.level; S.gjlo = task.jlo;
                S.N = 1; S.nkey[0] = 0; S.nkey[1] = M; S.nb0[0] = 0; S.nb0[1] = (u16)(task.jhi - task.jlo + 1);
                S.npos[0] = 0; S.nm[0] = (u16)M; S.ngap[0] = 0; S.ndeg[0] = 0;
            }
            for (u32 i = threadIdx.x; i < MC; i += K7_THREADS) S.GM[i] = i == 0 ? 1 : 0;
            __syncthreads();
            sub_place<K, true>(c, S, S.A, S.B, S.glevel);
            prof_mark(c, S, 3);
            leaf_phase(S);
            if (threadIdx.x == 0) { S.tail = S.new_tail; S.level_end = S.tail; }
            reset_leaf_lists(S);
            __syncthreads();
            prof_mark(c, S, 4);
            L = S.glevel + 1;
            xbuf = 1;
        }
        // ---- recursion levels (Alg. 1 on every recursing bucket, level by level)
        for (;;) {
            if (S.head == S.tail) break;
            if (S.head == S.level_end) {   // uniform: shared values read after a barrier
                __syncthreads();
                if (threadIdx.x == 0) S.level_end = S.tail;
                __syncthreads();
                L += 1;
                xbuf ^= 1u;
            }
            u64 *X = xbuf ? S.B : S.A;
            u64 *Y = xbuf ? S.A : S.B;
            sub_setup(c, S);
            prof_mark(c, S, 5);
            sub_minmax(S, X);
            prof_mark(c, S, 6);
            sub_sample<K>(c, S, X, L, task.off);
            prof_mark(c, S, 7);
            sub_fit(c, S, L);
            prof_mark(c, S, 8);
            sub_place<K, false>(c, S, X, Y, L);
            prof_mark(c, S, 10);
            leaf_phase(S);
            if (c->rec) sub_records<K>(c, S, L, task.off);
            if (threadIdx.x == 0) {
                S.head += S.N;
                S.tail = S.new_tail;
                if (S.tail - S.head > (u32)RING) atomicOr(c->err_flag, 2u);
            }
            reset_leaf_lists(S);
            __syncthreads();
            prof_mark(c, S, 4);
        }
        store_task<K>(S, gout, M);
        prof_mark(c, S, 13);
        __syncthreads();
    }
    if (c->k7_prof && threadIdx.x == 0)
        for (int i = 0; i < K7_PROF_SLOTS; ++i) atomicAdd(&c->k7_prof[i], S.prof[i]);
}

}  // namespace pcf
