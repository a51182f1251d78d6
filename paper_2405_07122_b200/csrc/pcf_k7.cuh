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
// Work split inside the CTA:
//  * CTA-wide (16 warps): the K7_GROUP placement by the global model, and any
//    node of more than 2 GCAP keys (its children are < delta <= 861 keys).
//  * Every other node is run, start to finish, by as few warps as hold its keys
//    in registers (<= 16 per thread): double teams of 8 warps (nodes <= 4096,
//    named barriers 5-6), teams of 4 (<= 2048, barriers 1-4), single warps
//    (<= 512, with their whole subtrees, depth-first on a per-warp stack).
//    A node step: min/max, alpha seeded samples (R3) -> per-bin
//    counts, b = prefix, T, classify + per-warp counts, one
//    column pass (bucket sizes, destinations, Alg. 1 lines 160-167 dispatch),
//    placement, and Standard-Sort of the leaf buckets.  Teams publish their
//    children to a small-node list that the single warps drain; no set of warps
//    waits for another inside a task.  The next task is claimed early and
//    bulk-copied into B while the current one is written out.
//  * Buffers: a node at relative depth r lives in A (r even) or B (r odd);
//    recursing buckets are placed into the other buffer, leaf buckets of
//    >= 2 keys into B (scratch) and then sorted into A, single keys straight
//    into A.  Every position ends in A, sorted.
//  * Stable placement (Append order; readings R4, R16): warp
//    w of a group owns a contiguous range of the node's keys.  Leaf keys take an
//    unstable rank from a shared-memory atomic (their bucket is sorted next);
//    keys of recursing buckets are re-ranked stably (chunk order, MATCH) when
//    they are placed.  The K7_GROUP placement ranks every key stably.
#pragma once
#include "pcf_common.cuh"

namespace pcf {

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
__device__ __forceinline__ u64 warp_sum_u64(u64 v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
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

// Key-value mode: the tie-break of equal keys is their task-local source index
// (IA / IB), i.e. input order -- the stable permutation (reading R18).
template <bool PR>
__device__ __forceinline__ u32 tie_of(const u16 *I, u32 j) { return PR ? (u32)I[j] : j; }

// ------------------------------------------------------------------ Standard-Sort (R2) on ordered keys
// Rank of (v, p) among (B[j], j), j in [st, st + h): keys below v, and equal
// keys before p.  One 96-bit subtract chain per comparison; PTX's carry after
// it is set iff (B[j], j) >= (v, p), so r counts the others and rank = h - r.
template <bool PR = false>
__device__ __forceinline__ u32 rank_in_leaf(const u64 *B, u32 st, u32 h, u64 v, u32 p, const u16 *IB = nullptr) {
    u32 r = 0;
    const u32 vlo = (u32)v, vhi = (u32)(v >> 32);
    for (u32 j = st; j < st + h; ++j) {
        const u64 x = B[j];
        asm("{\n\t.reg .u32 t;\n\t"
            "sub.cc.u32 t, %1, %2;\n\t"
            "subc.cc.u32 t, %3, %4;\n\t"
            "subc.cc.u32 t, %5, %6;\n\t"
            "addc.u32 %0, %0, 0;\n\t}"
            : "+r"(r) : "r"(tie_of<PR>(IB, j)), "r"(p), "r"((u32)x), "r"(vlo), "r"((u32)(x >> 32)), "r"(vhi));
    }
    return h - r;
}

// ------------------------------------------------------------------ Standard-Sort of a whole task (R2)
// Sort the NT * 8 ordered keys at X (keys-only; positions >= m are padding) into Y by
// one CTA of NT threads: each thread sorts 8 keys with Batcher's 19-comparator network,
// each warp merges its runs up to 256 keys in registers (bitonic merges over lane
// shuffles), then log2(NT / 32) merge-path levels through shared memory (each thread
// emits 8 consecutive outputs).  Padding (~0) sorts last.  X and Y are both written;
// the result ends in Y.  Ends with __syncthreads().
__device__ __forceinline__ void cx8(u64 &a, u64 &b) { const u64 x = a < b ? a : b; b = a < b ? b : a; a = x; }
__device__ __forceinline__ u32 mp_split(const u64 *A, u32 la, const u64 *B, u32 lb, u32 d) {   // A first among equal keys
    u32 lo = d > lb ? d - lb : 0, hi = d < la ? d : la;
    while (lo < hi) {
        const u32 mid = (lo + hi) >> 1;
        if (A[mid] <= B[d - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    return lo;
}
template <int NT>
__device__ void block_sort_tile(u64 *X, u64 *Y, u32 m) {
    constexpr u32 IPT = 8, TILE = NT * IPT;
    const u32 t = threadIdx.x, L = t & 31, t0 = t * IPT;
    u64 r[IPT];
#pragma unroll
    for (u32 k = 0; k < IPT; ++k) {   // rotated loads (fewer bank conflicts); the network sorts them anyway
        const u32 p = t0 + ((k + t) & (IPT - 1));
        r[k] = p < m ? X[p] : ~0ull;
    }
    cx8(r[0], r[1]); cx8(r[2], r[3]); cx8(r[4], r[5]); cx8(r[6], r[7]);
    cx8(r[0], r[2]); cx8(r[1], r[3]); cx8(r[4], r[6]); cx8(r[5], r[7]);
    cx8(r[1], r[2]); cx8(r[5], r[6]);
    cx8(r[0], r[4]); cx8(r[1], r[5]); cx8(r[2], r[6]); cx8(r[3], r[7]);
    cx8(r[2], r[4]); cx8(r[3], r[5]);
    cx8(r[1], r[2]); cx8(r[3], r[4]); cx8(r[5], r[6]);
    // runs of 16 .. 256 keys inside the warp: element i = 8 lane + q; each stage compares i with
    // its mirror i ^ (k - 1), then half-cleaners i ^ j
#pragma unroll
    for (u32 k = 16; k <= 32u * IPT; k <<= 1) {
        {
            const bool lo = (L & (k / (2 * IPT))) == 0;
            u64 pv[IPT];
#pragma unroll
            for (int q = 0; q < (int)IPT; ++q) pv[q] = __shfl_xor_sync(0xffffffffu, r[IPT - 1 - q], k / IPT - 1);
#pragma unroll
            for (int q = 0; q < (int)IPT; ++q) r[q] = (lo == (pv[q] < r[q])) ? pv[q] : r[q];
        }
#pragma unroll
        for (u32 j = k / 4; j >= 1; j >>= 1) {
            if (j >= IPT) {
                const bool lo = (L & (j / IPT)) == 0;
#pragma unroll
                for (int q = 0; q < (int)IPT; ++q) {
                    const u64 pv = __shfl_xor_sync(0xffffffffu, r[q], j / IPT);
                    r[q] = (lo == (pv < r[q])) ? pv : r[q];
                }
            } else {
#pragma unroll
                for (u32 q = 0; q < IPT; ++q)
                    if (!(q & j)) cx8(r[q], r[q | j]);
            }
        }
    }
    // merge levels 256 -> TILE through shared memory; an odd number of levels starts in X
    constexpr u32 LEVELS = NT >= 1024 ? 5 : NT >= 512 ? 4 : NT >= 256 ? 3 : NT >= 128 ? 2 : 1;
    static_assert((32u << LEVELS) == (u32)NT, "NT must be a power of two >= 64");
    u64 *sa = (LEVELS & 1) ? X : Y, *sb = (LEVELS & 1) ? Y : X;
    __syncthreads();   // every thread's loads of X are done
#pragma unroll
    for (u32 k = 0; k < IPT; ++k) sa[t0 + k] = r[k];
    __syncthreads();
    for (u32 run = 32 * IPT; run < TILE; run <<= 1) {
        const u32 p0 = (t0 / (2 * run)) * (2 * run), d = t0 - p0;
        const u64 *A = sa + p0, *B = sa + p0 + run;
        u32 ia = mp_split(A, run, B, run, d), ib = d - ia;
        u64 xa = ia < run ? A[ia] : ~0ull, xb = ib < run ? B[ib] : ~0ull;
#pragma unroll
        for (u32 k = 0; k < IPT; ++k) {
            const bool ta = ib >= run || (ia < run && xa <= xb);
            r[k] = ta ? xa : xb;
            if (ta) { ++ia; xa = ia < run ? A[ia] : ~0ull; }
            else { ++ib; xb = ib < run ? B[ib] : ~0ull; }
        }
#pragma unroll
        for (u32 k = 0; k < IPT; ++k) sb[t0 + k] = r[k];
        __syncthreads();
        u64 *tmp = sa; sa = sb; sb = tmp;
    }
}

// ------------------------------------------------------------------ global I/O
__device__ __forceinline__ ulonglong2 ld_stream2(const ulonglong2 *p) {
    ulonglong2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p));
    return r;
}

}  // namespace pcf

// The K7 body is compiled twice (pcf_k7_body.cuh): 512 threads (16 keys per
// thread in registers; every tau) and 1024 threads (8 keys per thread, a quad
// team tier; node lists sized for tau >= K7W_MIN_TAU, keys-only mode).  The host
// picks one per sort (pcf_api.cu: k7_wide).
#ifndef PCF_K7_NS0
#define PCF_K7_NS0 32      // small-list wait: first back-off (ns)
#endif
#ifndef PCF_K7_NSMAX
#define PCF_K7_NSMAX 512   // small-list wait: largest back-off (ns; longer sleeps delay the task end)
#endif
#ifndef PCF_K7_LEAFB
#define PCF_K7_LEAFB 1     // leaf sort: positions per thread whose loads are batched (2, 4: more spills, slower)
#endif
#ifndef PCF_K7_RELOAD
#define PCF_K7_RELOAD 1    // re-read the node's keys before placement instead of keeping them live
#endif
#ifndef PCF_K7_RELOAD2
#define PCF_K7_RELOAD2 0   // also re-read the keys before classify (not kept live through sampling and fit)
#endif
#ifndef PCF_K7_BULKST
#define PCF_K7_BULKST 1    // keys-only: store the finished task by one asynchronous bulk copy (overlaps the next task)
#endif
#ifndef PCF_K7_NPROF
#define PCF_K7_NPROF 0     // per-phase cycles of team nodes (profiling builds only)
#endif
#define PCF_K7_NT 512
namespace pcf { namespace k7n512 {
#include "pcf_k7_body.cuh"
} }
#undef PCF_K7_NT
#define PCF_K7_NT 1024
namespace pcf { namespace k7n1024 {
#include "pcf_k7_body.cuh"
} }
#undef PCF_K7_NT
