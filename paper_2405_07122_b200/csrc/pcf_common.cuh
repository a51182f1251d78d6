// pcf_common.cuh -- shared device definitions of the B200 PCF Learned Sort.
//
// Implements, independently of oracle/ (no shared code), the written specs of
// the ordered-key transform for IEEE totalOrder (R11), i(x) with
// explicitly rounded binary64 ops (R6, R15), floor(m^{3/4}) in exact 128-bit
// integers (R5), the counter-based sampler (R3, R4), the bucket table
// T[i] = floor(b_i*gamma/alpha)+1 (R7) and the order-independent digest (§3.4).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pcf {

typedef unsigned long long u64;
typedef unsigned int u32;
typedef unsigned short u16;
typedef unsigned char u8;

// ---------------------------------------------------------------- tunables
#ifndef PCF_S_CAP
#define PCF_S_CAP 8192
#endif
constexpr int S_CAP = PCF_S_CAP;             // keys a K7 CTA holds (two 64 KB buffers)
constexpr int NB_CAP = 862;              // max buckets of one K7 CTA-level partition (>= iroot34(S_CAP) + 1)
constexpr int WMAX = 1024;               // largest segment a single warp runs Alg. 1 on
constexpr int WNB = 184;                 // >= iroot34(WMAX) + 2 (warp scratch bins)
constexpr int WSTACK = 320;              // warp DFS stack entries (bound: DESIGN.md §5.3)
#ifndef PCF_GMAX
#define PCF_GMAX 1024
#endif
constexpr int GMAX = PCF_GMAX;           // digits per global split pass (a power of two)
static_assert((GMAX & (GMAX - 1)) == 0 && GMAX >= 256, "GMAX must be a power of two >= 256");
constexpr unsigned GMAX_LOG2 = GMAX >= 4096 ? 12 : GMAX >= 2048 ? 11 : GMAX >= 1024 ? 10 : GMAX >= 512 ? 9 : 8;
constexpr int SPLIT_THREADS = 512;       // split count kernel block
constexpr int SC_WARPS = 12;             // split scatter: warps per CTA
constexpr int SC_THREADS = SC_WARPS * 32;
#ifndef PCF_SC_KPL
#define PCF_SC_KPL 14
#endif
constexpr int SC_KPL = PCF_SC_KPL;             // keys per lane held in registers (2 CTAs/SM with the u32 rank counters)
constexpr int SC_PER_WARP = SC_KPL * 32; // 512 consecutive keys per warp
constexpr int SPLIT_TILE = SC_WARPS * SC_PER_WARP;   // 5376 keys per split tile
constexpr u64 GOLDEN = 0x9E3779B97F4A7C15ull;
#define K7_PROF_SLOTS_DECL 24

// ---------------------------------------------------------------- debug bounds checks
// compute-sanitizer is not available on the GPU pool, so a debug build
// (-DPCF_CHECKS=1, tools/checks.sh) asserts the shared- and global-memory index
// bounds of the hot kernels: a violation sets err_flag bit 5 and the call returns
// PCF_ERR_INTERNAL (the GPU parity suite run against that build must stay green).
#ifndef PCF_CHECKS
#define PCF_CHECKS 0
#endif
#define PCF_CHECK(ctx, cond)                                                              \
    do {                                                                                  \
        if (PCF_CHECKS && !(cond)) atomicOr((ctx)->err_flag, 32u);                        \
    } while (0)

// ---------------------------------------------------------------- key transforms
// totalOrder on binary64 == unsigned order of the "flipped" bits: set the sign
// bit of non-negative patterns, complement negative ones (R11).
struct KeyF64 {
    static constexpr bool is_f64 = true;
    __host__ __device__ static inline u64 to_okey(u64 raw) {
        return raw ^ ((u64)((long long)raw >> 63) | 0x8000000000000000ull);
    }
    __host__ __device__ static inline u64 from_okey(u64 k) {   // (k >> 63) ? k ^ sign : ~k
        return k ^ (~(u64)((long long)k >> 63) | 0x8000000000000000ull);
    }
};
struct KeyU64 {
    static constexpr bool is_f64 = false;
    __host__ __device__ static inline u64 to_okey(u64 raw) { return raw; }
    __host__ __device__ static inline u64 from_okey(u64 k) { return k; }
};

// ---------------------------------------------------------------- model of one bucketing node
// i(x) = floor((x - x_min) / (x_max - x_min) * beta) + 1
struct Model {
    double xmin;    // f64: x_min as a double
    double r;       // fl(x_max - x_min)  (f64)  or  RN(x_max - x_min) (u64, R15)
    double betad;   // (double)beta, exact
    double s;       // fl(beta / r): fast-path scale (NaN disables the fast path)
    double eps;     // beta * 2^-48: fast-path guard band
    u64 umin;       // u64: x_min
    u32 beta;
    u32 pad;
};

// Reading R6 evaluated exactly as written: d = x - x_min, q = d / r, t = q * beta,
// every op binary64 round-to-nearest-even, i = floor(t) + 1.
#ifndef PCF_EXACT_INLINE
#define PCF_EXACT_INLINE 0
#endif
#if PCF_EXACT_INLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
u32 interval_index_exact(double d, double r, double betad) {
    const double q = __ddiv_rn(d, r);
    const double t = __dmul_rn(q, betad);
    return __double2uint_rz(t) + 1u;   // t in [0, beta]  (R6: no clamp needed)
}

// Certified fast path for the same value.  With u = 2^-53 and
// every intermediate normal, the exact t = fl(fl(d/r)*beta) and the estimate
// t' = fl(d*s), s = fl(beta/r), satisfy t/t' = (1+e1)(1+e2)/((1+e3)(1+e4)),
// |e_k| <= u, so |t - t'| <= 4.0001 u t' <= 4.0001 u beta (1 + 4u) < eps =
// 2^-48 beta = 32 u beta.  Hence if frac(t') lies in [eps, 1 - eps], t lies in
// the same open unit interval (floor(t'), floor(t') + 1) and floor(t) =
// floor(t').  frac(t') >= eps also forces t' >= eps >= 32u, i.e. q and d*s
// normal, so the relative bounds apply; a subnormal or huge s is replaced by
// NaN in make_model (every comparison with NaN fails -> exact path), as is any
// t' that is NaN or infinite.  Keys inside the band (x_max itself, keys within
// a few ulps of a bin edge) take the exact path.
template <class K>
__device__ __forceinline__ double key_offset(u64 okey, const Model &md) {   // d = x - x_min (R6, R15)
    if (K::is_f64) return __dsub_rn(__longlong_as_double((long long)K::from_okey(okey)), md.xmin);
    return __ull2double_rn(okey - md.umin);
}
// The same d from the raw key bits (no ordered-key round trip: for f64 keys
// from_okey(to_okey(raw)) == raw, which the compiler cannot see).
template <class K>
__device__ __forceinline__ double key_offset_raw(u64 raw, const Model &md) {
    if (K::is_f64) return __dsub_rn(__longlong_as_double((long long)raw), md.xmin);
    return __ull2double_rn(raw - md.umin);
}
#ifndef PCF_FAST_FLOOR
#define PCF_FAST_FLOOR 0
#endif
__device__ __forceinline__ u32 fast_from_offset(double d, const Model &md, bool &ok) {
    const double t = __dmul_rn(d, md.s);
#if PCF_FAST_FLOOR
    // floor(t') without the conversion pipe (FRND / F2I): m = RN(RN(t' - 0.5) + 1.5 * 2^52) holds the
    // integer nearest to t' - 0.5 in its low mantissa bits (0 <= t' <= beta < 2^32; t' - 0.5 is exact
    // for t' >= 0.5, and a tiny t' fails the band test below anyway), which is floor(t') whenever
    // frac(t') is not 0; an integer t' (a tie) gives fl = t' or t' - 1, i.e. fr = 0 or 1, and the
    // band test sends it to the exact path like every other key within eps of a bin edge.
    const double MAGIC = 6755399441055744.0;   // 1.5 * 2^52
    const double m = __dadd_rn(__dadd_rn(t, -0.5), MAGIC);
    const double fl = __dsub_rn(m, MAGIC);
    const double fr = __dsub_rn(t, fl);
    ok = fr >= md.eps && fr <= 1.0 - md.eps;
    return (u32)__double2loint(m) + 1u;
#else
    const double fl = floor(t);
    const double fr = __dsub_rn(t, fl);
    ok = fr >= md.eps && fr <= 1.0 - md.eps;
    return (u32)fl + 1u;
#endif
}
// Branch-free fast path: floor(t') + 1 and whether it is certified (ok); the
// caller takes interval_index_exact for the rare uncertified keys.
template <class K>
__device__ __forceinline__ u32 interval_index_fast(u64 okey, const Model &md, bool &ok) {
    return fast_from_offset(key_offset<K>(okey, md), md, ok);
}
template <class K>
__device__ __forceinline__ u32 interval_index_fast_raw(u64 raw, const Model &md, bool &ok) {
    return fast_from_offset(key_offset_raw<K>(raw, md), md, ok);
}
template <class K>
__device__ __forceinline__ u32 interval_index(u64 okey, const Model &md) {
    double d;
    if (K::is_f64) {
        double x = __longlong_as_double((long long)K::from_okey(okey));
        d = __dsub_rn(x, md.xmin);
    } else {
        d = __ull2double_rn(okey - md.umin);
    }
    const double t = __dmul_rn(d, md.s);
    const double fl = floor(t);
    const double fr = __dsub_rn(t, fl);
    if (fr >= md.eps && fr <= 1.0 - md.eps) return (u32)fl + 1u;
    return interval_index_exact(d, md.r, md.betad);
}

// Build the model from the node's ordered min/max keys.  Returns false when
// the range is degenerate (not 0 < r < inf, R9/R10): Standard-Sort instead.
template <class K>
__device__ inline bool make_model(u64 kmin, u64 kmax, u32 beta, Model &md) {
    md.beta = beta;
    md.betad = (double)beta;
    md.pad = 0;
    bool ok;
    if (K::is_f64) {
        double xa = __longlong_as_double((long long)K::from_okey(kmin));
        double xb = __longlong_as_double((long long)K::from_okey(kmax));
        md.xmin = xa;
        md.umin = 0;
        md.r = __dsub_rn(xb, xa);
        ok = (md.r > 0.0) && (md.r <= 1.7976931348623157e308);
    } else {
        md.xmin = 0.0;
        md.umin = kmin;
        md.r = __ull2double_rn(kmax - kmin);
        ok = kmax > kmin;
    }
    const double s = ok ? __ddiv_rn(md.betad, md.r) : 0.0;
    md.s = (s >= 0x1p-1000 && s <= 0x1p1000) ? s : __longlong_as_double(0x7ff8000000000000ll);
    md.eps = __dmul_rn(md.betad, 0x1p-48);
    return ok;
}

// ---------------------------------------------------------------- floor(m^{3/4})  (R5)
__host__ __device__ inline u64 iroot34(u64 m) {
    if (m == 0) return 0;
    unsigned __int128 m3 = (unsigned __int128)m * m * m;   // m < 2^32 here
    u64 c = (u64)pow((double)m, 0.75);
    auto p4 = [](u64 c) -> unsigned __int128 {
        unsigned __int128 c2 = (unsigned __int128)c * c;
        return c2 * c2;
    };
    while (c > 0 && p4(c) > m3) --c;
    while (p4(c + 1) <= m3) ++c;
    return c;
}

// ---------------------------------------------------------------- sampler (R3, R4)
__host__ __device__ __forceinline__ u64 mix64(u64 z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ u64 node_key(u64 seed, u32 level, u64 o) {
    return mix64(seed ^ mix64(o + (u64)level * GOLDEN));
}
__device__ __forceinline__ u64 sample_pos(u64 nkey, u64 k, u64 m) {
    return __umul64hi(mix64(nkey + (k + 1) * GOLDEN), m);
}
// digest term of v_i at 1-based index i
__host__ __device__ __forceinline__ u64 digest_term(u64 i1, u32 v) { return mix64((i1 << 32) ^ (u64)v); }

// T[i] = floor(b_i * gamma / alpha) + 1   (R7; = b_i + 1 when alpha == gamma)
__host__ __device__ __forceinline__ u32 bucket_of(u32 b, u32 alpha, u32 gamma) {
    if (alpha == gamma) return b + 1;
    return (u32)(((u64)b * gamma) / alpha) + 1;
}

// ---------------------------------------------------------------- device records
struct NodeRec {   // == pcf_node_record (72 bytes)
    u32 level, alpha;
    u64 offset, m;
    u64 xmin_bits, xmax_bits;
    u64 digest_b, digest_h;
    u32 n_fallback, n_small, n_recurse, reserved;
};

// A bucketing node run by the global (multi-CTA) path.
struct GNode {
    u64 off;        // global offset of the segment (= its position in every buffer)
    u32 m;          // segment length
    u32 level;
    u64 kmin, kmax; // ordered keys (atomicMin/atomicMax targets)
    u32 alpha, beta, gamma, delta;
    u32 src;        // buffer holding the segment (0 in, 1 tmp, 2 out)
    u32 degenerate; // 1: range not in (0, inf) -> Standard-Sort
    Model md;
    u32 *cnt;       // [beta+2]  per-bin sample counts, then b (inclusive prefix), 1-based
    u32 *T;         // [beta+2]  bucket table, 1-based
    u32 *H;         // [gamma+2] bucket sizes, 1-based (written by the split/K7 leaves)
    u64 digest_b;
    // digit boundaries of the node's first split (large nodes; NULL otherwise):
    // bnd[d] = first bin i whose digit (T[i] - 1) >> bshift is >= d, d in [1, bG)
    u32 *bnd;
    u32 bshift, bG;
};

// Work item of the smem-subtree kernel (K7).
enum : u32 { K7_GROUP = 0, K7_NODE = 1, K7_SORT = 2 };
struct K7Task {
    u64 off;        // global offset == buffer position of the first key
    u32 size;
    u32 kind;       // K7_GROUP: buckets [jlo, jhi) of global node `node`
    u32 src;        // buffer holding the keys
    u32 level;      // K7_NODE: level of this node; K7_GROUP: level of `node`
    u32 node;
    u32 jlo, jhi;
    u32 pad;        // K7_SORT: 1 = the keys are all equal (copied, not sorted)
};

// A global split: stable partition of a segment by digit (j - jlo) >> shift.
struct SplitTask {
    u64 off;
    u32 m;
    u32 node;
    u32 jlo, jhi;   // bucket range of the segment (1-based, half-open)
    u32 shift, G;   // G = ceil((jhi - jlo) / 2^shift) <= GMAX
    u32 src, dst;
    u32 tile_begin, ntiles;  // filled by the host plan
    u64 cbase;      // offset of this split's digit-major count matrix
    u64 mbase;      // sum of m over earlier splits of the same launch
};

// Items the split leaves for the host (large recursing buckets / fallback).
struct SegItem {
    u64 off;
    u32 m;
    u32 level;      // level the segment would be processed at
    u32 src;
    u32 kind;       // 0 = recurse (new global node), 1 = fallback sort
};

// Sizes of one split round, computed on the device by k_round_plan.
struct RoundPlan {
    u32 ns;        // splits processed this round
    u32 tiles;     // total tiles
    u32 nblk;      // scan blocks over the count matrix
    u32 next_scan;    // block tickets of the count-matrix scan (k_scanp_lookback)
    u32 pad_;
    u32 cur;       // split list this round consumes (splits[cur]); the next round's is cur ^ 1
    u64 ctot;      // count-matrix entries
    u64 mtot;      // keys moved
};

// The batch of global nodes created on the device from the oversized recursing
// buckets of the previous batch (k_items_to_nodes): nodes [first, first + nb),
// their tables in arena[a0, a1), and the CTA chunk prefix sums of the batched
// min/max (MMB_CHUNK keys per chunk) and sampling (FSB_CHUNK samples) kernels.
struct BatchInfo {
    u32 first, nb;
    u32 mm_chunks, fs_chunks;   // totals
    u64 a0, a1;
};

// Device counters of one sort (zeroed / initialised by the host at the start of
// every call; read back only when the caller asks for a synchronous call).
struct Counters {
    u32 nan_flag, err_flag, k7_count, k7_next;
    u32 nsplits[2], nitems, k7_begin;
    unsigned long long rec_count, k7_keys, split_keys, global_keys;
    RoundPlan plan;
    u32 round, node_count, pad0, iters;   // iters: device-driven batches run
    unsigned long long arena_used, fb_keys;   // fb_keys: keys of Standard-Sort buckets > S_CAP
    BatchInfo batch;
    unsigned long long k7_prof[K7_PROF_SLOTS_DECL];
};

struct DevCtx {
    u64 *buf[3];            // in (const, never written unless in==out), tmp, out
    u32 *ibuf[3];           // key-value mode: the source index of every
                            // key of buf[i] (ibuf[0] == NULL: identity), or all NULL (keys only)
    Counters *cnt;          // device counters of this call
    u64 n;
    u64 gbase;              // global position of buffer position 0 (a shard of a sharded sort; else 0):
                            // sampler keys (R4) and node records use gbase + offset
    u64 seed;
    u32 tau;
    u32 flags;
    u32 root_external;      // sharded sort: node 0 is the global level-1 node, fitted across
                            // ranks; its record is written only where root_external == 2
    GNode *nodes;
    // K7 queue
    K7Task *k7;
    u32 *k7_order;          // claim order of the current K7 launch's tasks (largest first), or NULL
    u32 *k7_count;
    u32 k7_cap;
    u32 *k7_next;
    u32 *k7_begin;          // first task of the current K7 launch
    // split rounds, planned on the device: round r consumes splits[r & 1] and
    // appends the next round's splits to splits[(r + 1) & 1]
    SplitTask *splits[2];
    u32 *nsplits;           // [2]
    u32 splits_cap;
    struct RoundPlan *plan;
    u32 *cmat, *pmat, *bsum;
    unsigned long long *scan_status;   // per scan block: flag << 32 | value (k_scanp_lookback; zeroed by k_round_plan)
    u64 cmat_cap;
    unsigned long long *split_keys;   // keys moved by split passes (byte accounting)
    unsigned long long *k7_prof;      // PCF_FLAG_PROFILE: K7 cycles per phase (NULL = off)
    u16 *digs;              // split digit of the key at each array position (count -> scatter)
    u32 *tmap;              // split of each tile of the current round (k_tile_map)
    SegItem *items;
    u32 *nitems;
    u32 items_cap;
    // status
    u32 *nan_flag;
    u32 *err_flag;          // bit0 capacity overflow, bit1 internal
    unsigned long long *k7_keys;   // keys handed to K7 (for the byte accounting)
    // device-driven batches (k_items_to_nodes): node table and arena capacities,
    // CTA chunk prefix sums of the current batch
    u32 node_cap;
    u32 *arena;
    u64 arena_cap;
    u32 *bpre_mm, *bpre_fs;   // [node_cap + 1]
    // pass log
    NodeRec *rec;
    unsigned long long *rec_count;
    u64 rec_cap;
    u32 *l1_b, *l1_h;
    u64 l1_cap;
};

// ---------------------------------------------------------------- bulk copies (TMA, 1D) + mbarriers
__device__ __forceinline__ u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64 *b, u32 n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// one arrival that also announces `tx` bytes of bulk copies completing on the barrier
__device__ __forceinline__ void mbar_arrive_tx(u64 *b, u32 tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64 *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void named_bar(u32 id, u32 nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *b, u32 parity) {
    asm volatile("{\n\t.reg .pred p;\n\tW%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra W%=;\n\t}" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
// global -> shared bulk copy; dst, src 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, u32 bytes, u64 *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
// shared -> global bulk copy (16-byte aligned addresses and size) in the issuing thread's bulk group
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, u32 bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(dst), "r"(smem_u32(src)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }   // sources read
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }         // writes done
// generic-proxy accesses of a shared buffer before it is refilled by the async proxy
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Programmatic dependent launch: every kernel of the sort's chain first waits
// for its predecessor grid (complete, memory visible) and then lets its own
// successor start launching, so launch latency overlaps the tail of the
// previous kernel.  (No-ops for a kernel launched without the attribute.)
__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

constexpr u32 FLAG_SAMPLE_ALL = 2u;
constexpr u32 FLAG_EXACT_RANKS = 16u;
constexpr int K7_PROF_SLOTS = K7_PROF_SLOTS_DECL;

}  // namespace pcf
