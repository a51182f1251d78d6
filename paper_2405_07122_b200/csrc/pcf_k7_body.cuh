// pcf_k7_body.cuh -- the K7 kernel for one block size PCF_K7_NT (included twice
// by pcf_k7.cuh inside pcf::k7n512 / pcf::k7n1024; see pcf_k7.cuh for the design).
// No include guard on purpose.
constexpr int K7_THREADS = PCF_K7_NT;
constexpr int K7_WARPS = K7_THREADS / 32;


constexpr int GW = 4;                              // warps per team
constexpr int NGRP = K7_WARPS / GW;                // teams per CTA
constexpr int GT = GW * 32;                        // threads per team
constexpr int KPT = S_CAP / K7_THREADS;            // keys per thread held in registers (16)
constexpr int GCAP = GT * KPT;                     // largest node a team runs (2048)
constexpr int WCAP = 32 * KPT;                     // largest node a single warp runs (512)
constexpr int CCOLS = NB_CAP + 2;                  // counter columns (CTA view): >= iroot34(S_CAP) + 2 = 863
constexpr int WCOLS = K7_THREADS >= 1024 ? 72 : 128;   // T / size columns per warp slice: >= iroot34(WCAP) + 2 (66 / 109);
                                                   // a team's slices give 512 >= iroot34(GCAP) + 2 = 306
constexpr u32 SMALL_MAX = 64;                      // leaves up to this size: key-parallel rank sort
// Node lists live after K7Smem, sized for tau (nodes hold >= tau keys): the
// small-node list holds <= S_CAP / tau entries (+ one over-claimed ticket per
// warp), a warp's DFS stack <= WCAP / tau.  For the default tau = 64 that is
// ~1 KB instead of the 33 KB tau = 2 needs, which leaves L1 to the T gathers.
__host__ __device__ inline u32 k7_list_cap(u32 tau) { return (u32)S_CAP / tau > 0 ? (u32)S_CAP / tau : 1u; }
__host__ __device__ inline u32 k7_lsm_cap(u32 tau) { return k7_list_cap(tau) + K7_WARPS + 16; }
__host__ __device__ inline u32 k7_stk_cap(u32 tau) { return (u32)WCAP / tau > 0 ? (u32)WCAP / tau : 1u; }
__host__ __device__ inline size_t k7_lists_bytes(u32 tau) { return 4ull * (k7_lsm_cap(tau) + (u64)K7_WARPS * k7_stk_cap(tau)); }
constexpr int LBIG_CAP = 32;                       // nodes > WCAP keys of one task (<= 16)
constexpr int TBIG_CAP = 16;                       // children > WCAP of one team node: <= 4096 / 257
constexpr int STK_CAP = WCAP / 2;                  // per-warp DFS stack
constexpr int BL_CAP = 128;                        // leaves > SMALL_MAX keys of one node: <= S_CAP / 65
constexpr int BL_W = BL_CAP / K7_WARPS;            // per-warp slice (a warp's node has <= 7)
constexpr u32 NONE = 0xffffffffu;
// destination entries: node-relative position | target (Y: recursing bucket,
// A: leaf of one key -- final, B: larger leaf -- sorted into A next)
constexpr u32 DEST_A = 0x4000u, DEST_B = 0x8000u, POS_MASK = 0x3fffu;
constexpr int TCOLS = K7_WARPS * WCOLS > CCOLS ? K7_WARPS * WCOLS : CCOLS;   // CTA view of the column arrays
static_assert((CCOLS * 2) % 4 == 0, "counter rows must stay 4-byte aligned");
// 1024-thread builds add a tier of 4-team groups (4 GW warps, nodes of (2 GCAP, 4 GCAP] keys)
constexpr bool QUAD = K7_WARPS >= 8 * GW;
constexpr u32 CTA_MIN = (QUAD ? 4u : 2u) * (u32)GCAP;   // nodes above this size run on the whole CTA

// node entry: pos (13 bits) | m << 13 (14 bits) | relative depth << 27
__device__ __forceinline__ u32 ent_make(u32 pos, u32 m, u32 rel) { return pos | (m << 13) | (rel << 27); }
__device__ __forceinline__ u32 ent_pos(u32 e) { return e & 0x1fffu; }
__device__ __forceinline__ u32 ent_m(u32 e) { return (e >> 13) & 0x3fffu; }
__device__ __forceinline__ u32 ent_rel(u32 e) { return e >> 27; }

struct K7Smem {
    u64 A[S_CAP];
    u64 B[S_CAP + 2];             // + 2: the next task's bulk copy may start 8 bytes early
    u16 W[K7_WARPS * CCOLS];      // per-warp column counters -> destinations (rows of CCOLS);
                                  // a group's rows double as its u32 per-bin sample counts
    u16 T16[TCOLS];    // bucket table of the current node (slices of the node's warps)
    u16 hcol[TCOLS];   // bucket sizes of the current node (same slices)
    u16 LC[S_CAP];                // per position: bucket column of a B-leaf key, 0 otherwise
    u32 lbig[LBIG_CAP];           // nodes > WCAP keys
    // children of > WCAP keys of a double / quad team's node (1024-thread builds: nodes of
    // (1630, CTA_MIN] keys can have them), run next by the same team; per first warp
    u32 tbig[K7_WARPS][TBIG_CAP];
    u32 tbn[K7_WARPS];
    u32 bl[BL_CAP];               // leaves > SMALL_MAX keys of the current node (slices of the node's warps)
    u64 wmn[K7_WARPS], wmx[K7_WARPS];
    u32 wsum[K7_WARPS];
    // per node, indexed by the node's first warp
    unsigned long long db[K7_WARPS], dh[K7_WARPS];
    u32 ncnt[K7_WARPS];           // pass log: nf | ns << 10 | nr << 20
    u32 nbl[K7_WARPS];
    u32 top[K7_WARPS], cur[K7_WARPS], cur2[K7_WARPS], cur4[K7_WARPS];   // node claimed per team tier
    u32 stot, snext, btot, bnext, bnext2, bnext4, big_active;
    u32 task_idx, nidx;
    K7Task task, ntask;
    u32 lhead, ldirect;           // the loaded task: first key at B[lhead]; ldirect: not bulk-copied
    u64 tbar;                     // mbarrier of the task bulk copy
    Model gmd;
    const u32 *gT;
    u32 *gH;
    u32 gdelta, glevel, gjlo, gjhi;
    Model ngmd;                   // the same for the claimed next task (K7_GROUP), fetched with the claim
    const u32 *ngT;
    u32 *ngH;
    u32 ngdelta, nglevel;
    long long prof_t;                       // PCF_FLAG_PROFILE bookkeeping (thread 0)
    unsigned long long prof[K7_PROF_SLOTS];
    u16 *IA, *IB;                 // key-value mode (PR): task-local source index of every position
                                  // of A / B (dynamic shared memory past the lists), else NULL
    u32 *lsm;                     // nodes <= WCAP keys (tickets; 0 = not yet pushed)   [lsm_cap]
    u32 *stk;                     // per-warp DFS stacks, row w at stk + w * stk_cap (a team's rows:
                                  // its children before publication)                     [K7_WARPS * stk_cap]
    u32 lsm_cap, list_cap, stk_cap;
    unsigned char tail[];         // the lists (dynamic shared memory past the struct)
};

static_assert(K7_THREADS < 1024 || sizeof(K7Smem) + 4 * ((S_CAP / 32) + K7_WARPS + 16 + K7_WARPS * (WCAP / 32)) <= 232448,
              "K7 shared memory (1024 threads, tau = 32) exceeds 227 KB");
static_assert(K7_THREADS > 512 || sizeof(K7Smem) + 4 * ((S_CAP / 2) + K7_WARPS + 16 + K7_WARPS * (WCAP / 2)) <= 232448,
              "K7 shared memory (tau = 2) exceeds 227 KB");

// K7 phase profiling (PCF_FLAG_PROFILE): thread 0 charges the cycles since the
// previous mark to slot `id` (barrier waits included).  Slots: 0 claim, 1 load,
// 2 group placement (CTA), 4 CTA-run nodes, 5 node groups, 6 sort tasks,
// 11 tasks, 12 keys, 13 store.
__device__ __forceinline__ void prof_mark(const DevCtx *c, K7Smem &S, int id) {
    if (c->k7_prof && threadIdx.x == 0) {
        long long t = clock64();
        S.prof[id] += (unsigned long long)(t - S.prof_t);
        S.prof_t = t;
    }
}

// A set of NW warps that runs one node: the whole CTA (barrier 0) or a node
// group (named barrier g + 1).
template <int NW>
struct Grp {
    static constexpr int NT = NW * 32;
    u32 g;    // named barrier of the set (0: the CTA)
    u32 t;    // thread index inside the set
    u32 w0;   // first CTA warp of the set
    __device__ __forceinline__ void bar() const {
        if (NW == K7_WARPS) __syncthreads();
        else if (NW == 1) __syncwarp();
        else asm volatile("bar.sync %0, %1;" ::"r"(g), "r"(NT) : "memory");
    }
};

// Bitonic network over a[0, n) by a thread set; all merges ascending (the
// first step of each stage compares i with its mirror), so the virtual +inf
// padding never moves.
// compare-exchange of positions lo < hi: (key, tie) ascending; key-value mode
// carries (and breaks ties by) the source index
template <bool PR>
__device__ __forceinline__ void cx_pos(u64 *a, u16 *ia, u32 lo, u32 hi) {
    const u64 x = a[lo], y = a[hi];
    if (PR) {
        const u16 ix = ia[lo], iy = ia[hi];
        if (x > y || (x == y && ix > iy)) { a[lo] = y; a[hi] = x; ia[lo] = iy; ia[hi] = ix; }
    } else if (x > y) {
        a[lo] = y; a[hi] = x;
    }
}

template <int NW, bool PR = false>
__device__ void set_bitonic(u64 *a, u32 n, const Grp<NW> &G, u16 *ia = nullptr) {
    constexpr u32 NT = NW * 32;
    if (n <= 1) return;
    const u32 P = next_pow2(n);
    const u32 lgP = 31 - __clz(P);
    for (u32 lk = 1; lk <= lgP; ++lk) {
        const u32 k = 1u << lk, lh = lk - 1;
        for (u32 t = G.t; t < (P >> 1); t += NT) {
            const u32 blk = t >> lh, w = t & ((1u << lh) - 1);
            const u32 lo = (blk << lk) + w, hi = (blk << lk) + k - 1 - w;
            if (hi < n) cx_pos<PR>(a, ia, lo, hi);
        }
        G.bar();
        for (int lj = (int)lh - 1; lj >= 0; --lj) {
            const u32 j = 1u << lj;
            for (u32 t = G.t; t < (P >> 1); t += NT) {
                const u32 lo = ((t >> lj) << (lj + 1)) + (t & (j - 1)), hi = lo + j;
                if (hi < n) cx_pos<PR>(a, ia, lo, hi);
            }
            G.bar();
        }
    }
}

// Standard-Sort of the leaf B[st, st + h) into A[st, st + h) by a thread set.
// Ends with a barrier of the set.
template <int NW, bool PR = false>
__device__ void sort_range(K7Smem &S, u32 st, u32 h, const Grp<NW> &G) {
    constexpr u32 NT = NW * 32;
    if (h <= SMALL_MAX) {
        for (u32 p = st + G.t; p < st + h; p += NT) {
            const u32 r = st + rank_in_leaf<PR>(S.B, st, h, S.B[p], tie_of<PR>(S.IB, p), S.IB);
            S.A[r] = S.B[p];
            if (PR) S.IA[r] = S.IB[p];
        }
    } else {
        set_bitonic<NW, PR>(S.B + st, h, G, PR ? S.IB + st : nullptr);
        for (u32 p = st + G.t; p < st + h; p += NT) { S.A[p] = S.B[p]; if (PR) S.IA[p] = S.IB[p]; }
    }
    G.bar();
}

// ------------------------------------------------------------------ one bucketing node
// MODE_NODE:   a Learned-Sort call on keys X[pos, pos + m) (Alg. 1 lines
//              148-167; m >= tau): min/max, model, samples, fit, bucketing,
//              dispatch of every bucket, Standard-Sort of the leaves, record.
// MODE_GLOBAL: the K7_GROUP placement: model and T of the global node,
//              columns = buckets [jlo, jhi); keys in A[0, m).
// Recursing buckets become node entries: a single warp keeps them on its own
// stack; a team publishes them to the small-node list after placement; the CTA
// appends them to the task's lists by size.  Ends with a barrier of the set.
enum { MODE_NODE = 0, MODE_GLOBAL = 1 };

// i(x) of every valid slot (pk != NONE) into pk: certified fast path for all
// slots, the exact sub/div/mul evaluation (R6) only for the rare keys in the
// guard band, behind one warp-uniform branch.
// RAW: key[] holds the raw key bits (the K7_GROUP placement), else ordered keys.
template <class K, bool RAW = false>
__device__ __forceinline__ void classify_slots(const u64 (&key)[KPT], u32 (&pk)[KPT], const Model &md) {
    u32 bad = 0;
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
        bool ok;
        const u32 i = RAW ? interval_index_fast_raw<K>(key[q], md, ok) : interval_index_fast<K>(key[q], md, ok);
        const bool v = pk[q] != NONE;
        bad |= (v && !ok) ? (1u << q) : 0u;
        pk[q] = v ? i : NONE;
    }
    if (__any_sync(0xffffffffu, bad != 0)) {
#pragma unroll
        for (int q = 0; q < KPT; ++q)
            if (bad & (1u << q))
                pk[q] = interval_index_exact(RAW ? key_offset_raw<K>(key[q], md) : key_offset<K>(key[q], md), md.r, md.betad);
    }
}

template <class K, int NW, int MODE, bool PR, bool LOG>
__device__ void node_step(const DevCtx *c, K7Smem &S, const Grp<NW> &G, u32 pos, u32 m, u32 L, u32 rel, u64 gbase,
                          const u64 *raw = nullptr) {   // MODE_GLOBAL: raw keys (bulk-copied task) instead of A
    constexpr u32 NT = NW * 32;
    constexpr bool CTA = NW == K7_WARPS;
    // bins / columns per thread: node <= S_CAP (CTA, 862 bins; 1024 group columns) or <= GCAP (group, 305)
    constexpr u32 BPT = CTA ? 2 : NW == 1 ? 4 : 3;   // warp: node <= WCAP, 108 bins; double team: <= 2 GCAP, 513
    const u32 t = G.t, g = G.g, w = warp_id(), wg = w - G.w0, lane = lane_id();
    u64 *X = (rel & 1) ? S.B : S.A;
    u64 *Y = (rel & 1) ? S.A : S.B;
    u16 *IX = (rel & 1) ? S.IB : S.IA;   // key-value mode: source indices (NULL otherwise)
    u16 *IY = (rel & 1) ? S.IA : S.IB;
    u16 *Wg = S.W + G.w0 * CCOLS;
    u16 *Wrow = Wg + wg * CCOLS;
    u32 *row32 = reinterpret_cast<u32 *>(Wrow);
    u32 *cnt = reinterpret_cast<u32 *>(Wg);
    const u32 w0 = G.w0;
    u16 *T16 = S.T16 + w0 * WCOLS;
    u16 *hc = S.hcol + w0 * WCOLS;
    u32 *bl = S.bl + w0 * BL_W;
    constexpr bool logging = LOG;   // pass log on (c->rec != NULL): a separate kernel instance
    const u32 tau = c->tau;
    // PCF_K7_NPROF builds: cycles of each phase of the 4-warp team nodes (thread 0 of the
    // team; slots 3, 14, 15, 20-23: minmax, samples, fit, classify, columns, placement, leaves)
    constexpr bool NPROF = PCF_K7_NPROF && MODE == MODE_NODE && NW == GW;
    long long np_t = (NPROF && t == 0 && c->k7_prof) ? clock64() : 0;
    auto nmark = [&](int slot) {
        if (NPROF && t == 0 && c->k7_prof) {
            const long long x = clock64();
            atomicAdd(&S.prof[slot], (unsigned long long)(x - np_t));
            np_t = x;
        }
    };

    // ---- this thread's keys: warp wg owns [f0, f1), chunk q = 32 consecutive keys
    const u32 R = ((m + NT - 1) / NT) * 32;
    const u32 f0 = wg * R, f1 = min(f0 + R, m);
    const u32 nch = f1 > f0 ? (f1 - f0 + 31) / 32 : 0;   // uniform per warp
    // All KPT slots are processed branch-free (slots past the warp's range load
    // the node's first key and are marked NONE), so the unrolled loops compile
    // to straight-line code with the keys in registers.
    u64 key[KPT];
    u32 pk[KPT];
    u32 ix2[PR ? KPT / 2 : 1];   // key-value mode: two u16 source indices per register
    u64 mn = ~0ull, mx = 0;
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
        const u32 f = f0 + q * 32 + lane;
        const bool v = f < f1;
        // the K7_GROUP placement classifies raw key bits (converted to ordered keys after)
        key[q] = MODE == MODE_GLOBAL ? (raw ? raw[v ? f : 0u] : K::from_okey(X[pos + (v ? f : 0u)])) : X[pos + (v ? f : 0u)];
        if (PR) {
            const u32 i = (MODE == MODE_GLOBAL && raw) ? f : (u32)IX[pos + (v ? f : 0u)];
            if (q & 1) ix2[q / 2] |= i << 16; else ix2[q / 2] = i & 0xffffu;
        }
        pk[q] = v ? 0u : NONE;
        mn = v && key[q] < mn ? key[q] : mn;
        mx = v && key[q] > mx ? key[q] : mx;
    }
    auto idx_of = [&](int q) -> u16 { return PR ? (u16)((q & 1) ? ix2[q / 2] >> 16 : ix2[q / 2] & 0xffffu) : (u16)0; };

    if (c->k7_prof && t == 0) {   // node statistics: slots 7/8 group nodes / keys, 9/10 CTA nodes / keys
        atomicAdd(&S.prof[CTA ? 9 : 7], 1ull);
        atomicAdd(&S.prof[CTA ? 10 : 8], (unsigned long long)m);
    }
    u32 P = 0, alpha = 0, ncol, delta;
    Model md;
    if (MODE == MODE_NODE) {
        P = iroot34_small(m);
        alpha = (c->flags & FLAG_SAMPLE_ALL) ? m : P;
        ncol = P + 1;
        delta = P;
        for (u32 i = t; i < P + 2; i += NT) cnt[i] = 0;
        mn = warp_min_u64(mn);
        mx = warp_max_u64(mx);
        if (lane == 0) { S.wmn[w] = mn; S.wmx[w] = mx; }
        if (t == 0) { S.db[w0] = 0; S.dh[w0] = 0; S.ncnt[w0] = 0; S.nbl[w0] = 0; if (NW > 1 && !CTA) S.top[w0] = 0; }
        G.bar();
        nmark(3);
        mn = S.wmn[G.w0];
        mx = S.wmx[G.w0];
#pragma unroll
        for (int i = 1; i < NW; ++i) {
            const u64 a = S.wmn[G.w0 + i], b = S.wmx[G.w0 + i];
            mn = a < mn ? a : mn;
            mx = b > mx ? b : mx;
        }
        if (!make_model<K>(mn, mx, P, md)) {
            // R9/R10: the whole node goes to Standard-Sort (no bucketing, no record)
            if (!(rel & 1)) {
#pragma unroll
                for (int q = 0; q < KPT; ++q)
                    if (pk[q] != NONE) { S.B[pos + f0 + q * 32 + lane] = key[q]; if (PR) S.IB[pos + f0 + q * 32 + lane] = idx_of(q); }
            }
            G.bar();
            sort_range<NW, PR>(S, pos, m, G);
            return;
        }
        // ---- alpha samples (R3, R4) -> per-bin counts
        {
            const bool all = (c->flags & FLAG_SAMPLE_ALL) != 0;
            const u64 nk = node_key(c->seed, L, gbase + pos);
            for (u32 s = t; s < alpha; s += NT) {
                const u32 p = all ? s : (u32)sample_pos(nk, s, m);
                atomicAdd(&cnt[interval_index<K>(X[pos + p], md)], 1u);
            }
        }
        G.bar();
        nmark(14);
        if (CTA && MODE == MODE_NODE) prof_mark(c, S, 3);
        // ---- fit: b = inclusive prefix over bins 1..P+1, T = floor(b*gamma/alpha)+1 (R7)
        {
            const u32 e0 = 1 + t * BPT;
            u32 v[BPT], loc = 0;
#pragma unroll
            for (u32 k = 0; k < BPT; ++k) { v[k] = e0 + k <= P + 1 ? cnt[e0 + k] : 0; loc += v[k]; }
            const u32 incl = warp_incl_scan(loc);
            if (lane == 31) S.wsum[w] = incl;
            G.bar();
            u32 run = incl - loc;
            for (u32 i = 0; i < wg; ++i) run += S.wsum[G.w0 + i];
            for (u32 i = lane; i < (P + 3) / 2; i += 32) row32[i] = 0;   // counts are dead: zero this warp's row
            u64 db = 0;
#pragma unroll
            for (u32 k = 0; k < BPT; ++k) {
                const u32 e = e0 + k;
                run += v[k];
                if (e <= P + 1) {
                    T16[e] = (u16)bucket_of(run, alpha, P);
                    if (logging) {
                        db += digest_term(e, run);
                        if (L == 1 && c->l1_b && e - 1 < c->l1_cap) c->l1_b[e - 1] = run;
                    }
                }
            }
            if (logging) {
                db = warp_sum_u64(db);
                if (lane == 0) atomicAdd(&S.db[w0], (unsigned long long)db);
            }
        }
        G.bar();
        nmark(15);
        // ---- classify (i(x) -> T) and count per (warp, column); unstable rank
#if PCF_K7_RELOAD2
        // the keys were dead through sampling and the fit: re-read them (X is unchanged until placement)
#pragma unroll
        for (int q = 0; q < KPT; ++q) {
            const u32 f = f0 + q * 32 + lane;
            key[q] = X[pos + (f < f1 ? f : 0u)];
            pk[q] = f < f1 ? 0u : NONE;
        }
#endif
        classify_slots<K>(key, pk, md);
#pragma unroll
        for (int q = 0; q < KPT; ++q) {
            const bool v = pk[q] != NONE;
            PCF_CHECK(c, !v || (pk[q] >= 1u && pk[q] <= P + 1 && w0 * WCOLS + P + 1 < (u32)TCOLS));
            const u32 u = T16[v ? pk[q] : 1u];
            u32 old = 0;
            PCF_CHECK(c, !v || (u >= 1u && u <= ncol));
            if (v) old = atomicAdd(&row32[u >> 1], (u & 1) ? 0x10000u : 1u);
            pk[q] = v ? u | ((((u & 1) ? old >> 16 : old) & 0xffffu) << 16) : NONE;
        }
    } else {
        md = S.gmd;
        ncol = S.gjhi - S.gjlo;
        delta = S.gdelta;
        for (u32 i = lane; i < (ncol + 2) / 2; i += 32) row32[i] = 0;
        if (t == 0) S.nbl[w0] = 0;
        const u32 *gT = S.gT;
        const u32 jb = S.gjlo - 1u;
        classify_slots<K, true>(key, pk, md);
#pragma unroll
        for (int q = 0; q < KPT; ++q) key[q] = K::to_okey(key[q]);
#pragma unroll
        for (int q = 0; q < KPT; ++q) {
            const bool v = pk[q] != NONE;
            u32 j = 0;
            PCF_CHECK(c, !v || (pk[q] >= 1u && pk[q] <= md.beta + 1));
            if (v) j = __ldg(gT + pk[q]);
            pk[q] = v ? j - jb : NONE;   // column 1 + (j - jlo)
        }
        __syncwarp();
        // stable ranks (Append order): chunk by chunk, MATCH per chunk
#pragma unroll
        for (int q = 0; q < KPT; ++q) {
            if ((u32)q < nch) {
                const u32 u = pk[q];
                const u32 peers = __match_any_sync(0xffffffffu, u);
                const u32 leader = __ffs(peers) - 1;
                u32 old = 0;
                if (u != NONE && lane == leader) { old = Wrow[u]; Wrow[u] = (u16)(old + __popc(peers)); }
                old = __shfl_sync(0xffffffffu, old, leader);
                if (u != NONE) pk[q] = u | ((old + __popc(peers & lanemask_lt())) << 16);
                __syncwarp();
            }
        }
    }
    G.bar();
    nmark(20);
    if (CTA && MODE == MODE_NODE) prof_mark(c, S, 14);

    // ---- column pass: sizes, positions, Alg. 1 lines 160-167 dispatch, destinations per warp
    {
        const u32 c0 = 1 + t * BPT;
        u32 h[BPT], sum = 0;
#pragma unroll
        for (u32 k = 0; k < BPT; ++k) {
            const u32 col = c0 + k;
            h[k] = 0;
            if (col <= ncol) {
#pragma unroll
                for (int ww = 0; ww < NW; ++ww) h[k] += Wg[ww * CCOLS + col];
            }
            sum += h[k];
        }
        const u32 isum = warp_incl_scan(sum);
        if (lane == 31) S.wsum[w] = isum;
        G.bar();
        u32 run = isum - sum;
        for (u32 i = 0; i < wg; ++i) run += S.wsum[G.w0 + i];
        u32 ncc = 0;
        unsigned long long dh = 0;
#pragma unroll
        for (u32 k = 0; k < BPT; ++k) {
            const u32 col = c0 + k;
            if (col <= ncol) {
                const u32 hh = h[k];
                hc[col] = (u16)hh;
                if (hh) {
                    const bool leaf = hh >= delta || hh < tau;   // Alg. 1
                    u32 d = run | (!leaf ? 0u : hh == 1 ? DEST_A : DEST_B);
#pragma unroll
                    for (int ww = 0; ww < NW; ++ww) { const u32 o = Wg[ww * CCOLS + col]; Wg[ww * CCOLS + col] = (u16)d; d += o; }
                    if (!leaf) {
                        const u32 e = ent_make(pos + run, hh, rel + 1);
                        if (hh > (u32)WCAP) {   // too large for one warp: the CTA's big list / the team's own
                            if (CTA) {
                                const u32 sl = atomicAdd(&S.btot, 1u);
                                if (sl < (u32)LBIG_CAP) S.lbig[sl] = e; else atomicOr(c->err_flag, 2u);
                            } else {
                                const u32 sl = atomicAdd(&S.tbn[w0], 1u);
                                if (NW > 1 && sl < (u32)TBIG_CAP) S.tbig[w0][sl] = e; else atomicOr(c->err_flag, 2u);
                            }
                        } else if (CTA) {
                            const u32 sl = atomicAdd(&S.stot, 1u);
                            if (sl < S.list_cap) S.lsm[sl] = e; else atomicOr(c->err_flag, 2u);
                        } else {   // warp: own stack; team: staged in its warps' stacks (contiguous rows)
                            const u32 sl = atomicAdd(&S.top[w0], 1u);
                            if (sl < S.stk_cap * NW) S.stk[w0 * S.stk_cap + sl] = e; else atomicOr(c->err_flag, 2u);
                        }
                    } else if (hh > SMALL_MAX) {
                        const u32 sl = atomicAdd(&S.nbl[w0], 1u);
                        if (sl < (u32)(BL_W * NW)) bl[sl] = run | (hh << 13);
                        else atomicOr(c->err_flag, 2u);
                    }
                    ncc += hh >= delta ? 1u : hh < tau ? (1u << 10) : (1u << 20);
                }
                if (MODE == MODE_GLOBAL) {
                    S.gH[S.gjlo + col - 1] = hh;
                } else if (logging) {
                    dh += digest_term(col, hh);
                    if (L == 1 && c->l1_h && col - 1 < c->l1_cap) c->l1_h[col - 1] = hh;
                }
                run += hh;
            }
        }
        if (MODE == MODE_NODE && logging) {
            dh = warp_sum_u64(dh);
            for (int o = 16; o > 0; o >>= 1) ncc += __shfl_xor_sync(0xffffffffu, ncc, o);
            if (lane == 0) { atomicAdd(&S.dh[w0], dh); atomicAdd(&S.ncnt[w0], ncc); }
        }
    }
#if PCF_K7_RELOAD
    // the keys are dead from classify to placement: re-read them (still intact: nothing is
    // written before the barrier below) instead of holding 2 x KPT registers across the column pass
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
        const u32 f = f0 + q * 32 + lane;
        const u32 ff = f < f1 ? f : 0u;
        key[q] = (MODE == MODE_GLOBAL && raw) ? K::to_okey(raw[ff]) : X[pos + ff];
    }
#endif
    // the K7_GROUP placement is the task's first write to A: the previous task's bulk store has read it
    if (PCF_K7_BULKST && !PR && MODE == MODE_GLOBAL && threadIdx.x == 0) bulk_wait_read();
    G.bar();
    nmark(21);

    // ---- placement (chunk order: stable re-rank of recursing keys)
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
        {
            const u32 u = pk[q] & 0xffffu;
            const bool valid = pk[q] != NONE;
            u32 d = valid ? (u32)Wrow[u] + (pk[q] >> 16) : 0u;
            if (MODE == MODE_NODE) {
                const bool nd = valid && (d & (DEST_A | DEST_B)) == 0;
                if (__any_sync(0xffffffffu, nd)) {
                    const u32 peers = __match_any_sync(0xffffffffu, nd ? u : NONE);
                    const u32 leader = __ffs(peers) - 1;
                    u32 base = 0;
                    if (nd && lane == leader) { base = Wrow[u]; Wrow[u] = (u16)(base + __popc(peers)); }
                    base = __shfl_sync(0xffffffffu, base, leader);
                    if (nd) d = base + __popc(peers & lanemask_lt());
                    __syncwarp();
                }
            }
            const u32 p = pos + (d & POS_MASK);
            u64 *dst = (d & DEST_A) ? S.A : (d & DEST_B) ? S.B : Y;
            if (valid) {
                PCF_CHECK(c, p < pos + m && (d & POS_MASK) < m && u <= ncol);
                dst[p] = key[q];
                if (PR) ((d & DEST_A) ? S.IA : (d & DEST_B) ? S.IB : IY)[p] = idx_of(q);
                S.LC[p] = (d & DEST_B) ? (u16)u : (u16)0;
            }
        }
    }
    G.bar();
    nmark(22);
    if (CTA && MODE == MODE_NODE) prof_mark(c, S, 15);
    if (NW > 1 && !CTA) {   // team: publish the children (their keys are placed) to the small-node list
        const u32 nc = S.top[w0];
        if (nc) {
            __threadfence_block();
            for (u32 i = t; i < nc; i += NT) {
                const u32 sl = atomicAdd(&S.stot, 1u);
                if (sl < S.list_cap) *(volatile u32 *)&S.lsm[sl] = S.stk[w0 * S.stk_cap + i]; else atomicOr(c->err_flag, 2u);
            }
        }
    }

    // ---- Standard-Sort of the leaves: <= SMALL_MAX keys key-parallel, larger ones by bitonic networks
    // (a thread's positions p = t + q NT, q < KPT, in batches of LB: the dependent shared-memory
    // loads of a batch -- leaf column, its size and start, the key -- are issued together)
    constexpr int LB = PCF_K7_LEAFB;
    for (int q0 = 0; q0 < KPT; q0 += LB) {
        if (t + (u32)q0 * NT >= m) break;
        u32 lc[LB], lh[LB], ls[LB];
        u64 lv[LB];
#pragma unroll
        for (int q = 0; q < LB; ++q) { const u32 p = t + (u32)(q0 + q) * NT; lc[q] = p < m ? (u32)S.LC[pos + p] : 0u; }
#pragma unroll
        for (int q = 0; q < LB; ++q) {
            const u32 p = t + (u32)(q0 + q) * NT;
            lh[q] = lc[q] ? (u32)hc[lc[q]] : 0u;
            ls[q] = pos + ((u32)Wg[lc[q]] & POS_MASK);
            lv[q] = S.B[pos + (p < m ? p : 0u)];
        }
#pragma unroll
        for (int q = 0; q < LB; ++q) {
            const u32 p = t + (u32)(q0 + q) * NT;
            if (!lc[q] || lh[q] > SMALL_MAX) continue;
            const u32 r = ls[q] + rank_in_leaf<PR>(S.B, ls[q], lh[q], lv[q], tie_of<PR>(S.IB, pos + p), S.IB);
            PCF_CHECK(c, r >= ls[q] && r < ls[q] + lh[q] && ls[q] + lh[q] <= pos + m);
            S.A[r] = lv[q];
            if (PR) S.IA[r] = S.IB[pos + p];
        }
    }
    const u32 nb = S.nbl[w0];
    for (u32 i = 0; i < nb; ++i) {
        const u32 e = bl[i];
        const u32 st = pos + (e & 0x1fffu), hh = e >> 13;
        set_bitonic<NW, PR>(S.B + st, hh, G, PR ? S.IB + st : nullptr);
        for (u32 p = st + t; p < st + hh; p += NT) { S.A[p] = S.B[p]; if (PR) S.IA[p] = S.IB[p]; }
    }
    if (MODE == MODE_NODE && logging && t == 0) {
        const u32 cc = S.ncnt[w0];
        write_record(c, L, alpha, gbase + pos, m, K::from_okey(mn), K::from_okey(mx), S.db[w0], S.dh[w0],
                     cc & 1023u, (cc >> 10) & 1023u, cc >> 20);
    }
    G.bar();
    nmark(23);
}


// Load src[0, m) into dst (A or B) as ordered keys; returns true if a NaN was seen (f64).
template <class K, bool PR>
__device__ __forceinline__ bool load_task(u64 *dst, u16 *idst, const u64 *src, u32 m) {
    bool nan = false;
    auto put = [&](u32 k, u64 raw) {
        if (K::is_f64) nan |= (raw & 0x7fffffffffffffffull) > 0x7ff0000000000000ull;
        dst[k] = K::to_okey(raw);
        if (PR) idst[k] = (u16)k;
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

// Key-value mode: the global source index of the task's output positions,
// perm[off + p] = index of the key (ibuf[src][off + IA[p]], identity for the input
// buffer), gathered into registers before any thread writes (ibuf[src] may be the
// destination array itself).
template <bool PR>
__device__ __forceinline__ void store_task_idx(const DevCtx *c, const K7Smem &S, const K7Task &t, u32 m) {
    if (!PR) return;
    const u32 *isrc = c->ibuf[t.src];
    u32 g[KPT];
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
        const u32 p = threadIdx.x + q * K7_THREADS;
        g[q] = 0;
        if (p < m) {
            const u32 i = S.IA[p];
            g[q] = isrc ? isrc[t.off + i] : (u32)(t.off + i);
        }
    }
    __syncthreads();
    u32 *idst = c->ibuf[2] + t.off;
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
        const u32 p = threadIdx.x + q * K7_THREADS;
        if (p < m) idst[p] = g[q];
    }
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

// The same by one bulk copy (PCF_K7_BULKST, keys-only): A is converted to raw keys in place --
// shifted down by one key when dst is not 16-byte aligned, so that the shared and the global
// address of the copied body are both aligned; the odd first / last key is stored directly --
// and thread 0 issues the copy, which runs while the CTA starts its next task.  A must not be
// written before thread 0 has waited for the copy's reads (bulk_wait_read) and a barrier.
template <class K>
__device__ __forceinline__ void store_task_bulk(K7Smem &S, u64 *dst, u32 m) {
    const u32 sh = ((uintptr_t)dst & 15) ? 1u : 0u;
    u64 r[KPT];
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
        const u32 i = threadIdx.x + q * K7_THREADS;
        r[q] = i < m ? K::from_okey(S.A[i]) : 0ull;
    }
    const u32 body = (m - min(sh, m)) & ~1u;   // keys [sh, sh + body) go by the bulk copy
    if (sh) __syncthreads();                    // in-place shift: every key is read before any is written
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
        const u32 i = threadIdx.x + q * K7_THREADS;
        if (i < m) {
            if (i < sh || i >= sh + body) dst[i] = r[q];
            else S.A[i - sh] = r[q];
        }
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0 && body) bulk_s2g(dst + sh, S.A, body * 8u);
}

// ------------------------------------------------------------------ the kernel
// Bulk copy of the raw keys of task t into B (issued while the previous task
// is stored).  The copy covers the 16-byte aligned superset of the task; a task
// whose superset leaves the buffer is loaded by plain loads instead.
__device__ __forceinline__ void k7_issue(const DevCtx *c, K7Smem &S, const K7Task &t) {
    const u64 *base = c->buf[t.src];
    const uintptr_t a = (uintptr_t)(base + t.off);
    const uintptr_t a0 = a & ~(uintptr_t)15, a1 = (a + 8ull * t.size + 15) & ~(uintptr_t)15;
    S.lhead = (u32)((a - a0) >> 3);
    if (a0 < (uintptr_t)base || a1 > (uintptr_t)(base + c->n)) {
        S.ldirect = 1;
        mbar_arrive_tx(&S.tbar, 0);
    } else {
        S.ldirect = 0;
        fence_proxy_async();
        mbar_arrive_tx(&S.tbar, (u32)(a1 - a0));
        bulk_g2s(S.B, (const void *)a0, (u32)(a1 - a0), &S.tbar);
    }
}

// Thread 0, with the claim of the next task: the global node's model and tables of a K7_GROUP task
// (read by its placement), so that the task does not start with a chain of global loads.
__device__ __forceinline__ void k7_fetch_node(const DevCtx *c, K7Smem &S) {
    if (S.ntask.kind == K7_GROUP) {
        const GNode &gn = c->nodes[S.ntask.node];
        S.ngmd = gn.md; S.ngT = gn.T; S.ngH = gn.H;
        S.ngdelta = gn.delta; S.nglevel = gn.level;
    }
}

// Node entry of size m from the CTA phases: big list (> WCAP keys) or small list.
__device__ __forceinline__ void push_root(const DevCtx *c, K7Smem &S, u32 e) {
    if (ent_m(e) > (u32)WCAP) {
        const u32 sl = atomicAdd(&S.btot, 1u);
        if (sl < (u32)LBIG_CAP) S.lbig[sl] = e; else atomicOr(c->err_flag, 2u);
    } else {
        const u32 sl = atomicAdd(&S.stot, 1u);
        if (sl < S.list_cap) S.lsm[sl] = e; else atomicOr(c->err_flag, 2u);
    }
}

// One team tier: every set of NW warps claims nodes of (lo, hi] keys from the
// task's big list and runs them until none is left.
template <class K, int NW, bool PR, bool LOG>
__device__ __forceinline__ void run_tier(const DevCtx *c, K7Smem &S, const Grp<NW> &G, u32 *ctr, u32 *cur, u32 lo, u32 hi,
                                         u32 Lb, u64 gb, bool wprof, unsigned long long &wc) {
    for (;;) {
        if (G.t == 0) {
            u32 e = 0;
            if (S.tbn[G.w0] > 0) {   // the team's own children of > WCAP keys first (< delta(hi) keys: fit)
                e = S.tbig[G.w0][--S.tbn[G.w0]];
            } else {
                for (;;) {
                    const u32 i = atomicAdd(ctr, 1u);
                    if (i >= S.btot) break;
                    e = S.lbig[i];
                    if (ent_m(e) > lo && ent_m(e) <= hi) break;
                    e = 0;
                }
            }
            cur[G.w0] = e;
        }
        G.bar();
        const u32 e = cur[G.w0];
        if (!e) break;
        const long long t0 = wprof ? clock64() : 0;
        node_step<K, NW, MODE_NODE, PR, LOG>(c, S, G, ent_pos(e), ent_m(e), Lb + ent_rel(e), ent_rel(e), gb);
        if (wprof) wc += clock64() - t0;
    }
}

template <class K, bool PR, bool LOG>
__global__ void __launch_bounds__(K7_THREADS, K7_THREADS >= 512 ? 1 : 2) k7_kernel(const DevCtx *__restrict__ c) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char k7_smem_raw[];
    K7Smem &S = *reinterpret_cast<K7Smem *>(k7_smem_raw);
    if (*c->nan_flag) return;
    constexpr bool BULKST = PCF_K7_BULKST && !PR;   // the finished task leaves by an asynchronous bulk copy
    const u32 ntasks = *c->k7_count;
    const u32 begin = *c->k7_begin;
    const u32 w = warp_id(), lane = lane_id();
    const Grp<K7_WARPS> CT{0u, threadIdx.x, 0u};
    const Grp<GW> GG{1 + w / GW, threadIdx.x % GT, (w / GW) * GW};            // barriers 1..4
    const Grp<2 * GW> GH{1 + NGRP + w / (2 * GW), threadIdx.x % (2 * GT), (w / (2 * GW)) * (2 * GW)};   // 5..6
    const Grp<1> GS{w, lane, w};
    const Grp<(QUAD ? 4 * GW : 1)> GQ{1 + NGRP + NGRP / 2 + w / (4 * GW), threadIdx.x % (4 * GT), (w / (4 * GW)) * (4 * GW)};
    if (threadIdx.x == 0) {
        S.lsm_cap = k7_lsm_cap(c->tau); S.list_cap = k7_list_cap(c->tau); S.stk_cap = k7_stk_cap(c->tau);
        S.lsm = reinterpret_cast<u32 *>(S.tail);
        S.stk = S.lsm + S.lsm_cap;
        S.IA = PR ? reinterpret_cast<u16 *>(S.stk + K7_WARPS * S.stk_cap) : nullptr;
        S.IB = PR ? S.IA + S_CAP : nullptr;
    }
    __syncthreads();
    for (u32 i = threadIdx.x; i < S.lsm_cap; i += K7_THREADS) S.lsm[i] = 0;   // tickets read 0 until pushed
    if (threadIdx.x < (u32)K7_WARPS) S.tbn[threadIdx.x] = 0;   // (each team empties its own list)
    if (c->k7_prof && threadIdx.x == 0) {
        for (int i = 0; i < K7_PROF_SLOTS; ++i) S.prof[i] = 0;
        S.prof_t = clock64();
    }
    if (threadIdx.x == 0) {   // first task: claim + bulk copy
        mbar_init(&S.tbar, 1);
        mbar_init_fence();
        S.nidx = begin + atomicAdd(c->k7_next, 1u);
        if (S.nidx < ntasks) { S.ntask = c->k7[c->k7_order ? c->k7_order[S.nidx] : S.nidx]; k7_issue(c, S, S.ntask); k7_fetch_node(c, S); }
    }
    __syncthreads();
#ifndef PCF_K7_WPROF
#define PCF_K7_WPROF 0   // per-warp busy / wait cycles (slots 16-19): profiling builds only (costs registers)
#endif
    const bool wprof = PCF_K7_WPROF && c->k7_prof != nullptr && lane == 0;
    unsigned long long wcyc[4] = {0, 0, 0, 0};
    for (u32 it = 0;; ++it) {
        if (threadIdx.x == 0) {
            S.task_idx = S.nidx;
            S.task = S.ntask;
            S.gmd = S.ngmd; S.gT = S.ngT; S.gH = S.ngH; S.gdelta = S.ngdelta; S.glevel = S.nglevel;
            S.gjlo = S.ntask.jlo; S.gjhi = S.ntask.jhi;
            S.stot = 0; S.snext = 0; S.btot = 0; S.bnext = 0; S.bnext2 = 0; S.bnext4 = 0; S.big_active = NGRP;
        }
        __syncthreads();
        if (S.task_idx >= ntasks) break;
        prof_mark(c, S, 0);
        u32 nclaim = 0;
        if (threadIdx.x == 0) nclaim = begin + atomicAdd(c->k7_next, 1u);   // used when this task is done
        const K7Task task = S.task;   // (task / M / offsets are re-read from S.task where they are used
        const u32 M = task.size;      //  after the node phase: fewer registers live across it)
        // pad != 0: a K7_SORT chunk of equal keys (Standard-Sort split of one key value): copied
        const bool presorted = task.kind == K7_SORT && task.pad != 0;
        const bool sort_task = !presorted && (task.kind == K7_SORT || (task.kind == K7_NODE && M < c->tau));
        u64 *dst = sort_task ? S.B : S.A;
        bool nan_here = false;
        mbar_wait(&S.tbar, it & 1u);
        // a K7_GROUP task's placement reads the raw bulk-copied keys itself (no pass over B)
        const bool raw_group = task.kind == K7_GROUP && !S.ldirect;
        if (BULKST && !raw_group) {   // A is written next: the previous task's bulk store must have read it
            if (threadIdx.x == 0) bulk_wait_read();
            __syncthreads();
        }
        if (raw_group) {
        } else if (S.ldirect) {
            nan_here = load_task<K, PR>(dst, sort_task ? S.IB : S.IA, c->buf[task.src] + task.off, M);
        } else {   // raw keys at B[lhead + i] -> ordered keys at dst[i]
            const u32 hd = S.lhead;
            u64 r[KPT];
#pragma unroll
            for (int q = 0; q < KPT; ++q) {
                const u32 i = threadIdx.x + q * K7_THREADS;
                r[q] = i < M ? S.B[hd + i] : 0ull;
            }
            if (sort_task && hd) __syncthreads();   // in-place shift
#pragma unroll
            for (int q = 0; q < KPT; ++q) {
                const u32 i = threadIdx.x + q * K7_THREADS;
                if (i < M) {
                    if (K::is_f64) nan_here |= (r[q] & 0x7fffffffffffffffull) > 0x7ff0000000000000ull;
                    dst[i] = K::to_okey(r[q]);
                    if (PR) (sort_task ? S.IB : S.IA)[i] = (u16)i;
                }
            }
        }
        if (K::is_f64 && task.level == 1) {   // (uniform) the NaN vote is this point's barrier
            if (__syncthreads_or(nan_here)) {
                if (threadIdx.x == 0) { atomicOr(c->nan_flag, 1u); if (BULKST) bulk_wait_all(); }
                return;
            }
        } else {
            __syncthreads();
        }
        prof_mark(c, S, 1);
        if (threadIdx.x == 0 && c->k7_prof) { S.prof[11] += 1; S.prof[12] += M; }
        if (presorted) {
        } else if (sort_task) {
            if (!PR && K7_THREADS * 8 == S_CAP && M > SMALL_MAX) block_sort_tile<K7_THREADS>(S.B, S.A, M);   // B -> A
            else sort_range<K7_WARPS, PR>(S, 0, M, CT);
            prof_mark(c, S, 6);
        } else {
            u32 Lb;
            if (task.kind == K7_GROUP) {   // finish the global node's placement for buckets [jlo, jhi)
                Lb = S.glevel;
                node_step<K, K7_WARPS, MODE_GLOBAL, PR, LOG>(c, S, CT, 0, M, Lb, 0, c->gbase + task.off, raw_group ? S.B + S.lhead : nullptr);
                prof_mark(c, S, 2);
            } else {   // K7_NODE: a fresh Learned-Sort call on the whole task
                Lb = task.level;
                if (threadIdx.x == 0) push_root(c, S, ent_make(0, M, 0));
                __syncthreads();
            }
            // nodes larger than the largest team tier holds in registers: the whole CTA, one level
            for (u32 i = 0; i < S.btot; ++i) {
                const u32 e = S.lbig[i];
                if (ent_m(e) > CTA_MIN) {
                    __syncthreads();
                    if (threadIdx.x == 0) S.lbig[i] = 0;
                    node_step<K, K7_WARPS, MODE_NODE, PR, LOG>(c, S, CT, ent_pos(e), ent_m(e), Lb + ent_rel(e), ent_rel(e), c->gbase + S.task.off);
                }
            }
            const u64 gb = c->gbase + S.task.off;
            // quad teams (1024-thread builds): (2 GCAP, 4 GCAP]; double teams: (GCAP, 2 GCAP]
            if constexpr (QUAD) run_tier<K, 4 * GW, PR, LOG>(c, S, GQ, &S.bnext4, S.cur4, 2u * GCAP, 4u * GCAP, Lb, gb, wprof, wcyc[0]);
            run_tier<K, 2 * GW, PR, LOG>(c, S, GH, &S.bnext2, S.cur2, (u32)GCAP, 2u * GCAP, Lb, gb, wprof, wcyc[0]);
            prof_mark(c, S, 4);
            // teams of GW warps take the nodes of (WCAP, GCAP] keys (their children go to the small
            // list); then every warp runs small nodes and their whole subtrees on its own
            run_tier<K, GW, PR, LOG>(c, S, GG, &S.bnext, S.cur, (u32)WCAP, (u32)GCAP, Lb, gb, wprof, wcyc[1]);
            if (GG.t == 0) { __threadfence_block(); atomicSub(&S.big_active, 1u); }
            if (lane == 0) S.top[w] = 0;
            __syncwarp();
            for (;;) {
                u32 e = 0;
                const long long tw = wprof ? clock64() : 0;
                if (lane == 0) {
                    if (S.top[w] > 0) {
                        e = S.stk[w * S.stk_cap + (--S.top[w])];
                    } else {
                        const u32 tk = atomicAdd(&S.snext, 1u);
                        volatile u32 *slot = &S.lsm[tk < S.lsm_cap ? tk : S.lsm_cap - 1];
                        u32 ns = PCF_K7_NS0;
                        for (;;) {   // wait (backing off, so the working teams keep the issue slots)
                            e = *slot;
                            if (e) { *slot = 0; break; }
                            if (*(volatile u32 *)&S.big_active == 0) {   // no more pushes
                                __threadfence_block();
                                e = *slot;
                                if (e) *slot = 0;
                                break;
                            }
                            __nanosleep(ns);
                            ns = ns < PCF_K7_NSMAX ? ns * 2 : ns;
                        }
                    }
                }
                e = __shfl_sync(0xffffffffu, e, 0);
                const long long t0 = wprof ? clock64() : 0;
                if (wprof) wcyc[3] += t0 - tw;
                if (!e) break;
                node_step<K, 1, MODE_NODE, PR, LOG>(c, S, GS, ent_pos(e), ent_m(e), Lb + ent_rel(e), ent_rel(e), c->gbase + S.task.off);
                if (wprof) wcyc[2] += clock64() - t0;
            }
            __syncthreads();
            prof_mark(c, S, 5);
        }
        if (threadIdx.x == 0) {   // B is free: the next task streams in while this one is stored
            S.nidx = nclaim;
            if (nclaim < ntasks) { S.ntask = c->k7[c->k7_order ? c->k7_order[nclaim] : nclaim]; k7_issue(c, S, S.ntask); k7_fetch_node(c, S); }
        }
        if (BULKST) {
            store_task_bulk<K>(S, c->buf[2] + S.task.off, S.task.size);
        } else {
            store_task_idx<PR>(c, S, S.task, S.task.size);
            store_task<K>(S, c->buf[2] + S.task.off, S.task.size);
        }
        prof_mark(c, S, 13);
        __syncthreads();
    }
    if (BULKST && threadIdx.x == 0) bulk_wait_all();
    if (PCF_K7_WPROF) {
        if (wprof)
            for (int i = 0; i < 4; ++i) atomicAdd(&S.prof[16 + i], wcyc[i]);
        __syncthreads();
    }
    if (c->k7_prof && threadIdx.x == 0)
        for (int i = 0; i < K7_PROF_SLOTS; ++i) atomicAdd(&c->k7_prof[i], S.prof[i]);
}


// Host-side description of this block size (pcf_api.cu)
struct Variant {
    static constexpr int threads = K7_THREADS;
    static size_t smem(u32 tau, bool pr) { return sizeof(K7Smem) + k7_lists_bytes(tau < 2 ? 2 : tau) + (pr ? 4ull * S_CAP : 0ull); }
};
