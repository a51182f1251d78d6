// pcf_api.cu -- host orchestration and the C ABI of libpcfsort.so (include/pcf_sort.h).
//
// Call structure for one sort of n keys:
//   n <= S_CAP          one K7 task: the whole Algorithm 1 in one CTA's shared memory.
//   n >  S_CAP          level-1 node on the global path: k_minmax -> k_node_model ->
//                       k_fit_sample -> k_fit_scan, then split rounds (count, scan,
//                       scatter, taskgen) until every group fits a K7 CTA; oversized
//                       recursing buckets become new global nodes (next round);
//                       then one persistent K7 launch over all groups.  Buckets that
//                       Alg. 1 sends to Standard-Sort and that exceed S_CAP are sorted
//                       by MSD radix splits (the same count / scatter rounds) + K7.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pcf_sort.h"
#include "pcf_common.cuh"
#include "pcf_global.cuh"
#include "pcf_k7.cuh"
#include "pcf_bucketing.cuh"
#include "pcf_shard.cuh"

namespace pcf {

static thread_local std::string g_last_error;

static int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            return fail(PCF_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));        \
        }                                                                                          \
    } while (0)

static inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// ---------------------------------------------------------------- capacities
struct Caps {
    u64 n;
    u32 P;            // iroot34(n)
    u32 node_cap;
    u64 arena_u32;
    u32 k7_cap;
    u32 split_cap;
    u32 items_cap;
    u64 cmat_cap;     // entries of the C / P count matrices
    u64 bsum_cap;
};

constexpr u32 BND_MIN_LOG2 = 24;   // nodes of >= 2^24 keys get the gather-free digit table

// root_n: size of the level-1 node (n itself; N for a shard of a sharded sort, whose
// root tables are the global node's)
static Caps caps_for(u64 n, u64 root_n = 0) {
    Caps c;
    c.n = n;
    c.P = (u32)iroot34(root_n > n ? root_n : n);
    // global nodes hold > S_CAP keys; nodes of one level are disjoint, and a global
    // node nests in another only if the parent has > S_CAP^{4/3} keys: 2 n / S_CAP bounds them
    c.node_cap = (u32)(2 * (n / S_CAP) + 64);
    // root tables + every oversized node: sum of 3*(m^{3/4}+2) over disjoint m > S_CAP
    // is <= 3*(n^{3/4} + n / S_CAP^{1/4} + 2*node_cap)  (S_CAP^{1/4} > 9.5), twice for nesting
    c.arena_u32 = 3ull * ((u64)c.P + 2) + 6ull * (n * 2 / 19 + 2ull * c.node_cap) + 64
                  + (u64)GMAX * ((n >> BND_MIN_LOG2) + 1);   // digit boundaries of large nodes
    c.k7_cap = (u32)std::min<u64>(n / 32 + 65536, 0xffffffffull);
    c.split_cap = (u32)(n / 1024 + 4096);
    c.items_cap = (u32)(2 * (n / S_CAP) + 64);   // items hold > S_CAP keys (see node_cap)
    // every split of a round has <= GMAX digits and ceil(m/SPLIT_TILE) tiles; a round's
    // splits are disjoint segments of > S_CAP keys (or of wider-than-NB_CAP bucket ranges)
    c.cmat_cap = (n / SPLIT_TILE + n / S_CAP + 64) * (u64)GMAX;
    c.bsum_cap = c.cmat_cap / SCAN_CHUNK + 2;
    return c;
}

struct Layout {
    size_t ctx, counters, tmp, tidx, digs, tmap, k7_order, bpre_mm, bpre_fs, nodes, arena, k7, splits_a, splits_b, items, fb,
        cmat, pmat, bsum, scan_status, status, total;
};

static Layout layout_for(const Caps &c, bool pr = false) {   // (caps_for(n, root_n))
    Layout L;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    L.ctx = take(sizeof(DevCtx));
    L.counters = take(sizeof(Counters));
    L.status = take(16);
    L.tmp = take(c.n * 8);
    L.tidx = pr ? take(c.n * 4) : 0;   // key-value mode: source indices of tmp
    L.digs = take(c.n * 2);
    L.tmap = take((c.n / SPLIT_TILE + c.split_cap + 64) * 4);
    L.nodes = take((size_t)c.node_cap * sizeof(GNode));
    L.arena = take(c.arena_u32 * 4);
    L.k7 = take((size_t)c.k7_cap * sizeof(K7Task));
    L.k7_order = take((size_t)c.k7_cap * 4);
    L.bpre_mm = take(((u64)c.node_cap + 1) * 4);   // a batch's chunk prefix sums
    L.bpre_fs = take(((u64)c.node_cap + 1) * 4);
    L.splits_a = take((size_t)c.split_cap * sizeof(SplitTask));
    L.splits_b = take((size_t)c.split_cap * sizeof(SplitTask));
    L.items = take((size_t)c.items_cap * sizeof(SegItem));
    L.cmat = take(c.cmat_cap * 4);
    L.pmat = take(c.cmat_cap * 4);
    L.bsum = take(c.bsum_cap * 4);
    L.scan_status = take(c.bsum_cap * 8);
    L.total = off;
    return L;
}

static size_t small_layout_bytes() {
    // n <= S_CAP: ctx + counters + status + one K7 task
    return align_up(sizeof(DevCtx), 256) + align_up(sizeof(Counters), 256) + 256 + align_up(sizeof(K7Task), 256);
}

static size_t workspace_bytes_impl(size_t n, bool pr = false) {
    if (n == 0) return 0;
    if (n <= (size_t)S_CAP) return small_layout_bytes();
    return layout_for(caps_for(n), pr).total;
}

// ---------------------------------------------------------------- phase timer
struct PhaseTimer {
    bool on = false;
    cudaStream_t st;
    struct Ev { int phase; cudaEvent_t a, b; };
    std::vector<Ev> evs;
    int cur = -1;
    cudaEvent_t cur_a = nullptr;
    void begin(int phase) {
        if (!on) return;
        cudaEvent_t a;
        cudaEventCreate(&a);
        cudaEventRecord(a, st);
        cur = phase;
        cur_a = a;
    }
    void end() {
        if (!on || cur < 0) return;
        cudaEvent_t b;
        cudaEventCreate(&b);
        cudaEventRecord(b, st);
        evs.push_back({cur, cur_a, b});
        cur = -1;
    }
    void collect(float *ms) {
        for (auto &e : evs) {
            float t = 0;
            cudaEventElapsedTime(&t, e.a, e.b);
            ms[e.phase] += t;
            cudaEventDestroy(e.a);
            cudaEventDestroy(e.b);
        }
        evs.clear();
    }
};

enum { PH_MINMAX = 0, PH_FIT = 1, PH_COUNT = 2, PH_SCATTER = 3, PH_K7 = 4, PH_LOG = 5, PH_OTHER = 6, PH_TOTAL = 7,
       PH_BATCHES = 8 };

// K7 dynamic shared memory: the struct, the node lists (sized for tau) and, in
// key-value mode, the two u16 source-index arrays IA / IB behind them
namespace k7s = k7n512;    // 512 threads: every tau, key-value mode
namespace k7w = k7n1024;   // 1024 threads: keys-only sorts with tau >= K7W_MIN_TAU
constexpr u32 PR_MIN_TAU = 16;   constexpr u32 K7W_MIN_TAU = 32;
constexpr int SMEM_MAX = 232448;
// The wide variant (32 warps per SM) unless the sort is key-value, tau is small or
// PCF_K7_VARIANT=512 is set (A/B experiments).
static bool k7_wide(u32 tau, bool pr) {
    static int force = -1;
    if (force < 0) {
        const char *e = getenv("PCF_K7_VARIANT");
        force = e && !strcmp(e, "512") ? 1 : 0;
    }
    return !pr && !force && tau >= K7W_MIN_TAU && k7w::Variant::smem(tau, false) <= (size_t)SMEM_MAX;
}
static int k7_smem_bytes(u32 tau, bool pr) {
    return (int)(k7_wide(tau, pr) ? k7w::Variant::smem(tau, pr) : k7s::Variant::smem(tau, pr));
}
// K7 instance: block size (wide: 1024 threads), key-value mode, pass log (the logging code
// is compiled out of the benchmarked instance: fewer live registers, fewer spills)
template <class K, bool PR>
static void (*k7_fn(bool wide, bool log))(const DevCtx *) {
    if constexpr (!PR) { if (wide) return log ? k7w::k7_kernel<K, false, true> : k7w::k7_kernel<K, false, false>; }
    return log ? k7s::k7_kernel<K, PR, true> : k7s::k7_kernel<K, PR, false>;
}
static int split_smem_bytes() { return (int)sizeof(SplitScatterSmem); }

// Launch with programmatic stream serialization (see pdl_entry()).
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
}

// Per-device caches: occupancy results and the raised shared-memory limits apply to
// the device they were queried / set on (cudaFuncSetAttribute is per device).
constexpr int MAX_DEVS = 64;
static int cur_dev() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= MAX_DEVS) d = 0;
    return d;
}

template <class K, bool PR>
static int k7_ctas_per_sm(bool wide) {   // resident K7 CTAs per SM (persistent grid size)
    static thread_local int v[2][MAX_DEVS] = {{0}};
    const int d = cur_dev();
    if (!v[wide][d]) {
        int b = 1;
        const int nt = wide ? k7w::Variant::threads : k7s::Variant::threads;
        const int sm = (int)(wide ? k7w::Variant::smem(K7W_MIN_TAU, false) : k7s::Variant::smem(PR ? PR_MIN_TAU : 2, PR));
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k7_fn<K, PR>(wide, false), nt, sm) != cudaSuccess || b < 1) b = 1;
        v[wide][d] = b;
    }
    return v[wide][d];
}

template <class K>
static int count_ctas_per_sm() {
    static thread_local int v[MAX_DEVS] = {0};
    const int d = cur_dev();
    if (!v[d]) {
        int b = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_split_count<K>, CNT_THREADS, (int)sizeof(CountSmem)) != cudaSuccess || b < 1) b = 1;
        v[d] = b;
    }
    return v[d];
}

template <class K>
static int configure_kernels() {
    static thread_local bool done[MAX_DEVS] = {false};
    const int d = cur_dev();
    if (done[d]) return PCF_OK;
    for (int lg = 0; lg < 2; ++lg) {
        CK(cudaFuncSetAttribute(k7_fn<K, false>(false, lg), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k7s::Variant::smem(2, false)));
        CK(cudaFuncSetAttribute(k7_fn<K, true>(false, lg), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k7s::Variant::smem(PR_MIN_TAU, true)));
        CK(cudaFuncSetAttribute(k7_fn<K, false>(true, lg), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k7w::Variant::smem(K7W_MIN_TAU, false)));
    }
    CK(cudaFuncSetAttribute(k_split_scatter<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, split_smem_bytes()));
    CK(cudaFuncSetAttribute(k_split_scatter<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, split_smem_bytes()));
    CK(cudaFuncSetAttribute(k_split_count<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CountSmem)));
    done[d] = true;
    return PCF_OK;
}

// ---------------------------------------------------------------- launch helpers
#ifndef PCF_SCAN_LOOKBACK
#define PCF_SCAN_LOOKBACK 2   // count-matrix scan by one decoupled look-back kernel: 0 never, 1 always, 2 sorts of n <= 2^25
#endif
#ifndef PCF_TAIL_CTAS_PER_SM
#define PCF_TAIL_CTAS_PER_SM 32   // grid bound of the tail graph's per-tile kernels (CTAs per SM)
#endif
struct Launch {   // the kernel-launch configuration of this device and sort size
    int nsm;
    int k7_grid;
    int k7_threads;
    bool k7_wide;
    bool log;         // pass log on: the logging K7 instance
    int count_grid;
    int tau_smem;
    u32 tile_grid;    // tail graph: CTAs of the per-tile kernels (grid-stride over the round's tiles; idle CTAs exit)
};

// ---------------------------------------------------------------- device-driven tail (CUDA graph)
// Everything after the host-launched first batch runs from one executable graph:
//   k_items_to_nodes -> WHILE (more work) {
//       batched min/max, sampling, fit of the new global nodes;
//       two split rounds (plan, tile map, count [model, radix], scan x3, scatter, taskgen);
//       K7 (order, kernel, advance); k_items_to_nodes }
// k_items_to_nodes turns oversized recursing buckets into global nodes and oversized
// Standard-Sort buckets into MSD radix splits.  A sort with no oversized bucket runs
// one kernel here (k_items_to_nodes); with a pass log, k_log_finalize follows.
// The loop conditions are set on the device (cudaGraphSetConditional), so the
// recursion over oversized buckets needs no host round trip.
// Graphs depend only on (device, key type, DevCtx address, tau); they are cached
// per thread (a repeated sort with the same workspace reuses them).
struct TailGraph {
    int dev;
    int kt;   // key type * 4 + key-value mode * 2 + pass log (selects the K7 instance)
    const void *ctx;
    u32 tau;
    u64 n;    // grid bounds depend on it
    cudaGraph_t g;
    cudaGraphExec_t ex;
    u32 body_kernels;
};

static thread_local std::vector<TailGraph> g_tails;
static thread_local cudaStream_t g_cap[2] = {nullptr, nullptr};

template <class K, bool PR>
static int add_round(cudaStream_t cs, const DevCtx *d_ctx, const Launch &lc, u32 *nk) {
    CK(launch_pdl(k_round_plan, 1, 1024, 0, cs, d_ctx));
    CK(launch_pdl(k_tile_map, lc.nsm * 2, 256, 0, cs, d_ctx));
    CK(launch_pdl(k_split_count_tile<K>, lc.tile_grid, SC_THREADS, 0, cs, d_ctx));
    CK(launch_pdl(k_split_count_radix<K>, lc.nsm * 8, SC_THREADS, 0, cs, d_ctx));   // Standard-Sort splits
#if PCF_SCAN_LOOKBACK == 1
    CK(launch_pdl(k_scanp_lookback, lc.nsm * 2, SCAN_THREADS, 0, cs, d_ctx));
    *nk -= 2;
#else
    CK(launch_pdl(k_scanp_partials, lc.nsm * 2, SCAN_THREADS, 0, cs, d_ctx));
    CK(launch_pdl(k_scanp_bsums, 1, SCAN_THREADS, 0, cs, d_ctx));
    CK(launch_pdl(k_scanp_final, lc.nsm * 2, SCAN_THREADS, 0, cs, d_ctx));
#endif
    CK(launch_pdl(k_split_scatter<K, PR>, lc.tile_grid, SC_THREADS, split_smem_bytes(), cs, d_ctx));
    CK(launch_pdl(k_split_taskgen, lc.nsm * 2, TG_THREADS, 0, cs, d_ctx));
    *nk += 9;
    return PCF_OK;
}

template <class K, bool PR>
static int add_k7(cudaStream_t cs, const DevCtx *d_ctx, const Launch &lc, u32 *nk) {
    CK(launch_pdl(k_k7_order, 1, 1024, 0, cs, d_ctx));
    CK(launch_pdl(k7_fn<K, PR>(lc.k7_wide, lc.log), lc.k7_grid, lc.k7_threads, lc.tau_smem, cs, d_ctx));
    CK(launch_pdl(k_k7_advance, 1, 1, 0, cs, d_ctx));
    *nk += 3;
    return PCF_OK;
}

// Add a conditional node (WHILE / IF) after the current capture dependencies of
// `cs`, capture its body from `body` (launched on the second capture stream), and
// continue the capture of `cs` after the node.
template <class F>
static int add_cond(cudaStream_t cs, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type, F body) {
    cudaStreamCaptureStatus cst;
    cudaGraph_t cg;
    const cudaGraphNode_t *deps = nullptr;
    size_t ndeps = 0;
    CK(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &cg, &deps, &ndeps));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = type;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, cg, deps, ndeps, &cp));
    cudaGraph_t bg = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(g_cap[1], bg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    const int rc = body(g_cap[1]);
    cudaGraph_t tmp;
    const cudaError_t e = cudaStreamEndCapture(g_cap[1], &tmp);
    if (rc) return rc;
    CK(e);
    CK(cudaStreamUpdateCaptureDependencies(cs, &node, 1, cudaStreamSetCaptureDependencies));
    return PCF_OK;
}

template <class K, bool PR>
static int build_tail(TailGraph &tg, const DevCtx *d_ctx, const Launch &lc) {
    for (int i = 0; i < 2; ++i)
        if (!g_cap[i]) CK(cudaStreamCreateWithFlags(&g_cap[i], cudaStreamNonBlocking));
    cudaStream_t cs = g_cap[0];
    tg.body_kernels = 0;
    // ---- the device-driven batches of oversized buckets
    {
        CK(cudaGraphCreate(&tg.g, 0));
        cudaGraphConditionalHandle hb;
        CK(cudaGraphConditionalHandleCreate(&hb, tg.g, 0, cudaGraphCondAssignDefault));
        CK(cudaStreamBeginCaptureToGraph(cs, tg.g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        int rc = PCF_OK;
        auto cap = [&]() -> int {
            CK(launch_pdl(k_items_to_nodes<K>, 1, 1024, 0, cs, d_ctx, hb, 0u));
            return add_cond(cs, hb, cudaGraphCondTypeWhile, [&](cudaStream_t bs) -> int {
                u32 nk = 0;
                CK(launch_pdl(k_minmax_batch<K>, lc.nsm * 8, MM_THREADS, 0, bs, d_ctx));
                CK(launch_pdl(k_fit_sample_batch<K>, lc.nsm * 8, FSB_CHUNK, 0, bs, d_ctx));
                CK(launch_pdl(k_fit_batch, lc.nsm * 2, SCAN_THREADS, 0, bs, d_ctx));
                nk += 3;
                for (int r = 0; r < 2; ++r) { int e = add_round<K, PR>(bs, d_ctx, lc, &nk); if (e) return e; }
                int e = add_k7<K, PR>(bs, d_ctx, lc, &nk);
                if (e) return e;
                CK(launch_pdl(k_items_to_nodes<K>, 1, 1024, 0, bs, d_ctx, hb, 1u));
                nk += 1;
                tg.body_kernels = nk;
                return PCF_OK;
            });
        };
        rc = cap();
        cudaGraph_t out;
        const cudaError_t e = cudaStreamEndCapture(cs, &out);
        if (rc) return rc;
        CK(e);
    }
    CK(cudaGraphInstantiate(&tg.ex, tg.g, 0));
    return PCF_OK;
}

template <class K, bool PR>
static int get_tail(const DevCtx *d_ctx, u32 tau, u64 n, const Launch &lc, TailGraph **out) {
    const int dev = cur_dev();
    const int kt = (K::is_f64 ? 0 : 4) + (PR ? 2 : 0) + (lc.log ? 1 : 0);
    for (auto &t : g_tails)
        if (t.dev == dev && t.kt == kt && t.ctx == d_ctx && t.tau == tau && t.n == n) { *out = &t; return PCF_OK; }
    constexpr size_t MAX_TAILS = 8;
    if (g_tails.size() >= MAX_TAILS) {   // evict the oldest
        TailGraph &o = g_tails.front();
        cudaGraphExecDestroy(o.ex);
        cudaGraphDestroy(o.g);
        g_tails.erase(g_tails.begin());
    }
    TailGraph tg;
    memset(&tg, 0, sizeof tg);
    tg.dev = dev; tg.kt = kt; tg.ctx = d_ctx; tg.tau = tau; tg.n = n;
    const int rc = build_tail<K, PR>(tg, d_ctx, lc);
    if (rc) {
        if (tg.ex) cudaGraphExecDestroy(tg.ex);
        if (tg.g) cudaGraphDestroy(tg.g);
        return rc;
    }
    g_tails.push_back(tg);
    *out = &g_tails.back();
    return PCF_OK;
}

// ---------------------------------------------------------------- the sort
// A shard of a sharded sort (pcf_shard.cuh): the keys are buckets [jlo, jhi) of the
// global level-1 node of N keys, at global offset range_off.
struct ShardRoot {
    u64 N, range_off;
    u32 jlo, jhi;
    u32 record;              // write the global level-1 record (and level-1 dumps) here
    const ShardState *S;     // all-reduced extremes
    const u32 *cnt;          // all-reduced per-bin sample counts [beta + 2]
    const u32 *Hg;           // global bucket sizes [gamma + 2]
};

// Model and R9/R10 verdict of the shard's root (the global level-1 node); a
// degenerate range sends the whole shard range to Standard-Sort.
template <class K>
__global__ void k_shard_root(const DevCtx *__restrict__ c, const ShardState *__restrict__ S, u64 m) {
    GNode &g = c->nodes[0];
    g.kmin = i64_to_okey(S->mm[0]);
    g.kmax = i64_to_okey(S->mm[1]);
    Model md;
    const bool ok = make_model<K>(g.kmin, g.kmax, g.beta, md);
    g.md = md;
    g.degenerate = ok ? 0u : 1u;
    if (!ok) push_item(c, 0, (u32)m, 1, 0, 1u);
}

// in, out: device keys; perm (key-value mode, PR): device u32[n] that receives the
// stable sorting permutation (reading R18), NULL otherwise.
template <class K, bool PR = false>
static int sort_device(const u64 *in, u64 *out, size_t n, const pcf_params *pp, cudaStream_t st, u32 *perm = nullptr,
                       const ShardRoot *shard = nullptr) {
    pcf_params p;
    pcf_params_init(&p);
    if (pp) {
        if (pp->struct_size < PCF_PARAMS_V1_SIZE) return fail(PCF_ERR_INVALID_ARG, "pcf_params.struct_size too small");
        memcpy(&p, pp, std::min<size_t>(pp->struct_size, sizeof(pcf_params)));
        p.struct_size = sizeof(pcf_params);
    }
    if (p.tau < 2) return fail(PCF_ERR_INVALID_ARG, "tau must be >= 2");
    if (PR && p.tau < PR_MIN_TAU) return fail(PCF_ERR_INVALID_ARG, "key-value / argsort mode needs tau >= 16");
    if (PR && n && !perm) return fail(PCF_ERR_INVALID_ARG, "NULL permutation pointer with n > 0");
    if (PR && ((uintptr_t)perm & 3)) return fail(PCF_ERR_INVALID_ARG, "permutation must be 4-byte aligned");
    if (!in || !out) { if (n) return fail(PCF_ERR_INVALID_ARG, "NULL key pointer with n > 0"); }
    if (n >= (1ull << 32)) return fail(PCF_ERR_INVALID_ARG, "n must be < 2^32 in ABI v1");
    if (((uintptr_t)in & 7) || ((uintptr_t)out & 7)) return fail(PCF_ERR_INVALID_ARG, "keys must be 8-byte aligned");
    if (n && in != out) {
        uintptr_t a0 = (uintptr_t)in, a1 = a0 + n * 8, b0 = (uintptr_t)out, b1 = b0 + n * 8;
        if (a0 < b1 && b0 < a1) return fail(PCF_ERR_INVALID_ARG, "in and out overlap (only in == out is allowed)");
    }
    if (p.log && !p.log->count) return fail(PCF_ERR_INVALID_ARG, "pass log needs a count pointer");
    const bool timing = (p.flags & PCF_FLAG_TIMING) != 0;
    const bool sync = timing || (p.flags & PCF_FLAG_SYNC) != 0;
    pcf_stats stats;
    memset(&stats, 0, sizeof stats);
    if (n == 0) {
        if (p.status_out) CK(cudaMemsetAsync(p.status_out, 0, sizeof(int), st));
        if (p.stats) *p.stats = stats;
        return PCF_OK;
    }
    int rc = configure_kernels<K>();
    if (rc) return rc;

    const bool logging = p.log != nullptr;
    PhaseTimer tm;
    tm.on = timing;
    tm.st = st;
    cudaEvent_t ev_total0 = nullptr, ev_total1 = nullptr;
    if (timing) {
        cudaEventCreate(&ev_total0);
        cudaEventCreate(&ev_total1);
        cudaEventRecord(ev_total0, st);
    }

    const size_t need = shard ? layout_for(caps_for(n, shard->N), PR).total : workspace_bytes_impl(n, PR);
    char *ws = (char *)p.workspace;
    bool own = false;
    if (ws) {
        if (p.workspace_bytes < need) return fail(PCF_ERR_WORKSPACE_TOO_SMALL, "workspace smaller than pcf_workspace_bytes()");
        if ((uintptr_t)ws & 255) return fail(PCF_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
    } else {
        cudaError_t e = cudaMallocAsync((void **)&ws, need, st);
        if (e != cudaSuccess) { cudaGetLastError(); return fail(PCF_ERR_OOM, "cudaMallocAsync workspace failed"); }
        own = true;
    }
    struct Freer {
        bool own; char *ws; cudaStream_t st;
        ~Freer() { if (own) cudaFreeAsync(ws, st); }
    } freer{own, ws, st};

    DevCtx hc;
    memset(&hc, 0, sizeof hc);
    hc.buf[0] = const_cast<u64 *>(in);
    hc.buf[2] = out;
    hc.n = n;
    hc.seed = p.seed;
    hc.tau = p.tau;
    hc.flags = p.flags;
    if (shard) {
        hc.gbase = shard->range_off;
        hc.root_external = shard->record ? 2u : 1u;
    }
    if (logging) {
        hc.rec = reinterpret_cast<NodeRec *>(p.log->records);
        hc.rec_cap = p.log->records ? p.log->capacity : 0;
        hc.l1_b = p.log->level1_b;
        hc.l1_h = p.log->level1_h;
        hc.l1_cap = p.log->level1_capacity;
        if (shard && !shard->record) { hc.l1_b = nullptr; hc.l1_h = nullptr; }
        hc.rec_count = reinterpret_cast<unsigned long long *>(p.log->count);
        if (!hc.rec) hc.rec = reinterpret_cast<NodeRec *>(1);   // non-null marks logging on; cap 0
        CK(cudaMemsetAsync(p.log->count, 0, 8, st));
    }

    const bool small = n <= (size_t)S_CAP && !shard;
    DevCtx *d_ctx;
    Counters *d_cnt;
    int *d_status;
    Caps caps;
    Layout L;
    memset(&L, 0, sizeof L);
    memset(&caps, 0, sizeof caps);
    if (small) {
        d_ctx = (DevCtx *)ws;
        d_cnt = (Counters *)(ws + align_up(sizeof(DevCtx), 256));
        d_status = (int *)(ws + align_up(sizeof(DevCtx), 256) + align_up(sizeof(Counters), 256));
        K7Task *d_task = (K7Task *)((char *)d_status + 256);
        hc.k7 = d_task;
        hc.k7_cap = 1;
        hc.buf[1] = nullptr;
    } else {
        caps = caps_for(n, shard ? shard->N : 0);
        L = layout_for(caps, PR);
        d_ctx = (DevCtx *)(ws + L.ctx);
        d_cnt = (Counters *)(ws + L.counters);
        d_status = (int *)(ws + L.status);
        hc.buf[1] = (u64 *)(ws + L.tmp);
        hc.nodes = (GNode *)(ws + L.nodes);
        hc.node_cap = caps.node_cap;
        hc.arena = (u32 *)(ws + L.arena);
        hc.arena_cap = caps.arena_u32;
        hc.bpre_mm = (u32 *)(ws + L.bpre_mm);
        hc.bpre_fs = (u32 *)(ws + L.bpre_fs);
        hc.k7 = (K7Task *)(ws + L.k7);
        hc.k7_order = (u32 *)(ws + L.k7_order);
        hc.k7_cap = caps.k7_cap;
        hc.splits[0] = (SplitTask *)(ws + L.splits_a);
        hc.splits[1] = (SplitTask *)(ws + L.splits_b);
        hc.splits_cap = caps.split_cap;
        hc.items = (SegItem *)(ws + L.items);
        hc.items_cap = caps.items_cap;
        hc.cmat = (u32 *)(ws + L.cmat);
        hc.pmat = (u32 *)(ws + L.pmat);
        hc.bsum = (u32 *)(ws + L.bsum);
        hc.scan_status = (unsigned long long *)(ws + L.scan_status);
        hc.cmat_cap = caps.cmat_cap;
        hc.digs = (u16 *)(ws + L.digs);
        hc.tmap = (u32 *)(ws + L.tmap);
        if (PR) hc.ibuf[1] = (u32 *)(ws + L.tidx);
    }
    if (PR) hc.ibuf[2] = perm;   // ibuf[0] stays NULL: the input's index is its position
    hc.cnt = d_cnt;
    hc.nan_flag = &d_cnt->nan_flag;
    hc.err_flag = &d_cnt->err_flag;
    hc.k7_count = &d_cnt->k7_count;
    hc.k7_next = &d_cnt->k7_next;
    hc.nsplits = d_cnt->nsplits;
    hc.nitems = &d_cnt->nitems;
    hc.k7_keys = &d_cnt->k7_keys;
    hc.k7_begin = &d_cnt->k7_begin;
    hc.split_keys = &d_cnt->split_keys;
    hc.plan = &d_cnt->plan;
    hc.k7_prof = (p.flags & PCF_FLAG_PROFILE) ? d_cnt->k7_prof : nullptr;
    if (!logging) hc.rec_count = &d_cnt->rec_count;

    const bool sample_all = (p.flags & PCF_FLAG_SAMPLE_ALL) != 0;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    Launch lc;
    lc.nsm = nsm;
    lc.k7_wide = k7_wide(p.tau, PR);
    lc.log = logging;
    lc.k7_threads = lc.k7_wide ? k7w::Variant::threads : k7s::Variant::threads;
    lc.k7_grid = nsm * k7_ctas_per_sm<K, PR>(lc.k7_wide);
    lc.count_grid = nsm * count_ctas_per_sm<K>();
    lc.tau_smem = k7_smem_bytes(p.tau, PR);
    // fallback segments hold > S_CAP keys each: <= n / S_CAP partial tiles
    // (the tail graph's count / scatter kernels are grid-stride: a bounded grid keeps the cost of
    // an almost empty batch -- c5f's few wide tail groups -- away from n / SPLIT_TILE idle CTAs)
    lc.tile_grid = (u32)std::min<u64>(n / SPLIT_TILE + 4096, (u64)nsm * PCF_TAIL_CTAS_PER_SM);

    // initial counters (host-built: the root node and its tables are carved here)
    Counters h0;
    memset(&h0, 0, sizeof h0);
    u32 launches = 0;
    u64 bytes[PCF_PHASES] = {0};
    TailGraph *tail = nullptr;
    if (small) {
        h0.k7_count = 1;
        CK(cudaMemcpyAsync(d_ctx, &hc, sizeof hc, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d_cnt, &h0, sizeof h0, cudaMemcpyHostToDevice, st));
        K7Task t;
        memset(&t, 0, sizeof t);
        t.off = 0; t.size = (u32)n; t.kind = K7_NODE; t.src = 0; t.level = 1;
        CK(cudaMemcpyAsync(hc.k7, &t, sizeof t, cudaMemcpyHostToDevice, st));
        tm.begin(PH_K7);
        k7_fn<K, PR>(lc.k7_wide, lc.log)<<<1, lc.k7_threads, lc.tau_smem, st>>>(d_ctx);
        CK(cudaGetLastError());
        tm.end();
        launches++;
        bytes[PH_K7] += 16ull * n;
    } else {
        // ------------------------------------------------ level 1 (host-launched, exact grids)
        const u64 rootn = shard ? shard->N : n;
        const u32 P = (u32)iroot34(rootn);
        GNode g;
        memset(&g, 0, sizeof g);
        g.off = shard ? (u64)0 - shard->range_off : 0;   // the record's offset is gbase + off = 0
        g.m = (u32)rootn; g.level = 1;
        g.kmin = ~0ull; g.kmax = 0;
        g.alpha = sample_all ? (u32)rootn : P; g.beta = P; g.gamma = P; g.delta = P;
        g.src = 0;
        u64 arena_used = 3ull * ((u64)P + 2);
        u32 *arena = hc.arena;
        g.cnt = arena;
        g.T = g.cnt + (P + 2);
        g.H = g.T + (P + 2);
        const u32 jlo0 = shard ? shard->jlo : 1u, jhi0 = shard ? shard->jhi : P + 2;
        const u32 sh0 = choose_shift(jhi0 - jlo0, (u32)n);
        if (!shard && n >= (1ull << BND_MIN_LOG2)) {   // digit boundaries: gather-free digits in the first count pass
            g.bnd = arena + arena_used;
            arena_used += GMAX;
            g.bshift = sh0;
            g.bG = (P + 1 + (1u << sh0) - 1) >> sh0;
        }
        SplitTask s0;
        memset(&s0, 0, sizeof s0);
        s0.off = 0; s0.m = (u32)n; s0.node = 0; s0.jlo = jlo0; s0.jhi = jhi0;
        s0.shift = sh0;
        s0.G = (jhi0 - jlo0 + (1u << sh0) - 1) >> sh0;
        s0.src = 0; s0.dst = 1;
        h0.node_count = 1;
        h0.arena_used = arena_used;
        h0.nsplits[0] = 1;
        h0.global_keys = n;
        CK(cudaMemcpyAsync(d_ctx, &hc, sizeof hc, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d_cnt, &h0, sizeof h0, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(hc.nodes, &g, sizeof g, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(hc.splits[0], &s0, sizeof s0, cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(g.cnt, 0, 3ull * ((u64)P + 2) * 4, st));
        const DevCtx *dc = d_ctx;
        if (shard) {   // the global node: all-reduced counts and histogram, model from the all-reduced extremes
            CK(cudaMemcpyAsync(g.cnt, shard->cnt, ((u64)P + 2) * 4, cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(g.H, shard->Hg, ((u64)P + 2) * 4, cudaMemcpyDeviceToDevice, st));
            k_shard_root<K><<<1, 1, 0, st>>>(d_ctx, shard->S, (u64)n);
            CK(cudaGetLastError());
            launches++;
        }
        if (!shard) {
        tm.begin(PH_MINMAX);
        {
            const u64 nvec = n / 2 + 1;
            const u32 grid = (u32)std::min<u64>(148ull * 8, (nvec + MM_THREADS * MM_UNROLL - 1) / (MM_THREADS * MM_UNROLL));
            CK(launch_pdl(k_minmax<K>, grid, MM_THREADS, 0, st, dc, 0u));
        }
        tm.end();
        }
        tm.begin(PH_FIT);
        {
            if (!shard) CK(launch_pdl(k_fit_sample<K>, (g.alpha + 255) / 256, 256, 0, st, dc, 0u));
            const u64 nbins = (u64)P + 1;
            const u32 nblk = (u32)((nbins + SCAN_CHUNK - 1) / SCAN_CHUNK);
            u32 *bs = hc.bsum;
            CK(launch_pdl(k_scan_partials, nblk, SCAN_THREADS, 0, st, (const u32 *)(g.cnt + 1), (u64)nbins, bs));
            CK(launch_pdl(k_scan_bsums, 1, SCAN_THREADS, 0, st, bs, nblk));
            CK(launch_pdl(k_fit_final, nblk, SCAN_THREADS, 0, st, dc, 0u, (const u32 *)bs));
        }
        tm.end();
        CK(cudaGetLastError());
        launches += 5;
        if (!shard) bytes[PH_MINMAX] += 8ull * n;
        bytes[PH_FIT] += shard ? 8ull * (P + 2) : 8ull * g.alpha + 8ull * (P + 2);
        // two split rounds with grids sized from n (an upper bound on each round's tiles)
        u64 splits_bound = 1;
        for (int r = 0; r < 2; ++r) {
            const u32 tile_grid = (u32)std::min<u64>(n / SPLIT_TILE + 1 + splits_bound, 0x7fffffffull);
            splits_bound = std::min<u64>(splits_bound * (GMAX + 1), caps.split_cap);
            tm.begin(PH_OTHER);
            CK(launch_pdl(k_round_plan, 1, 1024, 0, st, dc));
            CK(launch_pdl(k_tile_map, nsm * 2, 256, 0, st, dc));
            tm.end();
            tm.begin(PH_COUNT);
            // one CTA per tile for small sorts and the second round (their T gathers are
            // local to a split: they need L1, which the persistent kernel's 2 x 111 KB of
            // staging takes); the persistent bulk-copy kernel for the first round of a
            // large sort (gather-free digit table)
            if (n <= (1ull << 25) || r > 0) CK(launch_pdl(k_split_count_tile<K>, tile_grid, SC_THREADS, 0, st, dc));
            else CK(launch_pdl(k_split_count<K>, lc.count_grid, CNT_THREADS, sizeof(CountSmem), st, dc));
            tm.end();
            tm.begin(PH_OTHER);
            // the count-matrix scan (a6): one decoupled look-back kernel for small sorts (two launches
            // less per round); for large matrices the three-phase scan is faster (ab_scan_lookback.txt)
            const bool lookback = PCF_SCAN_LOOKBACK == 1 || (PCF_SCAN_LOOKBACK == 2 && n <= (1ull << 25));
            if (lookback) {
                CK(launch_pdl(k_scanp_lookback, nsm * 2, SCAN_THREADS, 0, st, dc));
                launches -= 2;
            } else {
                CK(launch_pdl(k_scanp_partials, nsm * 2, SCAN_THREADS, 0, st, dc));
                CK(launch_pdl(k_scanp_bsums, 1, SCAN_THREADS, 0, st, dc));
                CK(launch_pdl(k_scanp_final, nsm * 2, SCAN_THREADS, 0, st, dc));
            }
            tm.end();
            tm.begin(PH_SCATTER);
            CK(launch_pdl(k_split_scatter<K, PR>, tile_grid, SC_THREADS, split_smem_bytes(), st, dc));
            tm.end();
            tm.begin(PH_OTHER);
            CK(launch_pdl(k_split_taskgen, nsm * 2, TG_THREADS, 0, st, dc));
            tm.end();
            launches += 8;
        }
        // K7 over every group produced so far (persistent grid; reads the task count on the device)
        tm.begin(PH_K7);
        {
            u32 nk = 0;
            rc = add_k7<K, PR>(st, dc, lc, &nk);
            if (rc) return rc;
            launches += nk;
        }
        tm.end();
        CK(cudaGetLastError());
        // ------------------------------------------------ everything after: device-driven (graphs)
        rc = get_tail<K, PR>(d_ctx, p.tau, n, lc, &tail);
        if (rc) return rc;
        tm.begin(PH_BATCHES);
        CK(cudaGraphLaunch(tail->ex, st));
        tm.end();
        launches += 1;   // k_items_to_nodes; the loop bodies are counted from the device counters
        if (logging) {   // the records of the global nodes (all levels)
            tm.begin(PH_LOG);
            CK(launch_pdl(k_log_finalize<K>, lc.nsm * 4, 256, 0, st, d_ctx));
            tm.end();
            launches += 1;
        }
    }
    if (p.status_out) {
        k_status<<<1, 1, 0, st>>>(d_ctx, p.status_out);
        CK(cudaGetLastError());
        launches++;
    }
    if (timing) cudaEventRecord(ev_total1, st);
    int status = PCF_OK;
    if (sync) {
        Counters hcnt;
        CK(cudaMemcpyAsync(&hcnt, d_cnt, sizeof hcnt, cudaMemcpyDeviceToHost, st));
        unsigned long long rcnt = 0;
        if (logging) CK(cudaMemcpyAsync(&rcnt, p.log->count, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        stats.host_syncs = 1;
        if (hcnt.nan_flag) status = fail(PCF_ERR_NAN, "input contains NaN");
        else if (hcnt.err_flag) status = fail(PCF_ERR_INTERNAL, "device capacity exceeded (err_flag=" + std::to_string(hcnt.err_flag) + ")");
        else if (logging && rcnt > p.log->capacity) status = fail(PCF_ERR_LOG_OVERFLOW, "pass log capacity exceeded");
        for (int i = 0; i < K7_PROF_SLOTS; ++i) stats.k7_cycles[i] = hcnt.k7_prof[i];
        stats.rounds = hcnt.round;
        stats.groups_smem = hcnt.k7_count;
        stats.global_nodes = small ? 0 : hcnt.node_count;
        stats.split_keys_moved = hcnt.split_keys;
        stats.fallback_keys_global = hcnt.fb_keys;
        if (tail) {
            launches += hcnt.iters * tail->body_kernels;
            stats.device_batches = hcnt.iters;
        }
        if (!small) {
            // one classify (8 B/key) and one stable scatter (16 B/key) per
            // bucketing level of every key the global path buckets; extra digit rounds are
            // traffic, not algorithmic bytes (reported as split_keys_moved)
            bytes[PH_COUNT] = 8ull * hcnt.global_keys;
            bytes[PH_SCATTER] = 16ull * hcnt.global_keys;
            bytes[PH_K7] = 16ull * hcnt.k7_keys;
            bytes[PH_MINMAX] = 8ull * hcnt.global_keys;
        }
    }
    stats.kernel_launches = launches;
    if (timing) {
        tm.collect(stats.phase_ms);
        float tot = 0;
        cudaEventElapsedTime(&tot, ev_total0, ev_total1);
        stats.phase_ms[PH_TOTAL] = tot;
        cudaEventDestroy(ev_total0);
        cudaEventDestroy(ev_total1);
    }
    for (int i = 0; i < PCF_PHASES; ++i) stats.phase_bytes[i] = bytes[i];
    if (p.stats) *p.stats = stats;
    return status;
}

template <class K>
static int sort_host(const u64 *in_h, u64 *out_h, size_t n, const pcf_params *pp, cudaStream_t st) {
    if (n == 0) return PCF_OK;
    if (!in_h || !out_h) return fail(PCF_ERR_INVALID_ARG, "NULL host pointer with n > 0");
    u64 *d = nullptr;
    cudaError_t e = cudaSuccess;
    const size_t key_bytes = align_up(n * 8, 256);
    const size_t sort_ws = workspace_bytes_impl(n);
    pcf_params p;
    pcf_params_init(&p);
    if (pp) {
        if (pp->struct_size < PCF_PARAMS_V1_SIZE) return fail(PCF_ERR_INVALID_ARG, "pcf_params.struct_size too small");
        memcpy(&p, pp, std::min<size_t>(pp->struct_size, sizeof(pcf_params)));
        p.struct_size = sizeof(pcf_params);
    }
    const bool own_keys = !(p.workspace && p.workspace_bytes >= key_bytes + sort_ws);
    if (own_keys) {
        p.workspace = nullptr;
        p.workspace_bytes = 0;
        e = cudaMallocAsync((void **)&d, n * 8, st);
        if (e != cudaSuccess) { cudaGetLastError(); return fail(PCF_ERR_OOM, "cudaMallocAsync keys failed"); }
    } else {   // caller workspace: [keys | sort workspace]
        d = (u64 *)p.workspace;
        p.workspace = (char *)p.workspace + key_bytes;
        p.workspace_bytes -= key_bytes;
    }
    // one synchronisation for the whole call: the sort runs asynchronously and
    // reports through a device status word read after the result's D2H copy
    int *d_status = nullptr;
    int *user_status = p.status_out;
    e = cudaMallocAsync((void **)&d_status, sizeof(int), st);
    if (e != cudaSuccess) { cudaGetLastError(); if (own_keys) cudaFreeAsync(d, st); return fail(PCF_ERR_OOM, "cudaMallocAsync status failed"); }
    p.status_out = d_status;
    p.flags &= ~(PCF_FLAG_SYNC | PCF_FLAG_TIMING);
    int rc = PCF_OK;
    e = cudaMemcpyAsync(d, in_h, n * 8, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rc = fail(PCF_ERR_CUDA, cudaGetErrorString(e));
    if (!rc) rc = sort_device<K>(d, d, n, &p, st);
    if (!rc) {
        e = cudaMemcpyAsync(out_h, d, n * 8, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) rc = fail(PCF_ERR_CUDA, cudaGetErrorString(e));
    }
    int hs = PCF_OK;
    if (!rc) {
        e = cudaMemcpyAsync(&hs, d_status, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) rc = fail(PCF_ERR_CUDA, cudaGetErrorString(e));
        if (!rc && user_status) cudaMemcpyAsync(user_status, d_status, sizeof(int), cudaMemcpyDefault, st);
    }
    cudaFreeAsync(d_status, st);
    if (own_keys) cudaFreeAsync(d, st);
    e = cudaStreamSynchronize(st);
    if (!rc && e != cudaSuccess) rc = fail(PCF_ERR_CUDA, cudaGetErrorString(e));
    if (!rc && hs != PCF_OK) rc = fail(hs, hs == PCF_ERR_NAN ? "input contains NaN" : "device status " + std::to_string(hs));
    return rc;
}

// ---------------------------------------------------------------- key-value mode
// vals_out[p] = vals_in[perm[p]]: the payload follows its key's stable permutation.
template <class V>
__global__ void __launch_bounds__(256) k_gather_vals(const DevCtx *__restrict__ c, const u32 *__restrict__ perm,
                                                     const V *__restrict__ vin, V *__restrict__ vout, u64 n) {
    pdl_entry();
    if (c && *c->nan_flag) return;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) vout[i] = vin[perm[i]];
}

static size_t pairs_perm_bytes(size_t n) { return align_up(n * 4, 256); }

template <class K, class V>
static int sort_pairs(const u64 *kin, const V *vin, u64 *kout, V *vout, size_t n, const pcf_params *pp, cudaStream_t st) {
    pcf_params p;
    pcf_params_init(&p);
    if (pp) {
        if (pp->struct_size < PCF_PARAMS_V1_SIZE) return fail(PCF_ERR_INVALID_ARG, "pcf_params.struct_size too small");
        memcpy(&p, pp, std::min<size_t>(pp->struct_size, sizeof(pcf_params)));
        p.struct_size = sizeof(pcf_params);
    }
    if (n == 0) return sort_device<K, true>(kin, kout, 0, &p, st, nullptr);
    if (!vin || !vout) return fail(PCF_ERR_INVALID_ARG, "NULL value pointer with n > 0");
    if (((uintptr_t)vin % sizeof(V)) || ((uintptr_t)vout % sizeof(V))) return fail(PCF_ERR_INVALID_ARG, "misaligned values");
    {
        const uintptr_t a0 = (uintptr_t)vin, a1 = a0 + n * sizeof(V), b0 = (uintptr_t)vout, b1 = b0 + n * sizeof(V);
        if (a0 < b1 && b0 < a1) return fail(PCF_ERR_INVALID_ARG, "vals_in and vals_out must not overlap");
    }
    const size_t pb = pairs_perm_bytes(n), sw = workspace_bytes_impl(n, true);
    char *ws = (char *)p.workspace;
    bool own = false;
    if (ws) {
        if (p.workspace_bytes < pb + sw) return fail(PCF_ERR_WORKSPACE_TOO_SMALL, "workspace smaller than pcf_workspace_bytes(PCF_KEY_PAIRS)");
        if ((uintptr_t)ws & 255) return fail(PCF_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
    } else {
        if (cudaMallocAsync((void **)&ws, pb + sw, st) != cudaSuccess) { cudaGetLastError(); return fail(PCF_ERR_OOM, "cudaMallocAsync workspace failed"); }
        own = true;
    }
    struct Freer {
        bool own; char *ws; cudaStream_t st;
        ~Freer() { if (own) cudaFreeAsync(ws, st); }
    } freer{own, ws, st};
    u32 *perm = (u32 *)ws;
    const bool sync = (p.flags & (PCF_FLAG_SYNC | PCF_FLAG_TIMING)) != 0;
    int *user_status = p.status_out;
    int *d_status = nullptr;
    if (sync) {   // the gather runs after the sort: synchronise once, after it
        if (cudaMallocAsync((void **)&d_status, sizeof(int), st) != cudaSuccess) { cudaGetLastError(); return fail(PCF_ERR_OOM, "status alloc failed"); }
        p.status_out = d_status;
    }
    p.flags &= ~(PCF_FLAG_SYNC | PCF_FLAG_TIMING);
    p.workspace = ws + pb;
    p.workspace_bytes = sw;
    int rc = sort_device<K, true>(kin, kout, n, &p, st, perm);
    if (!rc) {
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const DevCtx *dc = n <= (size_t)S_CAP ? (const DevCtx *)p.workspace
                                              : (const DevCtx *)((char *)p.workspace + layout_for(caps_for(n), true).ctx);
        const u32 grid = (u32)std::min<u64>((n + 255) / 256, (u64)nsm * 16);
        CK(launch_pdl(k_gather_vals<V>, grid, 256, 0, st, dc, (const u32 *)perm, vin, vout, (u64)n));
    }
    if (sync) {
        int hs = PCF_OK;
        if (!rc) {
            if (user_status) CK(cudaMemcpyAsync(user_status, d_status, sizeof(int), cudaMemcpyDefault, st));
            CK(cudaMemcpyAsync(&hs, d_status, sizeof(int), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (p.stats) p.stats->host_syncs = 1;
        }
        cudaFreeAsync(d_status, st);
        if (!rc && hs != PCF_OK) rc = fail(hs, hs == PCF_ERR_NAN ? "input contains NaN" : "device status " + std::to_string(hs));
    }
    return rc;
}

// ---------------------------------------------------------------- sharded sort (pcf_shard.cuh)
struct ShardLayout {
    size_t S, cnt, T, Hloc, Hall, Hg, C, Pm, bsum, total;
    u32 P, ntmax;
};
static ShardLayout shard_layout(u64 N, u32 R) {
    ShardLayout L;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    L.P = (u32)iroot34(N);
    const u64 nb = (u64)L.P + 2;
    L.ntmax = (u32)(N / SH_TILE + 1);
    L.S = take(sizeof(ShardState));
    L.cnt = take(nb * 4);
    L.T = take(nb * 4);
    L.Hloc = take(nb * 4);
    L.Hall = take(nb * 4 * R);
    L.Hg = take(nb * 4);
    L.C = take((u64)R * L.ntmax * 4);
    L.Pm = take((u64)R * L.ntmax * 4);
    L.bsum = take(((u64)R * L.ntmax / SCAN_CHUNK + 2) * 4);
    L.total = off;
    return L;
}

static int shard_check(const pcf_shard *sh) {
    if (!sh || !sh->state) return fail(PCF_ERR_INVALID_ARG, "NULL shard descriptor / state");
    if (sh->R < 1 || sh->R > SHARD_RMAX || sh->rank >= sh->R) return fail(PCF_ERR_INVALID_ARG, "R must be in [1, 64], rank < R");
    if (sh->N < 2 || sh->N >= (1ull << 32)) return fail(PCF_ERR_INVALID_ARG, "N must be in [2, 2^32)");
    if (((uintptr_t)sh->state & 255) || sh->state_bytes < shard_layout(sh->N, sh->R).total)
        return fail(PCF_ERR_WORKSPACE_TOO_SMALL, "shard state smaller than pcf_shard_state_bytes() or misaligned");
    return PCF_OK;
}

template <class K>
static int shard_minmax(const u64 *x, size_t n, const pcf_shard *sh, cudaStream_t st) {
    int rc = shard_check(sh);
    if (rc) return rc;
    ShardState *S = (ShardState *)((char *)sh->state + shard_layout(sh->N, sh->R).S);
    long long init[4] = {0x7fffffffffffffffll, (long long)0x8000000000000000ull, 0, 0};
    CK(cudaMemcpyAsync(S->mm, init, sizeof init, cudaMemcpyHostToDevice, st));
    if (n) {
        k_shard_minmax<K><<<(u32)std::min<u64>((n + 255) / 256, 148ull * 8), 256, 0, st>>>(x, n, S);
        CK(cudaGetLastError());
    }
    return PCF_OK;
}

template <class K>
static int shard_counts(const u64 *x, size_t n, const pcf_shard *sh, const pcf_params *pp, cudaStream_t st) {
    int rc = shard_check(sh);
    if (rc) return rc;
    pcf_params p;
    pcf_params_init(&p);
    if (pp) memcpy(&p, pp, std::min<size_t>(pp->struct_size, sizeof(pcf_params)));
    const ShardLayout L = shard_layout(sh->N, sh->R);
    char *b = (char *)sh->state;
    u32 *cnt = (u32 *)(b + L.cnt);
    CK(cudaMemsetAsync(cnt, 0, ((u64)L.P + 2) * 4, st));
    const u32 alpha = (p.flags & PCF_FLAG_SAMPLE_ALL) ? (u32)sh->N : L.P;
    k_shard_counts<K><<<(alpha + 255) / 256, 256, 0, st>>>(x, n, sh->offset, sh->N, alpha, L.P, p.seed, p.flags,
                                                            (const ShardState *)(b + L.S), cnt);
    CK(cudaGetLastError());
    return PCF_OK;
}

template <class K>
static int shard_histogram(const u64 *x, size_t n, const pcf_shard *sh, const pcf_params *pp, cudaStream_t st) {
    int rc = shard_check(sh);
    if (rc) return rc;
    pcf_params p;
    pcf_params_init(&p);
    if (pp) memcpy(&p, pp, std::min<size_t>(pp->struct_size, sizeof(pcf_params)));
    const ShardLayout L = shard_layout(sh->N, sh->R);
    char *b = (char *)sh->state;
    const u32 alpha = (p.flags & PCF_FLAG_SAMPLE_ALL) ? (u32)sh->N : L.P;
    u32 *T = (u32 *)(b + L.T), *H = (u32 *)(b + L.Hloc);
    ShardState *S = (ShardState *)(b + L.S);
    k_shard_table<<<1, 1024, 0, st>>>((const u32 *)(b + L.cnt), L.P, alpha, L.P, T);
    CK(cudaMemsetAsync(H, 0, ((u64)L.P + 2) * 4, st));
    // a degenerate global range (R9/R10) puts every key in bucket 1: the plan then
    // gives the whole array to rank 0, which Standard-Sorts it
    k_shard_deg_hist<K><<<1, 1, 0, st>>>(S, L.P, (u64)n, H);
    if (n) k_shard_hist<K><<<(u32)std::min<u64>((n + 255) / 256, 148ull * 8), 256, 0, st>>>(x, n, L.P, S, T, H);
    CK(cudaGetLastError());
    return PCF_OK;
}

template <class K>
static int shard_partition(const u64 *x, size_t n, const pcf_shard *sh, u64 *y, uint64_t *send_h, uint64_t *recv_h,
                           uint64_t *range_h, cudaStream_t st) {
    int rc = shard_check(sh);
    if (rc) return rc;
    const ShardLayout L = shard_layout(sh->N, sh->R);
    char *b = (char *)sh->state;
    ShardState *S = (ShardState *)(b + L.S);
    const u32 R = sh->R;
    k_shard_plan<<<1, 1024, 0, st>>>((const u32 *)(b + L.Hall), R, sh->rank, L.P, sh->N, (u32 *)(b + L.Hg), S);
    CK(cudaGetLastError());
    if (n) {
        const u32 nt = (u32)((n + SH_TILE - 1) / SH_TILE);
        if (nt > L.ntmax) return fail(PCF_ERR_INVALID_ARG, "shard larger than N");
        u32 *C = (u32 *)(b + L.C), *Pm = (u32 *)(b + L.Pm), *bs = (u32 *)(b + L.bsum);
        const u32 *T = (const u32 *)(b + L.T);
        k_shard_dcount<K><<<nt, SH_WARPS * 32, 0, st>>>(x, n, L.P, R, S, T, C, nt);
        const u64 tot = (u64)R * nt;
        const u32 nblk = (u32)((tot + SCAN_CHUNK - 1) / SCAN_CHUNK);
        k_scan_partials<<<nblk, SCAN_THREADS, 0, st>>>(C, tot, bs);
        k_scan_bsums<<<1, SCAN_THREADS, 0, st>>>(bs, nblk);
        k_scan_final<<<nblk, SCAN_THREADS, 0, st>>>(C, tot, bs, Pm);
        k_shard_dscatter<K><<<nt, SH_WARPS * 32, 0, st>>>(x, n, L.P, R, S, T, Pm, nt, y);
        CK(cudaGetLastError());
    }
    ShardState hs;
    CK(cudaMemcpyAsync(&hs, S, sizeof hs, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));   // the exchange needs the split sizes on the host (all-to-all)
    for (u32 r = 0; r < R; ++r) { if (send_h) send_h[r] = hs.send[r]; if (recv_h) recv_h[r] = hs.recv[r]; }
    if (range_h) { range_h[0] = hs.range_off; range_h[1] = hs.range_m; range_h[2] = hs.J[sh->rank]; range_h[3] = hs.J[sh->rank + 1]; }
    if (hs.mm[2]) return fail(PCF_ERR_NAN, "input contains NaN");
    return PCF_OK;
}

template <class K>
static int shard_sort_range(const u64 *in, u64 *out, size_t m, const pcf_shard *sh, const uint64_t *range_h,
                            const pcf_params *p, cudaStream_t st) {
    int rc = shard_check(sh);
    if (rc) return rc;
    if (!range_h) return fail(PCF_ERR_INVALID_ARG, "NULL range");
    if (range_h[1] != m) return fail(PCF_ERR_INVALID_ARG, "m differs from the planned range size");
    const ShardLayout L = shard_layout(sh->N, sh->R);
    char *b = (char *)sh->state;
    ShardRoot sr;
    sr.N = sh->N; sr.range_off = range_h[0];
    sr.jlo = (u32)range_h[2]; sr.jhi = (u32)range_h[3];
    sr.record = sh->rank == 0;
    sr.S = (const ShardState *)(b + L.S);
    sr.cnt = (const u32 *)(b + L.cnt);
    sr.Hg = (const u32 *)(b + L.Hg);
    if (m == 0) {   // nothing to sort here; the level-1 record still belongs to rank 0
        if (!sr.record || !p || !p->log) return PCF_OK;
    }
    return sort_device<K, false>(in, out, m, p, st, nullptr, &sr);
}

// §4.3 experiment: one M_PCF step with decoupled alpha, beta, gamma (pcf_bucketing.cuh)
static int bucket_counts_f64(const u64 *x, size_t n, u64 alpha, u64 beta, u64 gamma, u64 seed, u32 *b, u32 *H,
                             uint64_t *max_bucket, cudaStream_t st) {
    if (!x || !b || !H) return fail(PCF_ERR_INVALID_ARG, "NULL pointer");
    if (((uintptr_t)x & 7) || ((uintptr_t)b & 3) || ((uintptr_t)H & 3))
        return fail(PCF_ERR_INVALID_ARG, "misaligned pointer (keys 8-byte, b/H 4-byte)");
    if (n < 2 || n >= (1ull << 32)) return fail(PCF_ERR_INVALID_ARG, "n must be in [2, 2^32)");
    if (!alpha || !beta || !gamma || alpha >= (1ull << 32) || beta >= 0xffffffffull || gamma >= 0xffffffffull)
        return fail(PCF_ERR_INVALID_ARG, "alpha, beta, gamma must be in [1, 2^32 - 1)");
    u64 *mm = nullptr;
    CK(cudaMallocAsync(&mm, 3 * sizeof(u64), st));
    int rc = PCF_OK;
    u64 h[3] = {0, 0, 0};
    auto run = [&]() -> int {
        CK(cudaMemsetAsync(mm, 0xff, sizeof(u64), st));
        CK(cudaMemsetAsync(mm + 1, 0, 2 * sizeof(u64), st));
        CK(cudaMemsetAsync(b, 0, (beta + 1) * sizeof(u32), st));
        CK(cudaMemsetAsync(H, 0, (gamma + 1) * sizeof(u32), st));
        int dev = 0, sms = 148;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const u32 gx = (u32)std::min<u64>((n + BK_THREADS - 1) / BK_THREADS, (u64)sms * 8);
        const u32 ga = (u32)std::min<u64>((alpha + BK_THREADS - 1) / BK_THREADS, (u64)sms * 8);
        const u32 gh = (u32)std::min<u64>((gamma + BK_THREADS) / BK_THREADS, (u64)sms * 8);
        k_bk_minmax<<<gx, BK_THREADS, 0, st>>>(x, n, mm);
        k_bk_train<<<ga, BK_THREADS, 0, st>>>(x, n, (u32)alpha, (u32)beta, seed, mm, b);
        k_bk_scan<<<1, 1024, 0, st>>>(b, (u32)(beta + 1));
        k_bk_classify<<<gx, BK_THREADS, 0, st>>>(x, n, (u32)alpha, (u32)beta, (u32)gamma, mm, b, H);
        k_bk_max<<<gh, BK_THREADS, 0, st>>>(H, (u32)(gamma + 1), mm);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h, mm, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return PCF_OK;
    };
    rc = run();
    cudaFreeAsync(mm, st);
    if (rc) return rc;
    double lo, hi;
    const u64 rlo = KeyF64::from_okey(h[0]), rhi = KeyF64::from_okey(h[1]);
    memcpy(&lo, &rlo, 8);
    memcpy(&hi, &rhi, 8);
    if (lo != lo || hi != hi) return fail(PCF_ERR_NAN, "NaN key");
    if (!(hi - lo > 0.0) || !(hi - lo <= 1.7976931348623157e308))
        return fail(PCF_ERR_DEGENERATE, "x_max - x_min is not in (0, inf): M_PCF undefined");
    if (max_bucket) *max_bucket = h[2];
    return PCF_OK;
}

}  // namespace pcf

// ---------------------------------------------------------------- C ABI
extern "C" {

void pcf_params_init(pcf_params *p) {
    if (!p) return;
    memset(p, 0, sizeof *p);
    p->struct_size = sizeof(pcf_params);
    p->tau = 64;
    p->seed = 0;
    p->flags = PCF_FLAG_SYNC;
    p->status_out = NULL;
}

size_t pcf_workspace_bytes(size_t n, int key_type, const pcf_params *p) {
    (void)p;
    if (key_type & PCF_KEY_PAIRS) return n ? pcf::pairs_perm_bytes(n) + pcf::workspace_bytes_impl(n, true) : 0;
    return pcf::workspace_bytes_impl(n, (key_type & PCF_KEY_ARGSORT) != 0);
}

int pcf_sort_f64(const double *in, double *out, size_t n, const pcf_params *p, void *stream) {
    return pcf::sort_device<pcf::KeyF64>(reinterpret_cast<const pcf::u64 *>(in), reinterpret_cast<pcf::u64 *>(out), n, p,
                                         (cudaStream_t)stream);
}

int pcf_sort_u64(const uint64_t *in, uint64_t *out, size_t n, const pcf_params *p, void *stream) {
    return pcf::sort_device<pcf::KeyU64>(reinterpret_cast<const pcf::u64 *>(in), reinterpret_cast<pcf::u64 *>(out), n, p,
                                         (cudaStream_t)stream);
}

int pcf_argsort_f64(const double *in, double *out, uint32_t *perm, size_t n, const pcf_params *p, void *stream) {
    return pcf::sort_device<pcf::KeyF64, true>(reinterpret_cast<const pcf::u64 *>(in), reinterpret_cast<pcf::u64 *>(out), n, p,
                                               (cudaStream_t)stream, perm);
}

int pcf_argsort_u64(const uint64_t *in, uint64_t *out, uint32_t *perm, size_t n, const pcf_params *p, void *stream) {
    return pcf::sort_device<pcf::KeyU64, true>(reinterpret_cast<const pcf::u64 *>(in), reinterpret_cast<pcf::u64 *>(out), n, p,
                                               (cudaStream_t)stream, perm);
}

int pcf_sort_pairs_f64_u32(const double *keys_in, const uint32_t *vals_in, double *keys_out, uint32_t *vals_out, size_t n,
                           const pcf_params *p, void *stream) {
    return pcf::sort_pairs<pcf::KeyF64, uint32_t>(reinterpret_cast<const pcf::u64 *>(keys_in), vals_in,
                                                  reinterpret_cast<pcf::u64 *>(keys_out), vals_out, n, p, (cudaStream_t)stream);
}

int pcf_sort_pairs_f64_u64(const double *keys_in, const uint64_t *vals_in, double *keys_out, uint64_t *vals_out, size_t n,
                           const pcf_params *p, void *stream) {
    return pcf::sort_pairs<pcf::KeyF64, unsigned long long>(reinterpret_cast<const pcf::u64 *>(keys_in),
                                                            reinterpret_cast<const unsigned long long *>(vals_in),
                                                            reinterpret_cast<pcf::u64 *>(keys_out),
                                                            reinterpret_cast<unsigned long long *>(vals_out), n, p, (cudaStream_t)stream);
}

int pcf_sort_pairs_u64_u32(const uint64_t *keys_in, const uint32_t *vals_in, uint64_t *keys_out, uint32_t *vals_out, size_t n,
                           const pcf_params *p, void *stream) {
    return pcf::sort_pairs<pcf::KeyU64, uint32_t>(reinterpret_cast<const pcf::u64 *>(keys_in), vals_in,
                                                  reinterpret_cast<pcf::u64 *>(keys_out), vals_out, n, p, (cudaStream_t)stream);
}

int pcf_sort_pairs_u64_u64(const uint64_t *keys_in, const uint64_t *vals_in, uint64_t *keys_out, uint64_t *vals_out, size_t n,
                           const pcf_params *p, void *stream) {
    return pcf::sort_pairs<pcf::KeyU64, unsigned long long>(reinterpret_cast<const pcf::u64 *>(keys_in),
                                                            reinterpret_cast<const unsigned long long *>(vals_in),
                                                            reinterpret_cast<pcf::u64 *>(keys_out),
                                                            reinterpret_cast<unsigned long long *>(vals_out), n, p, (cudaStream_t)stream);
}

int pcf_sort_f64_host(const double *in_host, double *out_host, size_t n, const pcf_params *p, void *stream) {
    return pcf::sort_host<pcf::KeyF64>(reinterpret_cast<const pcf::u64 *>(in_host), reinterpret_cast<pcf::u64 *>(out_host),
                                       n, p, (cudaStream_t)stream);
}

int pcf_sort_u64_host(const uint64_t *in_host, uint64_t *out_host, size_t n, const pcf_params *p, void *stream) {
    return pcf::sort_host<pcf::KeyU64>(reinterpret_cast<const pcf::u64 *>(in_host), reinterpret_cast<pcf::u64 *>(out_host),
                                       n, p, (cudaStream_t)stream);
}

const char *pcf_status_string(int s) {
    switch (s) {
        case PCF_OK: return "PCF_OK";
        case PCF_ERR_INVALID_ARG: return "PCF_ERR_INVALID_ARG";
        case PCF_ERR_NAN: return "PCF_ERR_NAN";
        case PCF_ERR_WORKSPACE_TOO_SMALL: return "PCF_ERR_WORKSPACE_TOO_SMALL";
        case PCF_ERR_OOM: return "PCF_ERR_OOM";
        case PCF_ERR_CUDA: return "PCF_ERR_CUDA";
        case PCF_ERR_LOG_OVERFLOW: return "PCF_ERR_LOG_OVERFLOW";
        case PCF_ERR_INTERNAL: return "PCF_ERR_INTERNAL";
        case PCF_ERR_DEGENERATE: return "PCF_ERR_DEGENERATE";
        default: return "PCF_ERR_UNKNOWN";
    }
}

int pcf_bucket_counts_f64(const double *keys, size_t n, uint64_t alpha, uint64_t beta, uint64_t gamma,
                          uint64_t seed, uint32_t *b_out, uint32_t *H_out, uint64_t *max_bucket, void *stream) {
    return pcf::bucket_counts_f64(reinterpret_cast<const pcf::u64 *>(keys), n, alpha, beta, gamma, seed, b_out, H_out,
                                  max_bucket, (cudaStream_t)stream);
}

size_t pcf_level1_entries(size_t n, const pcf_params *p) {
    (void)p;
    return n ? (size_t)pcf::iroot34(n) + 2 : 2;
}

size_t pcf_shard_state_bytes(uint64_t N, uint32_t R) { return pcf::shard_layout(N, R ? R : 1).total; }

size_t pcf_shard_workspace_bytes(size_t m, uint64_t N) {
    return pcf::layout_for(pcf::caps_for(m ? m : 1, N), false).total;
}

int pcf_shard_views(const pcf_shard *sh, void **views, uint64_t *sizes) {
    int rc = pcf::shard_check(sh);
    if (rc) return rc;
    const pcf::ShardLayout L = pcf::shard_layout(sh->N, sh->R);
    char *b = (char *)sh->state;
    const uint64_t nb = (uint64_t)L.P + 2;
    views[0] = b + L.S;   // mm is the first member of ShardState
    views[1] = b + L.cnt;
    views[2] = b + L.Hloc;
    views[3] = b + L.Hall;
    sizes[0] = 4; sizes[1] = nb; sizes[2] = nb; sizes[3] = nb * sh->R;
    return PCF_OK;
}

#define PCF_SHARD_DISPATCH(call_f64, call_u64)                                                     \
    do {                                                                                           \
        if (key_type == PCF_KEY_F64) return call_f64;                                              \
        if (key_type == PCF_KEY_U64) return call_u64;                                              \
        return pcf::fail(PCF_ERR_INVALID_ARG, "key_type must be PCF_KEY_F64 or PCF_KEY_U64");      \
    } while (0)

int pcf_shard_minmax(const void *keys, size_t n, int key_type, const pcf_shard *sh, void *stream) {
    const pcf::u64 *k = (const pcf::u64 *)keys;
    PCF_SHARD_DISPATCH(pcf::shard_minmax<pcf::KeyF64>(k, n, sh, (cudaStream_t)stream),
                       pcf::shard_minmax<pcf::KeyU64>(k, n, sh, (cudaStream_t)stream));
}

int pcf_shard_counts(const void *keys, size_t n, int key_type, const pcf_shard *sh, const pcf_params *p, void *stream) {
    const pcf::u64 *k = (const pcf::u64 *)keys;
    PCF_SHARD_DISPATCH(pcf::shard_counts<pcf::KeyF64>(k, n, sh, p, (cudaStream_t)stream),
                       pcf::shard_counts<pcf::KeyU64>(k, n, sh, p, (cudaStream_t)stream));
}

int pcf_shard_histogram(const void *keys, size_t n, int key_type, const pcf_shard *sh, const pcf_params *p, void *stream) {
    const pcf::u64 *k = (const pcf::u64 *)keys;
    PCF_SHARD_DISPATCH(pcf::shard_histogram<pcf::KeyF64>(k, n, sh, p, (cudaStream_t)stream),
                       pcf::shard_histogram<pcf::KeyU64>(k, n, sh, p, (cudaStream_t)stream));
}

int pcf_shard_partition(const void *keys, size_t n, int key_type, const pcf_shard *sh, void *keys_out,
                        uint64_t *send_counts, uint64_t *recv_counts, uint64_t *range, void *stream) {
    const pcf::u64 *k = (const pcf::u64 *)keys;
    pcf::u64 *y = (pcf::u64 *)keys_out;
    PCF_SHARD_DISPATCH(pcf::shard_partition<pcf::KeyF64>(k, n, sh, y, send_counts, recv_counts, range, (cudaStream_t)stream),
                       pcf::shard_partition<pcf::KeyU64>(k, n, sh, y, send_counts, recv_counts, range, (cudaStream_t)stream));
}

int pcf_shard_sort_range(const void *keys, void *out, size_t m, int key_type, const pcf_shard *sh,
                         const uint64_t *range, const pcf_params *p, void *stream) {
    const pcf::u64 *k = (const pcf::u64 *)keys;
    pcf::u64 *y = (pcf::u64 *)out;
    PCF_SHARD_DISPATCH(pcf::shard_sort_range<pcf::KeyF64>(k, y, m, sh, range, p, (cudaStream_t)stream),
                       pcf::shard_sort_range<pcf::KeyU64>(k, y, m, sh, range, p, (cudaStream_t)stream));
}

const char *pcf_last_error(void) { return pcf::g_last_error.c_str(); }

int pcf_abi_version(void) { return PCF_ABI_VERSION; }

}  // extern "C"
