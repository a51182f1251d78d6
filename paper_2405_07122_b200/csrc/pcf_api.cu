// pcf_api.cu -- host orchestration and the C ABI of libpcfsort.so (include/pcf_sort.h).
//
// Call structure for one sort of n keys:
//   n <= S_CAP          one K7 task: the whole Algorithm 1 in one CTA's shared memory.
//   n >  S_CAP          level-1 node on the global path: k_minmax -> k_node_model ->
//                       k_fit_sample -> k_fit_scan, then split rounds (count, scan,
//                       scatter, taskgen) until every group fits a K7 CTA; oversized
//                       recursing buckets become new global nodes (next round);
//                       then one persistent K7 launch over all groups; K8 for buckets
//                       that Alg. 1 sends to Standard-Sort and that exceed S_CAP.
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
#include "pcf_k8.cuh"
#include "pcf_bucketing.cuh"

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

constexpr u32 BND_MIN_LOG2 = 24;   // nodes of >= 2^20 keys get the gather-free digit table

static Caps caps_for(u64 n) {
    Caps c;
    c.n = n;
    c.P = (u32)iroot34(n);
    c.node_cap = (u32)(n / S_CAP + 2);
    // root tables + every oversized node: sum of 3*(m^{3/4}+2) over disjoint m > S_CAP
    // is <= 3*(n^{3/4} + n / S_CAP^{1/4} + 2*node_cap)  (S_CAP^{1/4} > 9.5)
    c.arena_u32 = 3ull * ((u64)c.P + 2) + 3ull * (n * 2 / 19 + 2ull * c.node_cap) + 64
                  + (u64)GMAX * ((n >> BND_MIN_LOG2) + 1);   // digit boundaries of large nodes
    c.k7_cap = (u32)std::min<u64>(n / 32 + 65536, 0xffffffffull);
    c.split_cap = (u32)(n / 1024 + 4096);
    c.items_cap = (u32)(n / S_CAP + 64);
    // every split of a round has <= GMAX digits and ceil(m/SPLIT_TILE) tiles; a round's
    // splits are disjoint segments of > S_CAP keys (or of wider-than-NB_CAP bucket ranges)
    c.cmat_cap = (n / SPLIT_TILE + n / S_CAP + 64) * (u64)GMAX;
    c.bsum_cap = c.cmat_cap / SCAN_CHUNK + 2;
    return c;
}

struct Counters {             // zeroed at the start of every call
    u32 nan_flag, err_flag, k7_count, k7_next;
    u32 nsplits[2], nitems, k7_begin;
    unsigned long long rec_count, k7_keys, split_keys, pad;
    RoundPlan plan;
    unsigned long long k7_prof[K7_PROF_SLOTS];
};

struct Layout {
    size_t ctx, counters, tmp, digs, tmap, k7_order, bmm, bfs, bnl, nodes, acc, arena, k7, splits_a, splits_b, items, cmat, pmat, bsum, total;
};

static Layout layout_for(const Caps &c) {
    Layout L;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    L.ctx = take(sizeof(DevCtx));
    L.counters = take(sizeof(Counters));
    L.tmp = take(c.n * 8);
    L.digs = take(c.n * 2);
    L.tmap = take((c.n / SPLIT_TILE + c.split_cap + 64) * 4);
    L.nodes = take((size_t)c.node_cap * sizeof(GNode));
    L.acc = take((size_t)c.node_cap * sizeof(NodeAcc));
    L.arena = take(c.arena_u32 * 4);
    L.k7 = take((size_t)c.k7_cap * sizeof(K7Task));
    L.k7_order = take((size_t)c.k7_cap * 4);
    // batched global nodes: chunk -> node maps (+ first chunk per node) and the node list
    L.bmm = take((c.n / MMB_CHUNK + 2ull * c.node_cap + 64) * 4);
    L.bfs = take((c.n / FSB_CHUNK + 2ull * c.node_cap + 64) * 4);
    L.bnl = take(((u64)c.node_cap + 64) * 4);
    L.splits_a = take((size_t)c.split_cap * sizeof(SplitTask));
    L.splits_b = take((size_t)c.split_cap * sizeof(SplitTask));
    L.items = take((size_t)c.items_cap * sizeof(SegItem));
    L.cmat = take(c.cmat_cap * 4);
    L.pmat = take(c.cmat_cap * 4);
    L.bsum = take(c.bsum_cap * 4);
    L.total = off;
    return L;
}

static size_t small_layout_bytes() {
    // n <= S_CAP: ctx + counters + one K7 task
    return align_up(sizeof(DevCtx), 256) + align_up(sizeof(Counters), 256) + align_up(sizeof(K7Task), 256);
}

static size_t workspace_bytes_impl(size_t n) {
    if (n == 0) return 0;
    if (n <= (size_t)S_CAP) return small_layout_bytes();
    return layout_for(caps_for(n)).total;
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

enum { PH_MINMAX = 0, PH_FIT = 1, PH_COUNT = 2, PH_SCATTER = 3, PH_K7 = 4, PH_K8 = 5, PH_OTHER = 6, PH_TOTAL = 7 };

static int k7_smem_bytes(u32 tau = 2) { return (int)(sizeof(K7Smem) + k7_lists_bytes(tau < 2 ? 2 : tau)); }
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

template <class K>
static int k7_ctas_per_sm() {   // resident K7 CTAs per SM (persistent grid size)
    static thread_local int v[MAX_DEVS] = {0};
    const int d = cur_dev();
    if (!v[d]) {
        int b = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k7_kernel<K>, K7_THREADS, k7_smem_bytes()) != cudaSuccess || b < 1) b = 1;
        v[d] = b;
    }
    return v[d];
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
    CK(cudaFuncSetAttribute(k7_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, k7_smem_bytes()));
    CK(cudaFuncSetAttribute(k_split_scatter<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, split_smem_bytes()));
    CK(cudaFuncSetAttribute(k_split_count<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CountSmem)));
    CK(cudaFuncSetAttribute(k8_merge<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, K8_MERGE_SMEM));
    CK(cudaFuncSetAttribute(k8_blocksort<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, K8_SORT_SMEM));
    done[d] = true;
    return PCF_OK;
}

// ---------------------------------------------------------------- the sort
template <class K>
static int sort_device(const u64 *in, u64 *out, size_t n, const pcf_params *pp, cudaStream_t st) {
    pcf_params p;
    pcf_params_init(&p);
    if (pp) {
        if (pp->struct_size < sizeof(pcf_params)) return fail(PCF_ERR_INVALID_ARG, "pcf_params.struct_size too small");
        p = *pp;
    }
    if (p.tau < 2) return fail(PCF_ERR_INVALID_ARG, "tau must be >= 2");
    if (n == 0) return PCF_OK;
    if (!in || !out) return fail(PCF_ERR_INVALID_ARG, "NULL key pointer with n > 0");
    if (n >= (1ull << 32)) return fail(PCF_ERR_INVALID_ARG, "n must be < 2^32 in ABI v1");
    if (((uintptr_t)in & 7) || ((uintptr_t)out & 7)) return fail(PCF_ERR_INVALID_ARG, "keys must be 8-byte aligned");
    if (in != out) {
        uintptr_t a0 = (uintptr_t)in, a1 = a0 + n * 8, b0 = (uintptr_t)out, b1 = b0 + n * 8;
        if (a0 < b1 && b0 < a1) return fail(PCF_ERR_INVALID_ARG, "in and out overlap (only in == out is allowed)");
    }
    int rc = configure_kernels<K>();
    if (rc) return rc;

    const bool timing = (p.flags & PCF_FLAG_TIMING) != 0;
    const bool sync = timing || (p.flags & PCF_FLAG_SYNC) != 0;
    const bool logging = p.log != nullptr;
    pcf_stats stats;
    memset(&stats, 0, sizeof stats);
    PhaseTimer tm;
    tm.on = timing;
    tm.st = st;
    cudaEvent_t ev_total0 = nullptr, ev_total1 = nullptr;
    if (timing) {
        cudaEventCreate(&ev_total0);
        cudaEventCreate(&ev_total1);
        cudaEventRecord(ev_total0, st);
    }

    const size_t need = workspace_bytes_impl(n);
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
    if (logging) {
        hc.rec = reinterpret_cast<NodeRec *>(p.log->records);
        hc.rec_cap = p.log->records ? p.log->capacity : 0;
        hc.l1_b = p.log->level1_b;
        hc.l1_h = p.log->level1_h;
        hc.l1_cap = p.log->level1_capacity;
        if (!p.log->count) return fail(PCF_ERR_INVALID_ARG, "pass log needs a count pointer");
        hc.rec_count = reinterpret_cast<unsigned long long *>(p.log->count);
        if (!hc.rec) hc.rec = reinterpret_cast<NodeRec *>(1);   // non-null marks logging on; cap 0
        CK(cudaMemsetAsync(p.log->count, 0, 8, st));
    }

    const bool small = n <= (size_t)S_CAP;
    DevCtx *d_ctx;
    Counters *d_cnt;
    Caps caps;
    Layout L;
    memset(&L, 0, sizeof L);
    if (small) {
        d_ctx = (DevCtx *)ws;
        d_cnt = (Counters *)(ws + align_up(sizeof(DevCtx), 256));
        K7Task *d_task = (K7Task *)(ws + align_up(sizeof(DevCtx), 256) + align_up(sizeof(Counters), 256));
        hc.k7 = d_task;
        hc.k7_cap = 1;
        hc.buf[1] = nullptr;
    } else {
        caps = caps_for(n);
        L = layout_for(caps);
        d_ctx = (DevCtx *)(ws + L.ctx);
        d_cnt = (Counters *)(ws + L.counters);
        hc.buf[1] = (u64 *)(ws + L.tmp);
        hc.nodes = (GNode *)(ws + L.nodes);
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
        hc.cmat_cap = caps.cmat_cap;
        hc.digs = (u16 *)(ws + L.digs);
        hc.tmap = (u32 *)(ws + L.tmap);
    }
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
    CK(cudaMemcpyAsync(d_ctx, &hc, sizeof hc, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(d_cnt, 0, sizeof(Counters), st));

    const bool sample_all = (p.flags & PCF_FLAG_SAMPLE_ALL) != 0;
    u32 launches = 0;
    int status = PCF_OK;
    std::vector<SegItem> fallbacks;
    u64 k7_tasks = 0, split_moved = 0, global_keys = 0;
    u64 bytes[PCF_PHASES] = {0};
    std::vector<u32> global_nodes;   // indices (for the pass-log finalisation)

    if (small) {
        K7Task t;
        memset(&t, 0, sizeof t);
        t.off = 0; t.size = (u32)n; t.kind = K7_NODE; t.src = 0; t.level = 1;
        CK(cudaMemcpyAsync(hc.k7, &t, sizeof t, cudaMemcpyHostToDevice, st));
        u32 one = 1;
        CK(cudaMemcpyAsync(&d_cnt->k7_count, &one, 4, cudaMemcpyHostToDevice, st));
        tm.begin(PH_K7);
        k7_kernel<K><<<1, K7_THREADS, k7_smem_bytes(p.tau), st>>>(d_ctx);
        CK(cudaGetLastError());
        tm.end();
        launches++;
        k7_tasks = 1;
        bytes[PH_K7] += 16ull * n;
    } else {
        // ------------------------------------------------ global nodes
        u64 arena_used = 0;
        u32 *arena = (u32 *)(ws + L.arena);
        u32 node_count = 0;
        std::vector<SplitTask> list;
        std::vector<u32> batch;   // nodes whose fit is launched together
        std::vector<GNode> batch_nodes;
        u64 batch_arena0 = 0;
        std::vector<u32> node_m, node_alpha;
        auto add_node = [&](u64 off, u32 m, u32 level, u32 src, bool batched) -> int {
            if (node_count >= caps.node_cap) return fail(PCF_ERR_INTERNAL, "global node capacity exceeded");
            GNode g;
            memset(&g, 0, sizeof g);
            u32 P = (u32)iroot34(m);
            g.off = off; g.m = m; g.level = level;
            g.kmin = ~0ull; g.kmax = 0;
            g.alpha = sample_all ? m : P; g.beta = P; g.gamma = P; g.delta = P;
            g.src = src;
            u64 need_u32 = 3ull * ((u64)P + 2);
            if (arena_used + need_u32 > caps.arena_u32) return fail(PCF_ERR_INTERNAL, "node table arena exceeded");
            g.cnt = arena + arena_used;
            g.T = g.cnt + (P + 2);
            g.H = g.T + (P + 2);
            arena_used += need_u32;
            const u32 sh0 = choose_shift(P + 1, m);
            if (!batched && m >= (1u << BND_MIN_LOG2) && arena_used + GMAX <= caps.arena_u32) {
                g.bnd = arena + arena_used;
                arena_used += GMAX;
                g.bshift = sh0;
                g.bG = (P + 1 + (1u << sh0) - 1) >> sh0;
            }
            u32 idx = node_count++;
            node_m.push_back(m);
            node_alpha.push_back(g.alpha);
            if (!batched) {
                CK(cudaMemcpyAsync(hc.nodes + idx, &g, sizeof g, cudaMemcpyHostToDevice, st));
                CK(cudaMemsetAsync(g.cnt, 0, need_u32 * 4, st));
            }
            const DevCtx *dc = d_ctx;
            if (batched) {   // uploaded (nodes, zeroed tables) with the rest of the batch
                if (batch.empty()) batch_arena0 = (u64)(g.cnt - arena);
                batch_nodes.push_back(g);
                batch.push_back(idx);
                bytes[PH_MINMAX] += 8ull * m;
                bytes[PH_FIT] += 8ull * g.alpha + 8ull * (P + 2);
            } else {
            tm.begin(PH_MINMAX);
            u64 nvec = m / 2 + 1;
            u32 grid = (u32)std::min<u64>(148ull * 8, (nvec + MM_THREADS * MM_UNROLL - 1) / (MM_THREADS * MM_UNROLL));
            CK(launch_pdl(k_minmax<K>, grid, MM_THREADS, 0, st, dc, idx));
            tm.end();
            tm.begin(PH_FIT);
            u32 alpha = g.alpha;
            CK(launch_pdl(k_fit_sample<K>, (alpha + 255) / 256, 256, 0, st, dc, idx));
            {
                u64 nbins = (u64)P + 1;
                u32 nblk = (u32)((nbins + SCAN_CHUNK - 1) / SCAN_CHUNK);
                u32 *bs = (u32 *)(ws + L.bsum);
                CK(launch_pdl(k_scan_partials, nblk, SCAN_THREADS, 0, st, (const u32 *)(g.cnt + 1), (u64)nbins, bs));
                CK(launch_pdl(k_scan_bsums, 1, SCAN_THREADS, 0, st, bs, nblk));
                CK(launch_pdl(k_fit_final, nblk, SCAN_THREADS, 0, st, dc, idx, (const u32 *)bs));
            }
            tm.end();
            CK(cudaGetLastError());
            launches += 5;
            bytes[PH_MINMAX] += 8ull * m;
            bytes[PH_FIT] += 8ull * alpha + 8ull * (P + 2);
            }
            stats.global_nodes++;
            global_nodes.push_back(idx);
            SplitTask s;
            memset(&s, 0, sizeof s);
            s.off = off; s.m = m; s.node = idx; s.jlo = 1; s.jhi = P + 2;
            s.shift = sh0;
            s.G = (P + 1 + (1u << s.shift) - 1) >> s.shift;
            s.src = src; s.dst = src == 1 ? 2 : 1;
            list.push_back(s);
            return PCF_OK;
        };
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        // host-side list of splits to append to the device list of the next round
        rc = add_node(0, (u32)n, 1, 0, false);
        if (rc) return rc;
        u32 round = 0;
        u32 pending = 0;   // splits already in the device list splits[round & 1]
        auto flush_list = [&]() -> int {
            if (list.empty()) return PCF_OK;
            const u32 cur = round & 1u;
            if (pending + list.size() > caps.split_cap) return fail(PCF_ERR_INTERNAL, "split list capacity exceeded");
            CK(cudaMemcpyAsync(hc.splits[cur] + pending, list.data(), list.size() * sizeof(SplitTask),
                               cudaMemcpyHostToDevice, st));
            pending += (u32)list.size();
            CK(cudaMemcpyAsync(&d_cnt->nsplits[cur], &pending, 4, cudaMemcpyHostToDevice, st));
            list.clear();
            return PCF_OK;
        };
        // upper bound on the tiles of the next round: its keys are <= n and it has at most
        // (splits in it) partial tiles; the first round has 1 split, the second <= GMAX
        u64 splits_bound = 0;   // upper bound on the splits of the round being enqueued
        auto enqueue_round = [&]() -> int {
            const u32 cur = round & 1u;
            const u32 tile_grid = (u32)std::min<u64>(n / SPLIT_TILE + 1 + splits_bound, 0x7fffffffull);
            // each split yields <= GMAX next splits; overflow carry-over adds <= the current ones
            splits_bound = std::min<u64>(splits_bound * (GMAX + 1), caps.split_cap);
            tm.begin(PH_OTHER);
            CK(launch_pdl(k_round_plan, 1, 1024, 0, st, (const DevCtx *)d_ctx, cur));
            CK(launch_pdl(k_tile_map, nsm * 2, 256, 0, st, (const DevCtx *)d_ctx, cur));
            tm.end();
            tm.begin(PH_COUNT);
            // one CTA per tile for small sorts and for rounds after the first (their T
            // gathers are local to a split: they need L1, which the persistent kernel's
            // 2 x 111 KB of staging takes); the persistent bulk-copy kernel for the first
            // round of a large sort (gather-free digit table)
            if (n <= (1ull << 25) || round > 0) CK(launch_pdl(k_split_count_tile<K>, tile_grid, SC_THREADS, 0, st, (const DevCtx *)d_ctx, cur));
            else CK(launch_pdl(k_split_count<K>, nsm * count_ctas_per_sm<K>(), CNT_THREADS, sizeof(CountSmem), st, (const DevCtx *)d_ctx, cur));
            tm.end();
            tm.begin(PH_OTHER);
            CK(launch_pdl(k_scanp_partials, nsm * 2, SCAN_THREADS, 0, st, (const DevCtx *)d_ctx));
            CK(launch_pdl(k_scanp_bsums, 1, SCAN_THREADS, 0, st, (const DevCtx *)d_ctx));
            CK(launch_pdl(k_scanp_final, nsm * 2, SCAN_THREADS, 0, st, (const DevCtx *)d_ctx));
            tm.end();
            tm.begin(PH_SCATTER);
            CK(launch_pdl(k_split_scatter<K>, tile_grid, SC_THREADS, split_smem_bytes(), st, (const DevCtx *)d_ctx, cur));
            tm.end();
            tm.begin(PH_OTHER);
            CK(launch_pdl(k_split_taskgen, nsm * 2, TG_THREADS, 0, st, (const DevCtx *)d_ctx, cur));
            tm.end();
            launches += 8;
            round++;
            return PCF_OK;
        };
        u32 rounds_per_batch = 2;   // enough for 10^6..10^9 keys of well-modelled data
        for (;;) {
            rc = flush_list();
            if (rc) return rc;
            splits_bound = pending;
            for (u32 k = 0; k < rounds_per_batch; ++k) {
                rc = enqueue_round();
                if (rc) return rc;
            }
            CK(cudaGetLastError());
            // K7 over every group produced so far (persistent grid; reads the task count on the device)
            tm.begin(PH_K7);
            CK(launch_pdl(k_k7_order, 1, 1024, 0, st, (const DevCtx *)d_ctx));
            CK(launch_pdl(k7_kernel<K>, nsm * k7_ctas_per_sm<K>(), K7_THREADS, k7_smem_bytes(p.tau), st, (const DevCtx *)d_ctx));
            CK(launch_pdl(k_k7_advance, 1, 1, 0, st, (const DevCtx *)d_ctx));
            tm.end();
            CK(cudaGetLastError());
            launches += 3;
            Counters hcnt;
            CK(cudaMemcpyAsync(&hcnt, d_cnt, sizeof hcnt, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            stats.host_syncs++;
            if (hcnt.nan_flag) { status = PCF_ERR_NAN; break; }
            if (hcnt.err_flag) return fail(PCF_ERR_INTERNAL, "device work-queue capacity exceeded (err_flag=" + std::to_string(hcnt.err_flag) + ")");
            k7_tasks = hcnt.k7_count;
            pending = hcnt.nsplits[round & 1u];
            std::vector<SegItem> items(hcnt.nitems);
            if (hcnt.nitems) {
                CK(cudaMemcpyAsync(items.data(), hc.items, hcnt.nitems * sizeof(SegItem), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                CK(cudaMemsetAsync(&d_cnt->nitems, 0, 4, st));
            }
            for (const SegItem &it : items) {
                if (it.kind == 0) { rc = add_node(it.off, it.m, it.level, it.src, true); if (rc) return rc; }
                else fallbacks.push_back(it);
            }
            if (!batch.empty()) {   // one min/max, one sampling and one fit launch for every new node
                std::vector<u32> cmm, fmm, cfs, ffs;
                u64 nkeys = 0;
                // the batch's node records (consecutive indices) and its zeroed table range
                CK(cudaMemcpyAsync(hc.nodes + batch[0], batch_nodes.data(), batch_nodes.size() * sizeof(GNode),
                                   cudaMemcpyHostToDevice, st));
                CK(cudaMemsetAsync(arena + batch_arena0, 0, (arena_used - batch_arena0) * 4, st));
                for (u32 idx : batch) {
                    fmm.push_back((u32)cmm.size());
                    ffs.push_back((u32)cfs.size());
                    const u32 m = node_m[idx], al = node_alpha[idx];
                    for (u32 q = 0; q < (m + MMB_CHUNK - 1) / MMB_CHUNK; ++q) cmm.push_back(idx);
                    for (u32 q = 0; q < (al + FSB_CHUNK - 1) / FSB_CHUNK; ++q) cfs.push_back(idx);
                    nkeys += m;
                }
                // first-chunk tables are indexed by node: scatter them into node-sized arrays
                std::vector<u32> nfm(node_count, 0), nfs(node_count, 0);
                for (size_t i = 0; i < batch.size(); ++i) { nfm[batch[i]] = fmm[i]; nfs[batch[i]] = ffs[i]; }
                u32 *d_cmm = (u32 *)(ws + L.bmm), *d_nfm = d_cmm + cmm.size();
                u32 *d_cfs = (u32 *)(ws + L.bfs), *d_nfs = d_cfs + cfs.size();
                u32 *d_nl = (u32 *)(ws + L.bnl);
                CK(cudaMemcpyAsync(d_cmm, cmm.data(), cmm.size() * 4, cudaMemcpyHostToDevice, st));
                CK(cudaMemcpyAsync(d_nfm, nfm.data(), nfm.size() * 4, cudaMemcpyHostToDevice, st));
                CK(cudaMemcpyAsync(d_cfs, cfs.data(), cfs.size() * 4, cudaMemcpyHostToDevice, st));
                CK(cudaMemcpyAsync(d_nfs, nfs.data(), nfs.size() * 4, cudaMemcpyHostToDevice, st));
                CK(cudaMemcpyAsync(d_nl, batch.data(), batch.size() * 4, cudaMemcpyHostToDevice, st));
                tm.begin(PH_MINMAX);
                CK(launch_pdl(k_minmax_batch<K>, (u32)cmm.size(), MM_THREADS, 0, st, (const DevCtx *)d_ctx,
                              (const u32 *)d_cmm, (const u32 *)d_nfm));
                tm.end();
                tm.begin(PH_FIT);
                CK(launch_pdl(k_fit_sample_batch<K>, (u32)cfs.size(), FSB_CHUNK, 0, st, (const DevCtx *)d_ctx,
                              (const u32 *)d_cfs, (const u32 *)d_nfs));
                CK(launch_pdl(k_fit_batch, (u32)batch.size(), SCAN_THREADS, 0, st, (const DevCtx *)d_ctx, (const u32 *)d_nl));
                tm.end();
                launches += 3;
                batch.clear();
                batch_nodes.clear();
            }
            split_moved = hcnt.split_keys;
            bytes[PH_K7] = 16ull * hcnt.k7_keys;
            if (pending == 0 && list.empty()) break;
            rounds_per_batch = 2;
        }
        stats.rounds = round;
        stats.split_keys_moved = split_moved;
        // one classify (8 B/key) and one stable scatter (16 B/key) per
        // bucketing level of every key the global path buckets; extra digit rounds are
        // traffic, not algorithmic bytes (reported as split_keys_moved)
        for (u32 m_ : node_m) global_keys += m_;
        bytes[PH_COUNT] = 8ull * global_keys;
        bytes[PH_SCATTER] = 16ull * global_keys;
        if (status == PCF_OK) {
            // K8: global Standard-Sort of large buckets (flags in pmat, merge splits in cmat:
            // both are free once the split rounds are done)
            u32 *k8_flags = hc.pmat, *k8_sp = hc.cmat;
            if (!fallbacks.empty()) CK(cudaMemsetAsync(k8_flags, 0, 4 * fallbacks.size(), st));
            for (size_t fi = 0; fi < fallbacks.size(); ++fi) {
                const SegItem &it = fallbacks[fi];
                const u64 m = it.m;
                u64 *src = (it.src == 0 ? const_cast<u64 *>(in) : it.src == 1 ? hc.buf[1] : out) + it.off;
                u64 *bo = out + it.off, *bt = hc.buf[1] + it.off;
                u32 *flag = k8_flags + fi;
                u32 npass = 1;
                for (u64 w = K8_TILE; w < m; w *= 2) npass++;
                // pass k writes `out` iff (npass - 1 - k) is even, so the last pass lands in out
                u64 *dst0 = ((npass - 1) % 2 == 0) ? bo : bt;
                const u32 nblk = (u32)((m + K8_TILE - 1) / K8_TILE);
                tm.begin(PH_K8);
                k8_check<<<(u32)std::min<u64>(4ull * nsm, (m + 255) / 256), 256, 0, st>>>(src, m, flag);
                k8_blocksort<K><<<nblk, K8_THREADS, K8_SORT_SMEM, st>>>(src, dst0, bo, m, flag);
                u64 *cur = dst0;
                for (u64 w = K8_TILE; w < m; w *= 2) {
                    u64 *nxt = cur == bo ? bt : bo;
                    const u32 nmt = (u32)((m + K8_MTILE - 1) / K8_MTILE);
                    k8_partition<K><<<(nmt + 255) / 256, 256, 0, st>>>(cur, m, w, nmt, k8_sp, flag);
                    k8_merge<K><<<nmt, K8_MTHREADS, K8_MERGE_SMEM, st>>>(cur, nxt, m, w, k8_sp, flag, 2 * w >= m ? 1u : 0u);
                    cur = nxt;
                    launches += 2;
                }
                tm.end();
                launches += 2;
                CK(cudaGetLastError());
                bytes[PH_K8] += 24ull * m;   // check + block sort; the merge passes are added below (timing)
                stats.fallback_keys_global += m;
            }
            if (timing && !fallbacks.empty()) {   // merge passes run only for buckets with two distinct keys
                std::vector<u32> fl(fallbacks.size());
                CK(cudaMemcpyAsync(fl.data(), k8_flags, 4 * fl.size(), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                for (size_t fi = 0; fi < fl.size(); ++fi) {
                    u32 npass = 1;
                    for (u64 w = K8_TILE; w < fallbacks[fi].m; w *= 2) npass++;
                    if (fl[fi]) bytes[PH_K8] += 16ull * fallbacks[fi].m * (npass - 1);
                }
            }
            // pass log: records of the global nodes (need the complete H)
            if (logging) {
                NodeAcc *acc = (NodeAcc *)(ws + L.acc);
                CK(cudaMemsetAsync(acc, 0, sizeof(NodeAcc) * node_count, st));
                for (u32 idx : global_nodes) {
                    k_node_finalize_acc<<<64, 256, 0, st>>>(d_ctx, idx, acc + idx);
                    k_node_finalize_rec<K><<<1, 1, 0, st>>>(d_ctx, idx, acc + idx);
                    launches += 2;
                }
                CK(cudaGetLastError());
            }
        }
    }
    stats.groups_smem = k7_tasks;
    if (timing) cudaEventRecord(ev_total1, st);
    if (sync) {
        Counters hcnt;
        CK(cudaMemcpyAsync(&hcnt, d_cnt, sizeof hcnt, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        stats.host_syncs++;
        if (hcnt.nan_flag) status = PCF_ERR_NAN;
        else if (hcnt.err_flag) status = fail(PCF_ERR_INTERNAL, "device capacity exceeded (err_flag=" + std::to_string(hcnt.err_flag) + ")");
        if (status == PCF_OK && logging) {
            unsigned long long cnt = 0;
            CK(cudaMemcpy(&cnt, p.log->count, 8, cudaMemcpyDeviceToHost));
            if (cnt > p.log->capacity) status = fail(PCF_ERR_LOG_OVERFLOW, "pass log capacity exceeded");
        }
        if (status == PCF_ERR_NAN) fail(PCF_ERR_NAN, "input contains NaN");
        for (int i = 0; i < K7_PROF_SLOTS; ++i) stats.k7_cycles[i] = hcnt.k7_prof[i];
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
        if (pp->struct_size < sizeof(pcf_params)) return fail(PCF_ERR_INVALID_ARG, "pcf_params.struct_size too small");
        p = *pp;
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
    int rc = PCF_OK;
    e = cudaMemcpyAsync(d, in_h, n * 8, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rc = fail(PCF_ERR_CUDA, cudaGetErrorString(e));
    if (!rc) rc = sort_device<K>(d, d, n, &p, st);
    if (!rc) {
        e = cudaMemcpyAsync(out_h, d, n * 8, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) rc = fail(PCF_ERR_CUDA, cudaGetErrorString(e));
    }
    if (own_keys) cudaFreeAsync(d, st);
    e = cudaStreamSynchronize(st);
    if (!rc && e != cudaSuccess) rc = fail(PCF_ERR_CUDA, cudaGetErrorString(e));
    return rc;
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
}

size_t pcf_workspace_bytes(size_t n, int key_type, const pcf_params *p) {
    (void)key_type;
    (void)p;
    return pcf::workspace_bytes_impl(n);
}

int pcf_sort_f64(const double *in, double *out, size_t n, const pcf_params *p, void *stream) {
    return pcf::sort_device<pcf::KeyF64>(reinterpret_cast<const pcf::u64 *>(in), reinterpret_cast<pcf::u64 *>(out), n, p,
                                         (cudaStream_t)stream);
}

int pcf_sort_u64(const uint64_t *in, uint64_t *out, size_t n, const pcf_params *p, void *stream) {
    return pcf::sort_device<pcf::KeyU64>(reinterpret_cast<const pcf::u64 *>(in), reinterpret_cast<pcf::u64 *>(out), n, p,
                                         (cudaStream_t)stream);
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

const char *pcf_last_error(void) { return pcf::g_last_error.c_str(); }

int pcf_abi_version(void) { return PCF_ABI_VERSION; }

}  // extern "C"
