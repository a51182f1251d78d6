// pcf_global.cuh -- multi-CTA kernels for bucketing nodes larger than one CTA's
// shared memory (the level-1 array and oversized recursing buckets).
//
//   k_minmax        x_min / x_max of the segment under totalOrder, NaN flag
//   k_node_model    i(x) parameters, degenerate-range test (R9, R10)
//   k_fit_sample    alpha seeded sample positions, i(a_k), per-bin counts
//   k_fit_scan      b = prefix of counts, T[i] = floor(b_i*gamma/alpha)+1    (R7)
//   k_split_count   per-tile digit counts of d(x) = (T[i(x)] - jlo) >> shift (digit-major matrix)
//   k_scan_*        exclusive scan of the count matrix -> per-(digit, tile) output offsets
//   k_split_scatter stable placement by digit (Append order)
//   k_split_taskgen one task per non-empty digit group (K7 group / node / sort,
//                   deeper split, or an item for the host: large node / fallback)
// A "split" is a stable partition of a segment by a digit of its bucket index
// j; composing splits with a final in-smem placement by j (K7) equals the
// paper's single stable placement by j because stable partitions compose.
#pragma once
#include "pcf_common.cuh"

namespace pcf {

constexpr int MM_THREADS = 256;
constexpr int MM_UNROLL = 4;

__device__ __forceinline__ ulonglong2 ld_stream(const ulonglong2 *p) {
    ulonglong2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p));
    return r;
}

template <class K>
__device__ __forceinline__ void mm_acc(u64 raw, u64 &mn, u64 &mx, bool &nan) {
    if (K::is_f64) nan |= (raw & 0x7fffffffffffffffull) > 0x7ff0000000000000ull;
    u64 k = K::to_okey(raw);
    mn = k < mn ? k : mn;
    mx = k > mx ? k : mx;
}

template <class K>
__global__ void __launch_bounds__(MM_THREADS) k_minmax(const DevCtx *__restrict__ c, u32 node) {
    pdl_entry();
    GNode &g = c->nodes[node];
    const u64 *x = c->buf[g.src] + g.off;
    const u64 m = g.m;
    u64 mn = ~0ull, mx = 0;
    bool nan = false;
    const u64 head = (((uintptr_t)x & 15) && m) ? 1 : 0;
    const ulonglong2 *v = reinterpret_cast<const ulonglong2 *>(x + head);
    const u64 nv = (m - head) / 2;
    const u64 gtid = (u64)blockIdx.x * MM_THREADS + threadIdx.x;
    const u64 stride = (u64)gridDim.x * MM_THREADS;
    u64 i = gtid;
    for (; i + (MM_UNROLL - 1) * stride < nv; i += MM_UNROLL * stride) {
        ulonglong2 r[MM_UNROLL];
#pragma unroll
        for (int u = 0; u < MM_UNROLL; ++u) r[u] = ld_stream(v + i + u * stride);
#pragma unroll
        for (int u = 0; u < MM_UNROLL; ++u) { mm_acc<K>(r[u].x, mn, mx, nan); mm_acc<K>(r[u].y, mn, mx, nan); }
    }
    for (; i < nv; i += stride) { ulonglong2 r = ld_stream(v + i); mm_acc<K>(r.x, mn, mx, nan); mm_acc<K>(r.y, mn, mx, nan); }
    if (gtid == 0) {
        if (head) mm_acc<K>(x[0], mn, mx, nan);
        if ((m - head) & 1) mm_acc<K>(x[m - 1], mn, mx, nan);
    }
    for (int o = 16; o > 0; o >>= 1) {
        u64 a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn; mx = b > mx ? b : mx;
    }
    __shared__ u64 smn[MM_THREADS / 32], smx[MM_THREADS / 32];
    __shared__ int snan;
    if (threadIdx.x == 0) snan = 0;
    __syncthreads();
    if (nan) snan = 1;
    if ((threadIdx.x & 31) == 0) { smn[threadIdx.x >> 5] = mn; smx[threadIdx.x >> 5] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < MM_THREADS / 32; ++w) { mn = smn[w] < mn ? smn[w] : mn; mx = smx[w] > mx ? smx[w] : mx; }
        atomicMin(&g.kmin, mn);
        atomicMax(&g.kmax, mx);
        if (snan) atomicOr(c->nan_flag, 1u);
    }
}

// cnt[bin] += 1, one atomic per distinct bin of the warp: skewed samples (c3's
// repeated value, c4's first bin) would otherwise serialise on one address.
__device__ __forceinline__ void warp_agg_add(u32 *cnt, u32 bin) {
    const u32 act = __activemask();
    const u32 peers = __match_any_sync(act, bin);
    if ((threadIdx.x & 31) == (u32)(__ffs(peers) - 1)) atomicAdd(&cnt[bin], (u32)__popc(peers));
}

__device__ __forceinline__ void push_item(const DevCtx *c, u64 off, u32 m, u32 level, u32 src, u32 kind) {
    u32 slot = atomicAdd(c->nitems, 1u);
    if (slot < c->items_cap) {
        SegItem it; it.off = off; it.m = m; it.level = level; it.src = src; it.kind = kind;
        c->items[slot] = it;
    } else {
        atomicOr(c->err_flag, 1u);
    }
}

// --- exclusive scan of a u32 array (3 phases)
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_CHUNK = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ u32 block_excl_scan_1024(u32 v, u32 *wsum, u32 &total) {
    const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u32 x = v;
    for (int o = 1; o < 32; o <<= 1) { u32 y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= (u32)o) x += y; }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        u32 s = wsum[lane];
        u32 t = s;
        for (int o = 1; o < 32; o <<= 1) { u32 y = __shfl_up_sync(0xffffffffu, t, o); if (lane >= (u32)o) t += y; }
        wsum[lane] = t - s;
        if (lane == 31) wsum[32] = t;
    }
    __syncthreads();
    u32 r = wsum[w] + x - v;
    total = wsum[32];
    __syncthreads();
    return r;
}

__host__ __device__ inline u32 ceil_log2_u32(u32 v) {   // v >= 1
    u32 r = 0;
    while ((1ull << r) < v) ++r;
    return r;
}
__host__ __device__ inline u32 floor_log2_u64(u64 v) {  // v >= 1
    u32 r = 0;
    while (v >> (r + 1)) ++r;
    return r;
}
// Digit shift for splitting W >= 2 consecutive buckets holding c keys:
// G = ceil(W / 2^s) <= GMAX, expected group ~ S_CAP/2 keys, G >= 2.
constexpr u32 NB_SHIFT_MAX = 9;
static_assert((1u << NB_SHIFT_MAX) <= (u32)NB_CAP, "NB_SHIFT_MAX");
__host__ __device__ inline u32 choose_shift(u32 W, u32 c) {
    u32 cl = ceil_log2_u32(W);
    u32 smin = cl > GMAX_LOG2 ? cl - GMAX_LOG2 : 0;
    u64 q = ((u64)(S_CAP / 2) * W) / (c ? c : 1);
    u32 st = floor_log2_u64(q ? q : 1);
    u32 s = st < NB_SHIFT_MAX ? st : NB_SHIFT_MAX;   // a digit group of 2^s buckets fits a K7 task (NB_CAP)
    if (s < smin) s = smin;
    if (s > cl - 1) s = cl - 1;
    return s;
}

template <class K>
__global__ void k_node_model(const DevCtx *__restrict__ c, u32 node) {
    pdl_entry();
    if (*c->nan_flag) return;
    GNode &g = c->nodes[node];
    Model md;
    bool ok = make_model<K>(g.kmin, g.kmax, g.beta, md);
    g.md = md;
    g.degenerate = ok ? 0u : 1u;
    if (!ok) push_item(c, g.off, g.m, g.level, g.src, 1u);   // Standard-Sort the whole segment
}

// The node's model (from the min/max) is built by every thread (cheap, one
// launch less); thread 0 of block 0 publishes it (and the degenerate verdict,
// R9/R10) for the later kernels.
template <class K>
__global__ void k_fit_sample(const DevCtx *__restrict__ c, u32 node) {
    pdl_entry();
    if (*c->nan_flag) return;
    GNode &g = c->nodes[node];
    Model md;
    const bool ok = make_model<K>(g.kmin, g.kmax, g.beta, md);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        g.md = md;
        g.degenerate = ok ? 0u : 1u;
        if (!ok) push_item(c, g.off, g.m, g.level, g.src, 1u);   // Standard-Sort the whole segment
    }
    if (!ok) return;
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= g.alpha) return;
    const bool sample_all = (c->flags & FLAG_SAMPLE_ALL) != 0;
    const u64 pos = sample_all ? (u64)k : sample_pos(node_key(c->seed, g.level, c->gbase + g.off), k, g.m);
    const u64 raw = c->buf[g.src][g.off + pos];
    warp_agg_add(&g.cnt[0], interval_index<K>(K::to_okey(raw), md));
}

// ------------------------------------------------------------------ batched global nodes
// The recursing buckets too large for a K7 CTA that one batch produces (up to
// thousands for skewed inputs at 10^8-10^9 keys) become global nodes on the
// device (k_items_to_nodes) and are fitted together: one min/max launch, one
// sampling launch and one fit launch for all of them.  Both chunked kernels are
// grid-stride over the batch's chunks; a chunk finds its node by a binary search
// over the batch's chunk prefix sums (bpre_mm / bpre_fs, built by k_items_to_nodes).
constexpr int MMB_CHUNK = 16384;   // keys per min/max chunk
constexpr int FSB_CHUNK = 256;     // samples per sampling chunk

__device__ __forceinline__ u32 batch_node_of(const u32 *__restrict__ pre, u32 nb, u32 chunk) {
    u32 lo = 0, hi = nb - 1;   // last k with pre[k] <= chunk
    while (lo < hi) {
        const u32 mid = (lo + hi + 1) >> 1;
        if (pre[mid] <= chunk) lo = mid; else hi = mid - 1;
    }
    return lo;
}

template <class K>
__global__ void __launch_bounds__(MM_THREADS) k_minmax_batch(const DevCtx *__restrict__ c) {
    pdl_entry();
    if (*c->nan_flag) return;
    const BatchInfo bi = c->cnt->batch;
    if (bi.nb == 0) return;
    {   // zero the batch's tables (per-bin counts, T, H) before the sampling kernel adds to them
        u32 *a = c->arena;
        for (u64 i = bi.a0 + (u64)blockIdx.x * MM_THREADS + threadIdx.x; i < bi.a1; i += (u64)gridDim.x * MM_THREADS) a[i] = 0u;
    }
    __shared__ u64 smn[MM_THREADS / 32], smx[MM_THREADS / 32];
    for (u32 ch = blockIdx.x; ch < bi.mm_chunks; ch += gridDim.x) {
        const u32 k = batch_node_of(c->bpre_mm, bi.nb, ch);
        GNode &g = c->nodes[bi.first + k];
        const u64 s0 = (u64)(ch - c->bpre_mm[k]) * MMB_CHUNK, s1 = min((u64)g.m, s0 + MMB_CHUNK);
        const u64 *x = c->buf[g.src] + g.off;
        u64 mn = ~0ull, mx = 0;
        bool nan = false;
        constexpr int U = MMB_CHUNK / MM_THREADS;   // 64 keys per thread, 8 loads in flight
#pragma unroll 8
        for (int q = 0; q < U; ++q) {
            const u64 i = s0 + threadIdx.x + (u64)q * MM_THREADS;
            if (i < s1) mm_acc<K>(x[i], mn, mx, nan);
        }
        for (int o = 16; o > 0; o >>= 1) {
            u64 a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
            mn = a < mn ? a : mn; mx = b > mx ? b : mx;
        }
        if ((threadIdx.x & 31) == 0) { smn[threadIdx.x >> 5] = mn; smx[threadIdx.x >> 5] = mx; }
        if (__syncthreads_or(nan) && threadIdx.x == 0) atomicOr(c->nan_flag, 1u);
        if (threadIdx.x == 0) {
            for (int w = 1; w < MM_THREADS / 32; ++w) { mn = smn[w] < mn ? smn[w] : mn; mx = smx[w] > mx ? smx[w] : mx; }
            atomicMin(&g.kmin, mn);
            atomicMax(&g.kmax, mx);
        }
        __syncthreads();
    }
}

// alpha samples of every node -> per-bin counts; the first chunk of a node
// publishes its model (and the R9/R10 verdict) like k_fit_sample.
template <class K>
__global__ void __launch_bounds__(FSB_CHUNK) k_fit_sample_batch(const DevCtx *__restrict__ c) {
    pdl_entry();
    if (*c->nan_flag) return;
    const BatchInfo bi = c->cnt->batch;
    if (bi.nb == 0) return;
    const bool sample_all = (c->flags & FLAG_SAMPLE_ALL) != 0;
    for (u32 ch = blockIdx.x; ch < bi.fs_chunks; ch += gridDim.x) {
        const u32 kb = batch_node_of(c->bpre_fs, bi.nb, ch);
        GNode &g = c->nodes[bi.first + kb];
        Model md;
        const bool ok = make_model<K>(g.kmin, g.kmax, g.beta, md);
        const u32 cb = ch - c->bpre_fs[kb];
        if (cb == 0 && threadIdx.x == 0) {
            g.md = md;
            g.degenerate = ok ? 0u : 1u;
            if (!ok) push_item(c, g.off, g.m, g.level, g.src, 1u);   // Standard-Sort the whole segment
        }
        if (!ok) continue;
        const u32 k = cb * FSB_CHUNK + threadIdx.x;
        if (k >= g.alpha) continue;
        const u64 pos = sample_all ? (u64)k : sample_pos(node_key(c->seed, g.level, c->gbase + g.off), k, g.m);
        warp_agg_add(&g.cnt[0], interval_index<K>(K::to_okey(c->buf[g.src][g.off + pos]), md));
    }
}

constexpr u32 RADIX_BITS = 10;   // digit bits of a Standard-Sort (MSD radix) split: G <= 1024 = GMAX
static_assert((1u << RADIX_BITS) <= (u32)GMAX, "radix digits");

// The first MSD radix split of a Standard-Sort bucket of m > S_CAP keys:
// the top RADIX_BITS bits of the ordered keys.
__device__ __forceinline__ SplitTask radix_split(u64 off, u32 m, u32 src, u32 shift) {
    SplitTask s;
    s.off = off; s.m = m; s.node = 0xffffffffu; s.jlo = 0; s.jhi = 0;
    s.shift = shift; s.G = 1u << (64u - shift < RADIX_BITS ? 64u - shift : RADIX_BITS);
    s.src = src; s.dst = src == 1 ? 2 : 1;
    s.tile_begin = 0; s.ntiles = 0; s.cbase = 0; s.mbase = 0;
    return s;
}
__device__ __forceinline__ u32 radix_next_shift(u32 shift) { return shift >= RADIX_BITS ? shift - RADIX_BITS : 0u; }

// Oversized recursing buckets (items of kind 0) -> new global nodes of the next
// batch, with their tables carved from the arena and their first split appended
// to the next round's list; Standard-Sort items (kind 1) -> an MSD radix split (same list).
// One CTA; consumes every item and resets the item count.  This replaces the
// host round trip of the previous design (recursion per bucket).
template <class K>
__global__ void __launch_bounds__(1024) k_items_to_nodes(const DevCtx *__restrict__ c, cudaGraphConditionalHandle h,
                                                        u32 count_iter) {
    pdl_entry();
    __shared__ u32 wsum[33];
    __shared__ unsigned long long wsum64[33];
    Counters &C = *c->cnt;
    const u32 nit = min(C.nitems, c->items_cap);
    const u32 t = threadIdx.x, lane = t & 31, w = t >> 5;
    const bool sample_all = (c->flags & FLAG_SAMPLE_ALL) != 0;
    const u32 first = C.node_count;
    const u64 a0 = C.arena_used;
    const u32 cur = C.round & 1u;   // the list the next round consumes
    u32 nb = 0, nfb = 0, cmm = 0, cfs = 0;
    u64 arena = a0;
    for (u32 base = 0; base < nit; base += 1024) {
        const u32 i = base + t;
        SegItem it;
        it.kind = 2;
        if (i < nit) it = c->items[i];
        const bool isn = !C.nan_flag && it.kind == 0, isf = !C.nan_flag && it.kind == 1;
        u32 P = 0, al = 0, need = 0, nmm = 0, nfs = 0;
        if (isn) {
            P = (u32)iroot34(it.m);
            al = sample_all ? it.m : P;
            need = 3u * (P + 2u);
            nmm = (it.m + MMB_CHUNK - 1) / MMB_CHUNK;
            nfs = (al + FSB_CHUNK - 1) / FSB_CHUNK;
        }
        u32 tot;
        const u32 ex_n = block_excl_scan_1024(isn ? 1u : 0u, wsum, tot);
        const u32 tot_n = tot;
        const u32 ex_f = block_excl_scan_1024(isf ? 1u : 0u, wsum, tot);
        const u32 tot_f = tot;
        const u32 ex_mm = block_excl_scan_1024(nmm, wsum, tot);
        const u32 tot_mm = tot;
        const u32 ex_fs = block_excl_scan_1024(nfs, wsum, tot);
        const u32 tot_fs = tot;
        // u64 exclusive scan of the table sizes
        u64 x = need;
        for (int o = 1; o < 32; o <<= 1) { u64 y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= (u32)o) x += y; }
        if (lane == 31) wsum64[w] = x;
        __syncthreads();
        if (w == 0) {
            u64 sv = wsum64[lane], t2 = sv;
            for (int o = 1; o < 32; o <<= 1) { u64 y = __shfl_up_sync(0xffffffffu, t2, o); if (lane >= (u32)o) t2 += y; }
            wsum64[lane] = t2 - sv;
            if (lane == 31) wsum64[32] = t2;
        }
        __syncthreads();
        const u64 ex_a = wsum64[w] + x - need, tot_a = wsum64[32];
        __syncthreads();
        if (isn) {
            const u32 k = nb + ex_n, idx = first + k;
            const u64 ao = arena + ex_a;
            if (idx < c->node_cap && ao + need <= c->arena_cap) {
                GNode g;
                memset(&g, 0, sizeof g);
                g.off = it.off; g.m = it.m; g.level = it.level;
                g.kmin = ~0ull; g.kmax = 0;
                g.alpha = al; g.beta = P; g.gamma = P; g.delta = P;
                g.src = it.src;
                g.cnt = c->arena + ao;
                g.T = g.cnt + (P + 2);
                g.H = g.T + (P + 2);
                g.bnd = nullptr;
                c->nodes[idx] = g;
                c->bpre_mm[k] = cmm + ex_mm;
                c->bpre_fs[k] = cfs + ex_fs;
                SplitTask s;
                s.off = it.off; s.m = it.m; s.node = idx; s.jlo = 1; s.jhi = P + 2;
                s.shift = choose_shift(P + 1, it.m);
                s.G = (P + 1 + (1u << s.shift) - 1) >> s.shift;
                s.src = it.src; s.dst = it.src == 1 ? 2 : 1;
                s.tile_begin = 0; s.ntiles = 0; s.cbase = 0; s.mbase = 0;
                const u32 slot = atomicAdd(&C.nsplits[cur], 1u);
                if (slot < c->splits_cap) c->splits[cur][slot] = s;
                else atomicOr(c->err_flag, 1u);
            } else {
                atomicOr(c->err_flag, 8u);   // node table / arena capacity
            }
            atomicAdd(&C.global_keys, (unsigned long long)it.m);
        }
        if (isf) {   // Standard-Sort of a bucket of > S_CAP keys: MSD radix splits
            const SplitTask sp = radix_split(it.off, it.m, it.src, 64u - RADIX_BITS);
            const u32 slot = atomicAdd(&C.nsplits[cur], 1u);
            if (slot < c->splits_cap) c->splits[cur][slot] = sp;
            else atomicOr(c->err_flag, 1u);
            atomicAdd(&C.fb_keys, (unsigned long long)it.m);
        }
        nb += tot_n; nfb += tot_f; cmm += tot_mm; cfs += tot_fs; arena += tot_a;
    }
    __syncthreads();
    if (t == 0) {
        const u32 nbc = first + nb <= c->node_cap ? nb : (c->node_cap > first ? c->node_cap - first : 0u);
        BatchInfo bi;
        bi.first = first; bi.nb = nbc; bi.mm_chunks = nbc == nb ? cmm : 0u; bi.fs_chunks = nbc == nb ? cfs : 0u;
        bi.a0 = a0; bi.a1 = arena <= c->arena_cap ? arena : a0;
        if (nbc != nb) bi.nb = 0;
        C.batch = bi;
        C.node_count = first + bi.nb;
        C.arena_used = bi.a1;
        (void)nfb;
        C.nitems = 0;
        // condition of the batch loop (a CUDA-graph WHILE node): another batch runs iff
        // this one made new global nodes or left unfinished splits (and no error)
        if (count_iter) C.iters += 1;
        if (C.iters > 64u) atomicOr(c->err_flag, 16u);   // bound: depth <= 6 levels, a few rounds each
        const bool more = !C.nan_flag && !C.err_flag && (bi.nb > 0 || C.nsplits[cur] > 0);
        cudaGraphSetConditional(h, more && C.iters <= 64u ? 1u : 0u);
    }
}

// b = prefix of the counts and T of one node per CTA (the batched nodes have
// up to a few thousand bins: the CTA walks them SCAN_CHUNK at a time); grid-stride
// over the batch's nodes.
__global__ void __launch_bounds__(SCAN_THREADS) k_fit_batch(const DevCtx *__restrict__ c) {
    pdl_entry();
    __shared__ u32 wsum[33];
    __shared__ unsigned long long dsum;
    if (*c->nan_flag) return;
    const BatchInfo bi = c->cnt->batch;
    const bool logging = c->rec != nullptr;
    for (u32 k = blockIdx.x; k < bi.nb; k += gridDim.x) {
        GNode &g = c->nodes[bi.first + k];
        if (g.degenerate) continue;   // uniform per CTA
        const u64 nb = (u64)g.beta + 1;
        u32 *in = g.cnt + 1;
        if (threadIdx.x == 0) dsum = 0;
        u32 carry = 0;
        u64 db = 0;
        for (u64 base0 = 0; base0 < nb; base0 += SCAN_CHUNK) {
            const u64 base = base0 + (u64)threadIdx.x * SCAN_ITEMS;
            u32 v[SCAN_ITEMS], sm = 0;
#pragma unroll
            for (int q = 0; q < SCAN_ITEMS; ++q) { v[q] = base + q < nb ? in[base + q] : 0; sm += v[q]; }
            u32 total;
            u32 e = block_excl_scan_1024(sm, wsum, total) + carry;
#pragma unroll
            for (int q = 0; q < SCAN_ITEMS; ++q) {
                e += v[q];
                if (base + q < nb) {
                    const u64 i = base + q + 1;
                    in[base + q] = e;
                    g.T[i] = bucket_of(e, g.alpha, g.gamma);
                    if (logging) db += digest_term(i, e);
                }
            }
            carry += total;
        }
        if (logging) {
            for (int o = 16; o > 0; o >>= 1) db += __shfl_xor_sync(0xffffffffu, db, o);
            if ((threadIdx.x & 31) == 0) atomicAdd(&dsum, (unsigned long long)db);
            __syncthreads();
            if (threadIdx.x == 0) atomicAdd((unsigned long long *)&g.digest_b, dsum);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ splits
__device__ __forceinline__ u32 find_split(const SplitTask *L, u32 ns, u32 tile) {
    u32 lo = 0, hi = ns - 1;
    while (lo < hi) {
        u32 mid = (lo + hi + 1) >> 1;
        if (L[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Split of every tile of round `cur` (one thread per tile): the count and
// scatter CTAs read it instead of each searching the split list.
__global__ void k_tile_map(const DevCtx *__restrict__ c) {
    pdl_entry();
    const RoundPlan pl = *c->plan;
    const SplitTask *__restrict__ L = c->splits[pl.cur];
    for (u32 si = blockIdx.x; si < pl.ns; si += gridDim.x) {   // one CTA per split
        const u32 tb = L[si].tile_begin, nt = L[si].ntiles;
        for (u32 t = threadIdx.x; t < nt; t += blockDim.x) c->tmap[tb + t] = si;
    }
}

// A Standard-Sort split (jhi == 0; model splits have jhi >= 2): an MSD radix pass on
// ordered-key bits [shift, shift + log2 G) of a bucket that Alg. 1 sends to Standard-Sort
// (PAPER.md:162-163); jlo bit 0 is set by the count pass if the split holds two distinct keys.
__host__ __device__ __forceinline__ bool is_radix(const SplitTask &st) { return st.jhi == 0; }

template <class K>
__device__ __forceinline__ u32 digit_of(u64 okey, const Model &md, const u32 *__restrict__ T, u32 jlo, u32 shift) {
    u32 j = __ldg(&T[interval_index<K>(okey, md)]);
    return (j - jlo) >> shift;
}

// Counts of the digit (T[i(x)] - jlo) >> shift per tile of SPLIT_TILE keys,
// written to the digit-major count matrix; every key's digit is cached (u16)
// for the scatter.  Persistent CTAs (grid-stride over the round's tiles); the
// keys of the next tile stream into a second shared buffer by one bulk copy
// (TMA, mbarrier completion) while the current tile is classified, so the pass
// keeps HBM busy instead of waiting on each tile's loads.
struct CountStage {
    SplitTask st;
    const u32 *T;
    const u32 *bnd;                // digit boundaries (first split of a large node) or NULL
    Model md;
    u32 tile, head, direct, deg;   // head: index of the tile's first key in `in`; direct: no bulk copy
    u32 node, beta;
};
// Digit lookup without gathers from T (the first split of a large node, where
// T is large and the keys are random): bins are grouped in NCELL cells of
// 2^cs bins; ct[c] = digit of the cell's first bin, and the digit of bin i is
// ct[c] plus the boundaries bnd[] inside its cell at or below i.
constexpr int NCELL = 8192;
struct CountSmem {
    u64 in[2][SPLIT_TILE + 2];
    u32 hist[GMAX];
    u32 bnd[GMAX];
    u16 ct[NCELL + 1];
    u32 tab_node, tab_cs, tab_step;
    CountStage meta[2];
    u64 full[2], empty[2];
};

// Producer (one thread): metadata of `tile` and the bulk copy of its keys into stage `sg`.
__device__ __forceinline__ void count_issue(const DevCtx *__restrict__ c, CountSmem &S, u32 cur, u32 tile, u32 sg) {   // cur: plan.cur
    CountStage &m = S.meta[sg];
    const SplitTask &st = c->splits[cur][c->tmap[tile]];
    m.st = st;
    const GNode &g = c->nodes[st.node];
    m.T = g.T;
    m.md = g.md;
    m.deg = g.degenerate;
    m.tile = tile;
    m.node = st.node;
    m.beta = g.beta;
    m.bnd = (g.bnd && st.jlo == 1u && st.shift == g.bshift && st.G == g.bG) ? g.bnd : nullptr;
    const u32 lt = tile - st.tile_begin;
    const u32 k0 = lt * SPLIT_TILE, nt = min(st.m, k0 + SPLIT_TILE) - k0;
    const u64 *base = c->buf[st.src];
    const uintptr_t a = (uintptr_t)(base + st.off + k0);
    const uintptr_t a0 = a & ~(uintptr_t)15, a1 = (a + 8ull * nt + 15) & ~(uintptr_t)15;
    m.head = (u32)((a - a0) >> 3);
    m.direct = 0;
    if (m.deg) {
        mbar_arrive_tx(&S.full[sg], 0);
    } else if (a0 < (uintptr_t)base || a1 > (uintptr_t)(base + c->n)) {   // edge of the buffer: plain loads
        m.direct = 1;
        mbar_arrive_tx(&S.full[sg], 0);
    } else {
        fence_proxy_async();
        mbar_arrive_tx(&S.full[sg], (u32)(a1 - a0));
        bulk_g2s(S.in[sg], (const void *)a0, (u32)(a1 - a0), &S.full[sg]);
    }
}

constexpr int CNT_THREADS = SC_THREADS + 32;   // 12 consumer warps + 1 producer warp

template <class K>
__global__ void __launch_bounds__(CNT_THREADS, 2) k_split_count(const DevCtx *__restrict__ c) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char cnt_smem_raw[];
    CountSmem &S = *reinterpret_cast<CountSmem *>(cnt_smem_raw);
    if (*c->nan_flag) return;
    const u32 ntiles = c->plan->tiles;
    const u32 cur = c->plan->cur;
    const u32 w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&S.full[0], 1); mbar_init(&S.full[1], 1);
        mbar_init(&S.empty[0], 1); mbar_init(&S.empty[1], 1);
        mbar_init_fence();
        S.tab_node = 0xffffffffu;
    }
    __syncthreads();
    if (w == SC_WARPS) {   // producer warp: metadata + bulk copy of each tile, two stages ahead of use
        if (lane == 0) {
            for (u32 it = 0;; ++it) {
                const u32 tile = blockIdx.x + it * gridDim.x;
                if (tile >= ntiles) break;
                const u32 sg = it & 1u;
                if (it >= 2) mbar_wait(&S.empty[sg], ((it - 2) >> 1) & 1u);
                count_issue(c, S, cur, tile, sg);
            }
        }
        return;
    }
    u32 *__restrict__ C = c->cmat;
    for (u32 it = 0;; ++it) {
        const u32 tile = blockIdx.x + it * gridDim.x;
        if (tile >= ntiles) break;
        const u32 sg = it & 1u;
        mbar_wait(&S.full[sg], (it >> 1) & 1u);
        const CountStage &m = S.meta[sg];
        const SplitTask &st = m.st;
        const u32 G = st.G;
        for (u32 d = threadIdx.x; d < G; d += SC_THREADS) S.hist[d] = 0;
        const u32 lt = tile - st.tile_begin;
        const u32 k0 = lt * SPLIT_TILE, nt = min(st.m, k0 + SPLIT_TILE) - k0;
        const bool tab = m.bnd != nullptr && !m.deg;
        if (tab && S.tab_node != m.node) {   // (re)build the cell table of this node's first split
            named_bar(1, SC_THREADS);
            for (u32 d = threadIdx.x; d < G; d += SC_THREADS) S.bnd[d] = d ? m.bnd[d] : 0u;
            u32 cs = 0;
            while ((m.beta >> cs) >= (u32)NCELL) ++cs;
            named_bar(1, SC_THREADS);
            for (u32 cc = threadIdx.x; cc <= (u32)NCELL; cc += SC_THREADS) {
                const u64 i0 = ((u64)cc << cs) + 1;   // first bin of the cell
                u32 lo = 0, hi = G - 1;               // largest d in [0, G) with bnd[d] <= i0 (bnd[0] := 0)
                while (lo < hi) { const u32 mid = (lo + hi + 1) >> 1; if ((u64)S.bnd[mid] <= i0) lo = mid; else hi = mid - 1; }
                S.ct[cc] = (u16)lo;
            }
            named_bar(1, SC_THREADS);
            u32 mx = 0;   // widest cell (digits it spans) -> largest search step
            for (u32 cc = threadIdx.x; cc < (u32)NCELL; cc += SC_THREADS) mx = max(mx, (u32)S.ct[cc + 1] - (u32)S.ct[cc]);
            mx = __reduce_max_sync(0xffffffffu, mx);
            if (threadIdx.x == 0) { S.tab_node = m.node; S.tab_cs = cs; S.tab_step = 0; }
            named_bar(1, SC_THREADS);
            if ((threadIdx.x & 31) == 0) atomicMax(&S.tab_step, mx ? 1u << (31 - __clz(mx)) : 0u);
        }
        named_bar(1, SC_THREADS);
        if (m.deg) {
            if (threadIdx.x == 0) S.hist[0] = nt;
        } else {
            const Model md = m.md;
            const u32 *T = m.T;
            const u32 jlo = st.jlo, shift = st.shift;
            const u64 *in = S.in[sg] + m.head;
            const u64 *gx = c->buf[st.src] + st.off + k0;
            const bool direct = m.direct != 0;
            u16 *dg = c->digs + st.off + k0;
            const u32 r0 = w * SC_PER_WARP + lane;
            u64 raw[SC_KPL];
            u32 ix[SC_KPL];
#pragma unroll
            for (u32 q = 0; q < SC_KPL; ++q) {
                const u32 k = r0 + q * 32;
                const u32 kk = k < nt ? k : 0u;
                raw[q] = direct ? gx[kk] : in[kk];
            }
            u32 bad = 0;
#pragma unroll
            for (u32 q = 0; q < SC_KPL; ++q) {
                bool ok;
                ix[q] = interval_index_fast_raw<K>(raw[q], md, ok);
                bad |= ok ? 0u : (1u << q);
            }
            if (bad) {   // rare: keys in the fast path's guard band
#pragma unroll
                for (u32 q = 0; q < SC_KPL; ++q)
                    if (bad & (1u << q)) ix[q] = interval_index_exact(key_offset_raw<K>(raw[q], md), md.r, md.betad);
            }
            if (tab) {
                const u32 cs = S.tab_cs;
#pragma unroll
                for (u32 q = 0; q < SC_KPL; ++q) {
                    const u32 i = ix[q], cc = (i - 1u) >> cs;
                    u32 d = S.ct[cc];   // largest d in [ct[cc], ct[cc + 1]] with bnd[d] <= i:
                    const u32 d1 = S.ct[cc + 1];   // power-of-two steps, the same count for every key
                    for (u32 step = S.tab_step; step; step >>= 1) {
                        const u32 nd = d + step;
                        if (nd <= d1 && S.bnd[nd] <= i) d = nd;
                    }
                    ix[q] = d;
                }
            } else {
#pragma unroll
                for (u32 q = 0; q < SC_KPL; ++q) ix[q] = (__ldg(&T[ix[q]]) - jlo) >> shift;
            }
#pragma unroll
            for (u32 q = 0; q < SC_KPL; ++q) {
                const u32 k = r0 + q * 32;
                if (k < nt) {
                    const u32 d = ix[q];
                    dg[k] = (u16)d;
                    PCF_CHECK(c, d < G);
                    atomicAdd(&S.hist[d], 1u);
                }
            }
        }
        named_bar(1, SC_THREADS);
        for (u32 d = threadIdx.x; d < G; d += SC_THREADS) C[st.cbase + (u64)d * st.ntiles + lt] = S.hist[d];
        named_bar(1, SC_THREADS);
        if (threadIdx.x == 0) mbar_arrive(&S.empty[sg]);   // stage sg (keys, metadata) is free
    }
}

// One CTA per tile (no pipeline): for rounds of few tiles per SM (n <= 2^25), where
// the persistent kernel's pipeline never fills.  Same outputs as k_split_count.
template <class K>
__global__ void __launch_bounds__(SC_THREADS, 2) k_split_count_tile(const DevCtx *__restrict__ c) {
    pdl_entry();
    __shared__ u32 hist[GMAX];
    if (*c->nan_flag) return;
    const RoundPlan pl = *c->plan;
    const SplitTask *__restrict__ L = c->splits[pl.cur];
    u32 *__restrict__ C = c->cmat;
    // one tile per CTA when the grid covers the round (host-launched first rounds);
    // grid-stride in the device-driven batches, whose grid cannot know the round's size
    for (u32 tile = blockIdx.x; tile < pl.tiles; tile += gridDim.x) {
    const u32 s = c->tmap[tile];
    const SplitTask st = L[s];
    if (is_radix(st)) continue;   // k_split_count_radix (uniform per CTA)
    const u32 lt = tile - st.tile_begin;
    if (tile != blockIdx.x) __syncthreads();   // the previous tile's histogram is written out
    for (u32 d = threadIdx.x; d < st.G; d += SC_THREADS) hist[d] = 0;
    const u32 k0 = lt * SPLIT_TILE, k1 = min(st.m, k0 + SPLIT_TILE);
    const bool deg = c->nodes[st.node].degenerate != 0;
    __syncthreads();
    if (deg) {
        if (threadIdx.x == 0) hist[0] = k1 - k0;
    } else {
        const GNode &g = c->nodes[st.node];
        const Model md = g.md;
        const u64 *x = c->buf[st.src] + st.off;
        const u32 *T = g.T;
        u16 *dg = c->digs + st.off;
        const u32 w = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const u32 r0 = k0 + w * SC_PER_WARP + lane;
        u64 raw[SC_KPL];
        u32 ix[SC_KPL];
#pragma unroll
        for (u32 q = 0; q < SC_KPL; ++q) { const u32 k = r0 + q * 32; raw[q] = k < k1 ? x[k] : x[k0]; }
        u32 bad = 0;
#pragma unroll
        for (u32 q = 0; q < SC_KPL; ++q) {
            bool ok;
            ix[q] = interval_index_fast_raw<K>(raw[q], md, ok);
            bad |= ok ? 0u : (1u << q);
        }
        if (bad) {   // rare: keys in the fast path's guard band
#pragma unroll
            for (u32 q = 0; q < SC_KPL; ++q)
                if (bad & (1u << q)) ix[q] = interval_index_exact(key_offset_raw<K>(raw[q], md), md.r, md.betad);
        }
#pragma unroll
        for (u32 q = 0; q < SC_KPL; ++q) ix[q] = __ldg(&T[ix[q]]);
#pragma unroll
        for (u32 q = 0; q < SC_KPL; ++q) {
            const u32 k = r0 + q * 32;
            if (k < k1) {
                const u32 d = (ix[q] - st.jlo) >> st.shift;
                PCF_CHECK(c, ix[q] >= st.jlo && ix[q] < st.jhi && d < st.G);
                dg[k] = (u16)d;
                atomicAdd(&hist[d], 1u);
            }
        }
    }
    __syncthreads();
    for (u32 d = threadIdx.x; d < st.G; d += SC_THREADS) C[st.cbase + (u64)d * st.ntiles + lt] = hist[d];
    }
}

// The count pass of the Standard-Sort (MSD radix) splits of a round: digit = ordered-key bits
// [shift, shift + log2 G); also sets jlo bit 0 of a split that holds two distinct keys.
// Grid-stride over the round's tiles; tiles of model splits are k_split_count_tile's.
template <class K>
__global__ void __launch_bounds__(SC_THREADS, 2) k_split_count_radix(const DevCtx *__restrict__ c) {
    pdl_entry();
    __shared__ u32 hist[GMAX];
    if (*c->nan_flag) return;
    const RoundPlan pl = *c->plan;
    SplitTask *L = c->splits[pl.cur];
    u32 *__restrict__ C = c->cmat;
    bool first_tile = true;
    for (u32 tile = blockIdx.x; tile < pl.tiles; tile += gridDim.x) {
        const u32 s = c->tmap[tile];
        const SplitTask st = L[s];
        if (!is_radix(st)) continue;
        const u32 lt = tile - st.tile_begin;
        if (!first_tile) __syncthreads();   // the previous tile's histogram is written out
        first_tile = false;
        for (u32 d = threadIdx.x; d < st.G; d += SC_THREADS) hist[d] = 0;
        const u32 k0 = lt * SPLIT_TILE, k1 = min(st.m, k0 + SPLIT_TILE);
        __syncthreads();
        const u64 *x = c->buf[st.src] + st.off;
        u16 *dg = c->digs + st.off;
        const u64 first = K::to_okey(x[0]);
        const u32 w = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const u32 r0 = k0 + w * SC_PER_WARP + lane;
        u64 ok[SC_KPL];
#pragma unroll
        for (u32 q = 0; q < SC_KPL; ++q) { const u32 k = r0 + q * 32; ok[q] = K::to_okey(k < k1 ? x[k] : x[k0]); }
        bool diff = false;
#pragma unroll
        for (u32 q = 0; q < SC_KPL; ++q) {
            const u32 k = r0 + q * 32;
            if (k < k1) {
                const u32 d = (u32)(ok[q] >> st.shift) & (st.G - 1u);
                diff |= ok[q] != first;
                dg[k] = (u16)d;
                atomicAdd(&hist[d], 1u);
            }
        }
        if (__any_sync(0xffffffffu, diff) && lane == 0) atomicOr(&L[s].jlo, 1u);   // two distinct keys
        __syncthreads();
        for (u32 d = threadIdx.x; d < st.G; d += SC_THREADS) C[st.cbase + (u64)d * st.ntiles + lt] = hist[d];
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_partials(const u32 *__restrict__ in, u64 n, u32 *__restrict__ bsum) {
    pdl_entry();
    __shared__ u32 wsum[33];
    u64 base = (u64)blockIdx.x * SCAN_CHUNK + (u64)threadIdx.x * SCAN_ITEMS;
    u32 s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) if (base + k < n) s += in[base + k];
    u32 total;
    block_excl_scan_1024(s, wsum, total);
    if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_bsums(u32 *__restrict__ bsum, u32 nb) {
    pdl_entry();
    __shared__ u32 wsum[33];
    u32 carry = 0;
    for (u32 base = 0; base < nb; base += SCAN_THREADS) {
        u32 i = base + threadIdx.x;
        u32 v = i < nb ? bsum[i] : 0;
        u32 total;
        u32 e = block_excl_scan_1024(v, wsum, total);
        if (i < nb) bsum[i] = carry + e;
        carry += total;
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_final(const u32 *__restrict__ in, u64 n, const u32 *__restrict__ bsum,
                                                             u32 *__restrict__ out) {
    pdl_entry();
    __shared__ u32 wsum[33];
    u64 base = (u64)blockIdx.x * SCAN_CHUNK + (u64)threadIdx.x * SCAN_ITEMS;
    u32 v[SCAN_ITEMS];
    u32 s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) { v[k] = base + k < n ? in[base + k] : 0; s += v[k]; }
    u32 total;
    u32 e = block_excl_scan_1024(s, wsum, total) + bsum[blockIdx.x];
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) { if (base + k < n) out[base + k] = e; e += v[k]; }
}

// Same three phases over the count matrix of a split round, sizes from the plan.
__global__ void __launch_bounds__(SCAN_THREADS) k_scanp_partials(const DevCtx *__restrict__ c) {
    pdl_entry();
    __shared__ u32 wsum[33];
    const RoundPlan pl = *c->plan;
    for (u32 b = blockIdx.x; b < pl.nblk; b += gridDim.x) {
        const u64 base = (u64)b * SCAN_CHUNK + (u64)threadIdx.x * SCAN_ITEMS;
        u32 sum = 0;
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) if (base + k < pl.ctot) sum += c->cmat[base + k];
        u32 total;
        block_excl_scan_1024(sum, wsum, total);
        if (threadIdx.x == 0) c->bsum[b] = total;
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scanp_bsums(const DevCtx *__restrict__ c) {
    pdl_entry();
    __shared__ u32 wsum[33];
    const u32 nb = c->plan->nblk;
    u32 carry = 0;
    for (u32 base = 0; base < nb; base += SCAN_THREADS) {
        const u32 i = base + threadIdx.x;
        const u32 v = i < nb ? c->bsum[i] : 0;
        u32 total;
        const u32 e = block_excl_scan_1024(v, wsum, total);
        if (i < nb) c->bsum[i] = carry + e;
        carry += total;
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scanp_final(const DevCtx *__restrict__ c) {
    pdl_entry();
    __shared__ u32 wsum[33];
    const RoundPlan pl = *c->plan;
    for (u32 b = blockIdx.x; b < pl.nblk; b += gridDim.x) {
        const u64 base = (u64)b * SCAN_CHUNK + (u64)threadIdx.x * SCAN_ITEMS;
        u32 v[SCAN_ITEMS];
        u32 sum = 0;
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) { v[k] = base + k < pl.ctot ? c->cmat[base + k] : 0; sum += v[k]; }
        u32 total;
        u32 e = block_excl_scan_1024(sum, wsum, total) + c->bsum[b];
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) { if (base + k < pl.ctot) c->pmat[base + k] = e; e += v[k]; }
    }
}

// The same scan in one kernel (decoupled look-back): CTAs take block tickets in order; a block
// publishes its aggregate (flag 1), sums its predecessors' aggregates back to the nearest
// inclusive prefix (flag 2), publishes its own inclusive prefix and writes its slice of the
// scanned matrix: one read and one write of the matrix instead of two reads and a write, one
// launch instead of three.  A ticket's predecessors are held by CTAs that are already running,
// so the waits always end.  Status words (flag << 32 | value, one 8-byte store) are zeroed and
// the ticket counter reset by k_round_plan.
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_status(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
#ifndef PCF_LB_ITEMS
#define PCF_LB_ITEMS 16   // matrix entries per thread and block of the look-back scan (4 x 16-byte loads)
#endif
constexpr int LB_ITEMS = PCF_LB_ITEMS;
constexpr int LB_CHUNK = SCAN_THREADS * LB_ITEMS;
static_assert(LB_ITEMS % 4 == 0 && LB_CHUNK % SCAN_CHUNK == 0, "look-back blocks are whole scan chunks (status words: one per SCAN_CHUNK)");
__global__ void __launch_bounds__(SCAN_THREADS) k_scanp_lookback(const DevCtx *__restrict__ c) {
    pdl_entry();
    __shared__ u32 wsum[33];
    __shared__ u32 s_b, s_pref;
    const RoundPlan pl = *c->plan;
    const u32 nblk = (u32)((pl.ctot + LB_CHUNK - 1) / LB_CHUNK);   // (<= pl.nblk status words)
    unsigned long long *st = c->scan_status;
    const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (;;) {
        if (threadIdx.x == 0) s_b = atomicAdd(&c->plan->next_scan, 1u);
        __syncthreads();
        const u32 b = s_b;
        if (b >= nblk) break;
        const u64 base = (u64)b * LB_CHUNK + (u64)threadIdx.x * LB_ITEMS;
        const bool full = base + LB_ITEMS <= pl.ctot;
        u32 v[LB_ITEMS];
        u32 sum = 0;
        if (full) {
#pragma unroll
            for (int k = 0; k < LB_ITEMS; k += 4) {
                const uint4 q = *reinterpret_cast<const uint4 *>(c->cmat + base + k);
                v[k] = q.x; v[k + 1] = q.y; v[k + 2] = q.z; v[k + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < LB_ITEMS; ++k) v[k] = base + k < pl.ctot ? c->cmat[base + k] : 0;
        }
#pragma unroll
        for (int k = 0; k < LB_ITEMS; ++k) sum += v[k];
        u32 total;
        u32 e = block_excl_scan_1024(sum, wsum, total);   // (ends with a barrier: s_b may be rewritten after it)
        if (w == 0) {
            u32 acc = 0;
            if (b > 0) {
                if (lane == 0) st_status(&st[b], (1ull << 32) | total);
                for (long long j = (long long)b - 1;; j -= 32) {   // windows of 32 predecessors, nearest first
                    const long long idx = j - lane;
                    unsigned long long x = idx >= 0 ? ld_status(&st[idx]) : (2ull << 32);
                    while (__any_sync(0xffffffffu, (x >> 32) == 0)) {
                        if ((x >> 32) == 0) x = ld_status(&st[idx]);
                    }
                    const u32 pm = __ballot_sync(0xffffffffu, (x >> 32) == 2);
                    const u32 first = pm ? (u32)__ffs(pm) - 1u : 31u;
                    u32 val = lane <= first ? (u32)x : 0u;
                    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                    acc += val;
                    if (pm) break;
                }
            }
            if (lane == 0) { st_status(&st[b], (2ull << 32) | (u32)(acc + total)); s_pref = acc; }
        }
        __syncthreads();
        e += s_pref;
        if (full) {
#pragma unroll
            for (int k = 0; k < LB_ITEMS; k += 4) {
                uint4 q;
                q.x = e; e += v[k]; q.y = e; e += v[k + 1]; q.z = e; e += v[k + 2]; q.w = e; e += v[k + 3];
                *reinterpret_cast<uint4 *>(c->pmat + base + k) = q;
            }
        } else {
#pragma unroll
            for (int k = 0; k < LB_ITEMS; ++k) { if (base + k < pl.ctot) c->pmat[base + k] = e; e += v[k]; }
        }
    }
}

// Plan split round `cur`: tiles, count-matrix offsets and key offsets of every
// split (one CTA).  Splits that do not fit the count matrix are carried over to
// the next round's list; the next list's counter is reset here.
__global__ void __launch_bounds__(1024) k_round_plan(const DevCtx *__restrict__ c) {
    pdl_entry();
    __shared__ u32 wsum[33];
    __shared__ unsigned long long wsum64[33];
    __shared__ u32 cut_s;
    const u32 cur = c->cnt->round & 1u;   // rounds alternate between the two split lists
    SplitTask *L = c->splits[cur];
    const u32 nxt = cur ^ 1u;
    u32 ns = *c->nan_flag ? 0u : min(c->nsplits[cur], c->splits_cap);
    if (threadIdx.x == 0) { c->nsplits[nxt] = 0; cut_s = ns; }
    const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u32 carry_t = 0;
    u64 carry_c = 0, carry_m = 0;
    for (u32 base = 0; base < ns; base += 1024) {
        const u32 s = base + threadIdx.x;
        u32 nt = 0;
        u64 cc = 0, mm = 0;
        if (s < ns) {
            const SplitTask &t = L[s];
            nt = (t.m + SPLIT_TILE - 1) / SPLIT_TILE;
            cc = (u64)nt * t.G;
            mm = t.m;
        }
        u32 tot_t;
        const u32 ex_t = block_excl_scan_1024(nt, wsum, tot_t);
        // u64 exclusive scans of cc and mm (two passes through the same helper)
        u64 vals[2] = {cc, mm}, ex[2], tot[2];
        for (int q = 0; q < 2; ++q) {
            u64 x = vals[q];
            for (int o = 1; o < 32; o <<= 1) { u64 y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= (u32)o) x += y; }
            if (lane == 31) wsum64[w] = x;
            __syncthreads();
            if (w == 0) {
                u64 sv = wsum64[lane], t2 = sv;
                for (int o = 1; o < 32; o <<= 1) { u64 y = __shfl_up_sync(0xffffffffu, t2, o); if (lane >= (u32)o) t2 += y; }
                wsum64[lane] = t2 - sv;
                if (lane == 31) wsum64[32] = t2;
            }
            __syncthreads();
            ex[q] = wsum64[w] + x - vals[q];
            tot[q] = wsum64[32];
            __syncthreads();
        }
        if (s < ns) {
            const u64 cb = carry_c + ex[0];
            L[s].tile_begin = carry_t + ex_t;
            L[s].ntiles = nt;
            L[s].cbase = cb;
            L[s].mbase = carry_m + ex[1];
            if (cb + cc > c->cmat_cap) atomicMin(&cut_s, s);   // does not fit this round
        }
        carry_t += tot_t; carry_c += tot[0]; carry_m += tot[1];
    }
    __syncthreads();
    const u32 cut = cut_s;
    // carry splits [cut, ns) over to the next round
    for (u32 s = cut + threadIdx.x; s < ns; s += 1024) c->splits[nxt][s - cut] = L[s];
    if (threadIdx.x == 0) {
        if (cut < ns) c->nsplits[nxt] = ns - cut;
        RoundPlan pl;
        if (cut == ns) {
            pl.ns = ns; pl.tiles = carry_t; pl.ctot = carry_c; pl.mtot = carry_m;
        } else if (cut == 0) {
            pl.ns = 0; pl.tiles = 0; pl.ctot = 0; pl.mtot = 0;
            if (ns) atomicOr(c->err_flag, 4u);   // a single split larger than the matrix
        } else {
            const SplitTask &lst = L[cut - 1];
            pl.ns = cut; pl.tiles = lst.tile_begin + lst.ntiles;
            pl.ctot = lst.cbase + (u64)lst.ntiles * lst.G; pl.mtot = lst.mbase + lst.m;
        }
        pl.nblk = (u32)((pl.ctot + SCAN_CHUNK - 1) / SCAN_CHUNK);
        pl.next_scan = 0; pl.pad_ = 0;
        pl.cur = cur;
        *c->plan = pl;
        atomicAdd(c->split_keys, (unsigned long long)pl.mtot);
        c->cnt->round += 1;   // every reader of this round takes cur from the plan
        cut_s = pl.nblk;
    }
    __syncthreads();
    // status words of the round's scan blocks (k_scanp_lookback): none published yet
    for (u32 i = threadIdx.x, nb = cut_s; i < nb; i += 1024) c->scan_status[i] = 0ull;
}

// b[i] = inclusive prefix of cnt[1..beta+1] (exclusive block offsets from the
// k_scan_partials/k_scan_bsums pass over cnt+1), T[i] = floor(b_i*gamma/alpha)+1
// (R7), digest of b and the level-1 dump for the pass log.
__global__ void __launch_bounds__(SCAN_THREADS) k_fit_final(const DevCtx *__restrict__ c, u32 node, const u32 *__restrict__ bsum) {
    pdl_entry();
    __shared__ u32 wsum[33];
    __shared__ unsigned long long dsum;
    if (*c->nan_flag) return;
    GNode &g = c->nodes[node];
    if (g.degenerate) return;
    const u64 n = g.beta + 1;
    const bool logging = c->rec != nullptr;
    const bool copy_l1 = g.level == 1 && c->l1_b != nullptr;
    u32 *in = g.cnt + 1;
    if (threadIdx.x == 0) dsum = 0;
    const u64 base = (u64)blockIdx.x * SCAN_CHUNK + (u64)threadIdx.x * SCAN_ITEMS;
    u32 v[SCAN_ITEMS];
    u32 s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) { v[k] = base + k < n ? in[base + k] : 0; s += v[k]; }
    u32 total;
    u32 e = block_excl_scan_1024(s, wsum, total) + bsum[blockIdx.x];
    u64 db = 0;
    u32 *bnd = g.bnd;
    const u32 bsh = g.bshift;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        const u32 eprev = e;
        e += v[k];
        if (base + k < n) {
            const u64 i = base + k + 1;   // 1-based interval index
            in[base + k] = e;
            const u32 Ti = bucket_of(e, g.alpha, g.gamma);
            g.T[i] = Ti;
            if (bnd) {   // digit boundaries of the first split: digit (T - 1) >> bshift rises at bin i
                const u32 d1 = (Ti - 1u) >> bsh, d0 = (bucket_of(eprev, g.alpha, g.gamma) - 1u) >> bsh;
                for (u32 d = d0 + 1; d <= d1; ++d) bnd[d] = (u32)i;
            }
            if (logging) db += digest_term(i, e);
            if (copy_l1 && i - 1 < c->l1_cap) c->l1_b[i - 1] = e;
        }
    }
    if (logging) {
        for (int o = 16; o > 0; o >>= 1) db += __shfl_xor_sync(0xffffffffu, db, o);
        if ((threadIdx.x & 31) == 0) atomicAdd(&dsum, (unsigned long long)db);
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd((unsigned long long *)&g.digest_b, dsum);
    }
}

// --- stable scatter by digit
// One CTA per tile of SPLIT_TILE keys; warp w owns keys [w*SC_PER_WARP, ...)
// of the tile (SC_KPL per lane, chunk q = 32 consecutive keys).  Each key
// takes a rank inside its warp from a shared-memory atomicAdd on the warp's
// counter of its digit (3 instructions; chunks are processed in order, so
// only keys of the same chunk with the same digit can come out of Append
// order), the tile is staged in digit order (digit run, then warp, then
// rank), and the write-out puts every such same-chunk group back in source
// order (groups are found from the staged source index; almost all are
// single keys).  Global writes are coalesced per digit run.
struct SplitScatterSmem {
    u64 buf[SPLIT_TILE];
    u32 dsrc[SPLIT_TILE];            // staged: digit | tile source index << 16
    u32 wc[SC_WARPS][GMAX / 2 + 1];  // per-warp u16 counters (2 per word) -> per-warp offsets in the run
    u32 tstart[GMAX + 1];            // tile-local start of each digit's run
    u32 goff[GMAX + 1];              // segment-relative destination of run position 0 (mod 2^32)
    u32 scan_tmp[SC_WARPS + 1];
};

// FULL: the tile holds SPLIT_TILE keys (every tile but the last of a split), so
// the per-slot validity tests compile away.
template <class K, bool FULL, bool PR>
__device__ __forceinline__ void split_scatter_tile(const DevCtx *__restrict__ c, SplitScatterSmem &S, const SplitTask &st,
                                                   u32 lt, const u32 *__restrict__ P) {
    const u32 deg = !is_radix(st) && c->nodes[st.node].degenerate;   // checked after the tile's loads are issued
    const u64 *x = c->buf[st.src] + st.off;
    u64 *y = c->buf[st.dst] + st.off;
    const u32 w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const u32 G = st.G, GW2 = (G + 1) / 2;
    const u32 k0 = lt * SPLIT_TILE, k1 = min(st.m, k0 + SPLIT_TILE);
    const u32 ntile = k1 - k0;
    const u32 r0 = k0 + w * SC_PER_WARP;
    for (u32 d = lane; d < GW2; d += 32) S.wc[w][d] = 0;
    const u16 *dg = c->digs + st.off;   // digits cached by k_split_count
    u64 key[SC_KPL];
    u32 pk[SC_KPL];
#pragma unroll
    for (u32 q = 0; q < SC_KPL; ++q) {
        const u32 k = r0 + q * 32 + lane;
        const bool v = FULL || k < k1;
        key[q] = v ? x[k] : 0ull;
        pk[q] = v ? (u32)dg[k] : 0xffffffffu;
    }
    // destinations of this tile's digit runs (scanned count matrix), needed after the scan
    constexpr u32 PPER = (GMAX + SC_THREADS - 1) / SC_THREADS;
    u32 pv[PPER];
#pragma unroll
    for (u32 i = 0; i < PPER; ++i) {
        const u32 d = threadIdx.x * PPER + i;
        pv[i] = d < G ? P[st.cbase + (u64)d * st.ntiles + lt] : 0u;
    }
    if (deg) return;   // uniform: the whole CTA leaves
    __syncwarp();
    // rank inside the warp: one atomicAdd per key on the warp's u16 counter of its digit
#pragma unroll
    for (u32 q = 0; q < SC_KPL; ++q) {
        const u32 d = pk[q];
        if (FULL || d != 0xffffffffu) {
            const u32 old = atomicAdd(&S.wc[w][d >> 1], (d & 1u) ? 0x10000u : 1u);
            pk[q] = d | ((((d & 1u) ? old >> 16 : old) & 0xffffu) << 16);
        }
    }
    __syncthreads();
    // per digit pair: warp-exclusive offsets and tile totals; run destinations from the scanned matrix
    for (u32 e = threadIdx.x; e < GW2; e += SC_THREADS) {
        u32 lo = 0, hi = 0;
#pragma unroll
        for (u32 ww = 0; ww < SC_WARPS; ++ww) {
            const u32 v = S.wc[ww][e];
            S.wc[ww][e] = lo | (hi << 16);
            lo += v & 0xffffu;
            hi += v >> 16;
        }
        S.tstart[2 * e] = lo;
        S.tstart[2 * e + 1] = hi;   // e == GW2 - 1 with G odd: digit G, count 0
    }
    __syncthreads();
    {   // exclusive scan of the tile totals over the digits (G <= GMAX)
        constexpr u32 PER = (GMAX + SC_THREADS - 1) / SC_THREADS;
        const u32 b0 = threadIdx.x * PER;
        u32 v[PER], loc = 0;
#pragma unroll
        for (u32 i = 0; i < PER; ++i) { v[i] = b0 + i < G ? S.tstart[b0 + i] : 0; loc += v[i]; }
        u32 incl = loc;
        for (int o = 1; o < 32; o <<= 1) { u32 y2 = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= (u32)o) incl += y2; }
        if (lane == 31) S.scan_tmp[w] = incl;
        __syncthreads();
        if (w == 0) {
            u32 t = lane < SC_WARPS ? S.scan_tmp[lane] : 0;
            u32 ti = t;
            for (int o = 1; o < 32; o <<= 1) { u32 y2 = __shfl_up_sync(0xffffffffu, ti, o); if (lane >= (u32)o) ti += y2; }
            if (lane < SC_WARPS) S.scan_tmp[lane] = ti - t;
        }
        __syncthreads();
        u32 run = S.scan_tmp[w] + incl - loc;
#pragma unroll
        for (u32 i = 0; i < PER; ++i) {
            const u32 d = b0 + i;
            if (d < G) {
                S.tstart[d] = run;
                if (v[i]) S.goff[d] = pv[i] - (u32)st.mbase - run;
                run += v[i];
            }
        }
    }
    __syncthreads();
    // stage in digit order: digit run, then warp, then in-warp rank
#pragma unroll
    for (u32 q = 0; q < SC_KPL; ++q) {
        if (FULL || pk[q] != 0xffffffffu) {
            const u32 d = pk[q] & 0xffffu;
            const u32 wo = (S.wc[w][d >> 1] >> ((d & 1u) * 16)) & 0xffffu;
            const u32 lp = S.tstart[d] + wo + (pk[q] >> 16);
            PCF_CHECK(c, d < G && lp < ntile);
            S.buf[lp] = key[q];
            S.dsrc[lp] = d | ((w * SC_PER_WARP + q * 32 + lane) << 16);
        }
    }
    __syncthreads();
    // Append order inside a group of keys of one chunk with one digit (same
    // dsrc >> 21 and digit, contiguous in the stage) depends on the order the
    // shared-memory atomics of one instruction were served in: check for an
    // inversion, and only then re-rank the groups by source index.
    // (Fused with the write-out: if an inversion is found, every position of the
    // tile is written again from the exact ranks below.)
    bool inv = false;
    // key-value mode: the source index of every key moves with it (gathered from the
    // tile's source range of ibuf[src], identity for the input buffer)
    const u32 *isrc = PR ? c->ibuf[st.src] : nullptr;
    u32 *idst = PR ? c->ibuf[st.dst] + st.off : nullptr;
    auto src_index = [&](u32 tl) -> u32 { return isrc ? isrc[st.off + k0 + tl] : (u32)(st.off + k0 + tl); };
    for (u32 i = threadIdx.x; i < ntile; i += SC_THREADS) {
        const u32 b = S.dsrc[i];
        if (i > 0) {   // same chunk (src >> 5) and digit, source indices out of order
            const u32 a = S.dsrc[i - 1];
            inv |= ((a ^ b) & 0xffe0ffffu) == 0u && a > b;
        }
        PCF_CHECK(c, (b & 0xffffu) < G && S.goff[b & 0xffffu] + i < st.m);
        y[S.goff[b & 0xffffu] + i] = S.buf[i];
        if (PR) idst[S.goff[b & 0xffffu] + i] = src_index(b >> 16);
    }
    if (!__syncthreads_or(inv || (c->flags & FLAG_EXACT_RANKS))) return;
    for (u32 i = threadIdx.x; i < ntile; i += SC_THREADS) {
        const u32 e = S.dsrc[i];
        const u32 d = e & 0xffffu;
        const u32 gk = (e >> 21) << 16 | d;   // group key: chunk, digit
        u32 pos = i;
        const bool sp = i > 0 && (((S.dsrc[i - 1] >> 21) << 16) | (S.dsrc[i - 1] & 0xffffu)) == gk;
        const bool sn = i + 1 < ntile && (((S.dsrc[i + 1] >> 21) << 16) | (S.dsrc[i + 1] & 0xffffu)) == gk;
        if (sp || sn) {
            u32 a = i, b = i + 1;
            while (a > 0 && (((S.dsrc[a - 1] >> 21) << 16) | (S.dsrc[a - 1] & 0xffffu)) == gk) --a;
            while (b < ntile && (((S.dsrc[b] >> 21) << 16) | (S.dsrc[b] & 0xffffu)) == gk) ++b;
            pos = a;
            for (u32 j = a; j < b; ++j) pos += (S.dsrc[j] >> 16) < (e >> 16) ? 1u : 0u;
        }
        y[S.goff[d] + pos] = S.buf[i];
        if (PR) idst[S.goff[d] + pos] = src_index(e >> 16);
    }
}

#ifndef PCF_SC_MINB
#define PCF_SC_MINB 2
#endif
template <class K, bool PR>
__global__ void __launch_bounds__(SC_THREADS, PCF_SC_MINB) k_split_scatter(const DevCtx *__restrict__ c) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char sc_smem_raw[];
    SplitScatterSmem &S = *reinterpret_cast<SplitScatterSmem *>(sc_smem_raw);
    if (*c->nan_flag) return;
    const RoundPlan pl = *c->plan;
    const SplitTask *__restrict__ L = c->splits[pl.cur];
    // one tile per CTA when the grid covers the round, grid-stride otherwise (device-driven batches)
    for (u32 tile = blockIdx.x; tile < pl.tiles; tile += gridDim.x) {
        if (tile != blockIdx.x) __syncthreads();   // the previous tile's stage is written out
        const SplitTask st = L[c->tmap[tile]];
        const u32 lt = tile - st.tile_begin;
        if ((lt + 1) * SPLIT_TILE <= st.m) split_scatter_tile<K, true, PR>(c, S, st, lt, c->pmat);
        else split_scatter_tile<K, false, PR>(c, S, st, lt, c->pmat);
    }
}

__device__ __forceinline__ void push_k7(const DevCtx *c, const K7Task &t) {
    u32 slot = atomicAdd(c->k7_count, 1u);
    atomicAdd(c->k7_keys, (unsigned long long)t.size);
    if (slot < c->k7_cap) c->k7[slot] = t;
    else atomicOr(c->err_flag, 1u);
}

// Tasks of the digit groups of every split of round `cur`.  Groups larger than
// a K7 CTA (keys > S_CAP or buckets > NB_CAP) become the next round's splits
// (or, for a single bucket, host items: a new global node / fallback sort).
// Runs of consecutive smaller groups are packed greedily into one K7 task of
// <= S_CAP keys and <= NB_CAP buckets: a K7_GROUP over the run's bucket range,
// or, for a run of one bucket, a K7_NODE / K7_SORT task (Alg. 1).
__device__ __forceinline__ void make_run_task(const DevCtx *c, const SplitTask &st, GNode &g, u32 d0, u32 d1, u32 keys,
                                              const u32 *__restrict__ P, K7Task &t) {
    const u32 start = P[st.cbase + (u64)d0 * st.ntiles] - (u32)st.mbase;
    const u32 jlo = st.jlo + (d0 << st.shift);
    const u32 jhi = min(st.jlo + ((d1 + 1) << st.shift), st.jhi);
    t.off = st.off + start; t.size = keys; t.src = st.dst; t.node = st.node; t.jlo = jlo; t.jhi = jhi; t.pad = 0;
    if (jhi - jlo == 1) {
        g.H[jlo] = keys;
        const bool sort = keys >= g.delta || keys < c->tau;
        t.kind = sort ? K7_SORT : K7_NODE;
        t.level = g.level + 1;
    } else {
        t.kind = K7_GROUP;
        t.level = g.level;
    }
}

constexpr int TG_THREADS = 256;

// Tasks of a Standard-Sort split after its scatter: runs of consecutive digit groups of
// <= S_CAP keys become K7_SORT tasks (the groups are in key order, so sorting the run sorts
// every group); larger groups become the next radix split (the next lower bits); a split
// whose keys are all equal (count pass) or whose bits are exhausted is sorted as it lies,
// in K7_SORT chunks of <= S_CAP keys.  A few warps' worth of work per split.
__device__ void radix_taskgen(const DevCtx *__restrict__ c, const SplitTask &st, const u32 *__restrict__ P, u32 nxt,
                              u32 *dcnt, u8 *dpack) {
    const u32 lane = threadIdx.x & 31;
    auto emit = [&](u64 off, u32 keys, u32 presorted) {
        K7Task t;
        t.off = off; t.size = keys; t.kind = K7_SORT; t.src = st.dst; t.level = 0; t.node = 0xffffffffu;
        t.jlo = 0; t.jhi = 0; t.pad = presorted;
        push_k7(c, t);
    };
    auto emit_chunks = [&](u64 off, u32 m, u32 t0, u32 nt) {   // keys all equal: sorted as they lie (copied)
        for (u32 k = t0 * (u32)S_CAP; k < m; k += nt * (u32)S_CAP) emit(off + k, min((u32)S_CAP, m - k), 1u);
    };
    if (!(st.jlo & 1u)) {   // all keys of the split are equal
        emit_chunks(st.off, st.m, threadIdx.x, TG_THREADS);
        return;
    }
    for (u32 d = threadIdx.x; d < st.G; d += TG_THREADS) {
        const u32 start = P[st.cbase + (u64)d * st.ntiles] - (u32)st.mbase;
        const u32 end = d + 1 < st.G ? P[st.cbase + (u64)(d + 1) * st.ntiles] - (u32)st.mbase : st.m;
        const u32 cn = end - start;
        dcnt[d] = cn;
        dpack[d] = cn <= (u32)S_CAP ? 1 : 0;
        if (cn > (u32)S_CAP) {
            if (st.shift == 0) {   // every bit consumed: the group's keys are equal
                emit_chunks(st.off + start, cn, 0, 1);
            } else {               // the next lower bits
                const SplitTask nt = radix_split(st.off + start, cn, st.dst, radix_next_shift(st.shift));
                const u32 slot = atomicAdd(&c->nsplits[nxt], 1u);
                if (slot < c->splits_cap) c->splits[nxt][slot] = nt;
                else atomicOr(c->err_flag, 1u);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    // warp 0, in digit order: greedy next-fit runs of packable groups of <= S_CAP keys
    u32 run_start = 0, run_keys = 0, pos = 0;
    for (u32 base = 0; base < st.G; base += 32) {
        const u32 d = base + lane;
        const u32 cn = d < st.G ? dcnt[d] : 0u;
        const u32 pk = d < st.G ? (u32)dpack[d] : 1u;
        const u32 nk = min(32u, st.G - base);
        for (u32 k = 0; k < nk; ++k) {
            const u32 ck = __shfl_sync(0xffffffffu, cn, k);
            const bool pkk = __shfl_sync(0xffffffffu, pk, k) != 0;
            if (!pkk) {
                if (run_keys && lane == 0) emit(st.off + run_start, run_keys, 0u);
                run_keys = 0;
                pos += ck;
                run_start = pos;
            } else {
                if (run_keys + ck > (u32)S_CAP) {
                    if (run_keys && lane == 0) emit(st.off + run_start, run_keys, 0u);
                    run_keys = 0;
                    run_start = pos;
                }
                run_keys += ck;
                pos += ck;
            }
        }
    }
    if (run_keys && lane == 0) emit(st.off + run_start, run_keys, 0u);
}

__global__ void __launch_bounds__(TG_THREADS) k_split_taskgen(const DevCtx *__restrict__ c) {
    pdl_entry();
    __shared__ u32 dcnt[GMAX];
    __shared__ u8 dpack[GMAX];
    __shared__ u32 rd0[GMAX], rd1[GMAX], rk[GMAX];   // packed runs of the split (warp 0)
    __shared__ u32 nrun, rbase;
    if (*c->nan_flag) return;
    const RoundPlan pl = *c->plan;
    const u32 cur = pl.cur, nxt = cur ^ 1u;
    const u32 *__restrict__ P = c->pmat;
    const u32 lane = threadIdx.x & 31;
    for (u32 si = blockIdx.x; si < pl.ns; si += gridDim.x) {   // one CTA per split
        const SplitTask st = c->splits[cur][si];
        if (is_radix(st)) {   // Standard-Sort split: its own task generation
            __syncthreads();
            radix_taskgen(c, st, P, nxt, dcnt, dpack);
            continue;
        }
        GNode &g = c->nodes[st.node];
        if (g.degenerate) continue;
        __syncthreads();
        // every digit in parallel: count, packable into a K7 task?  Groups too large
        // for a K7 CTA become the next round's splits or host items.
        for (u32 d = threadIdx.x; d < st.G; d += TG_THREADS) {
            const u32 start = P[st.cbase + (u64)d * st.ntiles] - (u32)st.mbase;
            const u32 end = d + 1 < st.G ? P[st.cbase + (u64)(d + 1) * st.ntiles] - (u32)st.mbase : st.m;
            const u32 cn = end - start;
            const u32 jlo = st.jlo + (d << st.shift);
            const u32 dhi = min(jlo + (1u << st.shift), st.jhi);
            const u32 W = dhi - jlo;
            const bool pk = cn <= (u32)S_CAP && W <= (u32)NB_CAP;
            dcnt[d] = cn;
            dpack[d] = pk ? 1 : 0;
            if (!pk && cn > 0) {
                const u64 goff = st.off + start;
                if (W == 1) {
                    g.H[jlo] = cn;
                    const bool sort = cn >= g.delta || cn < c->tau;   // Alg. 1
                    push_item(c, goff, cn, g.level + 1, st.dst, sort ? 1u : 0u);
                } else {
                    SplitTask nt;
                    nt.off = goff; nt.m = cn; nt.node = st.node; nt.jlo = jlo; nt.jhi = dhi;
                    nt.shift = choose_shift(W, cn);
                    nt.G = (W + (1u << nt.shift) - 1) >> nt.shift;
                    nt.src = st.dst; nt.dst = st.dst == 1 ? 2 : 1;
                    nt.tile_begin = 0; nt.ntiles = 0; nt.cbase = 0; nt.mbase = 0;
                    u32 slot = atomicAdd(&c->nsplits[nxt], 1u);
                    if (slot < c->splits_cap) c->splits[nxt][slot] = nt;
                    else atomicOr(c->err_flag, 1u);
                }
            }
        }
        if (threadIdx.x == 0) nrun = 0;
        __syncthreads();
        {
        // every warp: greedy next-fit packing of the packable digits of its own range of
        // the split's digits (32 digits per step); runs never cross a warp's range, which
        // only costs a few more (smaller) tasks and keeps the latency of a split short
        const u32 w = threadIdx.x >> 5;
        const u32 RW = ((st.G + TG_THREADS / 32 * 32 - 1) / (TG_THREADS / 32 * 32)) * 32;
        const u32 dbeg = min(st.G, w * RW), dend = min(st.G, dbeg + RW);
        u32 run_d0 = dbeg, run_keys = 0;
        auto emit = [&](u32 d0, u32 d1, u32 keys) {   // lane 0
            if (keys == 0) return;
            const u32 r = atomicAdd(&nrun, 1u);
            rd0[r] = d0; rd1[r] = d1; rk[r] = keys;
        };
        for (u32 base = dbeg; base < dend; base += 32) {
            const u32 d = base + lane;
            const bool valid = d < dend;
            const u32 cn = valid ? dcnt[d] : 0;
            const bool pk = valid ? dpack[d] != 0 : true;
            const u32 dhi = valid ? min(st.jlo + ((d + 1) << st.shift), st.jhi) : 0;
            const u32 npm = __ballot_sync(0xffffffffu, !pk);
            u32 incl = cn;   // inclusive prefix of the chunk's counts (once per chunk)
            for (int o = 1; o < 32; o <<= 1) { u32 y = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= (u32)o) incl += y; }
            u32 s = 0;   // first lane of the chunk not yet assigned to a run
            for (u32 guard = 0; s < 32 && guard < 64; ++guard) {   // each step retires >= 1 lane
                const u32 before_s = s ? __shfl_sync(0xffffffffu, incl, (s + 31) & 31) : 0u;
                const u32 run_jlo = st.jlo + (run_d0 << st.shift);
                const bool bad = valid && lane >= s && (!pk || run_keys + (incl - before_s) > (u32)S_CAP || dhi - run_jlo > (u32)NB_CAP);
                const u32 bm = __ballot_sync(0xffffffffu, bad);
                if (bm == 0) { run_keys += __shfl_sync(0xffffffffu, incl, 31) - before_s; s = 32; break; }
                const u32 b = __ffs(bm) - 1;
                const u32 upto = __shfl_sync(0xffffffffu, incl, (b + 31) & 31);
                const u32 keys = run_keys + (b > s ? upto - before_s : 0);
                if (lane == 0 && base + b > run_d0) emit(run_d0, base + b - 1, keys);
                run_keys = 0;
                if ((npm >> b) & 1u) {   // skip the non-packable digits at b, b+1, ...
                    const u32 rest = ~npm & (b == 31 ? 0u : (0xffffffffu << (b + 1)));
                    s = rest ? (u32)(__ffs(rest) - 1) : 32u;
                } else {
                    s = b;
                }
                run_d0 = base + s;
            }
            if (s < 32 && lane == 0) atomicOr(c->err_flag, 2u);   // unreachable: the loop retires a lane per step
        }
        if (lane == 0 && run_d0 < dend) emit(run_d0, dend - 1, run_keys);
        }
        __syncthreads();
        // all threads: reserve the K7 slots of the split's runs at once, write the tasks
        const u32 nr = nrun;
        {   // keys of the runs (block reduction), K7 slots reserved at once
            u32 tk = 0;
            for (u32 r = threadIdx.x; r < nr; r += TG_THREADS) tk += rk[r];
            for (int o = 16; o > 0; o >>= 1) tk += __shfl_xor_sync(0xffffffffu, tk, o);
            if (lane == 0 && tk) atomicAdd(c->k7_keys, (unsigned long long)tk);
            if (threadIdx.x == 0 && nr) rbase = atomicAdd(c->k7_count, nr);
        }
        __syncthreads();
        for (u32 r = threadIdx.x; r < nr; r += TG_THREADS) {
            K7Task t;
            make_run_task(c, st, g, rd0[r], rd1[r], rk[r], P, t);
            if (rbase + r < c->k7_cap) c->k7[rbase + r] = t;
            else atomicOr(c->err_flag, 1u);
        }
    }
}

// Claim order of the tasks [k7_begin, k7_count) for the next K7 launch:
// largest first (64 size classes of S_CAP/64 keys, a counting sort in one CTA),
// so the persistent grid ends on small tasks (shorter tail) -- for launches of
// up to ~16 tasks per SM; larger ones keep the order taskgen produced them in
// (neighbouring tasks are neighbours in memory, measured 2 % faster on c5f).
__global__ void __launch_bounds__(1024) k_k7_order(const DevCtx *__restrict__ c) {
    pdl_entry();
    __shared__ u32 cnt[64];
    const u32 b = *c->k7_begin, e = min(*c->k7_count, c->k7_cap);
    if (e - b > 16u * 148u) {   // many tasks per CTA: the tail is short anyway; keep the produced
        for (u32 i = b + threadIdx.x; i < e; i += blockDim.x) c->k7_order[i] = i;   // (memory-local) order
        return;
    }
    if (threadIdx.x < 64) cnt[threadIdx.x] = 0;
    __syncthreads();
    auto cls = [&](u32 i) { return 63u - min(c->k7[i].size / (u32)(S_CAP / 64), 63u); };
    for (u32 i = b + threadIdx.x; i < e; i += blockDim.x) atomicAdd(&cnt[cls(i)], 1u);
    __syncthreads();
    if (threadIdx.x < 32) {   // exclusive scan of the 64 class counts
        const u32 a0 = cnt[2 * threadIdx.x], a1 = cnt[2 * threadIdx.x + 1];
        u32 x = a0 + a1;
        for (int o = 1; o < 32; o <<= 1) { const u32 y = __shfl_up_sync(0xffffffffu, x, o); if (threadIdx.x >= (u32)o) x += y; }
        const u32 ex = x - a0 - a1;
        cnt[2 * threadIdx.x] = b + ex;
        cnt[2 * threadIdx.x + 1] = b + ex + a0;
    }
    __syncthreads();
    for (u32 i = b + threadIdx.x; i < e; i += blockDim.x) c->k7_order[atomicAdd(&cnt[cls(i)], 1u)] = i;
}

__global__ void k_k7_advance(const DevCtx *__restrict__ c) {
    pdl_entry();
    *c->k7_begin = *c->k7_count;
    *c->k7_next = 0;
}

// ------------------------------------------------------------------ pass-log records of the global nodes
// One CTA per global node (grid-stride): digest and dispatch counts of its
// complete H (written by the split rounds and the K7 groups), then the record.
template <class K>
__global__ void __launch_bounds__(256) k_log_finalize(const DevCtx *__restrict__ c) {
    pdl_entry();
    if (c->rec == nullptr || *c->nan_flag) return;
    __shared__ unsigned long long sdh[8];
    __shared__ u32 sn[8][3];
    const u32 nn = c->cnt->node_count, tau = c->tau;
    for (u32 node = blockIdx.x; node < nn; node += gridDim.x) {
        const GNode &g = c->nodes[node];
        if (g.degenerate) continue;   // uniform per CTA: Standard-Sort, no bucketing record (R9/R10)
        if (node == 0 && c->root_external == 1) continue;   // sharded: another rank records the root
        u64 dh = 0;
        u32 nf = 0, ns = 0, nr = 0;
        const bool copy_l1 = g.level == 1 && c->l1_h != nullptr;
        for (u32 u = threadIdx.x; u <= g.gamma; u += blockDim.x) {
            const u32 h = g.H[u + 1];
            dh += digest_term(u + 1, h);
            if (h) { if (h >= g.delta) nf++; else if (h < tau) ns++; else nr++; }
            if (copy_l1 && u < c->l1_cap) c->l1_h[u] = h;
        }
        for (int o = 16; o > 0; o >>= 1) {
            dh += __shfl_xor_sync(0xffffffffu, dh, o);
            nf += __shfl_xor_sync(0xffffffffu, nf, o);
            ns += __shfl_xor_sync(0xffffffffu, ns, o);
            nr += __shfl_xor_sync(0xffffffffu, nr, o);
        }
        const u32 w = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0) { sdh[w] = dh; sn[w][0] = nf; sn[w][1] = ns; sn[w][2] = nr; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (u32 i = 1; i < blockDim.x / 32; ++i) { dh += sdh[i]; nf += sn[i][0]; ns += sn[i][1]; nr += sn[i][2]; }
            const unsigned long long slot = atomicAdd(c->rec_count, 1ull);
            if (slot < c->rec_cap) {
                NodeRec r;
                r.level = g.level; r.alpha = g.alpha; r.offset = c->gbase + g.off; r.m = g.m;
                r.xmin_bits = K::from_okey(g.kmin); r.xmax_bits = K::from_okey(g.kmax);
                r.digest_b = g.digest_b; r.digest_h = dh;
                r.n_fallback = nf; r.n_small = ns; r.n_recurse = nr; r.reserved = 0;
                c->rec[slot] = r;
            }
        }
        __syncthreads();
    }
}

// Status of the call for asynchronous callers: PCF_OK, PCF_ERR_NAN,
// PCF_ERR_LOG_OVERFLOW or PCF_ERR_INTERNAL, written in stream order after all work.
__global__ void k_status(const DevCtx *__restrict__ c, int *status) {
    pdl_entry();
    const Counters &C = *c->cnt;
    int s = 0;                                   // PCF_OK
    if (C.nan_flag) s = 2;                        // PCF_ERR_NAN
    else if (C.err_flag) s = 7;                   // PCF_ERR_INTERNAL
    else if (c->rec != nullptr && c->rec_count && *c->rec_count > c->rec_cap) s = 6;   // PCF_ERR_LOG_OVERFLOW
    *status = s;
}

}  // namespace pcf
