/*
 * pcf_sort.h -- C ABI of libpcfsort.so, the B200 (sm_100a) PCF Learned Sort.
 *
 * The library sorts an array of 8-byte keys on one GPU with PCF Learned Sort
 * (Sato & Matsui, arXiv 2405.07122): Algorithm 1 "Learned-Sort"
 * with the piecewise-constant CDF model of §3.2
 * and alpha = beta = gamma = delta = floor(n^{3/4})
 * (Theorems 1-2).  Silent points of the paper are resolved
 * as listed in DESIGN.md §2 (readings R1-R16); the result is bit-identical to
 * the CPU oracle in oracle/ (tests/test_gpu_parity.py), including every
 * per-node bucket histogram when the pass log is enabled.
 *
 * Signatures use plain pointers and sizes only.  "device" pointers are CUDA
 * device (or managed) memory of the current device; "host" pointers are
 * ordinary host memory.  `stream` is a cudaStream_t passed as void* (NULL =
 * the legacy default stream).  All functions are thread-safe for distinct
 * streams; the library keeps no global state besides a thread-local error
 * string.
 */
#ifndef PCF_SORT_H
#define PCF_SORT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCF_ABI_VERSION 2   /* 2: pcf_params.status_out, pcf_stats.device_batches, 9 phases */

/* ---- status codes (every entry point returns one) ---------------------- */
#define PCF_OK 0
#define PCF_ERR_INVALID_ARG 1          /* NULL with n>0, tau<2, bad overlap, n >= 2^32, bad struct_size */
#define PCF_ERR_NAN 2                  /* f64 input contains a NaN (domain error)         */
#define PCF_ERR_WORKSPACE_TOO_SMALL 3  /* caller workspace smaller than pcf_workspace_bytes()          */
#define PCF_ERR_OOM 4                  /* device allocation failed                                     */
#define PCF_ERR_CUDA 5                 /* a CUDA runtime call failed (see pcf_last_error())            */
#define PCF_ERR_LOG_OVERFLOW 6         /* pass log capacity exceeded (records beyond capacity dropped) */
#define PCF_ERR_INTERNAL 7             /* internal capacity bound violated (bug)                       */
#define PCF_ERR_DEGENERATE 8           /* pcf_bucket_counts_f64: x_max == x_min, M_PCF undefined (R9)   */

/* ---- key types ---------------------------------------------------------- */
#define PCF_KEY_F64 0   /* IEEE binary64, ascending under IEEE-754 totalOrder (-0.0 before +0.0) */
#define PCF_KEY_U64 1   /* uint64_t, ascending numeric order                                      */
/* or'ed into pcf_workspace_bytes' key_type for the key-value entry points: */
#define PCF_KEY_ARGSORT 0x10  /* pcf_argsort_*: + one u32 index per key                      */
#define PCF_KEY_PAIRS   0x20  /* pcf_sort_pairs_*: + the permutation buffer as well          */

/* ---- flags -------------------------------------------------------------- */
#define PCF_FLAG_SYNC       1u  /* synchronise the stream once before returning, report NaN/overflow
                                   and fill *stats; without it the call never synchronises       */
#define PCF_FLAG_SAMPLE_ALL 2u  /* test mode (reading R14): sample = whole segment, alpha = m      */
#define PCF_FLAG_TIMING     4u  /* record CUDA events per phase into stats->phase_ms (implies SYNC) */
#define PCF_FLAG_PROFILE    8u  /* K7 per-phase SM cycle counters into stats->k7_cycles (with SYNC) */
#define PCF_FLAG_EXACT_RANKS 16u /* test mode: the split scatter always takes its exact (source-
                                    index) re-rank path instead of trusting the atomic ranks      */

/* One record per bucketing node, i.e. per call of Alg. 1 that reaches its
 * model-based bucketing step.  Identical layout to the
 * oracle's record; compared after sorting by (level, offset). */
typedef struct pcf_node_record {
    uint32_t level;       /* recursion level, 1 = whole array                       */
    uint32_t alpha;       /* sample size alpha (= beta = gamma = delta unless R14)   */
    uint64_t offset;      /* global offset of the segment in the array               */
    uint64_t m;           /* segment length                                          */
    uint64_t xmin_bits;   /* bit pattern of x_min, totalOrder min     */
    uint64_t xmax_bits;   /* bit pattern of x_max                                    */
    uint64_t digest_b;    /* digest of b[1..beta+1]               */
    uint64_t digest_h;    /* digest of H[1..gamma+1]  (bucket sizes |c_j|)           */
    uint32_t n_fallback;  /* non-empty buckets with |c_j| >= delta    */
    uint32_t n_small;     /* non-empty buckets with |c_j| < delta and < tau          */
    uint32_t n_recurse;   /* non-empty buckets with tau <= |c_j| < delta             */
    uint32_t reserved;
} pcf_node_record;        /* 72 bytes */

/* Optional pass log (parity / debugging).  All buffers are DEVICE memory
 * owned by the caller.  Off when params->log == NULL. */
typedef struct pcf_pass_log {
    pcf_node_record *records;  /* device array of `capacity` records, unordered      */
    uint64_t capacity;
    uint64_t *count;           /* device u64, set to the number of records produced  */
    uint32_t *level1_b;        /* device, level-1 b[1..beta+1] (0-based), or NULL    */
    uint32_t *level1_h;        /* device, level-1 H[1..gamma+1] (0-based), or NULL   */
    uint64_t level1_capacity;  /* entries available in level1_b / level1_h           */
} pcf_pass_log;

/* Host-side statistics, written when params->stats != NULL.  Fields read from
 * device counters (rounds, groups_smem, split_keys_moved, global_nodes,
 * fallback_keys_global, device_batches, phase_bytes, k7_cycles, and the
 * device-driven part of kernel_launches) are filled only by synchronous calls
 * (PCF_FLAG_SYNC or PCF_FLAG_TIMING); asynchronous calls leave them 0. */
#define PCF_PHASES 9
typedef struct pcf_stats {
    uint32_t kernel_launches;  /* kernels this call launched                                  */
    uint32_t rounds;           /* device work rounds (global bucketing / split waves)        */
    uint32_t host_syncs;       /* stream synchronisations inside the call: 1 with SYNC, else 0 */
    uint32_t device_batches;   /* device-driven batches of oversized recursing buckets run    */
    uint64_t groups_smem;      /* bucket groups finished in shared memory (K7 tasks)         */
    uint64_t split_keys_moved; /* keys moved by the global digit-split rounds (all rounds)    */
    uint64_t global_nodes;     /* bucketing nodes run by the global (multi-CTA) path          */
    uint64_t fallback_keys_global; /* keys of Standard-Sort buckets of > 8192 keys (radix splits) */
    /* PCF_FLAG_TIMING: milliseconds per phase, CUDA events on `stream`:
     * [0] min/max  [1] sample+fit  [2] classify+histogram  [3] stable scatter
     * [4] smem subtree (K7)  [5] pass-log records of the global nodes  [6] other
     * [7] total  [8] device-driven batches of oversized recursing buckets (all their
     * phases: the host cannot place events inside the device-driven loop) */
    float phase_ms[PCF_PHASES];
    uint64_t phase_bytes[PCF_PHASES];  /* algorithmic bytes per phase */
    /* PCF_FLAG_PROFILE: clock64 cycles summed over K7 CTAs per phase (see pcf_k7.cuh prof_mark);
     * [16..19]: warp-cycles inside node steps of double teams / teams / single warps, and
     * warp-cycles single warps spent waiting for small nodes */
    uint64_t k7_cycles[24];
} pcf_stats;

typedef struct pcf_params {
    uint32_t struct_size;      /* = sizeof(pcf_params); set by pcf_params_init             */
    uint32_t tau;              /* base-case threshold tau (reading R1), >= 2; default 64   */
    uint64_t seed;             /* sampler seed (reading R3); default 0                     */
    uint32_t flags;            /* PCF_FLAG_*; default PCF_FLAG_SYNC                        */
    uint32_t reserved0;
    void *workspace;           /* device scratch, >= pcf_workspace_bytes(); NULL = the      */
    size_t workspace_bytes;    /*   library allocates stream-ordered (cudaMallocAsync)     */
    pcf_pass_log *log;         /* host struct pointing at device buffers, or NULL          */
    pcf_stats *stats;          /* host struct, or NULL                                     */
    /* ABI v2: device (or mapped pinned host) int that receives, in stream order after
     * all of the sort's work, PCF_OK, PCF_ERR_NAN, PCF_ERR_LOG_OVERFLOW or
     * PCF_ERR_INTERNAL -- the status of an asynchronous call.  NULL = not written. */
    int *status_out;
} pcf_params;
#define PCF_PARAMS_V1_SIZE ((uint32_t)offsetof(pcf_params, status_out))   /* v1 callers: no status_out */

/* Fill *p with the defaults above.  Never fails. */
void pcf_params_init(pcf_params *p);

/* Upper bound on the device scratch one sort of n keys of `key_type` needs
 * with parameters p (NULL = defaults): one n-key buffer plus the PCF tables,
 * histograms and work queues.  Pure host arithmetic; no CUDA call. */
size_t pcf_workspace_bytes(size_t n, int key_type, const pcf_params *p);

/* Sort n keys (Alg. 1).  in/out: DEVICE pointers to n
 * contiguous keys, 8-byte aligned.  `in` is never written unless in == out
 * (in-place is allowed); any other overlap of [in, in+n) and [out, out+n) is
 * PCF_ERR_INVALID_ARG.  `out` is fully overwritten with the ascending
 * permutation of `in`.
 * Execution: every kernel is enqueued on `stream`; the recursion over buckets
 * too large for one CTA and the fallback sort run from CUDA
 * graphs whose loops are decided on the device, so the host never waits for the
 * GPU inside the call.  Without PCF_FLAG_SYNC the call returns right after
 * enqueueing (stats->host_syncs == 0); with it, it synchronises `stream` once.
 * Errors: argument errors return before any launch.  NaN (f64) is detected on
 * the device by the first pass (the level-1 min/max), which sets a
 * device flag; every later kernel then exits without work.  With PCF_FLAG_SYNC
 * the call returns PCF_ERR_NAN (out unspecified); without it the call returns
 * PCF_OK after enqueueing and the NaN is reported through params->status_out.
 * Device capacity violations (a bug) are PCF_ERR_INTERNAL the same way. */
int pcf_sort_f64(const double *in, double *out, size_t n, const pcf_params *p, void *stream);
int pcf_sort_u64(const uint64_t *in, uint64_t *out, size_t n, const pcf_params *p, void *stream);

/* ---- key-value mode (not in the paper, which sorts keys only,
 * PAPER.md:136-139).  Equal keys keep their input order: the result is THE stable
 * sorting permutation (reading R18), bit-identical to oracle stable_argsort.
 * The sort itself is unchanged (same buckets, same node records); every kernel that
 * moves keys also moves the key's source index: the stable split scatter (global
 * u32 indices), K7 (task-local u16 indices in shared memory, stable tie-break by
 * index in its leaf sorts; the stable radix splits of oversized Standard-Sort buckets
 * keep input order among equal keys).  Needs
 * tau >= 16 (PCF_ERR_INVALID_ARG otherwise: shared-memory room for the indices).
 *
 * pcf_argsort_*: in/out as pcf_sort_*; perm: DEVICE uint32_t[n], 4-byte aligned,
 *   receives perm[k] = input index of out[k].  Workspace: pcf_workspace_bytes(n,
 *   key_type | PCF_KEY_ARGSORT, p).  Other semantics (flags, errors, status_out) as
 *   pcf_sort_*.  n < 2^32. */
int pcf_argsort_f64(const double *in, double *out, uint32_t *perm, size_t n, const pcf_params *p, void *stream);
int pcf_argsort_u64(const uint64_t *in, uint64_t *out, uint32_t *perm, size_t n, const pcf_params *p, void *stream);

/* pcf_sort_pairs_<key>_<value>: keys_in/keys_out as pcf_sort_*; vals_in / vals_out:
 * DEVICE arrays of n values (aligned to their size) that must not overlap each
 * other; vals_out[k] = vals_in[perm[k]].  Workspace: pcf_workspace_bytes(n,
 * key_type | PCF_KEY_PAIRS, p) (the permutation lives in it).  With PCF_FLAG_SYNC the
 * call synchronises once, after the value gather. */
int pcf_sort_pairs_f64_u32(const double *keys_in, const uint32_t *vals_in, double *keys_out, uint32_t *vals_out,
                           size_t n, const pcf_params *p, void *stream);
int pcf_sort_pairs_f64_u64(const double *keys_in, const uint64_t *vals_in, double *keys_out, uint64_t *vals_out,
                           size_t n, const pcf_params *p, void *stream);
int pcf_sort_pairs_u64_u32(const uint64_t *keys_in, const uint32_t *vals_in, uint64_t *keys_out, uint32_t *vals_out,
                           size_t n, const pcf_params *p, void *stream);
int pcf_sort_pairs_u64_u64(const uint64_t *keys_in, const uint64_t *vals_in, uint64_t *keys_out, uint64_t *vals_out,
                           size_t n, const pcf_params *p, void *stream);

/* ---- sharded sort over R GPUs -------------------------
 * One process per GPU; the caller (paper_2405_07122_b200/sharded.py) runs the
 * collectives between the calls (NCCL all-reduce / all-gather / all-to-all over
 * NVLink).  Rank r holds keys [offset, offset + n) of the global array of N keys.
 * The result is Alg. 1 on the WHOLE array: the level-1 node's extremes, sample
 * (the single-GPU positions over [0, N)), b, T and H are the single-GPU ones;
 * bucket ranges of ~N/R keys go to ranks; rank r's output is the sorted slice of
 * the global output starting at range[0], bit-identical to the single-GPU sort, and
 * every node record is the single-GPU one (the level-1 record on rank 0 only).
 * Sequence (device pointers; `state` of pcf_shard_state_bytes(N, R) bytes):
 *   pcf_shard_minmax     -> all-reduce state mm[0] MIN, mm[1] MAX, mm[2] MAX (int64)
 *   pcf_shard_counts     -> all-reduce SUM of the counts (uint32[beta + 2])
 *   pcf_shard_histogram  -> all-gather of the local histogram into Hall (R rows)
 *   pcf_shard_partition  -> keys_out = local keys grouped by destination rank (stable);
 *                           send / recv counts (host) for the all-to-all; range (host):
 *                           {global offset, size, J_lo, J_hi} of this rank's buckets
 *   all-to-all (keys, in source-rank order)
 *   pcf_shard_sort_range -> out = the sorted range (workspace pcf_shard_workspace_bytes)
 * pcf_shard_views returns the device pointers the collectives act on. */
typedef struct pcf_shard {
    uint64_t N;        /* keys over all ranks, 2 <= N < 2^32                     */
    uint64_t offset;   /* global index of this rank's first key                  */
    uint32_t R, rank;  /* 1 <= R <= 64                                            */
    void *state;       /* DEVICE, pcf_shard_state_bytes(N, R) bytes, 256-aligned  */
    size_t state_bytes;
} pcf_shard;
size_t pcf_shard_state_bytes(uint64_t N, uint32_t R);
size_t pcf_shard_workspace_bytes(size_t m, uint64_t N);
/* views[0]: int64 mm[4]; [1]: uint32 counts[beta + 2]; [2]: uint32 Hloc[gamma + 2];
 * [3]: uint32 Hall[R][gamma + 2]; sizes[i]: element counts */
int pcf_shard_views(const pcf_shard *sh, void **views, uint64_t *sizes);
int pcf_shard_minmax(const void *keys, size_t n, int key_type, const pcf_shard *sh, void *stream);
int pcf_shard_counts(const void *keys, size_t n, int key_type, const pcf_shard *sh, const pcf_params *p, void *stream);
int pcf_shard_histogram(const void *keys, size_t n, int key_type, const pcf_shard *sh, const pcf_params *p, void *stream);
int pcf_shard_partition(const void *keys, size_t n, int key_type, const pcf_shard *sh, void *keys_out,
                        uint64_t *send_counts, uint64_t *recv_counts, uint64_t *range, void *stream);
int pcf_shard_sort_range(const void *keys, void *out, size_t m, int key_type, const pcf_shard *sh,
                         const uint64_t *range, const pcf_params *p, void *stream);

/* End-to-end entry: HOST pointers (pinned memory recommended).  Copies the n
 * keys to the device, sorts them with pcf_sort_* (asynchronously), copies the
 * result back and synchronises `stream` once; returns the sort's status
 * (PCF_ERR_NAN etc.; also written to p->status_out if set).  If p->workspace holds at least
 * round_up(8n, 256) + pcf_workspace_bytes(n) bytes it is used as [device keys |
 * sort workspace]; otherwise device buffers are stream-ordered allocations freed
 * before return.  in_host == out_host is allowed. */
int pcf_sort_f64_host(const double *in_host, double *out_host, size_t n, const pcf_params *p, void *stream);
int pcf_sort_u64_host(const uint64_t *in_host, uint64_t *out_host, size_t n, const pcf_params *p, void *stream);

/* ---- the paper's bucketing-failure experiment (§4.3, Fig. 4)
 * One model-based bucketing step M_PCF (Alg. 1, PAPER.md:152-158;
 * model PAPER.md:288-308) of n float64 keys with DECOUPLED alpha, beta, gamma
 * (the sort fixes alpha = beta = gamma = delta = floor(n^{3/4})):
 *   sample a_k = keys[pos_k], k = 0..alpha-1, pos_k from the sampler of reading
 *     R3 for the root node (level 1, offset 0) and `seed`, with replacement;
 *   b[i] = |{k : i(a_k) <= i}|, i = 1..beta+1, with i(x) of reading R6;
 *   H[j] = |c_j| = |{x : floor(b[i(x)] * gamma / alpha) + 1 = j}|, j = 1..gamma+1 (R7).
 * The paper's "bucketing failure" is max_j |c_j| > delta (the caller compares).
 * keys:       DEVICE, n f64 keys, 8-byte aligned, not modified.
 * b_out:      DEVICE, beta + 1 uint32 (b[1..beta+1], stored 0-based), overwritten.
 * H_out:      DEVICE, gamma + 1 uint32 (|c_1|..|c_{gamma+1}|), overwritten.
 * max_bucket: HOST, receives max_j |c_j|; may be NULL.
 * Synchronous on `stream` (one 24-byte device scratch, stream-ordered alloc).
 * Errors: PCF_ERR_INVALID_ARG (NULL or misaligned pointer, n < 2 or n >= 2^32, alpha, beta or
 * gamma 0 or >= 2^32, beta + 1 or gamma + 1 overflow) before any launch;
 * PCF_ERR_NAN if a key is NaN; PCF_ERR_DEGENERATE if all keys are equal (b_out,
 * H_out unspecified after either); PCF_ERR_CUDA / PCF_ERR_OOM. */
int pcf_bucket_counts_f64(const double *keys, size_t n, uint64_t alpha, uint64_t beta, uint64_t gamma,
                          uint64_t seed, uint32_t *b_out, uint32_t *H_out, uint64_t *max_bucket, void *stream);

/* Entries the pass log's level1_b / level1_h arrays need for a sort of n keys:
 * beta + 1 = gamma + 1 = floor(n^{3/4}) + 1 (reading R5), plus one
 * spare.  Pure host arithmetic. */
size_t pcf_level1_entries(size_t n, const pcf_params *p);

/* Human-readable name of a status code (static storage). */
const char *pcf_status_string(int status);

/* Detail of the last error on the calling thread (static thread-local storage). */
const char *pcf_last_error(void);

/* ABI version of the loaded library (PCF_ABI_VERSION it was built with). */
int pcf_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PCF_SORT_H */
