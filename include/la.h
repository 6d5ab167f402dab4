/*
 * la.h -- C ABI of the B200-native LeanAttention decode library (libleanattn.so).
 *
 * LeanAttention (arXiv 2405.10480): exact decode-phase attention (query length 1, or one
 * GQA query group per KV head) over a long KV cache, decomposed stream-K style.
 * Citations: P:n = line n of the paper text, S:n = line n of SPEC.md,
 * Alg1§k / Alg2§k = statement k of Algorithm 1 / 2, readings Cn = DESIGN.md §Readings.
 *
 * The operation (Eq. 1; Table 1 decode column): for every request b,
 * query head h_q (KV head h_kv = h_q / g, g = heads_q / heads_kv, reading C3) and the
 * n_b = ctx_lens[b] cached keys/values,
 *     s_j = scale * <q[b,h_q,:], k[b,h_kv,j,:]>            j = 0 .. n_b - 1
 *     O[b,h_q,:] = sum_j softmax(s)_j v[b,h_kv,j,:]         (fp32, reading C4)
 *     L[b,h_q]   = ln sum_j e^{s_j}                          (Alg2§39, reading C2)
 * computed by ONE persistent kernel launch: the flattened (unit x LeanTile) iteration
 * space is cut into G equal contiguous ranges (Eq. 2, Alg2§4-9), each
 * CTA runs Alg. 1 over its segments and boundary-straddling units are merged
 * in-kernel by the owning ("host") CTA with the softmax re-scaling operator (§4.1
 * P:286-294; Alg2§19-36), with no second launch.
 *
 * Conventions for every entry point:
 *  - Return LA_OK or an error code; no C++ exception crosses the ABI.  A human-readable
 *    message for the last error on the calling thread is available from la_last_error().
 *  - Device pointers are plain CUDA device addresses owned by the CALLER (e.g. torch
 *    tensors); the library never frees them.  `stream` is a cudaStream_t (NULL = legacy
 *    default stream).  Kernels run asynchronously on `stream`; device-side faults surface
 *    at the caller's next synchronisation.
 *  - A plan owns all device memory it allocates (schedule tables, per-CTA partial slots
 *    Op/mp/lp and flags, Alg2§20-23) until la_plan_destroy().  la_decode and la_plan_update
 *    never allocate.
 *  - Not thread-safe on one plan: two la_decode calls on the same plan must be ordered
 *    on one stream (they share the partial slots and flags).
 */
#ifndef LEANATTN_LA_H
#define LEANATTN_LA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LA_VERSION 1

typedef enum {
  LA_OK = 0,
  LA_ERR_INVALID = 1,      /* bad argument: null/misaligned pointer, bad shape or size  */
  LA_ERR_UNSUPPORTED = 2,  /* valid request this build does not implement (dtype, d, g)  */
  LA_ERR_CUDA = 3,         /* a CUDA runtime call failed (message in la_last_error)     */
  LA_ERR_NOMEM = 4,        /* device or host allocation failed                          */
  LA_ERR_STATE = 5,        /* e.g. la_decode on a host-only plan                         */
  LA_ERR_TIMEOUT = 6       /* an in-kernel wait gave up: a peer CTA (10 s) or a peer rank
                              (5 s) never signalled (reported by la_plan_status)          */
} la_status;

/* Storage type of Q, K and V ("FP16->32": 16-bit inputs, fp32 arithmetic).
   LA_FP8_E4M3 (NEXT-4, not in the paper): K and V hold OCP FP8 E4M3 codes (1 byte each;
   the cache is K = code x opts.k_scale, V = code x opts.v_scale) and q is bf16; head_dim
   128 only.  The codes are widened exactly to f16 on chip; q is rounded bf16 -> f16 for
   the tensor-core QK^T (reading C23: exact for 2^-14 <= |q| < 65504). */
typedef enum { LA_BF16 = 0, LA_FP16 = 1, LA_FP32 = 2, LA_FP8_E4M3 = 3 } la_dtype;

/* KV cache layouts (reading C14 fixes the unit linearisation order). */
typedef enum {
  /* (B, H_kv, max_ctx, d) contiguous, request b valid on rows [0, ctx_lens[b]).
     Units (b, h_kv) linearised batch -> heads. */
  LA_KV_BHSD = 0,
  /* The paper's unpadded ragged layout (H_kv, sum_b n_b, d), request b on rows
     cu_seqlens[b] .. cu_seqlens[b+1] (cu_seqlens = prefix sum of ctx_lens, built by the
     planner).  Units linearised heads -> total context. */
  LA_KV_PACKED = 1,
  /* Paged pools (num_pages, H_kv, page_size, d) (NEXT-4, serving layout): token t of request
     b lives in page block_table[b][t / page_size] at row t % page_size.  block_table and
     page_size come with the plan (opts); units linearised batch -> heads. */
  LA_KV_PAGED = 2
} la_layout;

/* Work decomposition.  STREAMK is the method; the other two are its
   special cases / the baselines it is compared with, kept for the NEXT-1 comparison. */
typedef enum {
  LA_SCHED_STREAMK = 0,    /* Eq. 2 + Alg. 2 exactly: G equal contiguous iteration ranges,
                              host CTAs wait on their peers' flags (cooperative launch)  */
  LA_SCHED_SEQUENTIAL = 1, /* FA2: one CTA per unit, G = #units            */
  LA_SCHED_DYNAMIC = 2,    /* Alg. 2's equal ranges, each cut into a HEAD (its first
                              dyn_first_permille / 1000) and <= 8 tail chunks of >= dyn_min_chunk
                              LeanTiles; the persistent CTAs claim every head, then the chunks
                              round by round (atomic counter), so fast SMs take more chunks.  A
                              unit's pieces are folded by its LAST arriving piece in ascending
                              order -- same result semantics, bitwise deterministic, balances
                              TIME instead of LeanTile counts                    */
  LA_SCHED_FIXED_SPLIT = 3,/* FlashDecoding's fixed-split decomposition: every
                              unit cut into `split` near-equal chunks (first chunks take the
                              extra LeanTile), chunks run in order on the persistent
                              CTAs like hardware waves, folded in-kernel (the comparison
                              baseline of the paper's evaluation, NEXT-1)                 */
  LA_SCHED_AUTO = 4        /* (default) LA_SCHED_DYNAMIC for one-row tiles (MHA, T_m = 1) of a
                              bf16 / fp16 / fp32 BHSD or packed cache whose Eq. 2 ranges hold
                              >= 64 LeanTiles, LA_SCHED_STREAMK otherwise (multi-row tiles, FP8,
                              paged pools, exchange plans) -- the faster of the two as measured
                              on B200; la_plan_info.schedule reports the choice   */
} la_schedule;

typedef struct {
  float scale;       /* softmax scale applied to every score before max/exp (reading C1);
                        0 -> 1/sqrt(head_dim) (Eq. 1)                              */
  int layout;        /* la_layout, default LA_KV_BHSD                                     */
  int64_t max_ctx;   /* BHSD row stride of one (b, h_kv) slab in tokens; 0 -> max(ctx_lens) */
  int grid;          /* G.  0 -> min(#co-resident CTAs = 148 x occupancy, I) (reading C15);
                        > 0 forces G (tests), clamped to the co-resident maximum on device
                        plans because hosts wait on peers (Alg2§28 needs co-residency)    */
  int num_sms;       /* host-only plans: SM count assumed when grid == 0 (default 148)    */
  int ctas_per_sm;   /* host-only plans: occupancy assumed when grid == 0 (default 1)     */
  int host_only;     /* 1 -> plan the schedule only, no device state (inspection/tests)   */
  int schedule;      /* la_schedule, default LA_SCHED_AUTO (resolved at la_plan)          */
  int trace;         /* 1 -> every la_decode records a per-CTA timeline (la_plan_trace)     */
  int dyn_first_permille; /* LA_SCHED_DYNAMIC: head share of each Eq. 2 range, permille (default 940;
                             1000 = no tail: Alg. 2's ranges exactly)                        */
  int dyn_min_chunk;      /* LA_SCHED_DYNAMIC: smallest tail chunk in LeanTiles (default 2)    */
  int split;              /* LA_SCHED_FIXED_SPLIT: chunks per unit; 0 -> FlashAttention-2's
                             num_splits heuristic (wave efficiency >= 85% of the best)     */
  /* LA_KV_PAGED only: */
  const int32_t* block_table; /* HOST [batch][pages_per_seq] physical page indices; copied
                                 into the plan (re-plan when it changes)                   */
  int pages_per_seq;          /* row stride of block_table (>= ceil(max ctx / page_size))   */
  int page_size;              /* tokens per page: 16, 32, 64, 128 or 256                    */
  int64_t num_pages;          /* pages in each pool; every table entry must be < num_pages  */
  /* N_q > 1 (NEXT-3: speculative / multi-token decode; the paper's T_m rows, Alg2§4): */
  int q_len;                  /* query tokens per request N_q (default 1); q, out are then
                                 (B, H_q, N_q, d) and lse (B, H_q, N_q).  The g * N_q rows of
                                 one KV head are cut into C_m = ceil(g N_q / T_m) query tiles
                                 of T_m <= 8 rows (Alg2§4); each tile is a work unit that
                                 streams the head's KV (MQA / large groups included)          */
  int causal;                 /* 1 (default): query i of N_q is the token at position
                                 n - N_q + i and attends to keys [0, n - N_q + i]; 0: every
                                 query attends to all n keys                                 */
  /* Fused cross-GPU sequence-shard exchange (NEXT-2; see la_plan_xchg_handle): */
  int xchg_world;             /* P ranks (2..8) each holding a contiguous shard of every
                                 request's context; 0 or 1 = off.  With P > 1, la_decode on
                                 rank r's shard returns the FULL result on every rank      */
  int xchg_rank;              /* this plan's rank r in [0, P)                               */
  /* Heterogeneous batches (NEXT-3: decode mixed with speculative / chunked-prefill blocks): */
  const int32_t* q_lens;      /* HOST [batch] query tokens N_b per request (>= 1, <= ctx_lens[b]),
                                 or NULL for q_len everywhere.  q / out / lse then hold, per
                                 request in order, an (H_q, N_b[, d]) block (rows (b, h_q, i)
                                 contiguous); with NULL this is exactly (B, H_q, N_q[, d])    */
  /* LA_FP8_E4M3 only (per-tensor dequantisation scales; 0 -> 1): */
  float k_scale;              /* K = code x k_scale (folded into the score scale)             */
  float v_scale;              /* V = code x v_scale (applied once, at finalize: O x v_scale)  */
  /* Tensor-core engine for T_m > 1 tiles (GQA groups / N_q > 1; MHA always runs on CUDA cores): */
  int engine;                 /* la_engine, default LA_ENGINE_AUTO.  LA_ENGINE_TCGEN05 needs
                                 bf16 / fp16 and head_dim 128 when T_m > 1, and its 16-row
                                 tiles (g * N_q > 8) the static schedules, else
                                 la_plan fails with LA_ERR_UNSUPPORTED; ignored for T_m = 1
                                 (MHA: a GEMV, CUDA cores) and FP8 caches                     */
  void* stream;               /* cudaStream_t for the plan's initial table upload: la_plan then
                                 returns with the ONE H2D copy of its tables still in flight on
                                 it (decode on the same stream).  NULL: la_plan waits for it   */
} la_plan_opts;

/* Which tensor-core instructions contract the T_m x T_n tiles (Alg1§20, §24). */
typedef enum {
  LA_ENGINE_MMA_SYNC = 0, /* warp-level mma.sync m16n8k16: every consumer warp owns its own
                             32-token rounds and accumulators in registers      */
  LA_ENGINE_TCGEN05 = 1,  /* 5th-gen tensor cores: one warpgroup per 128-token stage, one
                             thread issues tcgen05.mma (M = 128 tokens / dims, N = 16 / 32)
                             with S^T and the per-stage O^T in TMEM (N up to 32 / 64), read back by
                             tcgen05.ld; query tiles of up to 32 rows (T_m)                 */
  LA_ENGINE_AUTO = 2      /* tcgen05 where it applies (bf16 / fp16, d = 128): tiles of more than
                             8 rows per KV head (one KV pass instead of two; static schedules)
                             and 8-row tiles of a BHSD / packed cache; mma.sync otherwise
                             (paged 8-row tiles, dynamic schedules for g * N_q > 8)          */
} la_engine;

typedef struct la_plan_s* la_plan_t;

typedef struct {
  int batch, heads_q, heads_kv, head_dim, group;
  int dtype, layout, schedule;
  int tile_n;              /* LeanTile tokens T_n                                 */
  int stage_tokens;        /* tokens per shared-memory ring stage (<= tile_n)             */
  int grid;                /* CTAs launched (persistent, <= 148 x occupancy unless static) */
  int num_units;           /* output tiles = B * H_kv                                     */
  int64_t total_iters;     /* I = sum_u ceil(n_u / T_n)  (Alg2§6, reading C15)           */
  int64_t num_segments;    /* LeanTile() calls over all CTAs (rows of la_plan_export)     */
  int64_t num_partials;    /* non-host segments = partial slots actually written          */
  int64_t workspace_bytes; /* device bytes owned by the plan                              */
  int64_t kv_bytes;        /* algorithmic K+V bytes one la_decode reads                   */
  float scale;
  int64_t num_vctas;       /* Alg. 2's G: iteration ranges (= grid for static schedules)  */
  int split;               /* LA_SCHED_FIXED_SPLIT: chunks per unit (0 otherwise)         */
  int q_len;               /* N_q (0 when per-request q_lens differ)                      */
  int tile_rows;           /* T_m: query rows per work unit                               */
  int64_t q_rows;          /* query / output rows = sum_b H_q N_b                          */
  int engine;              /* la_engine chosen for T_m > 1 tiles; -1 for the CUDA-core (MHA)
                              and FP8 engines                                                */
  double quantization_efficiency; /* I / (W x max_w LeanTiles of worker w):
                              W = the ranges of a static schedule (1.0 - 1/ceil(I/G) at worst for
                              stream-K), the persistent CTAs for dynamic / fixed split (range
                              j on CTA j mod W, the launch-order wave model)                 */
  int slot_capacity;       /* (virtual) CTA ranges the plan's device state can hold           */
  int64_t updates;         /* la_plan_update calls so far                                     */
  int sm_weighted;         /* 1: stream-K ranges follow la_plan_set_weights / la_plan_calibrate */
} la_plan_info;

/* Fill *opts with defaults.  Always LA_OK for a non-null pointer. */
la_status la_plan_opts_init(la_plan_opts* opts);

/*
 * la_plan -- build the stream-K schedule for one decode step (host, synchronous).
 *
 * batch, heads_q, heads_kv >= 1, heads_q % heads_kv == 0 (reading C3; any group size); head_dim in
 * {64, 128}; ctx_lens: HOST array of `batch` int32, each >= 1 (reading C6); tile_n: LeanTile
 * tokens in {16, 32, 64, 128, 256, 512}, or 0 for the default (T_n giving 64 KiB of K+V per
 * LeanTile -- 128 tokens at d=128 bf16, 256 at d=64, as the paper's sweep found).
 * dtype: storage type of q, k, v (LA_FP8_E4M3: E4M3 k, v codes with a bf16 q).  opts may be
 * NULL (defaults).
 *
 * Implements Alg2§4-18: units in memory order, C_n(u) = ceil(n_u / T_n), I = sum C_n,
 * per-CTA ranges by the remainder rule (reading C8), per unit the owning host CTA and the
 * last contributing CTA (reading C9).  Device plans allocate and upload the tables, G
 * partial slots of (g x d + 2) fp32 (Alg2§20-22) and G flags, and query the kernel's
 * occupancy on the current device.  On success *out receives a plan to be released with
 * la_plan_destroy.  Errors: LA_ERR_INVALID (shape/size), LA_ERR_UNSUPPORTED (head_dim,
 * dtype or group this build lacks), LA_ERR_CUDA / LA_ERR_NOMEM (device setup).
 */
la_status la_plan(int batch, int heads_q, int heads_kv, int head_dim, const int32_t* ctx_lens,
                  int tile_n, la_dtype dtype, const la_plan_opts* opts, la_plan_t* out);

/*
 * la_plan_update -- re-plan for the next decode step's context lengths (Lean Ragged
 * Batching: serving steps change ctx_lens every step) WITHOUT allocating:
 * Alg2§4-18 is re-run on the host (O(units + G)), the new tables (and block table) are
 * staged in the plan's pinned buffer and uploaded by ONE cudaMemcpyAsync on `stream`
 * (cudaStream_t; decode on the same stream, or order it after).  Everything a kernel launch
 * takes by value is independent of ctx_lens, so a CUDA graph captured around la_decode on
 * this plan replays correctly after an update (BHSD and paged layouts; a packed cache's
 * row count changes with sum n_b, so its tensor maps -- and a graph -- are re-made).
 * The CTA count launched is fixed at la_plan: min(co-resident CTAs, I at the capacity
 * lengths) -- the capacity is max_ctx for BHSD when opts.max_ctx was given,
 * pages_per_seq * page_size for paged pools, else the first plan's lengths.
 *
 * ctx_lens: HOST [batch], each in [max(1, q_lens[b]), capacity] (BHSD: <= max_ctx; paged:
 * <= pages_per_seq * page_size).  block_table: HOST [batch][pages_per_seq] for paged plans
 * (NULL keeps the current table); must be NULL otherwise.  Every other plan parameter
 * (shape, dtype, layout, schedule options, q_lens) is unchanged.  The staging buffer is
 * reused: an update first waits for the previous update's copy (long done in a decode loop).
 * Host-only plans just re-plan (la_plan_export shows the new schedule).
 * Errors: LA_ERR_INVALID (lengths / table), LA_ERR_STATE (a dynamic or fixed-split schedule
 * needs more virtual-CTA slots than allocated at la_plan -- create a new plan), LA_ERR_CUDA.
 * On error the plan is unchanged.
 */
la_status la_plan_update(la_plan_t plan, const int32_t* ctx_lens, const int32_t* block_table, void* stream);

/*
 * la_plan_set_weights -- SM-rate-weighted stream-K (B200 extension of Eq. 2).
 * Eq. 2 gives every CTA I/G LeanTiles, which balances TIME only if every SM streams at the
 * same rate; on B200 the per-SM share of HBM bandwidth under full load is not uniform (a
 * stable property of the SM: DESIGN §6), so the slowest SMs set the kernel's end.  With
 * weights w_0 .. w_{G-1} (one per CTA of the plan's LA_SCHED_STREAMK grid; blockIdx g) the
 * ranges become contiguous with boundaries
 *     cta_begin[g] = floor(I * (w_0 + .. + w_{g-1}) / (w_0 + .. + w_{G-1}))
 * (integer arithmetic; equal weights give sizes differing by at most one) -- still Alg. 2's
 * contiguous ranges, hosts and fixup, so the result is exact for any weights and
 * bitwise reproducible for fixed weights.  The weights persist across la_plan_update.
 * weights: HOST [n] int32 in [1, 2^20], n == la_plan_info.grid; NULL restores equal ranges.
 * The new tables are uploaded on `stream` (as la_plan_update).
 * Errors: LA_ERR_INVALID (n, range), LA_ERR_STATE (the plan's schedule is not
 * LA_SCHED_STREAMK), LA_ERR_CUDA.
 */
la_status la_plan_set_weights(la_plan_t plan, const int32_t* weights, int n, void* stream);

/*
 * la_plan_calibrate -- measure each CTA's streaming rate and set the weights from it
 * (la_plan_set_weights).  Per round, `launches` + 1 samples of 3 back-to-back la_decode
 * calls on the given (device) tensors on `stream`, the last of each traced (a temporary
 * device buffer if the plan has none; the first sample is a warm-up): time_g =
 * t_stream_end - t_start of CTA g summed over the samples, then w_g <- w_g * (mean time /
 * time_g) (rate-proportional shares), so the CTAs finish streaming together.  out / lse receive the last launch's (correct) result.
 * Synchronises the device.  LA_SCHED_STREAMK plans without a cross-GPU exchange only
 * (LA_ERR_STATE otherwise: an exchange plan's launches wait for its peers' -- calibrate an
 * exchange-free plan of the same shape and pass its range lengths -- la_plan_export -- to
 * la_plan_set_weights);
 * launches, rounds >= 1.  Weights are a property of the GPU's SMs: calibrate once per plan
 * (la_plan_update keeps them).
 */
la_status la_plan_calibrate(la_plan_t plan, const void* q, const void* k_cache, const void* v_cache, float* out,
                            float* lse, int launches, int rounds, void* stream);

/* Scalar facts about a plan (host, synchronous). */
la_status la_plan_info_get(la_plan_t plan, la_plan_info* info);

/*
 * la_plan_export -- dump the schedule, one row of 7 int32 per segment (= LeanTile call),
 * in SPEC's dump order: cta, unit, local_begin, local_end, host, finishing,
 * last_cta (Alg2§11-18, §26 with reading C9); cta / last_cta are (virtual) CTA indices.  rows: HOST buffer of cap_rows * 7 int32 (may
 * be NULL with cap_rows = 0 to query the count); *n_rows receives the total row count.
 * LA_ERR_INVALID if cap_rows is non-zero but too small.
 */
la_status la_plan_export(la_plan_t plan, int32_t* rows, size_t cap_rows, size_t* n_rows);

/*
 * la_plan_export_claims -- the order in which the persistent CTAs take the (virtual) CTA
 * ranges: claim c runs range claims[c] (LA_SCHED_DYNAMIC: every head, then the tail chunks
 * round by round; the other schedules: 0, 1, 2, ...).  HOST buffer of cap int32 (NULL with
 * cap = 0 queries the count into *n).  LA_ERR_INVALID if cap is non-zero but too small.
 */
la_status la_plan_export_claims(la_plan_t plan, int32_t* claims, size_t cap, size_t* n);

/*
 * la_decode -- one decode-attention step on `stream` (asynchronous).
 *
 * q: device (B, H_q, d) of the plan's dtype (bf16 for LA_FP8_E4M3), contiguous.  k_cache, v_cache: device, plan's
 * layout and dtype, contiguous, 16-byte aligned.  out: device (B, H_q, d) fp32.  lse:
 * device (B, H_q) fp32 natural-log logsumexp L, or NULL to skip it.  ctx_lens are the
 * plan's (a serving loop re-plans when they change; planning is O(B*H_kv + G)).
 * One kernel launch; it may be captured into a CUDA graph and replayed (the Signal/Wait
 * epoch lives in the plan's device memory), one launch of a plan in flight at a time.
 * Errors: LA_ERR_INVALID (null or misaligned pointer), LA_ERR_STATE (host-only plan),
 * LA_ERR_CUDA (launch failure).
 */
la_status la_decode(la_plan_t plan, const void* q, const void* k_cache, const void* v_cache,
                    float* out, float* lse, void* stream);

/*
 * la_decode_partial -- la_decode on one sequence shard of the KV cache (BASELINE.json
 * north star, multi-GPU): identical computation, `lse` is mandatory because the shard's
 * (O_r, L_r) is then combined across ranks with la_combine.  On a plan with a cross-GPU
 * exchange (opts.xchg_world > 1) it returns this shard's partial only (no exchange).
 */
la_status la_decode_partial(la_plan_t plan, const void* q, const void* k_shard,
                            const void* v_shard, float* o_part, float* lse_part, void* stream);

/*
 * la_combine -- fold P normalised partials with the softmax re-scaling operator (§4.1,
 * P:286-294, exact for any split by associativity P:264), in ascending part order:
 *     L = ln sum_r e^{L_r},  O = sum_r e^{L_r - L} O_r
 * o_parts: device [parts][rows][head_dim] fp32; lse_parts: device [parts][rows] fp32;
 * out: device [rows][head_dim] fp32; lse: device [rows] fp32 or NULL.  head_dim in
 * {64, 128}; parts >= 1; rows >= 1.  Asynchronous on `stream`.
 */
la_status la_combine(const float* o_parts, const float* lse_parts, int parts, int rows,
                     int head_dim, float* out, float* lse, void* stream);

/*
 * la_combine_strided -- la_combine with part p's O at o_parts + p * o_part_stride and its L
 * at lse_parts + p * lse_part_stride (floats): a rank's (O_r, L_r) packed in ONE buffer
 * [rows * head_dim + rows] is exchanged by ONE all-gather and combined in place
 * (o_part_stride = lse_part_stride = rows * (head_dim + 1), lse_parts = o_parts + rows * head_dim).
 * Strides must be >= one part (LA_ERR_INVALID).
 */
la_status la_combine_strided(const float* o_parts, int64_t o_part_stride, const float* lse_parts,
                             int64_t lse_part_stride, int parts, int rows, int head_dim, float* out, float* lse,
                             void* stream);

/*
 * la_decode_host -- la_decode through HOST buffers (end-to-end path): copies q, k, v
 * (plan's layout; sizes from the plan) host->device into plan-owned staging buffers
 * (allocated on first use, kept until la_plan_destroy), decodes, copies out (and lse if
 * non-NULL) device->host, and synchronises `stream`.  Host buffers should be pinned for
 * full PCIe/NVLink-C2C bandwidth.  kv_rows: total rows of one cache (B*H_kv*max_ctx for
 * BHSD, H_kv*sum n for PACKED) -- checked against the plan.
 */
la_status la_decode_host(la_plan_t plan, const void* q, const void* k_cache, const void* v_cache,
                         int64_t kv_rows, float* out, float* lse, void* stream);

/*
 * la_plan_trace -- per-CTA timeline of the most recent la_decode on a plan created with
 * opts.trace = 1 (SURVEY §5 tracing; the E2 SM-balance analog of P:191).  Synchronises the
 * device.  out: HOST buffer of cap_ctas * LA_TRACE_FIELDS uint64, one record per CTA:
 * smid, t_start, t_publish (non-host partial signalled, Alg2§23; for a static waiting host:
 * its peers' partials folded; 0 if none), t_wait_begin,
 * t_wait_end (host fold wait, Alg2§28; 0 if none), t_end -- %globaltimer nanoseconds.
 * LA_SCHED_DYNAMIC / FIXED_SPLIT: t_publish = when the epilogue took the CTA's last segment,
 * t_wait_begin / t_wait_end = claims taken / LeanTiles streamed (counts, not times).
 * Field 6, every schedule: t_stream_end = when the epilogue took the CTA's last segment
 * (its consumers had streamed every LeanTile of its range(s); 0 if it had none) -- the
 * per-CTA streaming time t_stream_end - t_start is what la_plan_calibrate measures.
 * *n_ctas receives G.  LA_ERR_STATE if the plan has no trace buffer.
 */
#define LA_TRACE_FIELDS 7
la_status la_plan_trace(la_plan_t plan, uint64_t* out, size_t cap_ctas, size_t* n_ctas);

/*
 * Fused cross-GPU fixup: Alg. 2's in-kernel fixup (Alg2§19-36) extended
 * across the NVLink domain for a sequence-sharded decode.  Rank r's plan covers its shard
 * of every request's context (same batch, heads, head_dim, dtype, q_len on every rank).
 * When the kernel has reduced unit u (b, h_kv) on its shard, the CTA that would write the
 * output instead pushes the normalised shard partial (O_r, L_r) of the unit's rows into
 * EVERY rank's exchange buffer (plain stores to peer HBM over NVLink), releases flag
 * [r][u] there (st.release.sys), then acquires the P flags [*][u] in its own buffer and
 * folds the P partials with the §4.1 operator in ascending rank order -- bitwise the same
 * result on every rank, no NCCL launch and no combine kernel.  Exact by associativity
 * (P:264).  Buffers are double-buffered by launch parity, so ranks may run one launch
 * apart.  Every rank must issue the same sequence of la_decode calls.
 *
 * la_plan_xchg_handle: the CUDA IPC handle (LA_XCHG_HANDLE_BYTES bytes into `handle`) of
 *   this plan's exchange buffer, to be sent to the other ranks (e.g. all_gather_object).
 * la_plan_xchg_open: map peer `peer`'s buffer from its handle (cudaIpcOpenMemHandle; the
 *   peer must live in another process on a peer-accessible GPU).
 * la_plan_xchg_attach: use the buffer of `peer_plan` (same process) as rank `peer`'s --
 *   for one process driving several GPUs with peer access enabled, or several "ranks"
 *   sharing one GPU (tests).
 * la_decode on an exchange plan needs every peer opened/attached (LA_ERR_STATE otherwise).
 * la_plan_xchg_status: la_plan_status on an exchange plan (LA_ERR_STATE without one).
 * la_plan_xchg_open checks the peer's shape header (batch, heads, head_dim, dtype, rows,
 *   units, world, rank) written into its buffer at la_plan: LA_ERR_INVALID on a mismatch.
 * LA_SCHED_DYNAMIC on an exchange plan claims its ranges in iteration order (no tail chunks):
 *   deadlock freedom needs every CTA to visit units in increasing order.
 * The exchange flags carry an exchange sequence number that only exchange launches
 *   advance (la_decode_partial on the plan does not), and waits compare wrap-safe.
 * Requires q_len == 1 or causal == 0 (a causal multi-token mask is not shard-local).
 */
#define LA_XCHG_HANDLE_BYTES 64
la_status la_plan_xchg_handle(la_plan_t plan, void* handle);
la_status la_plan_xchg_open(la_plan_t plan, int peer, const void* handle);
la_status la_plan_xchg_attach(la_plan_t plan, int peer, la_plan_t peer_plan);
la_status la_plan_xchg_status(la_plan_t plan);

/*
 * la_plan_status -- synchronises the device and reports whether an in-kernel wait of a
 * previous launch on this plan gave up: a stream-K host CTA waiting for a peer's partial
 * (Alg2§28, 10 s) or a cross-GPU exchange wait (5 s).  LA_ERR_TIMEOUT (the output of that
 * launch is invalid; the error is cleared), LA_ERR_STATE for a host-only plan, else LA_OK.
 * A protocol failure therefore surfaces as an error instead of hanging the device.
 */
la_status la_plan_status(la_plan_t plan);

/* Release a plan and all device memory it owns.  NULL is a no-op. */
void la_plan_destroy(la_plan_t plan);

/* Kernel launches issued by this library since load (for the bench's gpu_launches). */
int64_t la_launch_count(void);

const char* la_status_string(la_status s);
const char* la_last_error(void);
int la_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LEANATTN_LA_H */
