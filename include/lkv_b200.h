/*
 * lkv_b200.h -- C ABI of the B200-native LKV inference-time eviction path.
 *
 * This is the drop-in boundary: plain pointers, sizes and POD descriptors, no
 * C++ or torch types.  It replaces the reference's C++ hot-path API in
 * /root/reference/proj/include/lkv (all calls there are host-side, synchronous,
 * fp64, exception-throwing):
 *
 *   lkv_budgets     <- allocate_budgets   policy.hpp:67  (policy.cpp:110-120)
 *                      + freeze_budgets   policy.hpp:70  (policy.cpp:122-129)
 *                      (+ soft_topk_forward / solve_threshold soft_topk.hpp:57-60)
 *   lkv_score       <- token_scores       policy.hpp:73  (policy.cpp:131-136)
 *   lkv_select      <- inference_select   policy.hpp:81  (policy.cpp:152-154)
 *                      -> hard_topk       soft_topk.hpp:71 (soft_topk.cpp:191-201)
 *   lkv_compact     <- the compaction loop of prefill_with_eviction (evictsim.cpp:202-215)
 *   lkv_cache_from_trace <- cache_from_trace model.hpp:99 (model.cpp:289-315): mask scan + gather
 *   lkv_evict       <- prefill_with_eviction's score->select->compact loop
 *                      (evictsim.hpp:74, evictsim.cpp:161-215), K/V-given form
 *   lkv_evict_host  <- the same, for a cache resident in (pinned) host memory
 *   lkv_evict_shard <- the same on one rank's head shard (multi-GPU; lkv_comm_* = NCCL)
 *   lkv_decode_step <- decode_step's append + attention block (model.hpp:95,
 *                      model.cpp:240-265) -> masked_attention_dense (attention.hpp:57)
 *   lkv_soft_topk_fwd/_vjp <- soft_topk_forward / soft_topk_vjp (soft_topk.hpp:60-67;
 *                      training)
 *   lkv_masked_attention_fwd/_bwd <- masked_attention_dense / masked_attention_vjp
 *                      (attention.hpp:57-69; training)
 *   lkv_model_*     <- the whole decode_step (model.hpp:95, model.cpp:209-287):
 *                      projections, RoPE at tokens_seen, attention, SwiGLU MLP, logits
 *
 * Status codes map 1:1 onto the reference's exception types
 * (proj/include/lkv/errors.hpp:10-32); lkv_last_error() returns a thread-local
 * message.  Every entry point is stream-ordered and asynchronous: host-side
 * validation errors return immediately; device-side errors (non-finite scores,
 * budgets outside [0, t], solve failures) are latched into the caller's
 * workspace and returned by lkv_workspace_status(), which synchronises.
 *
 * Memory: the library never allocates or frees caller memory; every device
 * buffer is caller-owned.  Dense caches are head-major
 *   keys/values [n_seq][n_layers][n_kv_heads][max_tokens][head_dim]
 * and a flat head id is (s * n_layers + l) * n_kv_heads + h.  The ragged
 * (compacted) cache stores head i's rows at [offsets[i], offsets[i] + lens[i])
 * with capacity offsets[i+1] - offsets[i] = budget_i + decode_slack.
 *
 * Target: NVIDIA B200 (sm_100a).  Built with nvcc -gencode arch=compute_100a,code=sm_100a.
 */
#ifndef LKV_B200_H
#define LKV_B200_H

#include <stddef.h>
#include <stdint.h>

/* the library is built with -fvisibility=hidden: only what this header declares is exported */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif
#ifdef __cplusplus
extern "C" {
#endif

#define LKV_ABI_VERSION 2
#define LKV_MAX_SEQ 256

typedef struct CUstream_st* lkv_stream_t; /* identical to cudaStream_t */

typedef enum lkv_status {
    LKV_OK = 0,
    LKV_ERR_CONTRACT = 1,        /* lkv::contract_error        errors.hpp:10-12 */
    LKV_ERR_NUMERIC = 2,         /* lkv::numeric_error         errors.hpp:15-17 */
    LKV_ERR_BUDGET = 3,          /* lkv::budget_error          errors.hpp:20-22 */
    LKV_ERR_OVERFLOW_GUARD = 4,  /* lkv::overflow_guard_error  errors.hpp:25-27 */
    LKV_ERR_DEGENERATE_MASK = 5, /* lkv::degenerate_mask_error errors.hpp:30-32 */
    LKV_ERR_CUDA = 6,            /* CUDA runtime / launch failure (no reference analogue) */
    LKV_ERR_UNSUPPORTED = 7,     /* device is not sm_100 or shape outside the kernel envelope */
    LKV_ERR_NCCL = 8             /* NCCL missing or a collective failed (multi-GPU plumbing only) */
} lkv_status;

typedef enum lkv_dtype { LKV_F32 = 0, LKV_BF16 = 1, LKV_F64 = 2 /* gather-only: lkv_compact / cache_from_trace */ } lkv_dtype;
typedef enum lkv_activation { LKV_ACT_SILU = 0, LKV_ACT_GELU_ERF = 1 } lkv_activation;
typedef enum lkv_scorer_input {
    LKV_SCORER_K = 1,  /* x = k            (BASELINE.json configs: head_dim -> hidden -> 1) */
    LKV_SCORER_KV = 2  /* x = [k ; v]      (reference: policy.cpp:135, 2d -> d -> 1)        */
} lkv_scorer_input;
typedef enum lkv_budget_mode {
    LKV_BUDGET_FLOOR = 0, /* freeze_budgets: floor(r * t), policy.cpp:126              */
    LKV_BUDGET_EXACT = 1  /* floor + largest-remainder fix-up to llround(R * n * t)     */
} lkv_budget_mode;

/* Dense, pre-eviction cache (K already post-RoPE, evictsim.cpp:143). */
typedef struct lkv_cache_desc {
    int32_t n_seq;       /* 1 .. LKV_MAX_SEQ */
    int32_t n_layers;
    int32_t n_kv_heads;
    int32_t head_dim;    /* multiple of 8 */
    int64_t max_tokens;  /* T: row capacity per head in keys/values */
    int32_t dtype;       /* lkv_dtype */
    int32_t _pad;
    const void* keys;    /* device */
    const void* values;  /* device */
    const int32_t* seq_lens; /* HOST [n_seq], 1 <= t_s <= max_tokens */
} lkv_cache_desc;

/* LKV-T token scorers u = act(x W1 + b1) . w2 (policy.hpp:24-32, no output bias). */
typedef struct lkv_scorer_desc {
    int32_t input;        /* lkv_scorer_input */
    int32_t activation;   /* lkv_activation */
    int32_t hidden;       /* 1..256; the tensor-core path needs a multiple of 16 */
    int32_t n_scorers;
    int32_t stride_layer; /* scorer id of (l, h) = l * stride_layer + h * stride_head */
    int32_t stride_head;  /*   per-(l,h): (n_kv_heads, 1); per-layer: (1, 0)          */
    const void* w1t;      /* device [n_scorers][hidden][in] in the cache dtype (W1 transposed) */
    const float* b1;      /* device [n_scorers][hidden] */
    const float* w2;      /* device [n_scorers][hidden] */
} lkv_scorer_desc;

/* Ragged compacted cache (KvCache/HeadCache, model.hpp:55-71). */
typedef struct lkv_ragged_desc {
    int32_t n_heads;       /* n_seq * n_layers * n_kv_heads */
    int32_t head_dim;
    int32_t dtype;
    int32_t decode_slack;  /* rows reserved per head for decode appends */
    int64_t capacity_rows; /* rows allocated in keys/values/positions */
    int64_t* offsets;      /* device [n_heads + 1] */
    int32_t* lens;         /* device [n_heads]: rows currently held */
    void* keys;            /* device [capacity_rows][head_dim] */
    void* values;          /* device [capacity_rows][head_dim] */
    int32_t* positions;    /* device [capacity_rows]: original token index, strictly increasing */
} lkv_ragged_desc;

/* ---- library / errors -------------------------------------------------- */
int lkv_abi_version(void);
/* Number of CUDA kernels this library has launched in the process (bench accounting). */
uint64_t lkv_launch_count(void);
const char* lkv_last_error(void);
const char* lkv_status_name(int status);
/* LKV_OK when the current device is sm_100 (B200); LKV_ERR_UNSUPPORTED otherwise. */
lkv_status lkv_device_check(void);

/* Workspace: one caller-owned device buffer per in-flight call chain.  Its
 * first bytes latch device-side errors.  lkv_workspace_status synchronises
 * `stream`, returns the latched status (and clears it). */
size_t lkv_workspace_bytes(const lkv_cache_desc* cache, int32_t n_logits);
lkv_status lkv_workspace_init(void* workspace, size_t bytes, lkv_stream_t stream);
lkv_status lkv_workspace_status(void* workspace, lkv_stream_t stream);

/* Total rows a ragged cache needs (exact in LKV_BUDGET_EXACT mode, an upper
 * bound in FLOOR mode): sum_s llround(R * n * t_s) + n_heads * decode_slack. */
int64_t lkv_ragged_capacity(const lkv_cache_desc* cache, double target_ratio, int32_t decode_slack);

/* ---- K2: LKV-H budgets -------------------------------------------------- */
/* ratios = soft_topk(logits, k = R*n, tau = 1) (fp64, the reference's exact
 * operation order); budgets[s*n + i] = freeze(ratios_i, seq_lens[s]) per mode;
 * offsets (nullable) = exclusive scan of (budget + decode_slack), length
 * n_seq*n + 1.  logits: device fp64 [n]; ratios (nullable): device fp64 [n].
 * R outside (0,1) -> LKV_ERR_BUDGET. */
lkv_status lkv_budgets(const double* logits, int32_t n, double target_ratio, int32_t mode,
                       const int32_t* seq_lens, int32_t n_seq, int32_t decode_slack,
                       double* ratios, int32_t* budgets, int64_t* offsets,
                       void* workspace, size_t workspace_bytes, lkv_stream_t stream);

/* freeze_budgets on an existing ratio table (policy.cpp:122-129): ratios device fp64 [n]
 * -> budgets [n_seq * n] per mode (EXACT needs target_ratio in (0,1)); offsets nullable. */
lkv_status lkv_freeze_budgets(const double* ratios, int32_t n, double target_ratio, int32_t mode,
                              const int32_t* seq_lens, int32_t n_seq, int32_t decode_slack,
                              int32_t* budgets, int64_t* offsets, void* workspace,
                              size_t workspace_bytes, lkv_stream_t stream);

/* Exclusive scan of (budgets[i] + decode_slack) -> offsets[n_heads+1] (device). */
lkv_status lkv_ragged_offsets(const int32_t* budgets, int32_t n_heads, int32_t decode_slack,
                              int64_t* offsets, lkv_stream_t stream);

/* ---- K1: LKV-T scorer ------------------------------------------------------ */
/* scores: device fp32 [n_heads][max_tokens]; rows >= t_s are left untouched.
 * bf16 + head_dim 128 + hidden % 16 == 0 runs on tcgen05 tensor cores (TMA ->
 * SMEM -> UMMA -> TMEM, activation and w2 reduction fused in the epilogue);
 * other shapes run a SIMT kernel (fp32 inputs always do: TF32 would break the
 * 1e-5 parity bar). */
lkv_status lkv_score(const lkv_cache_desc* cache, const lkv_scorer_desc* scorer, float* scores,
                     void* workspace, size_t workspace_bytes, lkv_stream_t stream);

/* ---- K3: per-head top-k ----------------------------------------------------- */
/* For every head keep the budgets[i] largest scores (ties -> lowest index,
 * -0.0 == +0.0, NaN -> LKV_ERR_NUMERIC, budget outside [0, t] -> LKV_ERR_BUDGET),
 * writing their positions ascending to out->positions[offsets[i] ...] and
 * out->lens[i] = budgets[i].  out->offsets must already be filled.  With
 * gather != 0 the kept K/V rows are also copied into out->keys/values in the
 * same pass (fused K3 + K4; needs cache->keys/values). */
lkv_status lkv_select(const lkv_cache_desc* cache, const float* scores, const int32_t* budgets,
                      const lkv_ragged_desc* out, int32_t gather, void* workspace, size_t workspace_bytes,
                      lkv_stream_t stream);

/* ---- K4: compaction ---------------------------------------------------------- */
/* Gathers rows positions[offsets[i] + r], r < lens[i], of head i from the dense
 * cache into out->keys/values[offsets[i] + r] (16-byte vectorised).  A position outside
 * [0, t_s) or lens overrunning a head's capacity is a contract_error (model.cpp:298-312),
 * latched in `workspace` (>= 256 bytes, lkv_workspace_status); those rows are not written. */
lkv_status lkv_compact(const lkv_cache_desc* cache, const lkv_ragged_desc* out, void* workspace,
                       size_t workspace_bytes, lkv_stream_t stream);

/* cache_from_trace (model.hpp:99, model.cpp:289-315) on the device: keep row j < t_s of flat
 * head i iff masks[i * mask_ld + j] != 0, ascending (the reference's `if (!m[j]) continue`).
 * lkv_mask_counts writes the kept rows per head (to size the ragged cache);
 * lkv_cache_from_trace writes out->lens, out->offsets (exclusive scan of count +
 * decode_slack), the positions and the gathered K/V rows.  A ragged cache too small for the
 * counts is a contract_error (latched; nothing is written for that head).  Workspace as
 * lkv_workspace_bytes(cache, 1); mask_ld >= max t_s. */
lkv_status lkv_mask_counts(const lkv_cache_desc* cache, const int32_t* masks, int64_t mask_ld, int32_t* counts,
                           void* workspace, size_t workspace_bytes, lkv_stream_t stream);
lkv_status lkv_cache_from_trace(const lkv_cache_desc* cache, const int32_t* masks, int64_t mask_ld,
                                const lkv_ragged_desc* out, void* workspace, size_t workspace_bytes,
                                lkv_stream_t stream);

/* ---- fused: budgets -> score -> select -> compact ----------------------------- */
/* scores_out, ratios_out, budgets_out may be NULL (workspace-backed). */
lkv_status lkv_evict(const lkv_cache_desc* cache, const lkv_scorer_desc* scorer, const double* logits,
                     double target_ratio, int32_t mode, const lkv_ragged_desc* out, float* scores_out,
                     double* ratios_out, int32_t* budgets_out, void* workspace, size_t workspace_bytes,
                     lkv_stream_t stream);

/* score -> select -> compact with budgets given (no LKV-H solve): the per-layer step of the
 * layer-wise prefill (evictsim.cpp:161-215 with the budgets of policy_budget_table) or budgets
 * from an external source (export-budgets CSV, tools/lkv.cpp:154-177).  out->offsets must hold the
 * exclusive scan of budget + decode_slack (lkv_ragged_offsets / lkv_budgets); workspace as
 * lkv_workspace_bytes(cache, 1). */
lkv_status lkv_evict_budgets(const lkv_cache_desc* cache, const lkv_scorer_desc* scorer, const int32_t* budgets,
                             const lkv_ragged_desc* out, float* scores_out, void* workspace, size_t workspace_bytes,
                             lkv_stream_t stream);

/* ---- fused, from a host-resident cache ------------------------------------------ */
/* The same eviction for a dense cache held in pinned, device-mapped host memory
 * (cudaHostAlloc / cudaHostRegister mapped): host_cache->keys/values are host pointers.
 * K is uploaded into dev_keys (device, dense shape) in (sequence, layers_per_chunk-layer)
 * chunks on a library copy stream, pipelined with scoring; the kept V rows are gathered
 * straight from host memory (only the retained fraction of V crosses PCIe); with [k;v]
 * scorers V is uploaded into dev_values too.  Each chunk is scored, selected and gathered
 * as soon as its K has landed.  host_out (nullable, pinned) receives the compacted cache
 * chunk by chunk on a third (device->host) stream while later chunks still upload; to size
 * those copies the call waits once on the host for the budget solve's ragged offsets (all
 * uploads are queued first, so the wait overlaps the transfer).  Everything else is ordered
 * on `stream`. */
lkv_status lkv_evict_host(const lkv_cache_desc* host_cache, void* dev_keys, void* dev_values,
                          const lkv_scorer_desc* scorer, const double* logits, double target_ratio,
                          int32_t mode, const lkv_ragged_desc* out, const lkv_ragged_desc* host_out,
                          int32_t layers_per_chunk, void* workspace, size_t workspace_bytes,
                          lkv_stream_t stream);

/* ---- head shards (multi-GPU: one process per GPU) -------------------- */
/* A rank owns a contiguous range of flat per-sequence heads [head_begin, head_begin +
 * n_layers*n_kv_heads) -- i.e. a layer range -- of every sequence; its local cache/scorers
 * describe only those layers.  LKV-H is one Soft-TopK over ALL n_logits heads
 * (policy.cpp:110-120), so every rank solves it redundantly from the full logit vector (see
 * lkv_comm_allgatherv) and freezes every head's budget bit-identically; only its own heads'
 * budgets ([n_seq][n_local]) and ragged offsets are kept. */
lkv_status lkv_budgets_shard(const double* logits, int32_t n_logits, double target_ratio, int32_t mode,
                             const int32_t* seq_lens, int32_t n_seq, int32_t decode_slack, int32_t head_begin,
                             int32_t n_local, double* ratios, int32_t* budgets_all, int32_t* budgets_local,
                             int64_t* offsets_local, void* workspace, size_t workspace_bytes, lkv_stream_t stream);
/* lkv_evict on a head shard; the workspace is lkv_workspace_bytes(local_cache, n_logits). */
lkv_status lkv_evict_shard(const lkv_cache_desc* local_cache, const lkv_scorer_desc* scorer, const double* logits,
                           int32_t n_logits, int32_t head_begin, double target_ratio, int32_t mode,
                           const lkv_ragged_desc* out, float* scores_out, double* ratios_out, int32_t* budgets_out,
                           void* workspace, size_t workspace_bytes, lkv_stream_t stream);
/* lkv_evict_host on a head shard (host_cache holds this rank's layers only; pinned + mapped). */
lkv_status lkv_evict_host_shard(const lkv_cache_desc* host_cache, void* dev_keys, void* dev_values,
                                const lkv_scorer_desc* scorer, const double* logits, int32_t n_logits,
                                int32_t head_begin, double target_ratio, int32_t mode, const lkv_ragged_desc* out,
                                const lkv_ragged_desc* host_out, int32_t layers_per_chunk, void* workspace,
                                size_t workspace_bytes, lkv_stream_t stream);
/* Shards that own an arbitrary list of heads (LPT placement by budget, shard.lpt_assign): the
 * local cache holds them per sequence in list order, grouped any way as n_layers x n_kv_heads =
 * n_local (e.g. groups of H, so lkv_evict_host_heads still uploads per group), and head_ids
 * (DEVICE int32 [n_local]) gives local head j = l * n_kv_heads + h its global flat index; the scorer
 * table is indexed by local head (stride_layer = n_kv_heads, stride_head = 1).  K2 still solves all
 * n_logits heads (bit-identical on every rank); budgets_local / offsets_local follow the list order. */
lkv_status lkv_budgets_heads(const double* logits, int32_t n_logits, double target_ratio, int32_t mode,
                             const int32_t* seq_lens, int32_t n_seq, int32_t decode_slack, const int32_t* head_ids,
                             int32_t n_local, double* ratios, int32_t* budgets_all, int32_t* budgets_local,
                             int64_t* offsets_local, void* workspace, size_t workspace_bytes, lkv_stream_t stream);
lkv_status lkv_evict_heads(const lkv_cache_desc* local_cache, const lkv_scorer_desc* scorer, const double* logits,
                           int32_t n_logits, const int32_t* head_ids, double target_ratio, int32_t mode,
                           const lkv_ragged_desc* out, float* scores_out, double* ratios_out, int32_t* budgets_out,
                           void* workspace, size_t workspace_bytes, lkv_stream_t stream);
lkv_status lkv_evict_host_heads(const lkv_cache_desc* host_cache, void* dev_keys, void* dev_values,
                                const lkv_scorer_desc* scorer, const double* logits, int32_t n_logits,
                                const int32_t* head_ids, double target_ratio, int32_t mode, const lkv_ragged_desc* out,
                                const lkv_ragged_desc* host_out, int32_t layers_per_chunk, void* workspace,
                                size_t workspace_bytes, lkv_stream_t stream);
/* Upper bound on a shard's compacted rows (caller allocates; -1 on bad input). */
int64_t lkv_ragged_capacity_shard(const lkv_cache_desc* local_cache, int32_t n_logits, double target_ratio,
                                  int32_t decode_slack);

/* NCCL over NVLink/NVSwitch (resolved at run time from libnccl.so.2).  The path's only
 * exchanges: the LKV-H logits (allgatherv, a few KB) and the decode outputs (gatherv to a
 * root, or allgatherv), both latency-bound.  Byte counts/displacements are per rank. */
#define LKV_COMM_ID_BYTES 128
typedef struct lkv_comm_s* lkv_comm_t;
lkv_status lkv_comm_get_unique_id(void* id /* LKV_COMM_ID_BYTES */);
lkv_status lkv_comm_init(lkv_comm_t* comm, const void* id, int32_t n_ranks, int32_t rank);
lkv_status lkv_comm_destroy(lkv_comm_t comm);
int32_t lkv_comm_size(lkv_comm_t comm);
int32_t lkv_comm_rank(lkv_comm_t comm);
lkv_status lkv_comm_allgatherv(lkv_comm_t comm, const void* send, void* recv, const int64_t* bytes,
                               const int64_t* displs, lkv_stream_t stream);
lkv_status lkv_comm_gatherv(lkv_comm_t comm, const void* send, void* recv, const int64_t* bytes,
                            const int64_t* displs, int32_t root, lkv_stream_t stream);

/* ---- training-time operators ---------------------------------- */
/* Multiplicative soft-mask attention, forward and backward: masked_attention_dense /
 * masked_attention_vjp (attention.hpp:52-69, attention.cpp:46-201) for a batch of heads with
 * GQA (query head h reads kv head h / (n_q_heads / n_kv_heads)); the per-query-head calls of
 * forward_masked (model.cpp:100-112) in one launch.  Layouts: q, out, d_out
 * [batch][n_q_heads][t_q][head_dim]; k, v [batch][n_kv_heads][t_k][head_dim] (dtype);
 * mask [batch][n_kv_heads][t_k] fp32 or NULL (all ones); lse [batch][n_q_heads][t_q] fp32
 * (log2-domain masked log-sum-exp of scale * q.k, saved by the forward for the backward);
 * gradients fp32, dk/dv/dmask summed over the query heads of a group.  bf16 needs
 * head_dim 128 (tensor cores); fp32 runs the exact SIMT path (head_dim <= 256).  Errors:
 * mask value < 0 or non-finite -> CONTRACT, a row whose masked mass vanishes ->
 * DEGENERATE_MASK (both latched in the workspace). */
/* Soft-TopK over n_seg independent segments of n scores (row stride ld):
 * soft_topk_forward (soft_topk.hpp:60, soft_topk.cpp:111-164) with k[seg] in (0, n), tau > 0;
 * optional noise: scores are x + noise_scale * noise (training_mask, policy.cpp:138-150).
 * Outputs values [n_seg][ld] (fp64), density (the VJP's saved state, nullable), values_f32
 * (nullable: an fp32 copy usable directly as the masked-attention mask) and lambda [n_seg]
 * (nullable).  Device-side errors: k outside (0, n) -> BUDGET, non-finite score -> NUMERIC,
 * |score| > 1e300 -> OVERFLOW_GUARD, constraint |sum - k| > 1e-9 n -> NUMERIC.
 * lkv_soft_topk_vjp: soft_topk_vjp (soft_topk.cpp:166-189) -> grad_x [n_seg][ld], grad_k [n_seg].
 * Workspace: >= 256 bytes (the error latch). */
lkv_status lkv_soft_topk_fwd(const double* x, const double* noise, double noise_scale, int32_t n_seg, int32_t n,
                             int64_t ld, const double* k, double tau, double* values, double* density,
                             float* values_f32, double* lambda, void* workspace, size_t workspace_bytes,
                             lkv_stream_t stream);
lkv_status lkv_soft_topk_vjp(const double* density, const double* upstream, int32_t n_seg, int32_t n, int64_t ld,
                             double tau, double* grad_x, double* grad_k, lkv_stream_t stream);

typedef struct lkv_attn_desc {
    int32_t batch, n_q_heads, n_kv_heads, t_q, t_k, head_dim, dtype;
    int32_t causal;               /* row r admits keys j <= query_pos_offset + r */
    int32_t query_pos_offset;
    int32_t self_always_retained; /* key j == query_pos_offset + r keeps multiplier 1 */
    double scale;
} lkv_attn_desc;
size_t lkv_attn_workspace_bytes(const lkv_attn_desc* attn);
lkv_status lkv_masked_attention_fwd(const lkv_attn_desc* attn, const void* q, const void* k, const void* v,
                                    const float* mask, void* out, float* lse, void* workspace,
                                    size_t workspace_bytes, lkv_stream_t stream);
lkv_status lkv_masked_attention_bwd(const lkv_attn_desc* attn, const void* q, const void* k, const void* v,
                                    const float* mask, const void* out, const float* lse, const void* d_out,
                                    float* dq, float* dk, float* dv, float* dmask, void* workspace,
                                    size_t workspace_bytes, lkv_stream_t stream);

/* ---- fp64 reference-precision operators --------------------------------------------- */
/* The reference computes in float64 (tensor.hpp:3).  These device operators back the
 * declaration-compatible C++ API (include/lkv/ headers), which keeps the reference's signatures and
 * precision: the LKV-H solve with its outputs (lambda, split m, density, permutation), the LKV-T
 * scorer, top-b selection on fp64 scores, and the toy GQA model's forward / decode operators.
 * Each output element is computed in an order independent of the number of rows in the call, so
 * a t-row prefill and a one-row decode agree bit for bit.  All row-major, device pointers. */

/* soft_topk_forward (soft_topk.hpp:60, soft_topk.cpp:111-164) with the reference's exact solve
 * (solve_threshold :58-109): values [n], density [n], permutation [n] (stable descending order of
 * x), lambda, split_m, clamped_k (each nullable but values).  Device-side errors latch: k outside
 * (0, n) -> BUDGET, non-finite -> NUMERIC, |x/tau| > 1e300 (n >= 2) -> OVERFLOW_GUARD, no bracket
 * -> NUMERIC. */
lkv_status lkv_soft_topk_exact(const double* x, int32_t n, double k, double tau, double* values, double* density,
                               int32_t* permutation, double* lambda, int32_t* split_m, double* clamped_k,
                               void* workspace, size_t workspace_bytes, lkv_stream_t stream);
/* C[M x N] (+)= A[M x K] B[K x N] (matmul, tensor.cpp:276-297); accumulate: C + (A B). */
lkv_status lkv_f64_gemm(int32_t M, int32_t N, int32_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
                        double* C, int64_t ldc, int32_t accumulate, lkv_stream_t stream);
/* out = x * gain / sqrt(mean(x^2) + eps) per row (rmsnorm, model.cpp:48-53) */
lkv_status lkv_f64_rmsnorm(int32_t rows, int32_t cols, const double* x, int64_t ldx, const double* gain, double eps,
                           double* out, int64_t ldo, lkv_stream_t stream);
/* rotary pairs of every head of row r at position pos0 + r, in place (rope, tensor.cpp:586-623) */
lkv_status lkv_f64_rope(int32_t rows, int32_t n_heads, int32_t head_dim, double* x, int64_t ldx, int32_t pos0,
                        double base, lkv_stream_t stream);
/* masked_attention_dense (attention.cpp:46-94) for n_q_heads query heads at once, query head h
 * reading kv head h / group; p_raw / p [n_q_heads][n_q][t] and renorm [n_q_heads][n_q] nullable
 * (AttentionSaved).  A row whose masked mass vanishes -> DEGENERATE_MASK (latched). */
typedef struct lkv_f64_attn_desc {
    int32_t n_q_heads, group, n_q, t, head_dim;
    int32_t causal, query_pos_offset, self_always_retained;
    double scale;
    const double* q;  int64_t ldq;    /* row r, head h at q[r * ldq + h * head_dim] */
    const double* k;  const double* v; int64_t ldkv;
    const double* mask; int64_t mask_ld; /* nullable; kv head g's mask at mask[g * mask_ld + j] */
    double* out;      int64_t ldo;
    double* p_raw;    double* p;       double* renorm;
} lkv_f64_attn_desc;
lkv_status lkv_f64_attention(const lkv_f64_attn_desc* attn, void* workspace, size_t workspace_bytes,
                             lkv_stream_t stream);
/* out = silu(gate) * up (model.cpp:112-115) */
lkv_status lkv_f64_swiglu(int64_t n, const double* gate, const double* up, double* out, lkv_stream_t stream);
/* out[r] = table[tokens[r]] (embedding_rows); a token outside [0, vocab) -> CONTRACT (latched) */
lkv_status lkv_f64_embed(const int32_t* tokens, int32_t n, const double* table, int32_t d_model, int32_t vocab,
                         double* out, void* workspace, size_t workspace_bytes, lkv_stream_t stream);
/* [t][n_heads * head_dim] (row stride ldx) -> head-major [n_heads][out_rows][head_dim] */
lkv_status lkv_f64_split_heads(int32_t t, int32_t n_heads, int32_t head_dim, const double* x, int64_t ldx, double* out,
                               int64_t out_rows, lkv_stream_t stream);
/* token_scores (policy.cpp:131-136): u = act(x W1 + b1) . w2, x = [k ; v] (input KV) or k;
 * W1 [in][hidden] as the reference stores it.  A non-finite score -> NUMERIC (latched). */
lkv_status lkv_f64_token_scores(int32_t t, int32_t head_dim, int32_t input, const double* keys, int64_t ldk,
                                const double* values, int64_t ldv, const double* w1, const double* b1, const double* w2,
                                int32_t hidden, int32_t activation, double* u, void* workspace, size_t workspace_bytes,
                                lkv_stream_t stream);
/* hard_topk / inference_select (soft_topk.cpp:191-201) on fp64 scores [n_heads][ld], one budget
 * per head: the budgets[h] largest of the first t scores (ties -> lowest index, -0.0 == +0.0),
 * positions written ascending at out->offsets[h], out->lens[h] = budgets[h].  Budget outside
 * [0, t] -> BUDGET, NaN -> NUMERIC (latched).  Rows are gathered by lkv_compact (LKV_F64). */
lkv_status lkv_f64_select(const double* scores, int32_t n_heads, int32_t t, int64_t ld, const int32_t* budgets,
                          const lkv_ragged_desc* out, void* workspace, size_t workspace_bytes, lkv_stream_t stream);

/* ---- K/V production for layer-by-layer prefill (the step before the path) -------- */
/* cos/sin table [t_max][head_dim/2] of float2 (cos, sin) for positions pos_offset + p,
 * theta = pos * base^(-2j/head_dim) evaluated in fp64 (tensor.cpp:586-623, model.cpp:38-46). */
lkv_status lkv_rope_table(int32_t t_max, int32_t head_dim, double base, int32_t pos_offset, void* table,
                          lkv_stream_t stream);
/* One layer's projections, token-major [n_seq][max_tokens][n_kv_heads * head_dim] (the K/V
 * GEMM outputs) -> the dense head-major layer [n_seq][n_kv_heads][max_tokens][head_dim] that
 * lkv_score / lkv_select read, K rotated pairwise with `table` (V copied).  `layer` gives the
 * shape (n_layers must be 1); k_out / v_out receive the dense layer. */
lkv_status lkv_rope_pack(const void* k_lin, const void* v_lin, const lkv_cache_desc* layer, const void* table,
                         void* k_out, void* v_out, lkv_stream_t stream);

/* One layer's K/V production on tcgen05 tensor cores (evictsim.cpp:133-145): [k | v] = h Wkv with
 * RoPE (K only, at the absolute positions of `table`, lkv_rope_table) and the token-major ->
 * head-major pack fused into the GEMM epilogue, written straight into the dense layer k_out /
 * v_out [n_seq][n_kv_heads][max_tokens][head_dim] that lkv_score / lkv_select read (the
 * rope_pack round trip disappears).  h: [n_seq][max_tokens][d_model] bf16 (the attention-normed
 * hidden states); wkv_t: [2 * n_kv_heads * head_dim][d_model] bf16 = [Wk | Wv] transposed (K
 * output columns first).  bf16, head_dim 128, d_model % 64 == 0; fp32 accumulation. */
lkv_status lkv_kv_project(const void* h, int32_t d_model, const void* wkv_t, const lkv_cache_desc* layer,
                          const void* table, void* k_out, void* v_out, lkv_stream_t stream);

/* ---- K5: decode over the ragged cache ------------------------------------------- */
/* lkv_decode_plan splits every head's capacity into work items of 128..1024 rows (once
 * per eviction, after offsets are final).  lkv_decode_step then runs one decode
 * step for every (seq, layer): append new_k/new_v (post-RoPE) and position
 * tokens_seen[s] to each KV head (lens += 1, capacity checked), and for each
 * query head qh attend over kv = qh / (n_q_heads / n_kv_heads):
 * out = softmax(scale * q K^T) V over all lens rows (causal = false, no mask).
 * q, out: [n_seq][n_layers][n_q_heads][head_dim]; new_k/new_v:
 * [n_seq][n_layers][n_kv_heads][head_dim]; all in the cache dtype.
 * tokens_seen: device int32 [n_seq], incremented by the call.
 * bf16 requires head_dim 128 and G = n_q_heads / n_kv_heads <= 16. */
size_t lkv_decode_workspace_bytes(const lkv_ragged_desc* cache, int32_t group_size);
lkv_status lkv_decode_plan(const lkv_ragged_desc* cache, void* workspace, size_t workspace_bytes,
                           lkv_stream_t stream);
/* The same with the work-item size fixed (rows_per_item: 0 = automatic, else a multiple of 64
 * in [128, 1024]; it may still be raised so a head's chunks fit the combine's table). */
lkv_status lkv_decode_plan_ex(const lkv_ragged_desc* cache, int32_t rows_per_item, void* workspace,
                              size_t workspace_bytes, lkv_stream_t stream);
/* The plan's work-item count and size, read back from the workspace of lkv_decode_plan(_ex) or
 * lkv_model_plan(_ex) (synchronises `stream`). */
lkv_status lkv_decode_plan_info(const lkv_ragged_desc* cache, const void* workspace, int32_t* n_items,
                                int32_t* rows_per_item, lkv_stream_t stream);
lkv_status lkv_decode_step(const lkv_ragged_desc* cache, int32_t n_seq, int32_t n_layers,
                           int32_t n_kv_heads, int32_t n_q_heads, const void* q, const void* new_k,
                           const void* new_v, int32_t* tokens_seen, void* out, double scale,
                           void* workspace, size_t workspace_bytes, lkv_stream_t stream);

/* ---- full decode step of the reference's toy GQA model --------------------
 * Replaces decode_step (model.hpp:95, model.cpp:209-287) for a batch of n_seq <= 16 sequences
 * whose compacted caches live in one ragged cache (flat head (s * L + l) * H + h).  Weights are
 * the reference's ModelWeights (model.hpp:35-47) in the reference layout (x W, row-major
 * [rows][cols]), repacked once into a library-owned blob by lkv_model_load_param:
 *   LKV_P_TOK_EMBED [vocab][dm], WQ [dm][dm], WK/WV [dm][H*d], WO [dm][dm], ATTN_NORM/MLP_NORM [dm],
 *   W_GATE/W_UP [dm][mlp_width], W_DOWN [mlp_width][dm], FINAL_NORM [dm], LM_HEAD [dm][vocab]
 * (dm = n_q_heads * head_dim), each in the model dtype.  The blob must be zero-filled before the
 * first load.  lkv_model_plan (after every eviction / change of the cache's offsets) plans the
 * per-layer decode attention and builds the RoPE table; lkv_model_decode_step then runs one
 * step: tokens [n_seq] and tokens_seen [n_seq] are device int32, logits [n_seq][vocab] fp32.
 * Token / position range errors are latched (lkv_workspace_status -> LKV_ERR_CONTRACT). */
typedef struct lkv_model_desc {
    int32_t n_layers, n_q_heads, n_kv_heads, head_dim, vocab_size, max_seq_len, mlp_width, dtype;
    double rope_base; /* 10000 (model.cpp:38) */
    double norm_eps;  /* 1e-6 (model.cpp:48) */
} lkv_model_desc;

enum {
    LKV_P_TOK_EMBED = 0,
    LKV_P_WQ = 1,
    LKV_P_WK = 2,
    LKV_P_WV = 3,
    LKV_P_WO = 4,
    LKV_P_ATTN_NORM = 5,
    LKV_P_MLP_NORM = 6,
    LKV_P_W_GATE = 7,
    LKV_P_W_UP = 8,
    LKV_P_W_DOWN = 9,
    LKV_P_FINAL_NORM = 10,
    LKV_P_LM_HEAD = 11
};

#define LKV_MODEL_MAX_SEQ 16

lkv_status lkv_model_validate(const lkv_model_desc* model); /* ModelConfig::validate, model.cpp:124-133 */
size_t lkv_model_weights_bytes(const lkv_model_desc* model);
lkv_status lkv_model_load_param(const lkv_model_desc* model, void* weights, int32_t param, int32_t layer,
                                const void* src, lkv_stream_t stream);
size_t lkv_model_workspace_bytes(const lkv_model_desc* model, int32_t n_seq, const lkv_ragged_desc* cache);
lkv_status lkv_model_plan(const lkv_model_desc* model, const lkv_ragged_desc* cache, int32_t n_seq, void* workspace,
                          size_t workspace_bytes, lkv_stream_t stream);
/* lkv_model_plan with the per-layer attention work-item size fixed (as lkv_decode_plan_ex) */
lkv_status lkv_model_plan_ex(const lkv_model_desc* model, const lkv_ragged_desc* cache, int32_t n_seq,
                             int32_t rows_per_item, void* workspace, size_t workspace_bytes, lkv_stream_t stream);
lkv_status lkv_model_decode_step(const lkv_model_desc* model, const void* weights, const lkv_ragged_desc* cache,
                                 int32_t n_seq, const int32_t* tokens, int32_t* tokens_seen, float* logits,
                                 void* workspace, size_t workspace_bytes, lkv_stream_t stream);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* LKV_B200_H */
