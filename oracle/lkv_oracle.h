/*
 * lkv_oracle.h -- CPU restatement of the LKV inference-time eviction path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2605_06676_b200/,
 * include/) may include, link or call this.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg use it, as the checker and
 * as the reported CPU baseline.
 *
 * Every function restates one reference routine in plain C, fp64, and cites the
 * reference file:line it follows (paths relative to /root/reference).  The
 * restatement is pinned by tests/test_oracle.py against every known-answer test
 * of the reference's own suite for this path (proj/tests/test_soft_topk.cpp,
 * test_policy.cpp, test_evictsim.cpp, test_attention.cpp) and, when the
 * reference sources are present, bit-for-bit against oracle/_ref (the
 * reference's own soft_topk.cpp / policy.cpp compiled over a tensor shim).
 *
 * Compile with -ffp-contract=off: the fp64 operation sequence must be the one
 * written in the source (no FMA contraction), so that budgets are reproducible.
 */
#ifndef LKV_ORACLE_H
#define LKV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror proj/include/lkv/errors.hpp:10-32 and include/lkv_b200.h */
enum {
    LKVO_OK = 0,
    LKVO_CONTRACT = 1,
    LKVO_NUMERIC = 2,
    LKVO_BUDGET = 3,
    LKVO_OVERFLOW_GUARD = 4,
    LKVO_DEGENERATE_MASK = 5
};

enum { LKVO_F32 = 0, LKVO_BF16 = 1, LKVO_F64 = 2 /* fp64 inputs (the reference API's own precision) */ };
enum { LKVO_SILU = 0, LKVO_GELU_ERF = 1 };

/* ---- rng.hpp:11-66 (mt19937_64 + hand-rolled conversions) -------------- */
typedef struct lkvo_rng {
    uint64_t mt[312];
    int idx;
    int has_spare;
    double spare;
} lkvo_rng;

uint64_t lkvo_mix64(uint64_t z);
uint64_t lkvo_derive_seed(uint64_t base, uint64_t a, uint64_t b, uint64_t c);
void lkvo_rng_seed(lkvo_rng* r, uint64_t seed);
uint64_t lkvo_rng_next(lkvo_rng* r);
double lkvo_rng_uniform(lkvo_rng* r);
double lkvo_rng_uniform_range(lkvo_rng* r, double lo, double hi);
int lkvo_rng_uniform_int(lkvo_rng* r, int lo, int hi);
double lkvo_rng_normal(lkvo_rng* r);
/* fill helpers for fixtures */
void lkvo_fill_uniform(uint64_t seed, double lo, double hi, double* out, int64_t n);

/* ---- soft_topk.cpp ------------------------------------------------------- */
double lkvo_laplace_cdf(double z);
int lkvo_solve_threshold(const double* x, int n, double k, double* lambda_out, int* m_out);
int lkvo_soft_topk_forward(const double* x, int n, double k, double tau, double* values,
                           double* lambda_out, int* m_out, double* clamped_k_out);
/* bisection oracle of proj/tests/oracles.hpp:25-40 */
double lkvo_bisect_lambda(const double* x, int n, double k, double tol);
/* hard_topk (soft_topk.cpp:191-201): mask with b ones, ties keep the lowest index */
int lkvo_hard_topk(const double* x, int n, int b, int32_t* mask);
/* the same selection over fp32 device scores; writes the b selected positions
 * in ascending order (the compaction order of evictsim.cpp:205-212) */
int lkvo_select_positions_f32(const float* x, int n, int b, int32_t* positions);

/* ---- policy.cpp ---------------------------------------------------------- */
int lkvo_allocate_budgets(const double* logits, int n, double target_ratio, double* ratios);
int lkvo_freeze_budgets(const double* ratios, int n, int t, int32_t* budgets);
/* exact-sum variant: sum == llround(R*n*t) */
int lkvo_freeze_budgets_exact(const double* ratios, int n, double target_ratio, int t,
                              int32_t* budgets);

/* token scorer (policy.cpp:30-34,131-136), fp64 over widened inputs.
 *   x_i = k_i (in = d) or [k_i ; v_i] (in = 2d)
 *   u_i = act(x_i W1 + b1) . w2
 * keys/values: [t][d] of dtype; w1: [in][hidden] fp64; b1, w2: [hidden] */
int lkvo_token_scores(int dtype, const void* keys, const void* values, int64_t t, int d,
                      int in_mode, const double* w1, const double* b1, const double* w2,
                      int hidden, int act, double* out);

/* ---- compaction (evictsim.cpp:202-215, model.cpp:289-315) -------------- */
void lkvo_compact_rows(int dtype, const void* src_k, const void* src_v, int d,
                       const int32_t* positions, int b, void* dst_k, void* dst_v);

/* ---- decode attention (model.cpp:240-265 + attention.cpp:46-94) --------- */
/* Query heads qh in [0, G) of one KV head attend over the head's retained rows
 * (the new row already appended).  q: [G][d] fp64; keys/values [t][d] dtype;
 * out [G][d] fp64.  n_q = 1, causal = false, no mask, scale given. */
int lkvo_decode_attention(int dtype, const double* q, int G, const void* keys,
                          const void* values, int64_t t, int d, double scale, double* out);

/* ---- evictsim.cpp:56-81 -------------------------------------------------- */
int lkvo_kv_memory_bytes(int n_layers, int n_kv_heads, int head_dim, double bytes_per_element,
                         int64_t tokens, double retention, double* full, double* compressed,
                         double* reduction);
int lkvo_kv_memory_bytes_budgets(int n_layers, int n_kv_heads, int head_dim,
                                 double bytes_per_element, int64_t tokens,
                                 const int32_t* budgets, int n, double* full,
                                 double* compressed, double* reduction);

/* ---- whole eviction of a batch of heads (the CPU baseline) -------------- */
/* For each head h (rows [h*T, h*T + t_h) of keys/values): score (fp64), select
 * budgets[h] rows, gather them to dst at offsets[h].  Heads are spread over
 * n_threads pthreads (n_threads = 1 reproduces the reference's single-threaded
 * loop, evictsim.cpp:131-222).  scorer weights are per head via head_scorer[h].
 * scores_out (nullable) gets the fp64 scores [h*T + j]. */
int lkvo_evict_heads(int dtype, const void* keys, const void* values, int n_heads, int64_t T,
                     const int32_t* t_per_head, int d, int in_mode, const double* w1_all,
                     const double* b1_all, const double* w2_all, int hidden, int act,
                     const int32_t* head_scorer, const int32_t* budgets, const int64_t* offsets,
                     void* dst_k, void* dst_v, int32_t* dst_pos, double* scores_out,
                     int n_threads);

/* ---- soft_topk.cpp:123,153,166-189 ----------------------------------------- */
int lkvo_soft_topk_density(const double* x, int n, double tau, double lambda, double clamped_k, double* density);
int lkvo_soft_topk_vjp(const double* density, const double* upstream, int n, double tau, double* grad_x,
                       double* grad_k);

/* ---- attention.cpp:46-94,145-201 (one head; mask nullable = all ones) ---------- */
int lkvo_masked_attention(const double* q, const double* k, const double* v, const double* mask, int n_q, int t,
                          int d, int causal, double scale, int pos_offset, int self_keep, double* out,
                          double* p_raw, double* p, double* renorm);
int lkvo_masked_attention_vjp(const double* q, const double* k, const double* v, const double* mask, int n_q,
                              int t, int d, int causal, double scale, int pos_offset, int self_keep,
                              const double* upstream, double* dq, double* dk, double* dv, double* dmask);

const char* lkvo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
