/*
 * lkv_oracle.c -- CPU restatement (fp64, plain C) of LKV's inference-time
 * eviction path.  TEST INFRASTRUCTURE ONLY: see lkv_oracle.h.
 *
 * Reference files (relative to /root/reference):
 *   proj/include/lkv/rng.hpp            rng stream used by the reference fixtures
 *   proj/src/soft_topk.cpp              LKV-H threshold solve, soft top-k, hard top-k
 *   proj/src/policy.cpp                 allocate/freeze budgets, token scorer
 *   proj/src/evictsim.cpp, model.cpp    compaction, decode attention, memory model
 *   proj/src/attention.cpp              dense attention semantics
 * Build: -O2 -ffp-contract=off (see Makefile); never -ffast-math.
 */
#define _GNU_SOURCE
#include "lkv_oracle.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* lkvo_last_error(void) { return g_err; }

/* std::max / std::min / std::clamp exactly as libstdc++ defines them */
static inline double std_max(double a, double b) { return (a < b) ? b : a; }
static inline double std_min(double a, double b) { return (b < a) ? b : a; }
static inline double std_clamp(double v, double lo, double hi) {
    return (v < lo) ? lo : (hi < v) ? hi : v;
}

/* ======================================================================== */
/* rng.hpp:11-66                                                             */
/* ======================================================================== */

uint64_t lkvo_mix64(uint64_t z) { /* rng.hpp:11-16 */
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t lkvo_derive_seed(uint64_t base, uint64_t a, uint64_t b, uint64_t c) { /* rng.hpp:20-25 */
    uint64_t s = lkvo_mix64(base);
    s = lkvo_mix64(s ^ a);
    s = lkvo_mix64(s ^ b);
    return lkvo_mix64(s ^ c);
}

/* std::mt19937_64, the engine under lkv::Rng (rng.hpp:29-30,62) */
void lkvo_rng_seed(lkvo_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
    r->has_spare = 0;
    r->spare = 0.0;
}

uint64_t lkvo_rng_next(lkvo_rng* r) {
    if (r->idx >= 312) {
        const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
        for (int i = 0; i < 312; ++i) {
            uint64_t y = (r->mt[i] & upper) | (r->mt[(i + 1) % 312] & lower);
            uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = v;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEB88D5F0ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

double lkvo_rng_uniform(lkvo_rng* r) { /* rng.hpp:37 */
    return (double)(lkvo_rng_next(r) >> 11) * 0x1.0p-53;
}

double lkvo_rng_uniform_range(lkvo_rng* r, double lo, double hi) { /* rng.hpp:39 */
    return lo + (hi - lo) * lkvo_rng_uniform(r);
}

int lkvo_rng_uniform_int(lkvo_rng* r, int lo, int hi) { /* rng.hpp:42-45 */
    const uint64_t span = (uint64_t)(hi - lo);
    return lo + (int)(lkvo_rng_next(r) % span);
}

double lkvo_rng_normal(lkvo_rng* r) { /* rng.hpp:48-61, Box-Muller with a cached spare */
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1 = lkvo_rng_uniform(r);
    double u2 = lkvo_rng_uniform(r);
    if (u1 < 1e-300) u1 = 1e-300;
    const double rad = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * M_PI * u2;
    r->spare = rad * sin(theta);
    r->has_spare = 1;
    return rad * cos(theta);
}

void lkvo_fill_uniform(uint64_t seed, double lo, double hi, double* out, int64_t n) {
    lkvo_rng r;
    lkvo_rng_seed(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = lkvo_rng_uniform_range(&r, lo, hi);
}

/* ======================================================================== */
/* stable descending order (std::stable_sort with x[a] > x[b])               */
/* ======================================================================== */

/* Bottom-up merge sort of index arrays.  A merge takes from the right run only
 * when right > left, so equal keys keep their input order: the permutation is
 * the one std::stable_sort produces with comparator x[a] > x[b]. */
#define DEFINE_STABLE_DESC(NAME, T)                                                     \
    static void NAME(const T* x, int32_t* idx, int32_t* tmp, int n) {                   \
        for (int i = 0; i < n; ++i) idx[i] = i;                                          \
        int32_t* src = idx;                                                              \
        int32_t* dst = tmp;                                                              \
        for (int w = 1; w < n; w *= 2) {                                                 \
            for (int lo = 0; lo < n; lo += 2 * w) {                                      \
                int mid = lo + w < n ? lo + w : n;                                       \
                int hi = lo + 2 * w < n ? lo + 2 * w : n;                                \
                int a = lo, b = mid, o = lo;                                             \
                while (a < mid && b < hi) {                                              \
                    if (x[src[b]] > x[src[a]]) dst[o++] = src[b++];                      \
                    else dst[o++] = src[a++];                                            \
                }                                                                        \
                while (a < mid) dst[o++] = src[a++];                                     \
                while (b < hi) dst[o++] = src[b++];                                      \
            }                                                                            \
            int32_t* t_ = src; src = dst; dst = t_;                                      \
        }                                                                                \
        if (src != idx) memcpy(idx, src, sizeof(int32_t) * (size_t)n);                   \
    }

DEFINE_STABLE_DESC(stable_desc_f64, double)
DEFINE_STABLE_DESC(stable_desc_f32, float)

/* ======================================================================== */
/* soft_topk.cpp                                                             */
/* ======================================================================== */

static double logaddexp(double a, double b) { /* soft_topk.cpp:20-25 */
    if (a == -INFINITY) return b;
    if (b == -INFINITY) return a;
    const double m = std_max(a, b);
    return m + log1p(exp(-fabs(a - b)));
}

static int clamp_budget(double k, int n, double* out) { /* soft_topk.cpp:27-33 */
    if (!(k > 0.0) || !(k < (double)n)) return fail(LKVO_BUDGET, "k must lie strictly inside (0, n)");
    const double eps = std_min(1e-3, 0.01 * n);
    *out = std_min(std_max(k, eps), (double)n - eps);
    return LKVO_OK;
}

static double candidate_lambda(int m, int n, double k, double l1, double l2) { /* soft_topk.cpp:38-48 */
    if (m == 0) return l2 - log(2.0 * k);
    if (m == n) return log(2.0 * ((double)n - k)) - l1;
    const double a = k - (double)m;
    const double d = l1 + l2;
    if (a == 0.0) return 0.5 * (l2 - l1);
    const double root = sqrt(a * a + exp(d));
    if (a < 0.0) return log(root - a) - l1;
    return d - log(root + a) - l1;
}

double lkvo_laplace_cdf(double z) { /* soft_topk.cpp:52-56 (finite z) */
    if (z >= 0.0) return 1.0 - 0.5 * exp(-z);
    return 0.5 * exp(z);
}

int lkvo_solve_threshold(const double* x, int n, double k, double* lambda_out, int* m_out) {
    /* soft_topk.cpp:58-109 */
    if (n < 2) return fail(LKVO_CONTRACT, "solve_threshold: need at least two scores");
    for (int i = 0; i < n; ++i) {
        if (!isfinite(x[i])) return fail(LKVO_NUMERIC, "solve_threshold: non-finite score");
        if (fabs(x[i]) > 1e300)
            return fail(LKVO_OVERFLOW_GUARD, "solve_threshold: score magnitude beyond float64 exponent range");
    }
    double kc;
    int st = clamp_budget(k, n, &kc);
    if (st) return st;

    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)n * 2);
    double* xs = (double*)malloc(sizeof(double) * (size_t)n);
    double* l1 = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    double* l2 = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    stable_desc_f64(x, order, order + n, n);
    for (int i = 0; i < n; ++i) xs[i] = x[order[i]];
    for (int i = 0; i <= n; ++i) l1[i] = l2[i] = -INFINITY;
    for (int m = 1; m <= n; ++m) l1[m] = logaddexp(l1[m - 1], -xs[m - 1]);
    for (int m = n - 1; m >= 0; --m) l2[m] = logaddexp(l2[m + 1], xs[m]);

    const double kSlack = 1e-12;
    double best_lambda = 0.0, best_violation = INFINITY;
    int best_m = -1;
    int rc = -1;
    for (int m = 0; m <= n; ++m) {
        const double lam = candidate_lambda(m, n, kc, l1[m], l2[m]);
        if (!isfinite(lam)) continue;
        const double hi_v = (m == 0) ? 0.0 : std_max(0.0, lam - xs[m - 1]);
        const double lo_v = (m == n) ? 0.0 : std_max(0.0, xs[m] - lam);
        const double violation = std_max(hi_v, lo_v);
        if (violation <= kSlack) {
            *lambda_out = lam;
            *m_out = m;
            rc = LKVO_OK;
            break;
        }
        if (violation < best_violation) {
            best_violation = violation;
            best_lambda = lam;
            best_m = m;
        }
    }
    if (rc != LKVO_OK) {
        rc = fail(LKVO_NUMERIC, "solve_threshold: no bracket admitted the closed-form root");
        if (best_m >= 0 && best_violation < 1e-6) { /* soft_topk.cpp:101-107 */
            double sum = 0.0;
            for (int i = 0; i < n; ++i) sum += lkvo_laplace_cdf(xs[i] - best_lambda);
            if (fabs(sum - kc) <= 1e-9 * n) {
                *lambda_out = best_lambda;
                *m_out = best_m;
                rc = LKVO_OK;
            }
        }
    }
    free(order);
    free(xs);
    free(l1);
    free(l2);
    return rc;
}

int lkvo_soft_topk_forward(const double* x, int n, double k, double tau, double* values,
                           double* lambda_out, int* m_out, double* clamped_k_out) {
    /* soft_topk.cpp:111-164 */
    if (!(tau > 0.0)) return fail(LKVO_CONTRACT, "soft_topk_forward: tau must be positive");
    if (n < 1) return fail(LKVO_CONTRACT, "soft_topk_forward: empty scores");
    if (n == 1) { /* :119-131 */
        if (!isfinite(x[0])) return fail(LKVO_NUMERIC, "soft_topk_forward: non-finite score");
        double kk;
        int st = clamp_budget(k, 1, &kk);
        if (st) return st;
        values[0] = kk;
        const double z = kk >= 0.5 ? -log(2.0 * (1.0 - kk)) : log(2.0 * kk);
        if (lambda_out) *lambda_out = x[0] / tau - z;
        if (m_out) *m_out = kk >= 0.5 ? 1 : 0;
        if (clamped_k_out) *clamped_k_out = kk;
        return LKVO_OK;
    }
    double* scaled = (double*)malloc(sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) scaled[i] = x[i] / tau;
    double lambda;
    int m;
    int st = lkvo_solve_threshold(scaled, n, k, &lambda, &m);
    if (st) {
        free(scaled);
        return st;
    }
    double kc = 0.0;
    clamp_budget(k, n, &kc);
    const double hi = 1.0 - DBL_EPSILON / 2;
    for (int i = 0; i < n; ++i) {
        const double z = scaled[i] - lambda;
        values[i] = std_clamp(lkvo_laplace_cdf(z), DBL_MIN, hi);
    }
    free(scaled);
    double sum = 0.0;
    for (int i = 0; i < n; ++i) sum += values[i];
    if (fabs(sum - kc) > 1e-9 * n) return fail(LKVO_NUMERIC, "soft_topk_forward: budget constraint violated");
    if (lambda_out) *lambda_out = lambda;
    if (m_out) *m_out = m;
    if (clamped_k_out) *clamped_k_out = kc;
    return LKVO_OK;
}

int lkvo_soft_topk_density(const double* x, int n, double tau, double lambda, double clamped_k, double* density) {
    /* soft_topk.cpp:123,153: density_terms = max(0.5 exp(-|z|), DBL_MIN), z = x/tau - lambda
     * (n == 1: z is the pinned-budget log ratio) */
    if (n == 1) {
        const double z = clamped_k >= 0.5 ? -log(2.0 * (1.0 - clamped_k)) : log(2.0 * clamped_k);
        density[0] = std_max(0.5 * exp(-fabs(z)), DBL_MIN);
        return LKVO_OK;
    }
    for (int i = 0; i < n; ++i) density[i] = std_max(0.5 * exp(-fabs(x[i] / tau - lambda)), DBL_MIN);
    return LKVO_OK;
}

int lkvo_soft_topk_vjp(const double* density, const double* upstream, int n, double tau, double* grad_x,
                       double* grad_k) {
    /* soft_topk.cpp:166-189: one summation order for both reductions, so a constant upstream
     * gives an exactly zero score gradient and an exactly unit budget gradient */
    if (!(tau > 0.0)) return fail(LKVO_CONTRACT, "soft_topk_vjp: tau must be positive");
    if (n == 1) {
        grad_x[0] = 0.0;
        *grad_k = 1.0;
        return LKVO_OK;
    }
    double sum_fp = 0.0, dot = 0.0;
    for (int i = 0; i < n; ++i) {
        sum_fp += density[i];
        dot += upstream[i] * density[i];
    }
    const double mean_up = dot / sum_fp;
    for (int i = 0; i < n; ++i) grad_x[i] = density[i] * (upstream[i] - mean_up) / tau;
    *grad_k = mean_up;
    return LKVO_OK;
}

/* ---- attention.cpp:20-201: multiplicative soft-mask attention, one head ---------------- */
static inline int adm_end(int causal, int t, int pos_offset, int r) { /* attention.cpp:27-30 */
    if (!causal) return t;
    const int e = pos_offset + r + 1;
    return e < t ? e : t;
}
static inline double mask_at(const double* mask, int self_keep, int j, int pos) { /* :21-24 */
    if (self_keep && j == pos) return 1.0;
    return mask ? mask[j] : 1.0;
}
static int attn_validate(const double* mask, int n_q, int t, int d, int causal, int pos_offset) { /* :33-44 */
    if (n_q < 1 || t < 1 || d < 1) return fail(LKVO_CONTRACT, "attention: empty extents");
    if (mask)
        for (int j = 0; j < t; ++j)
            if (!(mask[j] >= 0.0) || !isfinite(mask[j]))
                return fail(LKVO_CONTRACT, "attention: mask values must be finite and >= 0");
    if (causal && adm_end(causal, t, pos_offset, 0) < 1) return fail(LKVO_CONTRACT, "attention: first query row admits no key");
    return LKVO_OK;
}

int lkvo_masked_attention(const double* q, const double* k, const double* v, const double* mask, int n_q, int t,
                          int d, int causal, double scale, int pos_offset, int self_keep, double* out,
                          double* p_raw, double* p, double* renorm) {
    /* masked_attention_dense (attention.cpp:46-94): p_raw = softmax(s) over admissible keys,
     * p~ = p_raw m, p = p~ / sum p~ (degenerate if sum <= 1e-300), out = p V.  p_raw, p
     * [n_q][t] and renorm [n_q] are the AttentionSaved fields (nullable). */
    int st = attn_validate(mask, n_q, t, d, causal, pos_offset);
    if (st) return st;
    double* pr = (double*)calloc((size_t)t, sizeof(double));
    double* w = (double*)calloc((size_t)t, sizeof(double));
    for (int r = 0; r < n_q && st == LKVO_OK; ++r) {
        const int end = adm_end(causal, t, pos_offset, r), pos = pos_offset + r;
        const double* qr = q + (size_t)r * d;
        double mx = -INFINITY;
        for (int j = 0; j < end; ++j) {
            double dot = 0.0;
            for (int c = 0; c < d; ++c) dot += qr[c] * k[(size_t)j * d + c];
            pr[j] = scale * dot;
            mx = std_max(mx, pr[j]);
        }
        double z_raw = 0.0;
        for (int j = 0; j < end; ++j) {
            pr[j] = exp(pr[j] - mx);
            z_raw += pr[j];
        }
        double z_masked = 0.0;
        for (int j = 0; j < end; ++j) {
            pr[j] /= z_raw;
            w[j] = pr[j] * mask_at(mask, self_keep, j, pos);
            z_masked += w[j];
        }
        if (!(z_masked > 1e-300)) {
            st = fail(LKVO_DEGENERATE_MASK, "attention row lost all admissible mass");
            break;
        }
        for (int j = 0; j < end; ++j) w[j] /= z_masked;
        for (int c = 0; c < d; ++c) {
            double acc = 0.0;
            for (int j = 0; j < end; ++j) acc += w[j] * v[(size_t)j * d + c];
            out[(size_t)r * d + c] = acc;
        }
        if (p_raw)
            for (int j = 0; j < t; ++j) p_raw[(size_t)r * t + j] = j < end ? pr[j] : 0.0;
        if (p)
            for (int j = 0; j < t; ++j) p[(size_t)r * t + j] = j < end ? w[j] : 0.0;
        if (renorm) renorm[r] = z_masked;
    }
    free(pr);
    free(w);
    return st;
}

int lkvo_masked_attention_vjp(const double* q, const double* k, const double* v, const double* mask, int n_q,
                              int t, int d, int causal, double scale, int pos_offset, int self_keep,
                              const double* upstream, double* dq, double* dk, double* dv, double* dmask) {
    /* masked_attention_vjp (attention.cpp:145-201), forward state recomputed in place:
     * W = U V^T; per row wp = sum_j w p; d p~ = (w - wp) / z; dmask += d p~ p_raw (self keys
     * excluded); d p_raw = d p~ m; dp_dot = sum d p_raw p_raw; ds = p_raw (d p_raw - dp_dot) scale;
     * dV = P^T U, dQ = dS K, dK = dS^T Q.  Gradients are ACCUMULATED into dq/dk/dv/dmask. */
    double* P = (double*)malloc(sizeof(double) * (size_t)n_q * t);
    double* PR = (double*)malloc(sizeof(double) * (size_t)n_q * t);
    double* Z = (double*)malloc(sizeof(double) * (size_t)n_q);
    double* out = (double*)malloc(sizeof(double) * (size_t)n_q * d);
    int st = lkvo_masked_attention(q, k, v, mask, n_q, t, d, causal, scale, pos_offset, self_keep, out, PR, P, Z);
    double* ds = (double*)malloc(sizeof(double) * (size_t)t);
    double* w = (double*)malloc(sizeof(double) * (size_t)t);
    for (int r = 0; r < n_q && st == LKVO_OK; ++r) {
        const int end = adm_end(causal, t, pos_offset, r), pos = pos_offset + r;
        const double* u = upstream + (size_t)r * d;
        const double* p_raw = PR + (size_t)r * t;
        const double* p = P + (size_t)r * t;
        for (int j = 0; j < t; ++j) {
            double acc = 0.0;
            for (int c = 0; c < d; ++c) acc += u[c] * v[(size_t)j * d + c];
            w[j] = acc;
            ds[j] = 0.0;
        }
        double wp = 0.0;
        for (int j = 0; j < end; ++j) wp += w[j] * p[j];
        double dp_dot = 0.0;
        for (int j = 0; j < end; ++j) {
            const double d_ptilde = (w[j] - wp) / Z[r];
            if (mask && dmask && !(self_keep && j == pos)) dmask[j] += d_ptilde * p_raw[j];
            const double d_praw = d_ptilde * mask_at(mask, self_keep, j, pos);
            ds[j] = d_praw;
            dp_dot += d_praw * p_raw[j];
        }
        for (int j = 0; j < end; ++j) ds[j] = p_raw[j] * (ds[j] - dp_dot) * scale;
        for (int j = 0; j < t; ++j) {
            for (int c = 0; c < d; ++c) {
                dv[(size_t)j * d + c] += p[j] * u[c];
                dq[(size_t)r * d + c] += ds[j] * k[(size_t)j * d + c];
                dk[(size_t)j * d + c] += ds[j] * q[(size_t)r * d + c];
            }
        }
    }
    free(P);
    free(PR);
    free(Z);
    free(out);
    free(ds);
    free(w);
    return st;
}

double lkvo_bisect_lambda(const double* x, int n, double k, double tol) {
    /* proj/tests/oracles.hpp:25-40 */
    double lo = x[0], hi = x[0];
    for (int i = 1; i < n; ++i) {
        if (x[i] < lo) lo = x[i];
        if (x[i] > hi) hi = x[i];
    }
    lo -= 40.0;
    hi += 40.0;
    for (int it = 0; it < 200 && hi - lo > tol; ++it) {
        const double mid = 0.5 * (lo + hi);
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += lkvo_laplace_cdf(x[i] - mid);
        if (s - k > 0.0) lo = mid;
        else hi = mid;
    }
    return 0.5 * (lo + hi);
}

int lkvo_hard_topk(const double* x, int n, int b, int32_t* mask) { /* soft_topk.cpp:191-201 */
    if (b < 0 || b > n) return fail(LKVO_BUDGET, "hard_topk: b outside [0, n]");
    for (int i = 0; i < n; ++i)
        if (isnan(x[i])) return fail(LKVO_NUMERIC, "hard_topk: NaN score");
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * n + 1));
    stable_desc_f64(x, order, order + n, n);
    memset(mask, 0, sizeof(int32_t) * (size_t)n);
    for (int i = 0; i < b; ++i) mask[order[i]] = 1;
    free(order);
    return LKVO_OK;
}

int lkvo_select_positions_f32(const float* x, int n, int b, int32_t* positions) {
    /* hard_topk (soft_topk.cpp:191-201) on fp32 scores, then the ascending walk of
     * the compaction loop (evictsim.cpp:205-212) */
    if (b < 0 || b > n) return fail(LKVO_BUDGET, "hard_topk: b outside [0, n]");
    for (int i = 0; i < n; ++i)
        if (isnan(x[i])) return fail(LKVO_NUMERIC, "hard_topk: NaN score");
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * n + 1));
    uint8_t* mask = (uint8_t*)calloc((size_t)n + 1, 1);
    stable_desc_f32(x, order, order + n, n);
    for (int i = 0; i < b; ++i) mask[order[i]] = 1;
    int o = 0;
    for (int j = 0; j < n; ++j)
        if (mask[j]) positions[o++] = j;
    free(order);
    free(mask);
    return LKVO_OK;
}

/* ======================================================================== */
/* policy.cpp                                                                */
/* ======================================================================== */

int lkvo_allocate_budgets(const double* logits, int n, double target_ratio, double* ratios) {
    /* policy.cpp:110-120: soft_topk over the flattened head logits, k = R*n, tau = 1 */
    if (!(target_ratio > 0.0 && target_ratio < 1.0)) return fail(LKVO_BUDGET, "target ratio must lie in (0,1)");
    if (n < 1) return fail(LKVO_CONTRACT, "allocate_budgets: score length mismatch");
    return lkvo_soft_topk_forward(logits, n, target_ratio * n, 1.0, ratios, NULL, NULL, NULL);
}

int lkvo_freeze_budgets(const double* ratios, int n, int t, int32_t* budgets) {
    /* policy.cpp:122-129: plain floor, no minimum, no repair */
    if (t < 1) return fail(LKVO_CONTRACT, "freeze_budgets: t must be >= 1");
    for (int i = 0; i < n; ++i) budgets[i] = (int32_t)floor(ratios[i] * t);
    return LKVO_OK;
}

int lkvo_freeze_budgets_exact(const double* ratios, int n, double target_ratio, int t,
                              int32_t* budgets) {
    /* floor, then hand the deficit D = total - sum(floor)
     * out one unit per head.  D > 0: +1 to the D largest remainders r*t - floor(r*t),
     * ties to the lower flat index.  D < 0: -1 to the |D| smallest remainders among
     * heads with floor >= 1, ties to the higher index.  total = llround(R*n*t). */
    if (t < 1) return fail(LKVO_CONTRACT, "freeze_budgets: t must be >= 1");
    if (!(target_ratio > 0.0 && target_ratio < 1.0)) return fail(LKVO_BUDGET, "target ratio must lie in (0,1)");
    double* rem = (double*)malloc(sizeof(double) * (size_t)n);
    int64_t sum = 0;
    for (int i = 0; i < n; ++i) {
        const double p = ratios[i] * t;
        const double f = floor(p);
        budgets[i] = (int32_t)f;
        rem[i] = p - f;
        sum += budgets[i];
    }
    const int64_t total = llround(target_ratio * n * t);
    const int64_t D = total - sum;
    int rc = LKVO_OK;
    if (D > n || D < -n) {
        rc = fail(LKVO_NUMERIC, "freeze_budgets_exact: deficit exceeds one unit per head");
    } else if (D != 0) {
        int64_t given = 0;
        /* ranks are computed on the floored table, deltas applied afterwards */
        int32_t* delta = (int32_t*)calloc((size_t)n, sizeof(int32_t));
        for (int i = 0; i < n; ++i) {
            const int elig_i = D > 0 ? (budgets[i] < t) : (budgets[i] > 0);
            if (!elig_i) continue;
            int64_t rank = 0;
            for (int j = 0; j < n; ++j) {
                const int elig_j = D > 0 ? (budgets[j] < t) : (budgets[j] > 0);
                if (!elig_j || j == i) continue;
                if (D > 0) {
                    if (rem[j] > rem[i] || (rem[j] == rem[i] && j < i)) ++rank;
                } else {
                    if (rem[j] < rem[i] || (rem[j] == rem[i] && j > i)) ++rank;
                }
            }
            if (rank < (D > 0 ? D : -D)) {
                delta[i] = D > 0 ? 1 : -1;
                ++given;
            }
        }
        for (int i = 0; i < n; ++i) budgets[i] += delta[i];
        free(delta);
        if (given != (D > 0 ? D : -D)) rc = fail(LKVO_NUMERIC, "freeze_budgets_exact: not enough eligible heads");
    }
    free(rem);
    return rc;
}

static inline double widen(int dtype, const void* p, int64_t i) {
    if (dtype == LKVO_F64) return ((const double*)p)[i];
    if (dtype == LKVO_F32) return (double)((const float*)p)[i];
    uint32_t bits = (uint32_t)((const uint16_t*)p)[i] << 16;
    float f;
    memcpy(&f, &bits, 4);
    return (double)f;
}

static inline double act_apply(int act, double v) {
    if (act == LKVO_SILU) return v / (1.0 + exp(-v)); /* tensor.cpp:371-378 */
    return 0.5 * v * (1.0 + erf(v * 0.70710678118654752440)); /* GELU-erf (BASELINE.json configs) */
}

int lkvo_token_scores(int dtype, const void* keys, const void* values, int64_t t, int d,
                      int in_mode, const double* w1, const double* b1, const double* w2,
                      int hidden, int act, double* out) {
    /* policy.cpp:131-136 -> mlp2_forward policy.cpp:30-34:
     *   h = act(add_rowvec(matmul([k;v], W1), b1)); s = matmul(h, W2)  (no output bias) */
    if (t < 0 || d < 1 || hidden < 1 || (in_mode != 1 && in_mode != 2))
        return fail(LKVO_CONTRACT, "token_scores: bad geometry");
    if (in_mode == 2 && !values) return fail(LKVO_CONTRACT, "token_scores: values required");
    const int in = in_mode * d;
    /* rows in blocks of 4 so each W1 row is reused from cache four times; every row keeps the
     * reference's summation order (i ascending), so results are identical to a row-at-a-time loop */
    enum { RB = 4 };
    double* x = (double*)malloc(sizeof(double) * (size_t)in * RB);
    double* acc = (double*)malloc(sizeof(double) * (size_t)hidden * RB);
    int rc = LKVO_OK;
    for (int64_t r0 = 0; r0 < t && rc == LKVO_OK; r0 += RB) {
        const int nb = (int)(t - r0 < RB ? t - r0 : RB);
        for (int b = 0; b < nb; ++b) {
            double* xb = x + (size_t)b * in;
            const int64_t r = r0 + b;
            for (int c = 0; c < d; ++c) xb[c] = widen(dtype, keys, r * d + c);
            if (in_mode == 2)
                for (int c = 0; c < d; ++c) xb[d + c] = widen(dtype, values, r * d + c);
            for (int c = 0; c < in; ++c)
                if (!isfinite(xb[c])) rc = fail(LKVO_NUMERIC, "matmul: non-finite input");
            for (int j = 0; j < hidden; ++j) acc[(size_t)b * hidden + j] = 0.0;
        }
        for (int i = 0; i < in; ++i) {
            const double* wr = w1 + (size_t)i * hidden;
            for (int b = 0; b < nb; ++b) {
                const double xi = x[(size_t)b * in + i];
                double* ab = acc + (size_t)b * hidden;
                for (int j = 0; j < hidden; ++j) ab[j] += xi * wr[j];
            }
        }
        for (int b = 0; b < nb; ++b) {
            const double* ab = acc + (size_t)b * hidden;
            double s = 0.0;
            for (int j = 0; j < hidden; ++j) s += act_apply(act, ab[j] + b1[j]) * w2[j];
            out[r0 + b] = s;
        }
    }
    free(x);
    free(acc);
    return rc;
}

/* ======================================================================== */
/* compaction, decode attention, memory model                                */
/* ======================================================================== */

void lkvo_compact_rows(int dtype, const void* src_k, const void* src_v, int d,
                       const int32_t* positions, int b, void* dst_k, void* dst_v) {
    /* evictsim.cpp:205-212 / model.cpp:302-311: append rows in ascending position */
    const size_t row = (size_t)d * (dtype == LKVO_F32 ? 4 : 2);
    for (int r = 0; r < b; ++r) {
        memcpy((char*)dst_k + (size_t)r * row, (const char*)src_k + (size_t)positions[r] * row, row);
        memcpy((char*)dst_v + (size_t)r * row, (const char*)src_v + (size_t)positions[r] * row, row);
    }
}

int lkvo_decode_attention(int dtype, const double* q, int G, const void* keys,
                          const void* values, int64_t t, int d, double scale, double* out) {
    /* model.cpp:250-263 (per query head, kv = qh / group) + attention.cpp:46-94 with
     * n_q = 1, causal = false, empty mask: p_raw = softmax(scale * q K^T), p = p_raw / sum,
     * out = p V.  attention.cpp:33 rejects t < 1. */
    if (t < 1 || d < 1) return fail(LKVO_CONTRACT, "attention: empty extents");
    double* s = (double*)malloc(sizeof(double) * (size_t)t);
    int rc = LKVO_OK;
    for (int g = 0; g < G && rc == LKVO_OK; ++g) {
        const double* qg = q + (size_t)g * d;
        double mx = -INFINITY;
        for (int64_t j = 0; j < t; ++j) {
            double dot = 0.0;
            for (int c = 0; c < d; ++c) dot += qg[c] * widen(dtype, keys, j * d + c);
            s[j] = scale * dot;
            mx = std_max(mx, s[j]);
        }
        double z_raw = 0.0;
        for (int64_t j = 0; j < t; ++j) {
            s[j] = exp(s[j] - mx);
            z_raw += s[j];
        }
        double z_masked = 0.0;
        for (int64_t j = 0; j < t; ++j) {
            s[j] /= z_raw;
            z_masked += s[j] * 1.0;
        }
        if (!(z_masked > 1e-300)) {
            rc = fail(LKVO_DEGENERATE_MASK, "attention row lost all admissible mass");
            break;
        }
        double* o = out + (size_t)g * d;
        for (int c = 0; c < d; ++c) o[c] = 0.0;
        for (int64_t j = 0; j < t; ++j) {
            const double w = s[j] / z_masked;
            for (int c = 0; c < d; ++c) o[c] += w * widen(dtype, values, j * d + c);
        }
    }
    free(s);
    return rc;
}

int lkvo_kv_memory_bytes(int n_layers, int n_kv_heads, int head_dim, double bytes_per_element,
                         int64_t tokens, double retention, double* full, double* compressed,
                         double* reduction) {
    /* evictsim.cpp:50-65 */
    if (n_layers < 1 || n_kv_heads < 1 || head_dim < 1 || tokens < 1 || !(bytes_per_element > 0.0))
        return fail(LKVO_CONTRACT, "memory model: all extents must be positive");
    if (!(retention > 0.0) || retention > 1.0)
        return fail(LKVO_BUDGET, "kv_memory_bytes: retention must lie in (0, 1]");
    *full = (double)n_layers * n_kv_heads * head_dim * 2.0 * bytes_per_element * (double)tokens;
    *compressed = retention * *full;
    *reduction = *full / *compressed;
    return LKVO_OK;
}

int lkvo_kv_memory_bytes_budgets(int n_layers, int n_kv_heads, int head_dim,
                                 double bytes_per_element, int64_t tokens,
                                 const int32_t* budgets, int n, double* full,
                                 double* compressed, double* reduction) {
    /* evictsim.cpp:67-81 */
    if (n_layers < 1 || n_kv_heads < 1 || head_dim < 1 || tokens < 1 || !(bytes_per_element > 0.0))
        return fail(LKVO_CONTRACT, "memory model: all extents must be positive");
    if (n != n_layers * n_kv_heads) return fail(LKVO_CONTRACT, "kv_memory_bytes: one budget per head required");
    *full = (double)n_layers * n_kv_heads * head_dim * 2.0 * bytes_per_element * (double)tokens;
    double kept = 0.0;
    for (int i = 0; i < n; ++i) kept += (double)budgets[i];
    *compressed = kept * head_dim * 2.0 * bytes_per_element;
    *reduction = *compressed > 0.0 ? *full / *compressed : INFINITY;
    return LKVO_OK;
}

/* ======================================================================== */
/* batch eviction (CPU baseline): score -> hard_topk -> compact per head     */
/* ======================================================================== */

typedef struct {
    int dtype;
    const void* keys;
    const void* values;
    int n_heads;
    int64_t T;
    const int32_t* t_per_head;
    int d, in_mode, hidden, act;
    const double *w1_all, *b1_all, *w2_all;
    const int32_t* head_scorer;
    const int32_t* budgets;
    const int64_t* offsets;
    void *dst_k, *dst_v;
    int32_t* dst_pos;
    double* scores_out;
    int next;  /* atomic work counter */
    int status;
} evict_job;

static void* evict_worker(void* arg) {
    evict_job* J = (evict_job*)arg;
    const size_t esz = J->dtype == LKVO_F32 ? 4 : 2;
    const size_t row = (size_t)J->d * esz;
    const int in = J->in_mode * J->d;
    double* sc = NULL;
    float* scf = NULL;
    int32_t* pos = NULL;
    int64_t cap = 0;
    for (;;) {
        const int h = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
        if (h >= J->n_heads) break;
        const int64_t t = J->t_per_head[h];
        if (t > cap) {
            cap = t;
            sc = (double*)realloc(sc, sizeof(double) * (size_t)cap);
            scf = (float*)realloc(scf, sizeof(float) * (size_t)cap);
            pos = (int32_t*)realloc(pos, sizeof(int32_t) * (size_t)cap);
        }
        const char* kh = (const char*)J->keys + (size_t)h * (size_t)J->T * row;
        const char* vh = (const char*)J->values + (size_t)h * (size_t)J->T * row;
        const int s = J->head_scorer[h];
        int rc = lkvo_token_scores(J->dtype, kh, vh, t, J->d, J->in_mode,
                                   J->w1_all + (size_t)s * in * J->hidden,
                                   J->b1_all + (size_t)s * J->hidden,
                                   J->w2_all + (size_t)s * J->hidden, J->hidden, J->act, sc);
        if (rc) {
            J->status = rc;
            continue;
        }
        if (J->scores_out) memcpy(J->scores_out + (size_t)h * (size_t)J->T, sc, sizeof(double) * (size_t)t);
        /* inference_select on the fp64 scores (policy.cpp:152-154) */
        int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * t + 1));
        const int b = J->budgets[h];
        if (b < 0 || b > t) {
            J->status = LKVO_BUDGET;
            free(order);
            continue;
        }
        stable_desc_f64(sc, order, order + t, (int)t);
        uint8_t* mask = (uint8_t*)calloc((size_t)t + 1, 1);
        for (int i = 0; i < b; ++i) mask[order[i]] = 1;
        int o = 0;
        for (int64_t j = 0; j < t; ++j)
            if (mask[j]) pos[o++] = (int32_t)j;
        free(order);
        free(mask);
        const int64_t off = J->offsets[h];
        lkvo_compact_rows(J->dtype, kh, vh, J->d, pos, b, (char*)J->dst_k + (size_t)off * row,
                          (char*)J->dst_v + (size_t)off * row);
        if (J->dst_pos) memcpy(J->dst_pos + off, pos, sizeof(int32_t) * (size_t)b);
    }
    free(sc);
    free(scf);
    free(pos);
    return NULL;
}

int lkvo_evict_heads(int dtype, const void* keys, const void* values, int n_heads, int64_t T,
                     const int32_t* t_per_head, int d, int in_mode, const double* w1_all,
                     const double* b1_all, const double* w2_all, int hidden, int act,
                     const int32_t* head_scorer, const int32_t* budgets, const int64_t* offsets,
                     void* dst_k, void* dst_v, int32_t* dst_pos, double* scores_out,
                     int n_threads) {
    evict_job J;
    memset(&J, 0, sizeof J);
    J.dtype = dtype;
    J.keys = keys;
    J.values = values;
    J.n_heads = n_heads;
    J.T = T;
    J.t_per_head = t_per_head;
    J.d = d;
    J.in_mode = in_mode;
    J.hidden = hidden;
    J.act = act;
    J.w1_all = w1_all;
    J.b1_all = b1_all;
    J.w2_all = w2_all;
    J.head_scorer = head_scorer;
    J.budgets = budgets;
    J.offsets = offsets;
    J.dst_k = dst_k;
    J.dst_v = dst_v;
    J.dst_pos = dst_pos;
    J.scores_out = scores_out;
    if (n_threads < 1) n_threads = 1;
    if (n_threads == 1) {
        evict_worker(&J);
    } else {
        pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
        for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, evict_worker, &J);
        for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
        free(th);
    }
    if (J.status) return fail(J.status, "evict_heads: a head failed");
    return LKVO_OK;
}
