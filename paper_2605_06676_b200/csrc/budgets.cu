// budgets.cu -- K2: LKV-H integer budget allocator, one CTA.
//
// ratios = soft_topk(logits, k = R*n, tau = 1)   (policy.cpp:110-120)
//   -> soft_topk_forward (soft_topk.cpp:111-164) -> solve_threshold (:58-109)
// budgets = floor(r * t)                          (freeze_budgets, policy.cpp:122-129)
//   or the exact-sum variant, per sequence length.
//
// Bit-exactness: this TU is compiled with -fmad=false so every fp64 expression
// is evaluated as written (no FMA contraction), in the reference's order:
// stable descending sort (rank form), sequential log-space prefix/suffix
// log-sum-exp chains, first bracket with violation <= 1e-12, sequential sums.
// The only remaining source of difference from the CPU is the last-ulp
// behaviour of exp/log/log1p (CUDA libdevice vs glibc), which can only change a
// budget when r*t lies within ~1e-16 relative of an integer (tested over many
// seeds in tests/test_gpu_parity.py).
#include <float.h>
#include <math.h>
#include <math_constants.h>

#include <atomic>

#include "kernels.cuh"

namespace lkv_dev {

constexpr int kBudgetThreads = 1024;
constexpr int kMaxLogits = 3072;  // 7n doubles of shared memory (checked by lkv_budgets)
static_assert(kMaxLogits * 7 * 8 < 227 * 1024, "budget smem");


__device__ __forceinline__ double std_max(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double std_min(double a, double b) { return (b < a) ? b : a; }

__device__ __forceinline__ double logaddexp_ref(double a, double b) {  // soft_topk.cpp:20-25
    if (a == -CUDART_INF) return b;
    if (b == -CUDART_INF) return a;
    const double m = std_max(a, b);
    return m + log1p(exp(-fabs(a - b)));
}

__device__ __forceinline__ double laplace_cdf_ref(double z) {  // soft_topk.cpp:52-56
    if (z >= 0.0) return 1.0 - 0.5 * exp(-z);
    return 0.5 * exp(z);
}

__device__ __forceinline__ double candidate_lambda(int m, int n, double k, double l1, double l2) {  // :38-48
    if (m == 0) return l2 - log(2.0 * k);
    if (m == n) return log(2.0 * ((double)n - k)) - l1;
    const double a = k - (double)m;
    const double d = l1 + l2;
    if (a == 0.0) return 0.5 * (l2 - l1);
    const double root = sqrt(a * a + exp(d));
    if (a < 0.0) return log(root - a) - l1;
    return d - log(root + a) - l1;
}

// Freeze ratios into integer budgets per sequence and scan the ragged offsets
// (policy.cpp:122-129 + SURVEY A.2); shared by the solve path and the given-ratios path.
__device__ void freeze_and_offsets(const BudgetParams& p, const double* r, double* rem, int32_t* fl, int32_t* delta,
                                   long long* s_sum_p, int64_t* s_carry_p, uint32_t* s_scan) {
    const int n = p.n;
    const int tid = threadIdx.x;
    long long& s_sum = *s_sum_p;
    int64_t& s_carry = *s_carry_p;
    if (p.ratios_out)
        for (int i = tid; i < n; i += kBudgetThreads) p.ratios_out[i] = r[i];

    // -- freeze per sequence
    for (int s = 0; s < p.n_seq; ++s) {
        const int t = p.seq_len[s];
        if (tid == 0) s_sum = 0;
        __syncthreads();
        long long local = 0;
        for (int i = tid; i < n; i += kBudgetThreads) {
            const double prod = r[i] * t;
            const double f = floor(prod);
            fl[i] = (int32_t)f;
            rem[i] = prod - f;
            delta[i] = 0;
            local += (int32_t)f;
        }
        atomicAdd(reinterpret_cast<unsigned long long*>(&s_sum), (unsigned long long)local);
        __syncthreads();
        if (p.mode == LKV_BUDGET_EXACT) {
            const long long total = llround(p.R * n * t);
            const long long D = total - s_sum;
            if (D > n || D < -n) {
                if (tid == 0) latch_error(p.err, LKV_ERR_NUMERIC, 3);
                return;
            }
            if (D != 0) {
                const long long need = D > 0 ? D : -D;
                for (int i = tid; i < n; i += kBudgetThreads) {
                    const bool elig_i = D > 0 ? (fl[i] < t) : (fl[i] > 0);
                    if (!elig_i) continue;
                    const double ri = rem[i];
                    long long rank = 0;
                    for (int j = 0; j < n; ++j) {
                        const bool elig_j = D > 0 ? (fl[j] < t) : (fl[j] > 0);
                        if (!elig_j || j == i) continue;
                        const double rj = rem[j];
                        if (D > 0) rank += (rj > ri) || (rj == ri && j < i);
                        else rank += (rj < ri) || (rj == ri && j > i);
                    }
                    if (rank < need) delta[i] = D > 0 ? 1 : -1;
                }
                __syncthreads();
                if (tid == 0) {
                    long long given = 0;
                    for (int i = 0; i < n; ++i) given += delta[i] != 0;
                    if (given != need) latch_error(p.err, LKV_ERR_NUMERIC, 4);
                }
            }
        }
        __syncthreads();
        for (int i = tid; i < n; i += kBudgetThreads) p.budgets_out[(size_t)s * n + i] = fl[i] + delta[i];
        if (p.local_count > 0)
            for (int i = tid; i < p.local_count; i += kBudgetThreads)
            {
                const int g = p.local_ids ? p.local_ids[i] : p.local_begin + i;  // the local head's global index
                p.budgets_local_out[(size_t)s * p.local_count + i] = fl[g] + delta[g];
            }
        __syncthreads();
    }

    // -- offsets = exclusive scan of (budget + slack)
    if (p.offsets_out) {
        __threadfence_block();
        __syncthreads();
        const bool shard = p.local_count > 0;
        const int64_t total_heads = (int64_t)p.n_seq * (shard ? p.local_count : n);
        const int32_t* bsrc = shard ? p.budgets_local_out : p.budgets_out;
        if (tid == 0) s_carry = 0;
        __syncthreads();
        for (int64_t base = 0; base < total_heads; base += kBudgetThreads) {
            const int64_t i = base + tid;
            const uint32_t v = i < total_heads ? uint32_t(bsrc[i] + p.slack) : 0u;
            uint32_t tot;
            const uint32_t ex = block_exclusive_scan<kBudgetThreads>(v, s_scan, &tot);
            if (i < total_heads) p.offsets_out[i] = s_carry + ex;
            __syncthreads();
            if (tid == 0) s_carry += tot;
            __syncthreads();
        }
        if (tid == 0) p.offsets_out[total_heads] = s_carry;
    }
}

__global__ void __launch_bounds__(kBudgetThreads, 1) budgets_kernel(const BudgetParams p) {
    // lkv_evict launches K1 as this kernel's programmatic dependent: let it start now, on the
    // other SMs (K1 waits for this grid before it completes; the select kernels wait for K1)
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = p.n;
    double* x = reinterpret_cast<double*>(smem_raw);  // [n]
    double* xs = x + n;                               // [n] sorted descending
    double* l1 = xs + n;                              // [n+1]
    double* l2 = l1 + (n + 1);                        // [n+1]
    double* r = l2 + (n + 1);                         // [n] ratios
    double* rem = r + n;                              // [n] remainders (per sequence)
    int32_t* fl = reinterpret_cast<int32_t*>(rem + n);  // [n] floors
    int32_t* delta = fl + n;                            // [n]

    __shared__ int s_first_bad;
    __shared__ int s_first_ok;
    __shared__ unsigned long long s_best_v;
    __shared__ int s_best_m;
    __shared__ double s_lambda;
    __shared__ double s_kc;
    __shared__ int s_fail;
    __shared__ long long s_sum;
    __shared__ int64_t s_carry;
    __shared__ uint32_t s_scan[kBudgetThreads / 32 + 1];

    const int tid = threadIdx.x;
    if (p.ratios_in) {  // freeze caller-given ratios (freeze_budgets on an existing BudgetTable)
        for (int i = tid; i < n; i += kBudgetThreads) r[i] = p.ratios_in[i];
        __syncthreads();
        freeze_and_offsets(p, r, rem, fl, delta, &s_sum, &s_carry, s_scan);
        return;
    }
    if (tid == 0) {
        s_first_bad = INT_MAX;
        s_first_ok = INT_MAX;
        s_best_v = ~0ull;
        s_best_m = INT_MAX;
        s_fail = 0;
    }
    __syncthreads();

    // -- load + validate (solve_threshold :61-64: first offending element decides)
    // (soft_topk_forward solves on x / tau, soft_topk.cpp:140-143; the unscaled scores stay in
    // `rem` for the output permutation, which sorts them, :152-156)
    for (int i = tid; i < n; i += kBudgetThreads) {
        const double raw = p.logits[i];
        const double v = p.soft ? raw / p.tau : raw;
        x[i] = v;
        if (p.soft) rem[i] = raw;
        if (!isfinite(v) || fabs(v) > 1e300) atomicMin(&s_first_bad, i);
    }
    __syncthreads();
    if (s_first_bad != INT_MAX) {
        if (tid == 0) {
            const double v = x[s_first_bad];
            if (!isfinite(v)) latch_error(p.err, LKV_ERR_NUMERIC, s_first_bad);
            else if (n >= 2) latch_error(p.err, LKV_ERR_OVERFLOW_GUARD, s_first_bad);
            else s_first_bad = INT_MAX;  // n == 1 has no magnitude guard (:119-131)
        }
        __syncthreads();
        if (s_first_bad != INT_MAX) return;
    }

    // -- k = R * n (allocate_budgets, policy.cpp:118) or given (soft_topk_forward), clamp_budget (:27-33)
    const double k = p.soft ? p.k_abs : p.R * n;
    if (tid == 0) {
        if (!(k > 0.0) || !(k < (double)n)) {
            latch_error(p.err, LKV_ERR_BUDGET, 0);
            s_fail = 1;
        } else {
            const double eps = std_min(1e-3, 0.01 * n);
            s_kc = std_min(std_max(k, eps), (double)n - eps);
        }
    }
    __syncthreads();
    if (s_fail) return;
    const double kc = s_kc;

    if (n == 1) {  // soft_topk_forward :119-131: the single output is the clamped budget
        if (tid == 0) {
            r[0] = kc;
            if (p.soft) {
                const double z = kc >= 0.5 ? -log(2.0 * (1.0 - kc)) : log(2.0 * kc);
                if (p.lambda_out) *p.lambda_out = rem[0] / p.tau - z;
                if (p.m_out) *p.m_out = kc >= 0.5 ? 1 : 0;
                if (p.kc_out) *p.kc_out = kc;
                if (p.density_out) p.density_out[0] = std_max(0.5 * exp(-fabs(z)), DBL_MIN);
                if (p.perm_out) p.perm_out[0] = 0;
                if (p.ratios_out) p.ratios_out[0] = kc;
            }
        }
        __syncthreads();
        if (p.soft) return;
    } else {
        // -- stable descending sort in rank form: ties keep input order
        for (int i = tid; i < n; i += kBudgetThreads) {
            const double xi = x[i];
            int rank = 0;
            for (int j = 0; j < n; ++j) {
                const double xj = x[j];
                rank += (xj > xi) || (xj == xi && j < i);
            }
            xs[rank] = xi;
        }
        __syncthreads();
        // -- log prefix sums of e^{-x} and log suffix sums of e^{x} (:74-82) as two parallel
        //    log-sum-exp scans: each thread folds a contiguous segment of the sorted scores, a
        //    Hillis-Steele scan combines the segment totals (log2(1024) rounds), and each thread
        //    completes its segment.  The reference folds left to right in one chain; a scan
        //    associates differently, so l1 / l2 may differ from it in the last few ulps (ratios stay
        //    within 1e-13 relative; budgets bit-exact -- tests/test_gpu_parity.py), at ~15 steps of
        //    latency instead of n.
        {
            // scratch for the segment totals: r and the fl / delta pair are written only later (rem
            // holds the unscaled scores of a soft_topk_forward call)
            double* sa = r;
            double* sb = reinterpret_cast<double*>(fl);
            const int per = (n + kBudgetThreads - 1) / kBudgetThreads;
            const int i0 = min(n, tid * per), i1 = min(n, i0 + per);
            double a = -CUDART_INF, b = -CUDART_INF;
            for (int i = i0; i < i1; ++i) {  // local inclusive prefix of e^{-x}
                a = logaddexp_ref(a, -xs[i]);
                l1[i + 1] = a;
            }
            for (int i = i1 - 1; i >= i0; --i) {  // local inclusive suffix of e^{x}
                b = logaddexp_ref(b, xs[i]);
                l2[i] = b;
            }
            const int nt = (n + per - 1) / per;  // threads that own a segment (<= kBudgetThreads)
            if (tid < nt) {
                sa[tid] = a;
                sb[tid] = b;
            }
            __syncthreads();
            for (int off = 1; off < nt; off <<= 1) {
                double na = 0.0, nb = 0.0;
                if (tid < nt) {
                    na = tid >= off ? logaddexp_ref(sa[tid - off], sa[tid]) : sa[tid];
                    nb = tid + off < nt ? logaddexp_ref(sb[tid], sb[tid + off]) : sb[tid];
                }
                __syncthreads();
                if (tid < nt) {
                    sa[tid] = na;
                    sb[tid] = nb;
                }
                __syncthreads();
            }
            const double pre = (tid > 0 && tid <= nt) ? sa[tid - 1] : -CUDART_INF;  // segments before mine
            const double suf = tid + 1 < nt ? sb[tid + 1] : -CUDART_INF;           // segments after mine
            for (int i = i0; i < i1; ++i) {
                l1[i + 1] = logaddexp_ref(pre, l1[i + 1]);
                l2[i] = logaddexp_ref(suf, l2[i]);
            }
            if (tid == 0) {
                l1[0] = -CUDART_INF;
                l2[n] = -CUDART_INF;
            }
        }
        __syncthreads();
        // -- bracket scan m = 0..n (:84-100), evaluated in parallel, first accepted m wins
        for (int m = tid; m <= n; m += kBudgetThreads) {
            const double lam = candidate_lambda(m, n, kc, l1[m], l2[m]);
            if (!isfinite(lam)) continue;
            const double hi_v = (m == 0) ? 0.0 : std_max(0.0, lam - xs[m - 1]);
            const double lo_v = (m == n) ? 0.0 : std_max(0.0, xs[m] - lam);
            const double viol = std_max(hi_v, lo_v);
            if (viol <= 1e-12) atomicMin(&s_first_ok, m);
            atomicMin(&s_best_v, (unsigned long long)__double_as_longlong(viol));
        }
        __syncthreads();
        if (s_first_ok == INT_MAX) {  // fallback (:101-107): nearest candidate, lowest m
            for (int m = tid; m <= n; m += kBudgetThreads) {
                const double lam = candidate_lambda(m, n, kc, l1[m], l2[m]);
                if (!isfinite(lam)) continue;
                const double hi_v = (m == 0) ? 0.0 : std_max(0.0, lam - xs[m - 1]);
                const double lo_v = (m == n) ? 0.0 : std_max(0.0, xs[m] - lam);
                const double viol = std_max(hi_v, lo_v);
                if ((unsigned long long)__double_as_longlong(viol) == s_best_v) atomicMin(&s_best_m, m);
            }
            __syncthreads();
            if (tid == 0) {
                const int bm = s_best_m;
                bool ok = false;
                if (bm != INT_MAX && __longlong_as_double((long long)s_best_v) < 1e-6) {
                    const double lam = candidate_lambda(bm, n, kc, l1[bm], l2[bm]);
                    double sum = 0.0;
                    for (int i = 0; i < n; ++i) sum += laplace_cdf_ref(xs[i] - lam);
                    if (fabs(sum - kc) <= 1e-9 * n) {
                        ok = true;
                        s_lambda = lam;
                    }
                }
                if (!ok) {
                    latch_error(p.err, LKV_ERR_NUMERIC, 1);
                    s_fail = 1;
                }
            }
        } else if (tid == 0) {
            const int m = s_first_ok;
            s_lambda = candidate_lambda(m, n, kc, l1[m], l2[m]);
            s_best_m = m;
        }
        __syncthreads();
        if (s_fail) return;
        // -- values (:145-150): tau = 1, x/1.0 == x
        const double lambda = s_lambda;
        const double hi = 1.0 - DBL_EPSILON / 2;
        for (int i = tid; i < n; i += kBudgetThreads) {
            double v = laplace_cdf_ref(x[i] - lambda);
            v = (v < DBL_MIN) ? DBL_MIN : (hi < v) ? hi : v;
            r[i] = v;
        }
        __syncthreads();
        if (tid == 0) {  // sum check in index order (:158-162)
            double sum = 0.0;
            for (int i = 0; i < n; ++i) sum += r[i];
            if (fabs(sum - kc) > 1e-9 * n) {
                latch_error(p.err, LKV_ERR_NUMERIC, 2);
                s_fail = 1;
            }
        }
        __syncthreads();
        if (s_fail) return;
        if (p.soft) {  // soft_topk_forward's remaining outputs (:139-156)
            if (tid == 0) {
                if (p.lambda_out) *p.lambda_out = lambda;
                if (p.m_out) *p.m_out = s_best_m;
                if (p.kc_out) *p.kc_out = kc;
            }
            for (int i = tid; i < n; i += kBudgetThreads) {
                if (p.ratios_out) p.ratios_out[i] = r[i];
                if (p.density_out) p.density_out[i] = std_max(0.5 * exp(-fabs(x[i] - lambda)), DBL_MIN);
                if (p.perm_out) {  // stable descending order of the unscaled scores
                    const double xi = rem[i];
                    int rank = 0;
                    for (int j = 0; j < n; ++j) rank += (rem[j] > xi) || (rem[j] == xi && j < i);
                    p.perm_out[rank] = i;
                }
            }
            return;
        }
    }
    freeze_and_offsets(p, r, rem, fl, delta, &s_sum, &s_carry, s_scan);
}

// Exclusive scan of (budgets + slack) for caller-supplied budgets.
__global__ void __launch_bounds__(1024) offsets_kernel(const int32_t* budgets, int n_heads, int slack,
                                                       int64_t* offsets) {
    __shared__ uint32_t s_scan[1024 / 32 + 1];
    __shared__ int64_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < n_heads; base += 1024) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < n_heads ? uint32_t(max(budgets[i], 0) + slack) : 0u;
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan<1024>(v, s_scan, &tot);
        if (i < n_heads) offsets[i] = s_carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) offsets[n_heads] = s_carry;
}

size_t budgets_smem_bytes(int n) { return (size_t)n * 8 * 6 + 16 + (size_t)n * 8; }

static std::atomic<uint64_t> g_launches{0};
void note_launches(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

cudaError_t launch_budgets(const BudgetParams& p, cudaStream_t stream) {
    const size_t smem = budgets_smem_bytes(p.n);
    cudaError_t e = cudaFuncSetAttribute(budgets_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    budgets_kernel<<<1, kBudgetThreads, smem, stream>>>(p);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_offsets(const int32_t* budgets, int n_heads, int slack, int64_t* offsets, cudaStream_t stream) {
    offsets_kernel<<<1, 1024, 0, stream>>>(budgets, n_heads, slack, offsets);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace lkv_dev
