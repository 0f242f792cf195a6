// softtopk.cu -- Soft-TopK forward / VJP for many segments at once.
//
// Reference: soft_topk_forward (soft_topk.cpp:111-164) -> solve_threshold (:58-109), and
// soft_topk_vjp (:166-189); used at training time both for LKV-H's global budget relaxation
// (policy.cpp:118, n = L*H) and for LKV-T's per-head token mask (training_mask,
// policy.cpp:138-150: Gumbel-noised scores, n = t tokens, k = the head's continuous budget).
//
//   values_i = F(x_i / tau - lambda),  F = Laplace CDF,  sum_i values_i = k (clamped)
//   density_i = max(0.5 exp(-|x_i / tau - lambda|), DBL_MIN)
//   vjp: mean = sum u_i density_i / sum density_i;  grad_x_i = density_i (u_i - mean) / tau;
//        grad_k = mean
//
// The reference finds lambda by a stable sort + sequential log-space prefix/suffix sums and
// a scan over the split m.  Here one CTA per segment (fp64, data streamed from L2):
//   1. g(lam) = sum F(s_i - lam) - k is decreasing: bisection on [min - 40, max + 40] until
//      the bracket holds no sample or is a few ulps wide;
//   2. m = #{s_i > lam} then fixes the closed form of the reference
//      (candidate_lambda(m, n, k, log S1, log S2), soft_topk.cpp:38-48) with
//      S1 = sum_{s_i > lam} e^{-s_i}, S2 = sum_{s_i <= lam} e^{s_i} as max-shifted fp64 sums.
// Only the summation order differs from the reference (parallel tree vs sequential), so lambda
// and the values agree to ~1e-15 relative; the reference's constraint check
// |sum values - k| <= 1e-9 n is re-applied.  The VJP reduces both sums with the same tree, so a
// unit upstream gives exactly zero score gradients and a unit budget gradient, as in the
// reference (test_soft_topk.cpp:129-136).
#include <float.h>
#include <math.h>
#include <math_constants.h>

#include "kernels.cuh"

namespace lkv_dev {
namespace stk {

constexpr int kThreads = 1024;

__device__ __forceinline__ double laplace_cdf(double z) { return z >= 0.0 ? 1.0 - 0.5 * exp(-z) : 0.5 * exp(z); }

// deterministic block reduction (fixed tree)
__device__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < 32) {
        s = red[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) red[32] = s;
    }
    __syncthreads();
    return red[32];
}
__device__ double block_max(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        double s = red[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
        if (threadIdx.x == 0) red[32] = s;
    }
    __syncthreads();
    return red[32];
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

__global__ void __launch_bounds__(kThreads) fwd_kernel(const __grid_constant__ SoftTopKParams p) {
    __shared__ double red[33];
    __shared__ int s_bad;
    const int seg = blockIdx.x, n = p.n, tid = threadIdx.x;
    const double* x = p.x + (size_t)seg * p.ld;
    const double* nz = p.noise ? p.noise + (size_t)seg * p.ld : nullptr;
    const double tau = p.tau;
    auto sc = [&](int i) -> double {  // scaled (noised) score
        double v = x[i];
        if (nz) v = v + p.noise_scale * nz[i];  // training_mask: add(u, noise_scale * gumbel)
        return v / tau;
    };
    if (tid == 0) s_bad = 0;
    __syncthreads();
    // clamp_budget (:27-33): k strictly inside (0, n)
    const double k = p.k[seg];
    if (!(k > 0.0) || !(k < (double)n)) {
        if (tid == 0) latch_error(p.err, LKV_ERR_BUDGET, seg);
        return;
    }
    const double eps = fmin(1e-3, 0.01 * n);
    const double kc = fmin(fmax(k, eps), (double)n - eps);
    double lo_v = CUDART_INF, hi_v = -CUDART_INF;
    for (int i = tid; i < n; i += kThreads) {
        const double v = sc(i);
        if (!isfinite(v)) s_bad = 1;
        else if (n >= 2 && fabs(v) > 1e300) s_bad = 2;  // solve_threshold's overflow guard (:63)
        lo_v = fmin(lo_v, v);
        hi_v = fmax(hi_v, v);
    }
    __syncthreads();
    if (s_bad) {
        if (tid == 0) latch_error(p.err, s_bad == 1 ? LKV_ERR_NUMERIC : LKV_ERR_OVERFLOW_GUARD, seg);
        return;
    }
    const double mn = -block_max(-lo_v, red), mx = block_max(hi_v, red);
    double lambda;
    if (n == 1) {  // :119-131: the constraint pins the single value to kc
        const double z = kc >= 0.5 ? -log(2.0 * (1.0 - kc)) : log(2.0 * kc);
        lambda = mx - z;
    } else {
        // 1. bisection on g(lam) = sum F(s - lam) - kc (decreasing in lam)
        double lo = mn - 40.0, hi = mx + 40.0;
        for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (lo + hi);
            if (!(mid > lo && mid < hi)) break;  // bracket a few ulps wide
            double part = 0.0;
            int inside = 0;
            for (int i = tid; i < n; i += kThreads) {
                const double v = sc(i);
                part += laplace_cdf(v - mid);
                inside |= (v > lo && v <= hi);
            }
            const double g = block_sum(part, red) - kc;
            const int any_inside = __syncthreads_or(inside);
            if (!any_inside) break;  // no sample in (lo, hi]: the split m is fixed
            if (g > 0.0) lo = mid;
            else hi = mid;
        }
        const double lam0 = 0.5 * (lo + hi);
        // 2. closed form on the split m = #{s > lam0} (soft_topk.cpp:38-48, log-space sums)
        double cnt = 0.0, m1 = -CUDART_INF, m2 = -CUDART_INF;
        for (int i = tid; i < n; i += kThreads) {
            const double v = sc(i);
            if (v > lam0) {
                cnt += 1.0;
                m1 = fmax(m1, -v);
            } else {
                m2 = fmax(m2, v);
            }
        }
        const int m = (int)block_sum(cnt, red);
        const double M1 = block_max(m1, red), M2 = block_max(m2, red);
        double s1 = 0.0, s2 = 0.0;
        for (int i = tid; i < n; i += kThreads) {
            const double v = sc(i);
            if (v > lam0) s1 += exp(-v - M1);
            else s2 += exp(v - M2);
        }
        s1 = block_sum(s1, red);
        s2 = block_sum(s2, red);
        const double l1 = m > 0 ? M1 + log(s1) : -CUDART_INF, l2 = m < n ? M2 + log(s2) : -CUDART_INF;
        lambda = candidate_lambda(m, n, kc, l1, l2);
        if (!isfinite(lambda)) lambda = lam0;
    }
    // values, density, constraint check (:145-162)
    const double vhi = 1.0 - DBL_EPSILON / 2;
    double sum = 0.0;
    double* vals = p.values + (size_t)seg * p.ld;
    double* dens = p.density ? p.density + (size_t)seg * p.ld : nullptr;
    float* v32 = p.values_f32 ? p.values_f32 + (size_t)seg * p.ld : nullptr;
    for (int i = tid; i < n; i += kThreads) {
        const double z = n == 1 ? (kc >= 0.5 ? -log(2.0 * (1.0 - kc)) : log(2.0 * kc)) : sc(i) - lambda;
        const double v = n == 1 ? kc : fmin(fmax(laplace_cdf(z), DBL_MIN), vhi);
        vals[i] = v;
        if (dens) dens[i] = fmax(0.5 * exp(-fabs(z)), DBL_MIN);
        if (v32) v32[i] = (float)v;
        sum += v;
    }
    sum = block_sum(sum, red);
    if (tid == 0) {
        if (p.lambda) p.lambda[seg] = lambda;
        if (fabs(sum - kc) > 1e-9 * n) latch_error(p.err, LKV_ERR_NUMERIC, seg);  // constraint violated
    }
}

__global__ void __launch_bounds__(kThreads) vjp_kernel(const __grid_constant__ SoftTopKParams p) {
    __shared__ double red[33];
    const int seg = blockIdx.x, n = p.n, tid = threadIdx.x;
    const double* d = p.density + (size_t)seg * p.ld;
    const double* u = p.upstream + (size_t)seg * p.ld;
    double* gx = p.grad_x + (size_t)seg * p.ld;
    if (n == 1) {  // :172
        if (tid == 0) {
            gx[0] = 0.0;
            p.grad_k[seg] = 1.0;
        }
        return;
    }
    double sf = 0.0, dot = 0.0;
    for (int i = tid; i < n; i += kThreads) {
        sf += d[i];
        dot += u[i] * d[i];
    }
    // one tree for both sums: u == 1 gives dot == sum exactly (zero gradient, unit grad_k)
    sf = block_sum(sf, red);
    dot = block_sum(dot, red);
    const double mean = dot / sf;
    for (int i = tid; i < n; i += kThreads) gx[i] = d[i] * (u[i] - mean) / p.tau;
    if (tid == 0) p.grad_k[seg] = mean;
}

}  // namespace stk

cudaError_t launch_soft_topk_fwd(const SoftTopKParams& p, cudaStream_t stream) {
    stk::fwd_kernel<<<p.n_seg, stk::kThreads, 0, stream>>>(p);
    note_launches(1);
    return cudaGetLastError();
}
cudaError_t launch_soft_topk_vjp(const SoftTopKParams& p, cudaStream_t stream) {
    stk::vjp_kernel<<<p.n_seg, stk::kThreads, 0, stream>>>(p);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace lkv_dev
