// f64.cu -- reference-precision (fp64) device operators behind the declaration-compatible C++
// API (include/lkv/*.hpp).  The reference computes everything in float64 on the host
// (tensor.hpp:3); a caller that keeps the reference's signatures gets the reference's precision
// here, on the B200: SIMT fp64 kernels, each output computed in a fixed order that does not
// depend on how many rows a call carries, so a prefill over t rows and a decode step over one
// row produce bit-identical per-row results (the property test_evictsim.cpp:82-117 relies on).
//
//   f64_gemm_kernel       C (+)= A B                    matmul (tensor.cpp:276-297)
//   f64_rmsnorm_kernel    x * gain / rms                rmsnorm (tensor.cpp:540-566), model.cpp:48-53
//   f64_rope_kernel       rotary pairs at pos0 + row    rope (tensor.cpp:586-623), model.cpp:38-46
//   f64_attention_kernel  masked softmax attention      masked_attention_dense (attention.cpp:46-94)
//   f64_swiglu_kernel     silu(g) * u                   model.cpp:112-115, 275-278
//   f64_embed_kernel      table rows                    embedding_rows (tensor.cpp:625-640)
//   f64_split_heads       [t][H*d] -> [H][t][d]          slice_lastdim per head (model.cpp:88-93)
//   f64_scorer_kernel     act(x W1 + b1) . w2           mlp2_forward (policy.cpp:30-34), token_scores
//   f64_select_kernel     top-b, ties -> lowest index   hard_topk (soft_topk.cpp:191-201)
#include <math.h>

#include "kernels.cuh"

namespace lkv_dev {

// ---- GEMM ------------------------------------------------------------------------------------
constexpr int kGT = 16;
__global__ void __launch_bounds__(kGT * kGT) f64_gemm_kernel(const F64GemmParams p) {
    __shared__ double sa[kGT][kGT + 1];
    __shared__ double sb[kGT][kGT + 1];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int row = blockIdx.y * kGT + ty, col = blockIdx.x * kGT + tx;
    double acc = 0.0;
    for (int k0 = 0; k0 < p.K; k0 += kGT) {
        sa[ty][tx] = (row < p.M && k0 + tx < p.K) ? p.A[(size_t)row * p.lda + k0 + tx] : 0.0;
        sb[ty][tx] = (k0 + ty < p.K && col < p.N) ? p.B[(size_t)(k0 + ty) * p.ldb + col] : 0.0;
        __syncthreads();
        const int kn = min(kGT, p.K - k0);
        for (int k = 0; k < kn; ++k) acc = fma(sa[ty][k], sb[k][tx], acc);  // ascending k, any M
        __syncthreads();
    }
    if (row < p.M && col < p.N) {
        double* c = p.C + (size_t)row * p.ldc + col;
        *c = p.accumulate ? *c + acc : acc;
    }
}

// ---- rmsnorm: one CTA per row, fixed reduction tree ----------------------------------------
constexpr int kRowThreads = 128;
__device__ __forceinline__ double block_sum_f64(double v, double* s_red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) s_red[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < kRowThreads / 32; ++i) t += s_red[i];
    __syncthreads();
    return t;
}

__global__ void __launch_bounds__(kRowThreads) f64_rmsnorm_kernel(int cols, const double* x, int64_t ldx,
                                                                  const double* gain, double eps, double* out,
                                                                  int64_t ldo) {
    __shared__ double s_red[kRowThreads / 32];
    const double* xr = x + (size_t)blockIdx.x * ldx;
    double ms = 0.0;
    for (int c = threadIdx.x; c < cols; c += kRowThreads) ms += xr[c] * xr[c];
    ms = block_sum_f64(ms, s_red);
    const double inv = 1.0 / sqrt(ms / cols + eps);
    double* o = out + (size_t)blockIdx.x * ldo;
    for (int c = threadIdx.x; c < cols; c += kRowThreads) o[c] = xr[c] * gain[c] * inv;
}

// ---- rope: row r at absolute position pos0 + r, every head of the row ------------------------
__global__ void f64_rope_kernel(int rows, int n_heads, int d, double* x, int64_t ldx, int pos0, double base) {
    const int half = d / 2;
    const int64_t total = (int64_t)rows * n_heads * half;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(i % half);
        const int64_t rh = i / half;
        const int h = (int)(rh % n_heads);
        const int r = (int)(rh / n_heads);
        const double th = (double)(pos0 + r) * pow(base, -2.0 * j / d);
        const double cs = cos(th), sn = sin(th);
        double* v = x + (size_t)r * ldx + (size_t)h * d + 2 * j;
        const double a = v[0], b = v[1];
        v[0] = a * cs - b * sn;
        v[1] = a * sn + b * cs;
    }
}

// ---- attention: one warp per (query head, query row) -----------------------------------------
// attention.cpp:46-94 per row: scores s_j = scale * q.k_j over the admissible keys, mx = max,
// p_raw_j = exp(s_j - mx) / z_raw, w_j = p_raw_j * mask_j, z = sum w, out = sum (w_j / z) v_j.
// Lane l owns keys j = l (mod 32) for the reductions (fixed butterfly); the output columns are
// accumulated in ascending key order, so the result for a row depends only on its keys.
__device__ __forceinline__ double warp_max_f64(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum_f64(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(128) f64_attention_kernel(const F64AttnParams p) {
    const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (warp >= p.n_qh * p.n_q) return;
    const int h = warp / p.n_q, r = warp - h * p.n_q;
    const int kvh = h / p.G;
    const int d = p.d;
    const double* q = p.q + (size_t)r * p.ldq + (size_t)h * d;
    const double* K = p.k + (size_t)kvh * d;
    const double* V = p.v + (size_t)kvh * d;
    const double* mask = p.mask ? p.mask + (size_t)kvh * p.mask_ld : nullptr;
    const int pos = p.qpo + r;
    const int end = p.causal ? min(p.t, pos + 1) : p.t;
    auto score = [&](int j) {
        const double* kj = K + (size_t)j * p.ldk;
        double s = 0.0;
        for (int c = 0; c < d; ++c) s = fma(q[c], kj[c], s);
        return p.scale * s;
    };
    auto mask_at = [&](int j) { return (p.self_keep && j == pos) ? 1.0 : (mask ? mask[j] : 1.0); };
    double mx = -INFINITY;
    for (int j = lane; j < end; j += 32) mx = fmax(mx, score(j));
    mx = warp_max_f64(mx);
    double z_raw = 0.0;
    for (int j = lane; j < end; j += 32) z_raw += exp(score(j) - mx);
    z_raw = warp_sum_f64(z_raw);
    double z = 0.0;
    for (int j = lane; j < end; j += 32) z += exp(score(j) - mx) / z_raw * mask_at(j);
    z = warp_sum_f64(z);
    if (!(z > 1e-300)) {  // attention.cpp:83-85
        if (lane == 0) latch_error(p.err, LKV_ERR_DEGENERATE_MASK, warp);
        return;
    }
    const size_t prow = ((size_t)h * p.n_q + r) * p.t;
    if (p.renorm && lane == 0) p.renorm[(size_t)h * p.n_q + r] = z;
    // output columns c = lane + 32 i (d <= 256)
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0;
    for (int j0 = 0; j0 < end; j0 += 32) {
        const int j = j0 + lane;
        double w = 0.0;
        if (j < end) {
            const double pr = exp(score(j) - mx) / z_raw;
            const double wt = pr * mask_at(j);
            w = wt / z;
            if (p.p_raw) p.p_raw[prow + j] = pr;
            if (p.p) p.p[prow + j] = w;
        }
        const int nj = min(32, end - j0);
        for (int u = 0; u < nj; ++u) {
            const double wu = __shfl_sync(0xffffffffu, w, u);
            const double* vj = V + (size_t)(j0 + u) * p.ldk;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int c = lane + 32 * i;
                if (c < d) acc[i] = fma(wu, vj[c], acc[i]);
            }
        }
    }
    double* o = p.out + (size_t)r * p.ldo + (size_t)h * d;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int c = lane + 32 * i;
        if (c < d) o[c] = acc[i];
    }
    if (p.p_raw || p.p) {  // zero the inadmissible tail (attention.cpp:64-66: weights start at zero)
        for (int j = end + lane; j < p.t; j += 32) {
            if (p.p_raw) p.p_raw[prow + j] = 0.0;
            if (p.p) p.p[prow + j] = 0.0;
        }
    }
}

// ---- elementwise ---------------------------------------------------------------------------------
__global__ void f64_swiglu_kernel(int64_t n, const double* gate, const double* up, double* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = gate[i];
        out[i] = v / (1.0 + exp(-v)) * up[i];  // tensor.cpp:377 silu, then mul (model.cpp:114-115, 277)
    }
}

__global__ void f64_embed_kernel(const int32_t* tokens, int n, const double* table, int dm, int vocab, double* out,
                                 ErrWord* err) {
    const int64_t total = (int64_t)n * dm;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / dm), c = (int)(i % dm);
        const int tok = tokens[r];
        if (tok < 0 || tok >= vocab) {
            if (c == 0) latch_error(err, LKV_ERR_CONTRACT, r);
            continue;
        }
        out[i] = table[(size_t)tok * dm + c];
    }
}

__global__ void f64_split_heads_kernel(int t, int H, int d, const double* x, int64_t ldx, double* out, int64_t T) {
    const int64_t total = (int64_t)t * H * d;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % d);
        const int64_t rh = i / d;
        const int h = (int)(rh % H);
        const int r = (int)(rh / H);
        out[((size_t)h * T + r) * d + c] = x[(size_t)r * ldx + (size_t)h * d + c];
    }
}

// ---- LKV-T scorer, fp64 --------------------------------------------------------------------------
// u = act([k ; v] W1 + b1) . w2 (policy.cpp:30-34,131-136): per row, hidden unit j accumulates
// its dot product over the input in ascending order (k part, then v part), adds b1, activates;
// the row's score sums the hidden units in ascending order.
constexpr int kScRows = 8;
__global__ void __launch_bounds__(128) f64_scorer_kernel(const F64ScorerParams p) {
    extern __shared__ double smem[];
    const int in = p.in_mode * p.d;
    double* sx = smem;                        // [kScRows][in]
    double* sh = smem + kScRows * in;         // [kScRows][hidden]
    const int r0 = blockIdx.x * kScRows;
    const int nr = min(kScRows, p.t - r0);
    for (int i = threadIdx.x; i < nr * in; i += blockDim.x) {
        const int r = i / in, c = i - r * in;
        sx[i] = c < p.d ? p.k[(size_t)(r0 + r) * p.ldk + c] : p.v[(size_t)(r0 + r) * p.ldv + c - p.d];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < p.hidden; j += blockDim.x) {
        for (int r = 0; r < nr; ++r) {
            const double* x = sx + r * in;
            double acc = 0.0;
            for (int c = 0; c < in; ++c) acc = fma(x[c], p.w1[(size_t)c * p.hidden + j], acc);
            const double h = acc + p.b1[j];
            sh[r * p.hidden + j] = p.act == LKV_ACT_SILU ? h / (1.0 + exp(-h)) : 0.5 * h * (1.0 + erf(h * M_SQRT1_2));
        }
    }
    __syncthreads();
    if (threadIdx.x < nr) {
        const int r = threadIdx.x;
        double u = 0.0;
        for (int j = 0; j < p.hidden; ++j) u = fma(sh[r * p.hidden + j], p.w2[j], u);
        if (!isfinite(u)) latch_error(p.err, LKV_ERR_NUMERIC, r0 + r);  // check_finite (tensor.cpp:34-40)
        p.u[r0 + r] = u;
    }
}

// ---- top-b over fp64 scores: one CTA per head ---------------------------------------------------
// Order-preserving 64-bit key (-0.0 == +0.0, as x[a] > x[b] treats them); 8 radix passes of 8
// bits find the b-th largest key T and how many T-equal rows to keep (the lowest indices, the
// stable sort's tie rule); one ordered pass writes the kept positions ascending.
__device__ __forceinline__ unsigned long long f64_key(double x) {
    if (x == 0.0) x = 0.0;
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

constexpr int kF64SelThreads = 512;
__global__ void __launch_bounds__(kF64SelThreads) f64_select_kernel(const F64SelectParams p) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_scan[kF64SelThreads / 32 + 1];
    __shared__ unsigned long long s_prefix;
    __shared__ uint32_t s_rem, s_carry_eq, s_carry_keep;
    __shared__ int s_bad;
    const int head = blockIdx.x;
    const int t = p.t;
    const double* x = p.scores + (size_t)head * p.ld;
    const int b = p.budgets[head];
    if (b < 0 || b > t) {  // soft_topk.cpp:193
        if (threadIdx.x == 0) latch_error(p.err, LKV_ERR_BUDGET, head);
        return;
    }
    if (threadIdx.x == 0) {
        s_prefix = 0;
        s_rem = (uint32_t)b;
        s_bad = 0;
        s_carry_eq = 0;
        s_carry_keep = 0;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < t; j += kF64SelThreads)
        if (isnan(x[j])) s_bad = 1;
    __syncthreads();
    if (s_bad) {
        if (threadIdx.x == 0) latch_error(p.err, LKV_ERR_NUMERIC, head);
        return;
    }
    unsigned long long key_t = 0;
    uint32_t need_eq = 0;
    const bool all = b == t;
    if (b > 0 && !all) {
        for (int pass = 7; pass >= 0; --pass) {
            const int shift = pass * 8;
            for (int i = threadIdx.x; i < 256; i += kF64SelThreads) hist[i] = 0;
            __syncthreads();
            const unsigned long long prefix = s_prefix;
            for (int j = threadIdx.x; j < t; j += kF64SelThreads) {
                const unsigned long long k = f64_key(x[j]);
                if (pass == 7 || (k >> (shift + 8)) == (prefix >> (shift + 8)))
                    atomicAdd(&hist[(k >> shift) & 255u], 1u);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t above = 0, rem = s_rem;
                int bin = 255;
                for (; bin >= 0; --bin) {
                    if (above + hist[bin] >= rem) break;
                    above += hist[bin];
                }
                s_prefix = prefix | ((unsigned long long)bin << shift);
                s_rem = rem - above;
            }
            __syncthreads();
        }
        key_t = s_prefix;
        need_eq = s_rem;
    }
    if (b == 0) {
        if (threadIdx.x == 0) p.lens[head] = 0;
        return;
    }
    // ordered emit: keep key > T, or key == T while the running equal rank < need_eq
    int32_t* out = p.positions + p.offsets[head];
    for (int j0 = 0; j0 < t; j0 += kF64SelThreads) {
        const int j = j0 + threadIdx.x;
        bool gt = false, eq = false;
        if (j < t) {
            if (all) {
                gt = true;
            } else {
                const unsigned long long k = f64_key(x[j]);
                gt = k > key_t;
                eq = k == key_t;
            }
        }
        uint32_t tot;
        const uint32_t eq_before = s_carry_eq + block_exclusive_scan<kF64SelThreads>(eq ? 1u : 0u, s_scan, &tot);
        const bool keep = gt || (eq && eq_before < need_eq);
        uint32_t tot_keep;
        const uint32_t slot = s_carry_keep + block_exclusive_scan<kF64SelThreads>(keep ? 1u : 0u, s_scan, &tot_keep);
        if (keep) out[slot] = j;
        __syncthreads();
        if (threadIdx.x == 0) {
            s_carry_eq += tot;
            s_carry_keep += tot_keep;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        p.lens[head] = b;
        if (s_carry_keep != (uint32_t)b) latch_error(p.err, LKV_ERR_NUMERIC, head);
    }
}

// ---- launchers -----------------------------------------------------------------------------------
static int grid_for(int64_t n, int threads) {
    const int64_t g = (n + threads - 1) / threads;
    return (int)(g < 1 ? 1 : (g > 65535 ? 65535 : g));
}

cudaError_t launch_f64_gemm(const F64GemmParams& p, cudaStream_t s) {
    if (p.M == 0 || p.N == 0) return cudaSuccess;
    f64_gemm_kernel<<<dim3((p.N + kGT - 1) / kGT, (p.M + kGT - 1) / kGT), dim3(kGT, kGT), 0, s>>>(p);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_f64_rmsnorm(int rows, int cols, const double* x, int64_t ldx, const double* gain, double eps,
                               double* out, int64_t ldo, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    f64_rmsnorm_kernel<<<rows, kRowThreads, 0, s>>>(cols, x, ldx, gain, eps, out, ldo);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_f64_rope(int rows, int n_heads, int d, double* x, int64_t ldx, int pos0, double base,
                            cudaStream_t s) {
    const int64_t n = (int64_t)rows * n_heads * (d / 2);
    if (n == 0) return cudaSuccess;
    f64_rope_kernel<<<grid_for(n, 256), 256, 0, s>>>(rows, n_heads, d, x, ldx, pos0, base);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_f64_attention(const F64AttnParams& p, cudaStream_t s) {
    const int64_t warps = (int64_t)p.n_qh * p.n_q;
    if (warps == 0) return cudaSuccess;
    f64_attention_kernel<<<(unsigned)((warps + 3) / 4), 128, 0, s>>>(p);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_f64_swiglu(int64_t n, const double* gate, const double* up, double* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    f64_swiglu_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, gate, up, out);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_f64_embed(const int32_t* tokens, int n, const double* table, int dm, int vocab, double* out,
                             ErrWord* err, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    f64_embed_kernel<<<grid_for((int64_t)n * dm, 256), 256, 0, s>>>(tokens, n, table, dm, vocab, out, err);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_f64_split_heads(int t, int H, int d, const double* x, int64_t ldx, double* out, int64_t T,
                                   cudaStream_t s) {
    const int64_t n = (int64_t)t * H * d;
    if (n == 0) return cudaSuccess;
    f64_split_heads_kernel<<<grid_for(n, 256), 256, 0, s>>>(t, H, d, x, ldx, out, T);
    note_launches(1);
    return cudaGetLastError();
}

size_t f64_scorer_smem(int in, int hidden) { return (size_t)kScRows * (in + hidden) * sizeof(double); }

cudaError_t launch_f64_scorer(const F64ScorerParams& p, cudaStream_t s) {
    if (p.t == 0) return cudaSuccess;
    const size_t smem = f64_scorer_smem(p.in_mode * p.d, p.hidden);
    cudaError_t e = cudaFuncSetAttribute(f64_scorer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    f64_scorer_kernel<<<(p.t + kScRows - 1) / kScRows, 128, smem, s>>>(p);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_f64_select(const F64SelectParams& p, int n_heads, cudaStream_t s) {
    if (n_heads == 0) return cudaSuccess;
    f64_select_kernel<<<n_heads, kF64SelThreads, 0, s>>>(p);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace lkv_dev
