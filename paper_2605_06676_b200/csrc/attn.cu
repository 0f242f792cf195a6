// attn.cu -- training-time multiplicative-mask attention, forward + backward.
//
// Reference: masked_attention_dense / masked_attention_blocked / masked_attention_vjp
// (attention.cpp:46-201, attention.hpp:20-74).  Per query row r (absolute position
// pos = query_pos_offset + r), over the admissible keys j (j < t, and j <= pos when causal):
//   p_raw = softmax(s),  s = scale * q.k;   p~ = p_raw * m_j;   p = p~ / sum(p~);   out = p V
// with m_j = 1 at j == pos when self_always_retained; a row whose masked mass vanishes raises
// degenerate_mask_error.  The mask multiplies AFTER exponentiation (never an additive bias).
//
// Flash formulation (one pass, nothing t x t is materialised):
//   forward keeps, per row, the running max M of the admissible raw scores, the masked sum
//   L = sum exp(s - M) m_j (and the raw sum, for the degenerate check) and O = sum exp(s - M) m_j v_j;
//   it stores lse = M + log L (log2 domain), so p = exp(s - lse) m_j exactly as above.
//   backward (the reference's vjp, attention.cpp:145-201, reduced analytically):
//     w = dO V^T,  D_r = <dO_r, O_r> (= sum_j w_rj p_rj),
//     dS = p (w - D)            (the reference's dp_dot = sum_j d_praw p_raw is 0 since sum p = 1)
//     dV = p^T dO,  dQ = scale dS K,  dK = scale dS^T Q,
//     dmask_j = sum_r exp(s_rj - lse_r) (w_rj - D_r)   (= d p~ . p_raw; self rows excluded)
// GQA: query head h reads kv head h / G; dK, dV, dmask sum over the G query heads of a group
// (what the reference's autodiff accumulates over forward_masked's per-query-head calls,
// model.cpp:100-112).
//
// B200 design (bf16 inputs, fp32 accumulate, head_dim 128):
//   * forward: CTA = 64 queries of one (batch, q head), 4 consumer warps x 16 rows + 1 TMA
//     producer warp streaming 64-key K/V tiles (128 B swizzle) through a 3-stage mbarrier ring;
//     S = Q K^T and O += P V on tensor cores (mma.sync m16n8k16 + ldmatrix); causal tiles past
//     the block's last admissible key are never loaded;
//   * backward, two kernels with no atomics (deterministic):
//     dQ:  CTA = 64 queries (Q, dO in smem), K/V tiles streamed as in the forward; recomputes S, P,
//          dP = dO V^T, dS and accumulates dS K;
//     dKV: CTA = 64 keys (K, V in smem for the CTA's life), 4 warps x 16 keys, streams 32-query
//          Q/dO tiles of all G query heads; recomputes S^T, dP^T and accumulates dV, dK and the
//          mask gradient per key in registers.
// fp32 inputs run SIMT kernels (exact two-pass softmax, the 1e-5 correctness path).
#include <math.h>

#include <algorithm>

#include "kernels.cuh"

namespace lkv_dev {
namespace attn {

constexpr int kD = 128;
constexpr int kQB = 64;      // forward / dQ: query rows per CTA
constexpr int kKB = 64;      // key rows per tile (forward / dQ) and per CTA (dKV)
constexpr int kQT = 32;      // dKV: query rows per streamed tile
constexpr int kStages = 3;
constexpr int kConsumers = 4;
constexpr int kThreads = (kConsumers + 1) * 32;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }
__device__ __forceinline__ float fast_exp2(float x) {  // MUFU.EX2 (2 ulp); ex2(-inf) = +0
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// byte offset of (row, 16-byte chunk q in 0..15) of a ROWS x 256 B tile stored as two
// ROWS x 128 B TMA boxes with the 128-byte swizzle
template <int ROWS>
__device__ __forceinline__ uint32_t sw(int row, int q) {
    return (uint32_t)((q >> 3) * (ROWS * 128) + row * 128 + (((q & 7) ^ (row & 7)) << 4));
}
// load a ROWS x 128 bf16 tile (two 64-column boxes) at global row y
template <int ROWS>
__device__ __forceinline__ void tma_tile(unsigned char* dst, const CUtensorMap* m, uint64_t* bar, int y, uint64_t pol) {
    tma_load_2d(dst, m, bar, 0, y, pol);
    tma_load_2d(dst + ROWS * 128, m, bar, 64, y, pol);
}

// A fragments (16 rows x 16 k) of a swizzled ROWS-row tile, rows r0..r0+15, k-step kk
template <int ROWS>
__device__ __forceinline__ void frag_a(uint32_t base, int r0, int kk, int lane, uint32_t (&a)[4]) {
    const int row = r0 + (lane & 7) + (((lane >> 3) & 1) << 3);
    ldsm_x4(base + sw<ROWS>(row, kk * 2 + (lane >> 4)), a);
}
// B fragments for two n8 tiles whose n index runs over tile ROWS r0..r0+15 ("K^T" operand:
// element (k = feature, n = row)); b[0],b[1] -> n-tile rows r0..r0+7, b[2],b[3] -> r0+8..r0+15
template <int ROWS>
__device__ __forceinline__ void frag_bn(uint32_t base, int r0, int kk, int lane, uint32_t (&b)[4]) {
    const int j = lane >> 3;
    ldsm_x4(base + sw<ROWS>(r0 + ((j >> 1) << 3) + (lane & 7), kk * 2 + (j & 1)), b);
}
// B fragments for two n8 tiles of FEATURES (n = feature chunk n2*16..+15) with k running over
// tile rows r0..r0+15 ("V" operand: element (k = row, n = feature))
template <int ROWS>
__device__ __forceinline__ void frag_bk(uint32_t base, int r0, int n2, int lane, uint32_t (&b)[4]) {
    const int j = lane >> 3;
    ldsm_x4_t(base + sw<ROWS>(r0 + ((j & 1) << 3) + (lane & 7), n2 * 2 + (j >> 1)), b);
}

// mask values of key columns j, j+1 (j even): 0 past t_k, 1 without a mask
__device__ __forceinline__ float2 load_mask2(const float* mask, bool vec, int j, int t_k) {
    if (!mask) return make_float2(1.f, 1.f);
    if (vec && j + 1 < t_k) return __ldg(reinterpret_cast<const float2*>(mask + j));
    return make_float2(j < t_k ? __ldg(mask + j) : 0.f, j + 1 < t_k ? __ldg(mask + j + 1) : 0.f);
}

struct Geo {
    int n_q_heads, n_kv_heads, G, t_q, t_k, causal, pos_offset, self_keep;
    float c;      // scale * log2(e)
    float scale;  // natural scale (gradient factors)
};

__device__ __forceinline__ int key_end(const Geo& g, int q_last) {  // one past the last admissible key
    return g.causal ? min(g.t_k, g.pos_offset + q_last + 1) : g.t_k;
}
__device__ __forceinline__ bool admissible(const Geo& g, int j, int r) {
    return j < g.t_k && r < g.t_q && (!g.causal || j <= g.pos_offset + r);
}
__device__ __forceinline__ float mask_eff(const Geo& g, const float* mask, int j, int r) {
    if (g.self_keep && j == g.pos_offset + r) return 1.f;
    return mask ? __ldg(mask + j) : 1.f;
}

// =====================================================================================================
// forward
// =====================================================================================================
__global__ void __launch_bounds__(kThreads, 2)
    fwd_bf16_kernel(const __grid_constant__ AttnParams p, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tq) {
    constexpr int kStageBytes = 2 * kKB * 256;
    extern __shared__ unsigned char smem_dyn[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
    unsigned char* qs = smem + kStages * kStageBytes;  // Q tile [64][256 B]
    uint64_t* full = reinterpret_cast<uint64_t*>(qs + kQB * 256);
    uint64_t* empty = full + kStages;
    uint64_t* qbar = empty + kStages;
    const Geo g{p.n_q_heads, p.n_kv_heads, p.n_q_heads / p.n_kv_heads, p.t_q, p.t_k, p.causal, p.pos_offset,
                p.self_keep, p.scale * kLog2e, p.scale};
    const int b = blockIdx.z, qh = blockIdx.y, kvh = qh / g.G;
    const int q0 = blockIdx.x * kQB;
    const int kend = key_end(g, min(g.t_q, q0 + kQB) - 1);
    const int ntiles = kend > 0 ? (kend + kKB - 1) / kKB : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kConsumers);
        }
        mbar_init(qbar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    const size_t kv_row0 = ((size_t)b * g.n_kv_heads + kvh) * g.t_k;
    if (warp == kConsumers) {
        if (lane == 0) {
            tma_prefetch_desc(&tk);
            tma_prefetch_desc(&tv);
            const uint64_t pol = l2_policy_evict_last();  // K/V tiles are re-read by every query block
            mbar_arrive_expect_tx(qbar, kQB * 256);
            tma_tile<kQB>(qs, &tq, qbar, (int)(((size_t)b * g.n_q_heads + qh) * g.t_q + q0), pol);
            for (int t = 0; t < ntiles; ++t) {
                const int st = t % kStages;
                if (t >= kStages) mbar_wait(&empty[st], ((t / kStages) - 1) & 1);
                mbar_arrive_expect_tx(&full[st], kStageBytes);
                unsigned char* dst = smem + st * kStageBytes;
                tma_tile<kKB>(dst, &tk, &full[st], (int)(kv_row0 + t * kKB), pol);
                tma_tile<kKB>(dst + kKB * 256, &tv, &full[st], (int)(kv_row0 + t * kKB), pol);
            }
        }
        return;
    }
    const int gq = lane >> 2, cq = (lane & 3) * 2;
    const int r_lo = q0 + warp * 16 + gq, r_hi = r_lo + 8;  // this thread's two query rows
    const float* mask = p.mask ? p.mask + ((size_t)b * g.n_kv_heads + kvh) * g.t_k : nullptr;
    const bool mask_vec = (reinterpret_cast<uintptr_t>(mask) & 7) == 0;
    const uint32_t qsb = smem_u32(qs);
    mbar_wait(qbar, 0);
    float o[16][4];
#pragma unroll
    for (int n = 0; n < 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;
    for (int t = 0; t < ntiles; ++t) {
        const int st = t % kStages;
        mbar_wait(&full[st], (t / kStages) & 1);
        const uint32_t kb = smem_u32(smem + st * kStageBytes), vb = kb + kKB * 256;
        const int j0 = t * kKB;
        float s[8][4];
#pragma unroll
        for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            uint32_t qa[4];
            frag_a<kQB>(qsb, warp * 16, kk, lane, qa);
#pragma unroll
            for (int np = 0; np < 4; ++np) {
                uint32_t bf[4];
                frag_bn<kKB>(kb, np * 16, kk, lane, bf);
                mma(s[2 * np], qa, bf[0], bf[1]);
                mma(s[2 * np + 1], qa, bf[2], bf[3]);
            }
        }
        // interior tiles (every key admissible for all 16 rows of this warp) skip the per-element
        // admissibility tests; only the causal diagonal and the ragged ends take the slow path
        const int wr0 = q0 + warp * 16;
        const bool interior = j0 + kKB <= g.t_k && wr0 + 16 <= g.t_q && (!g.causal || j0 + kKB - 1 <= g.pos_offset + wr0) &&
                              !(g.self_keep && j0 + kKB - 1 >= g.pos_offset + wr0);
        // this thread's 16 mask values (the same key columns for both rows)
        float mx_lo = -INFINITY, mx_hi = -INFINITY;
        if (interior) {
#pragma unroll
            for (int n = 0; n < 8; ++n)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    s[n][e] *= g.c;
                    s[n][2 + e] *= g.c;
                    mx_lo = fmaxf(mx_lo, s[n][e]);
                    mx_hi = fmaxf(mx_hi, s[n][2 + e]);
                }
        } else {
#pragma unroll
            for (int n = 0; n < 8; ++n)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = j0 + n * 8 + cq + e;
                    s[n][e] = admissible(g, j, r_lo) ? s[n][e] * g.c : -INFINITY;
                    s[n][2 + e] = admissible(g, j, r_hi) ? s[n][2 + e] * g.c : -INFINITY;
                    mx_lo = fmaxf(mx_lo, s[n][e]);
                    mx_hi = fmaxf(mx_hi, s[n][2 + e]);
                }
        }
        mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 1));
        mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 2));
        mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 1));
        mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 2));
        const float mn_lo = fmaxf(m_lo, mx_lo), mn_hi = fmaxf(m_hi, mx_hi);
        const float a_lo = mn_lo == -INFINITY ? 1.f : fast_exp2(m_lo - mn_lo);
        const float a_hi = mn_hi == -INFINITY ? 1.f : fast_exp2(m_hi - mn_hi);
        m_lo = mn_lo;
        m_hi = mn_hi;
        // a row with no admissible key yet has mn = -inf: exp2(-inf - -inf) would be NaN
        const float sub_lo = mn_lo == -INFINITY ? 0.f : mn_lo, sub_hi = mn_hi == -INFINITY ? 0.f : mn_hi;
        float sl = 0.f, sh = 0.f;
#pragma unroll
        for (int n = 0; n < 8; ++n) {
            const float2 m2 = load_mask2(mask, mask_vec, j0 + n * 8 + cq, g.t_k);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                float ml = e ? m2.y : m2.x, mh = ml;
                if (!interior && g.self_keep) {
                    const int j = j0 + n * 8 + cq + e;
                    if (j == g.pos_offset + r_lo) ml = 1.f;
                    if (j == g.pos_offset + r_hi) mh = 1.f;
                }
                s[n][e] = fast_exp2(s[n][e] - sub_lo) * ml;  // exp2(-inf) = 0 for inadmissible keys
                s[n][2 + e] = fast_exp2(s[n][2 + e] - sub_hi) * mh;
                sl += s[n][e];
                sh += s[n][2 + e];
            }
        }
        l_lo = l_lo * a_lo + sl;
        l_hi = l_hi * a_hi + sh;
#pragma unroll
        for (int n = 0; n < 16; ++n) {
            o[n][0] *= a_lo;
            o[n][1] *= a_lo;
            o[n][2] *= a_hi;
            o[n][3] *= a_hi;
        }
        // O += P V  (P: 16 rows x 64 keys = 4 k16 steps)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            uint32_t pa[4] = {pack2(s[2 * kk][0], s[2 * kk][1]), pack2(s[2 * kk][2], s[2 * kk][3]),
                              pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]), pack2(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
            for (int n2 = 0; n2 < 8; ++n2) {
                uint32_t bf[4];
                frag_bk<kKB>(vb, kk * 16, n2, lane, bf);
                mma(o[2 * n2], pa, bf[0], bf[1]);
                mma(o[2 * n2 + 1], pa, bf[2], bf[3]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
#pragma unroll
    for (int x = 1; x <= 2; x <<= 1) {
        l_lo += __shfl_xor_sync(0xffffffffu, l_lo, x);
        l_hi += __shfl_xor_sync(0xffffffffu, l_hi, x);
    }
    const size_t row_base = ((size_t)b * g.n_q_heads + qh) * g.t_q;
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int r = h ? r_hi : r_lo;
        if (r >= g.t_q) continue;
        const float l = h ? l_hi : l_lo, m = h ? m_hi : m_lo;
        // attention.cpp:82-84: the masked mass z = l / raw must stay above 1e-300; every row
        // admits key 0, so raw >= 1 after the max shift and the test is l > 0 in fp32
        if (!(l > 0.f)) {
            if ((lane & 3) == 0) latch_error(p.err, LKV_ERR_DEGENERATE_MASK, r);
            continue;
        }
        const float inv = 1.f / l;
        __nv_bfloat16* orow = out + (row_base + r) * kD;
#pragma unroll
        for (int n = 0; n < 16; ++n)
            *reinterpret_cast<__nv_bfloat162*>(orow + n * 8 + cq) =
                __floats2bfloat162_rn(o[n][2 * h] * inv, o[n][2 * h + 1] * inv);
        if ((lane & 3) == 0) p.lse[row_base + r] = m + log2f(l);
    }
}

// validate_call (attention.cpp:40-42): every mask value finite and >= 0
__global__ void mask_check_kernel(const float* __restrict__ mask, int64_t n, ErrWord* err) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float m = mask[i];
        if (!(m >= 0.f) || isinf(m)) {
            latch_error(err, LKV_ERR_CONTRACT, (int)min(i, (int64_t)INT32_MAX));
            return;
        }
    }
}

// =====================================================================================================
// backward: D = rowsum(dO * O)
// =====================================================================================================
template <typename T>
__global__ void bwd_prep_kernel(const T* __restrict__ out, const T* __restrict__ dout, float* __restrict__ dsum,
                                int64_t rows, int d) {
    const int64_t r = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    float s = 0.f;
    for (int c = lane; c < d; c += 32) {
        float o, u;
        if constexpr (sizeof(T) == 2) {
            o = __bfloat162float(out[r * d + c]);
            u = __bfloat162float(dout[r * d + c]);
        } else {
            o = out[r * d + c];
            u = dout[r * d + c];
        }
        s = fmaf(o, u, s);
    }
#pragma unroll
    for (int x = 16; x > 0; x >>= 1) s += __shfl_xor_sync(0xffffffffu, s, x);
    if (lane == 0) dsum[r] = s;
}

// =====================================================================================================
// backward: dQ (query-block major; K/V streamed)
// =====================================================================================================
__global__ void __launch_bounds__(kThreads, 2)
    dq_bf16_kernel(const __grid_constant__ AttnParams p, const __grid_constant__ CUtensorMap tk,
                   const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tq,
                   const __grid_constant__ CUtensorMap tdo) {
    constexpr int kStageBytes = 2 * kKB * 256;
    extern __shared__ unsigned char smem_dyn[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
    unsigned char* qs = smem + kStages * kStageBytes;  // Q tile [64][256 B], then dO tile
    uint64_t* full = reinterpret_cast<uint64_t*>(qs + 2 * kQB * 256);
    uint64_t* empty = full + kStages;
    uint64_t* qbar = empty + kStages;
    const Geo g{p.n_q_heads, p.n_kv_heads, p.n_q_heads / p.n_kv_heads, p.t_q, p.t_k, p.causal, p.pos_offset,
                p.self_keep, p.scale * kLog2e, p.scale};
    const int b = blockIdx.z, qh = blockIdx.y, kvh = qh / g.G;
    const int q0 = blockIdx.x * kQB;
    const int kend = key_end(g, min(g.t_q, q0 + kQB) - 1);
    const int ntiles = kend > 0 ? (kend + kKB - 1) / kKB : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kConsumers);
        }
        mbar_init(qbar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    const size_t kv_row0 = ((size_t)b * g.n_kv_heads + kvh) * g.t_k;
    const size_t q_row0 = ((size_t)b * g.n_q_heads + qh) * g.t_q;
    if (warp == kConsumers) {
        if (lane == 0) {
            const uint64_t pol = l2_policy_evict_last();
            mbar_arrive_expect_tx(qbar, 2 * kQB * 256);
            tma_tile<kQB>(qs, &tq, qbar, (int)(q_row0 + q0), pol);
            tma_tile<kQB>(qs + kQB * 256, &tdo, qbar, (int)(q_row0 + q0), pol);
            for (int t = 0; t < ntiles; ++t) {
                const int st = t % kStages;
                if (t >= kStages) mbar_wait(&empty[st], ((t / kStages) - 1) & 1);
                mbar_arrive_expect_tx(&full[st], kStageBytes);
                unsigned char* dst = smem + st * kStageBytes;
                tma_tile<kKB>(dst, &tk, &full[st], (int)(kv_row0 + t * kKB), pol);
                tma_tile<kKB>(dst + kKB * 256, &tv, &full[st], (int)(kv_row0 + t * kKB), pol);
            }
        }
        return;
    }
    const int gq = lane >> 2, cq = (lane & 3) * 2;
    const int r_lo = q0 + warp * 16 + gq, r_hi = r_lo + 8;
    const float* mask = p.mask ? p.mask + ((size_t)b * g.n_kv_heads + kvh) * g.t_k : nullptr;
    const bool mask_vec = (reinterpret_cast<uintptr_t>(mask) & 7) == 0;
    const float lse_lo = r_lo < g.t_q ? p.lse[q_row0 + r_lo] : 0.f, lse_hi = r_hi < g.t_q ? p.lse[q_row0 + r_hi] : 0.f;
    const float d_lo = r_lo < g.t_q ? p.dsum[q_row0 + r_lo] : 0.f, d_hi = r_hi < g.t_q ? p.dsum[q_row0 + r_hi] : 0.f;
    const uint32_t qsb = smem_u32(qs), dob = qsb + kQB * 256;
    mbar_wait(qbar, 0);
    float dq[16][4];
#pragma unroll
    for (int n = 0; n < 16; ++n) dq[n][0] = dq[n][1] = dq[n][2] = dq[n][3] = 0.f;
    for (int t = 0; t < ntiles; ++t) {
        const int st = t % kStages;
        mbar_wait(&full[st], (t / kStages) & 1);
        const uint32_t kb = smem_u32(smem + st * kStageBytes), vb = kb + kKB * 256;
        const int j0 = t * kKB;
        float s[8][4], dp[8][4];
#pragma unroll
        for (int n = 0; n < 8; ++n)
#pragma unroll
            for (int e = 0; e < 4; ++e) s[n][e] = dp[n][e] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            uint32_t qa[4], ua[4];
            frag_a<kQB>(qsb, warp * 16, kk, lane, qa);
            frag_a<kQB>(dob, warp * 16, kk, lane, ua);
#pragma unroll
            for (int np = 0; np < 4; ++np) {
                uint32_t bk[4], bv[4];
                frag_bn<kKB>(kb, np * 16, kk, lane, bk);
                frag_bn<kKB>(vb, np * 16, kk, lane, bv);
                mma(s[2 * np], qa, bk[0], bk[1]);
                mma(s[2 * np + 1], qa, bk[2], bk[3]);
                mma(dp[2 * np], ua, bv[0], bv[1]);
                mma(dp[2 * np + 1], ua, bv[2], bv[3]);
            }
        }
        // dS = P (dP - D), P = exp2(s c - lse) m; interior tiles skip the admissibility tests
        const int wr0 = q0 + warp * 16;
        const bool interior = j0 + kKB <= g.t_k && wr0 + 16 <= g.t_q && (!g.causal || j0 + kKB - 1 <= g.pos_offset + wr0) &&
                              !(g.self_keep && j0 + kKB - 1 >= g.pos_offset + wr0);
#pragma unroll
        for (int n = 0; n < 8; ++n) {
            const float2 m2 = load_mask2(mask, mask_vec, j0 + n * 8 + cq, g.t_k);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const float el = fast_exp2(s[n][e] * g.c - lse_lo), eh = fast_exp2(s[n][2 + e] * g.c - lse_hi);
                const float mj = e ? m2.y : m2.x;
                float pl = el * mj, ph = eh * mj;
                if (!interior) {
                    const int j = j0 + n * 8 + cq + e;
                    pl = !admissible(g, j, r_lo) ? 0.f : (g.self_keep && j == g.pos_offset + r_lo) ? el : pl;
                    ph = !admissible(g, j, r_hi) ? 0.f : (g.self_keep && j == g.pos_offset + r_hi) ? eh : ph;
                }
                s[n][e] = pl * (dp[n][e] - d_lo);
                s[n][2 + e] = ph * (dp[n][2 + e] - d_hi);
            }
        }
        // dQ += dS K
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            uint32_t pa[4] = {pack2(s[2 * kk][0], s[2 * kk][1]), pack2(s[2 * kk][2], s[2 * kk][3]),
                              pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]), pack2(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
            for (int n2 = 0; n2 < 8; ++n2) {
                uint32_t bf[4];
                frag_bk<kKB>(kb, kk * 16, n2, lane, bf);
                mma(dq[2 * n2], pa, bf[0], bf[1]);
                mma(dq[2 * n2 + 1], pa, bf[2], bf[3]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int r = h ? r_hi : r_lo;
        if (r >= g.t_q) continue;
        float* drow = p.dq + (q_row0 + r) * kD;
#pragma unroll
        for (int n = 0; n < 16; ++n)
            *reinterpret_cast<float2*>(drow + n * 8 + cq) = make_float2(dq[n][2 * h] * g.scale, dq[n][2 * h + 1] * g.scale);
    }
}

// =====================================================================================================
// backward: dK, dV, dmask (key-block major; Q/dO tiles of every query head of the group streamed)
// =====================================================================================================
__global__ void __launch_bounds__(kThreads, 1)
    dkv_bf16_kernel(const __grid_constant__ AttnParams p, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tq32,
                    const __grid_constant__ CUtensorMap tdo32) {
    constexpr int kStageBytes = 2 * kQT * 256;
    extern __shared__ unsigned char smem_dyn[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
    unsigned char* kvs = smem + kStages * kStageBytes;  // K block [64][256 B], then V block
    uint64_t* full = reinterpret_cast<uint64_t*>(kvs + 2 * kKB * 256);
    uint64_t* empty = full + kStages;
    uint64_t* kvbar = empty + kStages;
    const Geo g{p.n_q_heads, p.n_kv_heads, p.n_q_heads / p.n_kv_heads, p.t_q, p.t_k, p.causal, p.pos_offset,
                p.self_keep, p.scale * kLog2e, p.scale};
    const int b = blockIdx.z, kvh = blockIdx.y;
    const int k0 = blockIdx.x * kKB;
    // query tiles that see any key of this block: pos_offset + r >= k0 when causal
    const int rstart = g.causal ? max(0, k0 - g.pos_offset) : 0;
    const int qt0 = rstart / kQT;
    const int qtn = rstart < g.t_q ? (g.t_q + kQT - 1) / kQT - qt0 : 0;  // per query head
    const int ntiles = qtn * g.G;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kConsumers);
        }
        mbar_init(kvbar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    const size_t kv_row0 = ((size_t)b * g.n_kv_heads + kvh) * g.t_k;
    auto q_row_of = [&](int tile) -> size_t {  // global row of streamed tile `tile`
        const int hg = tile / qtn, qt = qt0 + tile % qtn;
        return ((size_t)b * g.n_q_heads + kvh * g.G + hg) * g.t_q + (size_t)qt * kQT;
    };
    if (warp == kConsumers) {
        if (lane == 0) {
            const uint64_t pol = l2_policy_evict_last();
            mbar_arrive_expect_tx(kvbar, 2 * kKB * 256);
            tma_tile<kKB>(kvs, &tk, kvbar, (int)(kv_row0 + k0), pol);
            tma_tile<kKB>(kvs + kKB * 256, &tv, kvbar, (int)(kv_row0 + k0), pol);
            for (int t = 0; t < ntiles; ++t) {
                const int st = t % kStages;
                if (t >= kStages) mbar_wait(&empty[st], ((t / kStages) - 1) & 1);
                mbar_arrive_expect_tx(&full[st], kStageBytes);
                unsigned char* dst = smem + st * kStageBytes;
                const int y = (int)q_row_of(t);
                tma_tile<kQT>(dst, &tq32, &full[st], y, pol);
                tma_tile<kQT>(dst + kQT * 256, &tdo32, &full[st], y, pol);
            }
        }
        return;
    }
    const int gk = lane >> 2, cq = (lane & 3) * 2;
    const int j_lo = k0 + warp * 16 + gk, j_hi = j_lo + 8;  // this thread's two keys
    const float* mask = p.mask ? p.mask + kv_row0 : nullptr;
    const uint32_t kb = smem_u32(kvs), vb = kb + kKB * 256;
    mbar_wait(kvbar, 0);
    float dk[16][4], dv[16][4];
#pragma unroll
    for (int n = 0; n < 16; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) dk[n][e] = dv[n][e] = 0.f;
    float dm_lo = 0.f, dm_hi = 0.f;
    const float mk_lo = !mask ? 1.f : j_lo < g.t_k ? __ldg(mask + j_lo) : 0.f;
    const float mk_hi = !mask ? 1.f : j_hi < g.t_k ? __ldg(mask + j_hi) : 0.f;
    for (int t = 0; t < ntiles; ++t) {
        const int st = t % kStages;
        mbar_wait(&full[st], (t / kStages) & 1);
        const uint32_t qb = smem_u32(smem + st * kStageBytes), ub = qb + kQT * 256;
        const int hg = t / qtn, r0 = (qt0 + t % qtn) * kQT;
        const size_t qrow = ((size_t)b * g.n_q_heads + kvh * g.G + hg) * g.t_q;
        float s[4][4], dp[4][4];  // keys (rows) x 32 queries (4 n8 tiles)
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int e = 0; e < 4; ++e) s[n][e] = dp[n][e] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            uint32_t ka[4], va[4];
            frag_a<kKB>(kb, warp * 16, kk, lane, ka);
            frag_a<kKB>(vb, warp * 16, kk, lane, va);
#pragma unroll
            for (int np = 0; np < 2; ++np) {
                uint32_t bq[4], bu[4];
                frag_bn<kQT>(qb, np * 16, kk, lane, bq);
                frag_bn<kQT>(ub, np * 16, kk, lane, bu);
                mma(s[2 * np], ka, bq[0], bq[1]);
                mma(s[2 * np + 1], ka, bq[2], bq[3]);
                mma(dp[2 * np], va, bu[0], bu[1]);
                mma(dp[2 * np + 1], va, bu[2], bu[3]);
            }
        }
        // element (key j, query r): P = exp2(s c - lse_r) m_j, Pm = exp2(s c - lse_r); interior tiles
        // (all 16 keys of the warp admissible for all 32 queries, no self key) skip the tests
        const int wk0 = k0 + warp * 16;
        const bool interior = wk0 + 16 <= g.t_k && r0 + kQT <= g.t_q && (!g.causal || wk0 + 15 <= g.pos_offset + r0) &&
                              !(g.self_keep && wk0 + 15 >= g.pos_offset + r0);
        float pt[4][4];
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = r0 + n * 8 + cq + e;
                const bool rv = r < g.t_q;
                const float lse = rv ? __ldg(p.lse + qrow + r) : 0.f;
                const float dd = rv ? __ldg(p.dsum + qrow + r) : 0.f;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = h ? j_hi : j_lo;
                    float& sv = s[n][2 * h + e];
                    const float dpv = dp[n][2 * h + e] - dd;
                    float pm = fast_exp2(sv * g.c - lse), mj = h ? mk_hi : mk_lo;
                    if (!interior) {
                        if (!admissible(g, j, r)) pm = 0.f;
                        if (g.self_keep && j == g.pos_offset + r) mj = -1.f;  // self: multiplier 1, no dmask
                    }
                    const float pv = mj < 0.f ? pm : pm * mj;
                    if (mj >= 0.f) (h ? dm_hi : dm_lo) += pm * dpv;
                    pt[n][2 * h + e] = pv;
                    sv = pv * dpv;  // dS^T
                }
            }
        // dV += P^T dO, dK += dS^T Q  (k = the 32 queries: 2 k16 steps)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            const uint32_t pa[4] = {pack2(pt[2 * kk][0], pt[2 * kk][1]), pack2(pt[2 * kk][2], pt[2 * kk][3]),
                                    pack2(pt[2 * kk + 1][0], pt[2 * kk + 1][1]),
                                    pack2(pt[2 * kk + 1][2], pt[2 * kk + 1][3])};
            const uint32_t sa[4] = {pack2(s[2 * kk][0], s[2 * kk][1]), pack2(s[2 * kk][2], s[2 * kk][3]),
                                    pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]), pack2(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
            for (int n2 = 0; n2 < 8; ++n2) {
                uint32_t bu[4], bq[4];
                frag_bk<kQT>(ub, kk * 16, n2, lane, bu);
                frag_bk<kQT>(qb, kk * 16, n2, lane, bq);
                mma(dv[2 * n2], pa, bu[0], bu[1]);
                mma(dv[2 * n2 + 1], pa, bu[2], bu[3]);
                mma(dk[2 * n2], sa, bq[0], bq[1]);
                mma(dk[2 * n2 + 1], sa, bq[2], bq[3]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
#pragma unroll
    for (int x = 1; x <= 2; x <<= 1) {
        dm_lo += __shfl_xor_sync(0xffffffffu, dm_lo, x);
        dm_hi += __shfl_xor_sync(0xffffffffu, dm_hi, x);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int j = h ? j_hi : j_lo;
        if (j >= g.t_k) continue;
        float* krow = p.dk + (kv_row0 + j) * kD;
        float* vrow = p.dv + (kv_row0 + j) * kD;
#pragma unroll
        for (int n = 0; n < 16; ++n) {
            *reinterpret_cast<float2*>(krow + n * 8 + cq) = make_float2(dk[n][2 * h] * g.scale, dk[n][2 * h + 1] * g.scale);
            *reinterpret_cast<float2*>(vrow + n * 8 + cq) = make_float2(dv[n][2 * h], dv[n][2 * h + 1]);
        }
        if (p.dmask && (lane & 3) == 0) p.dmask[kv_row0 + j] = h ? dm_hi : dm_lo;
    }
}

// =====================================================================================================
// fp32 SIMT path (any head_dim <= 256): exact two-pass softmax per row, the 1e-5 correctness path
// =====================================================================================================
constexpr int kSimt = 128;

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
    for (int x = 16; x > 0; x >>= 1) v += __shfl_xor_sync(0xffffffffu, v, x);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    float s = 0.f;
    for (int w = 0; w < kSimt / 32; ++w) s += red[w];
    return s;
}
__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
    for (int x = 16; x > 0; x >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, x));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    float s = -INFINITY;
    for (int w = 0; w < kSimt / 32; ++w) s = fmaxf(s, red[w]);
    return s;
}

// one CTA per (row, q head, batch): s_j = scale q.k_j (natural), p = softmax, masked, renormalised
__global__ void __launch_bounds__(kSimt) fwd_f32_kernel(const __grid_constant__ AttnParams p, int d) {
    extern __shared__ float sm[];
    float* q = sm;          // [d]
    float* sc = sm + d;     // [t_k]
    __shared__ float red[kSimt / 32];
    const int r = blockIdx.x, qh = blockIdx.y, b = blockIdx.z;
    const int G = p.n_q_heads / p.n_kv_heads, kvh = qh / G;
    const Geo g{p.n_q_heads, p.n_kv_heads, G, p.t_q, p.t_k, p.causal, p.pos_offset, p.self_keep, 0.f, p.scale};
    const size_t qrow = ((size_t)b * p.n_q_heads + qh) * p.t_q + r;
    const size_t kv0 = ((size_t)b * p.n_kv_heads + kvh) * p.t_k;
    const float* K = static_cast<const float*>(p.k) + kv0 * d;
    const float* V = static_cast<const float*>(p.v) + kv0 * d;
    const float* mask = p.mask ? p.mask + kv0 : nullptr;
    for (int c = threadIdx.x; c < d; c += kSimt) q[c] = static_cast<const float*>(p.q)[qrow * d + c];
    __syncthreads();
    const int end = key_end(g, r);
    float mx = -INFINITY;
    for (int j = threadIdx.x; j < end; j += kSimt) {
        float dot = 0.f;
        for (int c = 0; c < d; ++c) dot = fmaf(q[c], K[(size_t)j * d + c], dot);
        sc[j] = p.scale * dot;
        mx = fmaxf(mx, sc[j]);
    }
    mx = block_max(mx, red);
    float zr = 0.f;
    for (int j = threadIdx.x; j < end; j += kSimt) {
        sc[j] = expf(sc[j] - mx);
        zr += sc[j];
    }
    zr = block_sum(zr, red);
    float zm = 0.f;
    for (int j = threadIdx.x; j < end; j += kSimt) {
        sc[j] = sc[j] / zr * mask_eff(g, mask, j, r);  // p~ = p_raw m (attention.cpp:78-81)
        zm += sc[j];
    }
    zm = block_sum(zm, red);
    if (!(zm > 0.f)) {
        if (threadIdx.x == 0) latch_error(p.err, LKV_ERR_DEGENERATE_MASK, r);
        return;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += kSimt) {
        float acc = 0.f;
        for (int j = 0; j < end; ++j) acc = fmaf(sc[j], V[(size_t)j * d + c], acc);
        static_cast<float*>(p.out)[qrow * d + c] = acc / zm;
    }
    if (threadIdx.x == 0) p.lse[qrow] = (mx + logf(zr * zm)) * kLog2e;  // log2-domain masked LSE
}

// dQ row: one CTA per (row, q head, batch)
__global__ void __launch_bounds__(kSimt) dq_f32_kernel(const __grid_constant__ AttnParams p, int d) {
    extern __shared__ float sm[];
    float* q = sm;          // [d]
    float* u = q + d;       // [d]
    float* ds = u + d;      // [t_k]
    const int r = blockIdx.x, qh = blockIdx.y, b = blockIdx.z;
    const int G = p.n_q_heads / p.n_kv_heads, kvh = qh / G;
    const Geo g{p.n_q_heads, p.n_kv_heads, G, p.t_q, p.t_k, p.causal, p.pos_offset, p.self_keep, 0.f, p.scale};
    const size_t qrow = ((size_t)b * p.n_q_heads + qh) * p.t_q + r;
    const size_t kv0 = ((size_t)b * p.n_kv_heads + kvh) * p.t_k;
    const float* K = static_cast<const float*>(p.k) + kv0 * d;
    const float* V = static_cast<const float*>(p.v) + kv0 * d;
    const float* mask = p.mask ? p.mask + kv0 : nullptr;
    for (int c = threadIdx.x; c < d; c += kSimt) {
        q[c] = static_cast<const float*>(p.q)[qrow * d + c];
        u[c] = static_cast<const float*>(p.dout)[qrow * d + c];
    }
    __syncthreads();
    const float lse = p.lse[qrow] / kLog2e, D = p.dsum[qrow];
    const int end = key_end(g, r);
    for (int j = threadIdx.x; j < end; j += kSimt) {
        float dot = 0.f, w = 0.f;
        for (int c = 0; c < d; ++c) {
            dot = fmaf(q[c], K[(size_t)j * d + c], dot);
            w = fmaf(u[c], V[(size_t)j * d + c], w);
        }
        const float pj = expf(p.scale * dot - lse) * mask_eff(g, mask, j, r);
        ds[j] = pj * (w - D);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += kSimt) {
        float acc = 0.f;
        for (int j = 0; j < end; ++j) acc = fmaf(ds[j], K[(size_t)j * d + c], acc);
        p.dq[qrow * d + c] = acc * p.scale;
    }
}

// dK, dV, dmask of one key: one CTA per (key, kv head, batch), looping over the group's rows
__global__ void __launch_bounds__(kSimt) dkv_f32_kernel(const __grid_constant__ AttnParams p, int d) {
    extern __shared__ float sm[];
    float* kj = sm;       // [d]
    float* vj = kj + d;   // [d]
    float* accv = vj + d; // [d]
    float* acck = accv + d;
    __shared__ float red[kSimt / 32];
    const int j = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
    const int G = p.n_q_heads / p.n_kv_heads;
    const Geo g{p.n_q_heads, p.n_kv_heads, G, p.t_q, p.t_k, p.causal, p.pos_offset, p.self_keep, 0.f, p.scale};
    const size_t kv0 = ((size_t)b * p.n_kv_heads + kvh) * p.t_k;
    for (int c = threadIdx.x; c < d; c += kSimt) {
        kj[c] = static_cast<const float*>(p.k)[(kv0 + j) * d + c];
        vj[c] = static_cast<const float*>(p.v)[(kv0 + j) * d + c];
        accv[c] = 0.f;
        acck[c] = 0.f;
    }
    __syncthreads();
    const float mj = p.mask ? p.mask[kv0 + j] : 1.f;
    float dmask = 0.f;
    const int r0 = g.causal ? max(0, j - g.pos_offset) : 0;
    for (int hg = 0; hg < G; ++hg) {
        const size_t qbase = ((size_t)b * p.n_q_heads + kvh * G + hg) * p.t_q;
        for (int r = r0; r < p.t_q; ++r) {
            const float* qr = static_cast<const float*>(p.q) + (qbase + r) * d;
            const float* ur = static_cast<const float*>(p.dout) + (qbase + r) * d;
            float dot = 0.f, w = 0.f;
            for (int c = threadIdx.x; c < d; c += kSimt) {
                dot = fmaf(qr[c], kj[c], dot);
                w = fmaf(ur[c], vj[c], w);
            }
            dot = block_sum(dot, red);
            w = block_sum(w, red);
            const float pm = expf(p.scale * dot - p.lse[qbase + r] / kLog2e);
            const bool self = g.self_keep && j == g.pos_offset + r;
            const float pj = pm * (self ? 1.f : mj);
            const float D = p.dsum[qbase + r];
            const float dsj = pj * (w - D);
            if (!self) dmask += pm * (w - D);
            for (int c = threadIdx.x; c < d; c += kSimt) {
                accv[c] = fmaf(pj, ur[c], accv[c]);
                acck[c] = fmaf(dsj, qr[c], acck[c]);
            }
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += kSimt) {
        p.dv[(kv0 + j) * d + c] = accv[c];
        p.dk[(kv0 + j) * d + c] = acck[c] * p.scale;
    }
    if (p.dmask && threadIdx.x == 0) p.dmask[kv0 + j] = dmask;
}

}  // namespace attn

// ---- host launchers ----------------------------------------------------------------------------------
size_t attn_fwd_smem() { return 1024 + attn::kStages * (2 * attn::kKB * 256) + attn::kQB * 256 + 2 * attn::kStages * 8 + 8; }
size_t attn_dq_smem() { return 1024 + attn::kStages * (2 * attn::kKB * 256) + 2 * attn::kQB * 256 + 2 * attn::kStages * 8 + 8; }
size_t attn_dkv_smem() {
    return 1024 + attn::kStages * (2 * attn::kQT * 256) + 2 * attn::kKB * 256 + 2 * attn::kStages * 8 + 8;
}

cudaError_t launch_attn_fwd(const AttnParams& p, int dtype, int d, const CUtensorMap* mk, const CUtensorMap* mv,
                            const CUtensorMap* mq, cudaStream_t stream) {
    if (p.mask) {
        const int64_t n = (int64_t)p.batch * p.n_kv_heads * p.t_k;
        attn::mask_check_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1184), 256, 0, stream>>>(p.mask, n, p.err);
        note_launches(1);
    }
    if (dtype == LKV_BF16) {
        const size_t smem = attn_fwd_smem();
        cudaError_t e = cudaFuncSetAttribute(attn::fwd_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attn::fwd_bf16_kernel<<<dim3((p.t_q + attn::kQB - 1) / attn::kQB, p.n_q_heads, p.batch), attn::kThreads, smem,
                                stream>>>(p, *mk, *mv, *mq);
    } else {
        const size_t smem = (size_t)(d + p.t_k) * 4;
        cudaError_t e = cudaFuncSetAttribute(attn::fwd_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attn::fwd_f32_kernel<<<dim3(p.t_q, p.n_q_heads, p.batch), attn::kSimt, smem, stream>>>(p, d);
    }
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_attn_bwd(const AttnParams& p, int dtype, int d, const CUtensorMap* mk, const CUtensorMap* mv,
                            const CUtensorMap* mq, const CUtensorMap* mdo, const CUtensorMap* mq32,
                            const CUtensorMap* mdo32, cudaStream_t stream) {
    const int64_t rows = (int64_t)p.batch * p.n_q_heads * p.t_q;
    cudaError_t e;
    if (dtype == LKV_BF16) {
        attn::bwd_prep_kernel<__nv_bfloat16><<<(unsigned)((rows + 3) / 4), 128, 0, stream>>>(
            static_cast<const __nv_bfloat16*>(p.out), static_cast<const __nv_bfloat16*>(p.dout), p.dsum, rows, d);
        const size_t s1 = attn_dq_smem(), s2 = attn_dkv_smem();
        if ((e = cudaFuncSetAttribute(attn::dq_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1)))
            return e;
        if ((e = cudaFuncSetAttribute(attn::dkv_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2)))
            return e;
        attn::dq_bf16_kernel<<<dim3((p.t_q + attn::kQB - 1) / attn::kQB, p.n_q_heads, p.batch), attn::kThreads, s1,
                               stream>>>(p, *mk, *mv, *mq, *mdo);
        attn::dkv_bf16_kernel<<<dim3((p.t_k + attn::kKB - 1) / attn::kKB, p.n_kv_heads, p.batch), attn::kThreads, s2,
                                stream>>>(p, *mk, *mv, *mq32, *mdo32);
    } else {
        attn::bwd_prep_kernel<float><<<(unsigned)((rows + 3) / 4), 128, 0, stream>>>(
            static_cast<const float*>(p.out), static_cast<const float*>(p.dout), p.dsum, rows, d);
        const size_t s1 = (size_t)(2 * d + p.t_k) * 4, s2 = (size_t)4 * d * 4;
        if ((e = cudaFuncSetAttribute(attn::dq_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1)))
            return e;
        attn::dq_f32_kernel<<<dim3(p.t_q, p.n_q_heads, p.batch), attn::kSimt, s1, stream>>>(p, d);
        attn::dkv_f32_kernel<<<dim3(p.t_k, p.n_kv_heads, p.batch), attn::kSimt, s2, stream>>>(p, d);
    }
    note_launches(3);
    return cudaGetLastError();
}

}  // namespace lkv_dev
