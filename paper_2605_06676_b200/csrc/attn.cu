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
//   * forward on tcgen05 (fwd_tc_kernel below): S, P and O in TMEM (P V takes its A operand from
//     TMEM), the V tile is the B operand of P V read MN-major straight from the TMA layout;
//     causal tiles past the block's last admissible key are never loaded;
//   * backward on tcgen05, two kernels with no atomics (deterministic):
//     dQ:  CTA = 128 queries (Q, dO in smem), K/V tiles streamed; S = Q K^T and dP = dO V^T in
//          TMEM, dS = P (dP - D) written by the row threads to smem, dQ += dS K accumulated in TMEM;
//     dKV: CTA = 128 keys (K, V in smem for the CTA's life), streams 64-query Q/dO tiles of
//          all G query heads; S^T, dP^T in TMEM; P^T, dS^T through smem; dV += P^T dO and
//          dK += dS^T Q in TMEM; the mask gradient per key accumulates in the key-row thread.
// fp32 inputs run SIMT kernels (exact two-pass softmax, the 1e-5 correctness path).
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "kernels.cuh"

namespace lkv_dev {
namespace attn {

constexpr int kD = 128;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float fast_exp2(float x) {  // MUFU.EX2 (2 ulp); ex2(-inf) = +0
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// load a ROWS x 128 bf16 tile (two 64-column boxes) at global row y
template <int ROWS>
__device__ __forceinline__ void tma_tile(unsigned char* dst, const CUtensorMap* m, uint64_t* bar, int y, uint64_t pol) {
    tma_load_2d(dst, m, bar, 0, y, pol);
    tma_load_2d(dst + ROWS * 128, m, bar, 64, y, pol);
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
// forward on tcgen05 (5th-gen tensor cores, accumulators in TMEM)
//   CTA = 128 queries (UMMA M) of one (batch, q head); 64-key tiles.
//   warp 4: TMA (Q once; K tiles [64 keys][128 d]; V^T tiles [128 d][64 keys] from a transposed
//           copy, so both UMMA B operands are K-major), 3-stage rings;
//   warp 5: one thread issues S_t = Q K_t^T (M128 N64 K128) into a double-buffered TMEM S and
//           O += P_t V_t (M128 N128 K64) into TMEM O, running S one tile ahead of P V;
//   warps 0-3: thread = query row = TMEM lane: tcgen05.ld of the S row, admissibility, online
//           max with lazy rescaling (O in TMEM is rescaled only when the row max grows by more
//           than 2^8, FA4-style), exp2 x mask, P row -> shared memory in the 128-byte-swizzled
//           K-major layout the UMMA descriptor reads; epilogue O / l from TMEM.
// =====================================================================================================
constexpr int kTcQ = 128, kTcK = 64, kTcWG = 2;  // kTcK: key tile of the dQ kernel
constexpr int kTcThreads = (kTcWG * 4 + 2) * 32;  // 2 softmax warpgroups + TMA warp + MMA warp
constexpr float kTcRescale = 8.f;  // log2 units
constexpr uint32_t kTcCols = 512;  // TMEM columns of the forward / dQ kernels

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// tiles of 64 keys that query rows [r0, r0 + 128) need (0 when no row is valid)
__device__ __forceinline__ int tc_tiles(const Geo& g, int r0) {
    if (r0 >= g.t_q) return 0;
    const int kend = key_end(g, min(g.t_q, r0 + kTcQ) - 1);
    return kend > 0 ? (kend + kTcK - 1) / kTcK : 0;
}

// =====================================================================================================
// forward on tcgen05: 128-key tiles, P kept in TMEM (the A operand of P V read from TMEM)
//   CTA = two 128-query tiles (softmax warpgroups 0 / 1) sharing every K / V tile.
//   TMEM: S_w at column w*128 (128 fp32 columns); P_w overwrites the first 64 of them as packed
//         bf16 pairs once the row threads have read S; O_w at 256 + w*128.
//   MMA order per tile t and warpgroup w: P V_w(t) then S_w(t+1) -- tcgen05.mma executes in issue
//   order, so P_w(t) is consumed before S_w(t+1) overwrites it, and when S_w(t+1) lands, P V_w(t)
//   has landed too: the row threads may rescale O_w with no extra barrier.
//   Row threads walk S in 32-key chunks (32 live registers): chunk max, lazy rescale against the
//   running max (threshold 2^8; a chunk that raises it past the threshold also rescales the P
//   chunks of this tile already in TMEM, and O), exp2 x mask, P chunk -> TMEM.
// =====================================================================================================
constexpr int kF2K = 128;        // keys per tile (UMMA N of S, K of P V)
constexpr int kF2Stages = 2;     // K / V tile ring
constexpr int kF2Chunk = 32;     // keys per row-thread chunk

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
// D (TMEM) += A (TMEM, M rows x 16 bf16 as 8 packed columns) * B (shared-memory descriptor)
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// tcgen05.wait::ld that also "defines" r: the registers of an asynchronous tcgen05.ld cannot be
// read (or the read hoisted by the compiler) before the wait
__device__ __forceinline__ void tmem_ld_wait_dep(uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.wait::ld.sync.aligned;"
        : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
          "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]),
          "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]),
          "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]),
          "+r"(r[30]), "+r"(r[31])
        :
        : "memory");
}
__device__ __forceinline__ float2 unpack2(uint32_t w) {
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}

// The rare lazy-rescale step of the forward row threads (warp-collective): O *= alpha (when a
// P V has landed in it) and the P chunks [0, c) of the current tile already in TMEM.  Out of line
// to keep the hot loop small.
__device__ __noinline__ void fwd_rescale(uint32_t lane_addr, uint32_t s_col, uint32_t o_col, int c, bool has_o,
                                         float alpha) {
    tmem_st_wait();
    if (has_o) {
        for (int q = 0; q < 4; ++q) {
            uint32_t orr[32];
            tmem_ld_32x32b_x32(lane_addr + o_col + q * 32, orr);
            tmem_ld_wait_dep(orr);
#pragma unroll
            for (int i = 0; i < 32; ++i) orr[i] = __float_as_uint(__uint_as_float(orr[i]) * alpha);
            tmem_st32(lane_addr + o_col + q * 32, orr);
        }
    }
    for (int pc = 0; pc < c; ++pc) {
        uint32_t pr[16];
        tmem_ld16(lane_addr + s_col + pc * 16, pr);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float2 f = unpack2(pr[i]);
            pr[i] = pack2(f.x * alpha, f.y * alpha);
        }
        tmem_st16(lane_addr + s_col + pc * 16, pr);
    }
    tmem_st_wait();
}

__device__ __forceinline__ int f2_tiles(const Geo& g, int r0) {
    if (r0 >= g.t_q) return 0;
    const int kend = key_end(g, min(g.t_q, r0 + kTcQ) - 1);
    return kend > 0 ? (kend + kF2K - 1) / kF2K : 0;
}

__global__ void __launch_bounds__(kTcThreads, 1)
    fwd_tc_kernel(const __grid_constant__ AttnParams p, const __grid_constant__ CUtensorMap tq,
                   const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv) {
    constexpr uint32_t kQBytes = kTcQ * 256, kKBytes = kF2K * 256, kVBytes = kF2K * 256;
    extern __shared__ unsigned char smem_dyn[];
    unsigned char* smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);  // aligned, still a __shared__ pointer
    unsigned char* qs = smem;                          // [wg] Q tiles
    unsigned char* ks = qs + kTcWG * kQBytes;          // [stage] K tiles
    unsigned char* vs = ks + kF2Stages * kKBytes;      // [stage] V tiles
    float* mw = reinterpret_cast<float*>(vs + kF2Stages * kVBytes);  // [8 warps][128] mask tile
    uint64_t* bars = reinterpret_cast<uint64_t*>(mw + kTcWG * 4 * kF2K);
    uint64_t* q_full = bars;
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = k_full + kF2Stages;
    uint64_t* v_full = k_empty + kF2Stages;
    uint64_t* v_empty = v_full + kF2Stages;
    uint64_t* s_full = v_empty + kF2Stages;  // [wg]
    uint64_t* p_full = s_full + kTcWG;       // [wg]
    uint64_t* o_done = p_full + kTcWG;       // [wg]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + kTcWG);

    const Geo g{p.n_q_heads, p.n_kv_heads, p.n_q_heads / p.n_kv_heads, p.t_q, p.t_k, p.causal, p.pos_offset,
                p.self_keep, p.scale * kLog2e, p.scale};
    const int b = blockIdx.z, qh = blockIdx.y, kvh = qh / g.G;
    // causal: the last query blocks see the most keys -- dispatch them first (longest first keeps
    // the last wave short)
    const int qb = p.causal ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x;
    const int q0 = qb * (kTcWG * kTcQ);
    int nt[kTcWG];
#pragma unroll
    for (int w = 0; w < kTcWG; ++w) nt[w] = f2_tiles(g, q0 + w * kTcQ);
    const int n_all = max(nt[0], nt[1]);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < kF2Stages; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
        }
        for (int w = 0; w < kTcWG; ++w) {
            mbar_init(&s_full[w], 1);
            mbar_init(&p_full[w], 4);
            mbar_init(&o_done[w], 1);
        }
        fence_barrier_init();
    }
    if (warp == kTcWG * 4 + 1) tmem_alloc(tmem_slot, kTcCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const size_t kv_row0 = ((size_t)b * g.n_kv_heads + kvh) * g.t_k;
    const size_t q_row0 = ((size_t)b * g.n_q_heads + qh) * g.t_q;

    if (warp == kTcWG * 4) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint64_t pol = l2_policy_evict_last();
            mbar_arrive_expect_tx(q_full, kTcWG * kQBytes);
#pragma unroll
            for (int w = 0; w < kTcWG; ++w) tma_tile<kTcQ>(qs + w * kQBytes, &tq, q_full, (int)(q_row0 + q0 + w * kTcQ), pol);
            for (int t = 0; t < n_all; ++t) {
                const int st = t % kF2Stages;
                if (t >= kF2Stages) mbar_wait(&k_empty[st], ((t / kF2Stages) - 1) & 1);
                mbar_arrive_expect_tx(&k_full[st], kKBytes);
                tma_tile<kF2K>(ks + st * kKBytes, &tk, &k_full[st], (int)(kv_row0 + t * kF2K), pol);
                if (t >= kF2Stages) mbar_wait(&v_empty[st], ((t / kF2Stages) - 1) & 1);
                mbar_arrive_expect_tx(&v_full[st], kVBytes);
                tma_tile<kF2K>(vs + st * kVBytes, &tv, &v_full[st], (int)(kv_row0 + t * kF2K), pol);
            }
        }
    } else if (warp == kTcWG * 4 + 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            constexpr uint32_t idesc_s = umma_idesc_bf16(kTcQ, kF2K), idesc_o = umma_idesc_bf16_bmn(kTcQ, kD);
            const uint32_t qa = smem_u32(qs), ka = smem_u32(ks), va = smem_u32(vs);
            auto issue_s = [&](int w, int t) {  // S_w(t) = Q_w K(t)^T into TMEM columns w*128
                const int st = t % kF2Stages;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t ad = umma_desc_sw128(qa + w * kQBytes + (kk >> 2) * (kTcQ * 128) + (kk & 3) * 32);
                    const uint64_t bd = umma_desc_sw128(ka + st * kKBytes + (kk >> 2) * (kF2K * 128) + (kk & 3) * 32);
                    umma_bf16(tmem + w * 128, ad, bd, idesc_s, kk > 0 ? 1u : 0u);
                }
            };
            mbar_wait(q_full, 0);
            if (n_all > 0) {
                mbar_wait(&k_full[0], 0);
                tc_fence_after();
#pragma unroll
                for (int w = 0; w < kTcWG; ++w)
                    if (nt[w] > 0) {
                        issue_s(w, 0);
                        umma_commit(&s_full[w]);
                    }
                umma_commit(&k_empty[0]);
            }
            for (int t = 0; t < n_all; ++t) {
                const int st = t % kF2Stages, st1 = (t + 1) % kF2Stages;
                mbar_wait(&v_full[st], (t / kF2Stages) & 1);
                bool k_next = false;
#pragma unroll
                for (int w = 0; w < kTcWG; ++w) {
                    if (t >= nt[w]) continue;
                    mbar_wait(&p_full[w], t & 1);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        // B = the V tile read MN-major: keys 16kk.. at +2048 B, d 64..127 one box on
                        const uint64_t bd = umma_desc_sw128_mn(va + st * kVBytes + kk * 2048, kF2K * 128);
                        umma_bf16_ts(tmem + 256 + w * 128, tmem + w * 128 + kk * 8, bd, idesc_o,
                                     (t > 0 || kk > 0) ? 1u : 0u);
                    }
                    if (t + 1 < nt[w]) {
                        if (!k_next) {
                            mbar_wait(&k_full[st1], ((t + 1) / kF2Stages) & 1);
                            tc_fence_after();
                            k_next = true;
                        }
                        issue_s(w, t + 1);
                        umma_commit(&s_full[w]);
                    } else {
                        umma_commit(&o_done[w]);
                    }
                }
                umma_commit(&v_empty[st]);
                if (k_next) umma_commit(&k_empty[st1]);
            }
        }
    } else {
        // ===================== softmax / epilogue: warpgroup wg, thread = query row = TMEM lane
        const int wg = warp >> 2, w4 = warp & 3;
        const int ntw = nt[wg];
        const int rl = w4 * 32 + lane, r = q0 + wg * kTcQ + rl;
        const uint32_t lane_addr = tmem + (uint32_t(w4 * 32) << 16);
        const uint32_t s_col = wg * 128, o_col = 256 + wg * 128;
        const float* mask = p.mask ? p.mask + kv_row0 : nullptr;
        float* mwarp = mw + warp * kF2K;
        float m_run = -INFINITY, l_run = 0.f;
        float mnext[4] = {0.f, 0.f, 0.f, 0.f};  // the mask of tile t + 1, fetched during tile t
        if (mask) {
#pragma unroll
            for (int i = 0; i < 4; ++i) mnext[i] = lane + 32 * i < g.t_k ? __ldg(mask + lane + 32 * i) : 0.f;
        }
        const int wr0 = q0 + wg * kTcQ + w4 * 32;
        for (int t = 0; t < ntw; ++t) {
            const int j0 = t * kF2K;
            if (mask) {
#pragma unroll
                for (int i = 0; i < 4; ++i) mwarp[lane + 32 * i] = mnext[i];
                __syncwarp();
                const int jn = j0 + kF2K;
#pragma unroll
                for (int i = 0; i < 4; ++i) mnext[i] = jn + lane + 32 * i < g.t_k ? __ldg(mask + jn + lane + 32 * i) : 0.f;
            }
            mbar_wait(&s_full[wg], t & 1);
            __syncwarp();  // reconverge before .sync.aligned tcgen05.ld
            tc_fence_after();
            const bool interior = j0 + kF2K <= g.t_k && wr0 + 32 <= g.t_q &&
                                  (!g.causal || j0 + kF2K - 1 <= g.pos_offset + wr0) &&
                                  !(g.self_keep && j0 + kF2K - 1 >= g.pos_offset + wr0);
            float ls[4] = {0.f, 0.f, 0.f, 0.f};
            // INT: every (row, key) of this warp's tile is admissible -> no per-element tests and the
            // scale folded into the exponent's FMA (scale > 0: max(c s) = c max(s)); interior tiles
            // run a fully unrolled loop with the next S chunk's load in flight, boundary tiles a
            // compact one (code size: the kernel is instruction-cache sensitive)
            auto chunk = [&](auto int_tag, int c, uint32_t (&sr)[32]) {
                constexpr bool INT = decltype(int_tag)::value;
                float x[32];
                float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    if constexpr (INT) {
                        x[i] = __uint_as_float(sr[i]);
                    } else {
                        x[i] = __uint_as_float(sr[i]) * g.c;
                        if (!admissible(g, j0 + c * kF2Chunk + i, r)) x[i] = -INFINITY;
                    }
                    mq[i & 3] = fmaxf(mq[i & 3], x[i]);
                }
                float mt = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
                if constexpr (INT) mt *= g.c;
                const float m_new = fmaxf(m_run, mt);
                const bool need = m_new != -INFINITY && (m_run == -INFINITY || m_new > m_run + kTcRescale);
                float alpha = 1.f;
                if (need) alpha = m_run == -INFINITY ? 0.f : fast_exp2(m_run - m_new);
                if (__any_sync(0xffffffffu, need) && (t > 0 || c > 0))
                    fwd_rescale(lane_addr, s_col, o_col, c, t > 0, alpha);  // rare
                if (need) {
                    l_run *= alpha;
#pragma unroll
                    for (int q = 0; q < 4; ++q) ls[q] *= alpha;
                    m_run = m_new;
                }
                const float sub = m_run == -INFINITY ? 0.f : m_run;
                float mk[32];
                if (mask) {
                    const float4* m4 = reinterpret_cast<const float4*>(mwarp + c * kF2Chunk);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float4 v = m4[q];
                        mk[4 * q] = v.x;
                        mk[4 * q + 1] = v.y;
                        mk[4 * q + 2] = v.z;
                        mk[4 * q + 3] = v.w;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) mk[i] = 1.f;
                }
                uint32_t pw[16];
                if constexpr (INT) {
                    // packed pairs (FFMA2 / FMUL2 / FADD2): the row math is issue-bound
                    const float2 c2 = make_float2(g.c, g.c), ns2 = make_float2(-sub, -sub);
                    float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        float2 a2 = __ffma2_rn(make_float2(x[2 * e], x[2 * e + 1]), c2, ns2);
                        a2 = make_float2(fast_exp2(a2.x), fast_exp2(a2.y));
                        a2 = __fmul2_rn(a2, make_float2(mk[2 * e], mk[2 * e + 1]));
                        acc2[e & 1] = __fadd2_rn(acc2[e & 1], a2);
                        pw[e] = pack2(a2.x, a2.y);
                    }
                    ls[0] += acc2[0].x;
                    ls[1] += acc2[0].y;
                    ls[2] += acc2[1].x;
                    ls[3] += acc2[1].y;
                } else {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        float pv[2];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int i = 2 * e + h;
                            float mj = mk[i];
                            if (g.self_keep && j0 + c * kF2Chunk + i == g.pos_offset + r) mj = 1.f;
                            pv[h] = fast_exp2(x[i] - sub) * mj;  // x = -inf -> 0
                            ls[i & 3] += pv[h];
                        }
                        pw[e] = pack2(pv[0], pv[1]);
                    }
                }
                tmem_st16(lane_addr + s_col + c * 16, pw);  // P chunk c over S columns already read
            };
            if (interior) {
                uint32_t sb[2][32];  // S chunk c + 1 is loaded while chunk c is processed
                tmem_ld_32x32b_x32(lane_addr + s_col, sb[0]);
                tmem_ld_wait_dep(sb[0]);
#pragma unroll
                for (int c = 0; c < kF2K / kF2Chunk; ++c) {
                    if (c + 1 < kF2K / kF2Chunk) tmem_ld_32x32b_x32(lane_addr + s_col + (c + 1) * kF2Chunk, sb[(c + 1) & 1]);
                    chunk(std::true_type{}, c, sb[c & 1]);
                    if (c + 1 < kF2K / kF2Chunk) tmem_ld_wait_dep(sb[(c + 1) & 1]);
                }
            } else {
#pragma unroll 1
                for (int c = 0; c < kF2K / kF2Chunk; ++c) {
                    uint32_t sr[32];
                    tmem_ld_32x32b_x32(lane_addr + s_col + c * kF2Chunk, sr);
                    tmem_ld_wait_dep(sr);
                    chunk(std::false_type{}, c, sr);
                }
            }
            l_run += (ls[0] + ls[1]) + (ls[2] + ls[3]);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[wg]);
        }
        // ---- epilogue: O / l from TMEM
        if (ntw > 0) {
            mbar_wait(&o_done[wg], 0);
            __syncwarp();  // reconverge before .sync.aligned tcgen05.ld
            tc_fence_after();
        }
        const bool ok = l_run > 0.f;
        if (r < g.t_q && !ok) latch_error(p.err, LKV_ERR_DEGENERATE_MASK, r);  // attention.cpp:82-84
        const float inv = ok ? 1.f / l_run : 0.f;
        __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(p.out) + (q_row0 + r) * kD;
        if (ntw > 0) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t orr[32];
                tmem_ld_32x32b_x32(lane_addr + o_col + c * 32, orr);
                tmem_ld_wait();
                if (r < g.t_q && ok) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t w4v[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            w4v[e] = pack2(__uint_as_float(orr[q * 8 + 2 * e]) * inv, __uint_as_float(orr[q * 8 + 2 * e + 1]) * inv);
                        *reinterpret_cast<uint4*>(orow + c * 32 + q * 8) = make_uint4(w4v[0], w4v[1], w4v[2], w4v[3]);
                    }
                }
            }
        }
        if (r < g.t_q && ok) p.lse[q_row0 + r] = m_run + log2f(l_run);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kTcWG * 4 + 1) {
        tc_fence_after();
        tmem_dealloc(tmem, kTcCols);
    }
}

// =====================================================================================================
// backward on tcgen05: dKV (key-major) and dQ (query-major); the transposed B operands (Q and dO
// for dK / dV, K for dQ) are the TMA tiles themselves read through MN-major UMMA descriptors.
// =====================================================================================================
__device__ __forceinline__ void named_bar_sync_attn(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }
constexpr int kBwK = 128;   // dKV: keys per CTA (UMMA M)
constexpr int kBwQ = 64;    // dKV: queries per streamed tile (UMMA N of S^T, K of dV / dK)
constexpr int kBwWG = 2;     // dKV compute warpgroups: warpgroup w takes the query tiles t = w mod 2
constexpr int kBwThreads = (kBwWG * 4 + 2) * 32;  // warps 0-7 compute (thread = key row = TMEM lane), 8 TMA, 9 MMA
constexpr int kBwTma = kBwWG * 4, kBwMma = kBwWG * 4 + 1;
constexpr int kBwStages = 4;  // Q / dO tile ring

__global__ void __launch_bounds__(kBwThreads, 1)
    dkv_tc_kernel(const __grid_constant__ AttnParams p, const __grid_constant__ CUtensorMap tk128,
                  const __grid_constant__ CUtensorMap tv128, const __grid_constant__ CUtensorMap tq64,
                  const __grid_constant__ CUtensorMap tdo64) {
    constexpr uint32_t kKB128 = kBwK * 256, kT64 = kBwQ * 256, kStage = 2 * kT64;
    extern __shared__ unsigned char smem_dyn[];
    unsigned char* smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);  // aligned, still a __shared__ pointer
    unsigned char* ks = smem;
    unsigned char* vs = ks + kKB128;
    unsigned char* stg = vs + kKB128;          // [kBwStages] x {Q, dO}
    float* cw = reinterpret_cast<float*>(stg + kBwStages * kStage);  // [8 warps][lse 64 | D 64]
    float* dmx = cw + kBwWG * 4 * 2 * kBwQ;                // [128] warpgroup 1's dmask partials
    uint64_t* bars = reinterpret_cast<uint64_t*>(dmx + kBwK);
    uint64_t* kv_full = bars;
    uint64_t* st_full = bars + 1;                  // [kBwStages]
    uint64_t* st_empty = st_full + kBwStages;      // [kBwStages]
    uint64_t* s_full = st_empty + kBwStages;       // [2] (buffer = warpgroup)
    uint64_t* pt_full = s_full + 2;                // [2]
    uint64_t* acc_done = pt_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

    const Geo g{p.n_q_heads, p.n_kv_heads, p.n_q_heads / p.n_kv_heads, p.t_q, p.t_k, p.causal, p.pos_offset,
                p.self_keep, p.scale * kLog2e, p.scale};
    const int b = blockIdx.z, kvh = blockIdx.y;
    const int k0 = blockIdx.x * kBwK;
    const int rstart = g.causal ? max(0, k0 - g.pos_offset) : 0;
    const int qt0 = rstart / kBwQ;
    const int nq = rstart < g.t_q ? (g.t_q + kBwQ - 1) / kBwQ - qt0 : 0;
    const int ntiles = nq * g.G;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(kv_full, 1);
        for (int i = 0; i < kBwStages; ++i) {
            mbar_init(&st_full[i], 1);
            mbar_init(&st_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&pt_full[i], 4);
        }
        mbar_init(acc_done, 1);
        fence_barrier_init();
    }
    if (warp == kBwMma) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // TMEM: S^T[2] 0/64, dP^T[2] 128/192 (buffer = warpgroup; P^T / dS^T written over their first 32
    // columns as packed bf16 once read: the A operands of dV / dK), dV 256, dK 384
    const uint32_t tmem = *tmem_slot;
    const size_t kv_row0 = ((size_t)b * g.n_kv_heads + kvh) * g.t_k;
    auto head_of = [&](int t) { return (b * g.n_q_heads + kvh * g.G + t / nq); };  // flat q head
    auto qtile_of = [&](int t) { return qt0 + t % nq; };

    if (warp == kBwTma) {
        if (lane == 0 && ntiles > 0) {
            const uint64_t pol = l2_policy_evict_last();
            mbar_arrive_expect_tx(kv_full, 2 * kKB128);
            tma_tile<kBwK>(ks, &tk128, kv_full, (int)(kv_row0 + k0), pol);
            tma_tile<kBwK>(vs, &tv128, kv_full, (int)(kv_row0 + k0), pol);
            for (int t = 0; t < ntiles; ++t) {
                const int st = t % kBwStages;
                if (t >= kBwStages) mbar_wait_backoff(&st_empty[st], ((t / kBwStages) - 1) & 1);
                mbar_arrive_expect_tx(&st_full[st], kStage);
                unsigned char* d = stg + st * kStage;
                const int hq = head_of(t), r0 = qtile_of(t) * kBwQ;
                const int qrow = (int)((size_t)hq * g.t_q + r0);
                tma_tile<kBwQ>(d, &tq64, &st_full[st], qrow, pol);
                tma_tile<kBwQ>(d + kT64, &tdo64, &st_full[st], qrow, pol);

            }
        }
    } else if (warp == kBwMma) {
        if (lane == 0 && ntiles > 0) {
            constexpr uint32_t id_s = umma_idesc_bf16(kBwK, kBwQ), id_o = umma_idesc_bf16_bmn(kBwK, kD);
            const uint32_t ka = smem_u32(ks), va = smem_u32(vs), sa = smem_u32(stg);
            mbar_wait_backoff(kv_full, 0);
            auto issue_s = [&](int t) {  // S^T, dP^T of tile t into buffer t & 1
                const int st = t % kBwStages, bb = t & 1;
                mbar_wait_backoff(&st_full[st], (t / kBwStages) & 1);
                tc_fence_after();
                const uint32_t qb = sa + st * kStage, ub = qb + kT64;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t ao = (kk >> 2) * (kBwK * 128) + (kk & 3) * 32, bo = (kk >> 2) * (kBwQ * 128) + (kk & 3) * 32;
                    umma_bf16(tmem + bb * 64, umma_desc_sw128(ka + ao), umma_desc_sw128(qb + bo), id_s, kk > 0);
                    umma_bf16(tmem + 128 + bb * 64, umma_desc_sw128(va + ao), umma_desc_sw128(ub + bo), id_s, kk > 0);
                }
                umma_commit(&s_full[bb]);
            };
            // issue order S(t+1), dV/dK(t), S(t+2), ...: the MMAs run in issue order, so dV/dK(t) has
            // read P^T(t) / dS^T(t) before S(t+2) overwrites buffer t & 1
            issue_s(0);
            for (int t = 0; t < ntiles; ++t) {
                if (t + 1 < ntiles) issue_s(t + 1);
                const int st = t % kBwStages, pb = t & 1;
                mbar_wait_backoff(&pt_full[pb], (t >> 1) & 1);
                tc_fence_after();
                // A = P^T / dS^T from TMEM; B = the dO / Q tiles read MN-major ([queries][d] rows)
                const uint32_t qb = sa + st * kStage, ub = qb + kT64;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    umma_bf16_ts(tmem + 256, tmem + pb * 64 + kk * 8, umma_desc_sw128_mn(ub + kk * 2048, kBwQ * 128), id_o,
                                 (t > 0 || kk > 0) ? 1u : 0u);
                    umma_bf16_ts(tmem + 384, tmem + 128 + pb * 64 + kk * 8, umma_desc_sw128_mn(qb + kk * 2048, kBwQ * 128),
                                 id_o, (t > 0 || kk > 0) ? 1u : 0u);
                }
                umma_commit(&st_empty[st]);
            }
            umma_commit(acc_done);
        }
    } else {
        // ===================== compute: warpgroup wg, thread = key row; tiles t = wg, wg + 2, ...
        const int wg = warp >> 2, w4 = warp & 3;
        const int kr = w4 * 32 + lane, j = k0 + kr;
        const uint32_t la = tmem + (uint32_t(w4 * 32) << 16);
        const float mkey = !p.mask ? 1.f : j < g.t_k ? __ldg(p.mask + kv_row0 + j) : 0.f;
        float* wl = cw + warp * 2 * kBwQ;  // lse[64], D[64]
        float dm = 0.f;
        float nl0 = 0.f, nl1 = 0.f, nd0 = 0.f, nd1 = 0.f;
        auto fetch = [&](int t) {
            if (t >= ntiles) return;
            const size_t rb = (size_t)head_of(t) * g.t_q;
            const int r0 = qtile_of(t) * kBwQ;
            nl0 = r0 + lane < g.t_q ? __ldg(p.lse + rb + r0 + lane) : 0.f;
            nl1 = r0 + lane + 32 < g.t_q ? __ldg(p.lse + rb + r0 + lane + 32) : 0.f;
            nd0 = r0 + lane < g.t_q ? __ldg(p.dsum + rb + r0 + lane) : 0.f;
            nd1 = r0 + lane + 32 < g.t_q ? __ldg(p.dsum + rb + r0 + lane + 32) : 0.f;
        };
        fetch(wg);
        const int jw0 = k0 + w4 * 32;
        const int bb = wg;  // this warpgroup's S^T / dP^T / P^T / dS^T TMEM buffers
        for (int t = wg; t < ntiles; t += kBwWG) {
            const int r0 = qtile_of(t) * kBwQ;
            wl[lane] = nl0;
            wl[lane + 32] = nl1;
            wl[kBwQ + lane] = nd0;
            wl[kBwQ + lane + 32] = nd1;
            __syncwarp();
            fetch(t + kBwWG);
            mbar_wait(&s_full[bb], (t >> 1) & 1);
            __syncwarp();  // reconverge before .sync.aligned tcgen05.ld
            tc_fence_after();
            const bool interior = jw0 + 32 <= g.t_k && r0 + kBwQ <= g.t_q && (!g.causal || jw0 + 31 <= g.pos_offset + r0) &&
                                  !(g.self_keep && jw0 + 31 >= g.pos_offset + r0);
            // two 32-query chunks: S^T and dP^T columns of a chunk (64 registers) -> P^T, dS^T rows
            // INT: every (query, key) of this warp's tile is admissible and none is a kept self key
            auto chunk = [&](auto int_tag, int h2, const uint32_t (&sv)[32], const uint32_t (&dv)[32]) {
                constexpr bool INT = decltype(int_tag)::value;
                float dmq[4] = {0.f, 0.f, 0.f, 0.f};  // dmask partial sums (4 independent chains)
                uint32_t pt[16], dt[16];
                if constexpr (INT) {
                    // packed pairs of adjacent queries (FFMA2 / FMUL2 / FADD2; lse / D pairs as 8-byte loads)
                    const float2 c2 = make_float2(g.c, g.c), mk2 = make_float2(mkey, mkey);
                    const float2* wl2 = reinterpret_cast<const float2*>(wl + h2 * 32);
                    const float2* wd2 = reinterpret_cast<const float2*>(wl + kBwQ + h2 * 32);
                    float2 dma[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const float2 l2 = wl2[e], d2 = wd2[e];
                        float2 a2 = __ffma2_rn(make_float2(__uint_as_float(sv[2 * e]), __uint_as_float(sv[2 * e + 1])), c2,
                                               make_float2(-l2.x, -l2.y));
                        const float2 pm = make_float2(fast_exp2(a2.x), fast_exp2(a2.y));
                        const float2 dpv = __fadd2_rn(make_float2(__uint_as_float(dv[2 * e]), __uint_as_float(dv[2 * e + 1])),
                                                      make_float2(-d2.x, -d2.y));
                        dma[e & 1] = __ffma2_rn(pm, dpv, dma[e & 1]);
                        const float2 pj = __fmul2_rn(pm, mk2);
                        const float2 ds = __fmul2_rn(pj, dpv);
                        pt[e] = pack2(pj.x, pj.y);
                        dt[e] = pack2(ds.x, ds.y);
                    }
                    dmq[0] = dma[0].x;
                    dmq[1] = dma[0].y;
                    dmq[2] = dma[1].x;
                    dmq[3] = dma[1].y;
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t pw[4], dw[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            float pv[2], dsv[2];
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int i = c * 8 + e * 2 + h, q = h2 * 32 + i, r = r0 + q;
                                float pm = fast_exp2(fmaf(__uint_as_float(sv[i]), g.c, -wl[q]));
                                if (!admissible(g, j, r)) pm = 0.f;
                                const bool self = g.self_keep && j == g.pos_offset + r;
                                const float dpv = __uint_as_float(dv[i]) - wl[kBwQ + q];
                                const float pj = self ? pm : pm * mkey;
                                if (!self) dmq[i & 3] = fmaf(pm, dpv, dmq[i & 3]);
                                pv[h] = pj;
                                dsv[h] = pj * dpv;
                            }
                            pw[e] = pack2(pv[0], pv[1]);
                            dw[e] = pack2(dsv[0], dsv[1]);
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            pt[c * 4 + e] = pw[e];
                            dt[c * 4 + e] = dw[e];
                        }
                    }
                }
                // P^T / dS^T chunk over S^T / dP^T columns this thread has already read
                tmem_st16(la + bb * 64 + h2 * 16, pt);
                tmem_st16(la + 128 + bb * 64 + h2 * 16, dt);
                dm += (dmq[0] + dmq[1]) + (dmq[2] + dmq[3]);
            };
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                uint32_t sv[32], dv[32];
                tmem_ld_32x32b_x32(la + bb * 64 + h2 * 32, sv);
                tmem_ld_32x32b_x32(la + 128 + bb * 64 + h2 * 32, dv);
                tmem_ld_wait_dep(sv);
                tmem_ld_wait_dep(dv);
                if (interior) chunk(std::true_type{}, h2, sv, dv);
                else chunk(std::false_type{}, h2, sv, dv);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&pt_full[bb]);
        }
        // ---- epilogue: warpgroup 0 writes dV, warpgroup 1 dK (x scale); dmask from both
        if (ntiles > 0) {
            mbar_wait(acc_done, 0);
            __syncwarp();  // reconverge before .sync.aligned tcgen05.ld
            tc_fence_after();
        }
        {
            const int which = wg;
            float* dst = (which ? p.dk : p.dv) + (kv_row0 + j) * kD;
            const float f = which ? g.scale : 1.f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t rr[32];
                if (ntiles > 0) {
                    tmem_ld_32x32b_x32(la + 256 + which * 128 + c * 32, rr);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) rr[i] = 0u;
                }
                if (j < g.t_k) {
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        *reinterpret_cast<float4*>(dst + c * 32 + q * 4) =
                            make_float4(__uint_as_float(rr[q * 4]) * f, __uint_as_float(rr[q * 4 + 1]) * f,
                                        __uint_as_float(rr[q * 4 + 2]) * f, __uint_as_float(rr[q * 4 + 3]) * f);
                }
            }
        }
        if (wg == 1) dmx[kr] = dm;
        named_bar_sync_attn(1, kBwWG * 4 * 32);
        if (wg == 0 && p.dmask && j < g.t_k) p.dmask[kv_row0 + j] = dm + dmx[kr];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kBwMma) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// dQ: CTA = two 128-query tiles, one compute warpgroup each (ping-pong on shared K/V tiles, as in
// the forward).  TMEM per warpgroup: S [0,64) (dS written over its first 32 columns as packed bf16,
// the A operand of dQ += dS K), dP [64,128), dQ [128,256) at wg * 256.
constexpr int kDqThreads = (kTcWG * 4 + 2) * 32;
constexpr int kDqStages = 3;  // K / V tile ring

__global__ void __launch_bounds__(kDqThreads, 1)
    dq_tc_kernel(const __grid_constant__ AttnParams p, const __grid_constant__ CUtensorMap tq128,
                 const __grid_constant__ CUtensorMap tdo128, const __grid_constant__ CUtensorMap tk64,
                 const __grid_constant__ CUtensorMap tv64) {
    constexpr uint32_t kQ128 = kTcQ * 256, kT64 = kTcK * 256, kStage = 2 * kT64;
    // ~226 KB of shared memory: no room for a manual 1024-byte round-up; the dynamic window starts
    // right after the 1 KB reserved block, which is 1024-aligned (checked below)
    extern __shared__ __align__(1024) unsigned char smem_dyn[];
    unsigned char* smem = smem_dyn;
    unsigned char* qs = smem;                        // [wg] Q tiles
    unsigned char* us = qs + kTcWG * kQ128;          // [wg] dO tiles
    unsigned char* stg = us + kTcWG * kQ128;         // [kDqStages] x {K, V}
    float* mw = reinterpret_cast<float*>(stg + kDqStages * kStage);  // [8 warps][64]
    uint64_t* bars = reinterpret_cast<uint64_t*>(mw + kTcWG * 4 * kTcK);
    uint64_t* q_full = bars;
    uint64_t* st_full = bars + 1;                 // [kDqStages]
    uint64_t* st_empty = st_full + kDqStages;     // [kDqStages]
    uint64_t* s_full = st_empty + kDqStages;      // [wg]
    uint64_t* ds_full = s_full + kTcWG;           // [wg]
    uint64_t* dq_done = ds_full + kTcWG;          // [wg]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + kTcWG);
    if ((smem_u32(smem) & 1023) != 0) {
        if (threadIdx.x == 0) latch_error(p.err, LKV_ERR_UNSUPPORTED, 1024);
        return;
    }

    const Geo g{p.n_q_heads, p.n_kv_heads, p.n_q_heads / p.n_kv_heads, p.t_q, p.t_k, p.causal, p.pos_offset,
                p.self_keep, p.scale * kLog2e, p.scale};
    const int b = blockIdx.z, qh = blockIdx.y, kvh = qh / g.G;
    // causal: the last query blocks see the most keys -- dispatch them first (longest first keeps
    // the last wave short)
    const int qb = p.causal ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x;
    const int q0 = qb * (kTcWG * kTcQ);
    int nt[kTcWG];
#pragma unroll
    for (int w = 0; w < kTcWG; ++w) nt[w] = tc_tiles(g, q0 + w * kTcQ);
    const int n_all = max(nt[0], nt[1]);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kTmaWarp = kTcWG * 4, kMmaWarp = kTcWG * 4 + 1;
    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < kDqStages; ++i) {
            mbar_init(&st_full[i], 1);
            mbar_init(&st_empty[i], 1);
        }
        for (int w = 0; w < kTcWG; ++w) {
            mbar_init(&s_full[w], 1);
            mbar_init(&ds_full[w], 4);
            mbar_init(&dq_done[w], 1);
        }
        fence_barrier_init();
    }
    if (warp == kMmaWarp) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const size_t kv_row0 = ((size_t)b * g.n_kv_heads + kvh) * g.t_k;
    const size_t q_row0 = ((size_t)b * g.n_q_heads + qh) * g.t_q;

    if (warp == kTmaWarp) {
        if (lane == 0 && n_all > 0) {
            const uint64_t pol = l2_policy_evict_last();
            mbar_arrive_expect_tx(q_full, 2 * kTcWG * kQ128);
#pragma unroll
            for (int w = 0; w < kTcWG; ++w) {
                tma_tile<kTcQ>(qs + w * kQ128, &tq128, q_full, (int)(q_row0 + q0 + w * kTcQ), pol);
                tma_tile<kTcQ>(us + w * kQ128, &tdo128, q_full, (int)(q_row0 + q0 + w * kTcQ), pol);
            }
            for (int t = 0; t < n_all; ++t) {
                const int st = t % kDqStages;
                if (t >= kDqStages) mbar_wait_backoff(&st_empty[st], ((t / kDqStages) - 1) & 1);
                mbar_arrive_expect_tx(&st_full[st], kStage);
                unsigned char* d = stg + st * kStage;
                tma_tile<kTcK>(d, &tk64, &st_full[st], (int)(kv_row0 + t * kTcK), pol);
                tma_tile<kTcK>(d + kT64, &tv64, &st_full[st], (int)(kv_row0 + t * kTcK), pol);
            }
        }
    } else if (warp == kMmaWarp) {
        if (lane == 0 && n_all > 0) {
            constexpr uint32_t id_s = umma_idesc_bf16(kTcQ, kTcK), id_o_mn = umma_idesc_bf16_bmn(kTcQ, kD);
            const uint32_t sa = smem_u32(stg);
            mbar_wait_backoff(q_full, 0);
            auto issue_s = [&](int w, int t) {  // S = Q K^T and dP = dO V^T of warpgroup w, tile t
                const uint32_t kb = sa + (t % kDqStages) * kStage, vb = kb + kT64;
                const uint32_t qa = smem_u32(qs + w * kQ128), ua = smem_u32(us + w * kQ128);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t ao = (kk >> 2) * (kTcQ * 128) + (kk & 3) * 32, bo = (kk >> 2) * (kTcK * 128) + (kk & 3) * 32;
                    umma_bf16(tmem + w * 256, umma_desc_sw128(qa + ao), umma_desc_sw128(kb + bo), id_s, kk > 0);
                    umma_bf16(tmem + w * 256 + 64, umma_desc_sw128(ua + ao), umma_desc_sw128(vb + bo), id_s, kk > 0);
                }
                umma_commit(&s_full[w]);
            };
            mbar_wait_backoff(&st_full[0], 0);
            tc_fence_after();
#pragma unroll
            for (int w = 0; w < kTcWG; ++w)
                if (nt[w] > 0) issue_s(w, 0);
            for (int t = 0; t < n_all; ++t) {
                const int st = t % kDqStages;
                const uint32_t kb = sa + st * kStage;
                bool next_ready = false;
                // per warpgroup: dQ of tile t as soon as its dS lands (A = dS from TMEM, over S), then
                // at once its S / dP of tile t + 1 -- in issue order, so dQ(t) has read dS(t) before
                // S(t+1) overwrites it -- so each warpgroup's row math overlaps the other's MMAs
#pragma unroll
                for (int w = 0; w < kTcWG; ++w) {
                    if (t >= nt[w]) continue;
                    mbar_wait_backoff(&ds_full[w], t & 1);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_bf16_ts(tmem + w * 256 + 128, tmem + w * 256 + kk * 8,
                                     umma_desc_sw128_mn(kb + kk * 2048, kTcK * 128), id_o_mn, (t > 0 || kk > 0) ? 1u : 0u);
                    if (t + 1 < nt[w]) {
                        if (!next_ready) {
                            mbar_wait_backoff(&st_full[(t + 1) % kDqStages], ((t + 1) / kDqStages) & 1);
                            tc_fence_after();
                            next_ready = true;
                        }
                        issue_s(w, t + 1);
                    } else {
                        umma_commit(&dq_done[w]);
                    }
                }
                umma_commit(&st_empty[st]);
            }
        }
    } else {
        // ===================== compute: warpgroup wg, thread = query row
        const int wg = warp >> 2, w4 = warp & 3;
        const int ntw = nt[wg];
        const int rl = w4 * 32 + lane, r = q0 + wg * kTcQ + rl;
        const uint32_t la = tmem + (uint32_t(w4 * 32) << 16) + wg * 256;
        const float lse = r < g.t_q ? p.lse[q_row0 + r] : 0.f, dd = r < g.t_q ? p.dsum[q_row0 + r] : 0.f;
        const float* mask = p.mask ? p.mask + kv_row0 : nullptr;
        float* mwarp = mw + warp * kTcK;
        float mn0 = 0.f, mn1 = 0.f;
        if (mask) {
            mn0 = lane < g.t_k ? __ldg(mask + lane) : 0.f;
            mn1 = lane + 32 < g.t_k ? __ldg(mask + lane + 32) : 0.f;
        }
        const int wr0 = q0 + wg * kTcQ + w4 * 32;
        for (int t = 0; t < ntw; ++t) {
            const int j0 = t * kTcK;
            if (mask) {
                mwarp[lane] = mn0;
                mwarp[lane + 32] = mn1;
                __syncwarp();
                const int jn = j0 + kTcK;
                mn0 = jn + lane < g.t_k ? __ldg(mask + jn + lane) : 0.f;
                mn1 = jn + lane + 32 < g.t_k ? __ldg(mask + jn + lane + 32) : 0.f;
            }
            mbar_wait(&s_full[wg], t & 1);
            __syncwarp();  // reconverge before .sync.aligned tcgen05.ld
            tc_fence_after();
            uint32_t sv[64], dv[64];
            tmem_ld_32x32b_x32(la, *reinterpret_cast<uint32_t(*)[32]>(sv));
            tmem_ld_32x32b_x32(la + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
            tmem_ld_32x32b_x32(la + 64, *reinterpret_cast<uint32_t(*)[32]>(dv));
            tmem_ld_32x32b_x32(la + 96, *reinterpret_cast<uint32_t(*)[32]>(dv + 32));
            tmem_ld_wait_dep(*reinterpret_cast<uint32_t(*)[32]>(sv));
            tmem_ld_wait_dep(*reinterpret_cast<uint32_t(*)[32]>(sv + 32));
            tmem_ld_wait_dep(*reinterpret_cast<uint32_t(*)[32]>(dv));
            tmem_ld_wait_dep(*reinterpret_cast<uint32_t(*)[32]>(dv + 32));
            const bool interior = j0 + kTcK <= g.t_k && wr0 + 32 <= g.t_q && (!g.causal || j0 + kTcK - 1 <= g.pos_offset + wr0) &&
                                  !(g.self_keep && j0 + kTcK - 1 >= g.pos_offset + wr0);
            uint32_t dsw[32];  // dS row, packed bf16 -> TMEM over S (all of S and dP already read)
            auto tile_body = [&](auto int_tag) {  // INT: no per-element admissibility tests
                constexpr bool INT = decltype(int_tag)::value;
                if constexpr (INT) {  // packed pairs of adjacent keys (FFMA2 / FMUL2 / FADD2)
                    const float2 c2 = make_float2(g.c, g.c), nl2 = make_float2(-lse, -lse), nd2 = make_float2(-dd, -dd);
                    const float2* m2 = reinterpret_cast<const float2*>(mwarp);
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const float2 a2 = __ffma2_rn(make_float2(__uint_as_float(sv[2 * e]), __uint_as_float(sv[2 * e + 1])), c2, nl2);
                        float2 pm = make_float2(fast_exp2(a2.x), fast_exp2(a2.y));
                        if (mask) pm = __fmul2_rn(pm, m2[e]);
                        const float2 dpv = __fadd2_rn(make_float2(__uint_as_float(dv[2 * e]), __uint_as_float(dv[2 * e + 1])), nd2);
                        const float2 ds = __fmul2_rn(pm, dpv);
                        dsw[e] = pack2(ds.x, ds.y);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        uint32_t dw[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            float dsv[2];
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int i = c * 8 + e * 2 + h, jj = j0 + i;
                                float mj = mask ? mwarp[i] : 1.f;
                                float pm = fast_exp2(fmaf(__uint_as_float(sv[i]), g.c, -lse));
                                if (!admissible(g, jj, r)) pm = 0.f;
                                if (g.self_keep && jj == g.pos_offset + r) mj = 1.f;
                                dsv[h] = pm * mj * (__uint_as_float(dv[i]) - dd);
                            }
                            dw[e] = pack2(dsv[0], dsv[1]);
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) dsw[c * 4 + e] = dw[e];
                    }
                }
            };
            if (interior) tile_body(std::true_type{});
            else tile_body(std::false_type{});
            tmem_st32(la, dsw);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&ds_full[wg]);
        }
        if (ntw > 0) {  // the last dQ of this warpgroup has landed
            mbar_wait(&dq_done[wg], 0);
            __syncwarp();  // reconverge before .sync.aligned tcgen05.ld
            tc_fence_after();
        }
        float* drw = p.dq + (q_row0 + r) * kD;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t rr[32];
            if (ntw > 0) {
                tmem_ld_32x32b_x32(la + 128 + c * 32, rr);
                tmem_ld_wait();
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) rr[i] = 0u;
            }
            if (r < g.t_q) {
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    *reinterpret_cast<float4*>(drw + c * 32 + q * 4) =
                        make_float4(__uint_as_float(rr[q * 4]) * g.scale, __uint_as_float(rr[q * 4 + 1]) * g.scale,
                                    __uint_as_float(rr[q * 4 + 2]) * g.scale, __uint_as_float(rr[q * 4 + 3]) * g.scale);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
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



size_t attn_fwd_tc_smem() {
    return 1024 + attn::kTcWG * attn::kTcQ * 256 + attn::kF2Stages * 2 * attn::kF2K * 256 +
           attn::kTcWG * 4 * attn::kF2K * 4 + 16 * 8 + 16;
}

// mk / mv / mq: 128-row boxes
cudaError_t launch_attn_fwd(const AttnParams& p, int dtype, int d, const CUtensorMap* mk, const CUtensorMap* mv,
                            const CUtensorMap* mq, cudaStream_t stream) {
    if (p.mask) {
        const int64_t n = (int64_t)p.batch * p.n_kv_heads * p.t_k;
        attn::mask_check_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1184), 256, 0, stream>>>(p.mask, n, p.err);
        note_launches(1);
    }
    if (dtype == LKV_BF16) {
        constexpr int rows_per_cta = attn::kTcWG * attn::kTcQ;
        const dim3 grid((p.t_q + rows_per_cta - 1) / rows_per_cta, p.n_q_heads, p.batch);
        const size_t smem = attn_fwd_tc_smem();
        cudaError_t e = cudaFuncSetAttribute(attn::fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attn::fwd_tc_kernel<<<grid, attn::kTcThreads, smem, stream>>>(p, *mq, *mk, *mv);
        note_launches(1);
    } else {
        const size_t smem = (size_t)(d + p.t_k) * 4;
        cudaError_t e = cudaFuncSetAttribute(attn::fwd_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attn::fwd_f32_kernel<<<dim3(p.t_q, p.n_q_heads, p.batch), attn::kSimt, smem, stream>>>(p, d);
    }
    note_launches(1);
    return cudaGetLastError();
}

size_t attn_dq_tc_smem() {  // no alignment slack (see dq_tc_kernel)
    return 2 * attn::kTcWG * attn::kTcQ * 256 + attn::kDqStages * 2 * attn::kTcK * 256 + attn::kTcWG * 4 * attn::kTcK * 4 +
           (1 + 2 * attn::kDqStages + 3 * attn::kTcWG) * 8 + 16;
}
size_t attn_dkv_tc_smem() {
    return 1024 + 2 * attn::kBwK * 256 + attn::kBwStages * 2 * attn::kBwQ * 256 + attn::kBwWG * 4 * 2 * attn::kBwQ * 4 +
           attn::kBwK * 4 + (2 * attn::kBwStages + 6) * 8 + 16;
}

// m: dQ maps {Q(128-row boxes), dO(128), K(64), V(64)}, dKV maps {K(128), V(128), Q(64), dO(64)}
cudaError_t launch_attn_bwd(const AttnParams& p, int dtype, int d, const CUtensorMap* m, cudaStream_t stream) {
    const int64_t rows = (int64_t)p.batch * p.n_q_heads * p.t_q;
    cudaError_t e;
    if (dtype == LKV_BF16) {
        attn::bwd_prep_kernel<__nv_bfloat16><<<(unsigned)((rows + 3) / 4), 128, 0, stream>>>(
            static_cast<const __nv_bfloat16*>(p.out), static_cast<const __nv_bfloat16*>(p.dout), p.dsum, rows, d);
        const size_t s1 = attn_dq_tc_smem(), s2 = attn_dkv_tc_smem();
        if ((e = cudaFuncSetAttribute(attn::dq_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1)))
            return e;
        if ((e = cudaFuncSetAttribute(attn::dkv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2)))
            return e;
        constexpr int dq_rows = attn::kTcWG * attn::kTcQ;
        attn::dq_tc_kernel<<<dim3((p.t_q + dq_rows - 1) / dq_rows, p.n_q_heads, p.batch), attn::kDqThreads, s1,
                             stream>>>(p, m[0], m[1], m[2], m[3]);
        attn::dkv_tc_kernel<<<dim3((p.t_k + attn::kBwK - 1) / attn::kBwK, p.n_kv_heads, p.batch), attn::kBwThreads, s2,
                              stream>>>(p, m[4], m[5], m[6], m[7]);
        note_launches(3);
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
