// model.cu -- the full decode step of the reference's toy GQA model: the
// step AFTER the eviction path.  Reference: decode_step (model.cpp:209-287): per layer
//   h = rmsnorm(x, attn_norm); q, k, v = h Wq, h Wk, h Wv; RoPE(q, k) at tokens_seen;
//   append (k, v) and attend (K5, decode.cu); x += attn Wo;
//   h2 = rmsnorm(x, mlp_norm); x += (silu(h2 Wgate) * (h2 Wup)) Wdown;
// then logits = rmsnorm(x, final_norm) lm_head.
//
// At decode batch sizes (B <= 16 sequences) every projection is a skinny GEMM whose cost is
// streaming the weights once from HBM (B flop per weight element, far below the ridge), so the
// kernel is a WEIGHT STREAM:
//  * weights are repacked once (lkv_model_load_param) into 16 KB units of 64 output columns x
//    128 k, stored in the register-fragment order of mma.m16n8k16 (A = W^T): one lds.128 per
//    lane per 16x16 tile, no ldmatrix, no bank conflicts; units of a matrix form one contiguous
//    stream [column group][k-unit];
//  * one wave of CTAs (2 per SM) splits the units evenly, so every SM streams about the same
//    bytes whatever the shape: narrow matrices as split-K thread-block clusters (S CTAs per
//    column group, partials summed by rank 0 over DSMEM), the rest as stream-K (CTA c owns units
//    [c U / P, (c+1) U / P)) on a grid aligned to column groups where one fits (S CTAs per group,
//    or k whole groups per CTA), so that no CTA stops its stream for a mid-stream fix-up;
//  * one producer thread moves each unit (plus the matching 2-4 KB slice of the packed
//    activations) with a 1-D bulk TMA copy into a 5-stage (one batch tile) / 4-stage mbarrier
//    ring; the first stages' WEIGHT copies, and 4 more units into L2, are issued before
//    griddepcontrol.wait, i.e. while the previous kernel of the step is still finishing (PDL);
//  * 4 consumer warps split each unit's 8 k-steps, accumulate on tensor cores (fp32), and
//    reduce across warps in fixed order; a column group shared by stream-K CTAs is finished by
//    the last-arriving CTA, which sums the partials in CTA order (deterministic);
//  * the epilogue is fused: RoPE + scatter into q / new k / new v (QKV), residual add + the
//    group's sum of squares + x * gain of the next rmsnorm written as the next GEMV's packed
//    activations (Wo, Wdown), SiLU(gate) * up written straight into the next GEMV's packed
//    activations (Wgate|Wup interleaved by 32 columns), fp32 logits;
//  * rmsnorm has no kernel of its own: rmsnorm(x) W = ((x * gain) W) / rms(x), so the GEMV that
//    consumes a normalised input scales its outputs by 1 / rms, computed from the producer's
//    per-group sums of squares (the bf16 rounding then applies to x * gain instead of
//    x * gain / rms -- the same relative error).
// fp32 models (correctness configs) run a SIMT kernel over plain row-major weights with the
// same virtual column order and the same epilogues.
#include <math.h>

#include <algorithm>

#include "kernels.cuh"

namespace lkv_dev {

constexpr int kWsCols = 64;                    // output columns per unit (4 m16 tiles)
constexpr int kWsK = 128;                      // k per unit (8 k16 steps)
constexpr int kWsUnitBytes = kWsCols * kWsK * 2;  // 16 KB of bf16
// ring depth: 5 stages with one batch tile (2 CTAs per SM still fit; n_seq 4 -0.3%, n_seq 1 equal,
// profiles/r02/xp_ws_stages.sh), 4 with two
template <int NBT>
constexpr int ws_stages() { return NBT == 1 ? 5 : 4; }
constexpr int kWsConsumers = 4;
constexpr int kWsThreads = (kWsConsumers + 1) * 32;
constexpr int kWsPerSm = 2;
constexpr int kYPad = 17;                      // y[64][17]: columns x batch (B <= 16)
constexpr int kWsMaxSplit = 1024;              // CTAs sharing one column group (<= KU + 1; K <= 130k)
constexpr int kWsMaxCluster = 8;               // split-K cluster size bound (launch_gemv)

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

__device__ __forceinline__ void mma_16816(float (&d)[4], const uint4& a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// ---- fused epilogues: y[n][b] = the finished fp32 product of column group ng ----------------------
template <typename T>
__device__ __forceinline__ void store2(void* base, size_t i, float a, float b) {
    if constexpr (sizeof(T) == 2) {
        *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(base) + i) = __floats2bfloat162_rn(a, b);
    } else {
        *reinterpret_cast<float2*>(static_cast<float*>(base) + i) = make_float2(a, b);
    }
}

// the next rmsnorm's input, x * gain (its 1 / rms is applied by the consuming GEMV's epilogue)
template <typename T>
__device__ __forceinline__ void store_norm_act(void* act, int b, int n, int dm, int nbt, float v) {
    if constexpr (sizeof(T) == 2) static_cast<__nv_bfloat16*>(act)[act_index(b, n, nbt)] = __float2bfloat16_rn(v);
    else static_cast<float*>(act)[(size_t)b * dm + n] = v;
}

// the decode step's deferred cache bookkeeping (DecodeParams::lens_deferred): every head of the step
// gained one row and every sequence one token; run by CTA 0 of the step's last GEMV, whose wait
// implies every layer's attention and combine have completed
__device__ __forceinline__ void gemv_step_bookkeeping(const GemvParams& p, int tid, int nthr) {
    if (blockIdx.x != 0) return;
    for (int i = tid; i < p.n_lens; i += nthr) p.lens_inc[i] += 1;
    for (int i = tid; i < p.n_seen; i += nthr) p.seen_inc[i] += 1;
}

// Per-CTA values every epilogue of the launch shares, computed once per CTA: the 1 / rms of the
// consumed activations' rmsnorm (model.cpp:48-53) and the step position of each batch row (RoPE,
// EPI_QKV).  The consumers issue the loads right after griddepcontrol.wait and finish the sums
// after their first group's units (the loads fly under the MMAs), so neither the stream's start nor
// any group epilogue waits on them.  Fast path: a warp per batch row (B <= 4 with the 4 consumer
// warps), <= 128 producer groups (four loads per lane); otherwise the sums run synchronously in the
// finish step.
__shared__ float ws_inv_rms[16];
__shared__ int ws_pos[16];
struct ProRegs {
    float v[4];
    int pos;
};
__device__ __forceinline__ bool prologue_fast(const GemvParams& p, int nthr) {
    return p.B * 32 <= nthr && p.norm_dm <= 128 * 64;
}
__device__ __forceinline__ ProRegs gemv_prologue_issue(const GemvParams& p, int tid, int nthr) {
    ProRegs r = {{0.f, 0.f, 0.f, 0.f}, 0};
    const int warp = tid >> 5, lane = tid & 31;
    if (p.ss_in && prologue_fast(p, nthr) && warp < p.B) {
        const int ngx = (p.norm_dm + 63) / 64;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (lane + 32 * k < ngx) r.v[k] = p.ss_in[(size_t)(lane + 32 * k) * p.B + warp];
    }
    if (p.epi == EPI_QKV && tid < p.B) r.pos = p.tokens_seen[tid];
    return r;
}
__device__ __forceinline__ void gemv_prologue_finish(const GemvParams& p, const ProRegs& r, int tid, int nthr) {
    const int B = p.B, warp = tid >> 5, lane = tid & 31;
    if (p.ss_in) {  // lanes stride over the producer's per-group sums of squares, fixed-order tree
        const int ngx = (p.norm_dm + 63) / 64;
        for (int b = warp; b < B; b += nthr >> 5) {
            float s;
            if (prologue_fast(p, nthr)) {
                s = ((r.v[0] + r.v[1]) + r.v[2]) + r.v[3];
            } else {
                s = 0.f;
                for (int gi = lane; gi < ngx; gi += 32) s += p.ss_in[(size_t)gi * B + b];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) ws_inv_rms[b] = 1.f / sqrtf(s / (float)p.norm_dm + p.norm_eps);
        }
    }
    if (p.epi == EPI_QKV && tid < B) ws_pos[tid] = min(max(r.pos, 0), p.max_seq - 1);
}

template <typename T>
__device__ void gemv_epilogue(const GemvParams& p, int ng, float (*y)[kYPad], int tid, int nthr) {
    const int B = p.B;
    if (p.ss_in) {  // rmsnorm of the consumed activations: W^T (x g / rms) = (W^T x g) / rms
        for (int e = tid; e < kWsCols * B; e += nthr) y[e & 63][e >> 6] *= ws_inv_rms[e >> 6];
        named_sync(1, nthr);
    }
    if (p.epi == EPI_QKV) {
        const int D = p.head_dim;
        for (int e = tid; e < 32 * B; e += nthr) {
            const int pr = e & 31, b = e >> 5;
            const int n = ng * kWsCols + 2 * pr;
            if (n >= p.N) continue;
            float a = y[2 * pr][b], c = y[2 * pr + 1][b];
            void* dst;
            int col, ld;
            bool rot = true;
            if (n < p.dm) {
                dst = p.q_out, col = n, ld = p.dm;
            } else if (n < p.dm + p.dkv) {
                dst = p.k_out, col = n - p.dm, ld = p.dkv;
            } else {
                dst = p.v_out, col = n - p.dm - p.dkv, ld = p.dkv, rot = false;
            }
            if (rot) {  // rope_row (model.cpp:38-46): pair j of the head, theta = pos * base^(-2j/d)
                const int pos = ws_pos[b];
                const float2 cs = p.rope[(size_t)pos * (D / 2) + (col % D) / 2];
                const float r0 = a * cs.x - c * cs.y, r1 = a * cs.y + c * cs.x;
                a = r0;
                c = r1;
            }
            store2<T>(dst, (size_t)b * ld + col, a, c);
        }
    } else if (p.epi == EPI_RESID) {
        for (int e = tid; e < kWsCols * B; e += nthr) {
            const int nl = e & 63, b = e >> 6;
            const int n = ng * kWsCols + nl;
            float v = 0.f;
            if (n < p.N) {
                v = p.x[(size_t)b * p.N + n] + y[nl][b];
                p.x[(size_t)b * p.N + n] = v;
                if (p.gain_next) store_norm_act<T>(p.act_next, b, n, p.N, p.nbt, v * p.gain_next[n]);
            }
            y[nl][b] = v * v;
        }
        named_sync(1, nthr);
        if (tid < B) {
            float s = 0.f;
            for (int nl = 0; nl < kWsCols; ++nl) s += y[nl][tid];
            p.ss_part[(size_t)ng * B + tid] = s;
        }
    } else if (p.epi == EPI_SWIGLU) {
        for (int e = tid; e < 32 * B; e += nthr) {
            const int i = e & 31, b = e >> 5;
            const int c = ng * 32 + i;
            if (c >= p.ff) continue;
            const float g = y[i][b], u = y[32 + i][b];
            const float a = g / (1.f + expf(-g)) * u;  // model.cpp:274-277
            if constexpr (sizeof(T) == 2)
                static_cast<__nv_bfloat16*>(p.act_out)[act_index(b, c, p.nbt_out)] = __float2bfloat16_rn(a);
            else
                static_cast<float*>(p.act_out)[(size_t)b * p.ff + c] = a;
        }
    } else {
        for (int e = tid; e < kWsCols * B; e += nthr) {
            const int nl = e & 63, b = e >> 6;
            const int n = ng * kWsCols + nl;
            if (n < p.N) p.f_out[(size_t)b * p.N + n] = y[nl][b];
        }
    }
}

// ---- bf16 weight-stream GEMV (tensor cores, stream-K) -------------------------------------------
__host__ __device__ __forceinline__ int64_t unit_begin(int c, int64_t U, int P) { return (int64_t)c * U / P; }
__device__ __forceinline__ int unit_owner(int64_t u, int64_t U, int P) { return (int)(((u + 1) * P - 1) / U); }

// SPLIT: narrow matrices (few column groups) run split-K instead of stream-K: each column group is
// cut into p.split equal k-ranges, one CTA each, forming a thread-block cluster; the partial
// products are summed by the cluster's rank-0 CTA straight from its peers' shared memory (DSMEM),
// in rank order (deterministic), instead of the stream-K global partials + arrival counter.
// ---- one GEMV phase over the CTA's unit range [u0, u1), shared by the single-GEMV kernel and the
// chained persistent kernel.  The ring (st, ph) carries over from phase to phase: producer and
// consumers walk the same unit sequence.
//
// Producer: weight unit + activation slice per stage.  The first min(n, stages) weight copies go out
// before `gate()` (griddepcontrol.wait for the first phase, the grid barrier of the previous phase in
// a chain): weights never depend on earlier work, activations do.
template <int NBT, typename Gate>
__device__ __forceinline__ void ws_produce(const GemvParams& p, int64_t u0, int64_t u1, unsigned char* smem,
                                           uint64_t* full, uint64_t* empty, int& st, uint32_t& ph, bool fresh,
                                           Gate&& gate) {
    constexpr int kActBytes = 8 * NBT * 256;
    constexpr int kStage = kWsUnitBytes + kActBytes;
    const uint64_t pol_w = l2_policy_evict_first(), pol_a = l2_policy_evict_last();
    const unsigned char* wsrc = static_cast<const unsigned char*>(p.w);
    const unsigned char* asrc = static_cast<const unsigned char*>(p.act);
    const int64_t n = u1 - u0;
    const int npre = (int)(n < ws_stages<NBT>() ? n : ws_stages<NBT>());
    const int st0 = st;
    for (int64_t i = 0; i < n; ++i) {
        if (!(fresh && i < ws_stages<NBT>())) mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], kStage);
        const int64_t u = u0 + i;
        bulk_g2s(smem + st * kStage, wsrc + (size_t)u * kWsUnitBytes, kWsUnitBytes, &full[st], pol_w);
        if (i >= npre)
            bulk_g2s(smem + st * kStage + kWsUnitBytes, asrc + (size_t)(u % p.KU) * kActBytes, kActBytes, &full[st],
                     pol_a);
        if (i == npre - 1) {
            // the next p.l2_ahead units after the ring's into L2 too, while the previous kernel finishes
            if (fresh)
                for (int64_t j = npre; j < n && j < npre + p.l2_ahead; ++j)
                    bulk_prefetch_l2(wsrc + (size_t)(u0 + j) * kWsUnitBytes, kWsUnitBytes);
            gate();
            for (int j = 0; j < npre; ++j) {
                const int sj = (st0 + j) % ws_stages<NBT>();
                bulk_g2s(smem + sj * kStage + kWsUnitBytes, asrc + (size_t)((u0 + j) % p.KU) * kActBytes, kActBytes,
                         &full[sj], pol_a);
            }
        }
        if (++st == ws_stages<NBT>()) {
            st = 0;
            ph ^= 1;
        }
    }
}

// Consumers (4 warps): mma.sync over each unit, fixed-order cross-warp reduction into y, stream-K
// fix-up of column groups cut by a CTA boundary (last-arriving CTA sums the partials in CTA order),
// fused epilogue.  SPLIT: one column group per CTA, reduced across the cluster by the caller.
template <int NBT, bool SPLIT>
__device__ __forceinline__ void ws_consume(const GemvParams& p, int64_t u0, int64_t u1, unsigned char* smem,
                                           uint64_t* full, uint64_t* empty, float* red, float (*y)[kYPad],
                                           int* s_last, int* s_slot, int& st, uint32_t& ph) {
    constexpr int kActBytes = 8 * NBT * 256;
    constexpr int kStage = kWsUnitBytes + kActBytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tid = threadIdx.x;  // 0..127
    const int64_t U = (int64_t)p.NG * p.KU;
    const int P = gridDim.x, c = blockIdx.x;
    const int g = lane >> 2, cq = (lane & 3) * 2;
    int64_t u = u0;
    const int ng_first = (int)(u0 / p.KU);
    const ProRegs pro = gemv_prologue_issue(p, tid, kWsConsumers * 32);
    if (p.n_lens | p.n_seen) gemv_step_bookkeeping(p, tid, kWsConsumers * 32);
    bool pro_done = false;
    while (u < u1) {
        const int ng = (int)(u / p.KU);
        const int64_t gbeg = (int64_t)ng * p.KU, gend = gbeg + p.KU;
        const int64_t se = min(u1, gend);
        const bool whole = (u == gbeg) && (se == gend);
        float acc[4][NBT][4];
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int bt = 0; bt < NBT; ++bt) acc[t][bt][0] = acc[t][bt][1] = acc[t][bt][2] = acc[t][bt][3] = 0.f;
        for (; u < se; ++u) {
            mbar_wait(&full[st], ph);
            const unsigned char* stg = smem + st * kStage;
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
                const int ks = warp * 2 + kk;
                uint2 bf[NBT];
#pragma unroll
                for (int bt = 0; bt < NBT; ++bt)
                    bf[bt] = *reinterpret_cast<const uint2*>(stg + kWsUnitBytes + ((ks * NBT + bt) * 32 + lane) * 8);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const uint4 a = *reinterpret_cast<const uint4*>(stg + ((ks * 4 + t) * 32 + lane) * 16);
#pragma unroll
                    for (int bt = 0; bt < NBT; ++bt) mma_16816(acc[t][bt], a, bf[bt].x, bf[bt].y);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (++st == ws_stages<NBT>()) {
                st = 0;
                ph ^= 1;
            }
        }
        if (!pro_done) {  // ordered before every epilogue by the named barriers below
            gemv_prologue_finish(p, pro, tid, kWsConsumers * 32);
            pro_done = true;
        }
        // ---- cross-warp reduction (fixed order) -> y[64][b]
        constexpr int BW = NBT * 8;
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int bt = 0; bt < NBT; ++bt) {
                float* r = red + (size_t)warp * kWsCols * BW;
                const int n = t * 16 + g, b = bt * 8 + cq;
                r[n * BW + b] = acc[t][bt][0];
                r[n * BW + b + 1] = acc[t][bt][1];
                r[(n + 8) * BW + b] = acc[t][bt][2];
                r[(n + 8) * BW + b + 1] = acc[t][bt][3];
            }
        named_sync(1, kWsConsumers * 32);
        for (int e = tid; e < kWsCols * BW; e += kWsConsumers * 32) {
            const int n = e / BW, b = e - n * BW;
            float v = red[e];
#pragma unroll
            for (int w = 1; w < kWsConsumers; ++w) v += red[(size_t)w * kWsCols * BW + e];
            y[n][b] = v;
        }
        named_sync(1, kWsConsumers * 32);
        if constexpr (SPLIT) break;  // one column group per CTA: reduced across the cluster by the caller
        if (!whole) {
            // stream-K fix-up: partial -> global slot; the last CTA of the group sums in CTA order
            const int slot = 2 * c + (ng == ng_first ? 0 : 1);
            float* mine = p.part + (size_t)slot * kWsCols * 16;
            for (int e = tid; e < kWsCols * 16; e += kWsConsumers * 32) __stcg(mine + e, y[e >> 4][e & 15]);
            // one release/acquire pair per CTA (bar.sync orders the other consumers' stores
            // before thread 0's fence, which is cumulative): a fence in every thread costs ~25 us
            named_sync(1, kWsConsumers * 32);
            const int cf = unit_owner(gbeg, U, P), cl = unit_owner(gend - 1, U, P);
            if (tid == 0) {
                __threadfence();
                const uint32_t old = atomicAdd(&p.cnt[ng], 1u);
                const int last = (int)old == cl - cf;
                if (last) {
                    p.cnt[ng] = 0u;  // self-reset for the next launch
                    __threadfence();
                }
                *s_last = last;
            }
            named_sync(1, kWsConsumers * 32);
            if (!*s_last) continue;
            // slot of every contributing CTA computed once (one 64-bit division each), then each
            // thread streams its two float4 of every partial with the loads of 4 CTAs in flight --
            // a division + dependent L2 round trip per element cost ~20 us per launch.  The sum
            // runs in CTA order, as before (deterministic).
            const int ncta = cl - cf + 1;
            for (int i = tid; i < ncta; i += kWsConsumers * 32) {
                const int cc = cf + i;
                s_slot[i] = 2 * cc + (ng == (int)(unit_begin(cc, U, P) / p.KU) ? 0 : 1);
            }
            named_sync(1, kWsConsumers * 32);
            float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
#pragma unroll 4
            for (int i = 0; i < ncta; ++i) {
                const float4* src = reinterpret_cast<const float4*>(p.part + (size_t)s_slot[i] * kWsCols * 16);
                const float4 a = __ldcg(src + tid), b = __ldcg(src + tid + kWsConsumers * 32);
                v0.x += a.x, v0.y += a.y, v0.z += a.z, v0.w += a.w;
                v1.x += b.x, v1.y += b.y, v1.z += b.z, v1.w += b.w;
            }
            {
                const int e0 = 4 * tid, e1 = 4 * (tid + kWsConsumers * 32);  // 16 | e: one y row each
                y[e0 >> 4][(e0 & 15) + 0] = v0.x, y[e0 >> 4][(e0 & 15) + 1] = v0.y;
                y[e0 >> 4][(e0 & 15) + 2] = v0.z, y[e0 >> 4][(e0 & 15) + 3] = v0.w;
                y[e1 >> 4][(e1 & 15) + 0] = v1.x, y[e1 >> 4][(e1 & 15) + 1] = v1.y;
                y[e1 >> 4][(e1 & 15) + 2] = v1.z, y[e1 >> 4][(e1 & 15) + 3] = v1.w;
            }
            named_sync(1, kWsConsumers * 32);
        }
        gemv_epilogue<__nv_bfloat16>(p, ng, y, tid, kWsConsumers * 32);
        named_sync(1, kWsConsumers * 32);
    }
}

// The split-K cluster's tail (after every CTA's units): rank 0 sums the partial products and runs
// the epilogue.  KE: outputs per consumer thread (1 when B <= 2, 8 up to B = 16).
template <int KE>
__device__ __forceinline__ void ws_split_tail(const GemvParams& p, int c, int rank, float (*y)[kYPad], float* red) {
    constexpr int kE = KE;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // Rank 0 sums the cluster's partial products (DSMEM, rank order) and runs the epilogue.  Only
    // the live batch columns are summed, every peer load of a thread's (up to 8) outputs in
    // flight at once.  The residual epilogue (Wo, down) is inlined: its x / gain loads are
    // issued before the cluster barrier and the group's sums of squares are warp reductions
    // (element e = tid + 128 k: a warp holds 32 columns of one batch row).  Peers leave as soon
    // as rank 0 has read their partials (split arrive / wait), freeing their slots for the
    // next kernel's CTAs while rank 0 finishes the epilogue.
    const int S = p.split, B = p.B, ngc = c / S;
    const int tid = threadIdx.x;
    const bool lead = rank == 0 && warp < kWsConsumers;
    const bool resid_fast = p.epi == EPI_RESID && !p.ss_in;
    float xr[kE], gr[kE];
#pragma unroll
    for (int k = 0; k < kE; ++k) {
        xr[k] = gr[k] = 0.f;
        const int e = tid + k * kWsConsumers * 32, n = ngc * kWsCols + (e & (kWsCols - 1));
        if (resid_fast && lead && e < B * kWsCols && n < p.N) {
            xr[k] = p.x[(size_t)(e >> 6) * p.N + n];
            if (p.gain_next) gr[k] = __ldg(p.gain_next + n);
        }
    }
    cluster_sync_all();  // every thread of every CTA in the cluster (the producer warp too)
    if (lead) {
        const uint32_t ybase = smem_u32(&y[0][0]);
        float t[kE][kWsMaxCluster];
#pragma unroll
        for (int k = 0; k < kE; ++k) {
            const int e = tid + k * kWsConsumers * 32;
            if (e < B * kWsCols) {
                const uint32_t a = ybase + (uint32_t)((e & (kWsCols - 1)) * kYPad + (e >> 6)) * 4u;
#pragma unroll
                for (int r = 1; r < kWsMaxCluster; ++r)
                    if (r < S) t[k][r] = dsmem_ld(dsmem_map(a, r));
            }
        }
#pragma unroll
        for (int k = 0; k < kE; ++k) {
            const int e = tid + k * kWsConsumers * 32;
            if (e < B * kWsCols) {
                float v = y[e & (kWsCols - 1)][e >> 6];
#pragma unroll
                for (int r = 1; r < kWsMaxCluster; ++r)
                    if (r < S) v += t[k][r];
                y[e & (kWsCols - 1)][e >> 6] = v;
            }
        }
    }
    __syncwarp();
    cluster_arrive();  // rank 0's consumers: after their peer reads; everyone else: now
    if (lead) {
        if (resid_fast) {
#pragma unroll
            for (int k = 0; k < kE; ++k) {
                const int e = tid + k * kWsConsumers * 32;  // warp-uniform row e >> 6
                if (e >= B * kWsCols) break;
                const int nl = e & (kWsCols - 1), bb = e >> 6, n = ngc * kWsCols + nl;
                float v = 0.f;
                if (n < p.N) {
                    v = xr[k] + y[nl][bb];
                    p.x[(size_t)bb * p.N + n] = v;
                    if (p.gain_next) store_norm_act<__nv_bfloat16>(p.act_next, bb, n, p.N, p.nbt, v * gr[k]);
                }
                float q = v * v;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
                if (lane == 0) red[2 * bb + (nl >> 5)] = q;
            }
            named_sync(1, kWsConsumers * 32);
            if (tid < B) p.ss_part[(size_t)ngc * B + tid] = red[2 * tid] + red[2 * tid + 1];
        } else {
            named_sync(1, kWsConsumers * 32);
            gemv_epilogue<__nv_bfloat16>(p, ngc, y, tid, kWsConsumers * 32);
        }
    }
    cluster_wait();  // peers stay resident until rank 0 has read their partials
}

template <int NBT, bool SPLIT>
__global__ void __launch_bounds__(kWsThreads, kWsPerSm) wstream_gemv_kernel(const __grid_constant__ GemvParams p) {
    constexpr int kActBytes = 8 * NBT * 256;  // 8 k16 steps x NBT tiles x 32 lanes x 8 B
    constexpr int kStage = kWsUnitBytes + kActBytes;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);  // aligned, still a __shared__ pointer
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + ws_stages<NBT>() * kStage);
    uint64_t* empty = full + ws_stages<NBT>();
    float* red = reinterpret_cast<float*>(empty + ws_stages<NBT>());  // [4][64][NBT * 8]
    float(*y)[kYPad] = reinterpret_cast<float(*)[kYPad]>(red + kWsConsumers * kWsCols * NBT * 8);
    int* s_last = reinterpret_cast<int*>(y + kWsCols);
    int* s_slot = s_last + 4;  // [kWsMaxSplit]: partial slots of the CTAs sharing a column group

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t U = (int64_t)p.NG * p.KU;
    const int P = gridDim.x, c = blockIdx.x;
    int64_t u0, u1;
    int rank = 0;
    if constexpr (SPLIT) {
        const int S = p.split, ng = c / S;
        rank = c - ng * S;  // == %cluster_ctarank (clusters of S consecutive CTAs)
        u0 = (int64_t)ng * p.KU + (int64_t)rank * p.KU / S;
        u1 = (int64_t)ng * p.KU + (int64_t)(rank + 1) * p.KU / S;
    } else {
        u0 = unit_begin(c, U, P);
        u1 = unit_begin(c + 1, U, P);
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < ws_stages<NBT>(); ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kWsConsumers);
        }
        fence_barrier_init();
    }
    __syncthreads();
    pdl_trigger();
    int st = 0;
    uint32_t ph = 0;
    if (warp == kWsConsumers) {
        // weights do not depend on the previous kernel: the first stages stream before the wait
        if (lane == 0 && u1 > u0) ws_produce<NBT>(p, u0, u1, smem, full, empty, st, ph, true, [] { pdl_wait(); });
        if constexpr (!SPLIT) return;
    } else {
        pdl_wait();
        ws_consume<NBT, SPLIT>(p, u0, u1, smem, full, empty, red, y, s_last, s_slot, st, ph);
    }
    if constexpr (SPLIT) {
        // B <= 2 batch rows: one output per thread (the decode step's common case, fewest registers)
        if (p.B * kWsCols <= kWsConsumers * 32) ws_split_tail<1>(p, c, rank, y, red);
        else ws_split_tail<kWsCols * 16 / (kWsConsumers * 32)>(p, c, rank, y, red);
    }
}

// ---- fp32 SIMT GEMV (correctness configs): one 64-thread block per column group ------------------
__global__ void __launch_bounds__(64) gemv_f32_kernel(const __grid_constant__ GemvParams p) {
    pdl_wait();
    gemv_prologue_finish(p, gemv_prologue_issue(p, threadIdx.x, 64), threadIdx.x, 64);
    if (p.n_lens | p.n_seen) gemv_step_bookkeeping(p, threadIdx.x, 64);
    __shared__ float y[kWsCols][kYPad];
    const int ng = blockIdx.x, nl = threadIdx.x;
    const int ldw = p.NG * kWsCols;
    const float* w = static_cast<const float*>(p.w) + ng * kWsCols + nl;
    const float* act = static_cast<const float*>(p.act);
    float acc[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) acc[b] = 0.f;
    for (int k = 0; k < p.K; ++k) {
        const float wv = w[(size_t)k * ldw];
#pragma unroll
        for (int b = 0; b < 16; ++b)
            if (b < p.B) acc[b] = fmaf(act[(size_t)b * p.K + k], wv, acc[b]);
    }
#pragma unroll
    for (int b = 0; b < 16; ++b) y[nl][b] = acc[b];
    __syncthreads();
    gemv_epilogue<float>(p, ng, y, nl, 64);
}

// ---- embedding (model.cpp:218-219): x = tok_embed[token]; per-group sums of squares --------------
template <typename T>
__global__ void __launch_bounds__(64) embed_kernel(const T* __restrict__ tab, const int32_t* tokens, int B, int dm,
                                                  int vocab, const int32_t* tokens_seen, int max_seq, float* x,
                                                  float* ss_part, const float* gain, void* act, int nbt, ErrWord* err) {
    pdl_trigger();  // let the next GEMV start streaming its weights
    pdl_wait();
    __shared__ float s_w[2];
    const int ng = blockIdx.x, b = blockIdx.y, n = ng * 64 + threadIdx.x;
    int tok = tokens[b];
    if (tok < 0 || tok >= vocab) {
        if (threadIdx.x == 0 && ng == 0) latch_error(err, LKV_ERR_CONTRACT, b);  // "token id out of vocab"
        tok = 0;
    }
    if (threadIdx.x == 0 && ng == 0 && (tokens_seen[b] < 0 || tokens_seen[b] >= max_seq))
        latch_error(err, LKV_ERR_CONTRACT, b);  // "sequence exceeds max_seq_len" (model.cpp:215)
    float v = 0.f;
    if (n < dm) {
        if constexpr (sizeof(T) == 2) v = __bfloat162float(tab[(size_t)tok * dm + n]);
        else v = tab[(size_t)tok * dm + n];
        x[(size_t)b * dm + n] = v;
        if (gain) store_norm_act<T>(act, b, n, dm, nbt, v * gain[n]);  // layer 0's attn_norm input
    }
    float s = v * v;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) ss_part[(size_t)ng * B + b] = s_w[0] + s_w[1];
}

// ---- weight repacking (once per model load) -----------------------------------------------------------
// src [K][cols] row-major (reference layout, x W); column c lands on virtual column
//   col_mode 0: col_off + c;   col_mode 1/2 (gate/up): (c / 32) * 64 + (mode == 2 ? 32 : 0) + c % 32.
__device__ __forceinline__ int virt_col(int c, int mode, int off) {
    return mode == 0 ? off + c : (c >> 5) * 64 + (mode == 2 ? 32 : 0) + (c & 31);
}
template <typename T>
__global__ void pack_weight_kernel(const T* __restrict__ src, int K, int cols, int mode, int off, int NG, int KU,
                                   T* __restrict__ dst) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)K * cols) return;
    const int k = (int)(i / cols), c = (int)(i - (int64_t)k * cols);
    const int vn = virt_col(c, mode, off);
    if constexpr (sizeof(T) == 4) {
        dst[(size_t)k * NG * 64 + vn] = src[i];
    } else {
        const int ng = vn >> 6, r = vn & 63, t = r >> 4, m = r & 15;
        const int ku = k >> 7, kk = k & 127, s = kk >> 4, kc = kk & 15;
        const int lane = (m & 7) * 4 + ((kc & 7) >> 1);
        const int reg = (m >> 3) + 2 * (kc >> 3);
        const size_t unit = (size_t)ng * KU + ku;
        dst[unit * (kWsUnitBytes / 2) + (((size_t)(s * 4 + t) * 32 + lane) * 8) + reg * 2 + (kc & 1)] = src[i];
    }
}

template <typename T>
__global__ void to_f32_kernel(const T* src, int n, float* dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        if constexpr (sizeof(T) == 2) dst[i] = __bfloat162float(src[i]);
        else dst[i] = src[i];
    }
}

// ---- host launchers ----------------------------------------------------------------------------------
size_t gemv_max_grid(int num_sms) { return (size_t)kWsPerSm * num_sms; }

static size_t wstream_smem(int nbt) {
    const size_t stage = kWsUnitBytes + 8 * nbt * 256;
    const int stages = nbt == 1 ? ws_stages<1>() : ws_stages<2>();
    return 128 + stages * stage + 2 * stages * 8 + (size_t)kWsConsumers * kWsCols * nbt * 8 * 4 +
           (size_t)kWsCols * kYPad * 4 + 16 + 4 * kWsMaxSplit;
}

cudaError_t launch_gemv(const GemvParams& p, int dtype, int num_sms, cudaStream_t stream) {
    if (dtype == LKV_BF16) {
        const int64_t U = (int64_t)p.NG * p.KU;
        const int64_t cap = (int64_t)kWsPerSm * num_sms;
        const size_t smem = wstream_smem(p.nbt);
        // narrow matrices: cluster split-K with S CTAs per column group, S a power of two <= 8, used
        // when the NG * S CTAs still fill >= 60% of the one-wave slots (measured on the Llama-3-8B
        // step: Wo / down at S = 4 beat stream-K; QKV at S = 2 (192 CTAs) beats the group-aligned
        // stream-K by 2% of the step, S = 3 is 3% slower -- profiles/r02/xp_qkv_cluster.sh)
        int S = 1;
        while (S < 8 && (int64_t)p.NG * S * 2 <= cap && S * 2 <= p.KU) S *= 2;
        if (S >= 2 && (int64_t)p.NG * S * 5 >= cap * 3) {
            GemvParams q = p;
            q.split = S;
            auto kern = q.nbt == 1 ? wstream_gemv_kernel<1, true> : wstream_gemv_kernel<2, true>;
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            e = launch_pdl_cluster(kern, dim3(q.NG * S), dim3(kWsThreads), smem, stream, S, q);
            note_launches(1);
            return e;
        }
        int grid = (int)(U < cap ? U : cap);
        // group-aligned stream-K grids: every column group split evenly over S CTAs (NG * S CTAs,
        // >= 90% of the slots), or every CTA holding k whole groups (NG / k CTAs, >= 75%): no CTA's
        // range crosses a group boundary, so no CTA pauses its weight stream for a mid-stream
        // fix-up (Llama-3-8B step, profiles/r02/xp_align.sh: QKV 296 -> 288 CTAs, gate/up 296 ->
        // 224, 3.136 -> 2.979 ms on the same box)
        if (p.NG <= cap) {
            const int64_t g2 = (int64_t)p.NG * (cap / p.NG);
            if (g2 * 10 >= cap * 9 && g2 <= U) grid = (int)g2;
        } else {
            const int k = (int)((p.NG + cap - 1) / cap);
            if (p.NG % k == 0 && (int64_t)(p.NG / k) * 4 >= cap * 3) grid = p.NG / k;
        }
        auto kern = p.nbt == 1 ? wstream_gemv_kernel<1, false> : wstream_gemv_kernel<2, false>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = launch_pdl(kern, dim3(grid), dim3(kWsThreads), smem, stream, p);
        note_launches(1);
        return e;
    }
    cudaError_t e = launch_pdl(gemv_f32_kernel, dim3(p.NG), dim3(64), 0, stream, p);
    note_launches(1);
    return e;
}

cudaError_t launch_embed(const void* tok_embed, int dtype, const int32_t* tokens, int B, int dm, int vocab,
                         const int32_t* tokens_seen, int max_seq, float* x, float* ss_part, const float* gain,
                         void* act, int nbt, ErrWord* err, cudaStream_t stream) {
    const dim3 grid((dm + 63) / 64, B);
    cudaError_t e;
    // a plain (fully serialised) launch: every kernel of the step starts after the previous
    // step has completed, which the per-layer attention's early K/V prefetch relies on
    if (dtype == LKV_BF16)
        embed_kernel<__nv_bfloat16><<<grid, 64, 0, stream>>>(static_cast<const __nv_bfloat16*>(tok_embed), tokens, B,
                                                             dm, vocab, tokens_seen, max_seq, x, ss_part, gain, act,
                                                             nbt, err);
    else
        embed_kernel<float><<<grid, 64, 0, stream>>>(static_cast<const float*>(tok_embed), tokens, B, dm, vocab,
                                                     tokens_seen, max_seq, x, ss_part, gain, act, nbt, err);
    e = cudaGetLastError();
    note_launches(1);
    return e;
}

cudaError_t launch_pack_weight(const void* src, int dtype, int K, int cols, int col_mode, int col_off, int NG, int KU,
                               void* dst, cudaStream_t stream) {
    const int64_t n = (int64_t)K * cols;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (dtype == LKV_BF16)
        pack_weight_kernel<__nv_bfloat16><<<blocks, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(src), K, cols,
                                                                      col_mode, col_off, NG, KU,
                                                                      static_cast<__nv_bfloat16*>(dst));
    else
        pack_weight_kernel<float><<<blocks, 256, 0, stream>>>(static_cast<const float*>(src), K, cols, col_mode,
                                                              col_off, NG, KU, static_cast<float*>(dst));
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_to_f32(const void* src, int dtype, int n, float* dst, cudaStream_t stream) {
    if (dtype == LKV_BF16)
        to_f32_kernel<__nv_bfloat16><<<(n + 255) / 256, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(src), n, dst);
    else
        to_f32_kernel<float><<<(n + 255) / 256, 256, 0, stream>>>(static_cast<const float*>(src), n, dst);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace lkv_dev
