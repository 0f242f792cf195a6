// score.cu -- K1: LKV-T token scorer  u = act(x W1 + b1) . w2   (policy.cpp:30-34,131-136)
//
// Two kernels:
//  * score_tc_kernel  (bf16, head_dim 128, hidden % 16 == 0): persistent,
//    warp-specialised tcgen05 kernel.  Warp 0 streams 128-row K (and V) tiles
//    with TMA (128-byte swizzle) into a multi-stage shared-memory ring; warp 1
//    issues tcgen05.mma (M=128, N=hidden, K=16) into a double-buffered TMEM
//    accumulator; two 4-warp epilogue groups drain TMEM with tcgen05.ld
//    (thread = row), add b1, apply SiLU / GELU-erf and reduce against w2 in
//    registers, writing one fp32 score per row.  QK^T is never formed.
//  * score_simt_kernel (fp32 inputs, or shapes outside the tensor-core
//    envelope): FP32 SIMT, warp per row.  TF32 would break the 1e-5 bar.
#include <math.h>

#include "kernels.cuh"

namespace lkv_dev {


__device__ __forceinline__ float act_f32(int act, float h) {
    if (act == LKV_ACT_SILU) return h / (1.0f + __expf(-h));
    return 0.5f * h * (1.0f + erff(h * 0.70710678118654752f));
}

// Epilogue activations on the MUFU path (approximations far inside the 1e-2 bf16 bar):
//  GELU-erf: gelu(h) = h * Phi(h) = 0.5 (h + |h| erf(|h|/sqrt2)); erf by Abramowitz-Stegun
//            7.1.28 (one rcp).  f() returns 2*gelu; w2 is
//            pre-scaled by 0.5.
//  SiLU:     h / (1 + e^{-h}) (tensor.cpp:371-378) with ex2 + rcp.
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// Packed-pair forms (sm_100 FFMA2/FMUL2/FADD2): the epilogue bounds K1 on the FMA pipe, so two
// accumulator columns go through every FP32 instruction at once (scalar FFMA measured 17% slower
// on K1, profiles/r02/k1_gelu_experiments.txt); MUFU stays scalar.
__device__ __forceinline__ float2 f2(float x, float y) { return make_float2(x, y); }
__device__ __forceinline__ float2 abs2(float2 v) { return make_float2(fabsf(v.x), fabsf(v.y)); }
template <int ACT>
struct EpiAct2;
template <>
struct EpiAct2<LKV_ACT_GELU_ERF> {  // 2 gelu(h)
    // Abramowitz-Stegun 7.1.28: erf(u) = 1 - (1 + a1 u + ... + a6 u^6)^-16, |error| <= 3e-7
    // (1.7e-6 in fp32); u = |h|/sqrt2 folded into the coefficients.  One MUFU (rcp) per element;
    // returns 2 gelu(h) = h + |h| erf(|h|/sqrt2), w2 pre-scaled by 0.5.
    static constexpr float kW2Scale = 0.5f;
    __device__ __forceinline__ static float2 f(float2 h) {
        const float2 ah = abs2(h);
        float2 y = __ffma2_rn(f2(5.382975000e-06f, 5.382975000e-06f), ah, f2(4.889063564e-05f, 4.889063564e-05f));
        y = __ffma2_rn(y, ah, f2(3.800357500e-05f, 3.800357500e-05f));
        y = __ffma2_rn(y, ah, f2(3.277626324e-03f, 3.277626324e-03f));
        y = __ffma2_rn(y, ah, f2(2.114100615e-02f, 2.114100615e-02f));
        y = __ffma2_rn(y, ah, f2(4.986734697e-02f, 4.986734697e-02f));
        y = __ffma2_rn(y, ah, f2(1.0f, 1.0f));
        y = __fmul2_rn(y, y);
        y = __fmul2_rn(y, y);
        y = __fmul2_rn(y, y);
        y = __fmul2_rn(y, y);
        const float2 r = f2(rcp_approx(y.x), rcp_approx(y.y));
        return __ffma2_rn(f2(-ah.x, -ah.y), r, __fadd2_rn(h, ah));
    }
};
template <>
struct EpiAct2<LKV_ACT_SILU> {  // h / (1 + e^-h)
    static constexpr float kW2Scale = 1.0f;
    __device__ __forceinline__ static float2 f(float2 h) {
        const float2 z = __fmul2_rn(h, f2(-1.4426950408889634f, -1.4426950408889634f));
        const float2 d = __fadd2_rn(f2(ex2_approx(z.x), ex2_approx(z.y)), f2(1.0f, 1.0f));
        return __fmul2_rn(h, f2(rcp_approx(d.x), rcp_approx(d.y)));
    }
};

__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

template <int C>
__device__ __forceinline__ void tmem_ld_x(uint32_t taddr, uint32_t (&r)[C]);
template <>
__device__ __forceinline__ void tmem_ld_x<32>(uint32_t taddr, uint32_t (&r)[32]) {
    tmem_ld_32x32b_x32(taddr, r);
}
template <>
__device__ __forceinline__ void tmem_ld_x<16>(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

// Incremental walk over the (seq, head, 128-row tile) order: a CTA's tiles are consecutive, so
// each step is a few integer ops instead of a search over the sequence table.
struct TileCursor {
    int s, hs, j, tph, t;
};

struct TileInfo {
    int head;      // flat head
    int row0;      // first row inside the head
    int t;         // tokens of this head
    int scorer;
};

__device__ __forceinline__ TileCursor cursor_at(const ScoreParams& p, int tile, int tile_rows) {
    TileCursor c;
    c.s = 0;
    while (c.s + 1 < p.seq.n_seq && p.tile_base[c.s + 1] <= tile) ++c.s;
    c.t = p.seq.len[c.s];
    c.tph = (c.t + tile_rows - 1) / tile_rows;
    const int local = tile - p.tile_base[c.s];
    c.hs = local / c.tph;
    c.j = local - c.hs * c.tph;
    return c;
}
__device__ __forceinline__ void cursor_next(const ScoreParams& p, TileCursor& c, int tile_rows) {
    if (++c.j == c.tph) {
        c.j = 0;
        if (++c.hs == p.seq.n_layers * p.seq.n_kv_heads) {
            c.hs = 0;
            if (++c.s < p.seq.n_seq) {
                c.t = p.seq.len[c.s];
                c.tph = (c.t + tile_rows - 1) / tile_rows;
            }
        }
    }
}
__device__ __forceinline__ TileInfo cursor_info(const ScoreParams& p, const TileCursor& c, int tile_rows) {
    const int H = p.seq.n_kv_heads;
    const int l = c.hs / H, h = c.hs - l * H;
    TileInfo ti;
    ti.head = c.s * p.seq.n_layers * H + c.hs;
    ti.row0 = c.j * tile_rows;
    ti.t = c.t;
    ti.scorer = l * p.stride_layer + h * p.stride_head;
    return ti;
}

__device__ __forceinline__ TileInfo decode_tile(const ScoreParams& p, int tile, int tile_rows) {
    int s = 0;
    while (s + 1 < p.seq.n_seq && p.tile_base[s + 1] <= tile) ++s;
    const int t = p.seq.len[s];
    const int tph = (t + tile_rows - 1) / tile_rows;
    const int local = tile - p.tile_base[s];
    const int hs = local / tph;
    const int j = local - hs * tph;
    const int H = p.seq.n_kv_heads;
    const int l = hs / H, h = hs - l * H;
    TileInfo ti;
    ti.head = s * p.seq.n_layers * H + hs;
    ti.row0 = j * tile_rows;
    ti.t = t;
    ti.scorer = l * p.stride_layer + h * p.stride_head;
    return ti;
}

// ============================================================================
// tcgen05 kernel
// ============================================================================
constexpr int kTcRows = 128;  // UMMA M
// Epilogue groups of 4 warps (one TMEM lane quarter each); group g drains accumulator
// stage g, i.e. every E-th tile.  Warps 0..3: TMA producer, MMA issuer, TMEM allocator, spare.
constexpr int kHistBins = 2048;  // top 11 key bits: the first radix digit of the top-k (select.cu)

template <int N, int NBOX>
struct TcCfg {
    static constexpr int kABox = kTcRows * 128;            // bytes of one 128-row x 64-col box
    static constexpr int kAStage = NBOX * kABox;           // one tile (k or [k;v])
    static constexpr int kWBox = N * 128;
    static constexpr int kW = NBOX * kWBox;
    static constexpr int kStages = (NBOX == 2) ? (N <= 64 ? 5 : 4) : 2;
    // [k;v] tiles (NBOX = 4) leave room for two epilogue groups only
    static constexpr int kEpi = (NBOX == 2) ? 4 : 2;
    static constexpr int kThreads = 128 + 128 * kEpi;
    static constexpr int kEpiChunk = kEpi > 2 ? 16 : 32;  // TMEM columns per tcgen05.ld (register budget)
    static constexpr int kAcc = kEpi * N;  // accumulator columns: one N-wide stage per epilogue group
    static constexpr int kTmemCols = (kAcc <= 32) ? 32 : (kAcc <= 64) ? 64 : (kAcc <= 128) ? 128 : (kAcc <= 256) ? 256 : 512;
    static_assert(kAcc <= 512, "TMEM holds 512 fp32 columns");
    static constexpr int kSmem = kStages * kAStage + kW + 256 + 2 * kEpi * N * 4 + kEpi * kHistBins * 4 + 1024;
    static_assert(kSmem <= 227 * 1024, "shared memory budget");
};

template <int N, int NBOX, int ACT>
__global__ void __launch_bounds__(TcCfg<N, NBOX>::kThreads, 1)
    score_tc_kernel(const __grid_constant__ ScoreParams p, const __grid_constant__ CUtensorMap tmap_k,
                    const __grid_constant__ CUtensorMap tmap_v, const __grid_constant__ CUtensorMap tmap_w,
                    int total_tiles) {
    using Cfg = TcCfg<N, NBOX>;
    constexpr int S = Cfg::kStages;
    constexpr int kEpi = Cfg::kEpi;
    constexpr int kEpiChunk = Cfg::kEpiChunk;
    extern __shared__ unsigned char smem_dyn[];
    unsigned char* smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);  // aligned, still a __shared__ pointer
    unsigned char* sA = smem;
    unsigned char* sW = smem + S * Cfg::kAStage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sW + Cfg::kW);
    uint64_t* full = bars;              // [S]
    uint64_t* empty = bars + S;         // [S]
    uint64_t* tfull = bars + 2 * S;           // [kEpi]
    uint64_t* tempty = bars + 2 * S + kEpi;   // [kEpi]
    uint64_t* wfull = bars + 2 * S + 2 * kEpi;
    uint64_t* wempty = wfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wempty + 1);
    float* sEpi = reinterpret_cast<float*>(sW + Cfg::kW + 256);  // [kEpi groups][b1 | w2][N]
    uint32_t* sHist = reinterpret_cast<uint32_t*>(sEpi + 2 * kEpi * N);  // [kEpi groups][kHistBins]

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    // Tile schedule: one contiguous range of (seq, head, 128-row tile) per CTA, so the tiles of
    // a head and the heads of a scorer stay together (weights and histogram flushes amortised).
    const int t_begin = (int)((int64_t)total_tiles * blockIdx.x / gridDim.x);
    const int n_local = (int)((int64_t)total_tiles * (blockIdx.x + 1) / gridDim.x) - t_begin;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < kEpi; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        mbar_init(wfull, 1);
        mbar_init(wempty, 1);
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_k);
        if (NBOX == 4) tma_prefetch_desc(&tmap_v);
        tma_prefetch_desc(&tmap_w);
    }
    if (warp == 2) tmem_alloc(tmem_slot, Cfg::kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint64_t pol_stream = l2_policy_evict_first();
            const uint64_t pol_keep = l2_policy_evict_last();
            int cur = -1, wloads = 0;
            TileCursor cur_t = cursor_at(p, t_begin, kTcRows);
            for (int i = 0; i < n_local; ++i) {
                if (i > 0) cursor_next(p, cur_t, kTcRows);
                const TileInfo ti = cursor_info(p, cur_t, kTcRows);
                if (ti.scorer != cur) {
                    if (wloads > 0) mbar_wait(wempty, (wloads - 1) & 1);
                    mbar_arrive_expect_tx(wfull, Cfg::kW);
#pragma unroll
                    for (int b = 0; b < NBOX; ++b)
                        tma_load_2d(sW + b * Cfg::kWBox, &tmap_w, wfull, (b & 1) * 64 + (b >> 1) * 128, ti.scorer * N,
                                    pol_keep);
                    cur = ti.scorer;
                    ++wloads;
                }
                const int st = i % S;
                mbar_wait(&empty[st], ((i / S) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[st], Cfg::kAStage);
                const int grow = (int)((int64_t)ti.head * p.seq.T + ti.row0);
                unsigned char* dst = sA + st * Cfg::kAStage;
                tma_load_2d(dst, &tmap_k, &full[st], 0, grow, pol_stream);
                tma_load_2d(dst + Cfg::kABox, &tmap_k, &full[st], 64, grow, pol_stream);
                if (NBOX == 4) {
                    tma_load_2d(dst + 2 * Cfg::kABox, &tmap_v, &full[st], 0, grow, pol_stream);
                    tma_load_2d(dst + 3 * Cfg::kABox, &tmap_v, &full[st], 64, grow, pol_stream);
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(kTcRows, N);
            const uint32_t a_base = smem_u32(sA);
            const uint32_t w_base = smem_u32(sW);
            int cur = -1, wuses = 0;
            TileCursor cur_t = cursor_at(p, t_begin, kTcRows);
            for (int i = 0; i < n_local; ++i) {
                if (i > 0) cursor_next(p, cur_t, kTcRows);
                const TileInfo ti = cursor_info(p, cur_t, kTcRows);
                if (ti.scorer != cur) {
                    if (wuses > 0) umma_commit(wempty);  // old weights free once prior MMAs retire
                    mbar_wait(wfull, wuses & 1);
                    cur = ti.scorer;
                    ++wuses;
                }
                const int acc = i % kEpi;
                mbar_wait(&tempty[acc], ((i / kEpi) & 1) ^ 1);
                const int st = i % S;
                mbar_wait(&full[st], (i / S) & 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * N;
                const uint32_t a_st = a_base + st * Cfg::kAStage;
#pragma unroll
                for (int kk = 0; kk < NBOX * 4; ++kk) {
                    const int box = kk >> 2, within = kk & 3;
                    const uint64_t adesc = umma_desc_sw128(a_st + box * Cfg::kABox + within * 32);
                    const uint64_t bdesc = umma_desc_sw128(w_base + box * Cfg::kWBox + within * 32);
                    umma_bf16(d_tmem, adesc, bdesc, idesc, kk > 0 ? 1u : 0u);
                }
                umma_commit(&empty[st]);   // smem slot free when these MMAs retire
                umma_commit(&tfull[acc]);  // accumulator ready
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue (2 groups x 4 warps) =====================
        const int grp = (warp - 4) >> 2;
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        float* s_b1 = sEpi + grp * 2 * N;  // this group's copy of b1 and the pre-scaled w2
        float* s_w2 = s_b1 + N;
        uint32_t* hist_g = sHist + grp * kHistBins;  // this group's top-digit histogram (fused K3 pass 1)
        const int j128 = threadIdx.x & 127;
        if (p.hist) {
            for (int b = j128; b < kHistBins; b += 128) hist_g[b] = 0;
        }
        auto flush_hist = [&](int head) {
            named_bar_sync(1 + grp, 128);
            for (int b = j128; b < kHistBins; b += 128) {
                const uint32_t v = hist_g[b];
                if (v) {
                    atomicAdd(p.hist + (size_t)head * kHistBins + b, v);
                    hist_g[b] = 0;
                }
            }
            named_bar_sync(1 + grp, 128);
        };
        int cur = -1, cur_head = -1;
        TileCursor cur_t = cursor_at(p, t_begin + grp, kTcRows);
        for (int i = grp; i < n_local; i += kEpi) {
            if (i > grp)
                for (int k = 0; k < kEpi; ++k) cursor_next(p, cur_t, kTcRows);
            const TileInfo ti = cursor_info(p, cur_t, kTcRows);
            if (p.hist && ti.head != cur_head) {
                if (cur_head >= 0) flush_hist(cur_head);
                else named_bar_sync(1 + grp, 128);  // zeroing complete
                cur_head = ti.head;
            }
            if (ti.scorer != cur) {  // stage this scorer's b1 / w2 once (group-local barrier)
                named_bar_sync(1 + grp, 128);
                const int j = threadIdx.x & 127;
                if (j < N) {
                    s_b1[j] = p.b1[(size_t)ti.scorer * N + j];
                    s_w2[j] = p.w2[(size_t)ti.scorer * N + j] * EpiAct2<ACT>::kW2Scale;
                }
                named_bar_sync(1 + grp, 128);
                cur = ti.scorer;
            }
            mbar_wait(&tfull[grp], (i / kEpi) & 1);
            __syncwarp();  // reconverge before .sync.aligned tcgen05.ld
            tc_fence_after();
            const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + grp * N;
            float2 s2 = f2(0.f, 0.f);
#pragma unroll
            for (int c = 0; c < N / kEpiChunk; ++c) {
                uint32_t r[kEpiChunk];
                tmem_ld_x<kEpiChunk>(taddr + c * kEpiChunk, r);
                tmem_ld_wait();
                if (c == N / kEpiChunk - 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[grp]);
                }
#pragma unroll
                for (int q = 0; q < kEpiChunk; q += 4) {
                    const float4 bb = *reinterpret_cast<const float4*>(s_b1 + c * kEpiChunk + q);
                    const float4 ww = *reinterpret_cast<const float4*>(s_w2 + c * kEpiChunk + q);
                    const float2 h0 = __fadd2_rn(f2(__uint_as_float(r[q + 0]), __uint_as_float(r[q + 1])), f2(bb.x, bb.y));
                    const float2 h1 = __fadd2_rn(f2(__uint_as_float(r[q + 2]), __uint_as_float(r[q + 3])), f2(bb.z, bb.w));
                    s2 = __ffma2_rn(EpiAct2<ACT>::f(h0), f2(ww.x, ww.y), s2);
                    s2 = __ffma2_rn(EpiAct2<ACT>::f(h1), f2(ww.z, ww.w), s2);
                }
            }
            const float s = s2.x + s2.y;
            const int row = ti.row0 + quarter * 32 + lane;
            if (row < ti.t) {
                p.scores[(size_t)ti.head * p.seq.T + row] = s;
                if (p.hist) {
                    if (f32_is_nan(s)) latch_error(p.err, LKV_ERR_NUMERIC, ti.head);
                    atomicAdd(hist_g + (f32_key(s) >> 21), 1u);
                }
            }
        }
        if (p.hist && cur_head >= 0) flush_hist(cur_head);
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::kTmemCols);
    }
    // Launched as the PDL secondary of K2 (lkv_evict): no CTA of this grid may complete before
    // K2 has, so the select kernels behind this one (which wait for this grid) see the budgets
    // and offsets.  K2 is resident before this grid launches (it triggers at its start), so the
    // wait always makes progress.  A no-op for a normal launch.
    pdl_wait();
}

// ============================================================================
// SIMT kernel (fp32 / generic shapes)
// ============================================================================
constexpr int kSimtThreads = 256;
constexpr int kSimtRows = 256;  // rows per tile

template <typename T>
__device__ __forceinline__ float ld_elem(const T* p, size_t i);
template <>
__device__ __forceinline__ float ld_elem<float>(const float* p, size_t i) { return __ldg(p + i); }
template <>
__device__ __forceinline__ float ld_elem<__nv_bfloat16>(const __nv_bfloat16* p, size_t i) {
    return __bfloat162float(p[i]);
}

template <typename T>
__global__ void __launch_bounds__(kSimtThreads) score_simt_kernel(const __grid_constant__ ScoreParams p,
                                                                   int total_tiles) {
    extern __shared__ float w1s[];  // [in][hidden] fp32, then b1[hidden], w2[hidden]
    const int d = p.seq.head_dim;
    const int in = p.in_mode * d;
    const int hid = p.hidden;
    float* b1s = w1s + (size_t)in * hid;
    float* w2s = b1s + hid;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const T* keys = static_cast<const T*>(p.keys);
    const T* values = static_cast<const T*>(p.values);
    const T* w1t = static_cast<const T*>(p.w1t);
    int cur = -1;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const TileInfo ti = decode_tile(p, tile, kSimtRows);
        if (ti.scorer != cur) {
            __syncthreads();
            const T* w = w1t + (size_t)ti.scorer * hid * in;
            for (int e = threadIdx.x; e < in * hid; e += kSimtThreads) {
                const int j = e / in, i = e - j * in;  // source [hidden][in]
                w1s[(size_t)i * hid + j] = ld_elem<T>(w, e);
            }
            for (int j = threadIdx.x; j < hid; j += kSimtThreads) {
                b1s[j] = p.b1[(size_t)ti.scorer * hid + j];
                w2s[j] = p.w2[(size_t)ti.scorer * hid + j];
            }
            cur = ti.scorer;
            __syncthreads();
        }
        const int rows = min(kSimtRows, ti.t - ti.row0);
        for (int rr = warp; rr < rows; rr += kSimtThreads / 32) {
            const size_t base = ((size_t)ti.head * p.seq.T + ti.row0 + rr) * d;
            float acc[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = 0.f;
            for (int i0 = 0; i0 < in; i0 += 32) {
                const int i = i0 + lane;
                float xv = 0.f;
                if (i < in) xv = (i < d) ? ld_elem<T>(keys, base + i) : ld_elem<T>(values, base + (i - d));
                const int lim = min(32, in - i0);
                for (int ii = 0; ii < lim; ++ii) {
                    const float xi = __shfl_sync(0xffffffffu, xv, ii);
                    const float* wr = w1s + (size_t)(i0 + ii) * hid;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int j = lane + 32 * q;
                        if (j < hid) acc[q] = fmaf(xi, wr[j], acc[q]);
                    }
                }
            }
            float s = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int j = lane + 32 * q;
                if (j < hid) s = fmaf(act_f32(p.act, acc[q] + b1s[j]), w2s[j], s);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) p.scores[(size_t)ti.head * p.seq.T + ti.row0 + rr] = s;
        }
    }
}

// ============================================================================
// host launchers
// ============================================================================
static int compute_tiles(ScoreParams& p, int tile_rows) {
    int64_t acc = 0;
    for (int s = 0; s < p.seq.n_seq; ++s) {
        p.tile_base[s] = (int32_t)acc;
        acc += (int64_t)p.seq.n_layers * p.seq.n_kv_heads * ((p.seq.len[s] + tile_rows - 1) / tile_rows);
    }
    p.tile_base[p.seq.n_seq] = (int32_t)acc;
    return (int)acc;
}

cudaError_t launch_score_simt(ScoreParams p, int dtype, int num_sms, cudaStream_t stream) {
    const int tiles = compute_tiles(p, kSimtRows);
    if (tiles == 0) return cudaSuccess;
    const size_t smem = ((size_t)p.in_mode * p.seq.head_dim * p.hidden + 2 * p.hidden) * sizeof(float);
    const int grid = min(tiles, num_sms * 4);
    if (dtype == LKV_F32) {
        cudaError_t e = cudaFuncSetAttribute(score_simt_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        score_simt_kernel<float><<<grid, kSimtThreads, smem, stream>>>(p, tiles);
        note_launches(1);
    } else {
        cudaError_t e = cudaFuncSetAttribute(score_simt_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        score_simt_kernel<__nv_bfloat16><<<grid, kSimtThreads, smem, stream>>>(p, tiles);
        note_launches(1);
    }
    return cudaGetLastError();
}

size_t score_simt_smem_bytes(int in, int hidden) { return ((size_t)in * hidden + 2 * hidden) * sizeof(float); }

template <int N, int NBOX, int ACT>
static cudaError_t launch_tc_inst(const ScoreParams& p, const CUtensorMap& mk, const CUtensorMap& mv,
                                  const CUtensorMap& mw, int tiles, int grid, cudaStream_t stream) {
    using Cfg = TcCfg<N, NBOX>;
    auto kern = score_tc_kernel<N, NBOX, ACT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    if (e != cudaSuccess) return e;
    if (p.pdl)
        e = launch_pdl(kern, dim3(grid), dim3(Cfg::kThreads), Cfg::kSmem, stream, p, mk, mv, mw, tiles);
    else
        kern<<<grid, Cfg::kThreads, Cfg::kSmem, stream>>>(p, mk, mv, mw, tiles);
    if (e != cudaSuccess) return e;
    note_launches(1);
    return cudaGetLastError();
}

bool score_tc_supported(int dtype, int head_dim, int hidden, int in_mode) {
    if (dtype != LKV_BF16 || head_dim != 128) return false;
    if (in_mode == 1) return hidden == 64 || hidden == 128;
    return hidden == 128 || hidden == 64;
}

cudaError_t launch_score_tc(ScoreParams p, const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mw,
                            int num_sms, cudaStream_t stream) {
    const int tiles = compute_tiles(p, kTcRows);
    if (tiles == 0) return cudaSuccess;
    const int grid = min(tiles, num_sms);
    const bool silu = p.act == LKV_ACT_SILU;
    if (p.in_mode == 1) {
        if (p.hidden == 64)
            return silu ? launch_tc_inst<64, 2, LKV_ACT_SILU>(p, mk, mv, mw, tiles, grid, stream)
                        : launch_tc_inst<64, 2, LKV_ACT_GELU_ERF>(p, mk, mv, mw, tiles, grid, stream);
        return silu ? launch_tc_inst<128, 2, LKV_ACT_SILU>(p, mk, mv, mw, tiles, grid, stream)
                    : launch_tc_inst<128, 2, LKV_ACT_GELU_ERF>(p, mk, mv, mw, tiles, grid, stream);
    }
    if (p.hidden == 64)
        return silu ? launch_tc_inst<64, 4, LKV_ACT_SILU>(p, mk, mv, mw, tiles, grid, stream)
                    : launch_tc_inst<64, 4, LKV_ACT_GELU_ERF>(p, mk, mv, mw, tiles, grid, stream);
    return silu ? launch_tc_inst<128, 4, LKV_ACT_SILU>(p, mk, mv, mw, tiles, grid, stream)
                : launch_tc_inst<128, 4, LKV_ACT_GELU_ERF>(p, mk, mv, mw, tiles, grid, stream);
}

}  // namespace lkv_dev
