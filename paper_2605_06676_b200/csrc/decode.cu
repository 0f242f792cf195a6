// decode.cu -- K5: GQA decode attention over the ragged compacted cache.
//
// Reference: decode_step's attention block (model.cpp:240-265): append the new
// (post-RoPE) k, v and position to every KV head, then for every query head qh
// attend over kv = qh / G with n_q = 1, causal = false, no mask, scale 1/sqrt(d)
// (masked_attention_dense, attention.cpp:46-94).  The tiling follows the
// online-softmax form of masked_attention_blocked (attention.cpp:96-143).
//
// B200 design (HBM-bound, 4-8 flop/byte):
//  * work items = (head, ch-row chunk) over each head's capacity, planned once per eviction
//    (decode_plan_kernel, ch in 128..1024 chosen so one launch has enough items for every SM);
//    a persistent grid walks them;
//  * per CTA: one TMA producer warp streams 64-row K+V stages (128-byte
//    swizzle, 32 KB) through a 3-stage mbarrier ring (2 CTAs/SM); four consumer warps each
//    take 16 rows of a stage and run S = Q K^T and O += P V on tensor cores
//    (mma.sync m16n8k16 bf16, ldmatrix from the swizzled tiles), every K/V
//    byte read once for all G query heads of the group;
//  * the chunk containing the appended row patches it into shared memory and
//    writes it (plus its position) into the cache, so no separate append pass;
//  * split-K partials (m, l, o) are merged by decode_combine_kernel, which also
//    advances lens and tokens_seen (heads that fit one chunk are finalised in place).
#include <math.h>

#include "kernels.cuh"

namespace lkv_dev {

constexpr int kDecMaxCh = 1024;  // largest work item (rows); the plan picks 128..1024 per cache
constexpr int kDecStageRows = 64;   // rows per pipeline stage
constexpr int kDecStages = 2;       // x 32 KB per CTA (all-layer launches and G > 4)
constexpr int kDecStagesLayer = 3;  // per-layer launches at G <= 4: the whole one-wave item in flight
constexpr int kDecPerSm = 2;        // resident CTAs per SM
constexpr int kDecConsumers = 4;    // consumer warps (16 rows of a stage each)
constexpr int kDecThreads = (kDecConsumers + 1) * 32;



// ---- plan: work items over each head's capacity (once per eviction) -------------------------
// Heads are enumerated LAYER-major, j -> (l, s, h), head = (s * n_layers + l) * n_kv + h, so the
// items of one layer are contiguous: layer_begin[l] .. layer_begin[l + 1] (a per-layer decode
// launch, as in a full model decode step, walks just that range; an all-layer launch walks
// layer_begin[0] .. layer_begin[n_layers]).
// Work-item size: the largest ch in {1024, 512, 256, 128} that still gives a launch (one plan
// layer) >= target_items items, so a per-layer launch of a small cache still spreads over every
// SM while an all-layer launch keeps long items; ch never leaves G * chunks of a head above
// the combine's table (kCombMaxChunks).
constexpr int kCombMaxChunks = 8192;  // G * chunks per head (G=4: 2M rows, G=8: 1M rows at ch=1024)
constexpr int kPlanMaxLayers = 256;   // layers the one-wave policy tracks
__global__ void __launch_bounds__(1024) decode_plan_kernel(const int64_t* offsets, int n_seq, int n_layers, int n_kv,
                                                           DecodeItem* items, int32_t* item_base,
                                                           int32_t* layer_begin, int32_t* n_items, int32_t* ch_out,
                                                           int target_items, int G, int force_ch) {
    __shared__ uint32_t s_scan[33];
    __shared__ int32_t s_carry;
    __shared__ unsigned long long s_cnt[4];
    __shared__ unsigned long long s_maxcap;
    const int n_heads = n_seq * n_layers * n_kv;
    const int per_layer = n_seq * n_kv;
    if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        s_carry = 0;
        s_maxcap = 0;
    }
    __syncthreads();
    for (int h = threadIdx.x; h < n_heads; h += 1024) {
        const int64_t cap = offsets[h + 1] - offsets[h];
        for (int i = 0; i < 4; ++i) atomicAdd(&s_cnt[i], (unsigned long long)((cap + (128 << i) - 1) >> (7 + i)));
        atomicMax(&s_maxcap, (unsigned long long)cap);
    }
    __syncthreads();
    int ch = 128;
    if (force_ch > 0) {
        ch = force_ch;  // the caller fixes the work-item size (tests; profiling of one shape)
    } else if (target_items < 0 && n_layers <= kPlanMaxLayers) {
        // one-wave policy (per-layer launches, target = -slots): the smallest ch (a multiple of 64)
        // whose busiest layer has no more items than the launch has resident CTAs, so no layer's
        // attention runs a second, mostly idle wave
        __shared__ int32_t s_lay[kPlanMaxLayers];
        __shared__ int32_t s_ok;
        ch = kDecMaxCh;
        for (int c = 128; c <= kDecMaxCh; c += 64) {
            for (int l = threadIdx.x; l < n_layers; l += 1024) s_lay[l] = 0;
            __syncthreads();
            for (int h = threadIdx.x; h < n_heads; h += 1024) {
                const int64_t cap = offsets[h + 1] - offsets[h];
                atomicAdd(&s_lay[(h / n_kv) % n_layers], (int32_t)(cap > 0 ? (cap + c - 1) / c : 1));
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int mx = 0;
                for (int l = 0; l < n_layers; ++l) mx = max(mx, s_lay[l]);
                s_ok = mx <= -target_items;
            }
            __syncthreads();
            if (s_ok) {
                ch = c;
                break;
            }
        }
    } else {
        // the largest ch meeting the target, else the smallest
        const int tgt = target_items < 0 ? -target_items : target_items;
        for (int i = 0; i < 4; ++i)
            if ((long long)s_cnt[i] >= (long long)tgt * n_layers) ch = 128 << i;
    }
    // then grown until the combine fits
    while (ch < kDecMaxCh && (long long)((s_maxcap + ch - 1) / ch) * G > kCombMaxChunks) ch = min(kDecMaxCh, ch * 2);
    if (threadIdx.x == 0) *ch_out = ch;
    for (int base = 0; base < n_heads; base += 1024) {
        const int j = base + threadIdx.x;
        uint32_t nch = 0;
        int h = 0;
        if (j < n_heads) {
            const int l = j / per_layer, r = j - l * per_layer;
            const int s = r / n_kv, kh = r - s * n_kv;
            h = (s * n_layers + l) * n_kv + kh;
            const int64_t cap = offsets[h + 1] - offsets[h];
            nch = (uint32_t)(cap > 0 ? (cap + ch - 1) / ch : 1);  // >= 1: chunk 0 checks every append
        }
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan<1024>(nch, s_scan, &tot);
        if (j < n_heads) {
            const int b0 = s_carry + (int)ex;
            item_base[h] = b0;
            if (j % per_layer == 0) layer_begin[j / per_layer] = b0;
            for (uint32_t c = 0; c < nch; ++c) items[b0 + c] = DecodeItem{h, (int32_t)c};
        }
        __syncthreads();
        if (threadIdx.x == 0) s_carry += (int32_t)tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        layer_begin[n_layers] = s_carry;
        *n_items = s_carry;
    }
}

// (s, l, kv head) of a flat head, and the row of the q / out / new_k tensors of this launch,
// which hold the q_layers layers starting at layer0: qsl = s * q_layers + (l - layer0).
struct HeadCoord {
    int s, l, kvh, qsl;
};
__device__ __forceinline__ HeadCoord head_coord(const DecodeParams& p, int head) {
    HeadCoord c;
    const int sl = head / p.n_kv_heads;
    c.kvh = head - sl * p.n_kv_heads;
    c.s = sl / p.n_layers;
    c.l = sl - c.s * p.n_layers;
    c.qsl = c.s * p.q_layers + (c.l - p.layer0);
    return c;
}
// element (g, dd) of a head's G x D output block -> index into out.  Plain: [qsl][Hq][D].
// Packed (out_nbt > 0, q_layers == 1): the mma B-fragment layout the weight-streaming GEMV
// reads (model.cu act_index), with batch = s and feature = (kvh * G + g) * D + dd.
__device__ __forceinline__ size_t out_index(const DecodeParams& p, const HeadCoord& c, int g, int dd) {
    const int D = p.head_dim;
    if (p.out_nbt == 0) return ((size_t)c.qsl * p.n_q_heads + c.kvh * p.G + g) * D + dd;
    return act_index(c.s, (c.kvh * p.G + g) * D + dd, p.out_nbt);
}

// ---- helpers ---------------------------------------------------------------------------------
__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                                  uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// D = A B + C over an m16n8k16 tile; with HI == false the A rows 8..15 are zero and the
// rows-8..15 half of C/D is dead, so it is fed zeros and discarded (no live registers).
template <bool HI>
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    if constexpr (HI) {
        mma_bf16_16816(d, a, b0, b1);
    } else {
        float x2, x3;
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%10,%11,%12,%13};"
            : "=f"(d[0]), "=f"(d[1]), "=f"(x2), "=f"(x3)
            : "r"(a[0]), "r"(0u), "r"(a[2]), "r"(0u), "r"(b0), "r"(b1), "f"(d[0]), "f"(d[1]), "f"(0.f), "f"(0.f));
        d[2] = 0.f;
        d[3] = 0.f;
    }
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

// byte offset of (row, 16-byte chunk q in 0..15) inside a stage tile stored as two
// 64-row x 128-byte boxes with the TMA 128-byte swizzle
__device__ __forceinline__ uint32_t sw_off(int row, int q) {
    return (uint32_t)((q >> 3) * (kDecStageRows * 128) + row * 128 + (((q & 7) ^ (row & 7)) << 4));
}

// ---- bf16 attention kernel (tensor cores) ------------------------------------------------------
// HI: the group has more than 8 query heads, so rows 8..15 of the m16 fragments are live.
// For G <= 8 those rows are zero padding: their accumulators are never kept in registers.
template <bool HI, int ST>
__global__ void __launch_bounds__(kDecThreads, kDecPerSm)
    decode_attn_bf16_kernel(const __grid_constant__ DecodeParams p, const __grid_constant__ CUtensorMap tmap_k,
                            const __grid_constant__ CUtensorMap tmap_v) {
    constexpr int kStageBytes = 2 * kDecStageRows * 256;  // K + V, 64 rows x 256 B each
    extern __shared__ unsigned char smem_dyn[];
    unsigned char* smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);  // aligned, still a __shared__ pointer
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * kStageBytes);
    uint64_t* empty = full + ST;
    float* red = reinterpret_cast<float*>(empty + ST);  // [consumers][G][D + 2]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = p.G;
    const int D = 128;
    pdl_trigger();  // the combine's CTAs may become resident (they wait for this grid to finish)
    // q / new k / new v come from the previous kernel.  With early_kv the producer streams the
    // cached rows (written by earlier steps) while that kernel is still running; only the
    // consumers wait.
    if (!p.early_kv) pdl_wait();
    const int it_lo = *p.item_lo, it_hi = *p.item_hi;
    const int ch = *p.ch;
    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kDecConsumers);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kDecConsumers) {
        // ===================== producer =====================
        if (lane == 0) {
            tma_prefetch_desc(&tmap_k);
            tma_prefetch_desc(&tmap_v);
            const uint64_t pol = l2_policy_evict_first();
            int st = 0;
            uint32_t ph = 0;
            for (int it = it_lo + blockIdx.x; it < it_hi; it += gridDim.x) {
                const DecodeItem wi = p.items[it];
                const int len_new = p.lens[wi.head] + 1;
                const int r0 = wi.chunk * ch;
                if (r0 >= len_new) continue;
                const int rows = min(ch, len_new - r0);
                const int64_t grow0 = p.offsets[wi.head] + r0;
                for (int sr = 0; sr < rows; sr += kDecStageRows) {
                    mbar_wait(&empty[st], ph ^ 1);
                    mbar_arrive_expect_tx(&full[st], kStageBytes);
                    unsigned char* dst = smem + st * kStageBytes;
                    const int y = (int)(grow0 + sr);
                    tma_load_2d(dst, &tmap_k, &full[st], 0, y, pol);
                    tma_load_2d(dst + kDecStageRows * 128, &tmap_k, &full[st], 64, y, pol);
                    tma_load_2d(dst + 2 * kDecStageRows * 128, &tmap_v, &full[st], 0, y, pol);
                    tma_load_2d(dst + 3 * kDecStageRows * 128, &tmap_v, &full[st], 64, y, pol);
                    if (++st == ST) {
                        st = 0;
                        ph ^= 1;
                    }
                }
            }
        }
        return;
    }

    // ===================== consumers =====================
    if (p.early_kv) pdl_wait();
    const int g = lane >> 2;       // fragment row (query head within the group)
    const int cq = (lane & 3) * 2;  // fragment column pair
    int st = 0;
    uint32_t ph = 0;
    for (int it = it_lo + blockIdx.x; it < it_hi; it += gridDim.x) {
        const DecodeItem wi = p.items[it];
        const int head = wi.head;
        const int len_old = p.lens[head];
        const int len_new = len_old + 1;
        const int r0 = wi.chunk * ch;
        if (wi.chunk == 0 && threadIdx.x == 0) p.new_len[head] = len_new;  // for the combine (never reads lens)
        if (r0 >= len_new) continue;
        const int rows = min(ch, len_new - r0);
        const int64_t off = p.offsets[head];
        const bool has_new = (len_old >= r0) && (len_old < r0 + ch);
        const bool fits = off + len_new <= p.offsets[head + 1];
        if (has_new && !fits) {
            if (threadIdx.x == 0) latch_error(p.err, LKV_ERR_CONTRACT, head);
        }
        const __nv_bfloat16* qp;
        {
            const HeadCoord hc = head_coord(p, head);
            qp = static_cast<const __nv_bfloat16*>(p.q) + ((size_t)hc.qsl * p.n_q_heads + hc.kvh * G) * D;
        }

        // Q fragments (rows g and g+8 of the padded 16-row tile)
        uint32_t qa[8][4];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const int c0 = kk * 16 + cq;
            const uint32_t* r_lo = reinterpret_cast<const uint32_t*>(qp + (size_t)g * D);
            const uint32_t* r_hi = reinterpret_cast<const uint32_t*>(qp + (size_t)(g + 8) * D);
            qa[kk][0] = g < G ? __ldg(r_lo + (c0 >> 1)) : 0u;
            qa[kk][1] = (HI && g + 8 < G) ? __ldg(r_hi + (c0 >> 1)) : 0u;
            qa[kk][2] = g < G ? __ldg(r_lo + ((c0 + 8) >> 1)) : 0u;
            qa[kk][3] = (HI && g + 8 < G) ? __ldg(r_hi + ((c0 + 8) >> 1)) : 0u;
        }
        float o[16][4];
#pragma unroll
        for (int n = 0; n < 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
        float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;

        for (int sr = 0; sr < rows; sr += kDecStageRows) {
            mbar_wait(&full[st], ph);
            unsigned char* sbase = smem + st * kStageBytes;
            const uint32_t kbase = smem_u32(sbase);
            const uint32_t vbase = kbase + 2 * kDecStageRows * 128;
            const int wr0 = warp * 16;  // this warp's 16 rows inside the stage
            // patch the appended row (it is not in the cache yet)
            if (has_new) {
                const int nr = len_old - r0 - sr;  // row inside this stage
                if (nr >= wr0 && nr < wr0 + 16) {
                    const int hq = lane & 15;
                    const bool isv = lane >= 16;
                    const HeadCoord hc = head_coord(p, head);
                    const uint4* src =
                        static_cast<const uint4*>(isv ? p.new_v : p.new_k) + ((size_t)hc.qsl * p.n_kv_heads + hc.kvh) * 16;
                    const uint4 v = __ldg(src + hq);
                    *reinterpret_cast<uint4*>(sbase + (isv ? 2 * kDecStageRows * 128 : 0) + sw_off(nr, hq)) = v;
                    if (fits) {  // never write past the head's capacity (the error is latched above)
                        uint4* dstg = static_cast<uint4*>(isv ? p.values : p.keys) + (size_t)(off + len_old) * 16;
                        dstg[hq] = v;
                        if (lane == 0) p.positions[off + len_old] = p.tokens_seen[hc.s];
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                }
            }
            const int valid = min(kDecStageRows, rows - sr) - wr0;  // rows of this warp that exist
            if (valid > 0 && valid < 16) {
                // rows past the chunk end hold other heads' data or never-written slack:
                // zero their V so P = 0 cannot meet a NaN/Inf pattern in the MMA
                for (int e = lane; e < (16 - valid) * 16; e += 32) {
                    const int row = wr0 + valid + (e >> 4);
                    *reinterpret_cast<uint4*>(sbase + 2 * kDecStageRows * 128 + sw_off(row, e & 15)) =
                        make_uint4(0u, 0u, 0u, 0u);
                }
                fence_proxy_async_smem();
                __syncwarp();
            }
            if (valid > 0) {
                // ---- S = Q K^T for 16 rows (two n8 tiles)
                float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int j = lane >> 3;
                    const int row = wr0 + ((j >> 1) << 3) + (lane & 7);
                    const int q = kk * 2 + (j & 1);
                    uint32_t b0, b1, b2, b3;
                    ldmatrix_x4(kbase + sw_off(row, q), b0, b1, b2, b3);
                    mma16816<HI>(s0, qa[kk], b0, b1);
                    mma16816<HI>(s1, qa[kk], b2, b3);
                }
                // ---- mask, online softmax (log2 domain)
                float sv[8] = {s0[0], s0[1], s1[0], s1[1], s0[2], s0[3], s1[2], s1[3]};
                if constexpr (!HI) sv[4] = sv[5] = sv[6] = sv[7] = -INFINITY;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int col = ((e & 2) ? 8 : 0) + cq + (e & 1);
                    sv[e] = col < valid ? sv[e] * p.scale_log2 : -INFINITY;
                }
                float mx_lo = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
                float mx_hi = fmaxf(fmaxf(sv[4], sv[5]), fmaxf(sv[6], sv[7]));
                mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 1));
                mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 2));
                mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 1));
                mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 2));
                const float mn_lo = fmaxf(m_lo, mx_lo), mn_hi = fmaxf(m_hi, mx_hi);
                const float a_lo = (mn_lo == -INFINITY) ? 1.f : exp2f(m_lo - mn_lo);
                const float a_hi = (mn_hi == -INFINITY) ? 1.f : exp2f(m_hi - mn_hi);
                m_lo = mn_lo;
                m_hi = mn_hi;
                float pv[8];
#pragma unroll
                for (int e = 0; e < 4; ++e) pv[e] = (mn_lo == -INFINITY) ? 0.f : exp2f(sv[e] - mn_lo);
#pragma unroll
                for (int e = 4; e < 8; ++e) pv[e] = (mn_hi == -INFINITY) ? 0.f : exp2f(sv[e] - mn_hi);
                l_lo = l_lo * a_lo + (pv[0] + pv[1] + pv[2] + pv[3]);
                l_hi = l_hi * a_hi + (pv[4] + pv[5] + pv[6] + pv[7]);
#pragma unroll
                for (int n = 0; n < 16; ++n) {
                    o[n][0] *= a_lo;
                    o[n][1] *= a_lo;
                    if constexpr (HI) {
                        o[n][2] *= a_hi;
                        o[n][3] *= a_hi;
                    }
                }
                // P as the A operand (k = the 16 rows)
                uint32_t pa[4];
                pa[0] = pack_bf16(pv[0], pv[1]);  // row g,   cols cq..   (rows 0-7)
                pa[1] = pack_bf16(pv[4], pv[5]);  // row g+8, cols cq..
                pa[2] = pack_bf16(pv[2], pv[3]);  // row g,   cols 8+cq.. (rows 8-15)
                pa[3] = pack_bf16(pv[6], pv[7]);  // row g+8, cols 8+cq..
                // ---- O += P V
#pragma unroll
                for (int n2 = 0; n2 < 8; ++n2) {
                    const int j = lane >> 3;
                    const int row = wr0 + ((j & 1) << 3) + (lane & 7);
                    const int q = n2 * 2 + (j >> 1);
                    uint32_t b0, b1, b2, b3;
                    ldmatrix_x4_trans(vbase + sw_off(row, q), b0, b1, b2, b3);
                    mma16816<HI>(o[2 * n2], pa, b0, b1);
                    mma16816<HI>(o[2 * n2 + 1], pa, b2, b3);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (++st == ST) {
                st = 0;
                ph ^= 1;
            }
        }
        // ---- merge the 4 consumer warps (rows g < G live in the lo half; g+8 in the hi half)
        l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
        l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
        l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
        l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);
        const int stride = D + 2;
        float* rw = red + (size_t)warp * G * stride;
        if (g < G) {
#pragma unroll
            for (int n = 0; n < 16; ++n) {
                rw[g * stride + n * 8 + cq] = o[n][0];
                rw[g * stride + n * 8 + cq + 1] = o[n][1];
            }
            if ((lane & 3) == 0) {
                rw[g * stride + D] = m_lo;
                rw[g * stride + D + 1] = l_lo;
            }
        }
        if (HI && g + 8 < G) {
#pragma unroll
            for (int n = 0; n < 16; ++n) {
                rw[(g + 8) * stride + n * 8 + cq] = o[n][2];
                rw[(g + 8) * stride + n * 8 + cq + 1] = o[n][3];
            }
            if ((lane & 3) == 0) {
                rw[(g + 8) * stride + D] = m_hi;
                rw[(g + 8) * stride + D + 1] = l_hi;
            }
        }
        named_bar_sync(1, kDecConsumers * 32);
        const int nch = (len_new + ch - 1) / ch;
        __nv_bfloat16* outp = static_cast<__nv_bfloat16*>(p.out);
        const HeadCoord hc = head_coord(p, head);
        for (int e = threadIdx.x; e < G * D; e += kDecConsumers * 32) {
            const int gg = e / D, dd = e - gg * D;
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < kDecConsumers; ++w) M = fmaxf(M, red[((size_t)w * G + gg) * stride + D]);
            float L = 0.f, acc = 0.f;
#pragma unroll
            for (int w = 0; w < kDecConsumers; ++w) {
                const float* r = red + ((size_t)w * G + gg) * stride;
                const float f = (r[D] == -INFINITY) ? 0.f : exp2f(r[D] - M);
                L += r[D + 1] * f;
                acc += r[dd] * f;
            }
            if (nch == 1) {
                outp[out_index(p, hc, gg, dd)] = __float2bfloat16_rn(acc / L);
            } else {
                p.part_o[((size_t)it * G + gg) * D + dd] = acc;
                if (dd == 0) {
                    p.part_m[(size_t)it * G + gg] = M;
                    p.part_l[(size_t)it * G + gg] = L;
                }
            }
        }
        named_bar_sync(1, kDecConsumers * 32);
    }
}

// ---- fp32 attention kernel (SIMT; correctness configs) --------------------------------------------
constexpr int kDecSimtThreads = 128;

__global__ void __launch_bounds__(kDecSimtThreads) decode_attn_f32_kernel(const __grid_constant__ DecodeParams p) {
    extern __shared__ float sm[];
    const int D = p.head_dim, G = p.G;
    float* qs = sm;                 // [G][D]
    const int ch = *p.ch;
    float* sc = qs + G * D;         // [G][ch]
    const int it = *p.item_lo + blockIdx.x;
    if (it >= *p.item_hi) return;
    const DecodeItem wi = p.items[it];
    const int head = wi.head;
    const int len_old = p.lens[head];
    const int len_new = len_old + 1;
    const int r0 = wi.chunk * ch;
    if (wi.chunk == 0 && threadIdx.x == 0) p.new_len[head] = len_new;  // for the combine
    if (r0 >= len_new) return;
    const int rows = min(ch, len_new - r0);
    const int64_t off = p.offsets[head];
    const bool has_new = len_old >= r0 && len_old < r0 + ch;
    if (has_new && off + len_new > p.offsets[head + 1]) {
        if (threadIdx.x == 0) latch_error(p.err, LKV_ERR_CONTRACT, head);
        return;
    }
    const HeadCoord hc = head_coord(p, head);
    const float* qp = static_cast<const float*>(p.q) + ((size_t)hc.qsl * p.n_q_heads + hc.kvh * G) * D;
    for (int e = threadIdx.x; e < G * D; e += kDecSimtThreads) qs[e] = qp[e];
    float* K = static_cast<float*>(p.keys) + (size_t)off * D;
    float* V = static_cast<float*>(p.values) + (size_t)off * D;
    const float* nk = static_cast<const float*>(p.new_k) + ((size_t)hc.qsl * p.n_kv_heads + hc.kvh) * D;
    const float* nv = static_cast<const float*>(p.new_v) + ((size_t)hc.qsl * p.n_kv_heads + hc.kvh) * D;
    if (has_new) {
        for (int e = threadIdx.x; e < D; e += kDecSimtThreads) {
            K[(size_t)len_old * D + e] = nk[e];
            V[(size_t)len_old * D + e] = nv[e];
        }
        if (threadIdx.x == 0) p.positions[off + len_old] = p.tokens_seen[hc.s];
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = warp; r < rows; r += kDecSimtThreads / 32) {
        const int row = r0 + r;
        const float* kr = (row == len_old) ? nk : K + (size_t)row * D;
        for (int gg = 0; gg < G; ++gg) {
            float acc = 0.f;
            for (int c = lane; c < D; c += 32) acc = fmaf(qs[gg * D + c], kr[c], acc);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) sc[gg * ch + r] = acc * p.scale_log2;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < G * D; e += kDecSimtThreads) {
        const int gg = e / D, dd = e - gg * D;
        float M = -INFINITY;
        for (int r = 0; r < rows; ++r) M = fmaxf(M, sc[gg * ch + r]);
        float L = 0.f, acc = 0.f;
        for (int r = 0; r < rows; ++r) {
            const float w = exp2f(sc[gg * ch + r] - M);
            const int row = r0 + r;
            const float v = (row == len_old) ? nv[dd] : V[(size_t)row * D + dd];
            L += w;
            acc = fmaf(w, v, acc);
        }
        p.part_o[((size_t)it * G + gg) * D + dd] = acc;
        if (dd == 0) {
            p.part_m[(size_t)it * G + gg] = M;
            p.part_l[(size_t)it * G + gg] = L;
        }
    }
}

// ---- combine split-K partials; advance lens and tokens_seen ------------------------------------------
// One CTA per (head, 128 outputs).  Phase 1 turns the chunk maxima / sums into per-chunk weights in
// shared memory; phase 2 streams the partial outputs with independent (unrolled) loads, the
// chunks split over kCombSlices thread slices (a head's chunk count follows its budget, so a
// long head would otherwise set the kernel's latency) and the slices summed in fixed order.
// Heads that fit one chunk were finalised by the attention kernel (bf16 path).
constexpr int kCombCols = 128;    // outputs per CTA

template <typename T, int kCombSlices>  // chunk slices per output: 4 for a few heads, else 1
__global__ void __launch_bounds__(kCombCols * kCombSlices) decode_combine_kernel(const __grid_constant__ DecodeParams p,
                                                                                int single_chunk_done) {
    constexpr int kCombThreads = kCombCols * kCombSlices;
    pdl_trigger();  // the next GEMV may start streaming its weights
    __shared__ float s_w[kCombMaxChunks];  // [c * G + g] weight exp2(m_c - M_g) / L_g
    // blockIdx.x enumerates this launch's heads layer-major (as the plan does)
    const int per_layer = p.n_seq * p.n_kv_heads;
    const int jl = blockIdx.x / per_layer, jr = blockIdx.x - jl * per_layer;
    const int js = jr / p.n_kv_heads;
    const int head = (js * p.n_layers + p.layer0 + jl) * p.n_kv_heads + (jr - js * p.n_kv_heads);
    const int D = p.head_dim, G = p.G;
    const int ch = *p.ch;                  // the plan's (written before the step)
    const int base = p.item_base[head];
    // the length the attention kernel saw.  lens_deferred: lens is not written during the step, so
    // it is read before the wait.  Otherwise lens[head] is advanced below by the y = 0 CTA while
    // other CTAs of the head may not have started, so the attention kernel's copy is read.
    int len_new = p.lens_deferred ? p.lens[head] + 1 : 0;
    pdl_wait();
    if (!p.lens_deferred) len_new = p.new_len[head];
    const int nch = (len_new + ch - 1) / ch;
    if (!(single_chunk_done && nch == 1) && nch * G <= kCombMaxChunks) {
        const float* pm = p.part_m + (size_t)base * G;
        const float* pl = p.part_l + (size_t)base * G;
        const float* po = p.part_o + (size_t)base * G * D;
        static_assert(kCombSlices == 1 || kCombSlices == 4, "combine slices");
        constexpr int S = kCombSlices;
        const int col = threadIdx.x % kCombCols, sl = threadIdx.x / kCombCols;
        const int e = blockIdx.y * kCombCols + col;
        // per-layer launches (S = 4, a few heads): the first block of this thread's partial outputs
        // is requested now, together with phase 1's maxima and sums (one memory round trip fewer on
        // the step's critical path); all-layer launches keep their registers for occupancy
        float v[16];
        auto load_block = [&](int c) {
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (c + k * S < nch) v[k] = po[(size_t)(c + k * S) * G * D + e];
        };
        if constexpr (S == 4)
            if (e < G * D) load_block(sl);
        // weights: one warp per query head g reads its (chunk) maxima and sums straight from the
        // partials (lanes stride over chunks), reduces M and L by the xor tree, and writes
        // exp2(m_c - M) / L for its chunks -- one CTA barrier before the weighted sums
        {
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
            for (int g = warp; g < G; g += kCombThreads / 32) {
                float m0 = -INFINITY, l0 = 0.f;  // this lane's first chunk (nch <= 32: the only one)
                if (lane < nch) {
                    m0 = pm[lane * G + g];
                    l0 = pl[lane * G + g];
                }
                float M = m0;
                for (int c = lane + 32; c < nch; c += 32) M = fmaxf(M, pm[c * G + g]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
                float L = 0.f;
                if (lane < nch) L += l0 * exp2f(m0 - M);
                for (int c = lane + 32; c < nch; c += 32) L += pl[c * G + g] * exp2f(pm[c * G + g] - M);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
                if (lane < nch) s_w[lane * G + g] = exp2f(m0 - M) / L;
                for (int c = lane + 32; c < nch; c += 32) s_w[c * G + g] = exp2f(pm[c * G + g] - M) / L;
            }
        }
        __syncthreads();
        const HeadCoord hc = head_coord(p, head);
        T* out = static_cast<T*>(p.out);
        // grid.y tiles the G*D outputs.  Chunk c is summed into partial c % 4 and the four partials
        // are added in order, whether one thread holds all four (kCombSlices = 1) or slice sl of
        // the threads holds partial sl (kCombSlices = 4): the result does not depend on the launch
        // shape.  A thread's 16 chunk loads of a block are in flight together (the first block's
        // since before phase 1).
        __shared__ float s_part[S][kCombCols];
        const int g = min(e, G * D - 1) / D;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        if (e < G * D) {
            int c = sl;
            if constexpr (S != 4) load_block(c);
            for (;;) {
                const bool whole = c + 15 * S < nch;
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    if (whole || c + k * S < nch) {
                        float& a = acc[S == 4 ? 0 : (k & 3)];
                        a = fmaf(v[k], s_w[(c + k * S) * G + g], a);
                    }
                if (!whole) break;
                c += 16 * S;
                if (c >= nch) break;
                load_block(c);
            }
        }
        float sum;
        if constexpr (S == 4) {
            s_part[sl][col] = acc[0];
            __syncthreads();
            sum = ((s_part[0][col] + s_part[1][col]) + s_part[2][col]) + s_part[3][col];
        } else {
            sum = ((acc[0] + acc[1]) + acc[2]) + acc[3];
        }
        if (sl == 0 && e < G * D) {
            const size_t oi = out_index(p, hc, g, e - g * D);
            if constexpr (sizeof(T) == 2) out[oi] = __float2bfloat16_rn(sum);
            else out[oi] = sum;
        }
    } else if (nch * G > kCombMaxChunks && threadIdx.x == 0 && blockIdx.y == 0) {
        latch_error(p.err, LKV_ERR_UNSUPPORTED, head);
    }
    if (!p.lens_deferred && threadIdx.x == 0 && blockIdx.y == 0) {
        p.lens[head] = len_new;
        // tokens_seen advances once per step, after the last layer's append (the position of
        // every layer's new row is the step's starting tokens_seen, model.cpp:218,246)
        const HeadCoord hc = head_coord(p, head);
        if (hc.l == p.n_layers - 1 && hc.kvh == 0) p.tokens_seen[hc.s] += 1;
    }
}

// ---- host launchers ---------------------------------------------------------------------------------
cudaError_t launch_decode_plan(const int64_t* offsets, int n_seq, int n_layers, int n_kv, DecodeItem* items,
                               int32_t* item_base, int32_t* layer_begin, int32_t* n_items, int32_t* ch,
                               int target_items, int G, int force_ch, cudaStream_t stream) {
    decode_plan_kernel<<<1, 1024, 0, stream>>>(offsets, n_seq, n_layers, n_kv, items, item_base, layer_begin,
                                               n_items, ch, target_items, G, force_ch);
    note_launches(1);
    return cudaGetLastError();
}

size_t decode_bf16_smem(int G, int stages) {
    return 1024 + stages * (2 * kDecStageRows * 256) + 2 * stages * 8 + (size_t)kDecConsumers * G * (128 + 2) * 4;
}
// a per-layer launch (the model step) of a G <= 4 group keeps its whole one-wave work item in
// flight (3 stages, still 2 CTAs per SM); all-layer launches stream long items through 2 stages
static int decode_stages(int q_layers, int G) { return (q_layers == 1 && G <= 4) ? kDecStagesLayer : kDecStages; }
static void (*decode_bf16_kern(int G, int stages))(DecodeParams, CUtensorMap, CUtensorMap) {
    if (G > 8) return decode_attn_bf16_kernel<true, kDecStages>;
    return stages == kDecStagesLayer ? decode_attn_bf16_kernel<false, kDecStagesLayer>
                                     : decode_attn_bf16_kernel<false, kDecStages>;
}

// resident CTAs of one bf16 decode launch (its persistent grid size): the one-wave plan target
int decode_resident_ctas(int G, int num_sms) {  // of a per-layer launch (the model step's plan)
    const int stages = decode_stages(1, G);
    auto kern = decode_bf16_kern(G, stages);
    const size_t smem = decode_bf16_smem(G, stages);
    int per_sm = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDecThreads, smem) != cudaSuccess)
        per_sm = 1;
    return max(1, min(per_sm, kDecPerSm)) * num_sms;
}

cudaError_t launch_decode(const DecodeParams& p, int dtype, const CUtensorMap* mk, const CUtensorMap* mv, int num_sms,
                          cudaStream_t stream) {
    if (p.max_items == 0) return cudaSuccess;
    if (dtype == LKV_BF16) {
        const int stages = decode_stages(p.q_layers, p.G);
        const size_t smem = decode_bf16_smem(p.G, stages);
        auto kern = decode_bf16_kern(p.G, stages);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDecThreads, smem);
        if (e != cudaSuccess) return e;
        per_sm = max(1, min(per_sm, kDecPerSm));
        const int grid = min(p.max_items, per_sm * num_sms);
        e = launch_pdl(kern, dim3(grid), dim3(kDecThreads), smem, stream, p, *mk, *mv);
        if (e != cudaSuccess) return e;
        const dim3 cgrid(p.n_seq * p.q_layers * p.n_kv_heads, (p.G * p.head_dim + kCombCols - 1) / kCombCols);
        // few heads (a per-layer launch): split each head's chunks over 4 thread slices
        if (cgrid.x * cgrid.y < (unsigned)num_sms)
            e = launch_pdl(decode_combine_kernel<__nv_bfloat16, 4>, cgrid, dim3(kCombCols * 4), 0, stream, p, 1);
        else
            e = launch_pdl(decode_combine_kernel<__nv_bfloat16, 1>, cgrid, dim3(kCombCols), 0, stream, p, 1);
        if (e != cudaSuccess) return e;
        note_launches(2);
    } else {
        const size_t smem = ((size_t)p.G * p.head_dim + (size_t)p.G * kDecMaxCh) * sizeof(float);
        cudaError_t e = cudaFuncSetAttribute(decode_attn_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        decode_attn_f32_kernel<<<p.max_items, kDecSimtThreads, smem, stream>>>(p);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        decode_combine_kernel<float, 1><<<dim3(p.n_seq * p.q_layers * p.n_kv_heads, (p.G * p.head_dim + kCombCols - 1) / kCombCols), kCombCols, 0, stream>>>(p, 0);
        note_launches(2);
    }
    return cudaGetLastError();
}

}  // namespace lkv_dev
