// kvproj.cu -- K/V production for layer-by-layer prefill on tcgen05.
//
// The reference computes a layer's K and V as h Wk, h Wv, rotates K at absolute positions and
// splits the heads before scoring (evictsim.cpp:133-145, model.cpp:38-46, tensor.cpp:586-623).
// Here that is ONE persistent GEMM over the concatenated weights [Wk | Wv]:
//
//   C[tokens x 2HD] = h[tokens x d_model] * Wkv[d_model x 2HD]     (bf16 in, fp32 accumulate)
//
// with RoPE and the token-major -> head-major pack fused into the epilogue: each accumulator
// tile is read from TMEM once, K columns are rotated pairwise with the fp64-built cos/sin table,
// and the bf16 rows go straight into the dense layer [n_seq][H][T][D] that the scorer's TMA map
// and the gather read -- no token-major K/V round trip through HBM.
//
// Warp roles (persistent, one CTA per SM): warp 0 = TMA producer (A 128x64 and B 256x64 boxes,
// 128-byte swizzle, 4-stage ring), warp 1 = single-thread UMMA issuer (tcgen05.mma kind::f16,
// M=128 N=256 K=16), warps 2-5 = epilogue (one TMEM lane quarter each), two TMEM accumulators
// (2 x 256 columns) so the epilogue of tile i overlaps the MMAs of tile i+1.
#include "kernels.cuh"

namespace lkv_dev {

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}

constexpr int kPM = 128;     // UMMA M (token rows per tile)
constexpr int kPN = 256;     // UMMA N (output columns per tile: two heads of K or V)
constexpr int kPK = 64;      // K per stage (one 128-byte swizzle box of bf16)
constexpr int kPStages = 4;
constexpr int kPThreads = 192;
constexpr int kPABytes = kPM * kPK * 2;  // 16 KB
constexpr int kPBBytes = kPN * kPK * 2;  // 32 KB
constexpr int kPStageBytes = kPABytes + kPBBytes;
constexpr size_t kPSmem = (size_t)kPStages * kPStageBytes + 256 + 1024;

__global__ void __launch_bounds__(kPThreads, 1)
    kv_project_kernel(const __grid_constant__ KvProjParams p, const __grid_constant__ CUtensorMap tmap_a,
                      const __grid_constant__ CUtensorMap tmap_b) {
    extern __shared__ unsigned char smem_dyn[];
    unsigned char* smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kPStages * kPStageBytes);
    uint64_t* full = bars;                   // [kPStages]
    uint64_t* empty = bars + kPStages;       // [kPStages]
    uint64_t* tfull = bars + 2 * kPStages;   // [2]
    uint64_t* tempty = tfull + 2;            // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_tiles_n = p.N / kPN;
    const int n_tiles = ((p.M + kPM - 1) / kPM) * n_tiles_n;
    const int k_steps = p.K / kPK;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kPStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_b);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint64_t pol_a = l2_policy_evict_first();  // each A block is read by n_tiles_n CTAs in a row
            const uint64_t pol_b = l2_policy_evict_last();   // the weights: every tile reads them
            int it = 0;
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                const int m0 = (tile / n_tiles_n) * kPM, n0 = (tile % n_tiles_n) * kPN;
                for (int kb = 0; kb < k_steps; ++kb, ++it) {
                    const int st = it % kPStages;
                    mbar_wait_backoff(&empty[st], ((it / kPStages) & 1) ^ 1);
                    mbar_arrive_expect_tx(&full[st], kPStageBytes);
                    unsigned char* dst = smem + st * kPStageBytes;
                    tma_load_2d(dst, &tmap_a, &full[st], kb * kPK, m0, pol_a);
                    tma_load_2d(dst + kPABytes, &tmap_b, &full[st], kb * kPK, n0, pol_b);
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(kPM, kPN);
            const uint32_t base = smem_u32(smem);
            int it = 0, ti = 0;
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++ti) {
                const int acc = ti & 1;
                mbar_wait_backoff(&tempty[acc], ((ti >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * kPN;
                for (int kb = 0; kb < k_steps; ++kb, ++it) {
                    const int st = it % kPStages;
                    mbar_wait(&full[st], (it / kPStages) & 1);
                    tc_fence_after();
                    const uint32_t a_st = base + st * kPStageBytes, b_st = a_st + kPABytes;
#pragma unroll
                    for (int kk = 0; kk < kPK / 16; ++kk)
                        umma_bf16(d_tmem, umma_desc_sw128(a_st + kk * 32), umma_desc_sw128(b_st + kk * 32), idesc,
                                  (kb | kk) ? 1u : 0u);
                    umma_commit(&empty[st]);  // the stage is free once these MMAs retire
                }
                umma_commit(&tfull[acc]);
            }
        }
    } else {
        // ===================== epilogue: RoPE + head-major pack =====================
        const int quarter = warp & 3;  // the TMEM lane quarter this warp may read
        const int HD = p.H * p.D;
        int ti = 0;
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++ti) {
            const int acc = ti & 1;
            const int m0 = (tile / n_tiles_n) * kPM, n0 = (tile % n_tiles_n) * kPN;
            mbar_wait(&tfull[acc], (ti >> 1) & 1);
            __syncwarp();
            tc_fence_after();
            const int row = m0 + quarter * 32 + lane;  // token row of this thread
            const bool live = row < p.M;
            const int s = live ? row / p.T : 0, pos = live ? row - s * p.T : 0;
            const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + acc * kPN;
#pragma unroll 1
            for (int c = 0; c < kPN / 32; ++c) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(taddr + c * 32, r);
                tmem_ld_wait();
                if (c == kPN / 32 - 1) {  // accumulator drained: the MMA may reuse it
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                }
                const int gc = n0 + c * 32;  // first output column of this chunk
                const bool is_k = gc < HD;
                const int hc = is_k ? gc : gc - HD;
                const int h = hc / p.D, d0 = hc - h * p.D;
                float v[32];
#pragma unroll
                for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(r[q]);
                if (is_k) {  // rotary pairs (2j, 2j+1) at the row's absolute position
                    const float4* cs = reinterpret_cast<const float4*>(p.table + (size_t)pos * (p.D / 2) + d0 / 2);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float4 t2 = __ldg(cs + q);  // (cos, sin) of two consecutive pairs
                        const float a0 = v[4 * q], b0 = v[4 * q + 1], a1 = v[4 * q + 2], b1 = v[4 * q + 3];
                        v[4 * q] = a0 * t2.x - b0 * t2.y;
                        v[4 * q + 1] = a0 * t2.y + b0 * t2.x;
                        v[4 * q + 2] = a1 * t2.z - b1 * t2.w;
                        v[4 * q + 3] = a1 * t2.w + b1 * t2.z;
                    }
                }
                if (live) {
                    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(is_k ? p.k_out : p.v_out) +
                                         (((size_t)s * p.H + h) * p.T + pos) * p.D + d0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint4 w;
                        w.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
                        w.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
                        w.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
                        w.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
                        reinterpret_cast<uint4*>(out)[q] = w;
                    }
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

size_t kv_project_smem() { return kPSmem; }

cudaError_t launch_kv_project(const KvProjParams& p, const CUtensorMap& ma, const CUtensorMap& mb, int num_sms,
                              cudaStream_t stream) {
    const int tiles = ((p.M + kPM - 1) / kPM) * (p.N / kPN);
    if (tiles == 0) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kv_project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPSmem);
    if (e != cudaSuccess) return e;
    kv_project_kernel<<<min(tiles, num_sms), kPThreads, kPSmem, stream>>>(p, ma, mb);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace lkv_dev
