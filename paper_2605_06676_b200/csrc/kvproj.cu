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
// Warp roles (persistent, CTA pairs on the SMs of a TPC): warp 0 = TMA producer (this CTA's A and
// B 128x64 boxes, 128-byte swizzle, 6-stage ring), warp 1 = the leader's single-thread UMMA issuer
// (tcgen05.mma.cta_group::2 kind::f16, M=256 N=256 K=16), warps 2-5 = epilogue (one TMEM lane
// quarter each), two TMEM accumulators (2 x 256 columns) so the epilogue of tile i overlaps the
// MMAs of tile i+1.
#include "kernels.cuh"

namespace lkv_dev {

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}

// ---- 2-SM UMMA (cta_group::2): a CTA pair computes one 256 x 256 tile --------------------------
// Each CTA of the pair loads its own 128 rows of A (tokens) and 128 rows of B (output columns) per
// k-step -- 32 KB instead of the 48 KB a single-SM 128 x 256 tile needs -- and the pair's leader
// issues tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 16), which reads A and B halves from
// both CTAs' shared memory and writes each CTA's 128 accumulator rows into that CTA's TMEM.  Both
// CTAs' TMA loads complete on the leader's `full` barrier; the leader's commits are multicast to
// both CTAs' `empty` / `tfull` barriers; both CTAs' epilogue warps release the accumulator on the
// leader's `tempty` barrier.
constexpr int kPM = 256;     // UMMA M of the pair (token rows per tile)
constexpr int kPN = 256;     // UMMA N (output columns per tile: two heads of K or V)
constexpr int kPK = 64;      // K per stage (one 128-byte swizzle box of bf16)
constexpr int kPStages = 6;
constexpr int kPThreads = 192;
constexpr int kPHalf = 128;                   // rows of A and of B each CTA holds
constexpr int kPABytes = kPHalf * kPK * 2;    // 16 KB
constexpr int kPBBytes = kPHalf * kPK * 2;    // 16 KB
constexpr int kPStageBytes = kPABytes + kPBBytes;
constexpr size_t kPSmem = (size_t)kPStages * kPStageBytes + 256 + 1024;

__device__ __forceinline__ uint32_t pair_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t cluster_addr(const void* local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
    return r;
}
// 2-SM TMA: the box lands in this CTA's shared memory, its bytes count on the leader's barrier
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* m, uint32_t leader_bar, int x,
                                                 int y, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_bar), "r"(x), "r"(y), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// arrive on `bar` (same offset) in both CTAs when the leader's MMAs issued so far complete
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}

__global__ void __launch_bounds__(kPThreads, 1)
    kv_project_kernel(const __grid_constant__ KvProjParams p, const __grid_constant__ CUtensorMap tmap_a,
                      const __grid_constant__ CUtensorMap tmap_b) {
    extern __shared__ unsigned char smem_dyn[];
    unsigned char* smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kPStages * kPStageBytes);
    uint64_t* full = bars;                   // [kPStages]  (the leader's counts both CTAs' bytes)
    uint64_t* empty = bars + kPStages;       // [kPStages]
    uint64_t* tfull = bars + 2 * kPStages;   // [2]
    uint64_t* tempty = tfull + 2;            // [2]         (the leader's: 8 epilogue warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = pair_rank();
    const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
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
            mbar_init(&tempty[i], 8);
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_b);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer (both CTAs: their halves of A and B) =====================
        if (lane == 0) {
            const uint64_t pol_a = l2_policy_evict_first();  // each A block is read by n_tiles_n pairs in a row
            const uint64_t pol_b = l2_policy_evict_last();   // the weights: every tile reads them
            int it = 0;
            for (int tile = pair; tile < n_tiles; tile += n_pairs) {
                const int m0 = (tile / n_tiles_n) * kPM + (int)rank * kPHalf;
                const int n0 = (tile % n_tiles_n) * kPN + (int)rank * kPHalf;
                for (int kb = 0; kb < k_steps; ++kb, ++it) {
                    const int st = it % kPStages;
                    mbar_wait_backoff(&empty[st], ((it / kPStages) & 1) ^ 1);
                    if (rank == 0) mbar_arrive_expect_tx(&full[st], 2 * kPStageBytes);
                    const uint32_t lbar = cluster_addr(&full[st], 0);
                    unsigned char* dst = smem + st * kPStageBytes;
                    tma_load_2d_pair(dst, &tmap_a, lbar, kb * kPK, m0, pol_a);
                    tma_load_2d_pair(dst + kPABytes, &tmap_b, lbar, kb * kPK, n0, pol_b);
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (the leader) =====================
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(kPM, kPN);
            const uint32_t base = smem_u32(smem);
            int it = 0, ti = 0;
            for (int tile = pair; tile < n_tiles; tile += n_pairs, ++ti) {
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
                        umma_bf16_pair(d_tmem, umma_desc_sw128(a_st + kk * 32), umma_desc_sw128(b_st + kk * 32), idesc,
                                       (kb | kk) ? 1u : 0u);
                    umma_commit_pair(&empty[st]);  // the stage is free in both CTAs once these MMAs retire
                }
                umma_commit_pair(&tfull[acc]);
            }
        }
    } else {
        // ===================== epilogue: RoPE + head-major pack (both CTAs, own 128 rows) ==========
        const int quarter = warp & 3;  // the TMEM lane quarter this warp may read
        const int HD = p.H * p.D;
        const uint32_t lead_tempty[2] = {cluster_addr(&tempty[0], 0), cluster_addr(&tempty[1], 0)};
        int ti = 0;
        for (int tile = pair; tile < n_tiles; tile += n_pairs, ++ti) {
            const int acc = ti & 1;
            const int m0 = (tile / n_tiles_n) * kPM + (int)rank * kPHalf, n0 = (tile % n_tiles_n) * kPN;
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
                if (c == kPN / 32 - 1) {  // accumulator drained: the leader's MMA may reuse it
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote(lead_tempty[acc]);
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
    cluster_sync_all();  // both CTAs done with TMEM, no arrival in flight
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
    }
}

size_t kv_project_smem() { return kPSmem; }

cudaError_t launch_kv_project(const KvProjParams& p, const CUtensorMap& ma, const CUtensorMap& mb, int num_sms,
                              cudaStream_t stream) {
    const int tiles = ((p.M + kPM - 1) / kPM) * (p.N / kPN);
    if (tiles == 0) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kv_project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPSmem);
    if (e != cudaSuccess) return e;
    const int pairs = min(tiles, num_sms / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kPThreads);
    cfg.dynamicSmemBytes = kPSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kv_project_kernel, p, ma, mb);
    note_launches(1);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace lkv_dev
