// rope.cu -- K/V production for layer-by-layer prefill: the step before
// the eviction path.  The reference rotates keys with interleaved pairs
//   (x[2j], x[2j+1]) -> (a cos - b sin, a sin + b cos),  theta = pos * base^(-2j/d)
// (tensor.cpp:586-623, model.cpp:38-46) and scores the ROPED keys (evictsim.cpp:143,168).
//
//  * rope_table_kernel: cos/sin per (position, pair) evaluated in fp64 (theta reaches 1e5 rad
//    at 128k tokens, beyond fp32 argument reduction) and stored fp32; built once per prefill,
//    shared by every layer and head.
//  * rope_pack_kernel: token-major projections [s][t][H*D] (the GEMM output) -> head-major
//    dense layer [s][H][T][D] that the scorer's TMA map and the gather read, rotating K on the
//    way; 16-byte vectors, one warp per (s, t, h) row group.
#include "kernels.cuh"

namespace lkv_dev {

__global__ void __launch_bounds__(256) rope_table_kernel(int t_max, int half, double base, int pos_offset,
                                                         float2* cs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)t_max * half) return;
    const int p = (int)(i / half), j = (int)(i - (int64_t)p * half);
    const double freq = pow(base, -2.0 * j / (2.0 * half));
    const double th = (double)(pos_offset + p) * freq;
    double s, c;
    sincos(th, &s, &c);
    cs[i] = make_float2((float)c, (float)s);
}

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// grid: (ceil(t / rows_per_block), n_seq); each thread moves 8 elements (16 B for bf16).
template <typename T>
__global__ void __launch_bounds__(256) rope_pack_kernel(const T* __restrict__ k_lin, const T* __restrict__ v_lin,
                                                        int t_max, int t_len, int H, int D,
                                                        const float2* __restrict__ cs, T* __restrict__ k_out,
                                                        T* __restrict__ v_out) {
    const int s = blockIdx.y;
    const int per_row = H * D / 8;  // 8-element groups per token row
    const int64_t g0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)t_len * per_row;
    if (g0 >= total) return;
    const int p = (int)(g0 / per_row);
    const int r = (int)(g0 - (int64_t)p * per_row);
    const int h = (r * 8) / D, d0 = (r * 8) - h * D;
    const size_t src = ((size_t)s * t_max + p) * (size_t)H * D + (size_t)h * D + d0;
    const size_t dst = (((size_t)s * H + h) * t_max + p) * (size_t)D + d0;
    T kv[8], vv[8];
    if constexpr (sizeof(T) == 2) {
        *reinterpret_cast<uint4*>(kv) = *reinterpret_cast<const uint4*>(k_lin + src);
        *reinterpret_cast<uint4*>(vv) = *reinterpret_cast<const uint4*>(v_lin + src);
    } else {
        *reinterpret_cast<uint4*>(kv) = *reinterpret_cast<const uint4*>(k_lin + src);
        *reinterpret_cast<uint4*>(kv + 4) = *reinterpret_cast<const uint4*>(k_lin + src + 4);
        *reinterpret_cast<uint4*>(vv) = *reinterpret_cast<const uint4*>(v_lin + src);
        *reinterpret_cast<uint4*>(vv + 4) = *reinterpret_cast<const uint4*>(v_lin + src + 4);
    }
    const float2* row_cs = cs + (size_t)p * (D / 2) + d0 / 2;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float2 c = row_cs[q];
        const float a = to_f(kv[2 * q]), b = to_f(kv[2 * q + 1]);
        kv[2 * q] = from_f<T>(a * c.x - b * c.y);
        kv[2 * q + 1] = from_f<T>(a * c.y + b * c.x);
    }
    if constexpr (sizeof(T) == 2) {
        *reinterpret_cast<uint4*>(k_out + dst) = *reinterpret_cast<uint4*>(kv);
        *reinterpret_cast<uint4*>(v_out + dst) = *reinterpret_cast<uint4*>(vv);
    } else {
        *reinterpret_cast<uint4*>(k_out + dst) = *reinterpret_cast<uint4*>(kv);
        *reinterpret_cast<uint4*>(k_out + dst + 4) = *reinterpret_cast<uint4*>(kv + 4);
        *reinterpret_cast<uint4*>(v_out + dst) = *reinterpret_cast<uint4*>(vv);
        *reinterpret_cast<uint4*>(v_out + dst + 4) = *reinterpret_cast<uint4*>(vv + 4);
    }
}

cudaError_t launch_rope_table(int t_max, int head_dim, double base, int pos_offset, float2* cs, cudaStream_t stream) {
    const int64_t n = (int64_t)t_max * (head_dim / 2);
    rope_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(t_max, head_dim / 2, base, pos_offset, cs);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_rope_pack(const void* k_lin, const void* v_lin, int n_seq, int t_max, const int32_t* seq_lens,
                             int H, int D, int dtype, const float2* cs, void* k_out, void* v_out,
                             cudaStream_t stream) {
    int t_len = 0;
    for (int s = 0; s < n_seq; ++s) t_len = seq_lens[s] > t_len ? seq_lens[s] : t_len;
    const int64_t total = (int64_t)t_len * (H * D / 8);
    dim3 grid((unsigned)((total + 255) / 256), (unsigned)n_seq);
    if (dtype == LKV_BF16)
        rope_pack_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(
            static_cast<const __nv_bfloat16*>(k_lin), static_cast<const __nv_bfloat16*>(v_lin), t_max, t_len, H, D, cs,
            static_cast<__nv_bfloat16*>(k_out), static_cast<__nv_bfloat16*>(v_out));
    else
        rope_pack_kernel<float><<<grid, 256, 0, stream>>>(static_cast<const float*>(k_lin),
                                                          static_cast<const float*>(v_lin), t_max, t_len, H, D, cs,
                                                          static_cast<float*>(k_out), static_cast<float*>(v_out));
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace lkv_dev
