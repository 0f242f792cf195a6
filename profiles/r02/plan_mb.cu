// Microbenchmark (not product): which part of the plan kernel's score sweep costs what.
// 256 heads x 131072 fp32 scores ~ N(0,1); thresholds put ~15% of rows above the bin, ~5% inside.
// Variants share the plan kernel's structure (512 threads, 2 CTAs/SM, 16 rows/thread, half-CTA per
// chunk, double-buffered register loads) and add one piece of work at a time.
#include <cstdio>
#include <cstdint>
#include <curand_kernel.h>
constexpr int T = 131072, NH = 256, CH = 4096, NT = 512, R = 16, CAP = 8192;
__device__ __forceinline__ uint32_t f32_key(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
template <int V>
__global__ void __launch_bounds__(NT, 2) k_sweep(const float* scores, float g_thr, float lo_f, unsigned* out) {
    extern __shared__ uint32_t dyn[];
    uint32_t* s_cpos = dyn;
    uint32_t* s_ckey = dyn + CAP;
    __shared__ uint32_t cnt[2048], c_gt[64], s_ncand;
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < 2048; i += NT) cnt[i] = 0;
    if (tid < 64) c_gt[tid] = 0;
    if (tid == 0) s_ncand = 0;
    __syncthreads();
    const float* sc = scores + (size_t)blockIdx.x * T;
    const int u = tid / (CH / R), j0 = (tid % (CH / R)) * R;
    const int nc = T / CH;
    unsigned sink = 0;
    auto load = [&](float (&v)[R], int c0) {
#pragma unroll
        for (int h = 0; h < R / 4; ++h) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(sc + (c0 + u) * CH + j0 + 4 * h));
            v[4 * h] = f.x; v[4 * h + 1] = f.y; v[4 * h + 2] = f.z; v[4 * h + 3] = f.w;
        }
    };
    auto process = [&](const float (&v)[R], int c0) {
        const int c = c0 + u;
        if (V == 0) {  // loads only
#pragma unroll
            for (int q = 0; q < R; ++q) sink += __float_as_uint(v[q]);
            return;
        }
        uint32_t gt = 0, cm = 0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const bool above = v[q] > g_thr;
            gt += above;
            cm |= uint32_t(!above && v[q] >= lo_f) << q;
        }
        const uint32_t wgt = __reduce_add_sync(0xffffffffu, gt);
        if (lane == 0 && wgt) atomicAdd(&c_gt[c], wgt);
        if (V == 1) { sink += cm; return; }  // compare + per-chunk counts
        if (!__any_sync(0xffffffffu, cm)) return;
        const uint32_t ncd = __popc(cm);
        uint32_t incl = ncd;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        uint32_t base = 0;
        if (lane == 31) base = atomicAdd(&s_ncand, incl);
        base = __shfl_sync(0xffffffffu, base, 31) + incl - ncd;
        if (V == 2) { sink += base; return; }  // + warp scan and slot reservation
        const int r0 = c * CH + j0;
        while (cm) {
            const int q = __ffs(cm) - 1;
            cm &= cm - 1;
            if (V == 3) {  // + positions only
                if (base < CAP) s_cpos[base] = (uint32_t)(r0 + q);
                ++base;
                continue;
            }
            float h8[8], h4[4], h2[2];
#pragma unroll
            for (int z = 0; z < 8; ++z) h8[z] = (q & 8) ? v[z + 8] : v[z];
#pragma unroll
            for (int z = 0; z < 4; ++z) h4[z] = (q & 4) ? h8[z + 4] : h8[z];
#pragma unroll
            for (int z = 0; z < 2; ++z) h2[z] = (q & 2) ? h4[z + 2] : h4[z];
            const uint32_t key = f32_key((q & 1) ? h2[1] : h2[0]);
            if (V >= 5) atomicAdd(&cnt[(key >> 10) & 2047u], 1u);  // + pass-A histogram
            if (base < CAP) { s_cpos[base] = (uint32_t)(r0 + q); s_ckey[base] = key; }  // V4: + keys
            ++base;
        }
    };
    float va[R], vb[R];
    int c0 = 0;
    load(va, c0);
    while (c0 < nc) {
        if (c0 + 2 < nc) load(vb, c0 + 2);
        process(va, c0);
        c0 += 2;
        if (c0 >= nc) break;
        if (c0 + 2 < nc) load(va, c0 + 2);
        process(vb, c0);
        c0 += 2;
    }
    __syncthreads();
    if (sink == 0x12345678u) out[0] = sink;
    if (tid == 0) atomicAdd(out + 1, s_ncand + c_gt[0] + cnt[5]);
}
__global__ void init(float* s, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    curandStatePhilox4_32_10_t st;
    curand_init(7, i, 0, &st);
    for (; i < n; i += (size_t)gridDim.x * blockDim.x) s[i] = curand_normal(&st);
}
int main() {
    float* sc; unsigned* out; char* flush;
    cudaMalloc(&sc, (size_t)NH * T * 4);
    cudaMalloc(&out, 64);
    cudaMalloc(&flush, 256 << 20);
    init<<<1184, 256>>>(sc, (size_t)NH * T);
    // N(0,1): P(x > 1.0364) = 0.15, P(x > 0.9) ~ 0.184 -> ~3.4% in [0.9, 1.0364]
    const float g_thr = 1.0364f;
    float lo_f = 0.9f;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const size_t smem = 2 * CAP * 4;
    auto run = [&](const char* name, void (*k)(const float*, float, float, unsigned*)) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        float best = 1e9;
        for (int r = 0; r < 6; ++r) {
            cudaMemsetAsync(flush, r, 256 << 20);
            cudaEventRecord(e0);
            k<<<NH, NT, smem>>>(sc, g_thr, lo_f, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 0 && ms < best) best = ms;
        }
        printf("%-40s %8.1f us  %6.0f GB/s\n", name, best * 1e3, (double)NH * T * 4 / (best * 1e-3) / 1e9);
    };
    run("V0 loads only", k_sweep<0>);
    run("V1 + compare, per-chunk counts", k_sweep<1>);
    run("V2 + warp scan, slot reservation", k_sweep<2>);
    run("V3 + positions appended", k_sweep<3>);
    run("V4 + keys (select tree)", k_sweep<4>);
    run("V5 + pass-A histogram atomics", k_sweep<5>);
    lo_f = 0.8416f;  // ~5% of rows inside the bin (the C3 scorer's fraction at 11 bits)
    run("V5, 5% in the bin", k_sweep<5>);
    lo_f = 0.7f;     // ~9%
    run("V5, 9% in the bin", k_sweep<5>);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
