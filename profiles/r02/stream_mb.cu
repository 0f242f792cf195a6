// Microbenchmark (not product): how fast can per-head CTAs stream fp32 score rows?
// 256 heads x 131072 rows (134 MB), variants of layout / prefetch depth / grid shape.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int T = 131072, NH = 256, CH = 4096;

// one CTA per head, 512 threads, thread owns 8 contiguous rows of each chunk (2 float4), B chunks per step,
// double-buffered registers (the plan kernel's structure)
template <int B>
__global__ void __launch_bounds__(512, 2) k_head_contig(const float* sc, float thr, unsigned* out) {
    const float* s = sc + (size_t)blockIdx.x * T;
    unsigned cnt = 0;
    float4 a[B][2], b[B][2];
    auto load = [&](float4 (&v)[B][2], int c0) {
#pragma unroll
        for (int u = 0; u < B; ++u)
#pragma unroll
            for (int h = 0; h < 2; ++h) v[u][h] = __ldg(reinterpret_cast<const float4*>(s + (c0 + u) * CH + threadIdx.x * 8 + 4 * h));
    };
    auto proc = [&](const float4 (&v)[B][2]) {
#pragma unroll
        for (int u = 0; u < B; ++u)
#pragma unroll
            for (int h = 0; h < 2; ++h) cnt += (v[u][h].x > thr) + (v[u][h].y > thr) + (v[u][h].z > thr) + (v[u][h].w > thr);
    };
    const int nc = T / CH;
    load(a, 0);
    for (int c0 = 0; c0 < nc; c0 += 2 * B) {
        if (c0 + B < nc) load(b, c0 + B);
        proc(a);
        if (c0 + B >= nc) break;
        if (c0 + 2 * B < nc) load(a, c0 + 2 * B);
        proc(b);
    }
    if (cnt == 0xffffffffu) out[0] = cnt;
    atomicAdd(out + 1, cnt);
}
// same, coalesced: thread owns float4 j*512 + tid of the chunk (two float4 per chunk, 8 KB apart)
template <int B>
__global__ void __launch_bounds__(512, 2) k_head_coal(const float* sc, float thr, unsigned* out) {
    const float* s = sc + (size_t)blockIdx.x * T;
    unsigned cnt = 0;
    float4 a[B][2], b[B][2];
    auto load = [&](float4 (&v)[B][2], int c0) {
#pragma unroll
        for (int u = 0; u < B; ++u)
#pragma unroll
            for (int h = 0; h < 2; ++h) v[u][h] = __ldg(reinterpret_cast<const float4*>(s + (c0 + u) * CH) + h * 512 + threadIdx.x);
    };
    auto proc = [&](const float4 (&v)[B][2]) {
#pragma unroll
        for (int u = 0; u < B; ++u)
#pragma unroll
            for (int h = 0; h < 2; ++h) cnt += (v[u][h].x > thr) + (v[u][h].y > thr) + (v[u][h].z > thr) + (v[u][h].w > thr);
    };
    const int nc = T / CH;
    load(a, 0);
    for (int c0 = 0; c0 < nc; c0 += 2 * B) {
        if (c0 + B < nc) load(b, c0 + B);
        proc(a);
        if (c0 + B >= nc) break;
        if (c0 + 2 * B < nc) load(a, c0 + 2 * B);
        proc(b);
    }
    if (cnt == 0xffffffffu) out[0] = cnt;
    atomicAdd(out + 1, cnt);
}
// persistent balanced: grid G CTAs, each a contiguous range of the 8192 chunks, coalesced, B=2
__global__ void __launch_bounds__(512, 2) k_persist(const float* sc, float thr, unsigned* out, int nchunks) {
    const int c_lo = (int)((long long)nchunks * blockIdx.x / gridDim.x), c_hi = (int)((long long)nchunks * (blockIdx.x + 1) / gridDim.x);
    unsigned cnt = 0;
    constexpr int B = 2;
    float4 a[B][2], b[B][2];
    auto load = [&](float4 (&v)[B][2], int c0) {
#pragma unroll
        for (int u = 0; u < B; ++u)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = min(c0 + u, nchunks - 1);
                v[u][h] = __ldg(reinterpret_cast<const float4*>(sc + (size_t)c * CH) + h * 512 + threadIdx.x);
            }
    };
    auto proc = [&](const float4 (&v)[B][2], int c0) {
#pragma unroll
        for (int u = 0; u < B; ++u)
            if (c0 + u < c_hi)
#pragma unroll
                for (int h = 0; h < 2; ++h) cnt += (v[u][h].x > thr) + (v[u][h].y > thr) + (v[u][h].z > thr) + (v[u][h].w > thr);
    };
    int c0 = c_lo;
    if (c0 < c_hi) load(a, c0);
    while (c0 < c_hi) {
        if (c0 + B < c_hi) load(b, c0 + B);
        proc(a, c0);
        c0 += B;
        if (c0 >= c_hi) break;
        if (c0 + B < c_hi) load(a, c0 + B);
        proc(b, c0);
        c0 += B;
    }
    if (cnt == 0xffffffffu) out[0] = cnt;
    atomicAdd(out + 1, cnt);
}

int main() {
    float* sc; unsigned* out; char* flush;
    cudaMalloc(&sc, (size_t)NH * T * 4);
    cudaMalloc(&out, 64);
    cudaMalloc(&flush, 256 << 20);
    cudaMemset(sc, 0, (size_t)NH * T * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        float best = 1e9;
        for (int r = 0; r < 6; ++r) {
            cudaMemsetAsync(flush, r, 256 << 20);
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 0 && ms < best) best = ms;
        }
        printf("%-28s %8.1f us  %6.0f GB/s\n", name, best * 1e3, (double)NH * T * 4 / (best * 1e-3) / 1e9);
    };
    run("head_contig B=1", [&] { k_head_contig<1><<<NH, 512>>>(sc, 0.5f, out); });
    run("head_contig B=2", [&] { k_head_contig<2><<<NH, 512>>>(sc, 0.5f, out); });
    run("head_coal B=1", [&] { k_head_coal<1><<<NH, 512>>>(sc, 0.5f, out); });
    run("head_coal B=2", [&] { k_head_coal<2><<<NH, 512>>>(sc, 0.5f, out); });
    run("head_coal B=4", [&] { k_head_coal<4><<<NH, 512>>>(sc, 0.5f, out); });
    for (int g : {148, 296, 592})
        run(g == 148 ? "persist 148" : g == 296 ? "persist 296" : "persist 592",
            [&] { k_persist<<<g, 512>>>(sc, 0.5f, out, NH * T / CH); });
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
}
