// Per-launch cost of the pieces of a TMA-fed kernel (why small weight-stream GEMVs cost ~30 us):
// 296 CTAs (2 / SM), 86 KB dynamic smem, each CTA moves `units` x 16 KB with 1-D bulk copies.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2605_06676_b200/csrc/common.cuh"

using namespace lkv_dev;

template <int MODE>
__global__ void __launch_bounds__(160, 2) probe(const unsigned char* src, int units, float* out) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 4 * 18432);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&full[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (MODE == 0) return;  // launch + smem only
    const unsigned char* base = src + (size_t)blockIdx.x * units * 16384;
    if (MODE == 3) {  // plain vector loads
        float acc = 0.f;
        for (int u = 0; u < units; ++u)
            for (int i = threadIdx.x; i < 1024; i += blockDim.x) acc += reinterpret_cast<const float4*>(base + (size_t)u * 16384)[i].x;
        if (acc == 1234.5f) out[blockIdx.x] = acc;
        return;
    }
    if (threadIdx.x == 0) {
        const uint64_t pol = l2_policy_evict_first();
        for (int u = 0; u < units; ++u) {
            const int st = u & 3;
            if (u >= 4) mbar_wait(&full[st], ((u >> 2) - 1) & 1);
            mbar_arrive_expect_tx(&full[st], 16384);
            if (MODE == 1) bulk_g2s(smem + st * 18432, base + (size_t)u * 16384, 16384, &full[st], pol);
            else
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(smem + st * 18432)),
                    "l"(base + (size_t)u * 16384), "r"(16384), "r"(smem_u32(&full[st]))
                    : "memory");
        }
        for (int u = units > 4 ? units - 4 : 0; u < units; ++u) mbar_wait(&full[u & 3], (u >> 2) & 1);
    }
    __syncthreads();
}

int main(int argc, char** argv) {
    const int units = argc > 1 ? atoi(argv[1]) : 1;
    const int grid = 296;
    unsigned char* src;
    float* out;
    cudaMalloc(&src, (size_t)grid * units * 16384 + 1024);
    cudaMemset(src, 0, (size_t)grid * units * 16384);
    cudaMalloc(&out, grid * 4);
    const int smem = 86480;
    cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    void (*ks[4])(const unsigned char*, int, float*) = {probe<0>, probe<1>, probe<2>, probe<3>};
    const char* names[4] = {"empty (smem only)", "bulk copy + L2 hint", "bulk copy, no hint", "ld.global"};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int m = 0; m < 4; ++m) {
        for (int i = 0; i < 5; ++i) ks[m]<<<grid, 160, smem>>>(src, units, out);
        cudaEventRecord(e0);
        for (int i = 0; i < 100; ++i) ks[m]<<<grid, 160, smem>>>(src, units, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("units/CTA %3d  %-22s %8.2f us/launch  (%s)\n", units, names[m], ms * 10, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
