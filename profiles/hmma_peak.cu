// Legacy warp-level MMA (mma.sync m16n8k16 bf16 -> fp32) throughput on this GPU: the ceiling of
// the mma.sync kernels (decode attention, training attention).  Built + run under gpurun.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void hmma_loop(float* out, int iters) {
    float d[8][4] = {};
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0.f;
    for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    if (s == 1234.5f) out[0] = s;
}
int main() {
    float* out;
    cudaMalloc(&out, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int warps : {4, 8, 16, 32}) {
        const int iters = 4096;
        hmma_loop<<<sms, warps * 32>>>(out, iters);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        hmma_loop<<<sms, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = (double)sms * warps * iters * 8 * 4096;
        printf("warps/SM %2d: %.1f TFLOP/s (mma.sync bf16 m16n8k16)\n", warps, flops / ms / 1e9);
    }
    return 0;
}
