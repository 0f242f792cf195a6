// Microbenchmark of the weight-streaming GEMV (model.cu) per shape, outside ncu and graphs:
// `layers` distinct copies of each matrix are cycled so nothing is L2-resident, launches are
// PDL-chained on one stream as in the decode step.  Built by profiles/gemv_bench.sh.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2605_06676_b200/csrc/model.cu"  // the kernel itself, for launch variants

using namespace lkv_dev;

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e = (x);                                                                      \
        if (e != cudaSuccess) {                                                                   \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));    \
            exit(1);                                                                              \
        }                                                                                         \
    } while (0)

__global__ void fill_bf16(__nv_bfloat16* p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ seed;
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        p[i] = __float2bfloat16(((int)(h & 0xffff) - 32768) * (1.0f / 32768.f) * 0.02f);
    }
}

int main(int argc, char** argv) {
    const int layers = argc > 1 ? atoi(argv[1]) : 16;
    const int reps = argc > 2 ? atoi(argv[2]) : 8;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    struct Shape {
        const char* name;
        int N, K;
    } shapes[] = {{"qkv", 6144, 4096}, {"wo", 4096, 4096}, {"gate_up", 28672, 4096}, {"down", 4096, 14336},
                  {"lm_head", 128256, 4096}, {"tiny", 1024, 1024}};
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    float *part, *fout;
    uint32_t* cnt;
    CK(cudaMalloc(&part, gemv_max_grid(sms) * 2 * 64 * 16 * 4));
    CK(cudaMalloc(&cnt, 1 << 20));
    CK(cudaMemset(cnt, 0, 1 << 20));
    CK(cudaMalloc(&fout, 16 * 128256 * 4));
    for (const Shape& sh : shapes) {
        const int NG = (sh.N + 63) / 64, KU = (sh.K + 127) / 128;
        const size_t wbytes = (size_t)NG * KU * 16384;
        const int L = sh.N > 100000 ? 2 : layers;
        std::vector<void*> w(L);
        __nv_bfloat16* src;
        CK(cudaMalloc(&src, (size_t)sh.K * sh.N * 2));
        fill_bf16<<<1024, 256, 0, s>>>(src, (size_t)sh.K * sh.N, 7u);
        for (int l = 0; l < L; ++l) {
            CK(cudaMalloc(&w[l], wbytes));
            CK(cudaMemsetAsync(w[l], 0, wbytes, s));
            CK(launch_pack_weight(src, LKV_BF16, sh.K, sh.N, 0, 0, NG, KU, w[l], s));
        }
        CK(cudaFree(src));
        void* act;
        CK(cudaMalloc(&act, (size_t)KU * 8 * 256 * 2));
        fill_bf16<<<64, 256, 0, s>>>((__nv_bfloat16*)act, (size_t)KU * 8 * 256, 9u);
        GemvParams p{};
        p.NG = NG;
        p.KU = KU;
        p.N = sh.N;
        p.K = sh.K;
        p.B = 1;
        p.nbt = 1;
        p.act = act;
        p.part = part;
        p.cnt = cnt;
        p.epi = EPI_F32;
        p.f_out = fout;
        for (int l = 0; l < L; ++l) {  // warm
            p.w = w[l];
            CK(launch_gemv(p, LKV_BF16, sms, s));
        }
        const int mode = argc > 3 ? atoi(argv[3]) : 0;  // 0 launch_gemv, 1 plain <<<>>>, 2 plain + host timing
        const int64_t U = (int64_t)NG * KU;
        const int grid = (int)(U < 2 * sms ? U : 2 * sms);
        const size_t smem = wstream_smem(1);
        CK(cudaFuncSetAttribute(wstream_gemv_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        auto launch = [&]() {
            if (mode == 0) CK(launch_gemv(p, LKV_BF16, sms, s));
            else wstream_gemv_kernel<1, false><<<grid, kWsThreads, smem, s>>>(p);
        };
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, s));
        auto h0 = std::chrono::steady_clock::now();
        for (int r = 0; r < reps; ++r)
            for (int l = 0; l < L; ++l) {
                p.w = w[l];
                launch();
            }
        const double host_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count() / (reps * L);
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double us = ms * 1e3 / (reps * L);
        printf("mode %d %-8s N=%6d K=%6d  %8.1f MB  %8.2f us/launch  %7.1f GB/s  host %.2f us/launch\n", mode, sh.name,
               sh.N, sh.K, wbytes / 1e6, us, wbytes / us / 1e3, host_us);
#if LKV_GEMV_EXPT & 8
        {
            CK(cudaDeviceSynchronize());
            static unsigned long long z[512][8];
            memset(z, 0, sizeof z);
            CK(cudaMemcpyToSymbol(g_gemv_trace, z, sizeof z));
            p.w = w[0];
            launch();
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpyFromSymbol(z, g_gemv_trace, sizeof z));
            unsigned long long t0 = ~0ull, tend = 0;
            for (int c = 0; c < grid; ++c) if (z[c][5]) t0 = z[c][5] < t0 ? z[c][5] : t0;
            double mx[8] = {0}, av[8] = {0};
            int n[8] = {0};
            for (int c = 0; c < grid; ++c)
                for (int i = 0; i < 6; ++i)
                    if (z[c][i]) {
                        const double d = (z[c][i] - t0) * 1e-3;
                        mx[i] = d > mx[i] ? d : mx[i];
                        av[i] += d;
                        ++n[i];
                        tend = z[c][i] > tend ? z[c][i] : tend;
                    }
            printf("   trace (us from first CTA start): ");
            const char* nm[6] = {"cons_start", "data_done", "fixup_arrive", "epi_start", "epi_end", "cta_start"};
            for (int i = 0; i < 6; ++i) if (n[i]) printf("%s avg %.2f max %.2f | ", nm[i], av[i] / n[i], mx[i]);
            printf("\n");
        }
#endif
        for (int l = 0; l < L; ++l) CK(cudaFree(w[l]));
        CK(cudaFree(act));
    }
    return 0;
}
