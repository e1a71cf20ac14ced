// FP64 pipe probe: DMMA.8x8x4 alone, DFMA alone, and both interleaved in the
// same warps -- do the FP64 tensor and FP64 FMA pipes add up on sm_100a?
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>  // 0: DMMA only, 1: DFMA only, 2: both
__global__ void probe(double *out, int iters) {
    double c[8][2];
    double f[16];
    double a = threadIdx.x * 1e-9, b = 1.0 + blockIdx.x * 1e-9;
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = i * 1e-3;
    for (int it = 0; it < iters; ++it) {
        if (MODE != 1) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
        }
        if (MODE != 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = fma(f[i], b, a);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
#pragma unroll
    for (int i = 0; i < 16; ++i) s += f[i];
    if (s == 12345.0) out[0] = s;
}

int main() {
    double *out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 20000;
    for (int mode = 0; mode < 3; ++mode) {
        for (int warps : {4, 8, 16}) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            auto launch = [&]() {
                if (mode == 0) probe<0><<<sms * 2, warps * 32>>>(out, iters);
                if (mode == 1) probe<1><<<sms * 2, warps * 32>>>(out, iters);
                if (mode == 2) probe<2><<<sms * 2, warps * 32>>>(out, iters);
            };
            launch();
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double threads = (double)sms * 2 * warps * 32;
            double dmma_flops = mode != 1 ? (double)sms * 2 * warps * iters * 8 * (2.0 * 8 * 8 * 4) : 0;
            double dfma_flops = mode != 0 ? threads * iters * 16 * 2.0 : 0;
            printf("mode %d warps/CTA %2d: %.3f ms  DMMA %.1f TF  DFMA %.1f TF  total %.1f TF\n", mode, warps,
                   ms, dmma_flops / ms / 1e9, dfma_flops / ms / 1e9, (dmma_flops + dfma_flops) / ms / 1e9);
        }
    }
    return 0;
}
