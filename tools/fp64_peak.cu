// Measured fp64 FMA peak of this B200 (the Haralick / moments roofline denominator,
// SURVEY.md 8(d)): every SM runs independent DFMA chains; FLOP = 2 per DFMA.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_peak.cu -o tools/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8, kIters = 1 << 14;

__global__ void k_dfma(double* out, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x * 1e-9 + k;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int k = 0; k < kChains; ++k) x[k] = fma(x[k], a, b);
    double s = 0;
#pragma unroll
    for (int k = 0; k < kChains; ++k) s += x[k];
    if (s == 42.0) out[0] = s;  // keep the chains live
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    cudaMalloc(&d, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int tpb : {128, 256, 512}) {
        for (int bps : {1, 2, 4, 8}) {
            const int grid = sms * bps;
            k_dfma<<<grid, tpb>>>(d, 0.999999, 1e-7);
            cudaEventRecord(e0);
            for (int r = 0; r < 5; ++r) k_dfma<<<grid, tpb>>>(d, 0.999999, 1e-7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flop = 5.0 * grid * tpb * (double)kIters * kChains * 2.0;
            const double tf = flop / (ms * 1e-3) / 1e12;
            if (tf > best) best = tf;
            printf("tpb %d blocks/SM %d: %.2f TFLOP/s\n", tpb, bps, tf);
        }
    }
    printf("{\"fp64_fma_tflops\": %.3f, \"sms\": %d}\n", best, sms);
    return cudaGetLastError() != cudaSuccess;
}
