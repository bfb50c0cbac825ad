// TMA probe 2: triton-like sequencing (128 threads, bar.sync between steps).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
extern __shared__ __align__(1024) uint8_t dsm[];
template <int FA, int FB, int FC> __global__ void k(const __grid_constant__ CUtensorMap tm, uint16_t* out, int x0, int y0, int bw, int nthr_tma) {
    uint32_t tile = (uint32_t)__cvta_generic_to_shared(dsm);
    uint32_t bar = tile + 8192;
    if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        if (FA) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (FB) asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(bw * 16) : "memory");
    __syncthreads();
    if (threadIdx.x < nthr_tma) {
        if (FC) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        uint64_t d;
        asm volatile("cvta.param.u64 %0, %1;" : "=l"(d) : "l"(&tm));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(tile), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x0), "r"(y0), "r"(bar) : "memory");
    }
    __syncthreads();
    asm volatile("{\n\t.reg .pred p;\n\tW%=:\n\tmbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n\t@!p bra.uni W%=;\n\t}" ::"r"(bar) : "memory");
    __syncthreads();
    const uint16_t* t = (const uint16_t*)dsm;
    for (int i = threadIdx.x; i < 8 * bw; i += blockDim.x) out[i] = t[i];
}
int main(int argc, char** argv) {
    int bw = argc > 1 ? atoi(argv[1]) : 64, x0 = argc > 2 ? atoi(argv[2]) : 16, nthr = argc > 3 ? atoi(argv[3]) : 128, nt = argc > 4 ? atoi(argv[4]) : 1;
    const int W = 256, H = 256;
    uint16_t* h = (uint16_t*)malloc(W * H * 2);
    for (int i = 0; i < W * H; ++i) h[i] = (uint16_t)i;
    uint16_t *d, *o;
    cudaMalloc(&d, W * H * 2); cudaMalloc(&o, 8192);
    cudaMemcpy(d, h, W * H * 2, cudaMemcpyHostToDevice);
    alignas(64) CUtensorMap tm;
    cuuint64_t dims[2] = {W, H}; cuuint64_t str[1] = {W * 2};
    cuuint32_t box[2] = {(cuuint32_t)bw, 8}; cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int f = argc > 5 ? atoi(argv[5]) : 0;
    auto kk = f == 0 ? k<0,0,0> : f == 1 ? k<1,0,0> : f == 2 ? k<0,1,0> : f == 3 ? k<0,0,1> : k<1,1,1>;
    cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    kk<<<1, nthr, 16384>>>(tm, o, x0, 20, bw, nt);
    cudaError_t e = cudaDeviceSynchronize();
    uint16_t res[2048]; cudaMemcpy(res, o, 8 * bw * 2, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < 8; ++y) for (int x = 0; x < bw; ++x) if (res[y * bw + x] != (uint16_t)((20 + y) * W + x0 + x)) ++bad;
    printf("f %d enc %d bw %d x0 %d nthr %d: %s bad %d\n", f, (int)r, bw, x0, nthr, cudaGetErrorString(e), bad);
    return 0;
}
