// TMA probe 3: isolate static-vs-dynamic smem and expect_tx/TMA ordering.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
extern __shared__ __align__(1024) uint8_t dsm[];
template <int STATIC, int SYNC>
__global__ void k(const __grid_constant__ CUtensorMap tm, uint16_t* out, int x0, int y0, int bw) {
    __shared__ __align__(1024) uint8_t ssm[8192 + 64];
    uint8_t* base = STATIC ? ssm : dsm;
    uint32_t tile = (uint32_t)__cvta_generic_to_shared(base);
    uint32_t bar = tile + 8192;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(bw * 16) : "memory");
    if (SYNC) __syncthreads();
    if (threadIdx.x == 0)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(tile), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x0), "r"(y0), "r"(bar) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW%=:\n\tmbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n\t@!p bra.uni W%=;\n\t}" ::"r"(bar) : "memory");
    __syncthreads();
    const uint16_t* t = (const uint16_t*)base;
    for (int i = threadIdx.x; i < 8 * bw; i += blockDim.x) out[i] = t[i];
}
int main(int argc, char** argv) {
    int v = atoi(argv[1]), bw = 64, x0 = 16;
    const int W = 256, H = 256;
    uint16_t* h = (uint16_t*)malloc(W * H * 2);
    for (int i = 0; i < W * H; ++i) h[i] = (uint16_t)i;
    uint16_t *d, *o;
    cudaMalloc(&d, W * H * 2); cudaMalloc(&o, 8192);
    cudaMemcpy(d, h, W * H * 2, cudaMemcpyHostToDevice);
    alignas(64) CUtensorMap tm;
    cuuint64_t dims[2] = {W, H}; cuuint64_t str[1] = {W * 2};
    cuuint32_t box[2] = {(cuuint32_t)bw, 8}; cuuint32_t es[2] = {1, 1};
    cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    auto kk = v == 0 ? k<0,0> : v == 1 ? k<0,1> : v == 2 ? k<1,0> : k<1,1>;
    cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    kk<<<1, 32, 16384>>>(tm, o, x0, 20, bw);
    cudaError_t e = cudaDeviceSynchronize();
    uint16_t res[2048]; cudaMemcpy(res, o, 8 * bw * 2, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < 8; ++y) for (int x = 0; x < bw; ++x) if (res[y * bw + x] != (uint16_t)((20 + y) * W + x0 + x)) ++bad;
    printf("static %d sync %d: %s bad %d\n", v >> 1, v & 1, cudaGetErrorString(e), bad);
    return 0;
}
