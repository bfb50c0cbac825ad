// Standalone probe: 2D TMA tile load of a uint16 raster into shared memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, uint16_t* out, int x0, int y0, int getenv_bw, int dst_off = 0) {
    __shared__ __align__(1024) uint16_t tile[8 * 256 + 1024];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
        if (MODE != 2) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (MODE != 3) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const CUtensorMap* m = MODE == 1 ? gtm : &tm;
    if (MODE == 4) { if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&bar)) : "memory"); }
    else if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(getenv_bw * 16) : "memory");
        if (MODE == 6)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4}], [%2];" ::"r"(s32(tile)),
            "l"(reinterpret_cast<uint64_t>(m)), "r"(s32(&bar)), "r"(x0), "r"(y0)
            : "memory");
        else if (MODE == 7)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(s32(tile)), "l"(out + 4096), "r"(1024), "r"(s32(&bar)) : "memory");
        else
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4}], [%2];" ::"r"(s32(tile) + dst_off),
            "l"(reinterpret_cast<uint64_t>(m)), "r"(s32(&bar)), "r"(x0), "r"(y0)
            : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\tW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W%=;\n\t}" ::"r"(s32(&bar)) : "memory");
    for (int i = threadIdx.x; i < 8 * getenv_bw; i += blockDim.x) out[i] = tile[i + dst_off / 2];
}

int main(int argc, char** argv) {
    int mode = argc > 1 ? atoi(argv[1]) : 0;
    const int W = 256, H = 256;
    uint16_t* h = (uint16_t*)malloc(W * H * 2);
    for (int i = 0; i < W * H; ++i) h[i] = (uint16_t)i;
    uint16_t *d, *o;
    cudaMalloc(&d, W * H * 2);
    cudaMalloc(&o, 4096 + 8192*2);
    cudaMemcpy(d, h, W * H * 2, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    if (getenv("DIRECT")) enc = cuTensorMapEncodeTiled;
    alignas(64) CUtensorMap tm;
    cuuint64_t dims[2] = {W, H};
    cuuint64_t str[1] = {W * 2};
    cuuint32_t box[2] = {(cuuint32_t)(getenv("BW") ? atoi(getenv("BW")) : 64, getenv("OFF") ? atoi(getenv("OFF")) : 0), 8};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, (getenv("L2P") ? (CUtensorMapL2promotion)atoi(getenv("L2P")) : CU_TENSOR_MAP_L2_PROMOTION_L2_256B), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d fn=%p direct=%p\n", (int)r, fn, (void*)cuTensorMapEncodeTiled);
    for (int i = 0; i < 16; ++i) printf("%016llx ", ((unsigned long long*)&tm)[i]);
    printf("\n");
    CUtensorMap* gtm;
    cudaMalloc(&gtm, sizeof(CUtensorMap));
    cudaMemcpy(gtm, &tm, sizeof tm, cudaMemcpyHostToDevice);
    switch (mode) {
        case 0: k<0><<<1, 32>>>(tm, gtm, o, getenv("X0") ? atoi(getenv("X0")) : 10, 20, getenv("BW") ? atoi(getenv("BW")) : 64, getenv("OFF") ? atoi(getenv("OFF")) : 0); break;
        case 1: k<1><<<1, 32>>>(tm, gtm, o, 10, 20, 64); break;
        case 2: k<2><<<1, 32>>>(tm, gtm, o, 10, 20, 64); break;
        case 3: k<3><<<1, 32>>>(tm, gtm, o, 10, 20, 64); break;
        case 4: k<4><<<1, 32>>>(tm, gtm, o, 10, 20, 64); break;
        case 6: k<6><<<1, 32>>>(tm, gtm, o, 10, 20, 64); break;
        case 7: k<7><<<1, 32>>>(tm, gtm, o, 10, 20, 64); break;
        case 5: {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(1); cfg.blockDim = dim3(32);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            cudaError_t le = cudaLaunchKernelEx(&cfg, k<0>, tm, (const CUtensorMap*)gtm, o, 10, 20, 64, 0);
            printf("launch %s\n", cudaGetErrorString(le));
        } break;
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    uint16_t res[2048];
    cudaMemcpy(res, o, 4096, cudaMemcpyDeviceToHost);
    int bad = 0;
    int BW = getenv("BW") ? atoi(getenv("BW")) : 64;
    for (int y = 0; y < 8; ++y)
        for (int x = 0; x < BW; ++x)
            if (res[y * BW + x] != (uint16_t)((20 + y) * W + (getenv("X0") ? atoi(getenv("X0")) : 10) + x)) ++bad;
    printf("bad %d\n", bad);
    return 0;
}
