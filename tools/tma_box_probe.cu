// Standalone probe: 2-D TMA box loads of fp32 / fp64 padded arrays with the
// stage's box shapes, one variable at a time (diagnosing the fp32 tiled stage).
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 tools/tma_box_probe.cu -lcuda -o /tmp/probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>

struct alignas(128) Maps { CUtensorMap m; };

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <class T, int BX, int BY>
__global__ void k(const __grid_constant__ Maps M, int x0, int y0, T *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    T *dst = reinterpret_cast<T *>(sm);
    __shared__ alignas(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"((unsigned)(sizeof(T) * BX * BY)));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su32(dst)), "l"(reinterpret_cast<uint64_t>(&M.m)), "r"(x0), "r"(y0), "r"(su32(&bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(su32(&bar)) : "memory");
    for (int i = threadIdx.x; i < BX * BY; i += blockDim.x) out[i] = dst[i];
}

template <class T, int BX, int BY>
void run(const char *name, int dtype_override, int dx = 0) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    const int nx = 128, ny = 128, line = 128 / sizeof(T), xo = line - 2;
    const int pitch = (xo + nx + 4 + line - 1) / line * line, rows = ny + 4;
    T *a, *out;
    cudaMalloc(&a, sizeof(T) * pitch * rows);
    cudaMalloc(&out, sizeof(T) * BX * BY);
    cudaMemset(a, 0, sizeof(T) * pitch * rows);
    Maps M;
    cuuint64_t dims[2] = {(cuuint64_t)(xo + nx + 4), (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)pitch * sizeof(T)};
    cuuint32_t box[2] = {BX, BY}, es[2] = {1, 1};
    const CUtensorMapDataType dt = dtype_override >= 0 ? (CUtensorMapDataType)dtype_override
        : sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUresult r = enc(&M.m, dt, 2,
                     (char *)a, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k<T, BX, BY>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<T, BX, BY><<<1, 128, sizeof(T) * BX * BY + 128>>>(M, xo + 32 + dx, 30, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%-28s encode=%d launch=%s\n", name, (int)r, cudaGetErrorString(e));
    if (e != cudaSuccess) cudaDeviceReset();
    cudaFree(a);
    cudaFree(out);
}

#include <cstdlib>
int main(int argc, char **argv) {
    const int c = argc > 1 ? atoi(argv[1]) : 0;
    switch (c) {
    case 0: run<double, 36, 12>("f64 36x12", -1); break;
    case 1: run<float, 36, 12>("f32 36x12", -1); break;
    case 2: run<float, 32, 12>("f32 32x12", -1); break;
    case 3: run<float, 40, 12>("f32 40x12", -1); break;
    case 4: run<float, 36, 8>("f32 36x8", -1); break;
    case 5: run<float, 32, 11>("f32 32x11", -1); break;
    case 6: run<float, 64, 12>("f32 64x12", -1); break;
    case 7: run<double, 34, 12>("f64 34x12", -1); break;
    case 8: run<float, 36, 1>("f32 36x1", -1); break;
    case 9: run<float, 4, 12>("f32 4x12", -1); break;
    case 10: run<float, 12, 12>("f32 12x12", -1); break;
    case 11: run<float, 48, 12>("f32 48x12", -1); break;
    case 12: run<double, 18, 12>("f64 18x12", -1); break;
    case 13: run<double, 6, 12>("f64 6x12", -1); break;
    case 14: run<float, 36, 12>("f32 36x12 as UINT32", CU_TENSOR_MAP_DATA_TYPE_UINT32); break;
    case 15: run<float, 36, 12>("f32 36x12 as INT32", CU_TENSOR_MAP_DATA_TYPE_INT32); break;
    case 17: run<float, 40, 12>("f32 40x12 x0-2 (16B)", -1, -2); break;
    case 18: run<double, 36, 12>("f64 36x12 x0+1 (8 mod 16)", -1, 1); break;
    case 19: run<float, 36, 12>("f32 36x12 x0+2 (16B)", -1, 2); break;
    case 16: run<float, 36, 12>("f32 36x12 as FLOAT32_FTZ", CU_TENSOR_MAP_DATA_TYPE_FLOAT32_FTZ); break;
    }
    return 0;
}
