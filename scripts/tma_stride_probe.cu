// Dev probe (not product): DRAM bandwidth of TMA tile streams on 148 SMs -- 128-row x 128-byte boxes with a row
// pitch of P bytes (the batched MAC's M tiles: P = 2 nu_pad * 4 = 92 KB) vs. the same bytes contiguous (P = 128).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2208_11422_b200/csrc/tc_sm100.cuh"
using namespace lfm;
constexpr int kS = 8;

__global__ void __launch_bounds__(64, 1) tile_stream(const __grid_constant__ CUtensorMap tm, int ncols, int nrowblk, float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t full[kS];
    if (threadIdx.x == 0) { for (int i = 0; i < kS; ++i) tc::mbar_init(&full[i], 1); tc::mbar_fence_init(); }
    __syncthreads();
    const int ntiles = ncols * nrowblk;
    int my = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) ++my;
    if (threadIdx.x == 0) {
        float acc = 0.f;
        int issued = 0;
        auto issue = [&](int k) {
            const int t = blockIdx.x + k * gridDim.x, s = k % kS;
            tc::mbar_arrive_expect_tx(&full[s], 16384);
            tc::tma_load_3d(sm + s * 16384, &tm, (t % ncols) * 32, (t / ncols) * 128, 0, &full[s]);
        };
        for (; issued < kS && issued < my; ++issued) issue(issued);
        for (int k = 0; k < my; ++k) {
            tc::mbar_wait(&full[k % kS], (k / kS) & 1);
            acc += reinterpret_cast<float*>(sm + (k % kS) * 16384)[5];
            if (issued < my) issue(issued++);
        }
        if (acc == 1.2345f) out[0] = acc;
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    const size_t bytes = (size_t)8 << 30;
    float* d; float* o;
    cudaMalloc(&d, bytes); cudaMalloc(&o, 4); cudaMemset(d, 0, bytes);
    EncodeFn enc = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    cudaFuncSetAttribute(tile_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, kS * 16384);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const long long pitches[] = {128, 1024, 8192, 92160};
    for (long long P : pitches) {
        const long long rows = bytes / P;                  // rows of P bytes; the tile reads the first 128 B... of each
        const int ncols = (int)(P / 128);                  // column tiles per row band
        const int nrowblk = (int)(rows / 128);
        CUtensorMap tm;
        cuuint64_t dims[3] = {(cuuint64_t)(P / 4), (cuuint64_t)rows, 1}, str[2] = {(cuuint64_t)P, (cuuint64_t)bytes};
        cuuint32_t box[3] = {32, 128, 1}, es[3] = {1, 1, 1};
        if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode failed P=%lld\n", P); continue;
        }
        tile_stream<<<148, 64, kS * 16384>>>(tm, ncols, nrowblk, o);
        cudaEventRecord(a);
        tile_stream<<<148, 64, kS * 16384>>>(tm, ncols, nrowblk, o);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("row pitch %6lld B: %7.1f GB/s (%s)\n", P, (double)ncols * nrowblk * 16384 / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
