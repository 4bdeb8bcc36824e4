// Dev probe (not product): the building blocks of the v2 tensor-core direct kernel on sm_100a.
//   A: a 3-D TMA box {32 fp32, 128 rows, 1 slab} with SWIZZLE_128B, loaded at a NEGATIVE row coordinate
//      (partially out of bounds -> zero fill) from slab 1 of a [2][LP][32] array;
//   B: an N x 32 tile pre-swizzled on the host (sw128_off) and moved with one 1-D bulk copy;
//   C[128][N] = A * B^T with tcgen05.mma.kind::tf32 (M=128, N=240, 4 K-steps of 8, SW128 descriptors),
//   read back with tcgen05.ld 32x32b.x8.  Inputs are small integers (exact in TF32) -> the check is exact.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2208_11422_b200/csrc/tc_sm100.cuh"

using namespace lfm;

constexpr int LP = 300, NT = 240, ROW0 = -5;

__global__ void probe(const __grid_constant__ CUtensorMap tmA, const float* Bsw, float* C) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* a = sm;            // 16 KB
    unsigned char* b = sm + 16384;    // NT * 128 B
    __shared__ uint64_t bar_ld, bar_mma;
    __shared__ uint32_t tmem_base;
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar_ld, 1);
        tc::mbar_init(&bar_mma, 1);
        tc::mbar_fence_init();
    }
    if (threadIdx.x < 32) tc::tmem_alloc(&tmem_base, 256);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = tmem_base;
    if (threadIdx.x == 0) {
        tc::mbar_arrive_expect_tx(&bar_ld, 16384 + NT * 128);
        tc::tma_load_3d(a, &tmA, 0, ROW0, 1, &bar_ld);
        tc::bulk_g2s(b, Bsw, NT * 128, &bar_ld);
        tc::mbar_wait(&bar_ld, 0);
        tc::fence_after();
        const uint32_t idesc = tc::idesc_tf32(128, NT);
        for (int s = 0; s < 4; ++s)
            tc::mma_tf32(tm, tc::sdesc_sw128(tc::smem_u32(a) + 32 * s), tc::sdesc_sw128(tc::smem_u32(b) + 32 * s), idesc,
                         s > 0);
        tc::mma_commit(&bar_mma);
    }
    __syncwarp();
    tc::mbar_wait(&bar_mma, 0);
    tc::fence_after();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c0 = 0; c0 < NT; c0 += 8) {
        uint32_t r[8];
        tc::tmem_ld8_nowait(tm + ((uint32_t)(32 * w) << 16) + c0, r);
        tc::tmem_wait_ld();
        for (int i = 0; i < 8; ++i) C[(size_t)(32 * w + lane) * NT + c0 + i] = __uint_as_float(r[i]);
    }
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_dealloc(tm, 256);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    std::vector<float> A((size_t)2 * LP * 32), B((size_t)NT * 32), Bsw((size_t)NT * 32, 0.f);
    srand(1);
    for (auto& v : A) v = (float)(rand() % 17 - 8);
    for (auto& v : B) v = (float)(rand() % 13 - 6);
    for (int n = 0; n < NT; ++n)
        for (int k = 0; k < 32; ++k) Bsw[tc::sw128_off(n, k) / 4] = B[(size_t)n * 32 + k];
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dC, (size_t)128 * NT * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bsw.data(), Bsw.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dC, 0xff, (size_t)128 * NT * 4);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) != cudaSuccess || !enc) {
        printf("no cuTensorMapEncodeTiled\n");
        return 1;
    }
    CUtensorMap tm;
    cuuint64_t dims[3] = {32, LP, 2}, strides[2] = {128, (cuuint64_t)LP * 128};
    cuuint32_t box[3] = {32, 128, 1}, es[3] = {1, 1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dA, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)cr);
        return 1;
    }
    const int smem = 16384 + NT * 128;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<1, 128, smem>>>(tm, dB, dC);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("kernel error %s\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<float> C((size_t)128 * NT);
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 128; ++r)
        for (int n = 0; n < NT; ++n) {
            const int row = ROW0 + r;
            double ref = 0;
            if (row >= 0 && row < LP)
                for (int k = 0; k < 32; ++k) ref += (double)A[((size_t)LP + row) * 32 + k] * B[(size_t)n * 32 + k];
            if (C[(size_t)r * NT + n] != (float)ref) {
                if (bad < 8) printf("mismatch r=%d n=%d got %g want %g\n", r, n, C[(size_t)r * NT + n], ref);
                ++bad;
            }
        }
    printf("SW128 TMA + bulk + tcgen05 N=%d probe: %s (%d mismatches)\n", NT, bad ? "FAIL" : "PASS", bad);
    return bad ? 1 : 0;
}
