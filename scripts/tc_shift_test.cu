// Dev probe (not product): SWIZZLE_128B UMMA operand whose start is NOT 1024-byte aligned.  A TMA box of
// 136 rows x 32 fp32 lands 1024-aligned; the MMA reads rows [j, j+128) by starting the descriptor at +128*j,
// with the descriptor's base-offset field (bits 49-51) = 0 (variant 0) or (addr >> 7) & 7 (variant 1).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2208_11422_b200/csrc/tc_sm100.cuh"

using namespace lfm;
constexpr int NT = 64, ROWS = 136;

__global__ void probe(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, float* C, int variant) {
    extern __shared__ unsigned char sm_raw[];
    __shared__ uint64_t bar_ld, bar_mma;
    __shared__ uint32_t tmem_base;
    const uint32_t raw = tc::smem_u32(sm_raw);
    unsigned char* sm = sm_raw + (((raw + 1023u) & ~1023u) - raw);
    unsigned char* a = sm;                   // 136 * 128 = 17408 B
    unsigned char* b = sm + 18432;           // NT * 128
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar_ld, 1);
        tc::mbar_init(&bar_mma, 1);
        tc::mbar_fence_init();
    }
    if (threadIdx.x < 32) tc::tmem_alloc(&tmem_base, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = tmem_base;
    if (threadIdx.x == 0) {
        tc::mbar_arrive_expect_tx(&bar_ld, ROWS * 128 + NT * 128);
        tc::tma_load_3d(a, &tmA, 0, 0, 0, &bar_ld);
        tc::tma_load_3d(b, &tmB, 0, 0, 0, &bar_ld);
        tc::mbar_wait(&bar_ld, 0);
        tc::fence_after();
        const uint32_t idesc = tc::idesc_tf32(128, NT);
        for (int j = 0; j < 8; ++j) {
            const uint32_t as = tc::smem_u32(a) + 128 * j;
            for (int s = 0; s < 4; ++s) {
                uint64_t da = tc::sdesc_sw128(as + 32 * s);
                if (variant == 1) da |= (uint64_t)((as >> 7) & 7) << 49;
                tc::mma_tf32(tm + (uint32_t)(j * NT), da, tc::sdesc_sw128(tc::smem_u32(b) + 32 * s), idesc, s > 0);
            }
        }
        tc::mma_commit(&bar_mma);
    }
    __syncwarp();
    tc::mbar_wait(&bar_mma, 0);
    tc::fence_after();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c0 = 0; c0 < 8 * NT; c0 += 8) {
        uint32_t r[8];
        tc::tmem_ld8_nowait(tm + ((uint32_t)(32 * w) << 16) + c0, r);
        tc::tmem_wait_ld();
        for (int i = 0; i < 8; ++i) C[(size_t)(32 * w + lane) * 8 * NT + c0 + i] = __uint_as_float(r[i]);
    }
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_dealloc(tm, 512);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static bool encode(EncodeFn enc, CUtensorMap* tm, float* p, int rows) {
    cuuint64_t dims[3] = {32, (cuuint64_t)rows, 1}, strides[2] = {128, (cuuint64_t)rows * 128};
    cuuint32_t box[3] = {32, (cuuint32_t)rows, 1}, es[3] = {1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

int main() {
    std::vector<float> A((size_t)ROWS * 32), B((size_t)NT * 32);
    srand(3);
    for (auto& v : A) v = (float)(rand() % 17 - 8);
    for (auto& v : B) v = (float)(rand() % 13 - 6);
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dC, (size_t)128 * 8 * NT * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap ta, tb;
    if (!enc || !encode(enc, &ta, dA, ROWS) || !encode(enc, &tb, dB, NT)) {
        printf("encode failed\n");
        return 1;
    }
    const int smem = 18432 + NT * 128 + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int variant = 0; variant < 2; ++variant) {
        cudaMemset(dC, 0xff, (size_t)128 * 8 * NT * 4);
        probe<<<1, 128, smem>>>(ta, tb, dC, variant);
        if (cudaDeviceSynchronize() != cudaSuccess) {
            printf("kernel error\n");
            return 1;
        }
        std::vector<float> Cv((size_t)128 * 8 * NT);
        cudaMemcpy(Cv.data(), dC, Cv.size() * 4, cudaMemcpyDeviceToHost);
        int badj[8] = {0};
        for (int j = 0; j < 8; ++j)
            for (int r = 0; r < 128; ++r)
                for (int n = 0; n < NT; ++n) {
                    double ref = 0;
                    for (int k = 0; k < 32; ++k) ref += (double)A[(size_t)(r + j) * 32 + k] * B[(size_t)n * 32 + k];
                    if (Cv[(size_t)r * 8 * NT + j * NT + n] != (float)ref) ++badj[j];
                }
        printf("variant %d (base offset %s): mismatches per row shift j=0..7:", variant, variant ? "(addr>>7)&7" : "0");
        for (int j = 0; j < 8; ++j) printf(" %d", badj[j]);
        printf("\n");
    }
    return 0;
}
