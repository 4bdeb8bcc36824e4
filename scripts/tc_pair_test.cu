// Dev probe (not product): CTA-pair tcgen05 (cta_group::2) building blocks on sm_100a.
//   cluster (2,1,1); CTA r loads A rows [128r, 128r+128) and B rows [r*NT/2, (r+1)*NT/2) by TMA (SWIZZLE_128B),
//   both completing on the leader's mbarrier; the leader issues M=256 x N=NT x K=32 tcgen05.mma.cta_group::2;
//   a multicast commit releases both CTAs, each reads its 128 TMEM lanes.  Small-integer inputs -> exact check.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2208_11422_b200/csrc/tc_sm100.cuh"

using namespace lfm;
constexpr int NT = 240;

__global__ void __cluster_dims__(2, 1, 1) probe(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, float* C) {
    extern __shared__ unsigned char sm_raw[];
    __shared__ uint64_t bar_ld, bar_mma;
    __shared__ uint32_t tmem_base;
    const uint32_t raw = tc::smem_u32(sm_raw);
    unsigned char* sm = sm_raw + (((raw + 1023u) & ~1023u) - raw);
    unsigned char* a = sm;
    unsigned char* b = sm + 16384;
    const uint32_t rank = tc::cluster_ctarank();
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar_ld, 1);
        tc::mbar_init(&bar_mma, 1);
        tc::mbar_fence_init();
    }
    if (threadIdx.x < 32) tc::tmem_alloc_pair(&tmem_base, 256);
    tc::fence_before();
    tc::cluster_sync();
    tc::fence_after();
    const uint32_t tm = tmem_base;
    if (threadIdx.x == 0) {
        if (rank == 0) tc::mbar_arrive_expect_tx(&bar_ld, 2 * (16384 + NT / 2 * 128));
        tc::tma_load_3d_pair(a, &tmA, 0, 128 * rank, 0, &bar_ld);
        tc::tma_load_3d_pair(b, &tmB, 0, (NT / 2) * rank, 0, &bar_ld);
        if (rank == 0) {
            tc::mbar_wait(&bar_ld, 0);
            tc::fence_after();
            const uint32_t idesc = tc::idesc_tf32(256, NT);
            for (int s = 0; s < 4; ++s)
                tc::mma_tf32_pair(tm, tc::sdesc_sw128(tc::smem_u32(a) + 32 * s), tc::sdesc_sw128(tc::smem_u32(b) + 32 * s),
                                  idesc, s > 0);
            tc::mma_commit_pair(&bar_mma, 3);
        }
    }
    __syncwarp();
    tc::mbar_wait(&bar_mma, 0);
    tc::fence_after();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c0 = 0; c0 < NT; c0 += 8) {
        uint32_t r[8];
        tc::tmem_ld8_nowait(tm + ((uint32_t)(32 * w) << 16) + c0, r);
        tc::tmem_wait_ld();
        for (int i = 0; i < 8; ++i) C[(size_t)(128 * rank + 32 * w + lane) * NT + c0 + i] = __uint_as_float(r[i]);
    }
    tc::fence_before();
    tc::cluster_sync();
    if (threadIdx.x < 32) tc::tmem_dealloc_pair(tm, 256);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool encode(EncodeFn enc, CUtensorMap* tm, float* p, int rows, int boxrows) {
    cuuint64_t dims[3] = {32, (cuuint64_t)rows, 1}, strides[2] = {128, (cuuint64_t)rows * 128};
    cuuint32_t box[3] = {32, (cuuint32_t)boxrows, 1}, es[3] = {1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

int main() {
    std::vector<float> A((size_t)256 * 32), B((size_t)NT * 32);
    srand(2);
    for (auto& v : A) v = (float)(rand() % 17 - 8);
    for (auto& v : B) v = (float)(rand() % 13 - 6);
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dC, (size_t)256 * NT * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dC, 0xff, (size_t)256 * NT * 4);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap ta, tb;
    if (!enc || !encode(enc, &ta, dA, 256, 128) || !encode(enc, &tb, dB, NT, NT / 2)) {
        printf("encode failed\n");
        return 1;
    }
    const int smem = 16384 + NT / 2 * 128 + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<2, 128, smem>>>(ta, tb, dC);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("kernel error %s\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<float> Cv((size_t)256 * NT);
    cudaMemcpy(Cv.data(), dC, Cv.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 256; ++r)
        for (int n = 0; n < NT; ++n) {
            double ref = 0;
            for (int k = 0; k < 32; ++k) ref += (double)A[(size_t)r * 32 + k] * B[(size_t)n * 32 + k];
            if (Cv[(size_t)r * NT + n] != (float)ref) {
                if (bad < 8) printf("mismatch r=%d n=%d got %g want %g\n", r, n, Cv[(size_t)r * NT + n], ref);
                ++bad;
            }
        }
    printf("cta_group::2 M=256 N=%d probe: %s (%d mismatches)\n", NT, bad ? "FAIL" : "PASS", bad);
    return bad ? 1 : 0;
}
