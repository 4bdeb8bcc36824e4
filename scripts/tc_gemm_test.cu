// Dev test (not product): C[128][N] = A[128][K] * B[N][K]^T on tcgen05 kind::tf32 with the descriptors of
// paper_2208_11422_b200/csrc/tc_sm100.cuh, 1xTF32 and 3xTF32, compared with an fp64 CPU product.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2208_11422_b200/csrc/tc_sm100.cuh"

using namespace lfm;

template <bool THREE>
__global__ void tc_gemm(const float* A, const float* B, float* C, int K, int N) {
    extern __shared__ __align__(1024) unsigned char sm[];
    float* a_hi = reinterpret_cast<float*>(sm);
    float* a_lo = a_hi + 128 * K;
    float* b_hi = a_lo + 128 * K;
    float* b_lo = b_hi + N * K;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    for (int e = threadIdx.x; e < 128 * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        float h, l;
        tc::split_tf32(A[e], h, l);
        const uint32_t o = tc::kmajor_off(r, k, K) / 4;
        a_hi[o] = h;
        a_lo[o] = l;
    }
    for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        float h, l;
        tc::split_tf32(B[e], h, l);
        const uint32_t o = tc::kmajor_off(r, k, K) / 4;
        b_hi[o] = h;
        b_lo[o] = l;
    }
    tc::fence_proxy_async();
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar, 1);
        tc::mbar_fence_init();
    }
    if (threadIdx.x < 32) tc::tmem_alloc(&tmem_base, 256);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = tmem_base;
    if (threadIdx.x == 0) {
        const uint32_t idesc = tc::idesc_tf32(128, N);
        const uint32_t sboA = (K / 4) * 128, sboB = (K / 4) * 128;
        for (int s = 0; s < K / 8; ++s) {
            const uint64_t ah = tc::sdesc(tc::smem_u32(a_hi) + s * 256, 128, sboA);
            const uint64_t bh = tc::sdesc(tc::smem_u32(b_hi) + s * 256, 128, sboB);
            tc::mma_tf32(tm, ah, bh, idesc, s > 0);
            if (THREE) {
                const uint64_t al = tc::sdesc(tc::smem_u32(a_lo) + s * 256, 128, sboA);
                const uint64_t bl = tc::sdesc(tc::smem_u32(b_lo) + s * 256, 128, sboB);
                tc::mma_tf32(tm, ah, bl, idesc, 1);
                tc::mma_tf32(tm, al, bh, idesc, 1);
            }
        }
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::fence_after();
    const int w = threadIdx.x / 32;
    if (w < 4) {
        for (int c0 = 0; c0 < N; c0 += 16) {
            float v[16];
            tc::tmem_ld16(tm + ((uint32_t)(32 * w) << 16) + c0, v);
            const int row = 32 * w + (threadIdx.x & 31);
            for (int i = 0; i < 16 && c0 + i < N; ++i) C[row * N + c0 + i] = v[i];
        }
    }
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_dealloc(tm, 256);
}

int main() {
    int fails = 0;
    for (int N : {48, 64, 120, 232}) {
        for (int K : {32, 64}) {
            std::vector<float> A(128 * K), B(N * K), C(128 * N);
            srand(1234 + N + K);
            for (auto& x : A) x = (rand() / (float)RAND_MAX) * 2 - 1;
            for (auto& x : B) x = (rand() / (float)RAND_MAX) * 2 - 1;
            float *dA, *dB, *dC;
            cudaMalloc(&dA, A.size() * 4);
            cudaMalloc(&dB, B.size() * 4);
            cudaMalloc(&dC, C.size() * 4);
            cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
            cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
            const size_t smem = (size_t)(2 * 128 * K + 2 * N * K) * 4;
            for (int three = 0; three < 2; ++three) {
                cudaMemset(dC, 0, C.size() * 4);
                if (three) {
                    cudaFuncSetAttribute(tc_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    tc_gemm<true><<<1, 128, smem>>>(dA, dB, dC, K, N);
                } else {
                    cudaFuncSetAttribute(tc_gemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    tc_gemm<false><<<1, 128, smem>>>(dA, dB, dC, K, N);
                }
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("N=%d K=%d three=%d CUDA error %s\n", N, K, three, cudaGetErrorString(e));
                    return 2;
                }
                cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
                double maxerr = 0, maxref = 0;
                for (int i = 0; i < 128; ++i)
                    for (int j = 0; j < N; ++j) {
                        double ref = 0;
                        for (int k = 0; k < K; ++k) ref += (double)A[i * K + k] * B[j * K + k];
                        maxerr = fmax(maxerr, fabs(ref - C[i * N + j]));
                        maxref = fmax(maxref, fabs(ref));
                    }
                const double rel = maxerr / maxref;
                const bool ok = three ? rel < 2e-6 : rel < 3e-3;
                printf("N=%3d K=%2d %s max rel err %.3e %s\n", N, K, three ? "3xTF32" : "1xTF32", rel, ok ? "ok" : "FAIL");
                fails += !ok;
            }
            cudaFree(dA);
            cudaFree(dB);
            cudaFree(dC);
        }
    }
    printf(fails ? "TC GEMM TEST FAILED\n" : "TC GEMM TEST PASSED\n");
    return fails ? 1 : 0;
}
