// Dev test (not product): tcgen05 kind::tf32 with an MN-major A operand: A tile [M=128][K=32] stored as 4 blocks of
// 32 M-elements, each [32 K rows][128 B]; B K-major as in the product kernels.  C = A * B^T vs fp64, 1x and 3xTF32.
// Variants 0 / 1 (SWIZZLE_128B, 16-byte chunks ^ row & 7, LBO/SBO either way) leave the accumulator untouched;
// variant 2 (SWIZZLE_128B_BASE32B: 32-byte chunks ^ row & 3, LBO = 4 KB, SBO = 512 B, layout type 1) is the valid
// MN-major tf32 layout, used by the batched backward MAC (kernels_mac_tc.cu).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2208_11422_b200/csrc/tc_sm100.cuh"

using namespace lfm;
constexpr int K = 32;

// bytes, MN-major tile (M = 128, K = 32): variant 0/1 SWIZZLE_128B (16-byte chunks ^ row & 7); variant 2
// SWIZZLE_128B_BASE32B (32-byte chunks ^ row & 3), the layout the CUTLASS builders require for MN-major tf32
__host__ __device__ inline uint32_t mn_off(int m, int k, int variant) {
    const int b = m / 32, c = m % 32;
    if (variant == 2) return (uint32_t)(b * 4096 + k * 128 + (((c >> 3) ^ (k & 3)) << 5) + (c & 7) * 4);
    return (uint32_t)(b * 4096 + k * 128 + ((((c * 4) >> 4) ^ (k & 7)) << 4) + ((c * 4) & 15));
}
__host__ __device__ inline uint32_t k_off(int n, int k) {   // bytes, K-major SW128 tile (rows n of 32 floats)
    return (uint32_t)(n * 128 + ((((k * 4) >> 4) ^ (n & 7)) << 4) + ((k * 4) & 15));
}
__device__ inline uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

template <bool THREE>
__global__ void tc_mn(const float* A, const float* B, float* C, int N, int variant) {   // A [128][K] row-major, B [N][K]
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    const uint32_t raw = tc::smem_u32(sm_raw);
    unsigned char* sm = sm_raw + (((raw + 1023u) & ~1023u) - raw);
    unsigned char* a_hi = sm;
    unsigned char* a_lo = sm + 16384;
    unsigned char* b_hi = sm + 32768;
    unsigned char* b_lo = b_hi + ((N * 128 + 1023) & ~1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    for (int e = threadIdx.x; e < 128 * K; e += blockDim.x) {
        const int m = e / K, k = e % K;
        float h, l;
        tc::split_tf32(A[e], h, l);
        *reinterpret_cast<float*>(a_hi + mn_off(m, k, variant)) = h;
        *reinterpret_cast<float*>(a_lo + mn_off(m, k, variant)) = l;
    }
    for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
        const int n = e / K, k = e % K;
        float h, l;
        tc::split_tf32(B[e], h, l);
        *reinterpret_cast<float*>(b_hi + k_off(n, k)) = h;
        *reinterpret_cast<float*>(b_lo + k_off(n, k)) = l;
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
        const uint32_t idesc = tc::idesc_tf32(128, N) | (1u << 15);   // A MN-major
        for (int s = 0; s < K / 8; ++s) {
            const uint32_t lbo = variant == 1 ? 1024 : 4096, sbo = variant == 1 ? 4096 : (variant == 2 ? 512 : 1024);
            const uint32_t lay = variant == 2 ? 1u : 2u;
            const uint64_t ah = desc(tc::smem_u32(a_hi) + s * 1024, lbo, sbo, lay);
            const uint64_t al = desc(tc::smem_u32(a_lo) + s * 1024, lbo, sbo, lay);
            const uint64_t bh = tc::sdesc_sw128(tc::smem_u32(b_hi) + s * 32);
            const uint64_t bl = tc::sdesc_sw128(tc::smem_u32(b_lo) + s * 32);
            tc::mma_tf32(tm, ah, bh, idesc, s > 0);
            if (THREE) {
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
    for (int variant = 0; variant < 3; ++variant)
    for (int N : {32, 64}) {
        std::vector<float> A(128 * K), B(N * K), C(128 * N);
        srand(99 + N);
        for (auto& x : A) x = (rand() / (float)RAND_MAX) * 2 - 1;
        for (auto& x : B) x = (rand() / (float)RAND_MAX) * 2 - 1;
        float *dA, *dB, *dC;
        cudaMalloc(&dA, A.size() * 4);
        cudaMalloc(&dB, B.size() * 4);
        cudaMalloc(&dC, C.size() * 4);
        cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
        const size_t smem = 32768 + 2 * 8192 + 1024;
        for (int three = 0; three < 2; ++three) {
            cudaMemset(dC, 0, C.size() * 4);
            if (three) {
                cudaFuncSetAttribute(tc_mn<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                tc_mn<true><<<1, 128, smem>>>(dA, dB, dC, N, variant);
            } else {
                cudaFuncSetAttribute(tc_mn<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                tc_mn<false><<<1, 128, smem>>>(dA, dB, dC, N, variant);
            }
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("N=%d CUDA error %s\n", N, cudaGetErrorString(e));
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
            double r0 = 0;
            for (int k = 0; k < K; ++k) r0 += (double)A[k] * B[k];
            printf("variant %d MN-major A: N=%3d %s max rel err %.3e %s  C00 %.5f ref %.5f C01 %.5f\n", variant, N,
                   three ? "3xTF32" : "1xTF32", rel, ok ? "ok" : "FAIL", C[0], r0, C[1]);
            fails += !ok;
        }
    }
    printf(fails ? "MN TEST FAILED\n" : "MN TEST PASSED\n");
    return fails ? 1 : 0;
}
