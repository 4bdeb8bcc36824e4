// Dev probe (not product): tcgen05.mma.cta_group::2 kind::tf32 M=256 x N=240 x K=8 issue rate on sm_100a.
//   mode 0: R stages of 12 MMAs, a commit per stage, no waits
//   mode 1: as the direct kernel: accumulator groups of 2 stages alternate between 2 TMEM buffers and the
//           issuer waits for the commit of group g-2 before starting group g (drain = immediate)
//   mode 2: as mode 1 plus a per-stage commit + wait on stage it-3 (the smem ring's empty barrier)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2208_11422_b200/csrc/tc_sm100.cuh"

using namespace lfm;
constexpr int NT = 240;

__global__ void __cluster_dims__(2, 1, 1) rate(int mode, int R, long long* cyc, int n_mma) {
    extern __shared__ unsigned char sm_raw[];
    __shared__ uint64_t bar_st[3], bar_acc[2];
    __shared__ uint32_t tmem_base;
    const uint32_t raw = tc::smem_u32(sm_raw);
    unsigned char* sm = sm_raw + (((raw + 1023u) & ~1023u) - raw);
    const uint32_t rank = tc::cluster_ctarank();
    for (int i = threadIdx.x; i < 3 * 62 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.0f / (1 + i % 7);
    tc::fence_proxy_async();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 3; ++i) tc::mbar_init(&bar_st[i], 1);
        for (int i = 0; i < 2; ++i) tc::mbar_init(&bar_acc[i], 1);
        tc::mbar_fence_init();
    }
    if (threadIdx.x < 32) tc::tmem_alloc_pair(&tmem_base, 512);
    tc::fence_before();
    tc::cluster_sync();
    tc::fence_after();
    const uint32_t tm = tmem_base;
    if (mode == 3 && threadIdx.x < 32 && rank == 0) {   // whole warp, uniform loop, elected issue, precomputed descs
        const uint32_t idesc = tc::idesc_tf32(256, n_mma);
        long long t0 = clock64();
        int g = 0, gk = 0;
        for (int it = 0; it < R; ++it) {
            const int s = it % 3, j = g & 1;
            if (it >= 3) tc::mbar_wait(&bar_st[s], ((it / 3) - 1) & 1);
            if (gk == 0 && g >= 2) tc::mbar_wait(&bar_acc[j], ((g >> 1) - 1) & 1);
            tc::fence_after();
            const uint32_t a_hi = tc::smem_u32(sm + (size_t)s * 62 * 1024), a_lo = a_hi + 16384;
            const uint32_t b_hi = a_hi + 32768, b_lo = b_hi + NT / 2 * 128;
            const uint32_t acc = tm + (uint32_t)(j * 256);
            const uint64_t ah0 = tc::sdesc_sw128(a_hi), al0 = tc::sdesc_sw128(a_lo);
            const uint64_t bh0 = tc::sdesc_sw128(b_hi), bl0 = tc::sdesc_sw128(b_lo);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                tc::mma_tf32_pair_elect(acc, ah0 + 2 * k, bh0 + 2 * k, idesc, (gk == 0 && k == 0) ? 0u : 1u);
                tc::mma_tf32_pair_elect(acc, ah0 + 2 * k, bl0 + 2 * k, idesc, 1u);
                tc::mma_tf32_pair_elect(acc, al0 + 2 * k, bh0 + 2 * k, idesc, 1u);
            }
            gk += 4;
            tc::mma_commit_pair_elect(&bar_st[s], 1);
            if (gk >= 8) {
                tc::mma_commit_pair_elect(&bar_acc[j], 1);
                ++g;
                gk = 0;
            }
        }
        __shared__ uint64_t bar_end3;
        if (threadIdx.x == 0) tc::mbar_init(&bar_end3, 1);
        __syncwarp();
        tc::mbar_fence_init();
        tc::mma_commit_pair_elect(&bar_end3, 1);
        tc::mbar_wait(&bar_end3, 0);
        if (threadIdx.x == 0) cyc[0] = clock64() - t0;
    } else if (mode < 3 && threadIdx.x == 0 && rank == 0) {
        const uint32_t idesc = tc::idesc_tf32(256, n_mma);
        long long t0 = clock64();
        int g = 0, gk = 0;
        for (int it = 0; it < R; ++it) {
            const int s = it % 3, j = g & 1;
            if (mode == 2 && it >= 3) tc::mbar_wait(&bar_st[s], ((it / 3) - 1) & 1);
            if (mode >= 1 && gk == 0 && g >= 2) tc::mbar_wait(&bar_acc[j], ((g >> 1) - 1) & 1);
            tc::fence_after();
            const uint32_t a_hi = tc::smem_u32(sm + (size_t)s * 62 * 1024), a_lo = a_hi + 16384;
            const uint32_t b_hi = a_hi + 32768, b_lo = b_hi + NT / 2 * 128;
            const uint32_t acc = tm + (uint32_t)(j * 256);
            for (int k = 0; k < 4; ++k) {
                const uint64_t ah = tc::sdesc_sw128(a_hi + 32 * k), al = tc::sdesc_sw128(a_lo + 32 * k);
                const uint64_t bh = tc::sdesc_sw128(b_hi + 32 * k), bl = tc::sdesc_sw128(b_lo + 32 * k);
                tc::mma_tf32_pair(acc, ah, bh, idesc, (gk == 0 && k == 0) ? 0u : 1u);
                tc::mma_tf32_pair(acc, ah, bl, idesc, 1u);
                tc::mma_tf32_pair(acc, al, bh, idesc, 1u);
            }
            gk += 4;
            if (mode == 2) tc::mma_commit_pair(&bar_st[s], 1);
            if (gk >= 8) {
                if (mode >= 1) tc::mma_commit_pair(&bar_acc[j], 1);
                ++g;
                gk = 0;
            }
        }
        uint64_t fin;
        asm volatile("{\n\t.reg .b64 t;\n\tmov.b64 t, 0;\n\t}" ::: "memory");
        tc::mma_commit_pair(&bar_st[0], 1);
        (void)fin;
        // drain: wait for everything issued (commit tracks all prior MMAs)
        __shared__ uint64_t bar_end;
        tc::mbar_init(&bar_end, 1);
        tc::mbar_fence_init();
        tc::mma_commit_pair(&bar_end, 1);
        tc::mbar_wait(&bar_end, 0);
        cyc[0] = clock64() - t0;
    }
    tc::fence_before();
    tc::cluster_sync();
    if (threadIdx.x < 32) tc::tmem_dealloc_pair(tm, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    const int smem = 3 * 62 * 1024 + 1024;
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int n_mma : {240, 208, 160, 128, 64}) {   // MMA N (B rows split across the pair): does the time scale with N?
        for (int mode = 0; mode < 4; ++mode) {
            const int R = 2000;
            rate<<<2, 128, smem>>>(mode, R, d, n_mma);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("mode %d error %s\n", mode, cudaGetErrorString(e));
                return 1;
            }
            long long c;
            cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
            printf("N %d mode %d: %lld cycles for %d stages (%.1f cyc/MMA; N/2 = %d)\n", n_mma, mode, c, R,
                   (double)c / (R * 12), n_mma / 2);
        }
    }
    return 0;
}
