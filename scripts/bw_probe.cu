// Dev probe (not product): DRAM -> shared-memory streaming bandwidth vs. number of SMs, with 1-D bulk copies
// through a deep mbarrier ring (one CTA per SM, one producer thread, consumers touch each chunk once).
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2208_11422_b200/csrc/tc_sm100.cuh"
using namespace lfm;

constexpr int kChunk = 16384, kSlots = 12;   // 12 x 16 KB = 192 KB in flight per SM

__global__ void __launch_bounds__(288, 1) stream_kernel(const float4* __restrict__ src, size_t nchunks, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint64_t full[kSlots], empty[kSlots];
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSlots; ++i) { tc::mbar_init(&full[i], 1); tc::mbar_init(&empty[i], 8); }
        tc::mbar_fence_init();
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // chunks c = blockIdx.x + k * gridDim.x
    size_t my = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) ++my;
    if (warp == 8) {
        if (lane == 0)
        for (size_t k = 0; k < my; ++k) {
            const int s = k % kSlots;
            if (k >= kSlots) tc::mbar_wait(&empty[s], ((k / kSlots) - 1) & 1);
            tc::mbar_arrive_expect_tx(&full[s], kChunk);
            tc::bulk_g2s(sm + (size_t)s * kChunk, reinterpret_cast<const unsigned char*>(src) + (blockIdx.x + k * gridDim.x) * (size_t)kChunk, kChunk, &full[s]);
        }
        return;
    }
    float acc = 0.f;
    for (size_t k = 0; k < my; ++k) {
        const int s = k % kSlots;
        tc::mbar_wait(&full[s], (k / kSlots) & 1);
        const float4* v = reinterpret_cast<const float4*>(sm + (size_t)s * kChunk);
        for (int i = threadIdx.x; i < kChunk / 16; i += 256) acc += v[i].x;
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[s]);
    }
    if (acc == 12345.f) out[0] = acc;
    (void)warp;
}

int main() {
    const size_t bytes = (size_t)8 << 30;
    float4* d; float* o;
    cudaMalloc(&d, bytes); cudaMalloc(&o, 4);
    cudaMemset(d, 0, bytes);
    const int smem = kSlots * kChunk;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int ns[] = {148, 120, 96, 74, 56, 40, 28, 20};
    for (int n : ns) {
        stream_kernel<<<n, 288, smem>>>(d, bytes / kChunk, o);
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) stream_kernel<<<n, 288, smem>>>(d, bytes / kChunk, o);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double gbs = 3.0 * bytes / (ms / 1e3) / 1e9;
        printf("SMs %3d: %7.1f GB/s  (%.1f GB/s per SM)  err=%s\n", n, gbs, gbs / n, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
