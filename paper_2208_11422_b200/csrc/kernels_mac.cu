// kernels_mac.cu -- the two HBM-bound frequency-domain multiply-accumulates (K3 / K6).
//
// Transfer matrices M[kappa][b'][u] (complex64, u contiguous, row length nu_pad, a multiple of 16):
//   forward  (K3): Y[kappa][b']  = sum_u M[kappa][b'][u] * G[kappa][u]
//   backward (K6): Xh[kappa][u]  = sum_b' conj(M[kappa][b'][u]) * R[kappa][b']
// Both stream M exactly once per call at 1 complex MAC (8 flop) per 8-byte element, so they are
// bound by HBM bandwidth.  M is read with streaming (evict-first) 32-byte loads; every other operand
// is small and L2/shared-memory resident.
#include "lfm_internal.cuh"

namespace lfm {

struct f8 {
    float4 a, b;
};

// 32-byte streaming load (sm_100 requires 256-bit vectors for the L2::evict_first hint)
__device__ __forceinline__ f8 ld_stream8(const f8* p) {
    f8 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v.a.x), "=f"(v.a.y), "=f"(v.a.z), "=f"(v.a.w), "=f"(v.b.x), "=f"(v.b.y), "=f"(v.b.z),
                   "=f"(v.b.w)
                 : "l"(p));
    return v;
}

// acc += m * g for the 4 complex values packed in (m, g)
__device__ __forceinline__ void cmac4(const f8& m, const float4& g0, const float4& g1, float& ar, float& ai) {
    ar = fmaf(m.a.x, g0.x, ar);
    ar = fmaf(-m.a.y, g0.y, ar);
    ai = fmaf(m.a.x, g0.y, ai);
    ai = fmaf(m.a.y, g0.x, ai);
    ar = fmaf(m.a.z, g0.z, ar);
    ar = fmaf(-m.a.w, g0.w, ar);
    ai = fmaf(m.a.z, g0.w, ai);
    ai = fmaf(m.a.w, g0.z, ai);
    ar = fmaf(m.b.x, g1.x, ar);
    ar = fmaf(-m.b.y, g1.y, ar);
    ai = fmaf(m.b.x, g1.y, ai);
    ai = fmaf(m.b.y, g1.x, ai);
    ar = fmaf(m.b.z, g1.z, ar);
    ar = fmaf(-m.b.w, g1.w, ar);
    ai = fmaf(m.b.z, g1.w, ai);
    ai = fmaf(m.b.w, g1.z, ai);
}

// Persistent: each CTA owns a contiguous range of (kappa, b') rows; G[kappa] is staged in shared
// memory whenever kappa changes; one warp computes one row's dot product (lane-strided 32-byte
// loads, 8 in flight per lane = 8 KB per warp), then a warp-shuffle reduction.
__global__ void __launch_bounds__(512, 1) fwd_mac_kernel(const float2* __restrict__ M, const float2* __restrict__ G,
                                                      float2* __restrict__ Y, int N2, int nu_pad, long long rows) {
    extern __shared__ float4 gs[];
    const int nv = nu_pad >> 2;                       // 32-byte vectors per row
    const long long r_begin = rows * blockIdx.x / gridDim.x;
    const long long r_end = rows * (blockIdx.x + 1) / gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    long long r = r_begin;
    while (r < r_end) {
        const long long kap = r / N2;
        long long r_k_end = (kap + 1) * N2;
        if (r_k_end > r_end) r_k_end = r_end;
        __syncthreads();
        const float4* gsrc = reinterpret_cast<const float4*>(G + kap * nu_pad);
        for (int v = threadIdx.x; v < 2 * nv; v += blockDim.x) gs[v] = gsrc[v];
        __syncthreads();
        for (long long row = r + warp; row < r_k_end; row += nwarps) {
            const f8* mrow = reinterpret_cast<const f8*>(M + row * nu_pad);
            float ar0 = 0.f, ai0 = 0.f, ar1 = 0.f, ai1 = 0.f;
            int v = lane;
            for (; v + 7 * 32 < nv; v += 8 * 32) {
                f8 m[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) m[q] = ld_stream8(mrow + v + q * 32);
#pragma unroll
                for (int q = 0; q < 8; q += 2) {
                    cmac4(m[q], gs[2 * (v + q * 32)], gs[2 * (v + q * 32) + 1], ar0, ai0);
                    cmac4(m[q + 1], gs[2 * (v + (q + 1) * 32)], gs[2 * (v + (q + 1) * 32) + 1], ar1, ai1);
                }
            }
            for (; v < nv; v += 32) {
                const f8 m = ld_stream8(mrow + v);
                cmac4(m, gs[2 * v], gs[2 * v + 1], ar0, ai0);
            }
            float ar = ar0 + ar1, ai = ai0 + ai1;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                ar += __shfl_xor_sync(0xffffffffu, ar, o);
                ai += __shfl_xor_sync(0xffffffffu, ai, o);
            }
            if (lane == 0) Y[row] = make_float2(ar, ai);
        }
        r = r_k_end;
    }
}

// acc_k += conj(m_k) * r for 4 consecutive units
__device__ __forceinline__ void cjmac4(const f8& m, const float2 rr, float* acc) {
    // conj(m) * r = (mx rx + my ry) + i (mx ry - my rx)
    acc[0] = fmaf(m.a.x, rr.x, acc[0]);
    acc[0] = fmaf(m.a.y, rr.y, acc[0]);
    acc[1] = fmaf(m.a.x, rr.y, acc[1]);
    acc[1] = fmaf(-m.a.y, rr.x, acc[1]);
    acc[2] = fmaf(m.a.z, rr.x, acc[2]);
    acc[2] = fmaf(m.a.w, rr.y, acc[2]);
    acc[3] = fmaf(m.a.z, rr.y, acc[3]);
    acc[3] = fmaf(-m.a.w, rr.x, acc[3]);
    acc[4] = fmaf(m.b.x, rr.x, acc[4]);
    acc[4] = fmaf(m.b.y, rr.y, acc[4]);
    acc[5] = fmaf(m.b.x, rr.y, acc[5]);
    acc[5] = fmaf(-m.b.y, rr.x, acc[5]);
    acc[6] = fmaf(m.b.z, rr.x, acc[6]);
    acc[6] = fmaf(m.b.w, rr.y, acc[6]);
    acc[7] = fmaf(m.b.z, rr.y, acc[7]);
    acc[7] = fmaf(-m.b.w, rr.x, acc[7]);
}

// One CTA per (kappa, chunk of 4*blockDim units): each thread owns four consecutive units and walks
// the N2 rows of M[kappa] (32-byte loads coalesced across the warp, 9 in flight), R[kappa] broadcast
// from shared memory.
__global__ void __launch_bounds__(128) bwd_mac_kernel(const float2* __restrict__ M, const float2* __restrict__ R,
                                                      float2* __restrict__ Xh, int N2, int nu_pad) {
    extern __shared__ float2 rs[];
    const long long kap = blockIdx.y;
    for (int b = threadIdx.x; b < N2; b += blockDim.x) rs[b] = R[kap * N2 + b];
    __syncthreads();
    const int nv = nu_pad >> 2;
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    const f8* base = reinterpret_cast<const f8*>(M + kap * N2 * (long long)nu_pad) + v;
    const long long stride = nv;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int b = 0;
    for (; b + 8 < N2; b += 9) {
        f8 m[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) m[q] = ld_stream8(base + (b + q) * stride);
#pragma unroll
        for (int q = 0; q < 9; ++q) cjmac4(m[q], rs[b + q], acc);
    }
    for (; b < N2; ++b) cjmac4(ld_stream8(base + b * stride), rs[b], acc);
    float4* o = reinterpret_cast<float4*>(Xh + kap * nu_pad) + 2 * v;
    o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

cudaError_t launch_fwd_mac(const float2* M, const float2* G, float2* Y, int nkappa, int N2, int nu_pad, int num_sms,
                           cudaStream_t s) {
    const size_t smem = (size_t)nu_pad * sizeof(float2);
    cudaError_t e = cudaFuncSetAttribute(fwd_mac_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int per_sm = 1;   // 512 threads x ~121 registers: one persistent CTA per SM
    long long rows = (long long)nkappa * N2;
    long long grid = (long long)num_sms * per_sm;
    if (grid > rows) grid = rows;
    fwd_mac_kernel<<<(unsigned)grid, 512, smem, s>>>(M, G, Y, N2, nu_pad, rows);
    return cudaGetLastError();
}

cudaError_t launch_bwd_mac(const float2* M, const float2* R, float2* Xh, int nkappa, int N2, int nu_pad,
                           cudaStream_t s) {
    const int threads = 128;
    const int nv = nu_pad / 4;
    dim3 grid((nv + threads - 1) / threads, nkappa);
    bwd_mac_kernel<<<grid, threads, N2 * sizeof(float2), s>>>(M, R, Xh, N2, nu_pad);
    return cudaGetLastError();
}

}  // namespace lfm
