// kernels_mac.cu -- the two HBM-bound frequency-domain multiply-accumulates (K3 / K6).
//
// Transfer matrices M[kappa][b'][u] (complex64, u contiguous, row length nu_pad, a multiple of 16):
//   forward  (K3): Y[kappa][b']  = sum_u M[kappa][b'][u] * G[kappa][u]
//   backward (K6): Xh[kappa][u]  = sum_b' conj(M[kappa][b'][u]) * R[kappa][b']
// Both stream M exactly once per call at 1 complex MAC (8 flop) per 8-byte element, so they are
// bound by HBM bandwidth.  M is read with streaming (evict-first) 32-byte loads; every other operand
// is small and L2/shared-memory resident.
#include <algorithm>
#include <cstdlib>

#include "lfm_internal.cuh"
#include "tc_sm100.cuh"   // mbarrier / bulk-copy helpers

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
// memory whenever kappa changes; one warp computes one row's dot product (lane-strided 32-byte loads,
// NL in flight per lane = NL KB per warp), then a warp-shuffle reduction.  MINB CTAs per SM.  A lane's vectors
// j = 0, 1, 2, ... alternate between two accumulators in j order, so the result is bit-identical for every NL
// and launch shape (the SM-partition and whole-GPU variants agree exactly).
template <int NT, int NL, int MINB>
__global__ void __launch_bounds__(NT, MINB) fwd_mac_kernel(const float2* __restrict__ M, const float2* __restrict__ G,
                                                         float2* __restrict__ Y, int N2, int nu_pad, long long rows) {
    extern __shared__ float4 gs[];
    const int nv = nu_pad >> 2;                       // 32-byte vectors per row
    const long long r_begin = rows * blockIdx.x / gridDim.x;
    const long long r_end = rows * (blockIdx.x + 1) / gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int nwarps = NT / 32;
    long long r = r_begin;
    while (r < r_end) {
        const long long kap = r / N2;
        long long r_k_end = (kap + 1) * N2;
        if (r_k_end > r_end) r_k_end = r_end;
        const float4* gsrc = reinterpret_cast<const float4*>(G + kap * nu_pad);
        __syncthreads();
        // split planes: gs[v] = the first two complex values of vector v, gs[nv + v] = the last two, so that a
        // warp's lane-strided 16-byte reads are contiguous (conflict-free)
        for (int v = threadIdx.x; v < 2 * nv; v += NT) gs[(v & 1) * nv + (v >> 1)] = gsrc[v];
        __syncthreads();
        for (long long row = r + warp; row < r_k_end; row += nwarps) {
            const f8* mrow = reinterpret_cast<const f8*>(M + row * nu_pad);
            float ar0 = 0.f, ai0 = 0.f, ar1 = 0.f, ai1 = 0.f;
            int v = lane;
            for (; v + (NL - 1) * 32 < nv; v += NL * 32) {
                f8 m[NL];
#pragma unroll
                for (int q = 0; q < NL; ++q) m[q] = ld_stream8(mrow + v + q * 32);
#pragma unroll
                for (int q = 0; q < NL; q += 2) {
                    cmac4(m[q], gs[v + q * 32], gs[nv + v + q * 32], ar0, ai0);
                    cmac4(m[q + 1], gs[v + (q + 1) * 32], gs[nv + v + (q + 1) * 32], ar1, ai1);
                }
            }
            // tail: vector j of the lane still goes to accumulator j & 1, so every NL sums in the same order
            for (int jv = (v - lane) >> 5; v < nv; v += 32, ++jv) {
                const f8 m = ld_stream8(mrow + v);
                if (jv & 1) cmac4(m, gs[v], gs[nv + v], ar1, ai1);
                else cmac4(m, gs[v], gs[nv + v], ar0, ai0);
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

// ================================================================================================
// Frame-batched (lockstep time-lapse) versions: one pass over M serves F frames, turning each
// per-kappa GEMV into a (N2 x nu) x (nu x F) complex GEMM; arithmetic intensity rises from 1 to F flop/byte.
// ================================================================================================
constexpr int kBatchKT = 16;   // u (reduction) tile of the batched forward

// CTA per kappa, thread per output phase b' (N2 <= 256); M tile [k][b'] and G tile [k][f] staged in shared
// memory (double buffered through registers), F complex accumulators per thread.
template <int F>
__global__ void __launch_bounds__(256) fwd_mac_batch_kernel(const float2* __restrict__ M, const float2* __restrict__ G,
                                                            long long g_fstride, float2* __restrict__ Y,
                                                            long long y_fstride, int N2, int nu_pad) {
    extern __shared__ float4 smb[];
    auto ms = reinterpret_cast<float2 (*)[kBatchKT][257]>(smb);                                  // [2][KT][257]
    auto gs = reinterpret_cast<float4 (*)[kBatchKT][F / 2]>(smb + (2 * kBatchKT * 257 + 1) / 2);   // [2][KT][F/2]
    const long long kap = blockIdx.x;
    const int tid = threadIdx.x;
    const float2* Mk = M + kap * N2 * (long long)nu_pad;
    const int ntiles = nu_pad / kBatchKT;
    // staging assignment: 8 threads x float4 (2 complex) per row segment of 16 complex
    const int seg_row0 = tid >> 3, seg_q = tid & 7;    // rows seg_row0 + 32*i
    float4 mreg[8];
    float4 greg;
    auto load_tile = [&](int t) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int row = seg_row0 + 32 * i;
            mreg[i] = row < N2 ? __ldcs(reinterpret_cast<const float4*>(Mk + (long long)row * nu_pad + t * kBatchKT) + seg_q)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (tid < kBatchKT * F / 2) {   // G: F frames x 16 complex, as float4 pairs of frames
            const int k = tid / (F / 2), fp = tid - (tid / (F / 2)) * (F / 2);
            const float2 g0 = G[2 * fp * g_fstride + kap * nu_pad + t * kBatchKT + k];
            const float2 g1 = G[(2 * fp + 1) * g_fstride + kap * nu_pad + t * kBatchKT + k];
            greg = make_float4(g0.x, g0.y, g1.x, g1.y);
        }
    };
    auto store_tile = [&](int b) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int row = seg_row0 + 32 * i;
            ms[b][2 * seg_q][row] = make_float2(mreg[i].x, mreg[i].y);
            ms[b][2 * seg_q + 1][row] = make_float2(mreg[i].z, mreg[i].w);
        }
        if (tid < kBatchKT * F / 2) {
            const int k = tid / (F / 2), fp = tid - (tid / (F / 2)) * (F / 2);
            gs[b][k][fp] = greg;
        }
    };
    float accr[F], acci[F];
#pragma unroll
    for (int f = 0; f < F; ++f) accr[f] = acci[f] = 0.f;
    load_tile(0);
    store_tile(0);
    __syncthreads();
    for (int t = 0; t < ntiles; ++t) {
        const int b = t & 1;
        if (t + 1 < ntiles) load_tile(t + 1);
#pragma unroll
        for (int k = 0; k < kBatchKT; ++k) {
            const float2 m = ms[b][k][tid];
#pragma unroll
            for (int fp = 0; fp < F / 2; ++fp) {
                const float4 g = gs[b][k][fp];
                accr[2 * fp] = fmaf(m.x, g.x, accr[2 * fp]);
                accr[2 * fp] = fmaf(-m.y, g.y, accr[2 * fp]);
                acci[2 * fp] = fmaf(m.x, g.y, acci[2 * fp]);
                acci[2 * fp] = fmaf(m.y, g.x, acci[2 * fp]);
                accr[2 * fp + 1] = fmaf(m.x, g.z, accr[2 * fp + 1]);
                accr[2 * fp + 1] = fmaf(-m.y, g.w, accr[2 * fp + 1]);
                acci[2 * fp + 1] = fmaf(m.x, g.w, acci[2 * fp + 1]);
                acci[2 * fp + 1] = fmaf(m.y, g.z, acci[2 * fp + 1]);
            }
        }
        if (t + 1 < ntiles) store_tile(b ^ 1);
        __syncthreads();
    }
    if (tid < N2) {
#pragma unroll
        for (int f = 0; f < F; ++f) Y[f * y_fstride + kap * N2 + tid] = make_float2(accr[f], acci[f]);
    }
}

// thread per 4 consecutive units, walks the N2 rows of M[kappa] once for all F frames; R[f][kappa][b'] in smem
template <int F>
__global__ void __launch_bounds__(128) bwd_mac_batch_kernel(const float2* __restrict__ M, const float2* __restrict__ R,
                                                            long long r_fstride, float2* __restrict__ Xh,
                                                            long long x_fstride, int N2, int nu_pad) {
    extern __shared__ float2 rsb[];   // [b'][f]
    const long long kap = blockIdx.y;
    for (int e = threadIdx.x; e < N2 * F; e += blockDim.x) {
        const int bq = e / F, f = e - (e / F) * F;
        rsb[e] = R[f * r_fstride + kap * N2 + bq];
    }
    __syncthreads();
    const int nv = nu_pad >> 2;
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    const f8* base = reinterpret_cast<const f8*>(M + kap * N2 * (long long)nu_pad) + v;
    const long long stride = nv;
    float acc[F][8];
#pragma unroll
    for (int f = 0; f < F; ++f)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[f][i] = 0.f;
    int b = 0;
    for (; b + 3 < N2; b += 4) {
        f8 m[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) m[q] = ld_stream8(base + (b + q) * stride);
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int f = 0; f < F; ++f) cjmac4(m[q], rsb[(b + q) * F + f], acc[f]);
    }
    for (; b < N2; ++b) {
        const f8 m = ld_stream8(base + b * stride);
#pragma unroll
        for (int f = 0; f < F; ++f) cjmac4(m, rsb[b * F + f], acc[f]);
    }
#pragma unroll
    for (int f = 0; f < F; ++f) {
        float4* o = reinterpret_cast<float4*>(Xh + f * x_fstride + kap * nu_pad) + 2 * v;
        o[0] = make_float4(acc[f][0], acc[f][1], acc[f][2], acc[f][3]);
        o[1] = make_float4(acc[f][4], acc[f][5], acc[f][6], acc[f][7]);
    }
}

// Forward batched MAC for F >= 8: 128 threads per kappa, each owns output phases b' = tid and tid + 128, so every
// shared-memory broadcast of G feeds twice the FMAs (the F = 16 kernel above was bound by smem load issue).
template <int F>
__global__ void __launch_bounds__(128) fwd_mac_batch2_kernel(const float2* __restrict__ M, const float2* __restrict__ G,
                                                             long long g_fstride, float2* __restrict__ Y,
                                                             long long y_fstride, int N2, int nu_pad) {
    extern __shared__ float4 smb[];
    auto ms = reinterpret_cast<float2 (*)[kBatchKT][257]>(smb);                                  // [2][KT][257]
    auto gs = reinterpret_cast<float4 (*)[kBatchKT][F / 2]>(smb + (2 * kBatchKT * 257 + 1) / 2);   // [2][KT][F/2]
    const long long kap = blockIdx.x;
    const int tid = threadIdx.x;
    const float2* Mk = M + kap * N2 * (long long)nu_pad;
    const int ntiles = nu_pad / kBatchKT;
    const int seg_row0 = tid >> 3, seg_q = tid & 7;    // rows seg_row0 + 16*i, float4 column seg_q
    float4 mreg[16];
    float4 greg[(kBatchKT * F / 2 + 127) / 128];
    auto load_tile = [&](int t) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int row = seg_row0 + 16 * i;
            mreg[i] = row < N2 ? __ldcs(reinterpret_cast<const float4*>(Mk + (long long)row * nu_pad + t * kBatchKT) + seg_q)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < (kBatchKT * F / 2 + 127) / 128; ++j) {
            const int e = tid + 128 * j;
            if (e < kBatchKT * F / 2) {
                const int k = e / (F / 2), fp = e - (e / (F / 2)) * (F / 2);
                const float2 g0 = G[2 * fp * g_fstride + kap * nu_pad + t * kBatchKT + k];
                const float2 g1 = G[(2 * fp + 1) * g_fstride + kap * nu_pad + t * kBatchKT + k];
                greg[j] = make_float4(g0.x, g0.y, g1.x, g1.y);
            }
        }
    };
    auto store_tile = [&](int b) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int row = seg_row0 + 16 * i;
            ms[b][2 * seg_q][row] = make_float2(mreg[i].x, mreg[i].y);
            ms[b][2 * seg_q + 1][row] = make_float2(mreg[i].z, mreg[i].w);
        }
#pragma unroll
        for (int j = 0; j < (kBatchKT * F / 2 + 127) / 128; ++j) {
            const int e = tid + 128 * j;
            if (e < kBatchKT * F / 2) {
                const int k = e / (F / 2), fp = e - (e / (F / 2)) * (F / 2);
                gs[b][k][fp] = greg[j];
            }
        }
    };
    float ar0[F], ai0[F], ar1[F], ai1[F];
#pragma unroll
    for (int f = 0; f < F; ++f) ar0[f] = ai0[f] = ar1[f] = ai1[f] = 0.f;
    load_tile(0);
    store_tile(0);
    __syncthreads();
    for (int t = 0; t < ntiles; ++t) {
        const int b = t & 1;
        if (t + 1 < ntiles) load_tile(t + 1);
#pragma unroll 4
        for (int k = 0; k < kBatchKT; ++k) {
            const float2 m0 = ms[b][k][tid];
            const float2 m1 = ms[b][k][tid + 128];
#pragma unroll
            for (int fp = 0; fp < F / 2; ++fp) {
                const float4 g = gs[b][k][fp];
                ar0[2 * fp] = fmaf(m0.x, g.x, ar0[2 * fp]);
                ar0[2 * fp] = fmaf(-m0.y, g.y, ar0[2 * fp]);
                ai0[2 * fp] = fmaf(m0.x, g.y, ai0[2 * fp]);
                ai0[2 * fp] = fmaf(m0.y, g.x, ai0[2 * fp]);
                ar0[2 * fp + 1] = fmaf(m0.x, g.z, ar0[2 * fp + 1]);
                ar0[2 * fp + 1] = fmaf(-m0.y, g.w, ar0[2 * fp + 1]);
                ai0[2 * fp + 1] = fmaf(m0.x, g.w, ai0[2 * fp + 1]);
                ai0[2 * fp + 1] = fmaf(m0.y, g.z, ai0[2 * fp + 1]);
                ar1[2 * fp] = fmaf(m1.x, g.x, ar1[2 * fp]);
                ar1[2 * fp] = fmaf(-m1.y, g.y, ar1[2 * fp]);
                ai1[2 * fp] = fmaf(m1.x, g.y, ai1[2 * fp]);
                ai1[2 * fp] = fmaf(m1.y, g.x, ai1[2 * fp]);
                ar1[2 * fp + 1] = fmaf(m1.x, g.z, ar1[2 * fp + 1]);
                ar1[2 * fp + 1] = fmaf(-m1.y, g.w, ar1[2 * fp + 1]);
                ai1[2 * fp + 1] = fmaf(m1.x, g.w, ai1[2 * fp + 1]);
                ai1[2 * fp + 1] = fmaf(m1.y, g.z, ai1[2 * fp + 1]);
            }
        }
        if (t + 1 < ntiles) store_tile(b ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int f = 0; f < F; ++f) {
        if (tid < N2) Y[f * y_fstride + kap * N2 + tid] = make_float2(ar0[f], ai0[f]);
        if (tid + 128 < N2) Y[f * y_fstride + kap * N2 + tid + 128] = make_float2(ar1[f], ai1[f]);
    }
}

cudaError_t launch_fwd_mac_batch(const float2* M, const float2* G, long long g_fstride, float2* Y, long long y_fstride,
                                 int F, int nkappa, int N2, int nu_pad, cudaStream_t s) {
    if (N2 > 256 || nu_pad % kBatchKT) return cudaErrorInvalidValue;
    const size_t smem = ((2 * kBatchKT * 257 + 1) / 2) * sizeof(float4) + 2 * kBatchKT * (F / 2) * sizeof(float4);
    cudaError_t e = cudaSuccess;
#define LFM_FB(FV)                                                                                              \
    case FV:                                                                                                    \
        e = cudaFuncSetAttribute(fwd_mac_batch_kernel<FV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e != cudaSuccess) return e;                                                                         \
        fwd_mac_batch_kernel<FV><<<nkappa, 256, smem, s>>>(M, G, g_fstride, Y, y_fstride, N2, nu_pad);          \
        break;
#define LFM_FB2(FV)                                                                                              \
    case FV:                                                                                                     \
        e = cudaFuncSetAttribute(fwd_mac_batch2_kernel<FV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e != cudaSuccess) return e;                                                                          \
        fwd_mac_batch2_kernel<FV><<<nkappa, 128, smem, s>>>(M, G, g_fstride, Y, y_fstride, N2, nu_pad);          \
        break;
    if (N2 <= 256 && F >= 8) {
        switch (F) {
            LFM_FB2(8)
            LFM_FB2(16)
            default: return cudaErrorInvalidValue;
        }
    } else {
        switch (F) {
            LFM_FB(2)
            LFM_FB(4)
            LFM_FB(8)
            LFM_FB(16)
            default: return cudaErrorInvalidValue;
        }
    }
#undef LFM_FB2
#undef LFM_FB
    return cudaGetLastError();
}

// Backward batched MAC, staged version (F >= 8): a CTA of 256 threads owns 1024 units (4 per thread) of one kappa and
// all F frames; the rows M[kappa][b'][u0 .. u0+1024) stream into shared memory by 1-D bulk copies through a 4-deep
// mbarrier ring (4 rows per stage), so the 128 fp32 accumulators per thread never wait on HBM latency.
constexpr int kBBU = 1024, kBBRows = 4, kBBStages = 4;

template <int F>
__global__ void __launch_bounds__(288, 1) bwd_mac_batch_staged_kernel(const float2* __restrict__ M, const float2* __restrict__ R,
                                                                      long long r_fstride, float2* __restrict__ Xh,
                                                                      long long x_fstride, int N2, int nu_pad) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint64_t full[kBBStages], empty[kBBStages];
    float2* rs = reinterpret_cast<float2*>(sm);                                  // [N2][F]
    unsigned char* stage = sm + (((size_t)N2 * F * sizeof(float2) + 127) & ~(size_t)127);
    const long long kap = blockIdx.y;
    const int u0 = blockIdx.x * kBBU;
    const int nu_here = min(kBBU, nu_pad - u0);                                  // multiple of 16
    const uint32_t row_bytes = (uint32_t)nu_here * sizeof(float2);
    const uint32_t stage_bytes = kBBRows * kBBU * sizeof(float2);
    const int ngroups = (N2 + kBBRows - 1) / kBBRows;
    const float2* Mk = M + kap * N2 * (long long)nu_pad + u0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kBBStages; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], 8);   // the 8 compute warps
        }
        tc::mbar_fence_init();
    }
    for (int e = threadIdx.x; e < N2 * F; e += blockDim.x) {
        const int bq = e / F, f = e - (e / F) * F;
        rs[e] = R[f * r_fstride + kap * N2 + bq];
    }
    __syncthreads();
    if (warp == 8) {
        // ---- producer warp: rows of M into the ring ----
        if (lane == 0)
            for (int gi = 0; gi < ngroups; ++gi) {
                const int s = gi % kBBStages;
                if (gi >= kBBStages) tc::mbar_wait(&empty[s], ((gi / kBBStages) - 1) & 1);
                const int nr = min(kBBRows, N2 - gi * kBBRows);
                tc::mbar_arrive_expect_tx(&full[s], (uint32_t)nr * row_bytes);
                for (int q = 0; q < nr; ++q)
                    tc::bulk_g2s(stage + (size_t)s * stage_bytes + (size_t)q * kBBU * sizeof(float2),
                                 Mk + (long long)(gi * kBBRows + q) * nu_pad, row_bytes, &full[s]);
            }
        return;
    }
    float acc[F][8];
#pragma unroll
    for (int f = 0; f < F; ++f)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[f][i] = 0.f;
    const int v = threadIdx.x;   // units 4v .. 4v+3 of the tile
    for (int gi = 0; gi < ngroups; ++gi) {
        const int s = gi % kBBStages;
        tc::mbar_wait(&full[s], (gi / kBBStages) & 1);
        const f8* rows = reinterpret_cast<const f8*>(stage + (size_t)s * stage_bytes);
        const int nr = min(kBBRows, N2 - gi * kBBRows);
        if (4 * v < nu_here) {
#pragma unroll
            for (int q = 0; q < kBBRows; ++q) {
                if (q < nr) {
                    const f8 m = rows[q * (kBBU / 4) + v];
                    const float2* rr = rs + (gi * kBBRows + q) * F;
#pragma unroll
                    for (int f = 0; f < F; ++f) cjmac4(m, rr[f], acc[f]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[s]);   // this warp is done with slot s
    }
    if (4 * v < nu_here) {
#pragma unroll
        for (int f = 0; f < F; ++f) {
            float4* o = reinterpret_cast<float4*>(Xh + f * x_fstride + kap * nu_pad + u0) + 2 * v;
            o[0] = make_float4(acc[f][0], acc[f][1], acc[f][2], acc[f][3]);
            o[1] = make_float4(acc[f][4], acc[f][5], acc[f][6], acc[f][7]);
        }
    }
}

cudaError_t launch_bwd_mac_batch(const float2* M, const float2* R, long long r_fstride, float2* Xh, long long x_fstride,
                                 int F, int nkappa, int N2, int nu_pad, cudaStream_t s) {
    const int threads = 128;
    const int nv = nu_pad / 4;
    dim3 grid((nv + threads - 1) / threads, nkappa);
    const size_t smem = (size_t)N2 * F * sizeof(float2);
    switch (F) {
        case 2: bwd_mac_batch_kernel<2><<<grid, threads, smem, s>>>(M, R, r_fstride, Xh, x_fstride, N2, nu_pad); break;
        case 4: bwd_mac_batch_kernel<4><<<grid, threads, smem, s>>>(M, R, r_fstride, Xh, x_fstride, N2, nu_pad); break;
        default: break;
    }
    if (F == 2 || F == 4) return cudaGetLastError();
    if (F != 8 && F != 16) return cudaErrorInvalidValue;
    // F >= 8: staged kernel (fp32-ALU bound, rows streamed through shared memory)
    const size_t ssm = (((size_t)N2 * F * sizeof(float2) + 127) & ~(size_t)127) + (size_t)kBBStages * kBBRows * kBBU * sizeof(float2);
    const dim3 sgrid((nu_pad + kBBU - 1) / kBBU, nkappa);
    cudaError_t e;
    if (F == 8) {
        e = cudaFuncSetAttribute(bwd_mac_batch_staged_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
        if (e != cudaSuccess) return e;
        bwd_mac_batch_staged_kernel<8><<<sgrid, 288, ssm, s>>>(M, R, r_fstride, Xh, x_fstride, N2, nu_pad);
    } else {
        e = cudaFuncSetAttribute(bwd_mac_batch_staged_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
        if (e != cudaSuccess) return e;
        bwd_mac_batch_staged_kernel<16><<<sgrid, 288, ssm, s>>>(M, R, r_fstride, Xh, x_fstride, N2, nu_pad);
    }
    return cudaGetLastError();
}

template <int NT, int NL, int MINB>
static cudaError_t fwd_mac_v(const float2* M, const float2* G, float2* Y, int nkappa, int N2, int nu_pad, int num_sms,
                             cudaStream_t s) {
    const size_t smem = (size_t)nu_pad * sizeof(float2);
    cudaError_t e = cudaFuncSetAttribute(fwd_mac_kernel<NT, NL, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    // persistent: as many CTAs per SM as are resident at once (<= MINB; a large G[kappa] row in shared memory can
    // allow fewer -- a non-resident CTA would run its static row range after the others)
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fwd_mac_kernel<NT, NL, MINB>, NT, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    long long rows = (long long)nkappa * N2;
    long long grid = (long long)num_sms * std::min(per_sm, MINB);
    if (grid > rows) grid = rows;
    fwd_mac_kernel<NT, NL, MINB><<<(unsigned)grid, NT, smem, s>>>(M, G, Y, N2, nu_pad, rows);
    return cudaGetLastError();
}

// whole GPU: one 16-warp CTA per SM, 8 loads in flight per lane (HBM-bound at ~90 % of peak);
// SM partition (§5.5, below the HBM limit, bound per SM): four 8-warp CTAs per SM, 4 loads per lane (measured
// 4.53 vs 4.91 ms on 52 SMs at c3)
cudaError_t launch_fwd_mac(const float2* M, const float2* G, float2* Y, int nkappa, int N2, int nu_pad, int num_sms,
                           int partition, cudaStream_t s) {
    if (partition) return fwd_mac_v<256, 4, 4>(M, G, Y, nkappa, N2, nu_pad, num_sms, s);
    return fwd_mac_v<512, 8, 1>(M, G, Y, nkappa, N2, nu_pad, num_sms, s);
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
