// fft_warp.cuh -- warp-level radix stages and the per-image shared-memory geometry shared by the coarse transforms
// of kernels_fft_fast.cu (whole coarse images) and kernels_fft_tile.cu (overlap-save tiles).
#pragma once
#include "fft_smem.cuh"

#ifndef LFM_FFT_MINB
#define LFM_FFT_MINB 2   // resident CTAs per SM the register budget targets
#endif

namespace lfm {

struct Radices {
    int n;
    int r[12];
};

constexpr Radices factorize(int L) {
    Radices f{0, {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}};
    int x = L;
    const int order[4] = {4, 2, 3, 5};
    for (int i = 0; i < 4; ++i)
        while (x % order[i] == 0) {
            f.r[f.n++] = order[i];
            x /= order[i];
        }
    return f;
}

template <int L, int R, int NS, bool INV>
__device__ __forceinline__ void warp_stage(float2* base, int stride, const float2* __restrict__ tw, int lane) {
    constexpr int LR = L / R;
    constexpr int NB = (LR + 31) / 32;
    constexpr int TWS = L / (NS * R);
    float2 v[NB][R];
#pragma unroll
    for (int t = 0; t < NB; ++t) {
        const int j = lane + 32 * t;
        if (j < LR) {
#pragma unroll
            for (int q = 0; q < R; ++q) v[t][q] = base[(j + q * LR) * stride];
            if constexpr (NS > 1) {
                const int k = j % NS;
#pragma unroll
                for (int q = 1; q < R; ++q) {
                    float2 w = tw[q * k * TWS];
                    if (INV) w.y = -w.y;
                    v[t][q] = c_mul(v[t][q], w);
                }
            }
            small_dft<R, INV>(v[t]);
        }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < NB; ++t) {
        const int j = lane + 32 * t;
        if (j < LR) {
            const int k = j % NS;
            const int o = (j - k) * R + k;
#pragma unroll
            for (int q = 0; q < R; ++q) base[(o + q * NS) * stride] = v[t][q];
        }
    }
    __syncwarp();
}

template <int L, int S, int NS, bool INV>
__device__ __forceinline__ void warp_fft(float2* base, int stride, const float2* __restrict__ tw, int lane) {
    constexpr Radices F = factorize(L);
    if constexpr (S < F.n) {
        constexpr int R = F.r[S];
        warp_stage<L, R, NS, INV>(base, stride, tw, lane);
        warp_fft<L, S + 1, NS * R, INV>(base, stride, tw, lane);
    }
}

// Two independent transforms per warp (lanes 0-15 -> base0, 16-31 -> base1) for every stage whose butterfly count
// L/R fits in 16 lanes (both radix-5 stages of L = 75, all stages of L = 15, 16, 36): the radix-5 stages of a lone
// transform keep only 15 of 32 lanes busy, and the kernels are issue-bound.  Stages with more butterflies run the
// two transforms one after the other.  base1 == base0 (an odd task left over) is allowed: in a paired stage both
// halves then compute and store identical values; sequential stages skip the second pass.
template <int L, int R, int NS, bool INV>
__device__ __forceinline__ void warp_stage_pair(float2* base0, float2* base1, int stride, const float2* __restrict__ tw,
                                                int lane) {
    constexpr int LR = L / R;
    static_assert(LR <= 16, "paired stage needs L/R <= 16");
    constexpr int TWS = L / (NS * R);
    const int j = lane & 15;
    float2* base = (lane & 16) ? base1 : base0;
    float2 v[R];
    if (j < LR) {
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = base[(j + q * LR) * stride];
        if constexpr (NS > 1) {
            const int k = j % NS;
#pragma unroll
            for (int q = 1; q < R; ++q) {
                float2 w = tw[q * k * TWS];
                if (INV) w.y = -w.y;
                v[q] = c_mul(v[q], w);
            }
        }
        small_dft<R, INV>(v);
    }
    __syncwarp();
    if (j < LR) {
        const int k = j % NS;
        const int o = (j - k) * R + k;
#pragma unroll
        for (int q = 0; q < R; ++q) base[(o + q * NS) * stride] = v[q];
    }
    __syncwarp();
}

template <int L>
constexpr bool has_pair_stage() {
    constexpr Radices F = factorize(L);
    for (int i = 0; i < F.n; ++i)
        if (L / F.r[i] <= 16) return true;
    return false;
}

template <int L, int S, int NS, bool INV>
__device__ __forceinline__ void warp_fft2(float2* base0, float2* base1, int stride, const float2* __restrict__ tw,
                                          int lane) {
    constexpr Radices F = factorize(L);
    if constexpr (S == 0 && !has_pair_stage<L>()) {
        warp_fft<L, 0, 1, INV>(base0, stride, tw, lane);   // one transform per warp (PW = 1): base1 == base0
    } else if constexpr (S < F.n) {
        constexpr int R = F.r[S];
        if constexpr (L / R <= 16) {
            warp_stage_pair<L, R, NS, INV>(base0, base1, stride, tw, lane);
        } else {
            warp_stage<L, R, NS, INV>(base0, stride, tw, lane);
            if (base1 != base0) warp_stage<L, R, NS, INV>(base1, stride, tw, lane);
        }
        warp_fft2<L, S + 1, NS * R, INV>(base0, base1, stride, tw, lane);
    }
}

template <int L>
struct FastGeom {
    static constexpr int NK2 = L / 2 + 1;
    static constexpr int RHO = (NK2 % 2) ? NK2 : NK2 + 1;   // odd row stride, 2*RHO >= L
    static constexpr int S = (L + 1) * RHO;                 // complex per image (packed rows of an odd L fit)
    static constexpr int NBL = (L + 31) / 32;
    // images per CTA: ~100 KB of shared memory (two CTAs per SM) unless one image needs more
    static constexpr size_t PER = (size_t)S * 8;
    static constexpr int UBR = (int)((PER <= 50 * 1024 ? 100 * 1024 : 200 * 1024) / PER);
    static constexpr int UB = UBR > 8 ? 8 : (UBR < 1 ? 1 : UBR);
    static constexpr size_t SMEM = (size_t)(L + 1) * 8 + (size_t)UB * PER;
    static constexpr size_t smem_for(int ub) { return (size_t)(L + 1) * 8 + (size_t)ub * PER; }
};

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

}  // namespace lfm
