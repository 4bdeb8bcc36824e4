// fft_smem.cuh -- hand-written batched complex FFTs in shared memory for sm_100a.
//
// Stockham autosort, decimation in time, radices 2/3/4/5 (any 5-smooth length: the coarse transform
// sizes of DESIGN.md §2 -- 15, 36, 75, 144, ...).  One thread computes one radix-R butterfly per
// stage (R loads, twiddle, small DFT, R stores); stages ping-pong between two shared buffers.
// Twiddles W_L^t = exp(-2 pi i t / L) come from a table computed in fp64 on the host and rounded to
// fp32 (inverse transforms use the conjugate).  Element (b, t) of batch b lives at
//   base(b) + t,   base(b) = (b / per_unit) * unit_stride + (b % per_unit) * bstride.
#pragma once
#include "lfm_internal.cuh"

namespace lfm {

__device__ __forceinline__ float2 c_mul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ float2 c_mul_mi(float2 a) {
    return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

template <int R, bool INV>
__device__ __forceinline__ void small_dft(float2* v);

template <>
__device__ __forceinline__ void small_dft<2, false>(float2* v) {
    float2 a = v[0], b = v[1];
    v[0] = c_add(a, b);
    v[1] = c_sub(a, b);
}
template <>
__device__ __forceinline__ void small_dft<2, true>(float2* v) { small_dft<2, false>(v); }

template <int R, bool INV>
__device__ __forceinline__ void small_dft(float2* v) {
    if constexpr (R == 3) {
        const float s = INV ? -0.86602540378443864676f : 0.86602540378443864676f;  // sin(2pi/3)
        float2 t = c_add(v[1], v[2]);
        float2 d = c_sub(v[1], v[2]);
        float2 m = make_float2(v[0].x - 0.5f * t.x, v[0].y - 0.5f * t.y);
        // -i*s*d
        float2 q = make_float2(s * d.y, -s * d.x);
        v[0] = c_add(v[0], t);
        v[1] = c_add(m, q);
        v[2] = c_sub(m, q);
    } else if constexpr (R == 4) {
        float2 a = c_add(v[0], v[2]), b = c_sub(v[0], v[2]);
        float2 c = c_add(v[1], v[3]), d = c_mul_mi<INV>(c_sub(v[1], v[3]));
        v[0] = c_add(a, c);
        v[2] = c_sub(a, c);
        v[1] = c_add(b, d);
        v[3] = c_sub(b, d);
    } else if constexpr (R == 5) {
        const float c1 = 0.30901699437494742410f;    // cos(2pi/5)
        const float c2 = -0.80901699437494742410f;   // cos(4pi/5)
        const float s1 = INV ? -0.95105651629515357212f : 0.95105651629515357212f;  // sin(2pi/5)
        const float s2 = INV ? -0.58778525229247312917f : 0.58778525229247312917f;  // sin(4pi/5)
        float2 a1 = c_add(v[1], v[4]), b1 = c_sub(v[1], v[4]);
        float2 a2 = c_add(v[2], v[3]), b2 = c_sub(v[2], v[3]);
        float2 p1 = make_float2(v[0].x + c1 * a1.x + c2 * a2.x, v[0].y + c1 * a1.y + c2 * a2.y);
        float2 p2 = make_float2(v[0].x + c2 * a1.x + c1 * a2.x, v[0].y + c2 * a1.y + c1 * a2.y);
        // q1 = s1*b1 + s2*b2 ; q2 = s2*b1 - s1*b2 ; V1 = p1 - i q1, V4 = p1 + i q1, V2 = p2 - i q2, V3 = p2 + i q2
        float2 q1 = make_float2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y);
        float2 q2 = make_float2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y);
        v[0] = make_float2(v[0].x + a1.x + a2.x, v[0].y + a1.y + a2.y);
        v[1] = make_float2(p1.x + q1.y, p1.y - q1.x);
        v[4] = make_float2(p1.x - q1.y, p1.y + q1.x);
        v[2] = make_float2(p2.x + q2.y, p2.y - q2.x);
        v[3] = make_float2(p2.x - q2.y, p2.y + q2.x);
    }
}

struct BatchLayout {
    int per_unit;
    int unit_stride;
    int bstride;
};

template <int R, bool INV>
__device__ __forceinline__ void fft_stage(const float2* __restrict__ in, float2* __restrict__ out, int L, int Ns,
                                          const float2* __restrict__ tw, int nbatch, BatchLayout bl) {
    const int LR = L / R;
    const int total = nbatch * LR;
    const int twstep = L / (Ns * R);
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int b = idx / LR;
        const int j = idx - b * LR;
        const int bu = b / bl.per_unit;
        const int base = bu * bl.unit_stride + (b - bu * bl.per_unit) * bl.bstride;
        const int k = j % Ns;
        float2 v[R];
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = in[base + j + q * LR];
        if (Ns > 1) {
#pragma unroll
            for (int q = 1; q < R; ++q) {
                float2 w = tw[q * k * twstep];
                if (INV) w.y = -w.y;
                v[q] = c_mul(v[q], w);
            }
        }
        small_dft<R, INV>(v);
        const int o = base + (j - k) * R + k;   // (j / Ns) * Ns * R + k
#pragma unroll
        for (int q = 0; q < R; ++q) out[o + q * Ns] = v[q];
    }
}

// Runs all stages; returns the buffer holding the result (in or out).
template <bool INV>
__device__ float2* fft_run(float2* in, float2* out, const FftDesc& d, const float2* tw, int nbatch, BatchLayout bl) {
    int Ns = 1;
    for (int s = 0; s < d.nst; ++s) {
        const int R = d.radix[s];
        switch (R) {
            case 2: fft_stage<2, INV>(in, out, d.L, Ns, tw, nbatch, bl); break;
            case 3: fft_stage<3, INV>(in, out, d.L, Ns, tw, nbatch, bl); break;
            case 4: fft_stage<4, INV>(in, out, d.L, Ns, tw, nbatch, bl); break;
            default: fft_stage<5, INV>(in, out, d.L, Ns, tw, nbatch, bl); break;
        }
        __syncthreads();
        float2* t = in;
        in = out;
        out = t;
        Ns *= R;
    }
    return in;
}

}  // namespace lfm
