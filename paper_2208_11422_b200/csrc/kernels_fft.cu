// kernels_fft.cu -- coarse polyphase transforms (kernels K1/K2/K4/K5/K7).
//
// r2c_kernel: UB real Lh x Lw images per CTA (zero-padded coarse sub-aperture images, ratio-image
//   phases or wrapped PSF coarse kernels) -> Hermitian half-plane spectra written kappa-major
//   (out[kappa * ld + col]) so the multiply-accumulate kernels stream them contiguously.
//   Rows: two real rows packed into one complex FFT of length Lw, split with the Hermitian identity;
//   columns: nk2 complex FFTs of length Lh.
// c2r_kernel: the inverse (columns, then packed row pairs), cropped to the nh x nw coarse grid,
//   scaled by 1/(Lh Lw), followed by a fused epilogue (image scatter, polyphase store, or the RL
//   multiplicative update; the z max-projection is a separate deterministic pass, kernels_misc.cu).
//
// Polyphase facts used: with p = a + N m and s = b' + N m',
//   (H x)(b' + N m') = sum_a sum_m x_a[m] g_{a,b'}[m' - m],  g_{a,b'}[d] = h_a[b' - a + c + N d],
// a linear convolution of the coarse images; circular convolution of size L >= n + ceil(c/N) is
// alias-free on the cropped n outputs, and the adjoint uses conj(DFT g) with no extra scale.
#include "fft_smem.cuh"

namespace lfm {

template <int SRC>
__device__ __forceinline__ float src_val(const XformGeom& g, const R2CArgs& a, int t, int i, int j) {
    if constexpr (SRC == SRC_POLY) {
        const int lu = g.umap ? g.umap[t] : t;
        return a.in[((size_t)lu * g.nh + i) * g.nw + j];
    } else if constexpr (SRC == SRC_IMAGE) {
        const int u = g.unit0 + (g.umap ? g.umap[t] : t);
        const int N2 = g.N * g.N;
        const int z = u / N2, a1 = (u / g.N) % g.N, a2 = u % g.N;
        return a.in[((size_t)z * g.H + a1 + g.N * i) * g.W + a2 + g.N * j];
    } else if constexpr (SRC == SRC_RATIO) {
        const int b1 = t / g.N, b2 = t % g.N;
        const size_t pix = (size_t)(b1 + g.N * i) * g.W + b2 + g.N * j;
        return a.in[pix] / (fmaxf(a.in2[pix], 0.0f) + a.eps);
    } else if constexpr (SRC == SRC_ONES) {
        return 1.0f;
    } else if constexpr (SRC == SRC_IMAGE2D) {
        const int b1 = t / g.N, b2 = t % g.N;
        return a.in[(size_t)(b1 + g.N * i) * g.W + b2 + g.N * j];
    } else {  // SRC_KERNEL: t = b' * nu + uu ; wrapped coarse kernel g_{a,b'} at circular index (i, j)
        const int bp = t / g.nu, uu = t - bp * g.nu;
        const int b1 = bp / g.N, b2 = bp % g.N;
        const int lu = g.umap ? g.umap[uu] : uu;
        const int u = g.unit0 + lu;
        const int a1 = (u / g.N) % g.N, a2 = u % g.N;
        const float* ker = a.in + (size_t)lu * g.kh * g.kw;
        float v = 0.0f;
#pragma unroll
        for (int w1 = 0; w1 < 2; ++w1) {
            const int d1 = w1 ? i - g.Lh : i;
            const int k1 = b1 - a1 + g.ch + g.N * d1;
            if (k1 < 0 || k1 >= g.kh) continue;
#pragma unroll
            for (int w2 = 0; w2 < 2; ++w2) {
                const int d2 = w2 ? j - g.Lw : j;
                const int k2 = b2 - a2 + g.cw + g.N * d2;
                if (k2 < 0 || k2 >= g.kw) continue;
                v += ker[(size_t)k1 * g.kw + k2];
            }
        }
        return v;
    }
}

template <int SRC>
__global__ void __launch_bounds__(512) r2c_kernel(XformGeom g, FftDesc fh, FftDesc fw, const float2* __restrict__ twh_g,
                                                  const float2* __restrict__ tww_g, R2CArgs a, int UB, int S) {
    extern __shared__ float2 sm[];
    float2* twh = sm;
    float2* tww = sm + g.Lh;
    float2* bufA = tww + g.Lw;
    float2* bufB = bufA + (size_t)UB * S;
    for (int i = threadIdx.x; i < g.Lh; i += blockDim.x) twh[i] = twh_g[i];
    for (int i = threadIdx.x; i < g.Lw; i += blockDim.x) tww[i] = tww_g[i];
    const int t0 = blockIdx.x * UB;
    const int nt = min(UB, a.ntrans - t0);
    const bool full = (SRC == SRC_KERNEL);
    const int nrows = full ? g.Lh : g.nh;
    const int ncols = full ? g.Lw : g.nw;
    const int P = (nrows + 1) / 2;
    const int Lw = g.Lw, Lh = g.Lh, nk2 = g.nk2;

    // 1. load two real rows per complex row (zero-padded to Lw)
    const int nload = nt * P * Lw;
    for (int idx = threadIdx.x; idx < nload; idx += blockDim.x) {
        const int ui = idx / (P * Lw);
        const int rem = idx - ui * P * Lw;
        const int pr = rem / Lw;
        const int col = rem - pr * Lw;
        float re = 0.0f, im = 0.0f;
        if (col < ncols) {
            re = src_val<SRC>(g, a, t0 + ui, 2 * pr, col);
            if (2 * pr + 1 < nrows) im = src_val<SRC>(g, a, t0 + ui, 2 * pr + 1, col);
        }
        bufA[(size_t)ui * S + pr * Lw + col] = make_float2(re, im);
    }
    __syncthreads();
    // 2. row FFTs (length Lw)
    float2* res = fft_run<false>(bufA, bufB, fw, tww, nt * P, BatchLayout{P, S, Lw});
    float2* oth = (res == bufA) ? bufB : bufA;
    // 3. split packed rows (Hermitian identity) and transpose to column-major [k2][row]
    const int nun = nt * P * nk2;
    for (int idx = threadIdx.x; idx < nun; idx += blockDim.x) {
        const int ui = idx / (P * nk2);
        const int rem = idx - ui * P * nk2;
        const int pr = rem / nk2;
        const int k = rem - pr * nk2;
        const float2* row = res + (size_t)ui * S + pr * Lw;
        const float2 Z = row[k];
        float2 Q = row[k == 0 ? 0 : Lw - k];
        Q.y = -Q.y;  // conj(Z[-k])
        const float2 X0 = make_float2(0.5f * (Z.x + Q.x), 0.5f * (Z.y + Q.y));
        const float2 X1 = make_float2(0.5f * (Z.y - Q.y), -0.5f * (Z.x - Q.x));
        float2* col = oth + (size_t)ui * S + k * Lh;
        col[2 * pr] = X0;
        if (2 * pr + 1 < Lh) col[2 * pr + 1] = X1;
    }
    const int zr = Lh - 2 * P;
    if (zr > 0) {
        const int nz_ = nt * nk2 * zr;
        for (int idx = threadIdx.x; idx < nz_; idx += blockDim.x) {
            const int ui = idx / (nk2 * zr);
            const int rem = idx - ui * nk2 * zr;
            const int k = rem / zr;
            const int r = rem - k * zr;
            oth[(size_t)ui * S + k * Lh + 2 * P + r] = make_float2(0.0f, 0.0f);
        }
    }
    __syncthreads();
    // 4. column FFTs (length Lh)
    float2* res2 = fft_run<false>(oth, res, fh, twh, nt * nk2, BatchLayout{nk2, S, Lh});
    // 5. kappa-major store
    const int nkap = g.nkappa;
    const int nst = nkap * nt;
    for (int idx = threadIdx.x; idx < nst; idx += blockDim.x) {
        const int kap = idx / nt;
        const int ui = idx - kap * nt;
        const int k1 = kap / nk2;
        const int k2 = kap - k1 * nk2;
        const int t = t0 + ui;
        const int q = t / a.cdiv;
        const long long col = (long long)q * a.cmul + (t - q * a.cdiv);
        a.out[(long long)kap * a.out_ld + col] = res2[(size_t)ui * S + k2 * Lh + k1];
    }
}

template <int DST>
__global__ void __launch_bounds__(512) c2r_kernel(XformGeom g, FftDesc fh, FftDesc fw, const float2* __restrict__ twh_g,
                                                  const float2* __restrict__ tww_g, C2RArgs a, int UB, int S) {
    extern __shared__ float2 sm[];
    float2* twh = sm;
    float2* tww = sm + g.Lh;
    float2* bufA = tww + g.Lw;
    float2* bufB = bufA + (size_t)UB * S;
    for (int i = threadIdx.x; i < g.Lh; i += blockDim.x) twh[i] = twh_g[i];
    for (int i = threadIdx.x; i < g.Lw; i += blockDim.x) tww[i] = tww_g[i];
    const int t0 = blockIdx.x * UB;
    const int nt = min(UB, a.ntrans - t0);
    const int Lw = g.Lw, Lh = g.Lh, nk2 = g.nk2;
    // 1. gather spectra into column-major [k2][k1]
    const int nld = g.nkappa * nt;
    for (int idx = threadIdx.x; idx < nld; idx += blockDim.x) {
        const int kap = idx / nt;
        const int ui = idx - kap * nt;
        const int k1 = kap / nk2;
        const int k2 = kap - k1 * nk2;
        bufA[(size_t)ui * S + k2 * Lh + k1] = a.in[(long long)kap * a.in_ld + t0 + ui];
    }
    __syncthreads();
    // 2. inverse column FFTs
    float2* res = fft_run<true>(bufA, bufB, fh, twh, nt * nk2, BatchLayout{nk2, S, Lh});
    float2* oth = (res == bufA) ? bufB : bufA;
    // 3. rebuild full Hermitian rows for the nh needed rows, two real rows per complex row
    const int nh = g.nh, nw = g.nw;
    const int P = (nh + 1) / 2;
    const int npk = nt * P * Lw;
    for (int idx = threadIdx.x; idx < npk; idx += blockDim.x) {
        const int ui = idx / (P * Lw);
        const int rem = idx - ui * P * Lw;
        const int pr = rem / Lw;
        const int k = rem - pr * Lw;
        const bool mirror = (k >= nk2);
        const int kk = mirror ? Lw - k : k;
        const float2* col = res + (size_t)ui * S + kk * Lh;
        float2 A0 = col[2 * pr];
        float2 A1 = (2 * pr + 1 < nh) ? col[2 * pr + 1] : make_float2(0.0f, 0.0f);
        if (mirror) {
            A0.y = -A0.y;
            A1.y = -A1.y;
        }
        if (k == 0 || 2 * k == Lw) {  // DC / Nyquist of a real row: real part only
            A0.y = 0.0f;
            A1.y = 0.0f;
        }
        oth[(size_t)ui * S + pr * Lw + k] = make_float2(A0.x - A1.y, A0.y + A1.x);
    }
    __syncthreads();
    // 4. inverse row FFTs
    float2* res2 = fft_run<true>(oth, res, fw, tww, nt * P, BatchLayout{P, S, Lw});
    // 5. crop, scale, epilogue
    const float scale = 1.0f / (float)(Lh * Lw);
    const int nep = nt * nh * nw;
    for (int idx = threadIdx.x; idx < nep; idx += blockDim.x) {
        const int ui = idx / (nh * nw);
        const int rem = idx - ui * nh * nw;
        const int i = rem / nw;
        const int j = rem - i * nw;
        const float2 z = res2[(size_t)ui * S + (i >> 1) * Lw + j];
        const float v = ((i & 1) ? z.y : z.x) * scale;
        const int t = t0 + ui;
        if constexpr (DST == DST_IMAGE) {
            const int b1 = t / g.N, b2 = t % g.N;
            a.out[(size_t)(b1 + g.N * i) * g.W + b2 + g.N * j] = v;
        } else if constexpr (DST == DST_POLY) {
            a.out[((size_t)(g.umap ? g.umap[t] : t) * nh + i) * nw + j] = v;
        } else {
            const int lu = g.umap ? g.umap[t] : t;
            const int u = g.unit0 + lu;
            const int N2 = g.N * g.N;
            const int z = u / N2, a1 = (u / g.N) % g.N, a2 = u % g.N;
            if constexpr (DST == DST_VOLIMAGE) {
                a.out[((size_t)z * g.H + a1 + g.N * i) * g.W + a2 + g.N * j] = v;
            } else {  // DST_UPDATE / DST_ISRA
                const size_t pidx = ((size_t)lu * nh + i) * nw + j;
                a.out[pidx] = update_value<DST>(a.xold[pidx], a.norm[pidx], v, a.eps);
            }
        }
    }
}

static int xform_S(const XformGeom& g) {
    const int s1 = ((g.Lh + 1) / 2) * g.Lw;
    const int s2 = g.nk2 * g.Lh;
    return s1 > s2 ? s1 : s2;
}

static int xform_UB(const XformGeom& g, int S, size_t* smem) {
    const size_t budget = 200 * 1024;
    const size_t fixed = (size_t)(g.Lh + g.Lw) * sizeof(float2);
    int ub = (int)((budget - fixed) / (2 * (size_t)S * sizeof(float2)));
    if (ub > 4) ub = 4;
    if (ub < 1) ub = 1;
    *smem = fixed + 2 * (size_t)ub * S * sizeof(float2);
    return ub;
}

template <typename K>
static cudaError_t set_smem(K kernel, size_t smem) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

static bool g_fast = true;
void set_fast_fft_enabled(bool on) { g_fast = on; }

cudaError_t launch_r2c(const XformGeom& g, const FftDesc& fh, const FftDesc& fw, const float2* tw_h,
                       const float2* tw_w, const R2CArgs& a, cudaStream_t s) {
    if (a.ntrans <= 0) return cudaSuccess;
    if (g_fast && fast_fft_size(g.Lh, g.Lw)) return launch_r2c_fast(g, tw_h, a, s);
    const int S = xform_S(g);
    size_t smem;
    const int UB = xform_UB(g, S, &smem);
    const unsigned grid = (unsigned)((a.ntrans + UB - 1) / UB);
    const int threads = 512;
    cudaError_t e = cudaSuccess;
#define LFM_R2C_CASE(SRCV)                                                              \
    case SRCV:                                                                          \
        e = set_smem(r2c_kernel<SRCV>, smem);                                           \
        if (e != cudaSuccess) return e;                                                 \
        r2c_kernel<SRCV><<<grid, threads, smem, s>>>(g, fh, fw, tw_h, tw_w, a, UB, S);   \
        break;
    switch (a.src) {
        LFM_R2C_CASE(SRC_POLY)
        LFM_R2C_CASE(SRC_IMAGE)
        LFM_R2C_CASE(SRC_RATIO)
        LFM_R2C_CASE(SRC_ONES)
        LFM_R2C_CASE(SRC_KERNEL)
        LFM_R2C_CASE(SRC_IMAGE2D)
        default: return cudaErrorInvalidValue;
    }
#undef LFM_R2C_CASE
    return cudaGetLastError();
}

cudaError_t launch_c2r(const XformGeom& g, const FftDesc& fh, const FftDesc& fw, const float2* tw_h,
                       const float2* tw_w, const C2RArgs& a, cudaStream_t s) {
    if (a.ntrans <= 0) return cudaSuccess;
    if (g_fast && fast_fft_size(g.Lh, g.Lw)) return launch_c2r_fast(g, tw_h, a, s);
    const int S = xform_S(g);
    size_t smem;
    const int UB = xform_UB(g, S, &smem);
    const unsigned grid = (unsigned)((a.ntrans + UB - 1) / UB);
    const int threads = 512;
    cudaError_t e = cudaSuccess;
#define LFM_C2R_CASE(DSTV)                                                              \
    case DSTV:                                                                          \
        e = set_smem(c2r_kernel<DSTV>, smem);                                           \
        if (e != cudaSuccess) return e;                                                 \
        c2r_kernel<DSTV><<<grid, threads, smem, s>>>(g, fh, fw, tw_h, tw_w, a, UB, S);   \
        break;
    switch (a.dst) {
        LFM_C2R_CASE(DST_IMAGE)
        LFM_C2R_CASE(DST_POLY)
        LFM_C2R_CASE(DST_VOLIMAGE)
        LFM_C2R_CASE(DST_UPDATE)
        LFM_C2R_CASE(DST_ISRA)
        default: return cudaErrorInvalidValue;
    }
#undef LFM_C2R_CASE
    return cudaGetLastError();
}

bool fft_factor(int L, FftDesc* d) {
    d->L = L;
    d->nst = 0;
    int r = L;
    const int order[4] = {4, 2, 3, 5};
    for (int oi = 0; oi < 4; ++oi) {
        while (r % order[oi] == 0) {
            if (d->nst >= kMaxStages) return false;
            d->radix[d->nst++] = order[oi];
            r /= order[oi];
        }
    }
    return r == 1 && L >= 1;
}

int next_smooth(int n) {
    for (int m = n < 1 ? 1 : n;; ++m) {
        int r = m;
        const int ps[3] = {2, 3, 5};
        for (int k = 0; k < 3; ++k)
            while (r % ps[k] == 0) r /= ps[k];
        if (r == 1) return m;
    }
}

}  // namespace lfm
