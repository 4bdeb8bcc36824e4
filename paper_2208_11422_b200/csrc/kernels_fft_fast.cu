// kernels_fft_fast.cu -- compile-time-specialised coarse transforms for the square sizes the BASELINE
// configs use (Lc = 15, 16, 36, 75, 144).  Same mathematics as kernels_fft.cu (K2/K4/K5/K7),
// re-organised for throughput:
//   * one warp owns one 1-D transform; radix stages run in place with __syncwarp only (every lane loads
//     its butterflies' inputs into registers, syncs, writes outputs), so warps never wait on each other
//     between stages and all index arithmetic is compile-time (no runtime integer division);
//   * one shared buffer per image: rows of odd stride RHO (>= Lw/2+1, conflict-light column access) and
//     packed row pairs at stride 2*RHO, so the real-row packing / Hermitian split is done in place by the
//     warp that transformed the row (no transpose buffer, half the shared memory of the generic path);
//   * the C2R fuses rebuild-row -> inverse row FFT -> crop/scale -> epilogue per warp.
#include "fft_warp.cuh"

namespace lfm {


// sources read straight from one array at base(t) + i * row_pitch + j * col_stride (plus the yhat array for RATIO)
template <int SRC>
constexpr bool strided_src() {
    return SRC == SRC_POLY || SRC == SRC_IMAGE || SRC == SRC_IMAGE2D || SRC == SRC_RATIO;
}
template <int SRC>
__device__ __forceinline__ long long src_base(const XformGeom& g, int t) {
    if constexpr (SRC == SRC_POLY) {
        return (long long)(g.umap ? g.umap[t] : t) * g.nh * g.nw;
    } else if constexpr (SRC == SRC_IMAGE) {
        const int u = g.unit0 + (g.umap ? g.umap[t] : t);
        const int N2 = g.N * g.N;
        const int z = u / N2, a1 = (u / g.N) % g.N, a2 = u % g.N;
        return ((long long)z * g.H + a1) * g.W + a2;
    } else {   // IMAGE2D, RATIO: t = output phase (b1, b2)
        return (long long)(t / g.N) * g.W + t % g.N;
    }
}

template <int SRC>
__device__ __forceinline__ float src_value(const XformGeom& g, const R2CArgs& a, int t, int i, int j) {
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
    } else {
        const int bp = t / g.nu, uu = t - bp * g.nu;
        const int b1 = bp / g.N, b2 = bp % g.N;
        const int lu = g.umap ? g.umap[uu] : uu;
        const int u = g.unit0 + lu;
        const int a1 = (u / g.N) % g.N, a2 = u % g.N;
        const float* ker = a.in + (size_t)lu * g.kh * g.kw;
        float v = 0.0f;
        for (int w1 = 0; w1 < 2; ++w1) {
            const int k1 = b1 - a1 + g.ch + g.N * (w1 ? i - g.Lh : i);
            if (k1 < 0 || k1 >= g.kh) continue;
            for (int w2 = 0; w2 < 2; ++w2) {
                const int k2 = b2 - a2 + g.cw + g.N * (w2 ? j - g.Lw : j);
                if (k2 < 0 || k2 >= g.kw) continue;
                v += ker[(size_t)k1 * g.kw + k2];
            }
        }
        return v;
    }

}

// UBV images per CTA (FastGeom<L>::UB by default; 1 when a launch has fewer transforms than would fill the chip)
template <int L, int SRC, int UBV>
__global__ void __launch_bounds__(512, LFM_FFT_MINB) r2c_fast_kernel(XformGeom g, const float2* __restrict__ twg, R2CArgs a) {
    using FG = FastGeom<L>;
    constexpr int NK2 = FG::NK2, RHO = FG::RHO, S = FG::S, NBL = FG::NBL, UB = UBV;
    constexpr int PW = has_pair_stage<L>() ? 2 : 1;   // transforms per warp in the row / column phases
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* buf = sm + L + (L & 1);   // keep 16-byte alignment
    for (int i = threadIdx.x; i < L; i += blockDim.x) tw[i] = twg[i];
    const int t0 = blockIdx.x * UB;
    const int nt = min(UB, a.ntrans - t0);
    constexpr bool full = (SRC == SRC_KERNEL);
    const int nrows = full ? L : g.nh;
    const int ncols = full ? L : g.nw;
    const int P = (nrows + 1) / 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;

    // 1. packed rows (row 2pr in re, 2pr+1 in im) at buf[ui*S + pr*2*RHO + col]; unpacked rows >= 2P are zero.
    //    One warp per packed row.  Strided sources: per-unit base offsets are resolved once (umap) and the row
    //    elements go global -> shared by cp.async, so every lane keeps all its rows' loads in flight at once.
    __shared__ long long s_base[UB];
    if constexpr (strided_src<SRC>()) {
        if (threadIdx.x < nt) s_base[threadIdx.x] = src_base<SRC>(g, t0 + threadIdx.x);
        __syncthreads();
        const long long rp = (SRC == SRC_POLY) ? (long long)g.nw : (long long)g.N * g.W;
        const int cs = (SRC == SRC_POLY) ? 1 : g.N;
        for (int row = warp; row < nt * P; row += nwarps) {
            const int ui = row / P;
            const int pr = row - ui * P;
            float2* dst = buf + ui * S + pr * 2 * RHO;
            const bool two = (2 * pr + 1 < nrows);
            const long long o0 = s_base[ui] + 2 * pr * rp;
            if constexpr (SRC == SRC_RATIO) {
                float y0[NBL], y1[NBL], h0[NBL], h1[NBL];
#pragma unroll
                for (int t = 0; t < NBL; ++t) {
                    const int col = lane + 32 * t;
                    y0[t] = y1[t] = h0[t] = h1[t] = 0.0f;
                    if (col < ncols) {
                        y0[t] = a.in[o0 + (long long)col * cs];
                        h0[t] = a.in2[o0 + (long long)col * cs];
                        if (two) {
                            y1[t] = a.in[o0 + rp + (long long)col * cs];
                            h1[t] = a.in2[o0 + rp + (long long)col * cs];
                        }
                    }
                }
#pragma unroll
                for (int t = 0; t < NBL; ++t) {
                    const int col = lane + 32 * t;
                    if (col < L) {
                        float re = 0.0f, im = 0.0f;
                        if (col < ncols) {
                            re = y0[t] / (fmaxf(h0[t], 0.0f) + a.eps);
                            if (two) im = y1[t] / (fmaxf(h1[t], 0.0f) + a.eps);
                        }
                        dst[col] = make_float2(re, im);
                    }
                }
            } else {
#pragma unroll
                for (int t = 0; t < NBL; ++t) {
                    const int col = lane + 32 * t;
                    if (col < L) {
                        if (col < ncols) {
                            cp_async4(&dst[col].x, a.in + o0 + (long long)col * cs);
                            if (two)
                                cp_async4(&dst[col].y, a.in + o0 + rp + (long long)col * cs);
                            else
                                dst[col].y = 0.0f;
                        } else {
                            dst[col] = make_float2(0.0f, 0.0f);
                        }
                    }
                }
            }
        }
        cp_async_wait_all();
    } else
    for (int row = warp; row < nt * P; row += nwarps) {
        const int ui = row / P;
        const int pr = row - ui * P;
        float2* dst = buf + ui * S + pr * 2 * RHO;
        const bool two = (2 * pr + 1 < nrows);
        for (int col = lane; col < L; col += 32) {
            float re = 0.0f, im = 0.0f;
            if (col < ncols) {
                re = src_value<SRC>(g, a, t0 + ui, 2 * pr, col);
                if (two) im = src_value<SRC>(g, a, t0 + ui, 2 * pr + 1, col);
            }
            dst[col] = make_float2(re, im);
        }
    }
    const int zr = L - 2 * P;
    if (zr > 0) {
        const int per = zr * NK2;
        const int nz_ = nt * per;
        for (int idx = threadIdx.x; idx < nz_; idx += blockDim.x) {
            const int ui = idx / (per > 0 ? per : 1);
            const int rem = idx - ui * per;
            const int r = rem / NK2;
            const int k = rem - r * NK2;
            buf[ui * S + (2 * P + r) * RHO + k] = make_float2(0.0f, 0.0f);
        }
    }
    __syncthreads();
    // 2. per warp: row FFT of a packed pair, then the Hermitian split in place into rows 2pr, 2pr+1
    for (int tp = PW * warp; tp < nt * P; tp += PW * nwarps) {
        const int ntr = min(PW, nt * P - tp);
        int prs[2];
        float2* rows[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int tr = tp + (h < ntr ? h : 0);
            const int ui = tr / P;
            prs[h] = tr - ui * P;
            rows[h] = buf + ui * S + prs[h] * 2 * RHO;
        }
        warp_fft2<L, 0, 1, false>(rows[0], rows[PW - 1], 1, tw, lane);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (h >= ntr) break;
            float2* row = rows[h];
            const int pr = prs[h];
            float2 Z[NBL], Q[NBL];
#pragma unroll
            for (int t = 0; t < NBL; ++t) {
                const int k = lane + 32 * t;
                if (k < NK2) {
                    Z[t] = row[k];
                    Q[t] = row[k == 0 ? 0 : L - k];
                }
            }
            __syncwarp();
#pragma unroll
            for (int t = 0; t < NBL; ++t) {
                const int k = lane + 32 * t;
                if (k < NK2) {
                    const float2 q = make_float2(Q[t].x, -Q[t].y);   // conj(Z[-k])
                    row[k] = make_float2(0.5f * (Z[t].x + q.x), 0.5f * (Z[t].y + q.y));
                    if (2 * pr + 1 < L) row[RHO + k] = make_float2(0.5f * (Z[t].y - q.y), -0.5f * (Z[t].x - q.x));
                }
            }
            __syncwarp();
        }
    }
    __syncthreads();
    // 3. column FFTs (stride RHO)
    for (int tp = PW * warp; tp < nt * NK2; tp += PW * nwarps) {
        const int tq = min(tp + PW - 1, nt * NK2 - 1);
        const int ui0 = tp / NK2, ui1 = tq / NK2;
        warp_fft2<L, 0, 1, false>(buf + ui0 * S + (tp - ui0 * NK2), buf + ui1 * S + (tq - ui1 * NK2), RHO, tw, lane);
    }
    __syncthreads();
    // 4. kappa-major store, UB units contiguous per kappa (UB compile-time: no run-time division)
    __shared__ long long s_col[UB];
    if (threadIdx.x < UB) {
        const int t = t0 + threadIdx.x;
        const int q = t / a.cdiv;
        s_col[threadIdx.x] = (long long)q * a.cmul + (t - q * a.cdiv);
    }
    __syncthreads();
    constexpr int NKAP = L * NK2;
    for (int idx = threadIdx.x; idx < NKAP * UB; idx += blockDim.x) {
        const int kap = idx / UB;
        const int ui = idx - kap * UB;
        if (ui >= nt) continue;
        const int k1 = kap / NK2;
        const int k2 = kap - k1 * NK2;
        a.out[(long long)kap * a.out_ld + s_col[ui]] = buf[ui * S + k1 * RHO + k2];
    }
}

template <int L, int DST, int UBV>
__global__ void __launch_bounds__(512, LFM_FFT_MINB) c2r_fast_kernel(XformGeom g, const float2* __restrict__ twg, C2RArgs a) {
    using FG = FastGeom<L>;
    constexpr int NK2 = FG::NK2, RHO = FG::RHO, S = FG::S, NBL = FG::NBL, UB = UBV;
    constexpr int PW = has_pair_stage<L>() ? 2 : 1;   // transforms per warp in the row / column phases
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* buf = sm + L + (L & 1);
    for (int i = threadIdx.x; i < L; i += blockDim.x) tw[i] = twg[i];
    const int t0 = blockIdx.x * UB;
    const int nt = min(UB, a.ntrans - t0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    constexpr int NKAP = L * NK2;
    // 1. gather spectra into rows k1 (stride RHO); UB consecutive units per kappa
    for (int idx = threadIdx.x; idx < NKAP * UB; idx += blockDim.x) {
        const int kap = idx / UB;
        const int ui = idx - kap * UB;
        if (ui >= nt) continue;
        const int k1 = kap / NK2;
        const int k2 = kap - k1 * NK2;
        cp_async8(&buf[ui * S + k1 * RHO + k2], &a.in[(long long)kap * a.in_ld + t0 + ui]);
    }
    __shared__ int s_lu[UB];   // local unit of each transform (DST_POLY / VOLIMAGE / UPDATE / ISRA)
    if (threadIdx.x < nt) s_lu[threadIdx.x] = g.umap ? g.umap[t0 + threadIdx.x] : t0 + threadIdx.x;
    cp_async_wait_all();
    __syncthreads();
    // 2. inverse column FFTs
    for (int tp = PW * warp; tp < nt * NK2; tp += PW * nwarps) {
        const int tq = min(tp + PW - 1, nt * NK2 - 1);
        const int ui0 = tp / NK2, ui1 = tq / NK2;
        warp_fft2<L, 0, 1, true>(buf + ui0 * S + (tp - ui0 * NK2), buf + ui1 * S + (tq - ui1 * NK2), RHO, tw, lane);
    }
    __syncthreads();
    // 3. per warp and packed row pair: Hermitian row rebuild, inverse row FFT, crop / scale / epilogue
    const int nh = g.nh, nw = g.nw;
    const int P = (nh + 1) / 2;
    const float scale = 1.0f / (float)(L * L);
    for (int tp = PW * warp; tp < nt * P; tp += PW * nwarps) {
        const int ntr = min(PW, nt * P - tp);
        int uis[2], prs[2];
        float2* rows[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int tr = tp + (h < ntr ? h : 0);
            uis[h] = tr / P;
            prs[h] = tr - uis[h] * P;
            rows[h] = buf + uis[h] * S + prs[h] * 2 * RHO;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (h >= ntr) break;
            float2* row = rows[h];
            const bool has1 = (2 * prs[h] + 1 < nh);
            float2 Z[NBL];
#pragma unroll
            for (int t = 0; t < NBL; ++t) {
                const int k = lane + 32 * t;
                if (k < L) {
                    const bool mirror = (k >= NK2);
                    const int kk = mirror ? L - k : k;
                    float2 A0 = row[kk];
                    float2 A1 = has1 ? row[RHO + kk] : make_float2(0.0f, 0.0f);
                    if (mirror) {
                        A0.y = -A0.y;
                        A1.y = -A1.y;
                    }
                    if (k == 0 || 2 * k == L) {
                        A0.y = 0.0f;
                        A1.y = 0.0f;
                    }
                    Z[t] = make_float2(A0.x - A1.y, A0.y + A1.x);
                }
            }
            __syncwarp();
#pragma unroll
            for (int t = 0; t < NBL; ++t) {
                const int k = lane + 32 * t;
                if (k < L) row[k] = Z[t];
            }
            __syncwarp();
        }
        warp_fft2<L, 0, 1, true>(rows[0], rows[PW - 1], 1, tw, lane);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            if (hh >= ntr) break;
            const float2* row = rows[hh];
            const int pr = prs[hh];
            const bool has1 = (2 * pr + 1 < nh);
            const int t = t0 + uis[hh];
            if constexpr (DST == DST_UPDATE || DST == DST_ISRA) {
                // all of the row pair's x_old / aux loads first, then the update and the stores
                const size_t base = ((size_t)s_lu[uis[hh]] * nh + 2 * pr) * nw;
                float xo[NBL][2], ax[NBL][2];
#pragma unroll
                for (int c = 0; c < NBL; ++c) {
                    const int j = lane + 32 * c;
                    xo[c][0] = xo[c][1] = ax[c][0] = ax[c][1] = 0.0f;
                    if (j < nw) {
                        xo[c][0] = a.xold[base + j];
                        ax[c][0] = a.norm[base + j];
                        if (has1) {
                            xo[c][1] = a.xold[base + nw + j];
                            ax[c][1] = a.norm[base + nw + j];
                        }
                    }
                }
#pragma unroll
                for (int c = 0; c < NBL; ++c) {
                    const int j = lane + 32 * c;
                    if (j < nw) {
                        const float2 zz = row[j];
                        a.out[base + j] = update_value<DST>(xo[c][0], ax[c][0], zz.x * scale, a.eps);
                        if (has1) a.out[base + nw + j] = update_value<DST>(xo[c][1], ax[c][1], zz.y * scale, a.eps);
                    }
                }
            } else {
                for (int j = lane; j < nw; j += 32) {
                    const float2 zz = row[j];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (h == 1 && !has1) break;
                        const int i = 2 * pr + h;
                        const float v = (h ? zz.y : zz.x) * scale;
                        if constexpr (DST == DST_IMAGE) {
                            const int b1 = t / g.N, b2 = t % g.N;
                            a.out[(size_t)(b1 + g.N * i) * g.W + b2 + g.N * j] = v;
                        } else if constexpr (DST == DST_POLY) {
                            a.out[((size_t)s_lu[uis[hh]] * nh + i) * nw + j] = v;
                        } else {
                            const int u = g.unit0 + s_lu[uis[hh]];
                            const int N2 = g.N * g.N;
                            const int z = u / N2, a1 = (u / g.N) % g.N, a2 = u % g.N;
                            a.out[((size_t)z * g.H + a1 + g.N * i) * g.W + a2 + g.N * j] = v;
                        }
                    }
                }
            }
        }
    }
}

template <int L, int SRC, int UBV>
static cudaError_t r2c_fast_go(const XformGeom& g, const float2* tw, const R2CArgs& a, cudaStream_t s) {
    const size_t smem = FastGeom<L>::smem_for(UBV);
    cudaError_t e = cudaFuncSetAttribute(r2c_fast_kernel<L, SRC, UBV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    r2c_fast_kernel<L, SRC, UBV><<<(unsigned)((a.ntrans + UBV - 1) / UBV), 512, smem, s>>>(g, tw, a);
    return cudaGetLastError();
}

template <int L, int DST, int UBV>
static cudaError_t c2r_fast_go(const XformGeom& g, const float2* tw, const C2RArgs& a, cudaStream_t s) {
    const size_t smem = FastGeom<L>::smem_for(UBV);
    cudaError_t e = cudaFuncSetAttribute(c2r_fast_kernel<L, DST, UBV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    c2r_fast_kernel<L, DST, UBV><<<(unsigned)((a.ntrans + UBV - 1) / UBV), 512, smem, s>>>(g, tw, a);
    return cudaGetLastError();
}

// one image per CTA when the default packing would leave most SMs idle (the N^2 output-phase transforms)
constexpr int kFewTransforms = 2 * 148;

template <int L>
static cudaError_t r2c_fast_L(const XformGeom& g, const float2* tw, const R2CArgs& a, cudaStream_t s) {
    constexpr int UB = FastGeom<L>::UB;
    const bool few = UB > 1 && (a.ntrans + UB - 1) / UB < kFewTransforms;
    switch (a.src) {
        case SRC_POLY: return r2c_fast_go<L, SRC_POLY, UB>(g, tw, a, s);
        case SRC_IMAGE: return r2c_fast_go<L, SRC_IMAGE, UB>(g, tw, a, s);
        case SRC_KERNEL: return r2c_fast_go<L, SRC_KERNEL, UB>(g, tw, a, s);
        case SRC_RATIO: return few ? r2c_fast_go<L, SRC_RATIO, 1>(g, tw, a, s) : r2c_fast_go<L, SRC_RATIO, UB>(g, tw, a, s);
        case SRC_ONES: return few ? r2c_fast_go<L, SRC_ONES, 1>(g, tw, a, s) : r2c_fast_go<L, SRC_ONES, UB>(g, tw, a, s);
        case SRC_IMAGE2D:
            return few ? r2c_fast_go<L, SRC_IMAGE2D, 1>(g, tw, a, s) : r2c_fast_go<L, SRC_IMAGE2D, UB>(g, tw, a, s);
        default: return cudaErrorInvalidValue;
    }
}

template <int L>
static cudaError_t c2r_fast_L(const XformGeom& g, const float2* tw, const C2RArgs& a, cudaStream_t s) {
    constexpr int UB = FastGeom<L>::UB;
    const bool few = UB > 1 && (a.ntrans + UB - 1) / UB < kFewTransforms;
    switch (a.dst) {
        case DST_IMAGE: return few ? c2r_fast_go<L, DST_IMAGE, 1>(g, tw, a, s) : c2r_fast_go<L, DST_IMAGE, UB>(g, tw, a, s);
        case DST_POLY: return c2r_fast_go<L, DST_POLY, UB>(g, tw, a, s);
        case DST_VOLIMAGE: return c2r_fast_go<L, DST_VOLIMAGE, UB>(g, tw, a, s);
        case DST_UPDATE: return c2r_fast_go<L, DST_UPDATE, UB>(g, tw, a, s);
        case DST_ISRA: return c2r_fast_go<L, DST_ISRA, UB>(g, tw, a, s);
        default: return cudaErrorInvalidValue;
    }
}

bool fast_fft_size(int Lh, int Lw) {
    return Lh == Lw && (Lh == 15 || Lh == 16 || Lh == 36 || Lh == 75 || Lh == 144);
}

cudaError_t launch_r2c_fast(const XformGeom& g, const float2* tw, const R2CArgs& a, cudaStream_t s) {
    switch (g.Lh) {
        case 15: return r2c_fast_L<15>(g, tw, a, s);
        case 16: return r2c_fast_L<16>(g, tw, a, s);
        case 36: return r2c_fast_L<36>(g, tw, a, s);
        case 75: return r2c_fast_L<75>(g, tw, a, s);
        case 144: return r2c_fast_L<144>(g, tw, a, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_c2r_fast(const XformGeom& g, const float2* tw, const C2RArgs& a, cudaStream_t s) {
    switch (g.Lh) {
        case 15: return c2r_fast_L<15>(g, tw, a, s);
        case 16: return c2r_fast_L<16>(g, tw, a, s);
        case 36: return c2r_fast_L<36>(g, tw, a, s);
        case 75: return c2r_fast_L<75>(g, tw, a, s);
        case 144: return c2r_fast_L<144>(g, tw, a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lfm
