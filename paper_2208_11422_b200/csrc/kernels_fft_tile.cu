// kernels_fft_tile.cu -- coarse transforms of the overlap-save tiled frequency path.
//
// The whole-image frequency path transforms every coarse image once on an Lc x Lc grid (Lc >= n + ceil(c/N)) and
// streams transfer matrices of Lc x (Lc/2+1) frequencies per (output phase, unit).  The tiled path cuts the coarse grid
// into T1 x T2 tiles and transforms a window of L x L coarse pixels per (tile, item) instead, L = T + (dmax - dmin)
// (the span of the coarse taps): the linear convolution of the window with any pair's coarse kernel is exact on the
// tile's T1 x T2 valid outputs (overlap-save).  The transfer matrices shrink to L x (L/2+1) frequencies and every
// matrix element serves all tiles in one pass (the tiles are the N of a GEMM), at the price of transforming the
// overlap.  Forward (§2.2 forwardProject):
//   y_b'[m] = sum_a sum_d k_ab'[d] x_a[m - d]:  window w[i] = x_a[tile*T - dmax + i], y_b'[tile*T + j] = z[dmax + j];
// backward (the adjoint, conj M):
//   x_a[n] = sum_b' sum_d k_ab'[d] r_b'[n + d]: window w[i] = r_b'[tile*T + dmin + i], x_a[tile*T + j] = z[-dmin + j].
// Window pixels outside the coarse image are zeros.  Same shared-memory layout and warp radix stages as the
// whole-image kernels (kernels_fft_fast.cu); every row of the window is present (no zero rows beyond n).
#include <cmath>
#include <cstdlib>

#include "fft_warp.cuh"

namespace lfm {

namespace {

// element offset of item t's coarse image origin and its (row pitch, column stride), as the whole-image kernels
template <int SRC>
__device__ __forceinline__ long long tile_src_base(const XformGeom& g, int item) {
    if constexpr (SRC == SRC_POLY) {
        return (long long)(g.umap ? g.umap[item] : item) * g.nh * g.nw;
    } else if constexpr (SRC == SRC_IMAGE) {
        const int u = g.unit0 + (g.umap ? g.umap[item] : item);
        const int N2 = g.N * g.N;
        const int z = u / N2, a1 = (u / g.N) % g.N, a2 = u % g.N;
        return ((long long)z * g.H + a1) * g.W + a2;
    } else if constexpr (SRC == SRC_ONES) {
        return 0;
    } else {   // IMAGE2D, RATIO: item = output phase (b1, b2)
        return (long long)(item / g.N) * g.W + item % g.N;
    }
}

__device__ __forceinline__ void cp_async4_zfill(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src),
                 "r"(valid ? 4 : 0)
                 : "memory");
}

}  // namespace

template <int L, int SRC, int UBV>
__global__ void __launch_bounds__(512, LFM_FFT_MINB) r2c_tile_kernel(XformGeom g, TileGeom tg, const float2* __restrict__ twg,
                                                                     R2CArgs a, int o1, int o2, unsigned* __restrict__ amax) {
    using FG = FastGeom<L>;
    constexpr int NK2 = FG::NK2, RHO = FG::RHO, S = FG::S, NBL = FG::NBL, UB = UBV;
    constexpr int PW = has_pair_stage<L>() ? 2 : 1;
    constexpr int P = (L + 1) / 2;   // packed row pairs: every window row is present
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* buf = sm + L + (L & 1);
    for (int i = threadIdx.x; i < L; i += blockDim.x) tw[i] = twg[i];
    const int t0 = blockIdx.x * UB;
    const int nt = min(UB, a.ntrans - t0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    __shared__ long long s_base[UB], s_col[UB];
    __shared__ int s_r0[UB], s_c0[UB], s_tile[UB];
    __shared__ float s_rsum[UB][P];   // sum |window| per packed row pair (summed in row order: deterministic)
    if (threadIdx.x < nt) {
        const int t = t0 + threadIdx.x;
        const int tile = t / a.cdiv, item = t - tile * a.cdiv;
        const int ty = tile / tg.ntx, tx = tile - ty * tg.ntx;
        s_base[threadIdx.x] = tile_src_base<SRC>(g, item);
        s_col[threadIdx.x] = (long long)tile * a.cmul + item;
        s_r0[threadIdx.x] = ty * tg.T1 + o1;
        s_c0[threadIdx.x] = tx * tg.T2 + o2;
        s_tile[threadIdx.x] = tile;
    }
    __syncthreads();
    const long long rp = (SRC == SRC_POLY) ? (long long)g.nw : (long long)g.N * g.W;
    const int cs = (SRC == SRC_POLY) ? 1 : g.N;
    // 1. packed window rows (row 2pr in re, 2pr+1 in im), zero outside the coarse image; one warp per row pair
    for (int row = warp; row < nt * P; row += nwarps) {
        const int ui = row / P;
        const int pr = row - ui * P;
        float2* dst = buf + ui * S + pr * 2 * RHO;
        const int gr0 = s_r0[ui] + 2 * pr, gr1 = gr0 + 1;
        const bool v0 = gr0 >= 0 && gr0 < g.nh;
        const bool v1 = (2 * pr + 1 < L) && gr1 >= 0 && gr1 < g.nh;
        const long long o0 = s_base[ui] + (long long)gr0 * rp;
#pragma unroll
        for (int t = 0; t < NBL; ++t) {
            const int col = lane + 32 * t;
            if (col < L) {
                const int gc = s_c0[ui] + col;
                const bool vc = gc >= 0 && gc < g.nw;
                if constexpr (SRC == SRC_ONES) {
                    dst[col] = make_float2(v0 && vc ? 1.0f : 0.0f, v1 && vc ? 1.0f : 0.0f);
                } else if constexpr (SRC == SRC_RATIO) {
                    float re = 0.0f, im = 0.0f;
                    if (vc && v0) {
                        const long long q = o0 + (long long)gc * cs;
                        re = a.in[q] / (fmaxf(a.in2[q], 0.0f) + a.eps);
                    }
                    if (vc && v1) {
                        const long long q = o0 + rp + (long long)gc * cs;
                        im = a.in[q] / (fmaxf(a.in2[q], 0.0f) + a.eps);
                    }
                    dst[col] = make_float2(re, im);
                } else {
                    const float* p0 = a.in + (vc && v0 ? o0 + (long long)gc * cs : 0);
                    const float* p1 = a.in + (vc && v1 ? o0 + rp + (long long)gc * cs : 0);
                    cp_async4_zfill(&dst[col].x, p0, vc && v0);
                    cp_async4_zfill(&dst[col].y, p1, vc && v1);
                }
            }
        }
    }
    cp_async_wait_all();
    __syncthreads();
    // 2. per warp: sum |window| (scale bound of the tile MACs), row FFT of a packed pair, Hermitian split in place
    for (int tp = PW * warp; tp < nt * P; tp += PW * nwarps) {
        const int ntr = min(PW, nt * P - tp);
        int prs[2], uis[2];
        float2* rows[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int tr = tp + (h < ntr ? h : 0);
            uis[h] = tr / P;
            prs[h] = tr - uis[h] * P;
            rows[h] = buf + uis[h] * S + prs[h] * 2 * RHO;
        }
        if (amax) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h >= ntr) break;
                float sacc = 0.0f;
                for (int col = lane; col < L; col += 32) sacc += fabsf(rows[h][col].x) + fabsf(rows[h][col].y);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
                if (lane == 0) s_rsum[uis[h]][prs[h]] = sacc;
            }
            __syncwarp();
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
    if (amax && threadIdx.x < nt) {
        float sum = 0.0f;
        for (int pr = 0; pr < P; ++pr) sum += s_rsum[threadIdx.x][pr];
        atomicMax(amax + s_tile[threadIdx.x], __float_as_uint(sum));   // max: order-independent
    }
    // 3. column FFTs (stride RHO)
    for (int tp = PW * warp; tp < nt * NK2; tp += PW * nwarps) {
        const int tq = min(tp + PW - 1, nt * NK2 - 1);
        const int ui0 = tp / NK2, ui1 = tq / NK2;
        warp_fft2<L, 0, 1, false>(buf + ui0 * S + (tp - ui0 * NK2), buf + ui1 * S + (tq - ui1 * NK2), RHO, tw, lane);
    }
    __syncthreads();
    // 4. kappa-major store, UB transforms per kappa
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
__global__ void __launch_bounds__(512, LFM_FFT_MINB) c2r_tile_kernel(XformGeom g, TileGeom tg, const float2* __restrict__ twg,
                                                                     C2RArgs a, int j1, int j2) {
    using FG = FastGeom<L>;
    constexpr int NK2 = FG::NK2, RHO = FG::RHO, S = FG::S, NBL = FG::NBL, UB = UBV;
    constexpr int PW = has_pair_stage<L>() ? 2 : 1;
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* buf = sm + L + (L & 1);
    for (int i = threadIdx.x; i < L; i += blockDim.x) tw[i] = twg[i];
    const int t0 = blockIdx.x * UB;
    const int nt = min(UB, a.ntrans - t0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    constexpr int NKAP = L * NK2;
    __shared__ long long s_col[UB], s_ob[UB];
    __shared__ int s_m1[UB], s_m2[UB];
    if (threadIdx.x < nt) {
        const int t = t0 + threadIdx.x;
        const int tile = t / a.cdiv, item = t - tile * a.cdiv;
        const int ty = tile / tg.ntx, tx = tile - ty * tg.ntx;
        const int m1 = ty * tg.T1, m2 = tx * tg.T2;
        s_col[threadIdx.x] = (long long)tile * a.cmul + item;
        s_m1[threadIdx.x] = m1;
        s_m2[threadIdx.x] = m2;
        // destination offset of the window's first valid output (m1, m2), as the register kernel's prologue
        if constexpr (DST == DST_IMAGE) {
            const int b1 = item / g.N, b2 = item - (item / g.N) * g.N;
            s_ob[threadIdx.x] = (long long)(b1 + g.N * m1) * g.W + b2 + g.N * m2;
        } else if constexpr (DST == DST_VOLIMAGE) {
            const int u = g.unit0 + (g.umap ? g.umap[item] : item);
            const int N2 = g.N * g.N;
            const int z = u / N2, a1 = (u / g.N) % g.N, a2 = u % g.N;
            s_ob[threadIdx.x] = ((long long)z * g.H + a1 + g.N * m1) * g.W + a2 + g.N * m2;
        } else {
            const int lu = g.umap ? g.umap[item] : item;
            s_ob[threadIdx.x] = ((long long)lu * g.nh + m1) * g.nw + m2;
        }
    }
    __syncthreads();
    const long long ors = (DST == DST_IMAGE || DST == DST_VOLIMAGE) ? (long long)g.N * g.W : (long long)g.nw;
    const int ocs = (DST == DST_IMAGE || DST == DST_VOLIMAGE) ? g.N : 1;
    // 1. gather spectra into rows k1 (stride RHO)
    for (int idx = threadIdx.x; idx < NKAP * UB; idx += blockDim.x) {
        const int kap = idx / UB;
        const int ui = idx - kap * UB;
        if (ui >= nt) continue;
        const int k1 = kap / NK2;
        const int k2 = kap - k1 * NK2;
        const float2* src = &a.in[(long long)kap * a.in_ld + s_col[ui]];
        if (a.nsum > 1) {   // split-K partial spectra, summed in split order
            float2 v = src[0];
            for (int sp = 1; sp < a.nsum; ++sp) v = c_add(v, src[sp * a.in_sstride]);
            buf[ui * S + k1 * RHO + k2] = v;
        } else {
            cp_async8(&buf[ui * S + k1 * RHO + k2], src);
        }
    }
    cp_async_wait_all();
    __syncthreads();
    // 2. inverse column FFTs
    for (int tp = PW * warp; tp < nt * NK2; tp += PW * nwarps) {
        const int tq = min(tp + PW - 1, nt * NK2 - 1);
        const int ui0 = tp / NK2, ui1 = tq / NK2;
        warp_fft2<L, 0, 1, true>(buf + ui0 * S + (tp - ui0 * NK2), buf + ui1 * S + (tq - ui1 * NK2), RHO, tw, lane);
    }
    __syncthreads();
    // 3. the packed row pairs that hold valid rows j1 .. j1 + T1 - 1: Hermitian rebuild, inverse row FFT, epilogue
    const int pr_lo = j1 >> 1, npr = ((j1 + tg.T1 - 1) >> 1) - pr_lo + 1;
    const float scale = 1.0f / (float)(L * L);
    for (int tp = PW * warp; tp < nt * npr; tp += PW * nwarps) {
        const int ntr = min(PW, nt * npr - tp);
        int uis[2], prs[2];
        float2* rows[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int tr = tp + (h < ntr ? h : 0);
            uis[h] = tr / npr;
            prs[h] = pr_lo + tr - uis[h] * npr;
            rows[h] = buf + uis[h] * S + prs[h] * 2 * RHO;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (h >= ntr) break;
            float2* row = rows[h];
            const bool has1 = (2 * prs[h] + 1 < L);
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
            const int ui = uis[hh];
            for (int c = lane; c < tg.T2; c += 32) {
                const int m2 = s_m2[ui] + c;
                if (m2 >= g.nw) continue;
                const float2 zz = row[j2 + c];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int i = 2 * prs[hh] + h;   // window row
                    if (i < j1 || i >= j1 + tg.T1 || i >= L) continue;
                    const int m1 = s_m1[ui] + i - j1;
                    if (m1 >= g.nh) continue;
                    const float v = (h ? zz.y : zz.x) * scale;
                    const long long q = s_ob[ui] + (long long)(i - j1) * ors + (long long)c * ocs;
                    if constexpr (DST == DST_IMAGE) {
                        float* o = a.out + q;
                        *o = a.accum ? *o + v : v;
                    } else if constexpr (DST == DST_VOLIMAGE || DST == DST_POLY) {
                        a.out[q] = v;
                    } else {
                        a.out[q] = update_value<DST>(a.xold[q], a.norm[q], v, a.eps);
                    }
                }
            }
        }
    }
}

// ================================================================================================================
// Register-resident variant (default).  One thread owns one whole 1-D transform: it loads the L points from shared
// memory, runs every radix stage in registers (compile-time indices after unrolling, twiddles from a __constant__
// table, trivial ones skipped) and writes the result once -- two shared-memory passes per 2-D transform instead of two
// per radix stage, and no per-stage __syncwarp.  Layout per image (UB images per CTA):
//   real window rows in two planes (row 2pr -> plane 0 row pr, row 2pr+1 -> plane 1 row pr; odd row pitch RP);
//   spectrum rows (Hermitian half, NK2 columns) in two planes the same way (odd pitch CP, odd image stride CIMG), so
//   the threads of a warp -- consecutive packed rows, or consecutive images of one column -- hit distinct banks.
// R2C: stage A global -> real planes (cp.async, zero-fill outside the coarse image); stage B per packed row pair: row
// FFT of x[2pr] + i x[2pr+1], Hermitian split into the two spectrum rows, sum |x|; stage C per (column k, image):
// column FFT, stored straight to out[kappa * ld + col] (consecutive threads = consecutive images = consecutive cols).
// C2R: stage A per (column, image): load from global, inverse column FFT, to the spectrum planes; stage B per packed
// row pair of the valid rows: Hermitian rebuild, inverse row FFT, valid outputs to shared memory; stage C: the
// destination epilogue over the valid T1 x T2 outputs, consecutive threads on consecutive columns.
// ================================================================================================================
constexpr int kTwTotal = 228;
constexpr int kRegMaxL = 36;               // larger windows (c4: 45) run the warp-per-transform kernels above
__constant__ float2 c_tile_tw[kTwTotal];   // W_L^e = exp(-2 pi i e / L) for every L of tile_fft_size, fp64-rounded

__host__ __device__ constexpr int tw_off(int L) {
    return L == 16 ? 0 : L == 18 ? 16 : L == 20 ? 34 : L == 24 ? 54 : L == 25 ? 78 : L == 27 ? 103 : L == 30 ? 130
         : L == 32 ? 160 : 192;
}

template <int L, bool INV>
__device__ __forceinline__ float2 twl(int e) {
    float2 w = c_tile_tw[tw_off(L) + e];
    if (INV) w.y = -w.y;
    return w;
}

// Stockham stages in registers (the index algebra of warp_stage with the shared buffer replaced by register arrays)
template <int L, int S, int NS, bool INV>
__device__ __forceinline__ void reg_fft_stages(float2 (&a)[L]) {
    constexpr Radices F = factorize(L);
    if constexpr (S < F.n) {
        constexpr int R = F.r[S];
        constexpr int LR = L / R;
        constexpr int TWS = L / (NS * R);
        float2 b[L];
#pragma unroll
        for (int j = 0; j < LR; ++j) {
            const int k = j % NS;
            float2 v[R];
#pragma unroll
            for (int q = 0; q < R; ++q) v[q] = a[j + q * LR];
            if (NS > 1 && k != 0) {
#pragma unroll
                for (int q = 1; q < R; ++q) v[q] = c_mul(v[q], twl<L, INV>(q * k * TWS));
            }
            small_dft<R, INV>(v);
            const int o = (j - k) * R + k;
#pragma unroll
            for (int q = 0; q < R; ++q) b[o + q * NS] = v[q];
        }
#pragma unroll
        for (int i = 0; i < L; ++i) a[i] = b[i];
        reg_fft_stages<L, S + 1, NS * R, INV>(a);
    }
}

// Shared memory per window: one block of BLK floats per packed row pair pr, used in place -- first the two real
// window rows 2pr (floats 0 .. L-1) and 2pr+1 (L .. 2L-1), then (the thread that transformed them overwrites its own
// block) the two Hermitian-half spectrum rows (complex 0 .. NK2-1 and CP .. CP+NK2-1), and in the C2R the two output
// rows again.  Half the shared memory of separate real and spectrum planes; 8 windows per CTA (up to seven CTAs per SM
// at L <= 27: more, smaller CTAs measured 12 % faster than four of 16 windows).
// BLK / 2 and the window stride IMG / 2 are odd (64-bit accesses of consecutive blocks / windows hit distinct banks).
template <int L>
struct RegGeom {
    static constexpr int NK2 = L / 2 + 1;
    static constexpr int P = (L + 1) / 2;
    static constexpr int CP = (NK2 % 2) ? NK2 : NK2 + 1;      // spectrum row pitch within a block (complex)
    static constexpr int BLK0 = (2 * L > 4 * CP ? 2 * L : 4 * CP);
    static constexpr int BLK = ((BLK0 + 1) / 2 % 2) ? (BLK0 + 1) / 2 * 2 : (BLK0 + 1) / 2 * 2 + 2;   // floats, BLK/2 odd
    static constexpr int IMG0 = P * BLK;
    static constexpr int IMG = (IMG0 / 2 % 2) ? IMG0 : IMG0 + 2;   // floats per window, IMG/2 odd
    static constexpr int UB = 8;                                  // windows per CTA
    static constexpr int NT = ((P > NK2 ? P : NK2) * UB + 31) / 32 * 32;
    static constexpr int MINB = L <= 27 ? 7 : 4;                  // resident CTAs per SM (registers, shared memory)
    static constexpr size_t smem() { return (size_t)UB * IMG * 4; }
};

template <int L, int SRC>
__global__ void __launch_bounds__(RegGeom<L>::NT, RegGeom<L>::MINB) r2c_tile_reg_kernel(XformGeom g, TileGeom tg, R2CArgs a, int o1, int o2,
                                                                      unsigned* __restrict__ amax) {
    using RG = RegGeom<L>;
    constexpr int NK2 = RG::NK2, P = RG::P, UB = RG::UB, BLK = RG::BLK, IMG = RG::IMG, CP = RG::CP;
    extern __shared__ float4 smr[];
    float* sm = reinterpret_cast<float*>(smr);   // [UB][P][BLK]
    const int t0 = blockIdx.x * UB;
    const int nt = min(UB, a.ntrans - t0);
    __shared__ long long s_base[UB], s_col[UB];
    __shared__ int s_r0[UB], s_c0[UB], s_tile[UB];
    __shared__ float s_rsum[UB][P];
    if (threadIdx.x < nt) {
        const int t = t0 + threadIdx.x;
        const int tile = t / a.cdiv, item = t - tile * a.cdiv;
        const int ty = tile / tg.ntx, tx = tile - ty * tg.ntx;
        s_base[threadIdx.x] = tile_src_base<SRC>(g, item);
        s_col[threadIdx.x] = (long long)tile * a.cmul + item;
        s_r0[threadIdx.x] = ty * tg.T1 + o1;
        s_c0[threadIdx.x] = tx * tg.T2 + o2;
        s_tile[threadIdx.x] = tile;
    }
    __syncthreads();
    const long long rp = (SRC == SRC_POLY) ? (long long)g.nw : (long long)g.N * g.W;
    const int cs = (SRC == SRC_POLY) ? 1 : g.N;
    // A. window rows 0 .. L-1 -> their blocks (zero outside the coarse image): one warp per window row (ui, i), the
    //    lanes over its columns.  Per lane the column's validity, source pointer and shared-memory offset are set once
    //    per window and then stepped by NW rows (the flat element loop spent a third of this kernel's instructions on
    //    divisions and three shared-memory lookups per element, ncu r02)
    {
        constexpr int NW = RG::NT / 32;
        static_assert(NW <= L, "one wrap of the window-row counter per step");
        const int lane = threadIdx.x & 31;
        const long long rstep = (long long)NW * rp;
        for (int c = lane; c < L; c += 32) {
            int ui = 0, i = threadIdx.x >> 5;
            int gr = s_r0[0] + i;
            int gc = s_c0[0] + c;
            bool cv = gc >= 0 && gc < g.nw;
            long long q = s_base[0] + (long long)gr * rp + (long long)gc * cs;
            float* dwin = sm + c;
            for (;;) {
                float* dst = dwin + (i >> 1) * BLK + (i & 1) * L;
                const bool v = cv && (unsigned)gr < (unsigned)g.nh;
                if constexpr (SRC == SRC_ONES) {
                    *dst = v ? 1.0f : 0.0f;
                } else if constexpr (SRC == SRC_RATIO) {
                    *dst = v ? a.in[q] / (fmaxf(a.in2[q], 0.0f) + a.eps) : 0.0f;
                } else {
                    cp_async4_zfill(dst, a.in + (v ? q : 0), v);
                }
                i += NW;
                gr += NW;
                q += rstep;
                if (i >= L) {
                    i -= L;
                    if (++ui >= nt) break;
                    gr = s_r0[ui] + i;
                    gc = s_c0[ui] + c;
                    cv = gc >= 0 && gc < g.nw;
                    q = s_base[ui] + (long long)gr * rp + (long long)gc * cs;
                    dwin += IMG;
                }
            }
        }
    }
    cp_async_wait_all();
    __syncthreads();
    // B. per thread: its packed row pair x[2pr] + i x[2pr+1], row FFT, Hermitian split back into its own block
    for (int task = threadIdx.x; task < nt * P; task += blockDim.x) {
        const int ui = task / P, pr = task - ui * P;
        float* blk = sm + (size_t)ui * IMG + pr * BLK;
        const bool has1 = 2 * pr + 1 < L;
        float2 z[L];
        float sacc = 0.0f;
#pragma unroll
        for (int c = 0; c < L; ++c) {
            z[c] = make_float2(blk[c], has1 ? blk[L + c] : 0.0f);
            sacc += fabsf(z[c].x) + fabsf(z[c].y);
        }
        s_rsum[ui][pr] = sacc;
        reg_fft_stages<L, 0, 1, false>(z);
        float2* o = reinterpret_cast<float2*>(blk);
#pragma unroll
        for (int k = 0; k < NK2; ++k) {
            const float2 zk = z[k], zm = z[k == 0 ? 0 : L - k];
            const float2 q = make_float2(zm.x, -zm.y);   // conj(Z[-k])
            o[k] = make_float2(0.5f * (zk.x + q.x), 0.5f * (zk.y + q.y));
            o[CP + k] = make_float2(0.5f * (zk.y - q.y), -0.5f * (zk.x - q.x));
        }
    }
    __syncthreads();
    if (amax && threadIdx.x < nt) {
        float sum = 0.0f;
        for (int pr = 0; pr < P; ++pr) sum += s_rsum[threadIdx.x][pr];
        atomicMax(amax + s_tile[threadIdx.x], __float_as_uint(sum));
    }
    // C. column FFTs, stored kappa-major (kappa = k1 * NK2 + k2); row i of column k: block i >> 1, plane i & 1
    for (int task = threadIdx.x; task < NK2 * UB; task += blockDim.x) {
        const int k = task / UB, ui = task - k * UB;
        if (ui >= nt) continue;
        const float2* col = reinterpret_cast<const float2*>(sm + (size_t)ui * IMG) + k;
        float2 z[L];
#pragma unroll
        for (int i = 0; i < L; ++i) z[i] = col[(i >> 1) * (BLK / 2) + (i & 1) * CP];
        reg_fft_stages<L, 0, 1, false>(z);
        float2* out = a.out + s_col[ui] + (long long)k * a.out_ld;
#pragma unroll
        for (int i = 0; i < L; ++i) out[(long long)i * NK2 * a.out_ld] = z[i];
    }
}

template <int L, int DST>
__global__ void __launch_bounds__(RegGeom<L>::NT, RegGeom<L>::MINB) c2r_tile_reg_kernel(XformGeom g, TileGeom tg, C2RArgs a, int j1, int j2) {
    using RG = RegGeom<L>;
    constexpr int NK2 = RG::NK2, UB = RG::UB, BLK = RG::BLK, IMG = RG::IMG, CP = RG::CP;
    extern __shared__ float4 smr[];
    float* sm = reinterpret_cast<float*>(smr);   // [UB][P][BLK]
    const int T1 = tg.T1, T2 = tg.T2;
    const int t0 = blockIdx.x * UB;
    const int nt = min(UB, a.ntrans - t0);
    __shared__ long long s_col[UB], s_ob[UB];
    __shared__ int s_m1[UB], s_m2[UB];
    if (threadIdx.x < nt) {
        const int t = t0 + threadIdx.x;
        const int tile = t / a.cdiv, item = t - tile * a.cdiv;
        const int ty = tile / tg.ntx, tx = tile - ty * tg.ntx;
        const int m1 = ty * T1, m2 = tx * T2;
        s_col[threadIdx.x] = (long long)tile * a.cmul + item;
        s_m1[threadIdx.x] = m1;
        s_m2[threadIdx.x] = m2;
        // destination offset of the window's first valid output (m1, m2); the others follow at ii * rs + cc * cs
        if constexpr (DST == DST_IMAGE) {
            const int b1 = item / g.N, b2 = item - (item / g.N) * g.N;
            s_ob[threadIdx.x] = (long long)(b1 + g.N * m1) * g.W + b2 + g.N * m2;
        } else if constexpr (DST == DST_VOLIMAGE) {
            const int u = g.unit0 + (g.umap ? g.umap[item] : item);
            const int N2 = g.N * g.N;
            const int z = u / N2, a1 = (u / g.N) % g.N, a2 = u % g.N;
            s_ob[threadIdx.x] = ((long long)z * g.H + a1 + g.N * m1) * g.W + a2 + g.N * m2;
        } else {
            const int lu = g.umap ? g.umap[item] : item;
            s_ob[threadIdx.x] = ((long long)lu * g.nh + m1) * g.nw + m2;
        }
    }
    __syncthreads();
    // A. inverse column FFTs straight from global (consecutive threads: consecutive windows of one column)
    for (int task = threadIdx.x; task < NK2 * UB; task += blockDim.x) {
        const int k = task / UB, ui = task - k * UB;
        if (ui >= nt) continue;
        const float2* in = a.in + s_col[ui] + (long long)k * a.in_ld;
        float2 z[L];
#pragma unroll
        for (int i = 0; i < L; ++i) z[i] = in[(long long)i * NK2 * a.in_ld];
        for (int ks = 1; ks < a.nsum; ++ks) {   // split-K partial spectra, summed in split order
            const float2* ins = in + ks * a.in_sstride;
#pragma unroll
            for (int i = 0; i < L; ++i) z[i] = c_add(z[i], ins[(long long)i * NK2 * a.in_ld]);
        }
        reg_fft_stages<L, 0, 1, true>(z);
        float2* col = reinterpret_cast<float2*>(sm + (size_t)ui * IMG) + k;
#pragma unroll
        for (int i = 0; i < L; ++i) col[(i >> 1) * (BLK / 2) + (i & 1) * CP] = z[i];
    }
    __syncthreads();
    // B. the packed row pairs holding valid rows j1 .. j1 + T1 - 1: Hermitian rebuild, inverse row FFT, the two
    //    output rows back into the pair's own block (scaled)
    const int pr_lo = j1 >> 1, npr = ((j1 + T1 - 1) >> 1) - pr_lo + 1;
    const float scale = 1.0f / (float)(L * L);
    for (int task = threadIdx.x; task < nt * npr; task += blockDim.x) {
        const int ui = task / npr, pr = pr_lo + task - ui * npr;
        float* blk = sm + (size_t)ui * IMG + pr * BLK;
        const float2* s0 = reinterpret_cast<const float2*>(blk);
        const float2* s1 = s0 + CP;
        const bool has1 = 2 * pr + 1 < L;
        float2 z[L];
#pragma unroll
        for (int k = 0; k < L; ++k) {
            const bool mirror = k >= NK2;
            const int kk = mirror ? L - k : k;
            float2 A0 = s0[kk];
            float2 A1 = has1 ? s1[kk] : make_float2(0.0f, 0.0f);
            if (mirror) {
                A0.y = -A0.y;
                A1.y = -A1.y;
            }
            if (k == 0 || 2 * k == L) {
                A0.y = 0.0f;
                A1.y = 0.0f;
            }
            z[k] = make_float2(A0.x - A1.y, A0.y + A1.x);
        }
        reg_fft_stages<L, 0, 1, true>(z);
#pragma unroll
        for (int c = 0; c < L; ++c) {
            blk[c] = z[c].x * scale;
            if (has1) blk[L + c] = z[c].y * scale;
        }
    }
    __syncthreads();
    // C. epilogue over the valid outputs: LR lanes per output row (consecutive lanes: consecutive columns), 32 / LR rows
    //    per warp and step, each warp over a contiguous chunk of the CTA's (window, row) list; every lane handles two
    //    of its rows per pass with all global loads issued before the stores (the update's x_old / normaliser loads
    //    were the kernel's top stall, ncu r02), (ui, ii) advance incrementally (no per-element divisions)
    {
        constexpr int NW = RG::NT / 32;
        const int LR = T2 <= 16 ? 16 : 32;
        const int RPW = 32 / LR;
        const int lane = threadIdx.x & 31;
        const int nrows = nt * T1;
        const int chunk = ((nrows + NW - 1) / NW + RPW - 1) / RPW * RPW;
        const int rbeg = (threadIdx.x >> 5) * chunk + lane / LR;
        const int rend = min(nrows, (threadIdx.x >> 5) * chunk + chunk);
        const long long rs = (DST == DST_IMAGE || DST == DST_VOLIMAGE) ? (long long)g.N * g.W : (long long)g.nw;
        const int cst = (DST == DST_IMAGE || DST == DST_VOLIMAGE) ? g.N : 1;
        // output (ui, ii, c): false if outside the image, else its destination offset and value
        auto elem = [&](int ui, int ii, int c, long long& q, float& v) -> bool {
            if (s_m1[ui] + ii >= g.nh || s_m2[ui] + c >= g.nw) return false;
            const int i = j1 + ii;   // window row
            v = sm[(size_t)ui * IMG + (i >> 1) * BLK + (i & 1) * L + j2 + c];
            q = s_ob[ui] + (long long)ii * rs + (long long)c * cst;
            return true;
        };
        for (int c = lane & (LR - 1); c < T2; c += LR) {   // one pass unless T2 > 32
            int r = rbeg;
            int ui = r / T1, ii = r - (r / T1) * T1;
            while (r < rend) {
                int ui2 = ui, ii2 = ii + RPW;   // the lane's next row
                while (ii2 >= T1) {
                    ii2 -= T1;
                    ++ui2;
                }
                long long qa = 0, qb = 0;
                float va = 0.0f, vb = 0.0f;
                const bool oka = elem(ui, ii, c, qa, va);
                const bool okb = r + RPW < rend && elem(ui2, ii2, c, qb, vb);
                if constexpr (DST == DST_UPDATE || DST == DST_ISRA) {
                    float xa = 0.0f, na = 0.0f, xb = 0.0f, nb = 0.0f;
                    if (oka) {
                        xa = a.xold[qa];
                        na = a.norm[qa];
                    }
                    if (okb) {
                        xb = a.xold[qb];
                        nb = a.norm[qb];
                    }
                    if (oka) a.out[qa] = update_value<DST>(xa, na, va, a.eps);
                    if (okb) a.out[qb] = update_value<DST>(xb, nb, vb, a.eps);
                } else if constexpr (DST == DST_IMAGE) {
                    float oa = 0.0f, ob = 0.0f;
                    if (a.accum) {
                        if (oka) oa = a.out[qa];
                        if (okb) ob = a.out[qb];
                    }
                    if (oka) a.out[qa] = a.accum ? oa + va : va;
                    if (okb) a.out[qb] = a.accum ? ob + vb : vb;
                } else {
                    if (oka) a.out[qa] = va;
                    if (okb) a.out[qb] = vb;
                }
                r += 2 * RPW;
                ui = ui2;
                ii = ii2 + RPW;
                while (ii >= T1) {
                    ii -= T1;
                    ++ui;
                }
            }
        }
    }
}

namespace {

template <int L, int SRC>
cudaError_t r2c_tile_go(const XformGeom& g, const TileGeom& tg, const float2* tw, const R2CArgs& a, int o1, int o2,
                        unsigned* amax, cudaStream_t s) {
    constexpr int UB = FastGeom<L>::UB;
    const size_t smem = FastGeom<L>::smem_for(UB);
    cudaError_t e = cudaFuncSetAttribute(r2c_tile_kernel<L, SRC, UB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    r2c_tile_kernel<L, SRC, UB><<<(unsigned)((a.ntrans + UB - 1) / UB), 512, smem, s>>>(g, tg, tw, a, o1, o2, amax);
    return cudaGetLastError();
}

template <int L, int DST>
cudaError_t c2r_tile_go(const XformGeom& g, const TileGeom& tg, const float2* tw, const C2RArgs& a, int j1, int j2,
                        cudaStream_t s) {
    constexpr int UB = FastGeom<L>::UB;
    const size_t smem = FastGeom<L>::smem_for(UB);
    cudaError_t e = cudaFuncSetAttribute(c2r_tile_kernel<L, DST, UB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    c2r_tile_kernel<L, DST, UB><<<(unsigned)((a.ntrans + UB - 1) / UB), 512, smem, s>>>(g, tg, tw, a, j1, j2);
    return cudaGetLastError();
}

// dev A/B LFM_TILE_WARP: the warp-per-transform kernels above instead of the register-resident ones
bool tile_warp_kernels() {
    static const bool v = getenv("LFM_TILE_WARP") != nullptr;
    return v;
}

template <int L, int SRC>
cudaError_t r2c_tile_reg_go(const XformGeom& g, const TileGeom& tg, const R2CArgs& a, int o1, int o2, unsigned* amax,
                            cudaStream_t s) {
    if constexpr (L > kRegMaxL) {
        return cudaErrorInvalidValue;
    } else {
    using RG = RegGeom<L>;
    const size_t smem = RG::smem();
    cudaError_t e = cudaFuncSetAttribute(r2c_tile_reg_kernel<L, SRC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    r2c_tile_reg_kernel<L, SRC><<<(unsigned)((a.ntrans + RG::UB - 1) / RG::UB), RG::NT, smem, s>>>(g, tg, a, o1, o2, amax);
    return cudaGetLastError();
    }
}

template <int L, int DST>
cudaError_t c2r_tile_reg_go(const XformGeom& g, const TileGeom& tg, const C2RArgs& a, int j1, int j2, cudaStream_t s) {
    if constexpr (L > kRegMaxL) {
        return cudaErrorInvalidValue;
    } else {
    using RG = RegGeom<L>;
    const size_t smem = RG::smem();
    cudaError_t e = cudaFuncSetAttribute(c2r_tile_reg_kernel<L, DST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    c2r_tile_reg_kernel<L, DST><<<(unsigned)((a.ntrans + RG::UB - 1) / RG::UB), RG::NT, smem, s>>>(g, tg, a, j1, j2);
    return cudaGetLastError();
    }
}

template <int L>
cudaError_t r2c_tile_L(const XformGeom& g, const TileGeom& tg, const float2* tw, const R2CArgs& a, int o1, int o2,
                       unsigned* amax, cudaStream_t s) {
    if (!tile_warp_kernels() && L <= kRegMaxL) {
        switch (a.src) {
            case SRC_POLY: return r2c_tile_reg_go<L, SRC_POLY>(g, tg, a, o1, o2, amax, s);
            case SRC_IMAGE: return r2c_tile_reg_go<L, SRC_IMAGE>(g, tg, a, o1, o2, amax, s);
            case SRC_RATIO: return r2c_tile_reg_go<L, SRC_RATIO>(g, tg, a, o1, o2, amax, s);
            case SRC_ONES: return r2c_tile_reg_go<L, SRC_ONES>(g, tg, a, o1, o2, amax, s);
            case SRC_IMAGE2D: return r2c_tile_reg_go<L, SRC_IMAGE2D>(g, tg, a, o1, o2, amax, s);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (a.src) {
        case SRC_POLY: return r2c_tile_go<L, SRC_POLY>(g, tg, tw, a, o1, o2, amax, s);
        case SRC_IMAGE: return r2c_tile_go<L, SRC_IMAGE>(g, tg, tw, a, o1, o2, amax, s);
        case SRC_RATIO: return r2c_tile_go<L, SRC_RATIO>(g, tg, tw, a, o1, o2, amax, s);
        case SRC_ONES: return r2c_tile_go<L, SRC_ONES>(g, tg, tw, a, o1, o2, amax, s);
        case SRC_IMAGE2D: return r2c_tile_go<L, SRC_IMAGE2D>(g, tg, tw, a, o1, o2, amax, s);
        default: return cudaErrorInvalidValue;
    }
}

template <int L>
cudaError_t c2r_tile_L(const XformGeom& g, const TileGeom& tg, const float2* tw, const C2RArgs& a, int j1, int j2,
                       cudaStream_t s) {
    if (!tile_warp_kernels() && L <= kRegMaxL) {
        switch (a.dst) {
            case DST_IMAGE: return c2r_tile_reg_go<L, DST_IMAGE>(g, tg, a, j1, j2, s);
            case DST_POLY: return c2r_tile_reg_go<L, DST_POLY>(g, tg, a, j1, j2, s);
            case DST_VOLIMAGE: return c2r_tile_reg_go<L, DST_VOLIMAGE>(g, tg, a, j1, j2, s);
            case DST_UPDATE: return c2r_tile_reg_go<L, DST_UPDATE>(g, tg, a, j1, j2, s);
            case DST_ISRA: return c2r_tile_reg_go<L, DST_ISRA>(g, tg, a, j1, j2, s);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (a.dst) {
        case DST_IMAGE: return c2r_tile_go<L, DST_IMAGE>(g, tg, tw, a, j1, j2, s);
        case DST_POLY: return c2r_tile_go<L, DST_POLY>(g, tg, tw, a, j1, j2, s);
        case DST_VOLIMAGE: return c2r_tile_go<L, DST_VOLIMAGE>(g, tg, tw, a, j1, j2, s);
        case DST_UPDATE: return c2r_tile_go<L, DST_UPDATE>(g, tg, tw, a, j1, j2, s);
        case DST_ISRA: return c2r_tile_go<L, DST_ISRA>(g, tg, tw, a, j1, j2, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

// twiddle table of the register-resident kernels (plan time, before the first tile transform)
cudaError_t tile_fft_init() {
    static bool done = false;
    if (done) return cudaSuccess;
    float2 h[kTwTotal];
    const int Ls[] = {16, 18, 20, 24, 25, 27, 30, 32, 36};
    const double pi = 3.14159265358979323846;
    for (int L : Ls)
        for (int e = 0; e < L; ++e) {
            const double ang = -2.0 * pi * e / L;
            h[tw_off(L) + e] = make_float2((float)std::cos(ang), (float)std::sin(ang));
        }
    cudaError_t err = cudaMemcpyToSymbol(c_tile_tw, h, sizeof(h));
    if (err == cudaSuccess) done = true;
    return err;
}

// transform sizes with compiled tile kernels (5-smooth, radix-2/3/4/5 stages)
bool tile_fft_size(int L) {
    return L == 16 || L == 18 || L == 20 || L == 24 || L == 25 || L == 27 || L == 30 || L == 32 || L == 36 || L == 40 ||
           L == 45 || L == 48;
}

#define LFM_TILE_SIZES(X) X(16) X(18) X(20) X(24) X(25) X(27) X(30) X(32) X(36) X(40) X(45) X(48)

cudaError_t launch_r2c_tile(const XformGeom& g, const TileGeom& tg, const float2* tw, const R2CArgs& a, int dir,
                            unsigned* amax, cudaStream_t s) {
    if (a.ntrans <= 0) return cudaSuccess;
    const int o1 = dir ? tg.dmin1 : -tg.dmax1, o2 = dir ? tg.dmin2 : -tg.dmax2;
    switch (tg.L) {
#define LFM_R2C_TILE(LV) \
    case LV: return r2c_tile_L<LV>(g, tg, tw, a, o1, o2, amax, s);
        LFM_TILE_SIZES(LFM_R2C_TILE)
#undef LFM_R2C_TILE
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_c2r_tile(const XformGeom& g, const TileGeom& tg, const float2* tw, const C2RArgs& a, int dir,
                            cudaStream_t s) {
    if (a.ntrans <= 0) return cudaSuccess;
    const int j1 = dir ? -tg.dmin1 : tg.dmax1, j2 = dir ? -tg.dmin2 : tg.dmax2;
    switch (tg.L) {
#define LFM_C2R_TILE(LV) \
    case LV: return c2r_tile_L<LV>(g, tg, tw, a, j1, j2, s);
        LFM_TILE_SIZES(LFM_C2R_TILE)
#undef LFM_C2R_TILE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lfm
