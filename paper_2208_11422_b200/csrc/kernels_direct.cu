// kernels_direct.cu -- direct (spatial-domain) shift-variant projections for small PSFs
// (K9).  FP32-ALU bound: 2 flop per kernel tap per voxel.
//
//   forward : yhat(s,t) = sum_z sum_{i,j} x(z, s-i+ch, t-j+cw) * h[z][(s-i+ch)%N][(t-j+cw)%N][i][j]
//   backward: bp(z,p,q) = sum_{i,j} r(p+i-ch, q+j-cw) * h[z][p%N][q%N][i][j]
// (S:199, S:208 rewritten in gather form).  The CTA stages the input tile with its kernel halo in
// shared memory; the PSF of the owned units stays in L2 (read through the read-only path).
// Only voxels of the plan's owned units contribute / are written.
#include "lfm_internal.cuh"

namespace lfm {

constexpr int kTile = 16;

// x in polyphase layout [nu][nh][nw]; psf [nu][kh][kw] for owned units
__global__ void __launch_bounds__(256) direct_fwd_kernel(const float* __restrict__ xp, const float* __restrict__ psf,
                                                         float* __restrict__ y, XformGeom g) {
    extern __shared__ float tile[];
    const int tw = kTile + g.kw - 1, th = kTile + g.kh - 1;
    const int s0 = blockIdx.y * kTile, t0 = blockIdx.x * kTile;
    const int ls = threadIdx.x / kTile, lt = threadIdx.x % kTile;
    const int s = s0 + ls, t = t0 + lt;
    const int N = g.N, N2 = N * N;
    float acc = 0.0f;
    const int zb = g.unit0 / N2, ze = (g.unit0 + g.nu - 1) / N2;
    for (int z = zb; z <= ze; ++z) {
        __syncthreads();
        // input rows p in [s0 - ch, s0 + 15 + ch], cols q in [t0 - cw, ...]
        for (int e = threadIdx.x; e < th * tw; e += blockDim.x) {
            const int r = e / tw, c = e % tw;
            const int p = s0 - g.ch + r, q = t0 - g.cw + c;
            float v = 0.0f;
            if (p >= 0 && p < g.H && q >= 0 && q < g.W) {
                const int u = z * N2 + (p % N) * N + (q % N);
                if (u >= g.unit0 && u < g.unit0 + g.nu)
                    v = xp[((size_t)(u - g.unit0) * g.nh + p / N) * g.nw + q / N];
            }
            tile[e] = v;
        }
        __syncthreads();
        if (s < g.H && t < g.W) {
            for (int i = 0; i < g.kh; ++i) {
                const int p = s - i + g.ch;      // input row
                if (p < 0 || p >= g.H) continue;
                const int a1 = p % N;
                const float* trow = tile + (size_t)(ls - i + g.kh - 1) * tw;
                for (int j = 0; j < g.kw; ++j) {
                    const int q = t - j + g.cw;
                    if (q < 0 || q >= g.W) continue;
                    const int u = z * N2 + a1 * N + (q % N);
                    if (u < g.unit0 || u >= g.unit0 + g.nu) continue;
                    const float xv = trow[lt - j + g.kw - 1];
                    acc = fmaf(xv, __ldg(psf + ((size_t)(u - g.unit0) * g.kh + i) * g.kw + j), acc);
                }
            }
        }
    }
    if (s < g.H && t < g.W) y[(size_t)s * g.W + t] = acc;
}

// backward with the C2R epilogues; one thread per voxel of an owned unit, r tile with halo in smem
__global__ void __launch_bounds__(256) direct_bwd_kernel(const float* __restrict__ rimg, const float* __restrict__ psf,
                                                         float* __restrict__ out, int dst, const float* __restrict__ xold,
                                                         const float* __restrict__ norm, unsigned* __restrict__ mproj,
                                                         float eps, XformGeom g) {
    extern __shared__ float tile[];
    const int tw = kTile + g.kw - 1, th = kTile + g.kh - 1;
    const int p0 = blockIdx.y * kTile, q0 = blockIdx.x * kTile;
    const int lp = threadIdx.x / kTile, lq = threadIdx.x % kTile;
    const int p = p0 + lp, q = q0 + lq;
    const int N = g.N, N2 = N * N;
    // r rows s in [p0 - ch, p0 + 15 + ch]
    for (int e = threadIdx.x; e < th * tw; e += blockDim.x) {
        const int r = e / tw, c = e % tw;
        const int s = p0 - g.ch + r, t = q0 - g.cw + c;
        tile[e] = (s >= 0 && s < g.H && t >= 0 && t < g.W) ? rimg[(size_t)s * g.W + t] : 0.0f;
    }
    __syncthreads();
    if (p >= g.H || q >= g.W) return;
    const int zb = g.unit0 / N2, ze = (g.unit0 + g.nu - 1) / N2;
    for (int z = zb; z <= ze; ++z) {
        const int u = z * N2 + (p % N) * N + (q % N);
        if (u < g.unit0 || u >= g.unit0 + g.nu) continue;
        const float* ker = psf + (size_t)(u - g.unit0) * g.kh * g.kw;
        float acc = 0.0f;
        for (int i = 0; i < g.kh; ++i) {
            const float* trow = tile + (size_t)(lp + i) * tw + lq;   // s = p + i - ch
            for (int j = 0; j < g.kw; ++j) acc = fmaf(trow[j], __ldg(ker + i * g.kw + j), acc);
        }
        const int t = u - g.unit0;
        const size_t pidx = ((size_t)t * g.nh + p / N) * g.nw + q / N;
        if (dst == DST_POLY) {
            out[pidx] = acc;
        } else if (dst == DST_VOLIMAGE) {
            out[((size_t)z * g.H + p) * g.W + q] = acc;
        } else if (dst == DST_ISRA) {
            out[pidx] = update_value<DST_ISRA>(xold[pidx], norm[pidx], acc, eps);
        } else {  // DST_UPDATE
            out[pidx] = update_value<DST_UPDATE>(xold[pidx], norm[pidx], acc, eps);
        }
    }
}

cudaError_t launch_direct_fwd(const float* xp, const float* psf, float* yimg, const XformGeom& g, cudaStream_t s) {
    const size_t smem = (size_t)(kTile + g.kh - 1) * (kTile + g.kw - 1) * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(direct_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((g.W + kTile - 1) / kTile, (g.H + kTile - 1) / kTile);
    direct_fwd_kernel<<<grid, kTile * kTile, smem, s>>>(xp, psf, yimg, g);
    return cudaGetLastError();
}

cudaError_t launch_direct_bwd(const float* rimg, const float* psf, float* out, int dst, const float* xold,
                              const float* norm, unsigned* mproj, float eps, const XformGeom& g, cudaStream_t s) {
    const size_t smem = (size_t)(kTile + g.kh - 1) * (kTile + g.kw - 1) * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(direct_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((g.W + kTile - 1) / kTile, (g.H + kTile - 1) / kTile);
    direct_bwd_kernel<<<grid, kTile * kTile, smem, s>>>(rimg, psf, out, dst, xold, norm, mproj, eps, g);
    return cudaGetLastError();
}


// ================================================================================================
// Hybrid-plan direct kernels (K9b): per direct plane z, the polyphase form
//   forward : yhat_{b'}[m'] += sum_a sum_e g_z[b'][a][e] * x_{z,a}[m' - dlo(a,b') - e]
//   backward: xhat_{z,a}[m]  = sum_b' sum_e g_z[b'][a][e] * r_{b'}[m + dlo(a,b') + e]
// where g_z[b'][a][e] = h_{z,a}[b' - a + c + N (dlo + e)] are the (at most D x D) non-zero taps of the coarse
// kernel of the pair (a, b').  A CTA owns a 8x8 coarse output tile and 45 phases (output
// phases b' in the forward, input phases a in the backward); each thread register-blocks 4x4 outputs,
// reads its (4+D-1)^2 input window and D*D taps from shared memory per reduction phase and issues
// 16*D*D FMAs.  Taps and windows are staged in chunks of reduction phases.
// ================================================================================================
namespace {
constexpr int kDT = 8;     // coarse outputs per CTA per dimension
constexpr int kDB = 4;     // outputs per thread per dimension
constexpr int kDG = 45;    // phases per CTA (225 = 5 * 45)
template <int D>
struct DirCfg {
    static constexpr int AC = D <= 3 ? 45 : 15;   // reduction phases per shared-memory chunk
    static constexpr int WB = kDB + D - 1;        // per-thread window side
    static constexpr int THREADS = (kDT / kDB) * (kDT / kDB) * kDG;
};
}  // namespace

template <int D, int SRC>
__device__ __forceinline__ float dir_src(const DirArgs& d, const float* __restrict__ x, int z, int a, int m1, int m2) {
    if (m1 < 0 || m1 >= d.nh || m2 < 0 || m2 >= d.nw) return 0.0f;
    const int u = z * d.N * d.N + a;
    if (u < d.unit0 || u >= d.unit0 + d.nu) return 0.0f;
    if constexpr (SRC == 0) {
        return x[((size_t)(u - d.unit0) * d.nh + m1) * d.nw + m2];
    } else {
        const int a1 = a / d.N, a2 = a - a1 * d.N;
        return x[((size_t)z * d.H + a1 + d.N * m1) * d.W + a2 + d.N * m2];
    }
}

// SRC: 0 = polyphase volume, 1 = image-layout volume.  accumulate: yhat += (else =)
// one plane per blockIdx.z; writes the plane's contribution to part[zi][H][W] (summed in fixed order later)
template <int D, int SRC>
__global__ void __launch_bounds__(DirCfg<D>::THREADS) dir_fwd_kernel(DirArgs d, const float* __restrict__ x,
                                                                    float* __restrict__ part) {
    using C = DirCfg<D>;
    constexpr int AC = C::AC, WB = C::WB, DD = D * D;
    extern __shared__ float sm[];
    const int N = d.N, N2 = N * N;
    const int WH = kDT + (d.dmax1 - d.dmin1) + D - 1, WW = kDT + (d.dmax2 - d.dmin2) + D - 1;
    float* xs = sm;                                   // [AC][WH][WW]
    float* cs = xs + AC * WH * WW;                    // [AC][DD][kDG]
    int* dl = reinterpret_cast<int*>(cs + AC * DD * kDG);   // [2][N][N]
    const int tiles_w = (d.nw + kDT - 1) / kDT;
    const int M01 = (blockIdx.x / tiles_w) * kDT, M02 = (blockIdx.x % tiles_w) * kDT;
    const int sb = threadIdx.x / kDG, bb = threadIdx.x - sb * kDG;
    const int bp = blockIdx.y * kDG + bb;
    const bool act = bp < N2;
    const int b1 = act ? bp / N : 0, b2 = act ? bp - (bp / N) * N : 0;
    const int r0 = (sb / (kDT / kDB)) * kDB, c0 = (sb % (kDT / kDB)) * kDB;   // thread block origin in tile
    float acc[kDB][kDB];
#pragma unroll
    for (int i = 0; i < kDB; ++i)
#pragma unroll
        for (int j = 0; j < kDB; ++j) acc[i][j] = 0.0f;
    {
        const int zi = blockIdx.z;
        const int z = d.zlist[zi];
        for (int a0 = 0; a0 < N2; a0 += AC) {
            const int na = min(AC, N2 - a0);
            __syncthreads();
            for (int e = threadIdx.x; e < na * WH * WW; e += blockDim.x) {
                const int ai = e / (WH * WW);
                const int rem = e - ai * WH * WW;
                const int rr = rem / WW, cc = rem - (rem / WW) * WW;
                xs[e] = dir_src<D, SRC>(d, x, z, a0 + ai, M01 - d.dmax1 - (D - 1) + rr, M02 - d.dmax2 - (D - 1) + cc);
            }
            for (int e = threadIdx.x; e < na * DD * kDG; e += blockDim.x) {
                const int ai = e / (DD * kDG);
                const int rem = e - ai * DD * kDG;
                const int ee = rem / kDG, b = rem - ee * kDG;
                const int bq = blockIdx.y * kDG + b;
                cs[e] = bq < N2 ? d.coef_f[(((size_t)zi * N2 + a0 + ai) * DD + ee) * N2 + bq] : 0.0f;
            }
            if (a0 == 0)
                for (int e = threadIdx.x; e < 2 * N2; e += blockDim.x) dl[e] = d.dlo[(size_t)zi * 2 * N2 + e];
            __syncthreads();
            if (act) {
                for (int ai = 0; ai < na; ++ai) {
                    const int a = a0 + ai;
                    const int a1 = a / N, a2 = a - a1 * N;
                    const int o1 = dl[a1 * N + b1], o2 = dl[N2 + a2 * N + b2];
                    const float* ws = xs + ai * WH * WW + (r0 + d.dmax1 - o1) * WW + (c0 + d.dmax2 - o2);
                    float w[WB][WB];
#pragma unroll
                    for (int i = 0; i < WB; ++i)
#pragma unroll
                        for (int j = 0; j < WB; ++j) w[i][j] = ws[i * WW + j];
                    float c[DD];
#pragma unroll
                    for (int e = 0; e < DD; ++e) c[e] = cs[(ai * DD + e) * kDG + bb];
#pragma unroll
                    for (int e1 = 0; e1 < D; ++e1)
#pragma unroll
                        for (int e2 = 0; e2 < D; ++e2)
#pragma unroll
                            for (int i = 0; i < kDB; ++i)
#pragma unroll
                                for (int j = 0; j < kDB; ++j)
                                    acc[i][j] = fmaf(c[e1 * D + e2], w[i - e1 + D - 1][j - e2 + D - 1], acc[i][j]);
                }
            }
        }
    }
    if (!act) return;
#pragma unroll
    for (int i = 0; i < kDB; ++i)
#pragma unroll
        for (int j = 0; j < kDB; ++j) {
            const int m1 = M01 + r0 + i, m2 = M02 + c0 + j;
            if (m1 < d.nh && m2 < d.nw)
                part[(size_t)blockIdx.z * d.H * d.W + (size_t)(b1 + N * m1) * d.W + b2 + N * m2] = acc[i][j];
        }
}

// SRC: SRC_RATIO (img = y, img2 = yhat), SRC_ONES, SRC_IMAGE2D.  DST: DST_POLY, DST_VOLIMAGE, DST_UPDATE
template <int SRC>
__device__ __forceinline__ float dir_rsrc(const DirArgs& d, const float* __restrict__ img, const float* __restrict__ img2,
                                          float eps, int bp, int m1, int m2) {
    if (m1 < 0 || m1 >= d.nh || m2 < 0 || m2 >= d.nw) return 0.0f;
    if constexpr (SRC == SRC_ONES) {
        return 1.0f;
    } else {
        const int b1 = bp / d.N, b2 = bp - b1 * d.N;
        const size_t pix = (size_t)(b1 + d.N * m1) * d.W + b2 + d.N * m2;
        if constexpr (SRC == SRC_RATIO)
            return img[pix] / (fmaxf(img2[pix], 0.0f) + eps);
        else
            return img[pix];
    }
}

template <int D, int SRC, int DST>
__global__ void __launch_bounds__(DirCfg<D>::THREADS) dir_bwd_kernel(DirArgs d, const float* __restrict__ img,
                                                                    const float* __restrict__ img2, float eps,
                                                                    float* __restrict__ out, const float* __restrict__ xold,
                                                                    const float* __restrict__ norm) {
    using C = DirCfg<D>;
    constexpr int AC = C::AC, WB = C::WB, DD = D * D;
    extern __shared__ float sm[];
    const int N = d.N, N2 = N * N;
    const int WH = kDT + (d.dmax1 - d.dmin1) + D - 1, WW = kDT + (d.dmax2 - d.dmin2) + D - 1;
    float* rs = sm;                                   // [AC][WH][WW]   ratio windows of AC output phases
    float* cs = rs + AC * WH * WW;                    // [AC][DD][kDG]  taps, input phase fastest
    int* dl = reinterpret_cast<int*>(cs + AC * DD * kDG);
    const int tiles_w = (d.nw + kDT - 1) / kDT;
    const int M01 = (blockIdx.x / tiles_w) * kDT, M02 = (blockIdx.x % tiles_w) * kDT;
    const int sb = threadIdx.x / kDG, aa = threadIdx.x - sb * kDG;
    const int a = blockIdx.y * kDG + aa;
    const bool act = a < N2;
    const int a1 = act ? a / N : 0, a2 = act ? a - (a / N) * N : 0;
    const int r0 = (sb / (kDT / kDB)) * kDB, c0 = (sb % (kDT / kDB)) * kDB;
    {
        const int zi = blockIdx.z;
        const int z = d.zlist[zi];
        const int u = z * N2 + a;
        const bool own = act && u >= d.unit0 && u < d.unit0 + d.nu;
        float acc[kDB][kDB];
#pragma unroll
        for (int i = 0; i < kDB; ++i)
#pragma unroll
            for (int j = 0; j < kDB; ++j) acc[i][j] = 0.0f;
        for (int b0 = 0; b0 < N2; b0 += AC) {
            const int nb = min(AC, N2 - b0);
            __syncthreads();
            for (int e = threadIdx.x; e < nb * WH * WW; e += blockDim.x) {
                const int bi = e / (WH * WW);
                const int rem = e - bi * WH * WW;
                const int rr = rem / WW, cc = rem - (rem / WW) * WW;
                rs[e] = dir_rsrc<SRC>(d, img, img2, eps, b0 + bi, M01 + d.dmin1 + rr, M02 + d.dmin2 + cc);
            }
            for (int e = threadIdx.x; e < nb * DD * kDG; e += blockDim.x) {
                const int bi = e / (DD * kDG);
                const int rem = e - bi * DD * kDG;
                const int ee = rem / kDG, q = rem - ee * kDG;
                const int aq = blockIdx.y * kDG + q;
                cs[e] = aq < N2 ? d.coef_b[(((size_t)zi * N2 + b0 + bi) * DD + ee) * N2 + aq] : 0.0f;
            }
            if (b0 == 0)
                for (int e = threadIdx.x; e < 2 * N2; e += blockDim.x) dl[e] = d.dlo[(size_t)zi * 2 * N2 + e];
            __syncthreads();
            if (own) {
                for (int bi = 0; bi < nb; ++bi) {
                    const int bq = b0 + bi;
                    const int b1 = bq / N, b2 = bq - b1 * N;
                    const int o1 = dl[a1 * N + b1], o2 = dl[N2 + a2 * N + b2];
                    const float* ws = rs + bi * WH * WW + (r0 + o1 - d.dmin1) * WW + (c0 + o2 - d.dmin2);
                    float w[WB][WB];
#pragma unroll
                    for (int i = 0; i < WB; ++i)
#pragma unroll
                        for (int j = 0; j < WB; ++j) w[i][j] = ws[i * WW + j];
                    float c[DD];
#pragma unroll
                    for (int e = 0; e < DD; ++e) c[e] = cs[(bi * DD + e) * kDG + aa];
#pragma unroll
                    for (int e1 = 0; e1 < D; ++e1)
#pragma unroll
                        for (int e2 = 0; e2 < D; ++e2)
#pragma unroll
                            for (int i = 0; i < kDB; ++i)
#pragma unroll
                                for (int j = 0; j < kDB; ++j)
                                    acc[i][j] = fmaf(c[e1 * D + e2], w[i + e1][j + e2], acc[i][j]);
                }
            }
        }
        if (own) {
            const int lu = u - d.unit0;
#pragma unroll
            for (int i = 0; i < kDB; ++i)
#pragma unroll
                for (int j = 0; j < kDB; ++j) {
                    const int m1 = M01 + r0 + i, m2 = M02 + c0 + j;
                    if (m1 < d.nh && m2 < d.nw) {
                        const size_t pidx = ((size_t)lu * d.nh + m1) * d.nw + m2;
                        const float v = acc[i][j];
                        if constexpr (DST == DST_POLY) {
                            out[pidx] = v;
                        } else if constexpr (DST == DST_VOLIMAGE) {
                            out[((size_t)z * d.H + a1 + N * m1) * d.W + a2 + N * m2] = v;
                        } else {
                            out[pidx] = update_value<DST>(xold[pidx], norm[pidx], v, eps);
                        }
                    }
                }
        }
    }
}

template <int D>
static size_t dir_smem(const DirArgs& d) {
    using C = DirCfg<D>;
    const int WH = kDT + (d.dmax1 - d.dmin1) + D - 1, WW = kDT + (d.dmax2 - d.dmin2) + D - 1;
    return ((size_t)C::AC * WH * WW + (size_t)C::AC * D * D * kDG) * sizeof(float) + 2 * (size_t)d.N * d.N * sizeof(int);
}

// y (+)= sum over direct planes of part[zi] in plane order (deterministic)
__global__ void dir_reduce_kernel(const float* __restrict__ part, int nzd, size_t hw, float* __restrict__ y,
                                  int accumulate) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < hw; i += (size_t)gridDim.x * blockDim.x) {
        float v = accumulate ? y[i] : 0.0f;
        for (int zi = 0; zi < nzd; ++zi) v += part[(size_t)zi * hw + i];
        y[i] = v;
    }
}

template <int D>
static cudaError_t dir_fwd_D(const DirArgs& d, const float* x, int src_image, float* part, cudaStream_t s) {
    const size_t smem = dir_smem<D>(d);
    dim3 grid(((d.nh + kDT - 1) / kDT) * ((d.nw + kDT - 1) / kDT), (d.N * d.N + kDG - 1) / kDG, d.nzd);
    cudaError_t e;
    if (src_image) {
        e = cudaFuncSetAttribute(dir_fwd_kernel<D, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        dir_fwd_kernel<D, 1><<<grid, DirCfg<D>::THREADS, smem, s>>>(d, x, part);
    } else {
        e = cudaFuncSetAttribute(dir_fwd_kernel<D, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        dir_fwd_kernel<D, 0><<<grid, DirCfg<D>::THREADS, smem, s>>>(d, x, part);
    }
    return cudaGetLastError();
}

template <int D, int SRC, int DST>
static cudaError_t dir_bwd_DSD(const DirArgs& d, const float* img, const float* img2, float eps, float* out,
                               const float* xold, const float* norm, cudaStream_t s) {
    const size_t smem = dir_smem<D>(d);
    dim3 grid(((d.nh + kDT - 1) / kDT) * ((d.nw + kDT - 1) / kDT), (d.N * d.N + kDG - 1) / kDG, d.nzd);
    cudaError_t e = cudaFuncSetAttribute(dir_bwd_kernel<D, SRC, DST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dir_bwd_kernel<D, SRC, DST><<<grid, DirCfg<D>::THREADS, smem, s>>>(d, img, img2, eps, out, xold, norm);
    return cudaGetLastError();
}

template <int D>
static cudaError_t dir_bwd_D(const DirArgs& d, int src, const float* img, const float* img2, float eps, int dst,
                             float* out, const float* xold, const float* norm, cudaStream_t s) {
#define LFM_DIR_B(SRCV, DSTV) \
    if (src == SRCV && dst == DSTV) return dir_bwd_DSD<D, SRCV, DSTV>(d, img, img2, eps, out, xold, norm, s);
    LFM_DIR_B(SRC_RATIO, DST_UPDATE)
    LFM_DIR_B(SRC_IMAGE2D, DST_ISRA)
    LFM_DIR_B(SRC_ONES, DST_POLY)
    LFM_DIR_B(SRC_IMAGE2D, DST_VOLIMAGE)
    LFM_DIR_B(SRC_IMAGE2D, DST_POLY)
    LFM_DIR_B(SRC_RATIO, DST_POLY)
#undef LFM_DIR_B
    return cudaErrorInvalidValue;
}

cudaError_t launch_dir_fwd(const DirArgs& d, const float* x, int src_image, float* part, float* y, int accumulate,
                           cudaStream_t s) {
    if (d.nzd <= 0) return cudaSuccess;
    cudaError_t e;
    switch (d.D) {
        case 1: e = dir_fwd_D<1>(d, x, src_image, part, s); break;
        case 2: e = dir_fwd_D<2>(d, x, src_image, part, s); break;
        case 3: e = dir_fwd_D<3>(d, x, src_image, part, s); break;
        case 4: e = dir_fwd_D<4>(d, x, src_image, part, s); break;
        case 5: e = dir_fwd_D<5>(d, x, src_image, part, s); break;
        default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    return launch_plane_reduce(part, d.nzd, (size_t)d.H * d.W, y, accumulate, s);
}

cudaError_t launch_plane_reduce(const float* part, int nzd, size_t hw, float* y, int accumulate, cudaStream_t s) {
    dir_reduce_kernel<<<1184, 256, 0, s>>>(part, nzd, hw, y, accumulate);
    return cudaGetLastError();
}

cudaError_t launch_dir_bwd(const DirArgs& d, int src, const float* img, const float* img2, float eps, int dst, float* out,
                           const float* xold, const float* norm, cudaStream_t s) {
    if (d.nzd <= 0) return cudaSuccess;
    switch (d.D) {
        case 1: return dir_bwd_D<1>(d, src, img, img2, eps, dst, out, xold, norm, s);
        case 2: return dir_bwd_D<2>(d, src, img, img2, eps, dst, out, xold, norm, s);
        case 3: return dir_bwd_D<3>(d, src, img, img2, eps, dst, out, xold, norm, s);
        case 4: return dir_bwd_D<4>(d, src, img, img2, eps, dst, out, xold, norm, s);
        case 5: return dir_bwd_D<5>(d, src, img, img2, eps, dst, out, xold, norm, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lfm
