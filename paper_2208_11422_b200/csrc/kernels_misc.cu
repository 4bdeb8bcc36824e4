// kernels_misc.cu -- layout conversion, fills, deterministic fp64 reductions and the fp64 DCT-entropy
// metric (K8).
//
// Metric (§2.2): m = max_z x; F(u,v) = sum_{i,j} m(i,j) Cr[u][i] Cw[v][j] with the
// orthonormal DCT-II basis of Eqs. (2)-(4), only on the cutoff corner u < Y_S, v < X_S;
// ||F||_2 = ||m||_2 by Parseval (reading C13, pinned by the oracle's Parseval test);
// E = 2/(X_S Y_S) * sum_{(u,v) in T} -w log2 w, w = |F(u,v)| / ||m||_2 (Eq. 12, readings C12/C13).
// All reductions use fixed partitions and fixed shuffle trees, so E is bit-reproducible.
#include "lfm_internal.cuh"

namespace lfm {

__global__ void fill_kernel(float* p, size_t n, float v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void fill_dev_kernel(float* p, size_t n, const double* num, const double* den) {
    const float v = (float)(num[0] / den[0]);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

cudaError_t launch_fill(float* p, size_t n, float v, cudaStream_t s) {
    if (!n) return cudaSuccess;
    fill_kernel<<<1184, 256, 0, s>>>(p, n, v);
    return cudaGetLastError();
}

cudaError_t launch_fill_dev(float* p, size_t n, const double* num, const double* den, cudaStream_t s) {
    if (!n) return cudaSuccess;
    fill_dev_kernel<<<1184, 256, 0, s>>>(p, n, num, den);
    return cudaGetLastError();
}

// Row-tiled layout conversion: one CTA per image row (z, p).  The row's pixels q = a2 + N m2 belong to the N units
// u = z N^2 + (p mod N) N + a2, each a contiguous run of nw floats at coarse row m1 = p / N of the polyphase volume,
// so both sides are read / written coalesced and the interleave happens in shared memory (W floats).
template <bool TO_IMAGE>
__global__ void __launch_bounds__(256) poly_image_rows_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                                              XformGeom g, int ub, int uc, int zb) {
    extern __shared__ float rowbuf[];   // [N][nw]
    const int N = g.N, N2 = N * N, nw = g.nw;
    const int z = zb + (int)(blockIdx.x / g.H), p = (int)(blockIdx.x % g.H);
    const int a1 = p % N, m1 = p / N;
    const int u0 = z * N2 + a1 * N;   // unit of a2 = 0
    const size_t ppix = (size_t)g.nh * nw;
    float* row = dst + ((size_t)z * g.H + p) * g.W;
    const float* irow = src + ((size_t)z * g.H + p) * g.W;
    if (TO_IMAGE) {
        for (int e = threadIdx.x; e < N * nw; e += blockDim.x) {
            const int a2 = e / nw, m2 = e - a2 * nw, u = u0 + a2;
            if (u >= ub && u < ub + uc) rowbuf[e] = src[(size_t)(u - ub) * ppix + (size_t)m1 * nw + m2];
        }
        __syncthreads();
        for (int q = threadIdx.x; q < g.W; q += blockDim.x) {
            const int a2 = q % N, m2 = q / N, u = u0 + a2;
            if (u >= ub && u < ub + uc) row[q] = rowbuf[a2 * nw + m2];
        }
    } else {
        for (int q = threadIdx.x; q < g.W; q += blockDim.x) {
            const int a2 = q % N, m2 = q / N;
            rowbuf[a2 * nw + m2] = irow[q];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < N * nw; e += blockDim.x) {
            const int a2 = e / nw, m2 = e - a2 * nw, u = u0 + a2;
            if (u >= ub && u < ub + uc) dst[(size_t)(u - ub) * ppix + (size_t)m1 * nw + m2] = rowbuf[e];
        }
    }
}

template <bool TO_IMAGE>
static cudaError_t poly_image_rows(const float* src, float* dst, const XformGeom& g, int ub, int uc, cudaStream_t s) {
    if (uc <= 0) return cudaSuccess;
    const int N2 = g.N * g.N;
    const int zb = ub / N2, ze = (ub + uc - 1) / N2;
    const size_t smem = (size_t)g.N * g.nw * sizeof(float);
    poly_image_rows_kernel<TO_IMAGE><<<(unsigned)((ze - zb + 1) * g.H), 256, smem, s>>>(src, dst, g, ub, uc, zb);
    return cudaGetLastError();
}

cudaError_t launch_poly_to_image(const float* xp, float* x, const XformGeom& g, int unit_begin, int unit_count,
                                 cudaStream_t s) {
    return poly_image_rows<true>(xp, x, g, unit_begin, unit_count, s);
}

cudaError_t launch_image_to_poly(const float* x, float* xp, const XformGeom& g, int unit_begin, int unit_count,
                                 cudaStream_t s) {
    return poly_image_rows<false>(x, xp, g, unit_begin, unit_count, s);
}

// z max-projection of the owned units of an image-layout volume (lfm_quality)
__global__ void max_project_kernel(const float* __restrict__ x, unsigned* __restrict__ mproj, XformGeom g) {
    const int N = g.N, N2 = N * N;
    const size_t plane = (size_t)g.H * g.W;
    const size_t total = (size_t)g.nz * plane;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int z = (int)(e / plane);
        const int pix = (int)(e % plane);
        const int p = pix / g.W, q = pix % g.W;
        const int u = z * N2 + (p % N) * N + (q % N);
        if (u < g.unit0 || u >= g.unit0 + g.nu) continue;
        atomicMax(mproj + pix, __float_as_uint(fmaxf(x[e], 0.0f)));
    }
}

// z max-projection of the owned units of a POLYPHASE volume, deterministic and atomic-free:
// one thread per (input phase a, coarse pixel m) reads x[(z*N^2 + a) - unit0][m] for every owned plane z
// (coalesced along m) and writes max_z once to pixel (a1 + N m1, a2 + N m2); pixels whose phase this rank
// owns in no plane get 0 (the identity of the cross-rank max, x >= 0).
__global__ void max_project_poly_kernel(const float* __restrict__ xp, unsigned* __restrict__ mproj, XformGeom g) {
    const int N = g.N, N2 = N * N;
    const int per = g.nh * g.nw;
    const size_t total = (size_t)N2 * per;
    const int zb = g.unit0 / N2, ze = (g.unit0 + g.nu - 1) / N2;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int a = (int)(e / per);
        const int m = (int)(e - (size_t)a * per);
        float v = 0.0f;
        for (int z = zb; z <= ze; ++z) {
            const int u = z * N2 + a;
            if (u >= g.unit0 && u < g.unit0 + g.nu) v = fmaxf(v, xp[(size_t)(u - g.unit0) * per + m]);
        }
        const int m1 = m / g.nw, m2 = m - m1 * g.nw;
        const int a1 = a / N, a2 = a - a1 * N;
        mproj[(size_t)(a1 + N * m1) * g.W + a2 + N * m2] = __float_as_uint(v);
    }
}

// F frames: frame f reads base + (f * 3 + sel.b[f]) * vol (its current triple-buffer slot) into mproj + f H W
__global__ void max_project_poly_batch_kernel(const float* __restrict__ base, size_t vol, FrameSel sel,
                                              unsigned* __restrict__ mproj, XformGeom g) {
    const int f = blockIdx.y;
    const float* xp = base + ((size_t)f * 3 + sel.b[f]) * vol;
    unsigned* mp = mproj + (size_t)f * g.H * g.W;
    const int N = g.N, N2 = N * N;
    const int per = g.nh * g.nw;
    const size_t total = (size_t)N2 * per;
    const int zb = g.unit0 / N2, ze = (g.unit0 + g.nu - 1) / N2;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int a = (int)(e / per);
        const int m = (int)(e - (size_t)a * per);
        float v = 0.0f;
        for (int z = zb; z <= ze; ++z) {
            const int u = z * N2 + a;
            if (u >= g.unit0 && u < g.unit0 + g.nu) v = fmaxf(v, xp[(size_t)(u - g.unit0) * per + m]);
        }
        const int m1 = m / g.nw, m2 = m - m1 * g.nw;
        const int a1 = a / N, a2 = a - a1 * N;
        mp[(size_t)(a1 + N * m1) * g.W + a2 + N * m2] = __float_as_uint(v);
    }
}

cudaError_t launch_max_project_poly_batch(const float* base, size_t vol, const FrameSel& sel, int F, unsigned* mproj,
                                          const XformGeom& g, cudaStream_t s) {
    const size_t total = (size_t)g.N * g.N * g.nh * g.nw;
    const unsigned blocks = (unsigned)((total + 255) / 256 < 1184 ? (total + 255) / 256 : 1184);
    max_project_poly_batch_kernel<<<dim3(blocks, F), 256, 0, s>>>(base, vol, sel, mproj, g);
    return cudaGetLastError();
}

cudaError_t launch_max_project_poly(const float* xp, unsigned* mproj, const XformGeom& g, cudaStream_t s) {
    const size_t total = (size_t)g.N * g.N * g.nh * g.nw;
    const unsigned blocks = (unsigned)((total + 255) / 256 < 4736 ? (total + 255) / 256 : 4736);
    max_project_poly_kernel<<<blocks, 256, 0, s>>>(xp, mproj, g);
    return cudaGetLastError();
}

cudaError_t launch_max_project(const float* x, unsigned* mproj, const XformGeom& g, cudaStream_t s) {
    max_project_kernel<<<2368, 256, 0, s>>>(x, mproj, g);
    return cudaGetLastError();
}

// ---- deterministic fp64 sum / min / max ----
__global__ void stats_partial_kernel(const float* __restrict__ p, size_t n, double* __restrict__ partials) {
    __shared__ double ss[32], smn[32], smx[32];
    double s = 0.0, mn = 1e300, mx = -1e300;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const double v = p[i];
        s += v;
        mn = fmin(mn, v);
        mx = fmax(mx, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        ss[w] = s;
        smn[w] = mn;
        smx[w] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 1e300, c = -1e300;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            a += ss[k];
            b = fmin(b, smn[k]);
            c = fmax(c, smx[k]);
        }
        partials[3 * blockIdx.x] = a;
        partials[3 * blockIdx.x + 1] = b;
        partials[3 * blockIdx.x + 2] = c;
    }
}

__global__ void stats_final_kernel(const double* __restrict__ partials, int nparts, double* out3) {
    if (threadIdx.x == 0) {
        double a = 0.0, b = 1e300, c = -1e300;
        for (int k = 0; k < nparts; ++k) {
            a += partials[3 * k];
            b = fmin(b, partials[3 * k + 1]);
            c = fmax(c, partials[3 * k + 2]);
        }
        out3[0] = a;
        out3[1] = b;
        out3[2] = c;
    }
}

cudaError_t launch_sum_stats(const float* p, size_t n, double* partials, int nparts, double* out3, cudaStream_t s) {
    stats_partial_kernel<<<nparts, 256, 0, s>>>(p, n, partials);
    stats_final_kernel<<<1, 32, 0, s>>>(partials, nparts, out3);
    return cudaGetLastError();
}

// ---- metric ----
constexpr int kMetricRows = 4;

// T1[v][i] = sum_j m[i][j] Cw[v][j] (v < xs) and rowsq[i] = sum_j m[i][j]^2, fp64, kMetricRows rows per CTA
__global__ void __launch_bounds__(256) metric_rows_kernel(const unsigned* __restrict__ mbits, int H, int W, int xs,
                                                          const double* __restrict__ Cw, double* __restrict__ T1,
                                                          double* __restrict__ rowsq, size_t fs_m, size_t fs_t1) {
    extern __shared__ double mrow[];
    mbits += blockIdx.y * fs_m;   // frame blockIdx.y of a batch (fs_* = per-frame strides; 0 for one frame)
    T1 += blockIdx.y * fs_t1;
    rowsq += blockIdx.y * (size_t)H;
    const int i0 = blockIdx.x * kMetricRows;
    const int nr = min(kMetricRows, H - i0);
    for (int e = threadIdx.x; e < nr * W; e += blockDim.x)
        mrow[e] = (double)__uint_as_float(mbits[(size_t)i0 * W + e]);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int task = warp; task < xs + 1; task += nw) {
        double acc[kMetricRows];
#pragma unroll
        for (int r = 0; r < kMetricRows; ++r) acc[r] = 0.0;
        if (task < xs) {
            const double* c = Cw + (size_t)task * W;
            for (int j = lane; j < W; j += 32) {
                const double cv = c[j];
#pragma unroll
                for (int r = 0; r < kMetricRows; ++r)
                    if (r < nr) acc[r] = fma(mrow[r * W + j], cv, acc[r]);
            }
        } else {
            for (int j = lane; j < W; j += 32) {
#pragma unroll
                for (int r = 0; r < kMetricRows; ++r)
                    if (r < nr) acc[r] = fma(mrow[r * W + j], mrow[r * W + j], acc[r]);
            }
        }
#pragma unroll
        for (int r = 0; r < kMetricRows; ++r)
            for (int o = 16; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
        if (lane == 0) {
            for (int r = 0; r < nr; ++r) {
                if (task < xs)
                    T1[(size_t)task * H + i0 + r] = acc[r];   // column-major: member sums read it coalesced
                else
                    rowsq[i0 + r] = acc[r];
            }
        }
    }
}

// Parseval norm ||m|| from the row sums (every CTA, the same fixed order -> identical value everywhere)
__device__ double metric_norm(const double* __restrict__ rowsq, int H, double* red) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double t = 0.0;
    for (int i = threadIdx.x; i < H; i += blockDim.x) t += rowsq[i];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[warp] = t;
    __syncthreads();
    double v = lane < nw ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    return sqrt(v);
}

// F(u, v) = sum_i Cr[u][i] T1[v][i] for region member k (one warp each), entropy term -w log2 w, w = |F| / ||m||
__global__ void __launch_bounds__(256) metric_member_kernel(int H, const double* __restrict__ Cr,
                                                            const double* __restrict__ T1,
                                                            const double* __restrict__ rowsq,
                                                            const int2* __restrict__ mem, int nmem,
                                                            double* __restrict__ term, double* __restrict__ out,
                                                            size_t fs_t1, int fs_out) {
    __shared__ double red[32];
    T1 += blockIdx.y * fs_t1;
    term += blockIdx.y * fs_t1;
    rowsq += blockIdx.y * (size_t)H;
    out += blockIdx.y * fs_out;
    const double L = metric_norm(rowsq, H, red);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = blockIdx.x * (blockDim.x >> 5) + warp;
    if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = L;
    if (k >= nmem) return;
    const int u = mem[k].x, v = mem[k].y;
    const double* cr = Cr + (size_t)u * H;
    const double* t1 = T1 + (size_t)v * H;
    double f = 0.0;
    for (int i = lane; i < H; i += 32) f = fma(cr[i], t1[i], f);
    for (int o = 16; o > 0; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
    if (lane == 0) {
        double e = 0.0;
        if (L > 0.0) {
            const double w = fabs(f) / L;
            if (w > 0.0) e = -w * log2(w);
        }
        term[k] = e;
    }
}

// E = 2 / (xs ys) * sum_k term[k] in a fixed order (one CTA)
__global__ void __launch_bounds__(1024) metric_sum_kernel(int xs, int ys, const double* __restrict__ term, int nmem,
                                                          double* __restrict__ out, size_t fs_t1, int fs_out) {
    __shared__ double red[32];
    term += blockIdx.x * fs_t1;   // one CTA per frame
    out += blockIdx.x * fs_out;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double t = 0.0;
    for (int k = threadIdx.x; k < nmem; k += blockDim.x) t += term[k];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[warp] = t;
    __syncthreads();
    if (warp == 0) {
        double v = lane < nw ? red[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) out[0] = out[1] > 0.0 ? 2.0 / ((double)xs * (double)ys) * v : 0.0;
    }
}

cudaError_t launch_metric(const unsigned* mproj_bits, int H, int W, int xs, int ys, const double* Cr,
                          const double* Cw, const int2* members, int nmem, double* T1, double* rowsq,
                          double* out, cudaStream_t s) {
    const size_t smem = (size_t)kMetricRows * W * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(metric_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    metric_rows_kernel<<<(H + kMetricRows - 1) / kMetricRows, 256, smem, s>>>(mproj_bits, H, W, xs, Cw, T1, rowsq, 0, 0);
    // the per-member terms follow T1 ([xs][H] doubles) in the same allocation (MetricDev)
    double* term = T1 + (size_t)xs * H;
    metric_member_kernel<<<(nmem + 7) / 8, 256, 0, s>>>(H, Cr, T1, rowsq, members, nmem, term, out, 0, 0);
    metric_sum_kernel<<<1, 1024, 0, s>>>(xs, ys, term, nmem, out, 0, 0);
    return cudaGetLastError();
}

// the metric of F frames in three launches: frame f reads mproj_bits + f H W and writes out[2 f] (E) / out[2 f + 1]
// (its norm); T1 / rowsq hold F per-frame workspaces (T1: xs H + nmem doubles each, rowsq: H each).  Same arithmetic
// and reduction order per frame as launch_metric.
cudaError_t launch_metric_batch(const unsigned* mproj_bits, int F, int H, int W, int xs, int ys, const double* Cr,
                                const double* Cw, const int2* members, int nmem, double* T1, double* rowsq,
                                double* out, cudaStream_t s) {
    const size_t smem = (size_t)kMetricRows * W * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(metric_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const size_t fs_t1 = (size_t)xs * H + nmem;
    metric_rows_kernel<<<dim3((H + kMetricRows - 1) / kMetricRows, F), 256, smem, s>>>(mproj_bits, H, W, xs, Cw, T1, rowsq,
                                                                                       (size_t)H * W, fs_t1);
    double* term = T1 + (size_t)xs * H;
    metric_member_kernel<<<dim3((nmem + 7) / 8, F), 256, 0, s>>>(H, Cr, T1, rowsq, members, nmem, term, out, fs_t1, 2);
    metric_sum_kernel<<<F, 1024, 0, s>>>(xs, ys, term, nmem, out, fs_t1, 2);
    return cudaGetLastError();
}

// ---- ratio image (direct path): r = y / (max(yhat,0) + eps) ----
__global__ void ratio_kernel(const float* __restrict__ y, const float* __restrict__ yhat, float* __restrict__ r,
                             size_t n, float eps) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        r[i] = y[i] / (fmaxf(yhat[i], 0.0f) + eps);
}

cudaError_t launch_ratio(const float* y, const float* yhat, float* r, size_t n, float eps, cudaStream_t s) {
    ratio_kernel<<<1184, 256, 0, s>>>(y, yhat, r, n, eps);
    return cudaGetLastError();
}

// ---- image -> output-phase planes for the tiled path's image-side transforms: out[b'][i][j] = v(b1 + N i, b2 + N j),
//      v = y / (max(yhat, 0) + eps) (yhat != nullptr) or y; computed once per projection instead of once per tile group
__global__ void image_phase_planes_kernel(const float* __restrict__ y, const float* __restrict__ yhat, float eps,
                                          float* __restrict__ out, int N, int H, int W, int nh, int nw) {
    const size_t n = (size_t)H * W;
    for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < n; p += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(p / W), c = (int)(p - (size_t)r * W);
        const float v = yhat ? y[p] / (fmaxf(yhat[p], 0.0f) + eps) : y[p];
        out[((size_t)((r % N) * N + c % N) * nh + r / N) * nw + c / N] = v;
    }
}

cudaError_t launch_image_phase_planes(const float* y, const float* yhat, float eps, float* out, int N, int H, int W,
                                      cudaStream_t s) {
    image_phase_planes_kernel<<<1184, 256, 0, s>>>(y, yhat, eps, out, N, H, W, H / N, W / N);
    return cudaGetLastError();
}

// ---- device-resident auto-stop loop (LFM_PLAN_DEVICE_LOOP) ----
// The stop rule of lfm_rl_iterate (reading C15) evaluated on the device after each iteration: appends E_k to the
// series, counts strict decreases, tracks the argmax (ties -> smallest k) and sets the WHILE / IF conditions of the
// captured loop graph.  Same double comparisons as the host loop, so the decisions are identical.
__global__ void loop_reset_kernel(LoopState* st) {
    st->k = 0;
    st->dec = 0;
    st->best_k = 0;
    st->stop = 0;
    st->improved = 0;
    st->prev = 0.0;
    st->best_e = -INFINITY;
}

__global__ void stop_rule_kernel(LoopState* st, const double* __restrict__ e_dev, double* __restrict__ series, int mode,
                                 int n_iters, int min_iters, int patience, int cap, cudaGraphConditionalHandle h_loop,
                                 cudaGraphConditionalHandle h_second, int has_second) {
    const int k = ++st->k;
    const double e = e_dev[0];
    series[k - 1] = e;
    if (k > 1 && e < st->prev)
        ++st->dec;
    else
        st->dec = 0;
    st->prev = e;
    st->improved = e > st->best_e;
    if (st->improved) {
        st->best_e = e;
        st->best_k = k;
    }
    const bool stop = mode == LFM_MODE_FIXED ? k >= n_iters : ((k >= min_iters && st->dec >= patience) || k >= cap);
    st->stop = stop;
    cudaGraphSetConditional(h_loop, stop ? 0u : 1u);
    if (has_second) cudaGraphSetConditional(h_second, stop ? 0u : 1u);
}

// x_best <- x when the last iteration improved E (grid-stride, float4 when aligned)
__global__ void cond_copy_kernel(const LoopState* __restrict__ st, const float* __restrict__ src, float* __restrict__ dst,
                                 size_t n) {
    if (!st->improved) return;
    const size_t n4 = n / 4;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) d4[i] = s4[i];
    for (size_t i = 4 * n4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

cudaError_t launch_loop_reset(LoopState* st, cudaStream_t s) {
    loop_reset_kernel<<<1, 1, 0, s>>>(st);
    return cudaGetLastError();
}

cudaError_t launch_stop_rule(LoopState* st, const double* e_dev, double* series, const lfm_policy* pol, int cap,
                             cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_second, int has_second,
                             cudaStream_t s) {
    stop_rule_kernel<<<1, 1, 0, s>>>(st, e_dev, series, pol->mode, pol->n_iters, pol->min_iters, pol->patience, cap,
                                     h_loop, h_second, has_second);
    return cudaGetLastError();
}

cudaError_t launch_cond_copy(const LoopState* st, const float* src, float* dst, size_t n, cudaStream_t s) {
    cond_copy_kernel<<<592, 256, 0, s>>>(st, src, dst, n);
    return cudaGetLastError();
}

}  // namespace lfm
