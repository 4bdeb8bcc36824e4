/*
 * lfm_oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain fp64 CPU oracle of the light-field
 * forward / backward projections of AutoDeconJ (arXiv 2208.11422).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library.  It shares no code, header, table or helper with the CUDA product path
 * (paper_2208_11422_b200/csrc); neither includes nor links the other.
 *
 * What it computes (PAPER.md says "3D Richardson-Lucy (RL) deconvolution" P:29 §1 and that the
 * "convolution operation" is the GPU work P:29, §2.1; the shift-variant operator itself is
 * written out in SPEC.md S:196-213, module lfmodel):
 *
 *   forward:  y(s,t)      = sum_z sum_{p,q} x(z,p,q) * h[z][p%N][q%N](s-p+ch, t-q+cw)
 *   backward:  xhat(z,p,q) = sum_{s,t}       r(s,t)   * h[z][p%N][q%N](s-p+ch, t-q+cw)
 *
 * with ch=(kh-1)/2, cw=(kw-1)/2, zero outside kernel and image ("same" size).
 * Direct spatial convolution, double precision, no FFT, no blocking.  The only liberty taken is
 * that kernel rows/columns which are zero for every (a,b) kernel of a plane are not visited
 * (their products are exact zeros, so the sums are unchanged).
 *
 * Summation order is fixed: forward accumulates each output row over z, then input
 * row p ascending, then input column q ascending; backward accumulates each voxel over kernel
 * row i then kernel column j.  OpenMP parallelises over output rows (forward) or over (z,p)
 * rows (backward) only, so results do not depend on the thread count.
 *
 * Unit restriction: a "unit" is u = z*N*N + a*N + b (plane z, input phase (a,b)).  Passing a
 * unit range [u0,u1) restricts the forward sum to voxels of those units and the backward output
 * to those units (others are written 0).  This is the per-(z,a,b) decomposition of S:235 used
 * by the depth/phase sharding; [0, nz*N*N) is the full operator.
 */
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

/* per-plane bounding box of non-zero kernel taps over all (a,b) kernels of plane z */
static void plane_support(const double* h, int z, int N, int kh, int kw,
                          int* i0, int* i1, int* j0, int* j1) {
    int lo_i = kh, hi_i = -1, lo_j = kw, hi_j = -1;
    for (int ab = 0; ab < N * N; ++ab) {
        const double* k = h + ((size_t)z * N * N + ab) * (size_t)kh * kw;
        for (int i = 0; i < kh; ++i)
            for (int j = 0; j < kw; ++j)
                if (k[(size_t)i * kw + j] != 0.0) {
                    if (i < lo_i) lo_i = i;
                    if (i > hi_i) hi_i = i;
                    if (j < lo_j) lo_j = j;
                    if (j > hi_j) hi_j = j;
                }
    }
    *i0 = lo_i; *i1 = hi_i; *j0 = lo_j; *j1 = hi_j;   /* empty plane: i0 > i1 */
}

static int unit_of(int z, int p, int q, int N) { return (z * N + (p % N)) * N + (q % N); }

/* Forward projection, output rows [row0,row1) of y (other rows untouched). Returns 0 on success. */
int lfmo_forward(const double* x, const double* h, int nz, int N, int kh, int kw, int H, int W,
                 int u0, int u1, int row0, int row1, double* y) {
    if (nz < 1 || N < 1 || kh < 1 || kw < 1 || (kh % 2) == 0 || (kw % 2) == 0) return 1;
    if (H % N || W % N) return 2;
    const int ch = (kh - 1) / 2, cw = (kw - 1) / 2;
    int* sup = (int*)malloc(sizeof(int) * 4 * (size_t)nz);
    for (int z = 0; z < nz; ++z) plane_support(h, z, N, kh, kw, sup + 4 * z, sup + 4 * z + 1, sup + 4 * z + 2, sup + 4 * z + 3);
    #pragma omp parallel for schedule(dynamic, 1)
    for (int s = row0; s < row1; ++s) {
        double* yrow = y + (size_t)s * W;
        for (int t = 0; t < W; ++t) yrow[t] = 0.0;
        for (int z = 0; z < nz; ++z) {
            const int i0 = sup[4 * z], i1 = sup[4 * z + 1], j0 = sup[4 * z + 2], j1 = sup[4 * z + 3];
            if (i0 > i1) continue;
            /* kernel row i = s - p + ch  <=>  p = s + ch - i ; visit p ascending */
            int pmin = s + ch - i1, pmax = s + ch - i0;
            if (pmin < 0) pmin = 0;
            if (pmax > H - 1) pmax = H - 1;
            for (int p = pmin; p <= pmax; ++p) {
                const int i = s - p + ch;
                const int a = p % N;
                const double* xrow = x + ((size_t)z * H + p) * W;
                for (int q = 0; q < W; ++q) {
                    const int u = unit_of(z, p, q, N);
                    if (u < u0 || u >= u1) continue;
                    const double xv = xrow[q];
                    const int b = q % N;
                    const double* hrow = h + ((((size_t)z * N + a) * N + b) * kh + i) * (size_t)kw;
                    /* t - q + cw = j  <=>  t = q + j - cw */
                    int jlo = j0, jhi = j1;
                    if (q + jlo - cw < 0) jlo = cw - q;
                    if (q + jhi - cw > W - 1) jhi = W - 1 + cw - q;
                    for (int j = jlo; j <= jhi; ++j) yrow[q + j - cw] += xv * hrow[j];
                }
            }
        }
    }
    free(sup);
    return 0;
}

/* Backward projection for rows zp in [zp0,zp1) where zp = z*H + p (other rows untouched). */
int lfmo_backward(const double* r, const double* h, int nz, int N, int kh, int kw, int H, int W,
                  int u0, int u1, long zp0, long zp1, double* xhat) {
    if (nz < 1 || N < 1 || kh < 1 || kw < 1 || (kh % 2) == 0 || (kw % 2) == 0) return 1;
    if (H % N || W % N) return 2;
    const int ch = (kh - 1) / 2, cw = (kw - 1) / 2;
    int* sup = (int*)malloc(sizeof(int) * 4 * (size_t)nz);
    const int zlo = zp1 > zp0 ? (int)(zp0 / H) : 0, zhi = zp1 > zp0 ? (int)((zp1 - 1) / H) : -1;
    for (int z = zlo; z <= zhi; ++z)    /* only the planes this call visits */
        plane_support(h, z, N, kh, kw, sup + 4 * z, sup + 4 * z + 1, sup + 4 * z + 2, sup + 4 * z + 3);
    #pragma omp parallel for schedule(dynamic, 1)
    for (long zp = zp0; zp < zp1; ++zp) {
        const int z = (int)(zp / H), p = (int)(zp % H);
        const int a = p % N;
        const int i0 = sup[4 * z], i1 = sup[4 * z + 1], j0 = sup[4 * z + 2], j1 = sup[4 * z + 3];
        double* xo = xhat + (size_t)zp * W;
        for (int q = 0; q < W; ++q) {
            const int u = unit_of(z, p, q, N);
            double acc = 0.0;
            if (u >= u0 && u < u1 && i0 <= i1) {
                const int b = q % N;
                const double* k = h + (((size_t)z * N + a) * N + b) * (size_t)kh * kw;
                for (int i = i0; i <= i1; ++i) {
                    const int s = p + i - ch;          /* i = s - p + ch */
                    if (s < 0 || s >= H) continue;
                    const double* rrow = r + (size_t)s * W;
                    const double* hrow = k + (size_t)i * kw;
                    for (int j = j0; j <= j1; ++j) {
                        const int t = q + j - cw;      /* j = t - q + cw */
                        if (t < 0 || t >= W) continue;
                        acc += rrow[t] * hrow[j];
                    }
                }
            }
            xo[q] = acc;
        }
    }
    free(sup);
    return 0;
}

/* Forward projection at individual pixels (s_k, t_k): same sum as lfmo_forward, same order
 * (z, then p ascending, then q ascending), restricted to one output. */
int lfmo_forward_points(const double* x, const double* h, int nz, int N, int kh, int kw, int H, int W,
                        const int* s_idx, const int* t_idx, int npts, double* out) {
    if (nz < 1 || N < 1 || (kh % 2) == 0 || (kw % 2) == 0) return 1;
    if (H % N || W % N) return 2;
    const int ch = (kh - 1) / 2, cw = (kw - 1) / 2;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int k = 0; k < npts; ++k) {
        const int s = s_idx[k], t = t_idx[k];
        double acc = 0.0;
        for (int z = 0; z < nz; ++z)
            for (int p = s - ch; p <= s + ch; ++p) {
                if (p < 0 || p >= H) continue;
                const int i = s - p + ch, a = p % N;
                for (int q = t - cw; q <= t + cw; ++q) {
                    if (q < 0 || q >= W) continue;
                    const int j = t - q + cw, b = q % N;
                    acc += x[((size_t)z * H + p) * W + q] *
                           h[((((size_t)z * N + a) * N + b) * kh + i) * (size_t)kw + j];
                }
            }
        out[k] = acc;
    }
    return 0;
}

/* Backward projection at individual voxels (z_k, p_k, q_k). */
int lfmo_backward_points(const double* r, const double* h, int nz, int N, int kh, int kw, int H, int W,
                         const int* z_idx, const int* p_idx, const int* q_idx, int npts, double* out) {
    if (nz < 1 || N < 1 || (kh % 2) == 0 || (kw % 2) == 0) return 1;
    if (H % N || W % N) return 2;
    const int ch = (kh - 1) / 2, cw = (kw - 1) / 2;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int k = 0; k < npts; ++k) {
        const int z = z_idx[k], p = p_idx[k], q = q_idx[k];
        const int a = p % N, b = q % N;
        const double* ker = h + (((size_t)z * N + a) * N + b) * (size_t)kh * kw;
        double acc = 0.0;
        for (int i = 0; i < kh; ++i) {
            const int s = p + i - ch;
            if (s < 0 || s >= H) continue;
            for (int j = 0; j < kw; ++j) {
                const int t = q + j - cw;
                if (t < 0 || t >= W) continue;
                acc += r[(size_t)s * W + t] * ker[(size_t)i * kw + j];
            }
        }
        out[k] = acc;
    }
    return 0;
}
