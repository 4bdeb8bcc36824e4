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
        } else {  // DST_UPDATE
            out[pidx] = xold[pidx] * fmaxf(acc, 0.0f) / fmaxf(norm[pidx], eps);
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

}  // namespace lfm
