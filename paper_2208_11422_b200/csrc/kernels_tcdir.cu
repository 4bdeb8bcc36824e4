// kernels_tcdir.cu -- direct polyphase projections of near-focus planes on the 5th-generation tensor cores
// (K9tc).  fp32-accurate through the 3xTF32 split (a*b ~ ah*bh + ah*bl + al*bh).
//
// For one plane z the direct path is a sum over coarse tap offsets d of dense contractions over phases:
//   forward : Y[p][b']  += sum_a  X_a[m(p) - d] * G_d[b'][a]      (K = input phases a,  N = output phases b')
//   backward: Xh[p][a]   = sum_b' r_b'[m(p) + d] * G_d[b'][a]      (K = output phases b', N = input phases a)
// with G_d[b'][a] = h_{z,a}[b' - a + c + N d] (zero outside the kernel).  A CTA owns 128 coarse
// pixels (M, one TMEM lane each), one group of NG <= 48 N-phases (TMEM columns) and one plane, and loops over
// K chunks of 32 phases x taps:
//   * all 256 threads stage the chunk's source window (X planes or ratio-image phases, halo for every tap) in
//     shared memory, then for each tap build the shifted A tile (128 x 32, hi and lo) in the canonical K-major
//     core-matrix layout;
//   * the tap's coefficient tile (NG x 32, hi and lo, precomputed in the same layout) arrives by one bulk copy,
//     one iteration ahead, into a 3-deep ring;
//   * one thread issues 3 tcgen05.mma.kind::tf32 per K-step into the TMEM accumulator and commits to an
//     mbarrier; A tiles are double buffered so the next tap's tile is built while the tensor core works.
// The epilogue reads TMEM (tcgen05.ld 32x32b) and writes per-plane forward partials (summed across planes in a
// fixed order afterwards) or the backward result with the RL update / polyphase / image-layout epilogue.
#include "lfm_internal.cuh"
#include "tc_sm100.cuh"

namespace lfm {

namespace {
constexpr int kTcM = 128;          // pixels per CTA (TMEM lanes)
constexpr int kTcKC = 32;          // K phases per chunk (4 MMA K-steps)
constexpr int kTcP = 4;            // taps per drain group (accumulation chain = kTcP/2 taps x 12 MMAs)
constexpr int kTcBRing = 4;        // coefficient tiles in flight
constexpr int kDrainWarps = 4;     // warps 0-3: TMEM lane quarters -> fp32 running sums, epilogue
constexpr int kBuildWarps = 8;     // warps 4-11: window staging and A-tile builds
constexpr int kTcThreads = 32 * (kDrainWarps + kBuildWarps + 1);   // + warp 12: MMA issuer / B producer
constexpr uint32_t kTmemCols = 256;   // 2 regions x 2 accumulators x 64 columns (NG <= 48)
}  // namespace

struct TcSmem {
    uint32_t a[2];       // A tiles (hi then lo), 32 KB each
    uint32_t b[kTcBRing];// B tiles (hi then lo), NG x 32 x 8 bytes
    uint32_t win;        // source window [32][WR][WC]
    uint32_t total;
};

__host__ __device__ inline TcSmem tc_smem_layout(int NG, int WR, int WC) {
    TcSmem L{};
    uint32_t o = 0;
    const uint32_t atile = kTcM * kTcKC * 4 * 2;
    const uint32_t btile = (uint32_t)NG * kTcKC * 4 * 2;
    for (int i = 0; i < 2; ++i) {
        L.a[i] = o;
        o += atile;
    }
    for (int i = 0; i < kTcBRing; ++i) {
        L.b[i] = o;
        o += btile;
    }
    L.win = o;
    o += (uint32_t)kTcKC * WR * WC * 4;
    L.total = o;
    return L;
}

__device__ __forceinline__ void builders_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kBuildWarps) : "memory"); }

// SRC (forward): 0 polyphase volume, 1 image-layout volume.  (backward): SRC_RATIO, SRC_ONES, SRC_IMAGE2D
template <bool FWD, int SRC, int DST>
__global__ void __launch_bounds__(kTcThreads, 1) tcdir_kernel(TcDirArgs d, const float* __restrict__ src,
                                                              const float* __restrict__ src2, float eps,
                                                              float* __restrict__ out, const float* __restrict__ xold,
                                                              const float* __restrict__ norm) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t bar_afull[2], bar_aempty[2], bar_bfull[kTcBRing], bar_bempty[kTcBRing];
    __shared__ uint64_t bar_mma[2], bar_tfree[2];
    __shared__ uint32_t tmem_base;
    const int N = d.N, N2 = N * N;
    const int NG = d.NG;
    const int T2 = d.T2, NT = d.T1 * d.T2;
    const int npix = d.nh * d.nw;
    const int p0 = blockIdx.x * kTcM;
    const int grp = blockIdx.y;
    const int zi = blockIdx.z;
    const int z = d.zlist[zi];
    const int row0 = p0 / d.nw;
    const int WR = d.WR, WC = d.WC, wsz = WR * WC;
    const TcSmem L = tc_smem_layout(NG, WR, WC);
    float* win = reinterpret_cast<float*>(smem + L.win);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nchunks = (d.Kpad + kTcKC - 1) / kTcKC;
    const int total = nchunks * NT;
    const int ngroups_drain = (total + kTcP - 1) / kTcP;
    const uint32_t btile_bytes = (uint32_t)NG * kTcKC * 8;

    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&bar_afull[i], 32 * kBuildWarps);
            tc::mbar_init(&bar_aempty[i], 1);
            tc::mbar_init(&bar_mma[i], 1);
            tc::mbar_init(&bar_tfree[i], 32 * kDrainWarps);
        }
        for (int i = 0; i < kTcBRing; ++i) {
            tc::mbar_init(&bar_bfull[i], 1);
            tc::mbar_init(&bar_bempty[i], 1);
        }
        tc::mbar_fence_init();
    }
    if (warp == 0) tc::tmem_alloc(&tmem_base, kTmemCols);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;

    if (warp < kDrainWarps) {
        // ===================== drainers: TMEM -> fp32 (round-to-nearest) running sums =====================
        float acc[48];
#pragma unroll
        for (int i = 0; i < 48; ++i) acc[i] = 0.0f;
        const uint32_t lane_base = tmem + ((uint32_t)(32 * warp) << 16);
        for (int g = 0; g < ngroups_drain; ++g) {
            const int reg = g & 1;
            tc::mbar_wait(&bar_mma[reg], (g >> 1) & 1);
            tc::fence_after();
            const int nacc = min(2, total - g * kTcP);
            for (int j = 0; j < nacc; ++j) {
#pragma unroll
                for (int c0 = 0; c0 < 48; c0 += 16) {
                    if (c0 < NG) {
                        float v[16];
                        tc::tmem_ld16(lane_base + (uint32_t)(reg * 128 + j * 64 + c0), v);
#pragma unroll
                        for (int i = 0; i < 16; ++i) acc[c0 + i] += v[i];
                    }
                }
            }
            tc::fence_before();
            tc::mbar_arrive(&bar_tfree[reg]);
        }
        // ---- epilogue ----
        const int r = 32 * warp + lane;
        const int p = p0 + r;
        if (p < npix) {
            const int m1 = p / d.nw, m2 = p - (p / d.nw) * d.nw;
#pragma unroll
            for (int i = 0; i < 48; ++i) {
                const int n = grp * NG + i;
                if (i >= NG || n >= N2) break;
                if constexpr (FWD) {   // n = output phase b'
                    const int b1 = n / N, b2 = n - (n / N) * N;
                    out[(size_t)zi * d.H * d.W + (size_t)(b1 + N * m1) * d.W + b2 + N * m2] = acc[i];
                } else {               // n = input phase a of plane z
                    const int u = z * N2 + n;
                    if (u < d.unit0 || u >= d.unit0 + d.nu) continue;
                    const size_t pidx = ((size_t)(u - d.unit0) * d.nh + m1) * d.nw + m2;
                    if constexpr (DST == DST_POLY) {
                        out[pidx] = acc[i];
                    } else if constexpr (DST == DST_VOLIMAGE) {
                        const int a1 = n / N, a2 = n - (n / N) * N;
                        out[((size_t)z * d.H + a1 + N * m1) * d.W + a2 + N * m2] = acc[i];
                    } else {
                        out[pidx] = update_value<DST>(xold[pidx], norm[pidx], acc[i], eps);
                    }
                }
            }
        }
    } else if (warp < kDrainWarps + kBuildWarps) {
        // ===================== builders: windows and shifted A tiles (hi, lo) =====================
        const int bt = tid - 32 * kDrainWarps;           // 0..255
        const int r = bt & (kTcM - 1);                    // pixel row of the A tile
        const int kq0 = bt >> 7;                          // k-quads kq0, kq0+2, kq0+4, kq0+6
        const int p = p0 + r;
        const bool pv = p < npix;
        const int m1 = pv ? p / d.nw : 0, m2 = pv ? p - (p / d.nw) * d.nw : 0;
        // window offset of tap (0,0); a tap (td1, td2) moves it by -(td1*WC + td2) (fwd) or +(td1*WC + td2) (bwd)
        const int base0 = FWD ? (m1 - row0 + d.d1max - d.d1min) * WC + (m2 + d.d2max - d.d2min) : (m1 - row0) * WC + m2;
        const uint32_t aoff = (uint32_t)((r >> 3) * (kTcKC / 4) * 128 + (r & 7) * 16) / 4;   // + kq * 32 floats
        int it = 0;
        for (int c = 0; c < nchunks; ++c) {
            const int k0 = c * kTcKC;
            builders_sync();   // every A build of the previous chunk has read the window
            for (int row = bt >> 5; row < kTcKC * WR; row += kBuildWarps) {
                const int kk = row / WR, wr = row - (row / WR) * WR;
                const int k = k0 + kk;
                float* wrow = win + (size_t)row * WC;
                if (k >= N2) {
                    for (int wc = lane; wc < WC; wc += 32) wrow[wc] = 0.0f;
                    continue;
                }
                if constexpr (FWD) {
                    const int mm1 = row0 - d.d1max + wr;
                    const int u = z * N2 + k;
                    const bool ok = mm1 >= 0 && mm1 < d.nh && u >= d.unit0 && u < d.unit0 + d.nu;
                    const float* srow;
                    if constexpr (SRC == 0) {
                        srow = src + ((size_t)(u - d.unit0) * d.nh + mm1) * d.nw;
                    }
                    for (int wc = lane; wc < WC; wc += 32) {
                        const int mm2 = wc - d.d2max;
                        float v = 0.0f;
                        if (ok && mm2 >= 0 && mm2 < d.nw) {
                            if constexpr (SRC == 0) {
                                v = srow[mm2];
                            } else {
                                const int a1 = k / N, a2 = k - (k / N) * N;
                                v = src[((size_t)z * d.H + a1 + N * mm1) * d.W + a2 + N * mm2];
                            }
                        }
                        wrow[wc] = v;
                    }
                } else {
                    const int mm1 = row0 + d.d1min + wr;
                    const bool ok = mm1 >= 0 && mm1 < d.nh;
                    const int b1 = k / N, b2 = k - (k / N) * N;
                    const size_t rbase = (size_t)(b1 + N * mm1) * d.W + b2;
                    for (int wc = lane; wc < WC; wc += 32) {
                        const int mm2 = d.d2min + wc;
                        float v = 0.0f;
                        if (ok && mm2 >= 0 && mm2 < d.nw) {
                            if constexpr (SRC == SRC_ONES) {
                                v = 1.0f;
                            } else {
                                const size_t pix = rbase + (size_t)N * mm2;
                                if constexpr (SRC == SRC_RATIO)
                                    v = src[pix] / (fmaxf(src2[pix], 0.0f) + eps);
                                else
                                    v = src[pix];
                            }
                        }
                        wrow[wc] = v;
                    }
                }
            }
            builders_sync();
            for (int t = 0; t < NT; ++t, ++it) {
                const int sa = it & 1;
                const int td1 = t / T2, td2 = t - (t / T2) * T2;
                if (it >= 2) tc::mbar_wait(&bar_aempty[sa], ((it - 2) >> 1) & 1);
                float* ahi = reinterpret_cast<float*>(smem + L.a[sa]);
                float* alo = ahi + kTcM * kTcKC;
                const int off = FWD ? base0 - td1 * WC - td2 : base0 + td1 * WC + td2;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int kq = kq0 + 2 * q;
                    float4 hv = make_float4(0.f, 0.f, 0.f, 0.f), lv = hv;
                    if (pv) {
                        const float* w0 = win + (size_t)(4 * kq) * wsz + off;
                        tc::split_tf32(w0[0], hv.x, lv.x);
                        tc::split_tf32(w0[wsz], hv.y, lv.y);
                        tc::split_tf32(w0[2 * wsz], hv.z, lv.z);
                        tc::split_tf32(w0[3 * wsz], hv.w, lv.w);
                    }
                    *reinterpret_cast<float4*>(ahi + aoff + kq * 32) = hv;
                    *reinterpret_cast<float4*>(alo + aoff + kq * 32) = lv;
                }
                tc::fence_proxy_async();
                tc::mbar_arrive(&bar_afull[sa]);
            }
        }
    } else if (lane == 0) {
        // ===================== MMA issuer + coefficient producer (one thread) =====================
        const unsigned char* coef = reinterpret_cast<const unsigned char*>(d.coef) +
                                    ((size_t)zi * d.ngroups + grp) * (size_t)total * btile_bytes;
        const uint32_t idesc = tc::idesc_tf32(kTcM, NG);
        const int pre = min(kTcBRing - 1, total);
        for (int j = 0; j < pre; ++j) {
            tc::mbar_arrive_expect_tx(&bar_bfull[j], btile_bytes);
            tc::bulk_g2s(smem + L.b[j], coef + (size_t)j * btile_bytes, btile_bytes, &bar_bfull[j]);
        }
        for (int it = 0; it < total; ++it) {
            const int c = it / NT;
            const int ksteps = min(kTcKC, d.Kpad - c * kTcKC) / 8;
            const int g = it / kTcP, reg = g & 1;
            if (it % kTcP == 0 && g >= 2) tc::mbar_wait(&bar_tfree[reg], ((g - 2) >> 1) & 1);
            const int sa = it & 1, sb = it % kTcBRing;
            tc::mbar_wait(&bar_afull[sa], (it >> 1) & 1);
            tc::mbar_wait(&bar_bfull[sb], (it / kTcBRing) & 1);
            tc::fence_after();
            const uint32_t a_hi = tc::smem_u32(smem + L.a[sa]), a_lo = a_hi + kTcM * kTcKC * 4;
            const uint32_t b_hi = tc::smem_u32(smem + L.b[sb]), b_lo = b_hi + (uint32_t)NG * kTcKC * 4;
            const uint32_t acc_t = tmem + (uint32_t)(reg * 128 + (it & 1) * 64);
            const bool first = (it % kTcP) < 2;       // first use of this accumulator in the group
            for (int s = 0; s < ksteps; ++s) {
                const uint64_t ah = tc::sdesc(a_hi + s * 256, 128, (kTcKC / 4) * 128);
                const uint64_t al = tc::sdesc(a_lo + s * 256, 128, (kTcKC / 4) * 128);
                const uint64_t bh = tc::sdesc(b_hi + s * 256, 128, (kTcKC / 4) * 128);
                const uint64_t bl = tc::sdesc(b_lo + s * 256, 128, (kTcKC / 4) * 128);
                tc::mma_tf32(acc_t, ah, bh, idesc, (first && s == 0) ? 0u : 1u);
                tc::mma_tf32(acc_t, ah, bl, idesc, 1u);
                tc::mma_tf32(acc_t, al, bh, idesc, 1u);
            }
            tc::mma_commit(&bar_aempty[sa]);
            tc::mma_commit(&bar_bempty[sb]);
            if (it % kTcP == kTcP - 1 || it == total - 1) tc::mma_commit(&bar_mma[reg]);
            // refill the B ring: tile it+kTcBRing-1 goes to the slot of tile it-1 (wait for its MMAs)
            const int j = it + kTcBRing - 1;
            if (j < total) {
                const int sj = j % kTcBRing;
                if (j >= kTcBRing) tc::mbar_wait(&bar_bempty[sj], ((j - kTcBRing) / kTcBRing) & 1);
                tc::mbar_arrive_expect_tx(&bar_bfull[sj], btile_bytes);
                tc::bulk_g2s(smem + L.b[sj], coef + (size_t)j * btile_bytes, btile_bytes, &bar_bfull[sj]);
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, kTmemCols);
}

template <bool FWD, int SRC, int DST>
static cudaError_t tcdir_launch(const TcDirArgs& d, const float* src, const float* src2, float eps, float* out,
                                const float* xold, const float* norm, cudaStream_t s) {
    const TcSmem L = tc_smem_layout(d.NG, d.WR, d.WC);
    cudaError_t e = cudaFuncSetAttribute(tcdir_kernel<FWD, SRC, DST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)L.total);
    if (e != cudaSuccess) return e;
    dim3 grid((d.nh * d.nw + kTcM - 1) / kTcM, d.ngroups, d.nzd);
    tcdir_kernel<FWD, SRC, DST><<<grid, kTcThreads, L.total, s>>>(d, src, src2, eps, out, xold, norm);
    return cudaGetLastError();
}

size_t tcdir_smem_bytes(int NG, int WR, int WC) { return tc_smem_layout(NG, WR, WC).total; }

cudaError_t launch_tcdir_fwd(const TcDirArgs& d, const float* x, int src_image, float* part, float* y, int accumulate,
                             cudaStream_t s) {
    if (d.nzd <= 0) return cudaSuccess;
    cudaError_t e = src_image ? tcdir_launch<true, 1, 0>(d, x, nullptr, 0.f, part, nullptr, nullptr, s)
                              : tcdir_launch<true, 0, 0>(d, x, nullptr, 0.f, part, nullptr, nullptr, s);
    if (e != cudaSuccess) return e;
    return launch_plane_reduce(part, d.nzd, (size_t)d.H * d.W, y, accumulate, s);
}

cudaError_t launch_tcdir_bwd(const TcDirArgs& d, int src, const float* img, const float* img2, float eps, int dst,
                             float* out, const float* xold, const float* norm, cudaStream_t s) {
    if (d.nzd <= 0) return cudaSuccess;
#define LFM_TCB(SRCV, DSTV) \
    if (src == SRCV && dst == DSTV) return tcdir_launch<false, SRCV, DSTV>(d, img, img2, eps, out, xold, norm, s);
    LFM_TCB(SRC_RATIO, DST_UPDATE)
    LFM_TCB(SRC_IMAGE2D, DST_ISRA)
    LFM_TCB(SRC_ONES, DST_POLY)
    LFM_TCB(SRC_IMAGE2D, DST_VOLIMAGE)
    LFM_TCB(SRC_IMAGE2D, DST_POLY)
    LFM_TCB(SRC_RATIO, DST_POLY)
#undef LFM_TCB
    return cudaErrorInvalidValue;
}

}  // namespace lfm

namespace lfm {

// Coefficient tiles for the tensor-core direct path, built on the device from the owned PSF slice:
// tile (zi, grp, chunk, tap) = [hi | lo] of an NG x 32 K-major core-matrix tile whose element (n, k) is
//   forward : G_d[b' = grp*NG + n][a = chunk*32 + k]      backward: G_d[b' = chunk*32 + k][a = grp*NG + n]
// with G_d[b'][a] = h_{z,a}[b1 - a1 + ch + N d1][b2 - a2 + cw + N d2] (0 outside the kernel / phases).
__global__ void tcdir_coef_kernel(TcDirArgs d, const int* __restrict__ zlist_host_order, const float* __restrict__ psf,
                                  int kh, int kw, int ch, int cw, int fwd, float* __restrict__ out) {
    const int nchunks = d.Kpad / kTcKC + (d.Kpad % kTcKC ? 1 : 0);
    const int NT = d.T1 * d.T2;
    const int tile = blockIdx.x;   // ((zi * ngroups + grp) * nchunks + chunk) * NT + tap
    const int tap = tile % NT;
    const int chunk = (tile / NT) % nchunks;
    const int grp = (tile / (NT * nchunks)) % d.ngroups;
    const int zi = tile / (NT * nchunks * d.ngroups);
    const int z = zlist_host_order[zi];
    const int N = d.N, N2 = N * N;
    const int d1 = d.d1min + tap / d.T2, d2 = d.d2min + tap % d.T2;
    float* hi = out + (size_t)tile * d.NG * kTcKC * 2;
    float* lo = hi + (size_t)d.NG * kTcKC;
    for (int e = threadIdx.x; e < d.NG * kTcKC; e += blockDim.x) {
        const int n = e / kTcKC, k = e - (e / kTcKC) * kTcKC;
        const int ng = grp * d.NG + n, kg = chunk * kTcKC + k;
        const int bp = fwd ? ng : kg, a = fwd ? kg : ng;
        float v = 0.0f;
        if (bp < N2 && a < N2) {
            const int u = z * N2 + a;
            if (u >= d.unit0 && u < d.unit0 + d.nu) {
                const int b1 = bp / N, b2 = bp % N, a1 = a / N, a2 = a % N;
                const int k1 = b1 - a1 + ch + N * d1, k2 = b2 - a2 + cw + N * d2;
                if (k1 >= 0 && k1 < kh && k2 >= 0 && k2 < kw) v = psf[((size_t)(u - d.unit0) * kh + k1) * kw + k2];
            }
        }
        float h, l;
        tc::split_tf32(v, h, l);
        const uint32_t off = tc::kmajor_off(n, k, kTcKC) / 4;
        hi[off] = h;
        lo[off] = l;
    }
}

cudaError_t launch_tcdir_coef(const TcDirArgs& d, const int* zlist_dev, const float* psf_dev, int kh, int kw, int ch,
                              int cw, int fwd, float* out, cudaStream_t s) {
    const int nchunks = d.Kpad / kTcKC + (d.Kpad % kTcKC ? 1 : 0);
    const long long tiles = (long long)d.nzd * d.ngroups * nchunks * d.T1 * d.T2;
    if (tiles <= 0) return cudaSuccess;
    tcdir_coef_kernel<<<(unsigned)tiles, 256, 0, s>>>(d, zlist_dev, psf_dev, kh, kw, ch, cw, fwd, out);
    return cudaGetLastError();
}

size_t tcdir_coef_floats(const TcDirArgs& d) {
    const int nchunks = d.Kpad / kTcKC + (d.Kpad % kTcKC ? 1 : 0);
    return (size_t)d.nzd * d.ngroups * nchunks * d.T1 * d.T2 * d.NG * kTcKC * 2;
}

}  // namespace lfm
