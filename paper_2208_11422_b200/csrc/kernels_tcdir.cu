// kernels_tcdir.cu -- direct polyphase projections of near-focus planes on the 5th-generation tensor cores
// (K9tc).  fp32-accurate through the 3xTF32 split (a*b ~ ah*bh + ah*bl + al*bh).
//
// For one plane z the direct path is a sum over coarse taps d of dense contractions over phases
// (G_d[b'][a] = h_{z,a}[b1 - a1 + c + N d1][b2 - a2 + c + N d2], zero outside the kernel):
//   forward : Y[m'][b']  = sum_d sum_a  X_a[m' - d] * G_d[b'][a]      (K = input phases a,  N = output phases b')
//   backward: Xh[m][a]   = sum_d sum_b' r_b'[m + d] * G_d[b'][a]      (K = output phases b', N = input phases a)
// Mapping onto tcgen05 (M = 128 coarse pixels = TMEM lanes, N = all phases <= 256 TMEM columns, K = 32-phase
// chunks): every (tap, chunk) is one pipeline stage
//   * A (128 pixels x 32 phases, hi and lo) is ONE 3-D TMA box each from a per-iteration staged copy of the
//     source on a padded coarse grid -- a tap is only a row offset of the box, borders come from TMA's zero fill;
//   * B (the tap's Ntile x 32 coefficient tile, hi and lo, pre-swizzled at plan time) is one 1-D bulk copy;
//   * one thread issues 3 x ksteps tcgen05.mma.kind::tf32 (K = 8 each) into a fresh TMEM accumulator;
//   * 8 drainer warps add the accumulator into fp32 registers with round-to-nearest after every stage
//     (tcgen05's fp32 accumulation truncates; a 12-MMA chain keeps that bias below 1e-6 relative), while the
//     tensor core fills the other accumulator.
// One launch per direction covers every tensor-core plane: persistent CTAs walk a static LPT schedule of
// (plane, pixel tile) items; forward items write per-plane partial images (summed over planes in a fixed order
// afterwards -> deterministic), backward items write the plane's update epilogue directly.
#include <algorithm>

#include "lfm_internal.cuh"
#include "tc_sm100.cuh"

namespace lfm {

namespace {
constexpr int kM = 128;            // pixels per tile (TMEM lanes)
constexpr int kKC = 32;            // phases per chunk (one 128-byte swizzle row)
constexpr int kStages = 2;         // smem pipeline depth (A hi/lo + B hi/lo per stage)
constexpr int kDrainWarps = 8;     // warps 2..9: two per TMEM lane quarter, half of the columns each
constexpr int kThreads = 32 * (2 + kDrainWarps);
constexpr int kMaxNh = 128;        // columns per drainer thread
constexpr uint32_t kTmemCols = 512;   // 2 accumulators x 256 columns
constexpr uint32_t kATile = kM * kKC * 4;   // 16 KB

__host__ __device__ inline uint32_t stage_bytes(int Ntile) { return 2 * kATile + 2u * (uint32_t)Ntile * kKC * 4; }
}  // namespace

size_t tcdir_smem_bytes(int Ntile) { return (size_t)kStages * stage_bytes(Ntile) + 1024; }

// ------------------------------------------------------------------------------------------------
template <bool FWD, int DST>
__global__ void __launch_bounds__(kThreads, 1) tcdir_kernel(const __grid_constant__ TcDirArgs d, const float* __restrict__ xold,
                                                            const float* __restrict__ norm, float eps, float* __restrict__ out) {
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t bar_full[kStages], bar_empty[kStages], bar_acc[2], bar_tfree[2];
    __shared__ uint32_t tmem_base;
    const uint32_t raw = tc::smem_u32(smem_raw);
    unsigned char* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);   // SWIZZLE_128B tiles: 1024-byte aligned
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ib = d.item_off[blockIdx.x], ie = d.item_off[blockIdx.x + 1];
    const uint32_t sbytes = stage_bytes(d.Ntile);
    const uint32_t bbytes = 2u * (uint32_t)d.Ntile * kKC * 4;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            tc::mbar_init(&bar_full[i], 1);
            tc::mbar_init(&bar_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&bar_acc[i], 1);
            tc::mbar_init(&bar_tfree[i], kDrainWarps);
        }
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&d.tmap);
    }
    if (warp == 0) tc::tmem_alloc(&tmem_base, kTmemCols);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            // ============================ producer: TMA (A) + bulk copy (B) ============================
            int it = 0;
            for (int i = ib; i < ie; ++i) {
                const int item = d.items[i], zi = item / d.tiles, tile = item - zi * d.tiles;
                const TcPlane pl = d.planes[zi];
                const unsigned char* coef = reinterpret_cast<const unsigned char*>(d.coef + pl.coef_off);
                for (int c = 0; c < d.nch; ++c)
                    for (int t = 0; t < pl.T1 * pl.T2; ++t, ++it) {
                        const int s = it % kStages;
                        if (it >= kStages) tc::mbar_wait(&bar_empty[s], ((it / kStages) - 1) & 1);
                        unsigned char* st = smem + (size_t)s * sbytes;
                        const int e1 = pl.e1min + t / pl.T2, e2 = pl.e2min + t % pl.T2;
                        const int row = tile * kM + e1 * d.Wp + e2 - d.e2lo;
                        const int slab_hi = FWD ? (zi * 2) * d.nch + c : c;
                        const int slab_lo = FWD ? (zi * 2 + 1) * d.nch + c : d.nch + c;
                        tc::mbar_arrive_expect_tx(&bar_full[s], sbytes);
                        tc::tma_load_3d(st, &d.tmap, 0, row, slab_hi, &bar_full[s]);
                        tc::tma_load_3d(st + kATile, &d.tmap, 0, row, slab_lo, &bar_full[s]);
                        tc::bulk_g2s(st + 2 * kATile, coef + ((size_t)t * d.nch + c) * bbytes, bbytes, &bar_full[s]);
                    }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ============================ MMA issuer (one thread) ============================
            const uint32_t idesc = tc::idesc_tf32(kM, d.Ntile);
            int it = 0;
            for (int i = ib; i < ie; ++i) {
                const int zi = d.items[i] / d.tiles;
                const int NT = d.planes[zi].T1 * d.planes[zi].T2;
                for (int c = 0; c < d.nch; ++c) {
                        const int ks = c == d.nch - 1 ? d.kst_last : kKC / 8;
                    for (int t = 0; t < NT; ++t, ++it) {
                            const int s = it % kStages, j = it & 1;
                            tc::mbar_wait(&bar_full[s], (it / kStages) & 1);
                            if (it >= 2) tc::mbar_wait(&bar_tfree[j], ((it >> 1) - 1) & 1);
                            tc::fence_after();
                            const uint32_t a_hi = tc::smem_u32(smem + (size_t)s * sbytes), a_lo = a_hi + kATile;
                            const uint32_t b_hi = a_hi + 2 * kATile, b_lo = b_hi + (uint32_t)d.Ntile * kKC * 4;
                            const uint32_t acc = tmem + (uint32_t)(j * 256);
                            for (int k = 0; k < ks; ++k) {
                                const uint64_t ah = tc::sdesc_sw128(a_hi + 32 * k), al = tc::sdesc_sw128(a_lo + 32 * k);
                                const uint64_t bh = tc::sdesc_sw128(b_hi + 32 * k), bl = tc::sdesc_sw128(b_lo + 32 * k);
                                tc::mma_tf32(acc, ah, bh, idesc, k > 0 ? 1u : 0u);
                                tc::mma_tf32(acc, ah, bl, idesc, 1u);
                                tc::mma_tf32(acc, al, bh, idesc, 1u);
                            }
                            tc::mma_commit(&bar_empty[s]);
                            tc::mma_commit(&bar_acc[j]);
                        }
                    }
            }
        }
    } else {
        // ============================ drainers: TMEM -> fp32 running sums, epilogue ============================
        const int q = warp & 3;                       // TMEM lane quarter this warp may access
        const int half = (warp - 2) >> 2;             // column half
        const int Nh = d.Ntile >> 1;
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(half * Nh);
        const int r = 32 * q + lane;                  // tile row (pixel) of this thread
        float acc[kMaxNh];
#pragma unroll
        for (int i = 0; i < kMaxNh; ++i) acc[i] = 0.0f;
        int it = 0;
        for (int i = ib; i < ie; ++i) {
            const int item = d.items[i], zi = item / d.tiles, tile = item - zi * d.tiles;
            const int nst = d.nch * d.planes[zi].T1 * d.planes[zi].T2;
            for (int st = 0; st < nst; ++st, ++it) {
                const int j = it & 1;
                tc::mbar_wait(&bar_acc[j], (it >> 1) & 1);
                tc::fence_after();
                const uint32_t base = lane_base + (uint32_t)(j * 256);
#pragma unroll
                for (int c0 = 0; c0 < kMaxNh; c0 += 32) {
                    if (c0 < Nh) {
                        uint32_t v[32];
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (c0 + 8 * u < Nh) tc::tmem_ld8_nowait(base + (uint32_t)(c0 + 8 * u), v + 8 * u);
                        tc::tmem_wait_ld();
#pragma unroll
                        for (int u = 0; u < 32; ++u)
                            if (c0 + u < Nh) acc[c0 + u] += __uint_as_float(v[u]);
                    }
                }
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar_tfree[j]);
            }
            // ---- epilogue of the item ----
            const int L = tile * kM + r;
            const int m1 = L / d.Wp, m2 = L - (L / d.Wp) * d.Wp;
            if (m1 < d.nh && m2 < d.nw) {
                const size_t HW = (size_t)d.H * d.W;
#pragma unroll
                for (int i = 0; i < kMaxNh; ++i) {
                    const int n = half * Nh + i;
                    if (i < Nh && n < d.N2) {
                        const int n1 = n / d.N, n2 = n - (n / d.N) * d.N;
                        if constexpr (FWD) {   // n = output phase b'
                            d.part[(size_t)zi * HW + (size_t)(n1 + d.N * m1) * d.W + n2 + d.N * m2] = acc[i];
                        } else {               // n = input phase a of plane z
                            const int z = d.zlist[zi];
                            const int u = z * d.N2 + n;
                            if (u >= d.unit0 && u < d.unit0 + d.nu) {
                                const size_t pidx = ((size_t)(u - d.unit0) * d.nh + m1) * d.nw + m2;
                                if constexpr (DST == DST_POLY)
                                    out[pidx] = acc[i];
                                else if constexpr (DST == DST_VOLIMAGE)
                                    out[((size_t)z * d.H + n1 + d.N * m1) * d.W + n2 + d.N * m2] = acc[i];
                                else
                                    out[pidx] = update_value<DST>(xold[pidx], norm[pidx], acc[i], eps);
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < kMaxNh; ++i) acc[i] = 0.0f;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, kTmemCols);
}

// ------------------------------------------------------------------------------------------------
// Source staging: slab rows L of the padded grid (m1 = L / Wp, m2 = L % Wp + e2lo), 32 phases per row,
// hi = tf32(v), lo = tf32(v - hi).  A 32-row x 32-phase tile per block, transposed through shared memory.
//   forward  (SRC 0 polyphase volume [nu][nh][nw], 1 image-layout volume [nz][H][W]): plane blockIdx.z
//   backward (SRC_RATIO y / (max(yhat,0)+eps), SRC_ONES, SRC_IMAGE2D): one image
template <bool FWD, int SRC>
__global__ void __launch_bounds__(256) tc_stage_kernel(const __grid_constant__ TcDirArgs d, const float* __restrict__ src,
                                                       const float* __restrict__ src2, float eps) {
    __shared__ float tile[kKC][33];
    const int L0 = blockIdx.x * 32, c = blockIdx.y, zi = blockIdx.z;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    {
        const int L = L0 + tx;
        const int m1 = L / d.Wp, m2 = L - (L / d.Wp) * d.Wp + d.e2lo;
        const bool pv = L < d.Lp && m1 < d.nh && m2 >= 0 && m2 < d.nw;
        for (int k = ty; k < kKC; k += 8) {
            const int ph = c * kKC + k;
            float v = 0.0f;
            if (pv && ph < d.N2) {
                const int p1 = ph / d.N, p2 = ph - (ph / d.N) * d.N;
                if constexpr (FWD) {
                    const int z = d.zlist[zi];
                    const int u = z * d.N2 + ph;
                    if (u >= d.unit0 && u < d.unit0 + d.nu) {
                        if constexpr (SRC == 0)
                            v = src[((size_t)(u - d.unit0) * d.nh + m1) * d.nw + m2];
                        else
                            v = src[((size_t)z * d.H + p1 + d.N * m1) * d.W + p2 + d.N * m2];
                    }
                } else {
                    const size_t pix = (size_t)(p1 + d.N * m1) * d.W + p2 + d.N * m2;
                    if constexpr (SRC == SRC_ONES)
                        v = 1.0f;
                    else if constexpr (SRC == SRC_RATIO)
                        v = src[pix] / (fmaxf(src2[pix], 0.0f) + eps);
                    else
                        v = src[pix];
                }
            }
            tile[k][tx] = v;
        }
    }
    __syncthreads();
    const size_t slab_hi = FWD ? ((size_t)zi * 2) * d.nch + c : (size_t)c;
    const size_t slab_lo = FWD ? ((size_t)zi * 2 + 1) * d.nch + c : (size_t)d.nch + c;
    for (int rr = ty; rr < 32; rr += 8) {
        const int L = L0 + rr;
        if (L >= d.Lp) break;
        float h, l;
        tc::split_tf32(tile[tx][rr], h, l);
        d.src[(slab_hi * d.Lp + L) * kKC + tx] = h;
        d.src[(slab_lo * d.Lp + L) * kKC + tx] = l;
    }
}

// ------------------------------------------------------------------------------------------------
// Coefficient tiles of one plane (plan time), built on the device from the owned PSF slice: tile (tap, chunk) =
// [hi | lo] of an Ntile x 32 SWIZZLE_128B K-major tile with element (n, k) =
//   forward : G_d[b' = n][a = chunk*32 + k],   d = -e        backward: G_d[b' = chunk*32 + k][a = n],   d = +e
__global__ void tcdir_coef_kernel(const __grid_constant__ TcDirArgs d, TcPlane pl, int z, const float* __restrict__ psf,
                                  int kh, int kw, int ch, int cw, int fwd, float* __restrict__ out) {
    const int tileid = blockIdx.x;   // tap * nch + chunk
    const int chunk = tileid % d.nch;
    const int tap = tileid / d.nch;
    const int N = d.N, N2 = d.N2;
    const int e1 = pl.e1min + tap / pl.T2, e2 = pl.e2min + tap % pl.T2;
    const int d1 = fwd ? -e1 : e1, d2 = fwd ? -e2 : e2;
    float* hi = out + pl.coef_off + (size_t)tileid * d.Ntile * kKC * 2;
    float* lo = hi + (size_t)d.Ntile * kKC;
    for (int e = threadIdx.x; e < d.Ntile * kKC; e += blockDim.x) {
        const int n = e / kKC, k = e - (e / kKC) * kKC;
        const int kg = chunk * kKC + k;
        const int bp = fwd ? n : kg, a = fwd ? kg : n;
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
        const uint32_t off = tc::sw128_off(n, k) / 4;
        hi[off] = h;
        lo[off] = l;
    }
}

// ------------------------------------------------------------------------------------------------
// host side

bool tcdir_geometry(TcDirArgs* d, int fwd, const int* d1min, const int* d1max, const int* d2min, const int* d2max,
                    std::vector<TcPlane>* planes, int num_sms) {
    d->N2 = d->N * d->N;
    d->Ntile = (d->N2 + 15) / 16 * 16;
    if (d->Ntile > 2 * kMaxNh) return false;
    d->nch = (d->N2 + kKC - 1) / kKC;
    d->kst_last = ((d->N2 - (d->nch - 1) * kKC) + 7) / 8;
    planes->assign(d->nzd, TcPlane{});
    int e2lo = 1 << 30, e2hi = -(1 << 30);
    long long off = 0;
    for (int zi = 0; zi < d->nzd; ++zi) {
        TcPlane& pl = (*planes)[zi];
        pl.T1 = d1max[zi] - d1min[zi] + 1;
        pl.T2 = d2max[zi] - d2min[zi] + 1;
        pl.e1min = fwd ? -d1max[zi] : d1min[zi];
        pl.e2min = fwd ? -d2max[zi] : d2min[zi];
        pl.coef_off = off;
        off += (long long)pl.T1 * pl.T2 * d->nch * d->Ntile * kKC * 2;
        e2lo = std::min(e2lo, pl.e2min);
        e2hi = std::max(e2hi, pl.e2min + pl.T2 - 1);
    }
    d->e2lo = d->nzd > 0 ? e2lo : 0;
    d->Wp = d->nw + (d->nzd > 0 ? e2hi - e2lo : 0);
    d->Lp = d->nh * d->Wp;
    d->tiles = (d->Lp + kM - 1) / kM;
    d->grid = std::max(1, std::min(d->tiles * d->nzd, num_sms));
    return true;
}

void tcdir_schedule(const TcDirArgs& d, const std::vector<TcPlane>& planes, std::vector<int>* item_off,
                    std::vector<int>* items) {
    // longest-processing-time-first: items sorted by cost (taps), each to the least-loaded CTA
    std::vector<std::pair<long long, int>> it;
    for (int zi = 0; zi < d.nzd; ++zi)
        for (int t = 0; t < d.tiles; ++t) it.push_back({(long long)planes[zi].T1 * planes[zi].T2, zi * d.tiles + t});
    std::stable_sort(it.begin(), it.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
    std::vector<long long> load(d.grid, 0);
    std::vector<std::vector<int>> per(d.grid);
    for (const auto& x : it) {
        int best = 0;
        for (int b = 1; b < d.grid; ++b)
            if (load[b] < load[best]) best = b;
        load[best] += x.first;
        per[best].push_back(x.second);
    }
    item_off->assign(1, 0);
    items->clear();
    for (int b = 0; b < d.grid; ++b) {
        std::sort(per[b].begin(), per[b].end());   // plane-major within a CTA (L2 locality of the staged source)
        items->insert(items->end(), per[b].begin(), per[b].end());
        item_off->push_back((int)items->size());
    }
}

size_t tcdir_coef_floats(const TcDirArgs& d, const std::vector<TcPlane>& planes) {
    size_t n = 0;
    for (const TcPlane& pl : planes) n += (size_t)pl.T1 * pl.T2 * d.nch * d.Ntile * kKC * 2;
    return n;
}
size_t tcdir_src_floats(const TcDirArgs& d, int fwd) { return (size_t)(fwd ? 2 * d.nzd : 2) * d.nch * d.Lp * kKC; }
size_t tcdir_part_floats(const TcDirArgs& d, int fwd) { return fwd ? (size_t)d.nzd * d.H * d.W : 0; }

typedef CUresult (*TmapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t tcdir_encode(TcDirArgs* d, int fwd) {
    static TmapEncodeFn enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
        if (e != cudaSuccess || !enc || q != cudaDriverEntryPointSuccess) {
            enc = nullptr;
            return e != cudaSuccess ? e : cudaErrorSymbolNotFound;
        }
    }
    const cuuint64_t slabs = (cuuint64_t)(fwd ? 2 * d->nzd : 2) * d->nch;
    cuuint64_t dims[3] = {(cuuint64_t)kKC, (cuuint64_t)d->Lp, slabs};
    cuuint64_t strides[2] = {(cuuint64_t)kKC * 4, (cuuint64_t)d->Lp * kKC * 4};
    cuuint32_t box[3] = {(cuuint32_t)kKC, (cuuint32_t)kM, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&d->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d->src, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_tcdir_coef(const TcDirArgs& d, const TcPlane& pl, int zi, int z, const float* psf_dev, int kh,
                              int kw, int ch, int cw, int fwd, float* coef, cudaStream_t s) {
    (void)zi;
    const int tiles = pl.T1 * pl.T2 * d.nch;
    if (tiles <= 0) return cudaSuccess;
    tcdir_coef_kernel<<<tiles, 256, 0, s>>>(d, pl, z, psf_dev, kh, kw, ch, cw, fwd, coef);
    return cudaGetLastError();
}

template <bool FWD, int DST>
static cudaError_t tcdir_main(const TcDirArgs& d, const float* xold, const float* norm, float eps, float* out,
                              cudaStream_t s) {
    const size_t smem = tcdir_smem_bytes(d.Ntile);
    cudaError_t e = cudaFuncSetAttribute(tcdir_kernel<FWD, DST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    tcdir_kernel<FWD, DST><<<d.grid, kThreads, smem, s>>>(d, xold, norm, eps, out);
    return cudaGetLastError();
}

template <bool FWD, int SRC>
static cudaError_t tc_stage(const TcDirArgs& d, const float* src, const float* src2, float eps, cudaStream_t s) {
    dim3 grid((d.Lp + 31) / 32, d.nch, FWD ? d.nzd : 1);
    tc_stage_kernel<FWD, SRC><<<grid, 256, 0, s>>>(d, src, src2, eps);
    return cudaGetLastError();
}

cudaError_t launch_tcdir_fwd(const TcDirArgs& d, const float* x, int src_image, float* y, int accumulate,
                             cudaStream_t s) {
    if (d.nzd <= 0) return cudaSuccess;
    cudaError_t e = src_image ? tc_stage<true, 1>(d, x, nullptr, 0.f, s) : tc_stage<true, 0>(d, x, nullptr, 0.f, s);
    if (e != cudaSuccess) return e;
    e = tcdir_main<true, 0>(d, nullptr, nullptr, 0.f, nullptr, s);
    if (e != cudaSuccess) return e;
    return launch_plane_reduce(d.part, d.nzd, (size_t)d.H * d.W, y, accumulate, s);
}

cudaError_t launch_tcdir_bwd(const TcDirArgs& d, int src, const float* img, const float* img2, float eps, int dst,
                             float* out, const float* xold, const float* norm, cudaStream_t s) {
    if (d.nzd <= 0) return cudaSuccess;
    cudaError_t e;
    switch (src) {
        case SRC_RATIO: e = tc_stage<false, SRC_RATIO>(d, img, img2, eps, s); break;
        case SRC_ONES: e = tc_stage<false, SRC_ONES>(d, nullptr, nullptr, eps, s); break;
        case SRC_IMAGE2D: e = tc_stage<false, SRC_IMAGE2D>(d, img, nullptr, eps, s); break;
        default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    switch (dst) {
        case DST_UPDATE: return tcdir_main<false, DST_UPDATE>(d, xold, norm, eps, out, s);
        case DST_ISRA: return tcdir_main<false, DST_ISRA>(d, xold, norm, eps, out, s);
        case DST_POLY: return tcdir_main<false, DST_POLY>(d, xold, norm, eps, out, s);
        case DST_VOLIMAGE: return tcdir_main<false, DST_VOLIMAGE>(d, xold, norm, eps, out, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lfm
