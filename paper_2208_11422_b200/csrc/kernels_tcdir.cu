// kernels_tcdir.cu -- direct polyphase projections of near-focus planes on the 5th-generation tensor cores
// (K9tc).  fp32-accurate through a 2 x fp16 split of power-of-two scaled operands
// (a*b ~ ah*bh + ah*bl + al*bh, "3xFP16" on tcgen05 kind::f16: 22 significant bits per operand, as 3xTF32 has, at
// twice the tf32 tensor rate).
//
// For one plane z the direct path is a sum over coarse taps d of dense contractions over phases
// (G_d[b'][a] = h_{z,a}[b1 - a1 + c + N d1][b2 - a2 + c + N d2], zero outside the kernel):
//   forward : Y[m'][b']  = sum_d sum_a  X_a[m' - d] * G_d[b'][a]      (K = input phases a,  N = output phases b')
//   backward: Xh[m][a]   = sum_d sum_b' r_b'[m + d] * G_d[b'][a]      (K = output phases b', N = input phases a)
// Mapping onto tcgen05 (M = 128 coarse pixels = TMEM lanes, N = all phases <= 256 TMEM columns, K = 64-phase
// chunks, one 128-byte row of fp16): every (tap, chunk) is one pipeline stage
//   * A (128 pixels x 64 phases, hi and lo) is ONE 3-D TMA box each from a per-iteration staged copy of the
//     source on a padded coarse grid -- a tap is only a row offset of the box, borders come from TMA's zero fill;
//   * B (the tap's Ntile x 64 coefficient tile, hi and lo, split at plan time) is one TMA box each;
//   * CTA pairs (cta_group::2, M = 256 pixels); the issuer warp runs converged on warp-uniform values and one elected
//     lane issues 3 tcgen05.mma.kind::f16 (K = 16 each) per K-step, over the tile's nonzero column range;
//   * 8 drainer warps add the accumulator into fp32 registers with round-to-nearest after every drain group of
//     <= 24 K-steps (72 MMAs; tcgen05's fp32 accumulation truncates, the chain bounds that bias to ~3e-6 relative),
//     zero it with tcgen05.st and hand it back while the tensor core fills the other accumulator.
// One launch per direction covers every tensor-core plane: persistent CTA pairs walk a static LPT schedule of
// (plane, pixel tile) items; forward items write per-plane partial images (summed over planes in a fixed order
// afterwards -> deterministic), backward items write H^T r for the update kernel.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "lfm_internal.cuh"
#include "tc_sm100.cuh"

namespace lfm {

namespace {
constexpr int kM = 128;            // pixels per CTA tile (TMEM lanes); a CTA pair covers 2 * kM pixels
constexpr int kKC = 64;            // phases per chunk (one 128-byte swizzle row of fp16)
constexpr int kKS = kKC / 16;      // K-steps (kind::f16, K = 16) per full chunk
constexpr int kStagePB = 4;        // 32-pixel blocks per tc_stage_kernel CTA
constexpr int kASlots = 2;         // A windows in flight (one per 32-phase chunk x tap row e1)
constexpr int kBSlots = 5;         // coefficient tiles in flight (one per tap)
constexpr int kDrainWarps = 8;     // warps 2..9: two per TMEM lane quarter, half of the columns each
constexpr int kThreads = 32 * (2 + kDrainWarps);
constexpr int kMaxNh = 128;        // columns per drainer thread
constexpr uint32_t kTmemCols = 512;   // 2 accumulators x 256 columns
constexpr int kChainK = 24;        // default K-steps (x3 MMAs) accumulated in TMEM between round-to-nearest drains
                                   // (16 -> 24: -2 % tcgen05 time at c3; parity tests pass up to 32)

// per-CTA smem: A windows (hi | lo, Arows = 128 + T2max - 1 rows of 128 B each part) and B tiles (hi | lo,
// Ntile/2 rows each: the pair splits B along N); every part 1024-byte aligned (SWIZZLE_128B atoms)
__host__ __device__ inline uint32_t round1k(uint32_t v) { return (v + 1023u) & ~1023u; }
__host__ __device__ inline uint32_t apart_bytes(int Arows) { return round1k((uint32_t)Arows * 128u); }
__host__ __device__ inline uint32_t bhalf_bytes(int Ntile) { return round1k((uint32_t)(Ntile / 2) * 128u); }
}  // namespace

size_t tcdir_smem_bytes(int Ntile, int Arows) {
    return (size_t)kASlots * 2 * apart_bytes(Arows) + (size_t)kBSlots * 2 * bhalf_bytes(Ntile) + 1024;
}

// ------------------------------------------------------------------------------------------------
// CTA pair (cluster of 2, cta_group::2): CTA rank r owns pixel rows [pair_tile*256 + 128 r, +128) of the padded
// grid and B rows [r*Ntile/2, (r+1)*Ntile/2); the leader (rank 0) issues M=256 x N=Ntile MMAs for both; each CTA
// drains its own TMEM lanes.  A is loaded once per (chunk, tap row e1) as a window of 128 + T2 - 1 rows: the taps
// e2 of that row read it at a row offset (the 128-byte swizzle is address based, so any row start works).
// Barriers: fullA/fullB and tfree live in the leader (both CTAs' TMA bytes / drainer warps count there);
// emptyA/emptyB and acc in both CTAs (the leader's commits multicast to the pair).
template <bool FWD, int DST>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tcdir_kernel(const __grid_constant__ TcDirArgs d, const float* __restrict__ xold, const float* __restrict__ norm,
                 float eps, float* __restrict__ out) {
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t bar_fullA[kASlots], bar_emptyA[kASlots], bar_fullB[kBSlots], bar_emptyB[kBSlots];
    __shared__ uint64_t bar_acc[2], bar_tfree[2];
    __shared__ uint32_t tmem_base;
    const uint32_t raw = tc::smem_u32(smem_raw);
    unsigned char* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);   // SWIZZLE_128B tiles: 1024-byte aligned
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int pair = blockIdx.x >> 1;
    const int ib = d.item_off[pair], ie = d.item_off[pair + 1];
    const uint32_t apart = apart_bytes(d.Arows), bhalf = bhalf_bytes(d.Ntile);
    unsigned char* Abase = smem;
    unsigned char* Bbase = smem + (size_t)kASlots * 2 * apart;
    const int Nh = d.Ntile >> 1;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kASlots; ++i) {
            tc::mbar_init(&bar_fullA[i], 1);
            tc::mbar_init(&bar_emptyA[i], 1);
        }
        for (int i = 0; i < kBSlots; ++i) {
            tc::mbar_init(&bar_fullB[i], 1);
            tc::mbar_init(&bar_emptyB[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&bar_acc[i], 1);
            tc::mbar_init(&bar_tfree[i], 2 * kDrainWarps);
        }
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&d.tmap);
        tc::tma_prefetch_desc(&d.bmap);
    }
    if (warp == 0) tc::tmem_alloc_pair(&tmem_base, kTmemCols);
    tc::fence_before();
    tc::cluster_sync();
    tc::fence_after();
    const uint32_t tmem = tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            // ============================ producer (both CTAs): TMA A windows + B halves ============================
            int na = 0, nb = 0;
            long long dbg_empty = 0, dbg_t0 = clock64();
            // A windows and coefficient tiles are re-read from L2 by other CTAs (taps, pixel tiles): keep them there
            // ahead of a concurrent MAC's evict-first stream (§5.5; LFM_TC_EXP bit 8 turns the hint off)
            const uint64_t pol = tc::policy_evict_last();
            const bool hint = !(d.exp & 8);
            const bool ranged = !(d.exp & 16);   // LFM_TC_EXP bit 16: full-width MMAs (no column ranges)
            for (int i = ib; i < ie; ++i) {
                const int item = d.items[i], zi = item / d.tiles, tile = item - zi * d.tiles;
                const TcPlane pl = d.planes[zi];
                const int* rm = d.rowmask + pl.mask_off;
                const int row0 = tile * 2 * kM + (int)rank * kM - d.e2lo + pl.e2min;
                for (int c = 0; c < d.nch; ++c) {
                    // the last chunk's phases beyond N2 are zeros in both operands: full 128-byte boxes throughout
                    const void* am = (const void*)&d.tmap;
                    const void* bm = (const void*)&d.bmap;
                    const int slab_hi = FWD ? (zi * 2) * d.nch + c : c;
                    const int slab_lo = FWD ? (zi * 2 + 1) * d.nch + c : d.nch + c;
                    for (int t1 = 0; t1 < pl.T1; ++t1) {
                        if (!((rm[t1] >> c) & 1)) continue;   // all taps of this window are zero
                        const int sa = na % kASlots;
                        const long long c0 = (d.exp & 4) ? clock64() : 0;
                        if (na >= kASlots) tc::mbar_wait(&bar_emptyA[sa], ((na / kASlots) - 1) & 1);
                        if (d.exp & 4) dbg_empty += clock64() - c0;
                        unsigned char* as = Abase + (size_t)sa * 2 * apart;
                        const int row = row0 + (pl.e1min + t1) * d.Wp;
                        if (rank == 0) tc::mbar_arrive_expect_tx(&bar_fullA[sa], 2 * 2 * (uint32_t)d.Arows * 128u);
                        if (hint) {
                            tc::tma_load_3d_pair_hint(as, am, 0, row, slab_hi, &bar_fullA[sa], pol);
                            tc::tma_load_3d_pair_hint(as + apart, am, 0, row, slab_lo, &bar_fullA[sa], pol);
                        } else {
                            tc::tma_load_3d_pair(as, am, 0, row, slab_hi, &bar_fullA[sa]);
                            tc::tma_load_3d_pair(as + apart, am, 0, row, slab_lo, &bar_fullA[sa]);
                        }
                        for (int t2 = 0; t2 < pl.T2; ++t2, ++nb) {
                            const int sb = nb % kBSlots;
                            const long long c1 = (d.exp & 4) ? clock64() : 0;
                            if (nb >= kBSlots) tc::mbar_wait(&bar_emptyB[sb], ((nb / kBSlots) - 1) & 1);
                            if (d.exp & 4) dbg_empty += clock64() - c1;
                            unsigned char* bs = Bbase + (size_t)sb * 2 * bhalf;
                            const int bslab = (int)(pl.coef_off + (long long)((t1 * pl.T2 + t2) * d.nch + c) * 2);
                            // B rows of this CTA: its half of the tile's MMA column range [n0, n0 + nn) (the
                            // drainers zero every accumulator they hand back, so every MMA accumulates)
                            int brow = (int)rank * Nh;
                            if (ranged) {
                                const int rg = d.trange[bslab >> 1];
                                if (rg == 0) {   // all-zero tile: the issuer skips its MMAs, so nothing to load
                                    if (rank == 0) tc::mbar_arrive(&bar_fullB[sb]);
                                    continue;
                                }
                                brow = (rg & 0xFFFF) + (int)rank * (rg >> 17);
                            }
                            if (rank == 0) tc::mbar_arrive_expect_tx(&bar_fullB[sb], 2 * 2 * (uint32_t)Nh * 128u);
                            if (hint) {
                                tc::tma_load_3d_pair_hint(bs, bm, 0, brow, bslab, &bar_fullB[sb], pol);
                                tc::tma_load_3d_pair_hint(bs + bhalf, bm, 0, brow, bslab + 1, &bar_fullB[sb], pol);
                            } else {
                                tc::tma_load_3d_pair(bs, bm, 0, brow, bslab, &bar_fullB[sb]);
                                tc::tma_load_3d_pair(bs + bhalf, bm, 0, brow, bslab + 1, &bar_fullB[sb]);
                            }
                        }
                        ++na;
                    }
                }
            }
            if (d.exp & 4) {
                long long* o = d.dbg + (size_t)blockIdx.x * 8;
                o[3] = dbg_empty;
                o[7] = clock64() - dbg_t0;
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            // ==================== MMA issuer (leader CTA, whole warp, one elected lane issues) ====================
            // The loop runs converged on warp-uniform values, descriptors are built once per stage (+2 per 32-byte
            // K-step), so each MMA costs a few uniform instructions: a single-thread issue loop cost ~75-95 cycles
            // per MMA (scripts/tc_rate_test.cu), above the ~100-cycle MMAs of narrowed column ranges.
            const uint32_t idesc = tc::idesc_f16(2 * kM, d.Ntile);
            const bool ranged = !(d.exp & 16);
            long long dbg_full = 0, dbg_tfree = 0, dbg_t0 = clock64();
            int na = 0, nb = 0, g = 0, gk = 0;   // A windows, B tiles, drain group, K-steps in the open group
            for (int i = ib; i < ie; ++i) {
                const int zi = d.items[i] / d.tiles;
                const TcPlane pl = d.planes[zi];
                const int* rm = d.rowmask + pl.mask_off;
                const int T1 = pl.T1, T2 = pl.T2;
                for (int c = 0; c < d.nch; ++c) {
                    const int ks = c == d.nch - 1 ? d.kst_last : kKS;
                    const uint32_t rb = 128u;   // row bytes
                    for (int t1 = 0; t1 < T1; ++t1) {
                        if (!((rm[t1] >> c) & 1)) continue;
                        const int sa = na % kASlots;
                        const bool last_win = c * T1 + t1 == pl.last_win;
                        {
                            const long long c0 = (d.exp & 4) ? clock64() : 0;
                            tc::mbar_wait(&bar_fullA[sa], (na / kASlots) & 1);
                            if (d.exp & 4) dbg_full += clock64() - c0;
                        }
                        const uint32_t a_hi0 = tc::smem_u32(Abase + (size_t)sa * 2 * apart), a_lo0 = a_hi0 + apart;
                        for (int t2 = 0; t2 < T2; ++t2, ++nb) {
                            const int sb = nb % kBSlots, j = g & 1;
                            const long long c0 = (d.exp & 4) ? clock64() : 0;
                            tc::mbar_wait(&bar_fullB[sb], (nb / kBSlots) & 1);
                            const long long c1 = (d.exp & 4) ? clock64() : 0;
                            if (gk == 0) tc::mbar_wait(&bar_tfree[j], (g >> 1) & 1);   // zeroed by the drainers
                            if (d.exp & 4) {
                                dbg_full += c1 - c0;
                                dbg_tfree += clock64() - c1;
                            }
                            tc::fence_after();
                            const uint32_t a_hi = a_hi0 + (uint32_t)t2 * rb, a_lo = a_lo0 + (uint32_t)t2 * rb;
                            const uint32_t b_hi = tc::smem_u32(Bbase + (size_t)sb * 2 * bhalf), b_lo = b_hi + bhalf;
                            // column range of the tile (the zero columns outside it would only add exact zeros, so
                            // the accumulated sums are bit-identical to full-width MMAs)
                            uint32_t n0 = 0, nn = (uint32_t)d.Ntile, idesc_s = idesc;
                            if (ranged) {
                                const int rg = d.trange[(pl.coef_off >> 1) + (t1 * T2 + t2) * d.nch + c];
                                n0 = (uint32_t)(rg & 0xFFFF);
                                nn = (uint32_t)(rg >> 16);
                                idesc_s = tc::idesc_f16(2 * kM, (int)nn);
                            }
                            const uint32_t acc = tmem + (uint32_t)(j * 256) + n0;
                            const uint64_t ah = tc::sdesc_swz(a_hi, rb), al = tc::sdesc_swz(a_lo, rb);
                            const uint64_t bh = tc::sdesc_swz(b_hi, rb), bl = tc::sdesc_swz(b_lo, rb);
                            if (nn > 0)
                                for (int k = 0; k < ks; ++k) {   // K-step k (16 fp16): start + 32 k bytes = field + 2 k
                                    const uint64_t dk = 2 * (uint64_t)k;
                                    tc::mma_f16_pair_elect(acc, ah + dk, bh + dk, idesc_s, 1u);
                                    tc::mma_f16_pair_elect(acc, ah + dk, bl + dk, idesc_s, 1u);
                                    tc::mma_f16_pair_elect(acc, al + dk, bh + dk, idesc_s, 1u);
                                }
                            gk += ks;
                            tc::mma_commit_pair_elect(&bar_emptyB[sb], 3);
                            if (t2 == T2 - 1) tc::mma_commit_pair_elect(&bar_emptyA[sa], 3);
                            // close the drain group at the item's last stage or before it could exceed chain_k
                            if ((last_win && t2 == T2 - 1) || gk + kKS > d.chain_k) {
                                tc::mma_commit_pair_elect(&bar_acc[j], 3);
                                ++g;
                                gk = 0;
                            }
                        }
                        ++na;
                    }
                }
            }
            if ((d.exp & 4) && lane == 0) {
                long long* o = d.dbg + (size_t)blockIdx.x * 8;
                o[0] = dbg_full;
                o[1] = dbg_tfree;
                o[2] = clock64() - dbg_t0;
                o[6] = nb;
            }
        }
    } else {
        // ============================ drainers: TMEM -> fp32 running sums, epilogue ============================
        const int q = warp & 3;                       // TMEM lane quarter this warp may access
        const int half = (warp - 2) >> 2;             // column half
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(half * Nh);
        const int r = 32 * q + lane;                  // tile row (pixel) of this thread
        const int aexp = tc::f16_scale_exp(__uint_as_float(*d.amax));   // the staged source's scale (tc_stage_kernel)
        float acc[kMaxNh];
#pragma unroll
        for (int i = 0; i < kMaxNh; ++i) acc[i] = 0.0f;
        // zero both accumulators of this warp's lanes / columns and hand them to the issuer (first tfree phase)
        auto zero_acc = [&](uint32_t base) {
#pragma unroll
            for (int c0 = 0; c0 < kMaxNh; c0 += 32) {
                if (c0 < Nh) {
                    if (c0 + 32 <= Nh) {
                        tc::tmem_zero32(base + (uint32_t)c0);
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (c0 + 8 * u < Nh) tc::tmem_zero8(base + (uint32_t)(c0 + 8 * u));
                    }
                }
            }
            tc::tmem_wait_st();
        };
        for (int j = 0; j < 2; ++j) {
            zero_acc(lane_base + (uint32_t)(j * 256));
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_cluster(&bar_tfree[j], 0);
        }
        int g = 0;
        long long dbg_acc = 0, dbg_epi = 0;
        for (int i = ib; i < ie; ++i) {
            const int item = d.items[i], zi = item / d.tiles, tile = item - zi * d.tiles;
            const TcPlane pl = d.planes[zi];
            for (int gi = 0; gi < pl.ngroups; ++gi) {   // the item's drain groups (counted at plan time)
                const int j = g & 1;
                {
                    const long long c0 = (d.exp & 4) ? clock64() : 0;
                    tc::mbar_wait(&bar_acc[j], (g >> 1) & 1);
                    if (d.exp & 4) dbg_acc += clock64() - c0;
                }
                ++g;
                tc::fence_after();
                const uint32_t base = lane_base + (uint32_t)(j * 256);
#pragma unroll
                for (int c0 = 0; c0 < kMaxNh; c0 += 32) {
                    if (c0 < Nh && !(d.exp & 1)) {
                        uint32_t v[32];
                        if (c0 + 32 <= Nh) {
                            tc::tmem_ld32_nowait(base + (uint32_t)c0, v);
                        } else {
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                if (c0 + 8 * u < Nh) tc::tmem_ld8_nowait(base + (uint32_t)(c0 + 8 * u), v + 8 * u);
                        }
                        tc::tmem_wait_ld();
#pragma unroll
                        for (int u = 0; u < 32; ++u)
                            if (c0 + u < Nh) acc[c0 + u] += __uint_as_float(v[u]);
                    }
                }
                zero_acc(base);   // every later MMA of this accumulator adds (column ranges need no full-width start)
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive_cluster(&bar_tfree[j], 0);
            }
            // ---- epilogue of the item ----
            const long long ce0 = (d.exp & 4) ? clock64() : 0;
            {   // undo the operands' power-of-two scales (exact)
                const float inv = ldexpf(1.0f, -(aexp + pl.bexp));
#pragma unroll
                for (int i = 0; i < kMaxNh; ++i) acc[i] *= inv;
            }
            const int L = tile * 2 * kM + (int)rank * kM + r;
            const int m1 = L / d.Wp, m2 = L - (L / d.Wp) * d.Wp;
            if (m1 < d.nh && m2 < d.nw) {
                const size_t npix = (size_t)d.nh * d.nw;
                const int z = d.zlist[zi];
                const int n0 = half * Nh;
                // polyphase destinations: column n is npix floats after column n-1 (coalesced across lanes)
                const bool fast = FWD || DST == DST_UPDATE || DST == DST_ISRA || DST == DST_POLY;
                const bool owned_all = z * d.N2 >= d.unit0 && (z + 1) * d.N2 <= d.unit0 + d.nu;
                if (fast && (FWD || DST != DST_POLY || owned_all)) {
                    float* p;
                    if constexpr (FWD || DST == DST_UPDATE || DST == DST_ISRA)   // per-plane partial / H^T r scratch
                        p = d.part + ((size_t)zi * d.N2 + n0) * npix + (size_t)m1 * d.nw + m2;
                    else
                        p = out + ((size_t)(z * d.N2 + n0 - d.unit0)) * npix + (size_t)m1 * d.nw + m2;
                    if (owned_all || FWD) {
#pragma unroll
                        for (int i = 0; i < kMaxNh; ++i)
                            if (i < Nh && n0 + i < d.N2) p[(size_t)i * npix] = acc[i];
                    } else {
#pragma unroll
                        for (int i = 0; i < kMaxNh; ++i) {
                            const int uu = z * d.N2 + n0 + i;
                            if (i < Nh && n0 + i < d.N2 && uu >= d.unit0 && uu < d.unit0 + d.nu) p[(size_t)i * npix] = acc[i];
                        }
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < kMaxNh; ++i) {
                        const int n = n0 + i;
                        const int uu = z * d.N2 + n;
                        if (i < Nh && n < d.N2 && uu >= d.unit0 && uu < d.unit0 + d.nu) {
                            const int n1 = n / d.N, n2 = n - (n / d.N) * d.N;
                            if constexpr (DST == DST_VOLIMAGE)
                                out[((size_t)z * d.H + n1 + d.N * m1) * d.W + n2 + d.N * m2] = acc[i];
                            else
                                out[((size_t)(uu - d.unit0) * d.nh + m1) * d.nw + m2] = acc[i];
                        }
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < kMaxNh; ++i) acc[i] = 0.0f;
            if (d.exp & 4) dbg_epi += clock64() - ce0;
        }
        if ((d.exp & 4) && warp == 2 && lane == 0) {
            long long* o = d.dbg + (size_t)blockIdx.x * 8;
            o[4] = dbg_acc;
            o[5] = dbg_epi;
        }
    }
    tc::fence_before();
    tc::cluster_sync();
    if (warp == 0) tc::tmem_dealloc_pair(tmem, kTmemCols);
}

// ------------------------------------------------------------------------------------------------
// Source maximum (|v|, float bits, atomicMax into d.amax, zeroed before): the staged operands are scaled by
// 2^f16_scale_exp(amax) so that the fp16 hi / lo split keeps 22 significant bits.
//   forward  SRC 0: the tensor-core planes' owned units of the polyphase volume; SRC 1: their planes of [nz][H][W]
//   backward SRC_RATIO: y / (max(yhat,0)+eps); SRC_IMAGE2D: the image; SRC_ONES: 1
template <bool FWD, int SRC>
__global__ void __launch_bounds__(256) tc_amax_kernel(const __grid_constant__ TcDirArgs d, const float* __restrict__ src,
                                                      const float* __restrict__ src2, float eps) {
    float m = 0.0f;
    size_t n;
    const float* p = src;
    if constexpr (FWD) {
        const int z = d.zlist[blockIdx.y];
        if constexpr (SRC == 0) {
            const int ub = max(z * d.N2, d.unit0), ue = min((z + 1) * d.N2, d.unit0 + d.nu);
            n = ue > ub ? (size_t)(ue - ub) * d.nh * d.nw : 0;
            p = src + (size_t)(max(ub - d.unit0, 0)) * d.nh * d.nw;
        } else {
            n = (size_t)d.H * d.W;
            p = src + (size_t)z * d.H * d.W;
        }
    } else {
        n = SRC == SRC_ONES ? 0 : (size_t)d.H * d.W;
        if (SRC == SRC_ONES) m = 1.0f;
    }
    // four independent loads in flight per thread (the loop is latency-bound otherwise)
    const size_t st = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    float m1 = 0.0f, m2 = 0.0f, m3 = 0.0f;
    for (; i + 3 * st < n; i += 4 * st) {
        float v0 = __ldg(p + i), v1 = __ldg(p + i + st), v2 = __ldg(p + i + 2 * st), v3 = __ldg(p + i + 3 * st);
        if constexpr (!FWD && SRC == SRC_RATIO) {
            v0 = v0 / (fmaxf(src2[i], 0.0f) + eps);
            v1 = v1 / (fmaxf(src2[i + st], 0.0f) + eps);
            v2 = v2 / (fmaxf(src2[i + 2 * st], 0.0f) + eps);
            v3 = v3 / (fmaxf(src2[i + 3 * st], 0.0f) + eps);
        }
        m = fmaxf(m, fabsf(v0));
        m1 = fmaxf(m1, fabsf(v1));
        m2 = fmaxf(m2, fabsf(v2));
        m3 = fmaxf(m3, fabsf(v3));
    }
    for (; i < n; i += st) {
        float v = __ldg(p + i);
        if constexpr (!FWD && SRC == SRC_RATIO) v = v / (fmaxf(src2[i], 0.0f) + eps);
        m = fmaxf(m, fabsf(v));
    }
    m = fmaxf(fmaxf(m, m1), fmaxf(m2, m3));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ float wm[8];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) m = fmaxf(m, wm[w]);
        if (m > 0.0f) atomicMax(d.amax, __float_as_uint(m));
    }
}

// ------------------------------------------------------------------------------------------------
// Source staging: slab rows L of the padded grid (m1 = L / Wp, m2 = L % Wp + e2lo), 64 phases per row,
// v = x 2^aexp, hi = fp16(v), lo = fp16(v - hi).  A 32-row x 64-phase tile per block, transposed through shared memory.
//   forward  (SRC 0 polyphase volume [nu][nh][nw], 1 image-layout volume [nz][H][W]): plane blockIdx.z
//   backward (SRC_RATIO y / (max(yhat,0)+eps), SRC_ONES, SRC_IMAGE2D): one image
template <bool FWD, int SRC>
__global__ void __launch_bounds__(256) tc_stage_kernel(const __grid_constant__ TcDirArgs d, const float* __restrict__ src,
                                                       const float* __restrict__ src2, float eps) {
    // kStagePB blocks of 32 padded pixels per CTA; every thread issues all its loads before the first use
    __shared__ float tile[kStagePB][kKC][33];
    const int L0 = blockIdx.x * 32 * kStagePB, c = blockIdx.y, zi = blockIdx.z;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const float ascale = tc::pow2f(tc::f16_scale_exp(__uint_as_float(*d.amax)));
    {
        float v[kStagePB][kKC / 8];
        float w[kStagePB][kKC / 8];   // yhat for SRC_RATIO
#pragma unroll
        for (int j = 0; j < kStagePB; ++j) {
            const int L = L0 + 32 * j + tx;
            const int m1 = L / d.Wp, m2 = L - (L / d.Wp) * d.Wp + d.e2lo;
            const bool pv = L < d.Lp && m1 < d.nh && m2 >= 0 && m2 < d.nw;
#pragma unroll
            for (int i = 0; i < kKC / 8; ++i) {
                const int ph = c * kKC + ty + 8 * i;
                v[j][i] = 0.0f;
                w[j][i] = 0.0f;
                if (pv && ph < d.N2) {
                    const int p1 = ph / d.N, p2 = ph - (ph / d.N) * d.N;
                    if constexpr (FWD) {
                        const int z = d.zlist[zi];
                        const int u = z * d.N2 + ph;
                        if (u >= d.unit0 && u < d.unit0 + d.nu) {
                            if constexpr (SRC == 0)
                                v[j][i] = src[((size_t)(u - d.unit0) * d.nh + m1) * d.nw + m2];
                            else
                                v[j][i] = src[((size_t)z * d.H + p1 + d.N * m1) * d.W + p2 + d.N * m2];
                        }
                    } else {
                        const size_t pix = (size_t)(p1 + d.N * m1) * d.W + p2 + d.N * m2;
                        if constexpr (SRC == SRC_ONES) {
                            v[j][i] = 1.0f;
                        } else if constexpr (SRC == SRC_RATIO) {
                            v[j][i] = src[pix];
                            w[j][i] = src2[pix];
                        } else {
                            v[j][i] = src[pix];
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kStagePB; ++j)
#pragma unroll
            for (int i = 0; i < kKC / 8; ++i) {
                float x = v[j][i];
                if constexpr (!FWD && SRC == SRC_RATIO) {
                    const int L = L0 + 32 * j + tx;
                    const int m1 = L / d.Wp, m2 = L - (L / d.Wp) * d.Wp + d.e2lo;
                    const bool pv = L < d.Lp && m1 < d.nh && m2 >= 0 && m2 < d.nw;
                    const int ph = c * kKC + ty + 8 * i;
                    x = (pv && ph < d.N2) ? x / (fmaxf(w[j][i], 0.0f) + eps) : 0.0f;
                }
                tile[j][ty + 8 * i][tx] = x;
            }
    }
    __syncthreads();
    const size_t slab_hi = FWD ? ((size_t)zi * 2) * d.nch + c : (size_t)c;
    const size_t slab_lo = FWD ? ((size_t)zi * 2 + 1) * d.nch + c : (size_t)d.nch + c;
    uint32_t* dst = reinterpret_cast<uint32_t*>(d.src);   // two fp16 phases (2 tx, 2 tx + 1) per 32-bit store
#pragma unroll
    for (int j = 0; j < kStagePB; ++j)
        for (int rr = ty; rr < 32; rr += 8) {
            const int L = L0 + 32 * j + rr;
            if (L >= d.Lp) break;
            uint16_t h0, l0, h1, l1;
            tc::split_f16(tile[j][2 * tx][rr], ascale, h0, l0);
            tc::split_f16(tile[j][2 * tx + 1][rr], ascale, h1, l1);
            dst[(slab_hi * d.Lp + L) * (kKC / 2) + tx] = (uint32_t)h0 | ((uint32_t)h1 << 16);
            dst[(slab_lo * d.Lp + L) * (kKC / 2) + tx] = (uint32_t)l0 | ((uint32_t)l1 << 16);
        }
}

// ------------------------------------------------------------------------------------------------
// forward reduction: y (+)= sum_zi part[zi][b'][m] (plane order fixed -> deterministic), interleaved into the image
// y[b1 + N m1][b2 + N m2].  One CTA per lenslet row m1: reads are contiguous along m2, the N image rows of the CTA
// are written from shared memory.
__global__ void __launch_bounds__(256) tc_fwd_reduce_kernel(const __grid_constant__ TcDirArgs d, float* __restrict__ y,
                                                            int accumulate) {
    extern __shared__ float accs[];   // [N][nw]: output phases (b1, 0..N-1) of lenslet row m1
    const int m1 = blockIdx.x, b1 = blockIdx.y;
    const size_t npix = (size_t)d.nh * d.nw;
    const int per = d.N * d.nw;
    for (int e = threadIdx.x; e < per; e += blockDim.x) {
        const int b2 = e / d.nw, m2 = e - (e / d.nw) * d.nw;
        const float* src = d.part + (size_t)(b1 * d.N + b2) * npix + (size_t)m1 * d.nw + m2;
        float v = 0.0f;
#pragma unroll 8
        for (int zi = 0; zi < d.nzd; ++zi) v += __ldcs(src + (size_t)zi * d.N2 * npix);   // plane order fixed
        accs[e] = v;
    }
    __syncthreads();
    float* o = y + (size_t)(b1 + d.N * m1) * d.W;
    for (int t = threadIdx.x; t < d.W; t += blockDim.x) {
        const float v = accs[(t % d.N) * d.nw + t / d.N];
        o[t] = accumulate ? o[t] + v : v;
    }
}

// ------------------------------------------------------------------------------------------------
// multiplicative update of the tensor-core planes' units from the H^T r scratch (coalesced, float4)
template <int DST>
__global__ void __launch_bounds__(256) tc_update_kernel(const __grid_constant__ TcDirArgs d, const float* __restrict__ xold,
                                                        const float* __restrict__ norm, float eps, float* __restrict__ out) {
    const size_t npix = (size_t)d.nh * d.nw;
    const int zi = blockIdx.y / d.N2, a = blockIdx.y - (blockIdx.y / d.N2) * d.N2;
    const int u = d.zlist[zi] * d.N2 + a;
    if (u < d.unit0 || u >= d.unit0 + d.nu) return;
    const float* bp = d.part + ((size_t)zi * d.N2 + a) * npix;
    const size_t base = (size_t)(u - d.unit0) * npix;
    for (size_t m = (size_t)blockIdx.x * blockDim.x + threadIdx.x; m < npix; m += (size_t)gridDim.x * blockDim.x)
        out[base + m] = update_value<DST>(xold[base + m], norm[base + m], bp[m], eps);
}

// ------------------------------------------------------------------------------------------------
// Coefficient tiles of one plane (plan time), built on the device from the owned PSF slice: tile (tap, chunk) =
// fp16 slabs [hi], [lo] of Ntile x 64 row-major (the TMA load swizzles them) of g * 2^bexp with element (n, k) =
//   forward : G_d[b' = n][a = chunk*64 + k],   d = -e        backward: G_d[b' = chunk*64 + k][a = n],   d = +e
__global__ void tcdir_coef_kernel(const __grid_constant__ TcDirArgs d, TcPlane pl, int z, const float* __restrict__ psf,
                                  int kh, int kw, int ch, int cw, int fwd, uint16_t* __restrict__ out,
                                  int* __restrict__ nzflag) {
    __shared__ int any, nmin, nmax;
    if (threadIdx.x == 0) {
        any = 0;
        nmin = 1 << 30;
        nmax = -1;
    }
    __syncthreads();
    const int tileid = blockIdx.x;   // tap * nch + chunk
    const int chunk = tileid % d.nch;
    const int tap = tileid / d.nch;
    const int N = d.N, N2 = d.N2;
    const int e1 = pl.e1min + tap / pl.T2, e2 = pl.e2min + tap % pl.T2;
    const int d1 = fwd ? -e1 : e1, d2 = fwd ? -e2 : e2;
    uint16_t* hi = out + ((size_t)pl.coef_off + (size_t)tileid * 2) * d.Ntile * kKC;
    uint16_t* lo = hi + (size_t)d.Ntile * kKC;
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
        uint16_t h, l;
        tc::split_f16(v, tc::pow2f(pl.bexp), h, l);
        hi[e] = h;
        lo[e] = l;
        if (v != 0.0f) {
            any = 1;
            atomicMin(&nmin, n);
            atomicMax(&nmax, n);
        }
    }
    __syncthreads();
    // nonzero flag of the tile = its nonzero B-row (N) range, packed nmin | (nmax + 1) << 16 (0: all zero)
    if (threadIdx.x == 0) nzflag[tileid] = any ? (nmin | ((nmax + 1) << 16)) : 0;
}

// per-plane max |psf| of the owned units (float bits, atomicMax) -> the coefficient tiles' fp16 scales
__global__ void tc_plane_amax_kernel(const float* __restrict__ psf, const int* __restrict__ zlist, int N2, int kk,
                                     int unit0, int nu, unsigned* __restrict__ pmax) {
    const int zi = blockIdx.y, z = zlist[zi];
    const int ub = max(z * N2, unit0), ue = min((z + 1) * N2, unit0 + nu);
    const size_t n = ue > ub ? (size_t)(ue - ub) * kk : 0;
    const float* p = psf + (size_t)max(ub - unit0, 0) * kk;
    float m = 0.0f;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        m = fmaxf(m, fabsf(p[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0f) atomicMax(pmax + zi, __float_as_uint(m));
}

cudaError_t launch_tc_plane_amax(const float* psf_dev, const int* zlist, int nzd, int N2, int kk, int unit0, int nu,
                                 unsigned* pmax, cudaStream_t s) {
    if (nzd <= 0) return cudaSuccess;
    tc_plane_amax_kernel<<<dim3(64, nzd), 256, 0, s>>>(psf_dev, zlist, N2, kk, unit0, nu, pmax);
    return cudaGetLastError();
}

// per-tile MMA column ranges (§5.3 column ranges): n0 | nn << 16, the nonzero B rows [nmin, nmax] widened to n0 a
// multiple of 8 and nn a multiple of 16 (the pair MMA's N), inside [0, Ntile); nn = 0 for an all-zero tile
void tcdir_ranges(const TcDirArgs& d, const std::vector<int>& nzflags, std::vector<int>* ranges) {
    ranges->resize(nzflags.size());
    for (size_t i = 0; i < nzflags.size(); ++i) {
        const int f = nzflags[i];
        if (!f) {
            (*ranges)[i] = 0;
            continue;
        }
        const int nmin = f & 0xFFFF, nend = f >> 16;
        int n0 = nmin / 8 * 8;
        int nn = (nend - n0 + 15) / 16 * 16;
        if (n0 + nn > d.Ntile) n0 = d.Ntile - nn;
        (*ranges)[i] = n0 | (nn << 16);
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
    d->kst_last = ((d->N2 - (d->nch - 1) * kKC) + 15) / 16;   // the last chunk's zero phases beyond are skipped
    planes->assign(d->nzd, TcPlane{});
    int e2lo = 1 << 30, e2hi = -(1 << 30);
    long long off = 0;
    for (int zi = 0; zi < d->nzd; ++zi) {
        TcPlane& pl = (*planes)[zi];
        pl.T1 = d1max[zi] - d1min[zi] + 1;
        pl.T2 = d2max[zi] - d2min[zi] + 1;
        pl.e1min = fwd ? -d1max[zi] : d1min[zi];
        pl.e2min = fwd ? -d2max[zi] : d2min[zi];
        pl.coef_off = off;   // in slabs of Ntile x 64 fp16
        pl.bexp = 0;         // set from the plane's max tap before the coefficient tiles are built
        off += (long long)pl.T1 * pl.T2 * d->nch * 2;
        e2lo = std::min(e2lo, pl.e2min);
        e2hi = std::max(e2hi, pl.e2min + pl.T2 - 1);
    }
    d->nslabs = off;
    {
        const char* ev = getenv("LFM_TC_EXP");
        d->exp = ev ? atoi(ev) : 0;
        const char* ck = getenv("LFM_TC_CHAIN");   // dev: drain-group length override
        d->chain_k = ck ? std::max(1, atoi(ck)) : kChainK;
        d->dbg = nullptr;
        if (d->exp & 4) cudaMalloc(&d->dbg, (size_t)2 * num_sms * 8 * sizeof(long long));   // leaked: dev only
    }
    d->e2lo = d->nzd > 0 ? e2lo : 0;
    int t2max = 1;
    for (const TcPlane& pl : *planes) t2max = std::max(t2max, pl.T2);
    if (t2max > 65) return false;   // A window box rows <= 192 (TMA box <= 256, smem budget)
    d->Arows = kM + t2max - 1;
    if (tcdir_smem_bytes(d->Ntile, d->Arows) > 227 * 1024) return false;
    d->Wp = d->nw + (d->nzd > 0 ? e2hi - e2lo : 0);
    d->Lp = d->nh * d->Wp;
    d->tiles = (d->Lp + 2 * kM - 1) / (2 * kM);   // pair tiles
    d->grid = std::max(1, std::min(d->tiles * d->nzd, num_sms / 2));   // CTA pairs
    return true;
}

void tcdir_schedule(const TcDirArgs& d, const std::vector<TcPlane>& planes, std::vector<int>* item_off,
                    std::vector<int>* items) {
    // longest-processing-time-first: items sorted by cost (taps), each to the least-loaded CTA
    std::vector<std::pair<long long, int>> it;
    for (int zi = 0; zi < d.nzd; ++zi)
        for (int t = 0; t < d.tiles; ++t)
            it.push_back({(long long)std::max(1, planes[zi].active_windows) * planes[zi].T2, zi * d.tiles + t});
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
    // Each CTA pair runs its items in the order LPT assigned them, i.e. the global (cost, plane, tile) order: at any
    // moment all pairs work on neighbouring items of that order -- a few planes -- so a plane's coefficient tiles are
    // fetched from HBM once and served from L2 to all its pixel tiles (sorting each pair's items by plane instead
    // spread the pairs over many planes at once: a coefficient working set far beyond L2, re-read from HBM and
    // competing with the concurrent MAC for bandwidth).  LFM_TC_SCHED=1 (dev): the old per-pair plane sort.
    static const bool plane_sort = getenv("LFM_TC_SCHED") && atoi(getenv("LFM_TC_SCHED")) == 1;
    item_off->assign(1, 0);
    items->clear();
    for (int b = 0; b < d.grid; ++b) {
        if (plane_sort) std::sort(per[b].begin(), per[b].end());
        items->insert(items->end(), per[b].begin(), per[b].end());
        item_off->push_back((int)items->size());
    }
}

size_t tcdir_coef_elems(const TcDirArgs& d, const std::vector<TcPlane>& planes) {
    size_t n = 0;
    for (const TcPlane& pl : planes) n += (size_t)pl.T1 * pl.T2 * d.nch * 2;
    return n * d.Ntile * kKC;
}
size_t tcdir_src_elems(const TcDirArgs& d, int fwd) { return (size_t)(fwd ? 2 * d.nzd : 2) * d.nch * d.Lp * kKC; }
size_t tcdir_part_floats(const TcDirArgs& d, int fwd) {
    (void)fwd;   // forward: per-plane partials; backward: H^T r scratch -- both polyphase [nzd][N2][nh][nw]
    return (size_t)d.nzd * d.N2 * d.nh * d.nw;
}

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
    cuuint64_t strides[2] = {(cuuint64_t)kKC * 2, (cuuint64_t)d->Lp * kKC * 2};
    cuuint32_t box[3] = {(cuuint32_t)kKC, (cuuint32_t)d->Arows, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&d->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, d->src, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    // coefficient slabs [nslabs][Ntile][64] fp16, each CTA of a pair loads Ntile/2 rows
    cuuint64_t bdims[3] = {(cuuint64_t)kKC, (cuuint64_t)d->Ntile, (cuuint64_t)d->nslabs};
    cuuint64_t bstrides[2] = {(cuuint64_t)kKC * 2, (cuuint64_t)d->Ntile * kKC * 2};
    cuuint32_t bbox[3] = {(cuuint32_t)kKC, (cuuint32_t)(d->Ntile / 2), 1};
    r = enc(&d->bmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<uint16_t*>(d->coef), bdims, bstrides, bbox, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_tcdir_coef(const TcDirArgs& d, const TcPlane& pl, int zi, int z, const float* psf_dev, int kh,
                              int kw, int ch, int cw, int fwd, uint16_t* coef, int* nzflags, cudaStream_t s) {
    (void)zi;
    const int tiles = pl.T1 * pl.T2 * d.nch;
    if (tiles <= 0) return cudaSuccess;
    tcdir_coef_kernel<<<tiles, 256, 0, s>>>(d, pl, z, psf_dev, kh, kw, ch, cw, fwd, coef, nzflags);
    return cudaGetLastError();
}

void tcdir_window_masks(const TcDirArgs& d, std::vector<TcPlane>* planes, const std::vector<int>& nzflags,
                        std::vector<int>* rowmask) {
    rowmask->clear();
    long long tile0 = 0;   // first (tap, chunk) flag of the plane
    for (TcPlane& pl : *planes) {
        pl.mask_off = (int)rowmask->size();
        pl.last_win = -1;
        pl.active_windows = 0;
        for (int t1 = 0; t1 < pl.T1; ++t1) {
            int m = 0;
            for (int c = 0; c < d.nch; ++c)
                for (int t2 = 0; t2 < pl.T2; ++t2)
                    if (nzflags[(size_t)(tile0 + (long long)(t1 * pl.T2 + t2) * d.nch + c)]) m |= 1 << c;
            rowmask->push_back(m);
        }
        for (int c = 0; c < d.nch; ++c)
            for (int t1 = 0; t1 < pl.T1; ++t1)
                if (((*rowmask)[pl.mask_off + t1] >> c) & 1) {
                    pl.last_win = c * pl.T1 + t1;
                    ++pl.active_windows;
                }
        if (pl.last_win < 0) {   // an all-zero plane still runs one (zero) window so that its outputs are written
            (*rowmask)[pl.mask_off] |= 1;
            pl.last_win = 0;
            pl.active_windows = 1;
        }
        // drain groups of one item: the issuer's stage walk (c, t1 of nonzero windows, t2), closing a group at the
        // last window's last tap or before it would exceed chain_k K-steps -- the drainers only need the count
        pl.ngroups = 0;
        for (int c = 0, gk = 0; c < d.nch; ++c)
            for (int t1 = 0; t1 < pl.T1; ++t1) {
                if (!(((*rowmask)[pl.mask_off + t1] >> c) & 1)) continue;
                for (int t2 = 0; t2 < pl.T2; ++t2) {
                    gk += c == d.nch - 1 ? d.kst_last : kKS;
                    if ((c * pl.T1 + t1 == pl.last_win && t2 == pl.T2 - 1) || gk + kKS > d.chain_k) {
                        ++pl.ngroups;
                        gk = 0;
                    }
                }
            }
        tile0 += (long long)pl.T1 * pl.T2 * d.nch;
    }
}

template <bool FWD, int DST>
static cudaError_t tcdir_main(const TcDirArgs& d, const float* xold, const float* norm, float eps, float* out,
                              cudaStream_t s) {
    const size_t smem = tcdir_smem_bytes(d.Ntile, d.Arows);
    cudaError_t e = cudaFuncSetAttribute(tcdir_kernel<FWD, DST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // SMs configured for the largest shared-memory carveout, so that a co-resident MAC CTA fits beside it (§5.5)
    e = cudaFuncSetAttribute(tcdir_kernel<FWD, DST>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    tcdir_kernel<FWD, DST><<<2 * d.grid, kThreads, smem, s>>>(d, xold, norm, eps, out);
    if (d.exp & 4) {   // dev only: print the averaged wait counters of the leader CTAs
        cudaStreamSynchronize(s);
        std::vector<long long> h((size_t)2 * d.grid * 8);
        cudaMemcpy(h.data(), d.dbg, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
        double a[8] = {0};
        for (int b = 0; b < 2 * d.grid; b += 2)
            for (int k = 0; k < 8; ++k) a[k] += (double)h[(size_t)b * 8 + k] / d.grid;
        double p[8] = {0};
        for (int b = 1; b < 2 * d.grid; b += 2)
            for (int k = 0; k < 8; ++k) p[k] += (double)h[(size_t)b * 8 + k] / d.grid;
        fprintf(stderr,
                "[tc %s] leader: mma_total %.0f wait_full %.0f wait_tfree %.0f stages %.0f | prod_total %.0f "
                "wait_empty %.0f | drain wait_acc %.0f epi %.0f || peer: prod wait_empty %.0f drain wait_acc %.0f epi %.0f\n",
                FWD ? "fwd" : "bwd", a[2], a[0], a[1], a[6], a[7], a[3], a[4], a[5], p[3], p[4], p[5]);
    }
    return cudaGetLastError();
}

template <bool FWD, int SRC>
static cudaError_t tc_stage(const TcDirArgs& d, const float* src, const float* src2, float eps, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(d.amax, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    tc_amax_kernel<FWD, SRC><<<dim3(FWD ? 64 : 296, FWD ? d.nzd : 1), 256, 0, s>>>(d, src, src2, eps);
    dim3 grid((d.Lp + 32 * kStagePB - 1) / (32 * kStagePB), d.nch, FWD ? d.nzd : 1);
    tc_stage_kernel<FWD, SRC><<<grid, 256, 0, s>>>(d, src, src2, eps);
    return cudaGetLastError();
}

cudaError_t launch_tcdir_fwd(const TcDirArgs& d, const float* x, int src_image, float* y, int accumulate,
                             cudaStream_t s, int parts) {
    if (d.nzd <= 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    if (parts & TC_PART_STAGE) {
        e = src_image ? tc_stage<true, 1>(d, x, nullptr, 0.f, s) : tc_stage<true, 0>(d, x, nullptr, 0.f, s);
        if (e != cudaSuccess) return e;
    }
    if (parts & TC_PART_MAIN) {
        e = tcdir_main<true, 0>(d, nullptr, nullptr, 0.f, nullptr, s);
        if (e != cudaSuccess) return e;
    }
    if (!(parts & TC_PART_FINISH)) return cudaSuccess;
    const size_t rsm = (size_t)d.N * d.nw * sizeof(float);
    tc_fwd_reduce_kernel<<<dim3(d.nh, d.N), 256, rsm, s>>>(d, y, accumulate);
    return cudaGetLastError();
}

static cudaError_t tc_stage_bwd(const TcDirArgs& d, int src, const float* img, const float* img2, float eps,
                                cudaStream_t s) {
    switch (src) {
        case SRC_RATIO: return tc_stage<false, SRC_RATIO>(d, img, img2, eps, s);
        case SRC_ONES: return tc_stage<false, SRC_ONES>(d, nullptr, nullptr, eps, s);
        case SRC_IMAGE2D: return tc_stage<false, SRC_IMAGE2D>(d, img, nullptr, eps, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_tcdir_bwd(const TcDirArgs& d, int src, const float* img, const float* img2, float eps, int dst,
                             float* out, const float* xold, const float* norm, cudaStream_t s, int parts) {
    if (d.nzd <= 0) return cudaSuccess;
    cudaError_t e;
    if (parts & TC_PART_STAGE) {
        e = tc_stage_bwd(d, src, img, img2, eps, s);
        if (e != cudaSuccess) return e;
    }
    if (!(parts & TC_PART_MAIN)) return cudaSuccess;
    const dim3 ug((unsigned)std::min<size_t>(((size_t)d.nh * d.nw + 255) / 256, 8), (unsigned)(d.nzd * d.N2));
    switch (dst) {
        case DST_UPDATE:
            e = tcdir_main<false, DST_UPDATE>(d, xold, norm, eps, out, s);
            if (e != cudaSuccess) return e;
            tc_update_kernel<DST_UPDATE><<<ug, 256, 0, s>>>(d, xold, norm, eps, out);
            return cudaGetLastError();
        case DST_ISRA:
            e = tcdir_main<false, DST_ISRA>(d, xold, norm, eps, out, s);
            if (e != cudaSuccess) return e;
            tc_update_kernel<DST_ISRA><<<ug, 256, 0, s>>>(d, xold, norm, eps, out);
            return cudaGetLastError();
        case DST_POLY: return tcdir_main<false, DST_POLY>(d, xold, norm, eps, out, s);
        case DST_VOLIMAGE: return tcdir_main<false, DST_VOLIMAGE>(d, xold, norm, eps, out, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lfm
