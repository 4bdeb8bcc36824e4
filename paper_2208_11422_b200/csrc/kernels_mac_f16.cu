// kernels_mac_f16.cu -- frame-batched MACs for plans built for time-lapse batches (LFM_PLAN_FRAMES; SURVEY f1,
// DESIGN.md §5.2).  The transfer matrices are stored pre-split into power-of-two-scaled fp16 hi / lo parts (the same
// bytes as fp32), so the batched passes are a plain TMA -> tcgen05 kind::f16 pipeline: no SIMT warps touch the
// streamed operand (the 3xTF32 kernels of kernels_mac_tc.cu compute A_lo from every streamed tile), and kind::f16 runs
// at twice the tf32 rate.  Three products per K-step as in the direct path (reading C26): ah*bh + ah*bl + al*bh.
//
//   forward   per kappa  Y_f[b'] = sum_u M[b'][u] G_f[u]            A = M rows b' (K = (u, re/im) interleaved)
//   backward  per kappa  Xh_f[u] = sum_b' conj(M[b'][u]) R_f[b']    A = M^T rows u (K = (b', re/im) interleaved),
//             a transposed copy built at plan time, so both passes read K-major tiles.
// B (the frames' spectra, per chunk) is built by SIMT prep warps from a TMA-staged fp32 tile, scaled per frame by
// 2^eB[f] from the DC bound: for the non-negative sources of the RL iteration (x, y / yhat) |G_f[kappa][u]| <=
// G_f[0][u] = sum_m x (mf_frame_scale_kernel).  The epilogue multiplies by 2^-(eA + eB[f]) (exact).
//
// Split row format (in place of a complex64 row of n entries): [hi: 2n fp16][lo: 2n fp16], v = x 2^eA,
// hi = fp16(v), lo = fp16(v - hi), re / im interleaved -- 8n bytes, as before.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "lfm_internal.cuh"
#include "tc_sm100.cuh"

namespace lfm {

namespace {
constexpr int kFM = 128;                       // rows per CTA tile (TMEM lanes)
constexpr int kFK = 64;                        // K elements (fp16) per chunk = one 128-byte swizzle row
constexpr int kFKS = kFK / 16;                 // K-steps per chunk
constexpr uint32_t kFATile = kFM * 128;        // 16 KB per part
constexpr int kFPrep = 8;                      // prep warps
constexpr int kFThreads = 32 * (kFPrep + 6);   // producer + prep + MMA + 4 drainers
constexpr uint32_t kFSmemMax = 232448;

__host__ __device__ constexpr uint32_t f_round1k(uint32_t v) { return (v + 1023u) & ~1023u; }
__host__ __device__ constexpr uint32_t f_btile(int F) { return f_round1k((uint32_t)(4 * F) * 128u); }   // 4F fp16 rows
constexpr uint32_t kFAStage = 2 * kFATile;     // A hi + lo per chunk
// the two-ring kernel (F = 32): four prep groups of two warps, four B slots (>= the groups, see its prep warps)
__host__ __device__ constexpr int f_pg(int F) { return F >= 32 ? 4 : 8; }
__host__ __device__ constexpr int f_bslots(int F) { return f_pg(F); }
// the one-ring kernel (F <= 16): A hi + lo, B tile and fp32 source tile per stage
__host__ __device__ constexpr uint32_t f_stile(int F) { return f_round1k((uint32_t)F * kFK * 4u); }     // F fp32 rows
__host__ __device__ constexpr uint32_t f_stage(int F) { return 2 * kFATile + f_btile(F) + f_stile(F); }
__host__ __device__ constexpr int f_depth(int F) {
    return (int)((kFSmemMax - 1024) / f_stage(F)) < 8 ? (int)((kFSmemMax - 1024) / f_stage(F)) : 8;
}
__host__ __device__ constexpr int f_gcd(int a, int b) { return b == 0 ? a : f_gcd(b, a % b); }
// A ring depth: what shared memory holds beside the B ring (F = 32: 5 x 32 KB; the A bytes in flight per SM bound
// the MAC's streaming rate)
__host__ __device__ constexpr int f_adepth(int F) {
    return (int)((kFSmemMax - 1024 - f_bslots(F) * f_btile(F)) / kFAStage) < 8
               ? (int)((kFSmemMax - 1024 - f_bslots(F) * f_btile(F)) / kFAStage)
               : 8;
}
}  // namespace

size_t mac_f16_smem_bytes(int F) {
    return F >= 32 ? (size_t)f_adepth(F) * kFAStage + (size_t)f_bslots(F) * f_btile(F) + 1024
                   : (size_t)f_depth(F) * f_stage(F) + 1024;
}

// ---------------------------------------------------------------------------------------------------------------
// F <= 16 variant: one ring whose stages hold A hi + lo, the B tile and the frames' fp32 source tile (TMA, loaded with
// A).  Items as in mac_f16_kernel below.  Warps: 0 TMA producer, 1..8 prep (PG groups, alternate chunks; one fill
// barrier per (group, stage), see kernels_mac_tc.cu), 9 MMA issuer, 10..13 drainers (lane quarters 2, 3, 0, 1).
// At F <= 16 the stages are small enough to run five or six deep, and the TMA-staged source measured faster than the
// prep warps' L2 reads of the two-ring kernel (c2, F = 8: forward MAC 0.143 vs 0.160 ms).
template <int F, int PG, bool FWD>
__global__ void __launch_bounds__(kFThreads, 1) mac_f16_tma_kernel(const __grid_constant__ MacF16Args d) {
    constexpr int S = f_depth(F);
    constexpr int LG = PG * S / f_gcd(PG, S);
    constexpr int NB = 4 * F;      // stacked B rows: hi 0..2F-1, lo 2F..4F-1
    constexpr int NSET = 6 * F;    // accumulator columns: hi*hi | hi*lo | lo*hi
    static_assert(S >= PG, "every prep group needs a stage");
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t bar_full[PG][S], bar_ready[S], bar_empty[S], bar_acc[2], bar_tfree[2];
    __shared__ uint32_t tmem_base;
    __shared__ float s_scale[F], s_inv[F];   // per frame: 2^eB (prep) and 2^-(eA + eB) (epilogue)
    const uint32_t raw = tc::smem_u32(smem_raw);
    unsigned char* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sbytes = f_stage(F);
    const int ntile = FWD ? 2 : (d.nu_pad + kFM - 1) / kFM;
    const int ksp = d.ksplit > 1 ? d.ksplit : 1;   // K splits per (kappa, tile): partial outputs ksp apart
    const int nitems = d.nkappa * ntile * ksp;
    const int nchunks = FWD ? (2 * d.nu_pad + kFK - 1) / kFK : (2 * d.bpitch + kFK - 1) / kFK;
    // item -> kappa, row tile, K split and its chunk range [c_lo, c_hi)
    auto decode = [&](int item, int& kap, int& t, int& sp, int& c_lo, int& c_hi) {
        kap = item / (ntile * ksp);
        const int rem = item - kap * ntile * ksp;
        t = rem / ksp;
        sp = rem - t * ksp;
        c_lo = (int)((long long)sp * nchunks / ksp);
        c_hi = (int)((long long)(sp + 1) * nchunks / ksp);
    };
    const int kvalid_last = (FWD ? 2 * d.nu_pad : 2 * d.N2) - (nchunks - 1) * kFK;   // real K elements, last chunk
    const int ks_last = (kvalid_last + 15) / 16;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            for (int g = 0; g < PG; ++g) tc::mbar_init(&bar_full[g][i], 1);
            tc::mbar_init(&bar_ready[i], kFPrep / PG);
            tc::mbar_init(&bar_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&bar_acc[i], 1);
            tc::mbar_init(&bar_tfree[i], 4);
        }
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&d.tmapAh);
        tc::tma_prefetch_desc(&d.tmapAl);
        tc::tma_prefetch_desc(&d.tmapS);
    }
    if (warp == 0) tc::tmem_alloc(&tmem_base, 2 * NSET <= 256 ? 256 : 512);
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
        const int eb = d.bmax ? (f < d.nframes ? tc::f16_scale_exp(__uint_as_float(d.bmax[f])) : 0) : d.bexp[f];
        s_scale[f] = tc::pow2f(eb);
        s_inv[f] = ldexpf(1.0f, -(d.aexp + eb));
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;

    if (warp == 0) {
        if (lane == 0) {   // ---- producer: A hi / lo tiles and the frames' fp32 source tile per chunk ----
            int it = 0;
            for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
                int kap, t, sp, c_lo, c_hi;
                decode(item, kap, t, sp, c_lo, c_hi);
                for (int c = c_lo; c < c_hi; ++c, ++it) {
                    const int s = it % S;
                    if (it >= S) tc::mbar_wait(&bar_empty[s], ((it / S) - 1) & 1);
                    unsigned char* st = smem + (size_t)s * sbytes;
                    uint64_t* fb = &bar_full[it % PG][s];
                    tc::mbar_arrive_expect_tx(fb, 2 * kFATile + (uint32_t)F * kFK * 4u);
                    tc::tma_load_3d(st, &d.tmapAh, c * kFK, t * kFM, kap, fb);
                    tc::tma_load_3d(st + kFATile, &d.tmapAl, c * kFK, t * kFM, kap, fb);
                    tc::tma_load_3d(st + 2 * kFATile + f_btile(F), &d.tmapS, c * kFK, kap, 0, fb);
                }
            }
        }
    } else if (warp <= kFPrep) {
        // ---- prep: stacked B rows from the fp32 tile [F][32 complex], scaled by 2^eB[f], split hi | lo ----
        //   FWD  row 2f: (Gr, -Gi), row 2f+1: (Gi, Gr)   -> D[b'][2f] = Re Y_f, D[b'][2f+1] = Im Y_f
        //   BWD  row 2f: (Rr,  Ri), row 2f+1: (Ri, -Rr)  -> D[u][2f]  = Re Xh_f, D[u][2f+1] = Im Xh_f (conj(M) R)
        constexpr int NP = 32 * kFPrep / PG;
        constexpr int NE = (F * (kFK / 2) + NP - 1) / NP;   // complex source values per thread
        const int pt = (threadIdx.x - 32) % NP, grp = (threadIdx.x - 32) / NP;
        int it = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            int kap, t, sp, c_lo, c_hi;
            decode(item, kap, t, sp, c_lo, c_hi);
            for (int c = c_lo; c < c_hi; ++c, ++it) {
                if (it % PG != grp) continue;
                const int s = it % S;
                tc::mbar_wait(&bar_full[grp][s], (it / LG) & 1);
                unsigned char* st = smem + (size_t)s * sbytes;
                unsigned char* bt = st + 2 * kFATile;
                const float2* src = reinterpret_cast<const float2*>(bt + f_btile(F));   // [F][32]
#pragma unroll
                for (int i = 0; i < NE; ++i) {
                    const int e = pt + NP * i;
                    if (e < F * (kFK / 2)) {
                        const int f = e / (kFK / 2), j = e - f * (kFK / 2);
                        const float2 g = src[f * (kFK / 2) + j];
                        // two splits per complex value; the B entries are +-re / +-im, and -(h + l) = (-h) + (-l)
                        // is a sign flip of both fp16 halves
                        uint16_t rh, rl, ih, il;
                        tc::split_f16(g.x, s_scale[f], rh, rl);
                        tc::split_f16(g.y, s_scale[f], ih, il);
                        uint32_t h0, l0, h1, l1;   // rows 2f, 2f+1: (element 2j) | (element 2j+1) << 16
                        if constexpr (FWD) {       // (re, -im), (im, re)
                            h0 = (uint32_t)rh | ((uint32_t)(ih ^ 0x8000u) << 16);
                            l0 = (uint32_t)rl | ((uint32_t)(il ^ 0x8000u) << 16);
                            h1 = (uint32_t)ih | ((uint32_t)rh << 16);
                            l1 = (uint32_t)il | ((uint32_t)rl << 16);
                        } else {                   // (re, im), (im, -re)
                            h0 = (uint32_t)rh | ((uint32_t)ih << 16);
                            l0 = (uint32_t)rl | ((uint32_t)il << 16);
                            h1 = (uint32_t)ih | ((uint32_t)(rh ^ 0x8000u) << 16);
                            l1 = (uint32_t)il | ((uint32_t)(rl ^ 0x8000u) << 16);
                        }
#pragma unroll
                        for (int r = 0; r < 2; ++r) {
                            const int row = 2 * f + r, rowl = 2 * F + row;
                            // byte offset of elements (row, 2j .. 2j+1) in a K-major SWIZZLE_128B fp16 tile
                            const uint32_t off = (uint32_t)row * 128u + ((((uint32_t)(j >> 2)) ^ (row & 7)) & 7) * 16u + (j & 3) * 4u;
                            const uint32_t offl = (uint32_t)rowl * 128u + ((((uint32_t)(j >> 2)) ^ (rowl & 7)) & 7) * 16u + (j & 3) * 4u;
                            *reinterpret_cast<uint32_t*>(bt + off) = r ? h1 : h0;
                            *reinterpret_cast<uint32_t*>(bt + offl) = r ? l1 : l0;
                        }
                    }
                }
                tc::fence_proxy_async();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar_ready[s]);
            }
        }
    } else if (warp == kFPrep + 1) {
        // ---- MMA issuer (whole warp, uniform values, one elected lane issues) ----
        const uint32_t id1 = tc::idesc_f16(kFM, NB), id2 = tc::idesc_f16(kFM, 2 * F);
        int it = 0, g = 0, gk = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            int kap, t, sp, c_lo, c_hi;
            decode(item, kap, t, sp, c_lo, c_hi);
            for (int c = c_lo; c < c_hi; ++c, ++it) {
                const int s = it % S, j = g & 1;
                tc::mbar_wait(&bar_ready[s], (it / S) & 1);
                if (gk == 0 && g >= 2) tc::mbar_wait(&bar_tfree[j], ((g >> 1) - 1) & 1);
                tc::fence_after();
                const uint32_t a_hi = tc::smem_u32(smem + (size_t)s * sbytes), a_lo = a_hi + kFATile;
                const uint32_t b = a_hi + 2 * kFATile;
                const uint32_t acc = tmem + (uint32_t)(j * NSET);
                const uint64_t ah0 = tc::sdesc_sw128(a_hi), al0 = tc::sdesc_sw128(a_lo), bd0 = tc::sdesc_sw128(b);
                const int ks = c == nchunks - 1 ? ks_last : kFKS;
                for (int k = 0; k < ks; ++k) {   // K-step k (16 fp16 = 32 bytes): descriptor address + 2 k
                    const uint64_t dk = 2 * (uint64_t)k;
                    tc::mma_f16_elect(acc, ah0 + dk, bd0 + dk, id1, (gk == 0 && k == 0) ? 0u : 1u);           // hi*hi | hi*lo
                    tc::mma_f16_elect(acc + 4 * F, al0 + dk, bd0 + dk, id2, (gk == 0 && k == 0) ? 0u : 1u);   // lo*hi
                }
                tc::mma_commit_elect(&bar_empty[s]);
                gk += ks;
                if (gk + kFKS > d.chain_k || c == c_hi - 1) {
                    tc::mma_commit_elect(&bar_acc[j]);
                    ++g;
                    gk = 0;
                }
            }
        }
    } else {
        // ---- drainers: TMEM -> fp32 running sums (2F per thread), unscale per frame, store ----
        const int q = warp & 3;
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
        float acc[2 * F];
#pragma unroll
        for (int i = 0; i < 2 * F; ++i) acc[i] = 0.0f;
        int g = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            int kap, t, sp, c_lo, c_hi;
            decode(item, kap, t, sp, c_lo, c_hi);
            for (int c = c_lo, gk = 0; c < c_hi; ++c) {   // the issuer's drain groups
                gk += c == nchunks - 1 ? ks_last : kFKS;
                if (!(gk + kFKS > d.chain_k || c == c_hi - 1)) continue;
                gk = 0;
                const int j = g & 1;
                tc::mbar_wait(&bar_acc[j], (g >> 1) & 1);
                ++g;
                tc::fence_after();
                const uint32_t base = lane_base + (uint32_t)(j * NSET);
#pragma unroll
                for (int b0 = 0; b0 < 3; ++b0) {   // up to 32 columns in flight per wait (not one wait per 8)
#pragma unroll
                    for (int c8 = 0; c8 < 2 * F; c8 += 32) {
                        constexpr int W = 2 * F < 32 ? 2 * F : 32;
                        uint32_t v[W];
                        if constexpr (W == 32) {
                            tc::tmem_ld32_nowait(base + (uint32_t)(b0 * 2 * F + c8), v);
                        } else {
#pragma unroll
                            for (int c = 0; c < W; c += 8) tc::tmem_ld8_nowait(base + (uint32_t)(b0 * 2 * F + c8 + c), v + c);
                        }
                        tc::tmem_wait_ld();
#pragma unroll
                        for (int u = 0; u < W; ++u) acc[c8 + u] += __uint_as_float(v[u]);
                    }
                }
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar_tfree[j]);
            }
            const int row = t * kFM + 32 * q + lane;
            if (row < (FWD ? d.N2 : d.nu_pad)) {
#pragma unroll
                for (int f = 0; f < F; ++f) {
                    if (f >= d.nframes) break;
                    const float inv = s_inv[f];
                    const float2 v = make_float2(acc[2 * f] * inv, acc[2 * f + 1] * inv);
                    d.out[(long long)sp * d.out_sstride + (long long)f * d.out_fstride + (long long)kap * d.out_ld + row] = v;
                }
            }
#pragma unroll
            for (int i = 0; i < 2 * F; ++i) acc[i] = 0.0f;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 2 * NSET <= 256 ? 256 : 512);
}

// FWD: item = (kappa, half h of the output phases): D[b'][n] over all K chunks of the kappa row.
// BWD: item = (kappa, tile t of 128 units):        D[u][n] over the 8 K chunks of (b', re/im).
// Warps: 0 TMA producer (A only), 1..8 prep (PG groups, alternate chunks), 9 MMA issuer, 10..13 drainers (lane
// quarters 2, 3, 0, 1).  Two rings: A (hi + lo tiles, SA deep, TMA) and the stacked B tiles (f_bslots(F), written by the
// prep warps from the fp32 source read through L2).  Keeping the B tiles and the source out of the A stages lets the
// A ring run five deep at F = 32 instead of four (the F = 32 MAC streamed 5.5-5.8 TB/s with four, the F = 16 one 6.4
// with five, r02 ncu).  Used at F = 32; F <= 16 runs mac_f16_tma_kernel above.
template <int F, int PG, bool FWD>
__global__ void __launch_bounds__(kFThreads, 1) mac_f16_kernel(const __grid_constant__ MacF16Args d) {
    constexpr int SA = f_adepth(F);
    constexpr int SB = f_bslots(F);
    constexpr int NB = 4 * F;      // stacked B rows: hi 0..2F-1, lo 2F..4F-1
    constexpr int NSET = 6 * F;    // accumulator columns: hi*hi | hi*lo | lo*hi
    // a prep group waits for the MMA to release B slot (it % SB) from chunk it - SB; its own previous chunk (it - PG)
    // already waited for chunk it - PG - SB, so with PG <= SB the slot's earlier use it - 2 SB is released and the
    // parity wait cannot pass on a stale phase
    static_assert(SB >= PG, "B ring at least as deep as the prep groups");
    static_assert(SA >= 2, "A ring");
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t bar_afull[SA], bar_aempty[SA], bar_bready[SB], bar_bempty[SB], bar_acc[2], bar_tfree[2];
    __shared__ uint32_t tmem_base;
    __shared__ float s_scale[F], s_inv[F];   // per frame: 2^eB (prep) and 2^-(eA + eB) (epilogue)
    const uint32_t raw = tc::smem_u32(smem_raw);
    unsigned char* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    unsigned char* bring = smem + (size_t)SA * kFAStage;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntile = FWD ? 2 : (d.nu_pad + kFM - 1) / kFM;
    const int ksp = d.ksplit > 1 ? d.ksplit : 1;   // K splits per (kappa, tile): partial outputs ksp apart
    const int nitems = d.nkappa * ntile * ksp;
    const int nchunks = FWD ? (2 * d.nu_pad + kFK - 1) / kFK : (2 * d.bpitch + kFK - 1) / kFK;
    // item -> kappa, row tile, K split and its chunk range [c_lo, c_hi)
    auto decode = [&](int item, int& kap, int& t, int& sp, int& c_lo, int& c_hi) {
        kap = item / (ntile * ksp);
        const int rem = item - kap * ntile * ksp;
        t = rem / ksp;
        sp = rem - t * ksp;
        c_lo = (int)((long long)sp * nchunks / ksp);
        c_hi = (int)((long long)(sp + 1) * nchunks / ksp);
    };
    const int kvalid_last = (FWD ? 2 * d.nu_pad : 2 * d.N2) - (nchunks - 1) * kFK;   // real K elements, last chunk
    const int ks_last = (kvalid_last + 15) / 16;

    if (threadIdx.x == 0) {
        for (int i = 0; i < SA; ++i) {
            tc::mbar_init(&bar_afull[i], 1);
            tc::mbar_init(&bar_aempty[i], 1);
        }
        for (int i = 0; i < SB; ++i) {
            tc::mbar_init(&bar_bready[i], kFPrep / PG);
            tc::mbar_init(&bar_bempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&bar_acc[i], 1);
            tc::mbar_init(&bar_tfree[i], 4);
        }
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&d.tmapAh);
        tc::tma_prefetch_desc(&d.tmapAl);
    }
    if (warp == 0) tc::tmem_alloc(&tmem_base, 2 * NSET <= 256 ? 256 : 512);
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
        const int eb = d.bmax ? (f < d.nframes ? tc::f16_scale_exp(__uint_as_float(d.bmax[f])) : 0) : d.bexp[f];
        s_scale[f] = tc::pow2f(eb);
        s_inv[f] = ldexpf(1.0f, -(d.aexp + eb));
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;

    if (warp == 0) {
        if (lane == 0) {   // ---- producer: A hi / lo tiles per chunk ----
            int it = 0;
            for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
                int kap, t, sp, c_lo, c_hi;
                decode(item, kap, t, sp, c_lo, c_hi);
                for (int c = c_lo; c < c_hi; ++c, ++it) {
                    const int s = it % SA;
                    if (it >= SA) tc::mbar_wait(&bar_aempty[s], ((it / SA) - 1) & 1);
                    unsigned char* st = smem + (size_t)s * kFAStage;
                    tc::mbar_arrive_expect_tx(&bar_afull[s], kFAStage);
                    tc::tma_load_3d(st, &d.tmapAh, c * kFK, t * kFM, kap, &bar_afull[s]);
                    tc::tma_load_3d(st + kFATile, &d.tmapAl, c * kFK, t * kFM, kap, &bar_afull[s]);
                }
            }
        }
    } else if (warp <= kFPrep) {
        // ---- prep: stacked B rows from the fp32 source [F][32 complex] of the chunk (read through L2), scaled by
        //      2^eB[f], split hi | lo ----
        //   FWD  row 2f: (Gr, -Gi), row 2f+1: (Gi, Gr)   -> D[b'][2f] = Re Y_f, D[b'][2f+1] = Im Y_f
        //   BWD  row 2f: (Rr,  Ri), row 2f+1: (Ri, -Rr)  -> D[u][2f]  = Re Xh_f, D[u][2f+1] = Im Xh_f (conj(M) R)
        constexpr int NP = 32 * kFPrep / PG;
        constexpr int NE = (F * (kFK / 2) + NP - 1) / NP;   // complex source values per thread
        const int pt = (threadIdx.x - 32) % NP, grp = (threadIdx.x - 32) / NP;
        int it = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            int kap, t, sp, c_lo, c_hi;
            decode(item, kap, t, sp, c_lo, c_hi);
            for (int c = c_lo; c < c_hi; ++c, ++it) {
                if (it % PG != grp) continue;
                // the source values first (independent of the slot; L2 / DRAM), then wait for the slot
                const float2* gsrc = d.src + (long long)kap * d.src_n + (long long)c * (kFK / 2);
                float2 gv[NE];
#pragma unroll
                for (int i = 0; i < NE; ++i) {
                    const int e = pt + NP * i;
                    const int f = e / (kFK / 2), j = e - f * (kFK / 2);
                    gv[i] = (e < F * (kFK / 2) && f < d.nframes && c * (kFK / 2) + j < d.src_n)
                                ? __ldg(gsrc + (long long)f * d.src_fstride + j)
                                : make_float2(0.0f, 0.0f);
                }
                const int b = it % SB;
                if (it >= SB) tc::mbar_wait(&bar_bempty[b], ((it / SB) - 1) & 1);
                unsigned char* bt = bring + (size_t)b * f_btile(F);
#pragma unroll
                for (int i = 0; i < NE; ++i) {
                    const int e = pt + NP * i;
                    if (e < F * (kFK / 2)) {
                        const int f = e / (kFK / 2), j = e - f * (kFK / 2);
                        const float2 g = gv[i];
                        // two splits per complex value; the B entries are +-re / +-im, and -(h + l) = (-h) + (-l)
                        // is a sign flip of both fp16 halves
                        uint16_t rh, rl, ih, il;
                        tc::split_f16(g.x, s_scale[f], rh, rl);
                        tc::split_f16(g.y, s_scale[f], ih, il);
                        uint32_t h0, l0, h1, l1;   // rows 2f, 2f+1: (element 2j) | (element 2j+1) << 16
                        if constexpr (FWD) {       // (re, -im), (im, re)
                            h0 = (uint32_t)rh | ((uint32_t)(ih ^ 0x8000u) << 16);
                            l0 = (uint32_t)rl | ((uint32_t)(il ^ 0x8000u) << 16);
                            h1 = (uint32_t)ih | ((uint32_t)rh << 16);
                            l1 = (uint32_t)il | ((uint32_t)rl << 16);
                        } else {                   // (re, im), (im, -re)
                            h0 = (uint32_t)rh | ((uint32_t)ih << 16);
                            l0 = (uint32_t)rl | ((uint32_t)il << 16);
                            h1 = (uint32_t)ih | ((uint32_t)(rh ^ 0x8000u) << 16);
                            l1 = (uint32_t)il | ((uint32_t)(rl ^ 0x8000u) << 16);
                        }
#pragma unroll
                        for (int r = 0; r < 2; ++r) {
                            const int row = 2 * f + r, rowl = 2 * F + row;
                            // byte offset of elements (row, 2j .. 2j+1) in a K-major SWIZZLE_128B fp16 tile
                            const uint32_t off = (uint32_t)row * 128u + ((((uint32_t)(j >> 2)) ^ (row & 7)) & 7) * 16u + (j & 3) * 4u;
                            const uint32_t offl = (uint32_t)rowl * 128u + ((((uint32_t)(j >> 2)) ^ (rowl & 7)) & 7) * 16u + (j & 3) * 4u;
                            *reinterpret_cast<uint32_t*>(bt + off) = r ? h1 : h0;
                            *reinterpret_cast<uint32_t*>(bt + offl) = r ? l1 : l0;
                        }
                    }
                }
                tc::fence_proxy_async();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar_bready[b]);
            }
        }
    } else if (warp == kFPrep + 1) {
        // ---- MMA issuer (whole warp, uniform values, one elected lane issues) ----
        const uint32_t id1 = tc::idesc_f16(kFM, NB), id2 = tc::idesc_f16(kFM, 2 * F);
        int it = 0, g = 0, gk = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            int kap, t, sp, c_lo, c_hi;
            decode(item, kap, t, sp, c_lo, c_hi);
            for (int c = c_lo; c < c_hi; ++c, ++it) {
                const int s = it % SA, b = it % SB, j = g & 1;
                tc::mbar_wait(&bar_afull[s], (it / SA) & 1);
                tc::mbar_wait(&bar_bready[b], (it / SB) & 1);
                if (gk == 0 && g >= 2) tc::mbar_wait(&bar_tfree[j], ((g >> 1) - 1) & 1);
                tc::fence_after();
                const uint32_t a_hi = tc::smem_u32(smem + (size_t)s * kFAStage), a_lo = a_hi + kFATile;
                const uint32_t bsm = tc::smem_u32(bring + (size_t)b * f_btile(F));
                const uint32_t acc = tmem + (uint32_t)(j * NSET);
                const uint64_t ah0 = tc::sdesc_sw128(a_hi), al0 = tc::sdesc_sw128(a_lo), bd0 = tc::sdesc_sw128(bsm);
                const int ks = c == nchunks - 1 ? ks_last : kFKS;
                for (int k = 0; k < ks; ++k) {   // K-step k (16 fp16 = 32 bytes): descriptor address + 2 k
                    const uint64_t dk = 2 * (uint64_t)k;
                    tc::mma_f16_elect(acc, ah0 + dk, bd0 + dk, id1, (gk == 0 && k == 0) ? 0u : 1u);           // hi*hi | hi*lo
                    tc::mma_f16_elect(acc + 4 * F, al0 + dk, bd0 + dk, id2, (gk == 0 && k == 0) ? 0u : 1u);   // lo*hi
                }
                tc::mma_commit_elect(&bar_aempty[s]);
                tc::mma_commit_elect(&bar_bempty[b]);
                gk += ks;
                if (gk + kFKS > d.chain_k || c == c_hi - 1) {
                    tc::mma_commit_elect(&bar_acc[j]);
                    ++g;
                    gk = 0;
                }
            }
        }
    } else {
        // ---- drainers: TMEM -> fp32 running sums (2F per thread), unscale per frame, store ----
        const int q = warp & 3;
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
        float acc[2 * F];
#pragma unroll
        for (int i = 0; i < 2 * F; ++i) acc[i] = 0.0f;
        int g = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            int kap, t, sp, c_lo, c_hi;
            decode(item, kap, t, sp, c_lo, c_hi);
            for (int c = c_lo, gk = 0; c < c_hi; ++c) {   // the issuer's drain groups
                gk += c == nchunks - 1 ? ks_last : kFKS;
                if (!(gk + kFKS > d.chain_k || c == c_hi - 1)) continue;
                gk = 0;
                const int j = g & 1;
                tc::mbar_wait(&bar_acc[j], (g >> 1) & 1);
                ++g;
                tc::fence_after();
                const uint32_t base = lane_base + (uint32_t)(j * NSET);
#pragma unroll
                for (int b0 = 0; b0 < 3; ++b0) {   // up to 32 columns in flight per wait (not one wait per 8)
#pragma unroll
                    for (int c8 = 0; c8 < 2 * F; c8 += 32) {
                        constexpr int W = 2 * F < 32 ? 2 * F : 32;
                        uint32_t v[W];
                        if constexpr (W == 32) {
                            tc::tmem_ld32_nowait(base + (uint32_t)(b0 * 2 * F + c8), v);
                        } else {
#pragma unroll
                            for (int c = 0; c < W; c += 8) tc::tmem_ld8_nowait(base + (uint32_t)(b0 * 2 * F + c8 + c), v + c);
                        }
                        tc::tmem_wait_ld();
#pragma unroll
                        for (int u = 0; u < W; ++u) acc[c8 + u] += __uint_as_float(v[u]);
                    }
                }
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar_tfree[j]);
            }
            const int row = t * kFM + 32 * q + lane;
            if (row < (FWD ? d.N2 : d.nu_pad)) {
#pragma unroll
                for (int f = 0; f < F; ++f) {
                    if (f >= d.nframes) break;
                    const float inv = s_inv[f];
                    const float2 v = make_float2(acc[2 * f] * inv, acc[2 * f + 1] * inv);
                    d.out[(long long)sp * d.out_sstride + (long long)f * d.out_fstride + (long long)kap * d.out_ld + row] = v;
                }
            }
#pragma unroll
            for (int i = 0; i < 2 * F; ++i) acc[i] = 0.0f;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 2 * NSET <= 256 ? 256 : 512);
}

// ---------------------------------------------------------------------------------------------------------------
// plan time: max |M| (float bits), transposed copy M^T, in-place split of complex64 rows into [hi | lo] fp16 rows

__global__ void mf_amax_kernel(const float* __restrict__ p, size_t n, unsigned* __restrict__ out) {
    float m = 0.0f;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        m = fmaxf(m, fabsf(p[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0f) atomicMax(out, __float_as_uint(m));
}

// MT[kap][u][b'] (row pitch bpitch complex, zeros for b' >= N2) = M[kap][b'][u] (row pitch nu_pad)
__global__ void mf_transpose_kernel(const float2* __restrict__ M, float2* __restrict__ MT, int N2, int nu_pad, int bpitch) {
    __shared__ float2 tile[32][33];
    const int kap = blockIdx.z;
    const int u0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
    const float2* src = M + (size_t)kap * N2 * nu_pad;
    float2* dst = MT + (size_t)kap * nu_pad * bpitch;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int b = b0 + r, u = u0 + threadIdx.x;
        tile[r][threadIdx.x] = (b < N2 && u < nu_pad) ? src[(size_t)b * nu_pad + u] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int u = u0 + r, b = b0 + threadIdx.x;
        if (u < nu_pad && b < bpitch) dst[(size_t)u * bpitch + b] = tile[threadIdx.x][r];
    }
}

// one CTA per row of n complex: [re0 im0 re1 im1 ...] fp32 -> [hi: 2n fp16][lo: 2n fp16], scaled by 2^e
__global__ void mf_split_rows_kernel(float2* __restrict__ rows, int n, int e) {
    extern __shared__ float2 rowbuf[];
    float2* row = rows + (size_t)blockIdx.x * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) rowbuf[i] = row[i];
    __syncthreads();
    uint32_t* hi = reinterpret_cast<uint32_t*>(row);   // n uint32 = 2n fp16
    uint32_t* lo = hi + n;
    const float sc = tc::pow2f(e);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        uint16_t h0, l0, h1, l1;
        tc::split_f16(rowbuf[i].x, sc, h0, l0);
        tc::split_f16(rowbuf[i].y, sc, h1, l1);
        hi[i] = (uint32_t)h0 | ((uint32_t)h1 << 16);
        lo[i] = (uint32_t)l0 | ((uint32_t)l1 << 16);
    }
}

// per-frame scale exponents from the DC bound: eB[f] = f16_scale_exp(max_c |src[f][kappa = 0][c]|), c < n
__global__ void mf_frame_scale_kernel(const float2* __restrict__ src, long long fstride, int n, int* __restrict__ eb) {
    float m = 0.0f;
    const float2* p = src + (long long)blockIdx.x * fstride;
    for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmaxf(m, fmaxf(fabsf(p[i].x), fabsf(p[i].y)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ float wm[32];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, wm[w]);
        eb[blockIdx.x] = tc::f16_scale_exp(m);
    }
}

typedef CUresult (*MfEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static MfEncodeFn mf_encoder() {
    static MfEncodeFn enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            enc = nullptr;
    }
    return enc;
}

// plan time: split M (forward operand) and build + split M^T (backward operand); encode both directions' A maps
cudaError_t mac_f16_prepare(float2* M, const float2* Mb, float2* MT, int nkappa, int N2, int nu_pad, int bpitch,
                            MacF16Args* fwd, MacF16Args* bwd, cudaStream_t s) {
    unsigned* am = nullptr;
    cudaError_t e = cudaMalloc(&am, 2 * sizeof(unsigned));
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(am, 0, 2 * sizeof(unsigned), s);
    const size_t nf = (size_t)nkappa * N2 * nu_pad * 2;
    mf_amax_kernel<<<4 * 148, 256, 0, s>>>(reinterpret_cast<const float*>(M), nf, am);
    mf_amax_kernel<<<4 * 148, 256, 0, s>>>(reinterpret_cast<const float*>(Mb), nf, am + 1);
    // the transpose reads the backward matrices before M is split in place (Mb may be M)
    mf_transpose_kernel<<<dim3((nu_pad + 31) / 32, (bpitch + 31) / 32, nkappa), dim3(32, 8), 0, s>>>(Mb, MT, N2, nu_pad, bpitch);
    unsigned amh[2] = {0, 0};
    cudaMemcpyAsync(amh, am, sizeof(amh), cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    cudaFree(am);
    if (e != cudaSuccess) return e;
    float amf[2];
    memcpy(amf, amh, sizeof(amf));
    const int ea = tc::f16_scale_exp(amf[0]), eb = tc::f16_scale_exp(amf[1]);
    e = cudaFuncSetAttribute(mf_split_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(nu_pad * sizeof(float2)));
    if (e != cudaSuccess) return e;
    mf_split_rows_kernel<<<nkappa * N2, 256, nu_pad * sizeof(float2), s>>>(M, nu_pad, ea);
    mf_split_rows_kernel<<<nkappa * nu_pad, 256, bpitch * sizeof(float2), s>>>(MT, bpitch, eb);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    MfEncodeFn enc = mf_encoder();
    if (!enc) return cudaErrorSymbolNotFound;
    cuuint32_t es[3] = {1, 1, 1};
    for (int w = 0; w < 2; ++w) {
        MacF16Args* a = w ? bwd : fwd;
        a->nkappa = nkappa;
        a->N2 = N2;
        a->nu_pad = nu_pad;
        a->bpitch = bpitch;
        a->aexp = w ? eb : ea;
        a->chain_k = getenv("LFM_MF_CHAIN") ? std::max(4, atoi(getenv("LFM_MF_CHAIN"))) : 24;   // dev override
        const int n = w ? bpitch : nu_pad;               // complex per split row
        const int rows = w ? nu_pad : N2;
        unsigned char* base = reinterpret_cast<unsigned char*>(w ? MT : M);
        cuuint64_t dims[3] = {(cuuint64_t)2 * n, (cuuint64_t)rows, (cuuint64_t)nkappa};
        cuuint64_t strides[2] = {(cuuint64_t)n * 8, (cuuint64_t)rows * n * 8};
        cuuint32_t box[3] = {(cuuint32_t)kFK, (cuuint32_t)kFM, 1};
        for (int part = 0; part < 2; ++part) {
            CUresult r = enc(part ? &a->tmapAl : &a->tmapAh, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, base + (size_t)part * n * 4,
                             dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
        }
    }
    return cudaSuccess;
}

// per call: the frames' fp32 source spectra (FWD: G [F][kappa][nu_pad]; BWD: R [F][kappa][bpitch]), read by the prep
// warps (frames nframes .. F-1 and the K tail read as zeros)
cudaError_t mac_f16_encode_src(MacF16Args* a, int fwd, const float2* src, long long src_fstride, int F, int nframes) {
    if (nframes <= 0 || nframes > F) nframes = F;
    const int n = fwd ? a->nu_pad : a->bpitch;
    a->nframes = nframes;   // frames nframes .. F-1 read as zeros (TMA out of bounds / the prep warps' bounds check)
    a->src = src;
    a->src_fstride = src_fstride;
    a->src_n = n;
    if (F >= 32) return cudaSuccess;   // the two-ring kernel reads the source directly
    MfEncodeFn enc = mf_encoder();
    if (!enc) return cudaErrorSymbolNotFound;
    cuuint64_t dims[3] = {(cuuint64_t)2 * n, (cuuint64_t)a->nkappa, (cuuint64_t)nframes};
    cuuint64_t strides[2] = {(cuuint64_t)n * 8, (cuuint64_t)src_fstride * 8};
    cuuint32_t box[3] = {(cuuint32_t)kFK, 1, (cuuint32_t)F}, es[3] = {1, 1, 1};
    CUresult r = enc(&a->tmapS, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(src), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_frame_scales(const float2* src, long long fstride, int n, int F, int* eb, cudaStream_t s) {
    mf_frame_scale_kernel<<<F, 256, 0, s>>>(src, fstride, n, eb);
    return cudaGetLastError();
}

template <int F, bool FWD>
static cudaError_t launch_mf(const MacF16Args& d, int num_sms, cudaStream_t s) {
    const size_t smem = mac_f16_smem_bytes(F);
    const int ntile = FWD ? 2 : (d.nu_pad + kFM - 1) / kFM;
    const int grid = std::max(1, std::min(d.nkappa * ntile * std::max(1, d.ksplit), num_sms));
    if constexpr (F >= 32) {
        cudaError_t e = cudaFuncSetAttribute(mac_f16_kernel<F, f_pg(F), FWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        mac_f16_kernel<F, f_pg(F), FWD><<<grid, kFThreads, smem, s>>>(d);
    } else {
        cudaError_t e = cudaFuncSetAttribute(mac_f16_tma_kernel<F, 4, FWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        mac_f16_tma_kernel<F, 4, FWD><<<grid, kFThreads, smem, s>>>(d);
    }
    return cudaGetLastError();
}

cudaError_t launch_mac_f16(const MacF16Args& d, int fwd, int F, int num_sms, cudaStream_t s) {
    switch (F) {
        case 8: return fwd ? launch_mf<8, true>(d, num_sms, s) : launch_mf<8, false>(d, num_sms, s);
        case 16: return fwd ? launch_mf<16, true>(d, num_sms, s) : launch_mf<16, false>(d, num_sms, s);
        case 32: return fwd ? launch_mf<32, true>(d, num_sms, s) : launch_mf<32, false>(d, num_sms, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lfm
