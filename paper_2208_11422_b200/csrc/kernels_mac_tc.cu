// kernels_mac_tc.cu -- frame-batched forward MAC on the 5th-generation tensor cores ("FP32 SIMT first,
// then tcgen05 3xTF32").
//
// Per coarse frequency kappa the batched forward projection is a complex GEMM over the frequency-path units u:
//   Y_f[kappa][b'] = sum_u M[kappa][b'][u] G_f[kappa][u]          (F frames)
// written as a real GEMM over K = (u, re/im) interleaved, which is exactly M's memory layout [b'][u] complex:
//   D[b'][n] = sum_k A[b'][k] B[n][k],   A = M[kappa] viewed as real (K-major, streamed by TMA),
//   B rows n = 2f   : ( Gr(u0), -Gi(u0), Gr(u1), -Gi(u1), ...)  -> D[b'][2f]   = Re Y_f[b']
//   B rows n = 2f+1 : ( Gi(u0),  Gr(u0), Gi(u1),  Gr(u1), ...)  -> D[b'][2f+1] = Im Y_f[b']
// 3xTF32: A_hi is the raw fp32 tile (the tensor core truncates it to TF32 = hi), A_lo = rna_tf32(a - hi) is written
// next to it by SIMT warps; B_hi and B_lo (rna splits) are stacked in one tile of 4F rows, so one MMA with N = 4F
// gives A_hi·B_hi | A_hi·B_lo and a second with N = 2F (the B_hi half) gives A_lo·B_hi.  The three column blocks are
// summed by the drainers in fp32 with round-to-nearest after every 16 K-steps (tcgen05 accumulation truncates).
//
// CTA = (kappa, half of the output phases): M = 128 rows b' in [128 h, 128 h + 128) (rows >= N^2 are TMA zero fill).
// Warp roles: 0 TMA producer, 1-8 prep (A_lo + B build), 9 MMA issuer (one thread), 10-13 drainers / epilogue.
#include <algorithm>
#include <cstdlib>

#include "lfm_internal.cuh"
#include "tc_sm100.cuh"

namespace lfm {

namespace {
constexpr int kMtM = 128;                 // rows (output phases) per CTA
constexpr int kMtKC = 32;                 // K floats per chunk (16 complex units, one 128-byte swizzle row)
constexpr int kMtChain = 4;               // chunks (x 4 K-steps) per drain group
// warps: 1 producer + NPREP prep + 1 MMA + 4 drainers (NPREP = 8 or 16, template parameter)
__host__ __device__ constexpr int mt_threads(int NPREP) { return 32 * (NPREP + 6); }
// Prep groups: group g of kMtPrep / PG warps prepares the chunks it with it % PG == g (each warp's wait -> build ->
// fence -> arrive chain is serial per chunk, so PG groups keep PG chunks in preparation).  A ring stage s = it % S is
// reused by chunk it + S, which (unless PG divides S) another group prepares.  With one fill barrier per stage a
// group waiting for chunk it's fill could find that barrier one phase behind (chunk it - S not yet filled) or one
// phase ahead (chunk it filled, chunk it + S in flight) -- the same parity, so a parity wait cannot tell them apart
// and may pass on chunk it - S's completed phase (the fault 4 groups hit in r01).  Each (group, stage) pair
// therefore has its own fill barrier: bar_fullA[g][s] serves the chunks it = g (mod PG), s (mod S), i.e. every
// L = lcm(PG, S)-th chunk, all prepared by group g in order, so the phase of chunk it is it / L and unambiguous.
constexpr uint32_t kMtATile = kMtM * kMtKC * 4;   // 16 KB
constexpr uint32_t kMtSmemMax = 232448;           // 227 KB per CTA

__host__ __device__ constexpr uint32_t mt_round1k(uint32_t v) { return (v + 1023u) & ~1023u; }
__host__ __device__ constexpr uint32_t mt_btile(int F) { return mt_round1k((uint32_t)(4 * F) * kMtKC * 4); }
__host__ __device__ constexpr uint32_t mt_gtile(int F) { return (uint32_t)F * kMtKC * 4; }   // F rows of 128 B
__host__ __device__ constexpr uint32_t mt_stage(int F) { return 2 * kMtATile + mt_btile(F) + mt_round1k(mt_gtile(F)); }
// deepest ring that fits next to the 1 KB alignment slack, at most 8 stages
__host__ __device__ constexpr int ring_depth(uint32_t stage_bytes, int PG) {
    return (int)((kMtSmemMax - 1024) / stage_bytes) < 8 ? (int)((kMtSmemMax - 1024) / stage_bytes) : 8 + 0 * PG;
}
__host__ __device__ constexpr int mt_stages(int F, int PG) { return ring_depth(mt_stage(F), PG); }
__host__ __device__ constexpr int mt_gcd(int a, int b) { return b == 0 ? a : mt_gcd(b, a % b); }
}  // namespace

// prep configuration (warps, groups): (8, 2), (8, 4) default, (16, 4); dev overrides LFM_MT_PREP / LFM_MT_PG
int mac_tc_prep_warps() {
    static int np = [] {
        const char* e = getenv("LFM_MT_PREP");
        return e && atoi(e) == 16 ? 16 : 8;
    }();
    return np;
}
int mac_tc_prep_groups() {
    static int pg = [] {
        const char* e = getenv("LFM_MT_PG");
        const int v = e ? atoi(e) : 4;
        if (mac_tc_prep_warps() == 16) return 4;
        return v == 2 ? 2 : 4;
    }();
    return pg;
}

size_t mac_tc_smem_bytes(int F) { return (size_t)mt_stages(F, mac_tc_prep_groups()) * mt_stage(F) + 1024; }

template <int F, int PG, int NPREP>
__global__ void __launch_bounds__(mt_threads(NPREP), 1) fmb_tc_kernel(const __grid_constant__ MacTcArgs d) {
    constexpr int S = mt_stages(F, PG);
    constexpr int kMtPG = PG;
    constexpr int kMtPrep = NPREP;
    static_assert(S >= PG, "every prep group needs a stage");
    constexpr int NB = 4 * F;       // rows of the stacked B tile (B_hi: 0..2F-1, B_lo: 2F..4F-1)
    constexpr int NSET = 6 * F;     // TMEM columns per accumulator set: hi*hi | hi*lo | lo*hi
    extern __shared__ unsigned char smem_raw[];
    constexpr int LG = PG * S / mt_gcd(PG, S);   // chunks between two uses of one (group, stage) fill barrier
    __shared__ uint64_t bar_fullA[PG][S], bar_ready[S], bar_empty[S], bar_acc[2], bar_tfree[2];
    __shared__ uint32_t tmem_base;
    const uint32_t raw = tc::smem_u32(smem_raw);
    unsigned char* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sbytes = mt_stage(F);
    const int nitems = 2 * d.nkappa;
    const int nchunks = 2 * d.nu_pad / kMtKC;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            for (int g = 0; g < PG; ++g) tc::mbar_init(&bar_fullA[g][i], 1);
            tc::mbar_init(&bar_ready[i], kMtPrep / kMtPG);
            tc::mbar_init(&bar_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&bar_acc[i], 1);
            tc::mbar_init(&bar_tfree[i], 4);
        }
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&d.tmapM);
        tc::tma_prefetch_desc(&d.tmapG);
    }
    if (warp == 0) tc::tmem_alloc(&tmem_base, 2 * NSET <= 256 ? 256 : 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;

    if (warp == 0) {
        if (lane == 0) {   // ---- producer: A tiles (rows b' of M[kappa], 32 K floats) ----
            int it = 0;
            for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
                const int kap = item >> 1, h = item & 1;
                for (int c = 0; c < nchunks; ++c, ++it) {
                    const int s = it % S;
                    if (it >= S) tc::mbar_wait(&bar_empty[s], ((it / S) - 1) & 1);
                    unsigned char* st = smem + (size_t)s * sbytes;
                    uint64_t* fb = &bar_fullA[it % PG][s];
                    tc::mbar_arrive_expect_tx(fb, kMtATile + mt_gtile(F));
                    tc::tma_load_3d(st, &d.tmapM, c * kMtKC, h * kMtM, kap, fb);
                    // the frames' G for this chunk: F rows of 16 complex units (plain row-major)
                    tc::tma_load_3d(st + 2 * kMtATile + mt_btile(F), &d.tmapG,
                                    (int)((long long)kap * 2 * d.nu_pad % d.gsplit) + c * kMtKC,
                                    (int)((long long)kap * 2 * d.nu_pad / d.gsplit), 0, fb);
                }
            }
        }
    } else if (warp <= kMtPrep) {
        // ---- prep warps: A_lo = rna_tf32(a - trunc_tf32(a)); stacked B_hi | B_lo from the frames' G ----
        constexpr int NP = 32 * kMtPrep / kMtPG;         // prep threads per group
        constexpr int NA = (int)(kMtATile / 16) / NP;    // float4 of the A tile per thread
        constexpr int NE = (2 * F * kMtKC) / NP;         // B elements per thread (per stacked half)
        const int pt = (threadIdx.x - 32) % NP, grp = (threadIdx.x - 32) / NP;
        int it = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            for (int c = 0; c < nchunks; ++c, ++it) {
                if (it % kMtPG != grp) continue;
                const int s = it % S;
                tc::mbar_wait(&bar_fullA[grp][s], (it / LG) & 1);   // this group's own fill barrier (see above)
                unsigned char* st = smem + (size_t)s * sbytes;
                const float4* ahi = reinterpret_cast<const float4*>(st);
                float4* alo = reinterpret_cast<float4*>(st + kMtATile);
                unsigned char* bt = st + 2 * kMtATile;
                const float2* gt = reinterpret_cast<const float2*>(bt + mt_btile(F));   // [F][16] complex
                float4 a[NA];
                float2 gv[NE];
#pragma unroll
                for (int i = 0; i < NA; ++i) a[i] = ahi[pt + NP * i];   // loads first (ILP)
#pragma unroll
                for (int i = 0; i < NE; ++i) {
                    const int e = pt + NP * i, n = e / kMtKC, k = e - (e / kMtKC) * kMtKC;
                    gv[i] = gt[(n >> 1) * (kMtKC / 2) + (k >> 1)];
                }
#pragma unroll
                for (int i = 0; i < NA; ++i) {   // elementwise: the swizzle is irrelevant
                    float4 l;
                    l.x = tc::tf32_lo_of_trunc(a[i].x);
                    l.y = tc::tf32_lo_of_trunc(a[i].y);
                    l.z = tc::tf32_lo_of_trunc(a[i].z);
                    l.w = tc::tf32_lo_of_trunc(a[i].w);
                    alo[pt + NP * i] = l;
                }
                // B element (n, k), n < 2F: frame f = n / 2, unit j = k / 2 of the chunk, component k & 1
#pragma unroll
                for (int i = 0; i < NE; ++i) {
                    const int e = pt + NP * i, n = e / kMtKC, k = e - (e / kMtKC) * kMtKC;
                    const float2 g = gv[i];
                    const float v = (n & 1) == 0 ? ((k & 1) ? -g.y : g.x) : ((k & 1) ? g.x : g.y);
                    float hi, lo;
                    tc::split_tf32(v, hi, lo);
                    *reinterpret_cast<float*>(bt + tc::sw128_off(n, k)) = hi;
                    *reinterpret_cast<float*>(bt + tc::sw128_off(2 * F + n, k)) = lo;
                }
                tc::fence_proxy_async();   // generic-proxy smem writes -> visible to the tensor core
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar_ready[s]);
            }
        }
    } else if (warp == kMtPrep + 1) {
        {   // ---- MMA issuer: the whole warp on uniform values, one elected lane issues (§5.3) ----
            const uint32_t id1 = tc::idesc_tf32(kMtM, NB), id2 = tc::idesc_tf32(kMtM, 2 * F);
            int it = 0, g = 0, gk = 0;
            for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
                for (int c = 0; c < nchunks; ++c, ++it) {
                    const int s = it % S, j = g & 1;
                    tc::mbar_wait(&bar_ready[s], (it / S) & 1);
                    if (gk == 0 && g >= 2) tc::mbar_wait(&bar_tfree[j], ((g >> 1) - 1) & 1);
                    tc::fence_after();
                    const uint32_t a_hi = tc::smem_u32(smem + (size_t)s * sbytes), a_lo = a_hi + kMtATile;
                    const uint32_t b = a_hi + 2 * kMtATile;
                    const uint32_t acc = tmem + (uint32_t)(j * NSET);
                    const uint64_t ah0 = tc::sdesc_sw128(a_hi), al0 = tc::sdesc_sw128(a_lo), bd0 = tc::sdesc_sw128(b);
#pragma unroll
                    for (int k = 0; k < kMtKC / 8; ++k) {   // K-step k: start address + 32 k bytes = field + 2 k
                        const uint64_t dk = 2 * (uint64_t)k;
                        tc::mma_tf32_elect(acc, ah0 + dk, bd0 + dk, id1, (gk == 0 && k == 0) ? 0u : 1u);          // hi*hi | hi*lo
                        tc::mma_tf32_elect(acc + 4 * F, al0 + dk, bd0 + dk, id2, (gk == 0 && k == 0) ? 0u : 1u);  // lo*hi
                    }
                    tc::mma_commit_elect(&bar_empty[s]);
                    if (++gk == kMtChain || c == nchunks - 1) {
                        tc::mma_commit_elect(&bar_acc[j]);
                        ++g;
                        gk = 0;
                    }
                }
            }
        }
    } else {
        // ---- drainers: TMEM -> fp32 running sums (2F per thread), epilogue ----
        const int q = warp & 3;   // warps 10-13: lane quarters 2, 3, 0, 1
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
        float acc[2 * F];
#pragma unroll
        for (int i = 0; i < 2 * F; ++i) acc[i] = 0.0f;
        int g = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            const int kap = item >> 1, h = item & 1;
            for (int c0 = 0; c0 < nchunks; c0 += kMtChain) {
                const int j = g & 1;
                tc::mbar_wait(&bar_acc[j], (g >> 1) & 1);
                ++g;
                tc::fence_after();
                const uint32_t base = lane_base + (uint32_t)(j * NSET);
#pragma unroll
                for (int b0 = 0; b0 < 3; ++b0) {   // column blocks hi*hi, hi*lo, lo*hi (2F columns each)
#pragma unroll
                    for (int c8 = 0; c8 < 2 * F; c8 += 8) {
                        uint32_t v[8];
                        tc::tmem_ld8_nowait(base + (uint32_t)(b0 * 2 * F + c8), v);
                        tc::tmem_wait_ld();
#pragma unroll
                        for (int u = 0; u < 8; ++u) acc[c8 + u] += __uint_as_float(v[u]);
                    }
                }
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar_tfree[j]);
            }
            const int row = h * kMtM + 32 * q + lane;
            if (row < d.N2) {
#pragma unroll
                for (int f = 0; f < F; ++f)
                    d.Y[(long long)f * d.y_fstride + (long long)kap * d.N2 + row] = make_float2(acc[2 * f], acc[2 * f + 1]);
            }
#pragma unroll
            for (int i = 0; i < 2 * F; ++i) acc[i] = 0.0f;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 2 * NSET <= 256 ? 256 : 512);
}

// ================================================================================================================
// Frame-batched BACKWARD MAC on tcgen05: per kappa  Xh_f[u] = sum_b' conj(M[b'][u]) R_f[b'].
// M[kappa] is [b'][u] complex (u contiguous), so with u' = (u, re/im) interleaved as the GEMM's M dimension and b' as
// K, A[u'][b'] = M_float[b'][u'] is an MN-major operand (SWIZZLE_128B_BASE32B: the only MN-major tf32 layout),
// loaded by TMA straight from the transfer matrices.  B rows n = 2f + p hold R_f's real (p = 0) / imaginary (p = 1)
// parts, so D[u'][2f + p] = sum_b' A[u'][b'] R_p,f[b'] and, with (re, im) = rows (2u, 2u + 1),
//   Re Xh = D[2u][2f] + D[2u+1][2f+1],   Im Xh = D[2u][2f+1] - D[2u+1][2f]     (conj(m) r, no extra factor).
// 3xTF32 exactly as in the forward (A_hi raw, A_lo by the prep warps, B_hi | B_lo stacked).  Item = (kappa, 128 u').
// ================================================================================================================
namespace {
constexpr int kBmKC = 32;                                   // K rows (b') per chunk
__host__ __device__ constexpr uint32_t bm_stage(int F) { return 2 * kMtATile + mt_btile(F); }
}  // namespace

__host__ __device__ constexpr int bm_stages(int F, int PG) { return ring_depth(bm_stage(F), PG); }

size_t bmac_tc_smem_bytes(int F) { return (size_t)bm_stages(F, mac_tc_prep_groups()) * bm_stage(F) + 1024; }

template <int F, int PG, int NPREP>
__global__ void __launch_bounds__(mt_threads(NPREP), 1) bmb_tc_kernel(const __grid_constant__ BmacTcArgs d) {
    constexpr int S = bm_stages(F, PG);
    constexpr int kMtPG = PG;
    constexpr int kMtPrep = NPREP;
    static_assert(S >= PG, "every prep group needs a stage");
    constexpr int NB = 4 * F;
    constexpr int NSET = 6 * F;
    extern __shared__ unsigned char smem_raw[];
    constexpr int LG = PG * S / mt_gcd(PG, S);   // chunks between two uses of one (group, stage) fill barrier
    __shared__ uint64_t bar_fullA[PG][S], bar_ready[S], bar_empty[S], bar_acc[2], bar_tfree[2];
    __shared__ uint32_t tmem_base;
    const uint32_t raw = tc::smem_u32(smem_raw);
    unsigned char* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sbytes = bm_stage(F);
    const int ntile = (2 * d.nu_pad + kMtM - 1) / kMtM;
    const int nitems = d.nkappa * ntile;
    const int nchunks = (d.N2 + kBmKC - 1) / kBmKC;
    const int kst_last = ((d.N2 - (nchunks - 1) * kBmKC) + 7) / 8;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            for (int g = 0; g < PG; ++g) tc::mbar_init(&bar_fullA[g][i], 1);
            tc::mbar_init(&bar_ready[i], kMtPrep / kMtPG);
            tc::mbar_init(&bar_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&bar_acc[i], 1);
            tc::mbar_init(&bar_tfree[i], 4);
        }
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&d.tmapA);
    }
    if (warp == 0) tc::tmem_alloc(&tmem_base, 2 * NSET <= 256 ? 256 : 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;

    if (warp == 0) {
        if (lane == 0) {   // ---- producer: A = 4 MN blocks of 32 u' x 32 b' (4 KB each) ----
            int it = 0;
            for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
                const int kap = item / ntile, t = item - kap * ntile;
                for (int c = 0; c < nchunks; ++c, ++it) {
                    const int s = it % S;
                    if (it >= S) tc::mbar_wait(&bar_empty[s], ((it / S) - 1) & 1);
                    unsigned char* st = smem + (size_t)s * sbytes;
                    uint64_t* fb = &bar_fullA[it % PG][s];
                    tc::mbar_arrive_expect_tx(fb, kMtATile);
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        tc::tma_load_3d(st + b * 4096, &d.tmapA, t * kMtM + 32 * b, c * kBmKC, kap, fb);
                }
            }
        }
    } else if (warp <= kMtPrep) {
        // ---- prep warps: A_lo = rna_tf32(a - trunc_tf32(a)); stacked B_hi | B_lo rows (f, re/im) from R (global,
        //      L2-resident: a kappa row of R is 225 x 8 bytes, not a TMA-legal stride) ----
        constexpr int NP = 32 * kMtPrep / kMtPG;
        constexpr int NA = (int)(kMtATile / 16) / NP;
        constexpr int NE = (2 * F * kBmKC) / NP;
        const int pt = (threadIdx.x - 32) % NP, grp = (threadIdx.x - 32) / NP;
        int it = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            const int kap = item / ntile;
            for (int c = 0; c < nchunks; ++c, ++it) {
                if (it % kMtPG != grp) continue;
                const int s = it % S;
                float2 rv[NE];
#pragma unroll
                for (int i = 0; i < NE; ++i) {   // issued before the wait: overlaps the A tile's arrival
                    const int e = pt + NP * i, n = e / kBmKC, k = e - (e / kBmKC) * kBmKC, bq = c * kBmKC + k;
                    rv[i] = bq < d.N2 ? __ldg(d.R + (long long)(n >> 1) * d.r_fstride + (long long)kap * d.N2 + bq)
                                      : make_float2(0.f, 0.f);
                }
                tc::mbar_wait(&bar_fullA[grp][s], (it / LG) & 1);   // this group's own fill barrier (see above)
                unsigned char* st = smem + (size_t)s * sbytes;
                const float4* ahi = reinterpret_cast<const float4*>(st);
                float4* alo = reinterpret_cast<float4*>(st + kMtATile);
                unsigned char* bt = st + 2 * kMtATile;
                float4 a[NA];
#pragma unroll
                for (int i = 0; i < NA; ++i) a[i] = ahi[pt + NP * i];
#pragma unroll
                for (int i = 0; i < NA; ++i) {   // elementwise: the swizzle is irrelevant
                    float4 l;
                    l.x = tc::tf32_lo_of_trunc(a[i].x);
                    l.y = tc::tf32_lo_of_trunc(a[i].y);
                    l.z = tc::tf32_lo_of_trunc(a[i].z);
                    l.w = tc::tf32_lo_of_trunc(a[i].w);
                    alo[pt + NP * i] = l;
                }
#pragma unroll
                for (int i = 0; i < NE; ++i) {   // B element (n = 2f + p, k = b' in the chunk)
                    const int e = pt + NP * i, n = e / kBmKC, k = e - (e / kBmKC) * kBmKC;
                    const float v = (n & 1) ? rv[i].y : rv[i].x;
                    float hi, lo;
                    tc::split_tf32(v, hi, lo);
                    *reinterpret_cast<float*>(bt + tc::sw128_off(n, k)) = hi;
                    *reinterpret_cast<float*>(bt + tc::sw128_off(2 * F + n, k)) = lo;
                }
                tc::fence_proxy_async();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar_ready[s]);
            }
        }
    } else if (warp == kMtPrep + 1) {
        {   // ---- MMA issuer: whole warp, uniform values, one elected lane issues ----
            const uint32_t id1 = tc::idesc_tf32(kMtM, NB) | (1u << 15), id2 = tc::idesc_tf32(kMtM, 2 * F) | (1u << 15);
            int it = 0, g = 0, gk = 0;
            for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
                for (int c = 0; c < nchunks; ++c, ++it) {
                    const int s = it % S, j = g & 1;
                    tc::mbar_wait(&bar_ready[s], (it / S) & 1);
                    if (gk == 0 && g >= 2) tc::mbar_wait(&bar_tfree[j], ((g >> 1) - 1) & 1);
                    tc::fence_after();
                    const uint32_t a_hi = tc::smem_u32(smem + (size_t)s * sbytes), a_lo = a_hi + kMtATile;
                    const uint32_t b = a_hi + 2 * kMtATile;
                    const uint32_t acc = tmem + (uint32_t)(j * NSET);
                    // A: MN-major SWIZZLE_128B_BASE32B, LBO = 4 KB between 32-element M blocks, SBO = 512 B between
                    // 4-row K groups; K-step k starts 8 rows = 1 KB further.  B: K-major SW128 (+32 B per K-step).
                    const uint64_t ah0 = tc::sdesc(a_hi, 4096, 512) | ((uint64_t)1u << 61);
                    const uint64_t al0 = tc::sdesc(a_lo, 4096, 512) | ((uint64_t)1u << 61);
                    const uint64_t bd0 = tc::sdesc_sw128(b);
                    const int ks = c == nchunks - 1 ? kst_last : kBmKC / 8;
                    for (int k = 0; k < ks; ++k) {
                        const uint64_t da = 64 * (uint64_t)k, db = 2 * (uint64_t)k;
                        tc::mma_tf32_elect(acc, ah0 + da, bd0 + db, id1, (gk == 0 && k == 0) ? 0u : 1u);        // hi*hi | hi*lo
                        tc::mma_tf32_elect(acc + 4 * F, al0 + da, bd0 + db, id2, (gk == 0 && k == 0) ? 0u : 1u);  // lo*hi
                    }
                    tc::mma_commit_elect(&bar_empty[s]);
                    if (++gk == kMtChain || c == nchunks - 1) {
                        tc::mma_commit_elect(&bar_acc[j]);
                        ++g;
                        gk = 0;
                    }
                }
            }
        }
    } else {
        // ---- drainers: TMEM -> fp32 running sums (2F per thread, row u'), pair (re, im) rows, epilogue ----
        const int q = warp & 3;
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
        float acc[2 * F];
#pragma unroll
        for (int i = 0; i < 2 * F; ++i) acc[i] = 0.0f;
        int g = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            const int kap = item / ntile, t = item - kap * ntile;
            for (int c0 = 0; c0 < nchunks; c0 += kMtChain) {
                const int j = g & 1;
                tc::mbar_wait(&bar_acc[j], (g >> 1) & 1);
                ++g;
                tc::fence_after();
                const uint32_t base = lane_base + (uint32_t)(j * NSET);
#pragma unroll
                for (int b0 = 0; b0 < 3; ++b0) {
#pragma unroll
                    for (int c8 = 0; c8 < 2 * F; c8 += 8) {
                        uint32_t v[8];
                        tc::tmem_ld8_nowait(base + (uint32_t)(b0 * 2 * F + c8), v);
                        tc::tmem_wait_ld();
#pragma unroll
                        for (int u = 0; u < 8; ++u) acc[c8 + u] += __uint_as_float(v[u]);
                    }
                }
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar_tfree[j]);
            }
            const int row = t * kMtM + 32 * q + lane;   // u' = 2u + (re/im)
            const int u = row >> 1;
#pragma unroll
            for (int f = 0; f < F; ++f) {
                const float oR = __shfl_down_sync(0xffffffffu, acc[2 * f], 1);       // odd (im) row's values
                const float oI = __shfl_down_sync(0xffffffffu, acc[2 * f + 1], 1);
                if (!(lane & 1) && u < d.nu_pad)
                    d.Xh[(long long)f * d.x_fstride + (long long)kap * d.nu_pad + u] =
                        make_float2(acc[2 * f] + oI, acc[2 * f + 1] - oR);
            }
#pragma unroll
            for (int i = 0; i < 2 * F; ++i) acc[i] = 0.0f;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 2 * NSET <= 256 ? 256 : 512);
}

typedef CUresult (*MtEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t mac_tc_encode(MacTcArgs* d, const float2* M) {
    static MtEncodeFn enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
        if (e != cudaSuccess || !enc || q != cudaDriverEntryPointSuccess) {
            enc = nullptr;
            return e != cudaSuccess ? e : cudaErrorSymbolNotFound;
        }
    }
    // M as real floats [kappa][N2][2 * nu_pad]; box {32 floats, 128 rows, 1}; rows >= N2 are zero fill
    cuuint64_t dims[3] = {(cuuint64_t)2 * d->nu_pad, (cuuint64_t)d->N2, (cuuint64_t)d->nkappa};
    cuuint64_t strides[2] = {(cuuint64_t)d->nu_pad * 8, (cuuint64_t)d->N2 * d->nu_pad * 8};
    cuuint32_t box[3] = {(cuuint32_t)kMtKC, (cuuint32_t)kMtM, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&d->tmapM, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(M), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// G tiles: the frames' spectra [F][kappa][nu_pad] complex viewed as real floats with rows of gsplit floats
// (a divisor of 2 * nu_pad * nkappa so that a chunk never straddles two rows): dims {gsplit, rows, F}
cudaError_t mac_tc_encode_g(MacTcArgs* d, const float2* G, long long g_fstride, int F) {
    MtEncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    if (e != cudaSuccess || !enc || q != cudaDriverEntryPointSuccess) return e != cudaSuccess ? e : cudaErrorSymbolNotFound;
    const long long per_frame = 2LL * d->nu_pad * d->nkappa;   // floats
    d->gsplit = 2 * d->nu_pad;                                   // one kappa per row: chunks stay inside a row
    cuuint64_t dims[3] = {(cuuint64_t)d->gsplit, (cuuint64_t)(per_frame / d->gsplit), (cuuint64_t)F};
    cuuint64_t strides[2] = {(cuuint64_t)d->gsplit * 4, (cuuint64_t)g_fstride * 8};
    cuuint32_t box[3] = {(cuuint32_t)kMtKC, 1, (cuuint32_t)F}, es[3] = {1, 1, 1};
    CUresult r = enc(&d->tmapG, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(G), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int F, int PG, int NPREP>
static cudaError_t launch_fmb(const MacTcArgs& d, int grid, size_t smem, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(fmb_tc_kernel<F, PG, NPREP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fmb_tc_kernel<F, PG, NPREP><<<grid, mt_threads(NPREP), smem, s>>>(d);
    return cudaGetLastError();
}
template <int F>
static cudaError_t launch_fmb_cfg(const MacTcArgs& d, int grid, size_t smem, cudaStream_t s) {
    const int np = mac_tc_prep_warps(), pg = mac_tc_prep_groups();
    if (np == 16) return launch_fmb<F, 4, 16>(d, grid, smem, s);
    return pg == 2 ? launch_fmb<F, 2, 8>(d, grid, smem, s) : launch_fmb<F, 4, 8>(d, grid, smem, s);
}

cudaError_t launch_fwd_mac_batch_tc(const MacTcArgs& d, int F, int num_sms, cudaStream_t s) {
    const size_t smem = mac_tc_smem_bytes(F);
    const int grid = std::max(1, std::min(2 * d.nkappa, num_sms));
    switch (F) {
        case 8: return launch_fmb_cfg<8>(d, grid, smem, s);
        case 16: return launch_fmb_cfg<16>(d, grid, smem, s);
        case 32: return launch_fmb_cfg<32>(d, grid, smem, s);
        default: return cudaErrorInvalidValue;
    }
}

// A: M as real floats {2 nu_pad (u'), N2 (b'), kappa}, box {32, 32, 1}, SWIZZLE_128B_ATOM_32B (the MN-major tf32
// layout)
cudaError_t bmac_tc_encode(BmacTcArgs* d, const float2* M) {
    MtEncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    if (e != cudaSuccess || !enc || q != cudaDriverEntryPointSuccess) return e != cudaSuccess ? e : cudaErrorSymbolNotFound;
    cuuint64_t dims[3] = {(cuuint64_t)2 * d->nu_pad, (cuuint64_t)d->N2, (cuuint64_t)d->nkappa};
    cuuint64_t strides[2] = {(cuuint64_t)d->nu_pad * 8, (cuuint64_t)d->N2 * d->nu_pad * 8};
    cuuint32_t box[3] = {32, (cuuint32_t)kBmKC, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&d->tmapA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(M), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int F, int PG, int NPREP>
static cudaError_t launch_bmb(const BmacTcArgs& d, int grid, size_t smem, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(bmb_tc_kernel<F, PG, NPREP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    bmb_tc_kernel<F, PG, NPREP><<<grid, mt_threads(NPREP), smem, s>>>(d);
    return cudaGetLastError();
}
template <int F>
static cudaError_t launch_bmb_cfg(const BmacTcArgs& d, int grid, size_t smem, cudaStream_t s) {
    const int np = mac_tc_prep_warps(), pg = mac_tc_prep_groups();
    if (np == 16) return launch_bmb<F, 4, 16>(d, grid, smem, s);
    return pg == 2 ? launch_bmb<F, 2, 8>(d, grid, smem, s) : launch_bmb<F, 4, 8>(d, grid, smem, s);
}

cudaError_t launch_bwd_mac_batch_tc(const BmacTcArgs& d, int F, int num_sms, cudaStream_t s) {
    const size_t smem = bmac_tc_smem_bytes(F);
    const int nitems = d.nkappa * ((2 * d.nu_pad + kMtM - 1) / kMtM);
    const int grid = std::max(1, std::min(nitems, num_sms));
    switch (F) {
        case 8: return launch_bmb_cfg<8>(d, grid, smem, s);
        case 16: return launch_bmb_cfg<16>(d, grid, smem, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lfm
