// lfm_internal.cuh -- internal declarations of the B200 light-field RL path (not part of the ABI).
//
// Notation: N = Nnum, (nh, nw) = (H/N, W/N) lenslets, unit u = z*N*N + a1*N + a2
// (plane z, input phase a), output phase b' = b1*N + b2, coarse transform Lh x Lw, kappa = k1*nk2 + k2
// with nk2 = Lw/2 + 1 (Hermitian half plane).
#pragma once
#include <cuda.h>   // CUtensorMap (types only; the encoder is fetched through the runtime)
#include <cuda_runtime.h>
#include <nccl.h>
#include <cstddef>
#include <cstdint>
#include <vector>
#include "../../include/lfm.h"

namespace lfm {

constexpr int kMaxStages = 16;

struct FftDesc {
    int L;
    int nst;
    int radix[kMaxStages];
};

bool fft_factor(int L, FftDesc* d);         // radices 4,2,3,5; false if L is not 5-smooth
int next_smooth(int n);                     // smallest 5-smooth integer >= n

// ---- source / sink modes of the coarse transforms ----
enum R2CSrc : int {
    SRC_POLY = 0,     // polyphase volume [nu][nh][nw]            -> transform t = local unit
    SRC_IMAGE = 1,    // image-layout volume [nz][H][W]           -> transform t = local unit
    SRC_RATIO = 2,    // r = y / (max(yhat,0)+eps) on [H][W]       -> transform t = output phase b'
    SRC_ONES = 3,     // all-ones image                            -> transform t = output phase b'
    SRC_KERNEL = 4,   // PSF coarse kernels (plan)                 -> transform t = b'*nu + local unit
    SRC_IMAGE2D = 5   // plain image [H][W] (lfm_backward input)   -> transform t = output phase b'
};
enum C2RDst : int {
    DST_IMAGE = 0,    // yhat image [H][W] at (b1 + N i, b2 + N j); t = output phase
    DST_POLY = 1,     // polyphase volume; t = local unit
    DST_VOLIMAGE = 2, // image-layout volume [nz][H][W]; t = local unit
    DST_UPDATE = 3,   // RL:   x_new = x_old * max(bp,0) / max(norm,eps) (poly)
    DST_ISRA = 4      // ISRA: x_new = x_old * max(aux,0) / max(bp,eps), aux = H^T y, bp = H^T H x (poly)
};

// multiplicative update epilogues (aux = normalizer H^T 1 for RL, H^T y for ISRA)
template <int DST>
__device__ __forceinline__ float update_value(float xold, float aux, float bp, float eps) {
    if constexpr (DST == DST_ISRA)
        return xold * fmaxf(aux, 0.0f) / fmaxf(bp, eps);
    else
        return xold * fmaxf(bp, 0.0f) / fmaxf(aux, eps);
}

struct XformGeom {
    int N, H, W, nh, nw, nz;
    int Lh, Lw, nk2, nkappa;
    int unit0;              // first owned global unit
    int nu, nu_pad;         // transforms over units (FFT units of the plan) and their padded row length
    const int* umap;        // [nu] local unit index (u - unit0) of transform t; nullptr = identity
    int kh, kw, ch, cw;
};

struct R2CArgs {
    int src;
    const float* in;        // source array (see R2CSrc)
    const float* in2;       // yhat for SRC_RATIO
    float eps;
    int ntrans;             // number of transforms
    float2* out;            // out[kappa * out_ld + col(t)]
    long long out_ld;
    int cdiv, cmul;         // col(t) = (t / cdiv) * cmul + t % cdiv
};

struct C2RArgs {
    int dst;
    const float2* in;       // in[kappa * in_ld + t]
    long long in_ld;
    int ntrans;
    float* out;             // see C2RDst
    const float* xold;      // DST_UPDATE
    const float* norm;      // DST_UPDATE: H^T 1; DST_ISRA: H^T y
    float eps;
    int cdiv;               // overlap-save tiles (launch_c2r_tile): transform t = tile * cdiv + item reads column
    long long cmul;         //   tile * cmul + item of in[kappa * in_ld + .]
    int nsum;               //   summed over nsum partial inputs in_sstride apart (split-K MAC outputs; 0 / 1: one)
    long long in_sstride;
    int accum;              //   DST_IMAGE: add onto out instead of writing it (tile groups after the first)
};

// overlap-save tiles of the coarse grid: a square transform of L points per axis serves T1 x T2
// output coarse pixels; the coarse taps of every (phase pair, plane) lie in [dmin1, dmax1] x [dmin2, dmax2], so
// L >= T + dmax - dmin.  Forward windows start at tile * T - dmax (valid outputs at dmax ..), backward windows at
// tile * T + dmin (valid outputs at -dmin ..).
struct TileGeom {
    int L;
    int T1, T2, nty, ntx, ntile;
    int dmin1, dmax1, dmin2, dmax2;
};

// hybrid-plan direct part (kernels_direct.cu)
constexpr int kDirMaxD = 5;   // largest per-pair tap box handled by the register-blocked direct kernels
struct DirArgs {
    int N, H, W, nh, nw;
    int unit0, nu;            // owned units
    int nzd;                  // number of direct planes
    const int* zlist;         // [nzd] global plane index
    int D;                    // taps per dimension (box), coefficients zero-padded to D x D
    int dmin1, dmax1, dmin2, dmax2;   // range of the box origins dlo over all pairs and direct planes
    const float* coef_f;      // [nzd][a][D*D][b'] (forward: output phase fastest)
    const float* coef_b;      // [nzd][b'][D*D][a] (backward: input phase fastest)
    const int* dlo;           // [nzd][2][N][N]: dlo1[a1][b1], dlo2[a2][b2]
};
// tensor-core direct part (kernels_tcdir.cu).  One direction over ALL tensor-core planes of the
// plan (one launch).  Source offsets e = -d (forward: X_a[m' - d]) or e = +d (backward: r_b'[m + d]); the source
// is staged per iteration on a padded coarse grid shared by all planes (row pitch Wp >= nw + T2 - 1 for every
// plane, column c holds m2 = c + e2lo) so that a tap is a plain row offset of a TMA box.
struct TcPlane {
    int T1, T2, e1min, e2min;   // union tap box of the plane (source offsets)
    int bexp;                   // coefficient scale 2^bexp of the plane's fp16 split (f16_scale_exp of its max tap)
    long long coef_off;         // first coefficient slab (Ntile x 64 fp16) of the plane
    int mask_off;               // rowmask[mask_off + t1]: bit c set if window (chunk c, tap row t1) has a nonzero tap
    int last_win;               // c * T1 + t1 of the last nonzero window
    int active_windows;         // number of nonzero windows
    int ngroups;                // TMEM drain groups per (plane, tile) item (the issuer's stage walk, host-counted)
};
struct TcDirArgs {
    int N, H, W, nh, nw;
    int unit0, nu;            // owned units
    int nzd;                  // tensor-core planes
    const int* zlist;         // [nzd] global plane index (device)
    const TcPlane* planes;    // [nzd] (device)
    const int* rowmask;       // nonzero (chunk, tap row) windows, see TcPlane (device)
    int N2, Ntile;            // phases and TMEM columns per accumulator (N2 rounded up to 16, <= 256)
    int nch, kst_last;        // reduction chunks of 64 phases (one 128-byte fp16 row); K-steps of 16 in the last
    int e2lo;                 // column origin of the staged grid (min e2min over planes)
    int Wp, Lp, tiles;        // padded grid: Lp = nh * Wp rows of 64 phases, pair tiles of 256 rows
    int grid;                 // persistent CTA pairs (launch 2 * grid CTAs, clusters of 2)
    const int* item_off;      // [grid + 1] pair b runs items[item_off[b] .. item_off[b+1])   (LPT schedule)
    const int* items;         // item = zi * tiles + tile
    const uint16_t* coef;     // fp16 slabs [plane][tap][chunk][hi | lo] of Ntile x 64 (row-major), scaled 2^bexp
    long long nslabs;         // coefficient slabs
    int exp;                  // timing experiments only (env LFM_TC_EXP): 1 skip drains, 2 skip reloads, 4 counters
    long long* dbg;           // exp & 4: per-CTA wait-cycle counters [grid*2][8]
    uint16_t* src;            // staged fp16 source, slabs of [Lp][64] (hi / lo, scaled 2^aexp): fwd ((zi*2+part)*nch
                              // + c), bwd (part*nch + c)
    unsigned* amax;           // device scalar: max of the source (float bits) -> aexp = f16_scale_exp(amax)
    float* part;              // polyphase [nzd][N2][nh][nw]: forward per-plane partials (tc_fwd_reduce_kernel sums
                              // and interleaves them), backward H^T r (update epilogues apply it afterwards)
    int chain_k;              // K-steps (x3 MMAs) accumulated in TMEM between round-to-nearest drains
    const int* trange;        // [tiles] MMA column range per coefficient tile: n0 | nn << 16 (tcdir_ranges; device)
    alignas(64) CUtensorMap tmap;   // 3-D fp16 {64, Lp, slabs} over src, box {64, Arows, 1}, SWIZZLE_128B
    alignas(64) CUtensorMap bmap;   // 3-D fp16 {64, Ntile, nslabs} over coef, box {64, Ntile/2, 1}, SWIZZLE_128B
    int Arows;                      // A window rows: 128 + max T2 - 1
};
// geometry of one direction from the per-plane tap boxes d in [d1min, d1max] x [d2min, d2max] (host arrays)
bool tcdir_geometry(TcDirArgs* d, int fwd, const int* d1min, const int* d1max, const int* d2min, const int* d2max,
                    std::vector<TcPlane>* planes, int num_sms);
// LPT schedule of the (plane, tile) items over d->grid CTAs (host arrays)
void tcdir_schedule(const TcDirArgs& d, const std::vector<TcPlane>& planes, std::vector<int>* item_off,
                    std::vector<int>* items);
size_t tcdir_smem_bytes(int Ntile, int Arows);
size_t tcdir_coef_elems(const TcDirArgs& d, const std::vector<TcPlane>& planes);   // fp16 elements
size_t tcdir_src_elems(const TcDirArgs& d, int fwd);                                 // fp16 elements
size_t tcdir_part_floats(const TcDirArgs& d, int fwd);
cudaError_t tcdir_encode(TcDirArgs* d, int fwd);
// per-tile MMA column ranges from the packed nonzero-row flags of tcdir_coef_kernel (host)
void tcdir_ranges(const TcDirArgs& d, const std::vector<int>& nzflags, std::vector<int>* ranges);
cudaError_t launch_tcdir_coef(const TcDirArgs& d, const TcPlane& pl, int zi, int z, const float* psf_dev, int kh,
                              int kw, int ch, int cw, int fwd, uint16_t* coef, int* nzflags, cudaStream_t s);
// per-plane maxima of the owned PSF slice (float bits into pmax[zi], zeroed by the caller) for the fp16 scales
cudaError_t launch_tc_plane_amax(const float* psf_dev, const int* zlist, int nzd, int N2, int kk, int unit0, int nu,
                                 unsigned* pmax, cudaStream_t s);
// from the per-(tap, chunk) nonzero flags of every plane: row masks, last windows, active counts (host)
void tcdir_window_masks(const TcDirArgs& d, std::vector<TcPlane>* planes, const std::vector<int>& nzflags,
                        std::vector<int>* rowmask);
// launch pieces: stage the source (hi/lo split), the tcgen05 kernel (+ the backward update), the forward plane reduction
enum { TC_PART_STAGE = 1, TC_PART_MAIN = 2, TC_PART_FINISH = 4, TC_PART_ALL = 7 };
cudaError_t launch_tcdir_fwd(const TcDirArgs& d, const float* x, int src_image, float* y, int accumulate,
                             cudaStream_t s, int parts = TC_PART_ALL);
cudaError_t launch_tcdir_bwd(const TcDirArgs& d, int src, const float* img, const float* img2, float eps, int dst,
                             float* out, const float* xold, const float* norm, cudaStream_t s, int parts = TC_PART_ALL);
cudaError_t launch_plane_reduce(const float* part, int nzd, size_t hw, float* y, int accumulate, cudaStream_t s);
cudaError_t launch_dir_fwd(const DirArgs& d, const float* x, int src_image, float* part, float* y, int accumulate,
                           cudaStream_t s);  // part: [nzd][H][W] scratch
cudaError_t launch_dir_bwd(const DirArgs& d, int src, const float* img, const float* img2, float eps, int dst, float* out,
                           const float* xold, const float* norm, cudaStream_t s);

// C1 / C2 over NCCL symmetric memory (kernels_sym.cu, LFM_PLAN_SYMMETRIC): each rank writes its partial image into
// sym_buffer(st, 0) and its partial max-projection into sym_buffer(st, 1); sym_reduce(st, 0 | 1, out) leaves the sum /
// max over ranks in `out` (NVLS multimem.ld_reduce or rank-ordered peer loads)
struct SymState;
lfm_status sym_create(ncclComm_t comm, size_t n, int want_multimem, SymState** out, char* err, size_t errlen);
float* sym_buffer(SymState* st, int slot);
int sym_multimem(const SymState* st);
cudaError_t sym_reduce(SymState* st, int op, void* out, cudaStream_t s);
void sym_destroy(SymState* st);

// device-resident auto-stop loop state (kernels_misc.cu, LFM_PLAN_DEVICE_LOOP)
struct LoopState {
    int k, dec, best_k, stop, improved;
    double prev, best_e;
};
cudaError_t launch_loop_reset(LoopState* st, cudaStream_t s);
cudaError_t launch_stop_rule(LoopState* st, const double* e_dev, double* series, const lfm_policy* pol, int cap,
                             cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_second, int has_second,
                             cudaStream_t s);
cudaError_t launch_cond_copy(const LoopState* st, const float* src, float* dst, size_t n, cudaStream_t s);

// launchers (kernels_fft.cu)
cudaError_t launch_r2c(const XformGeom& g, const FftDesc& fh, const FftDesc& fw, const float2* tw_h,
                       const float2* tw_w, const R2CArgs& a, cudaStream_t s);
cudaError_t launch_c2r(const XformGeom& g, const FftDesc& fh, const FftDesc& fw, const float2* tw_h,
                       const float2* tw_w, const C2RArgs& a, cudaStream_t s);
// (kernels_fft_fast.cu) compile-time-specialised square sizes; used by launch_r2c / launch_c2r when available
bool fast_fft_size(int Lh, int Lw);
cudaError_t launch_r2c_fast(const XformGeom& g, const float2* tw, const R2CArgs& a, cudaStream_t s);
cudaError_t launch_c2r_fast(const XformGeom& g, const float2* tw, const C2RArgs& a, cudaStream_t s);
// (kernels_fft_tile.cu) overlap-save tile transforms.  R2C: transform t = tile * a.cdiv + item (item = FFT unit or
// output phase as in the whole-image modes), window of the item's coarse image at the tile's origin (dir 0: forward
// source, dir 1: backward source), spectrum to out[kappa * out_ld + tile * cmul + item]; with amax != nullptr the sum
// of |window| of every transform is max-reduced into amax[tile] (float bits; the fp16 scale bound of the tile MACs).
// C2R: the tile's valid T1 x T2 outputs (dir 0: forward image, dir 1: backward volume) into the C2RDst destination.
bool tile_fft_size(int L);
cudaError_t tile_fft_init();   // twiddle table of the tile kernels (once per process, plan time)
cudaError_t launch_r2c_tile(const XformGeom& g, const TileGeom& tg, const float2* tw, const R2CArgs& a, int dir,
                            unsigned* amax, cudaStream_t s);
cudaError_t launch_c2r_tile(const XformGeom& g, const TileGeom& tg, const float2* tw, const C2RArgs& a, int dir,
                            cudaStream_t s);
void set_fast_fft_enabled(bool on);
// (kernels_mac.cu)
cudaError_t launch_fwd_mac(const float2* M, const float2* G, float2* Y, int nkappa, int N2, int nu_pad, int num_sms,
                           int partition, cudaStream_t s);   // partition: launch shape for an SM partition (§5.5)
cudaError_t launch_bwd_mac(const float2* M, const float2* R, float2* Xh, int nkappa, int N2, int nu_pad,
                           cudaStream_t s);
cudaError_t launch_fwd_mac_batch(const float2* M, const float2* G, long long g_fstride, float2* Y, long long y_fstride,
                                 int F, int nkappa, int N2, int nu_pad, cudaStream_t s);   // F in {2,4,8,16}
cudaError_t launch_bwd_mac_batch(const float2* M, const float2* R, long long r_fstride, float2* Xh, long long x_fstride,
                                 int F, int nkappa, int N2, int nu_pad, cudaStream_t s);
// (kernels_mac_tc.cu) frame-batched forward MAC on tcgen05 (3xTF32), F in {8, 16, 32}
struct MacTcArgs {
    int nkappa, N2, nu_pad;
    const float2* G;          // [F][kappa][nu_pad] complex, frame stride g_fstride
    long long g_fstride;
    float2* Y;                // [F][kappa][N2] complex, frame stride y_fstride
    long long y_fstride;
    alignas(64) CUtensorMap tmapM;   // M as real floats [kappa][N2][2 nu_pad], box {32, 128, 1}, SWIZZLE_128B
    long long gsplit;                // floats per row of the G map (2 nu_pad: one kappa per row)
    alignas(64) CUtensorMap tmapG;   // G as real floats {gsplit, kappa, F}, box {32, 1, F}, no swizzle
};
cudaError_t mac_tc_encode_g(MacTcArgs* d, const float2* G, long long g_fstride, int F);
size_t mac_tc_smem_bytes(int F);
cudaError_t mac_tc_encode(MacTcArgs* d, const float2* M);
cudaError_t launch_fwd_mac_batch_tc(const MacTcArgs& d, int F, int num_sms, cudaStream_t s);
// frame-batched backward MAC on tcgen05 (MN-major transfer matrices, kernels_mac_tc.cu)
struct BmacTcArgs {
    int nkappa, N2, nu_pad;
    float2* Xh;               // [F][kappa][nu_pad] complex, frame stride x_fstride
    long long x_fstride;
    const float2* R;          // [F][kappa][N2] complex, frame stride r_fstride
    long long r_fstride;
    alignas(64) CUtensorMap tmapA;   // M as floats {2 nu_pad, N2, kappa}, box {32, 32, 1}, SWIZZLE_128B_ATOM_32B
};
// frame-batched MACs of LFM_PLAN_FRAMES plans: transfer matrices pre-split into scaled fp16 hi / lo rows, kind::f16
// (kernels_mac_f16.cu).  fwd: A = M rows b', src = G; bwd: A = M^T rows u (row pitch bpitch), src = R (pitch bpitch)
struct MacF16Args {
    int nkappa, N2, nu_pad, bpitch;
    int aexp;                 // the transfer matrices' scale exponent
    int chain_k;              // K-steps accumulated in TMEM between drains
    int ksplit;               // K splits per (kappa, row tile) (0 / 1: none): split sp writes out + sp * out_sstride
    long long out_sstride;
    const int* bexp;          // [F] the frames' source scale exponents (device, per call)
    const unsigned* bmax;     // or (non-null): [F] bounds of the frames' |source| (float bits), exponents derived in-kernel
    int nframes;              // frames actually present (<= F; the rest read as zeros, no output for them)
    float2* out;              // fwd: Y [F][kappa][N2]; bwd: Xh [F][kappa][nu_pad]
    long long out_fstride, out_ld;
    const float2* src;        // the frames' fp32 source spectra [nframes][kappa][src_n] (frame stride src_fstride),
    long long src_fstride;    //   read by the F = 32 kernel's prep warps (L2) into the stacked B tiles
    int src_n;
    alignas(64) CUtensorMap tmapAh;   // A hi parts {2n fp16, rows, kappa}, box {64, 128, 1}, SWIZZLE_128B
    alignas(64) CUtensorMap tmapAl;   // A lo parts (same rows, + 4n bytes)
    alignas(64) CUtensorMap tmapS;    // F <= 16: the frames' fp32 source {2n floats, kappa, F}, box {64, 1, F}
};
cudaError_t mac_f16_prepare(float2* M, const float2* Mb, float2* MT, int nkappa, int N2, int nu_pad, int bpitch,
                            MacF16Args* fwd, MacF16Args* bwd, cudaStream_t s);
cudaError_t mac_f16_encode_src(MacF16Args* a, int fwd, const float2* src, long long src_fstride, int F, int nframes = 0);
cudaError_t launch_frame_scales(const float2* src, long long fstride, int n, int F, int* eb, cudaStream_t s);
cudaError_t launch_mac_f16(const MacF16Args& d, int fwd, int F, int num_sms, cudaStream_t s);
size_t mac_f16_smem_bytes(int F);
size_t bmac_tc_smem_bytes(int F);
cudaError_t bmac_tc_encode(BmacTcArgs* d, const float2* M);
cudaError_t launch_bwd_mac_batch_tc(const BmacTcArgs& d, int F, int num_sms, cudaStream_t s);
// (kernels_misc.cu)
cudaError_t launch_fill(float* p, size_t n, float v, cudaStream_t s);
cudaError_t launch_fill_dev(float* p, size_t n, const double* num, const double* den, cudaStream_t s);
cudaError_t launch_poly_to_image(const float* xp, float* x, const XformGeom& g, int unit_begin, int unit_count,
                                 cudaStream_t s);
cudaError_t launch_image_to_poly(const float* x, float* xp, const XformGeom& g, int unit_begin, int unit_count,
                                 cudaStream_t s);
cudaError_t launch_max_project(const float* x, unsigned* mproj, const XformGeom& g, cudaStream_t s);
cudaError_t launch_max_project_poly(const float* xp, unsigned* mproj, const XformGeom& g, cudaStream_t s);
struct FrameSel {
    int b[32];   // per frame of a batch: the triple-buffer slot holding its current iterate
};
cudaError_t launch_max_project_poly_batch(const float* base, size_t vol, const FrameSel& sel, int F, unsigned* mproj,
                                          const XformGeom& g, cudaStream_t s);
cudaError_t launch_metric_batch(const unsigned* mproj_bits, int F, int H, int W, int xs, int ys, const double* Cr,
                                const double* Cw, const int2* members, int nmem, double* T1, double* rowsq,
                                double* out, cudaStream_t s);
cudaError_t launch_sum_stats(const float* p, size_t n, double* partials, int nparts, double* out3, cudaStream_t s);
cudaError_t launch_metric(const unsigned* mproj_bits, int H, int W, int xs, int ys, const double* Cr,
                          const double* Cw, const int2* members, int nmem, double* T1, double* rowsq,
                          double* out, cudaStream_t s);
// direct spatial path (kernels_direct.cu)
cudaError_t launch_direct_fwd(const float* xp, const float* psf, float* yimg, const XformGeom& g, cudaStream_t s);
cudaError_t launch_direct_bwd(const float* rimg, const float* psf, float* out, int dst, const float* xold,
                              const float* norm, unsigned* mproj, float eps, const XformGeom& g, cudaStream_t s);
cudaError_t launch_ratio(const float* y, const float* yhat, float* r, size_t n, float eps, cudaStream_t s);
cudaError_t launch_image_phase_planes(const float* y, const float* yhat, float eps, float* out, int N, int H, int W,
                                      cudaStream_t s);

}  // namespace lfm
