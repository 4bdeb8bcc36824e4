/*
 * lfm.h -- C ABI of the B200-native light-field Richardson-Lucy hot path (AutoDeconJ, arXiv 2208.11422).
 *
 * Citations: "P:n" = the paper (PAPER.md line n); "S:n" = SPEC.md line n (interfaces only);
 * "C1..C18" = the readings of silent / garbled passages listed in DESIGN.md §3.
 *
 * One iteration of the hot path (§1 "3D Richardson-Lucy (RL) deconvolution"; §2.2):
 *     yhat = H x                      forward projection
 *     r    = y / (max(yhat,0) + eps)  ratio image            (C3)
 *     bp   = H^T r                    backward projection (exact adjoint, C6)
 *     x    = x * bp / max(H^T 1, eps) multiplicative non-negative update (C1)
 *     m    = max_z x                  z max-projection
 *     E    = DCT entropy of m         Eqs. (1)-(12)
 *     stop when E shows a decreasing trend, return argmax-E iterate (Fig. 2d; C14-C15)
 * with  H x (s,t) = sum_z sum_{p,q} x(z,p,q) * psf[z][p mod N][q mod N](s-p+ch, t-q+cw),
 *       ch = (kh-1)/2, cw = (kw-1)/2, zero outside kernel and image ("same" size; C4, C5).
 *
 * Conventions for every entry point
 *   - Arrays are row-major fp32 unless stated.  Volumes are [nz][H][W]; images [H][W];
 *     the PSF bank is [nz][N][N][kh][kw] (page (z*N + a)*N + b holds the kernel of input phase
 *     (a,b) = (p mod N, q mod N) of plane z).
 *   - "device" pointers must be CUDA device memory of the plan's device; "host" pointers are
 *     ordinary (preferably pinned) host memory.  `stream` is a cudaStream_t (NULL = legacy default
 *     stream); device work is ordered on it.  Calls that return host values synchronise `stream`.
 *   - The caller owns every buffer it passes; the library never retains a caller pointer past
 *     the call.  The plan owns its transfer matrices, workspaces and communicator.
 *   - No call aborts or throws across the ABI.  Every call returns an lfm_status; on failure
 *     lfm_last_error() (thread-local) names the argument / term that was violated and nothing
 *     has been written to the caller's outputs unless stated.
 *   - Multi-GPU (depth / phase sharding, §2.1 "divide the 3D layers ... evenly among
 *     different GPUs"): one process per GPU.  The nz*N*N "units" u = z*N*N + a*N + b (plane z,
 *     input phase (a,b)) are split into contiguous ranges, the first (nu mod world) ranks owning
 *     one extra unit.  Volumes at the boundary are always the FULL [nz][H][W] on every rank; a rank
 *     reads / writes only the voxels of its own units unless stated.
 */
#ifndef LFM_H_
#define LFM_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lfm_plan_s* lfm_plan;

typedef enum {
    LFM_OK = 0,
    LFM_EINVAL = 1,   /* invalid argument / policy / NULL pointer                         */
    LFM_EDIM = 2,     /* H or W not divisible by N, even kernel or even N, size mismatch */
    LFM_ENEG = 3,     /* negative PSF entry or negative measurement                */
    LFM_EZERO = 4,    /* all-zero measurement, an all-zero PSF plane or a PSF whose
                         normalizer H^T 1 sums to 0 on this image (it projects nothing)              */
    LFM_ENOMEM = 5,   /* device memory budget exceeded; lfm_last_error names the limiting term */
    LFM_ECUDA = 6,    /* CUDA runtime error                                                        */
    LFM_ENCCL = 7,    /* NCCL error: any rank failure fails the whole run                  */
    LFM_EUNSUPPORTED = 8 /* valid request this build does not implement (message says which)     */
} lfm_status;

/* Optics for the metric's cutoff region, Eqs. (7) and (11).  All fields > 0, na <= 1.6. */
typedef struct {
    double wavelength_um;   /* lambda, emission wavelength                    */
    double na;              /* numerical aperture of the objective            */
    double mla_pitch_um;    /* d_ML, microlens pitch                          */
    double magnification;   /* Q, objective magnification                     */
} lfm_optics;

enum { LFM_MODE_FIXED = 0, LFM_MODE_AUTO = 1 };
enum { LFM_REGION_TRIANGLE = 0, LFM_REGION_RECTANGLE = 1 };     /* C11 */
enum { LFM_UPDATE_RL = 0, LFM_UPDATE_ISRA = 1 };                /* C1  */

/* Iteration / stopping policy ("stop iteration when the DCT entropy value shows a decreasing
 * trend"; reading C15).  Defaults: lfm_policy_default(). */
typedef struct {
    int mode;         /* LFM_MODE_FIXED: run n_iters; LFM_MODE_AUTO: stop at the first k >= min_iters
                         after `patience` consecutive strict decreases of E, or at max_iters      */
    int n_iters;      /* fixed mode iteration count (>= 1)                                         */
    int max_iters;    /* auto mode cap (default 50, Fig. 2d sweeps 1..50)                  */
    int min_iters;    /* default 2                                                                 */
    int patience;     /* default 1                                                                 */
    float eps;        /* division guard, default 1e-6 (C3)                                         */
    int region;       /* LFM_REGION_TRIANGLE (default) or LFM_REGION_RECTANGLE (C11)               */
    int init_from_x;  /* 0: x0 = c0 = sum(y) / sum(H^T 1) uniform (C2); 1: caller's x is x0 (resume) */
    int update;       /* LFM_UPDATE_RL (default) or LFM_UPDATE_ISRA (MATLAB-lineage x * H^T y / H^T H x, x0 = H^T y unless
                         init_from_x; reading C1)                                          */
} lfm_policy;

/* Distribution.  world == 1: single GPU, no communicator.  world > 1: nccl_id is the 128-byte
 * ncclUniqueId produced by lfm_comm_unique_id() on rank 0 and broadcast by the caller (e.g. with
 * torch.distributed); every rank passes the same id. */
typedef struct {
    int rank;
    int world;
    unsigned char nccl_id[128];
} lfm_dist;

/* lfm_plan_create flags */
enum {
    LFM_PLAN_NO_COMM = 1,   /* world > 1 without a communicator: the plan owns rank's units and all
                               cross-rank reductions are skipped (outputs are this rank's partials).
                               For testing the sharding on one device.                              */
    LFM_PLAN_DIRECT = 2,    /* every plane on the spatial (direct polyphase convolution) path, on the
                               CUDA-core kernels (with LFM_PLAN_TC_DIRECT: on the tensor-core kernel) */
    LFM_PLAN_FFT_ONLY = 4,  /* every plane on the frequency path.  Default (neither flag): hybrid --
                               per plane, the cheapest of frequency / CUDA-core direct / tensor-core
                               direct by the cost model of DESIGN.md §5                               */
    LFM_PLAN_TC_DIRECT = 16,/* with LFM_PLAN_DIRECT: every plane on the tcgen05 kernel                */
    LFM_PLAN_GRAPHS = 32,   /* lfm_rl_iterate replays each iteration as one captured CUDA graph (needs a
                               non-default stream; not combined with lfm_profile timing)             */
    LFM_PLAN_NO_TC = 64,    /* hybrid without the tensor-core direct kernel                          */
    LFM_PLAN_FORCE_COMM = 512, /* create the NCCL communicator even for world = 1 (dist->nccl_id required):
                               every collective of the sharded path runs, over one rank (testing)    */
    LFM_PLAN_EVEN_SHARDS = 256, /* world > 1: split the units evenly (lfm_shard_units) instead of by the
                               cost model (lfm_shard_units_balanced, the default)                     */
    LFM_PLAN_FRAMES = 2048, /* a plan for time-lapse frame batches (lfm_rl_iterate_batch, F = 8 / 16 / 32): every
                               plane on the frequency path, the transfer matrices stored split into scaled fp16
                               hi / lo rows plus a split transposed copy (twice the memory of M) so both batched
                               passes run as TMA -> tcgen05 kind::f16 pipelines.  The single-frame calls
                               (lfm_forward / _backward / _rl_step / _rl_iterate / lfm_deconvolve_host) return
                               LFM_EUNSUPPORTED on such a plan.  Excludes DIRECT, GRAPHS, DEVICE_LOOP.       */
    LFM_PLAN_SYMMETRIC = 1024, /* with a communicator: the forward's partial images live in an NCCL symmetric
                               window and C1 (their sum over ranks) is our own kernel -- NVLS
                               multimem.ld_reduce where the NVLink switch supports it, else rank-ordered
                               peer loads -- instead of ncclAllReduce                 */
    LFM_PLAN_TILES = 4096,  /* the frequency path on overlap-save tiles of the coarse grid: small
                               transforms whose transfer matrices serve every tile in one tcgen05 kind::f16 pass.
                               Default (neither TILES nor NO_TILES): chosen by the cost model when the tiles are
                               cheaper than whole-image transforms.  Not with FRAMES; on such a plan
                               lfm_rl_iterate_batch runs the frames one after the other.                       */
    LFM_PLAN_NO_TILES = 8192, /* never tile the frequency path                                               */
    LFM_PLAN_DEVICE_LOOP = 128 /* lfm_rl_iterate runs the whole loop as one CUDA graph: a conditional WHILE
                               node over two unrolled iterations, the stop rule and the argmax snapshot
                               evaluated on the device -- no host round trip per iteration (
                               needs a non-default stream; ms_host receives the per-iteration average) */
};

/* Information about a plan. */
typedef struct {
    int nnum, nz, kh, kw, height, width;
    int unit_begin, unit_end;       /* owned units [begin, end)                                   */
    int fft_h, fft_w;               /* coarse transform sizes Lh, Lw (0 in direct mode)           */
    int lc_min_h, lc_min_w;         /* alias-free minimum n + ceil(c/N)            */
    int n_kappa;                    /* Lh * (Lw/2 + 1) coarse frequencies kept                     */
    int units_padded;               /* row length of the transfer matrices (>= owned units)       */
    int x_s, y_s;                   /* cutoff region (Eqs. 9-10)                                   */
    int direct;                     /* 1 if no owned unit is on the frequency path                 */
    size_t transfer_bytes;          /* bytes of transfer matrices + direct taps held by this rank  */
    size_t device_bytes;            /* all device memory held by the plan                         */
    double plan_ms;                 /* wall time of lfm_plan_create                                */
    int direct_planes;              /* planes (touching owned units) on the direct path            */
    int fft_units;                  /* owned units on the frequency path                            */
    int tc_planes;                  /* direct planes on the tcgen05 (3-product fp16 split) kernels  */
    double tc_flops_executed;       /* per projection: tensor flops the tcgen05 kernel issues (3 kind::f16
                                       products, union tap boxes, column ranges, padded pixel rows)   */
    double tc_flops_algorithmic;    /* per projection: 2 * exact taps (D x D per phase pair) * pixels */
    int planes_moved_for_memory;    /* planes the hybrid planner moved off the frequency path so that the
                                       transfer matrices fit the device (memory-aware planning, §5.1)  */
    int partition_sms[2][2];        /* SM partitions of the [forward, backward] projection:
                                       [tensor-core SMs, frequency-path SMs]; 0 = run one after the other */
    int c1_mode;                    /* the forward's sum over ranks: 0 ncclAllReduce (or none, one rank without
                                       a communicator), 1 own kernel over symmetric memory with peer loads,
                                       2 the same with NVLS multimem.ld_reduce (LFM_PLAN_SYMMETRIC, §7)       */
    int tc_moved_to_fft;            /* tensor-core planes the partition-aware step moved to the frequency path */
    int tiles;                      /* overlap-save tiles of the frequency path (0: whole-image transforms); the
                                       transforms are then fft_h x fft_w windows serving tile_T1 x tile_T2 outputs
                                       (of the first tile group when several coarse-tap ranges have their own)      */
    int tile_T1, tile_T2;
    int tile_groups;                /* tile groups (one window geometry per coarse-tap range of the planes)        */
    double fft_bytes;               /* per projection: algorithmic bytes of the frequency-path MAC(s) -- transfer
                                       matrices of the owned frequency-path units + the spectra they read / write */
} lfm_info;

/* Default policy: auto, max 50, min 2, patience 1, eps 1e-6, triangle, uniform init, RL. */
lfm_policy lfm_policy_default(void);

/* Thread-local description of the last failure (empty string if none). */
const char* lfm_last_error(void);

/* Version string of the library (build identifier). */
const char* lfm_version(void);

/* Writes a fresh ncclUniqueId (128 bytes) into id_out (host).  Call on rank 0 only. */
lfm_status lfm_comm_unique_id(unsigned char* id_out);

/* Host-only: the SM partition the planner picks for one projection direction when its
 * tensor-core planes take t_tc_ms on the whole GPU and its frequency-path planes stream mac_bytes of transfer
 * matrices.  direction 0 forward, 1 backward; mac_rate_scale (0 < s <= 1) scales the MAC's per-SM rate (resident
 * CTAs per SM).  *tc_sms = tensor-core SMs (0: the two halves run one after the other on the whole GPU);
 * *predicted_ms (nullable) = the model's time of the projection's two halves.  The developer overrides
 * LFM_TC_SMS_F / LFM_TC_SMS_B are not consulted here.  LFM_EINVAL for negative inputs or num_sms < 32. */
lfm_status lfm_partition_model(double t_tc_ms, double mac_bytes, int direction, int num_sms, double mac_rate_scale,
                               int* tc_sms, double* predicted_ms);

/* Host-only: the overlap-save tiling the planner picks for frequency-path planes of an nnum-phase
 * height x width image whose coarse taps lie in [d1a, d1b] x [d2a, d2b] (flags: LFM_PLAN_NO_TILES etc. as for
 * lfm_plan_create).  *L = window size (0: no tiling possible: fewer than 2 or more than 32 tiles for every compiled
 * window size), *T1 x *T2 = valid outputs per window, *ntile = tiles; *cost_unit (nullable) = the cost model's
 * seconds per frequency-path unit and iteration (both projections) on these tiles, *cost_whole (nullable) = the
 * same on whole-image transforms of the alias-free size for a kernel of side kh = kw = nnum * (2 max(|d|) + 1).
 * LFM_EINVAL for nnum < 1, image sides not multiples of nnum, or d1a > d1b / d2a > d2b. */
lfm_status lfm_tile_model(int nnum, int height, int width, int d1a, int d1b, int d2a, int d2b, int flags, int* L,
                          int* T1, int* T2, int* ntile, double* cost_unit, double* cost_whole);

/* Host-only: the contiguous unit range [*unit_begin, *unit_end) that `rank` of `world` owns among the
 * nz*N*N units (z-major u = z*N*N + a*N + b); the first (nu mod world) ranks own one extra unit
 * (S:334's even split, refined from planes to (z,a) units). */
lfm_status lfm_shard_units(int nz, int nnum, int world, int rank, int* unit_begin, int* unit_end);

/* Host-only: the cost-balanced contiguous unit range of `rank` -- the ownership lfm_plan_create uses
 * for world > 1 unless LFM_PLAN_EVEN_SHARDS.  From the FULL PSF (host, [nz][N][N][kh][kw]) every plane's path and
 * per-iteration time are estimated with the hybrid cost model; frequency-path and CUDA-core
 * planes may be cut between any two units, tensor-core planes only at plane borders (their cost does not shrink
 * with the owned fraction).  Cuts are placed at the cost quantiles k/world.  `flags` as for lfm_plan_create
 * (LFM_PLAN_EVEN_SHARDS returns the even split).  *est_seconds (nullable) receives the estimated per-iteration
 * time of the returned range.  Deterministic: every rank computes the same partition. */
lfm_status lfm_shard_units_balanced(const float* psf_host, int nnum, int nz, int kh, int kw, int height, int width,
                                    int world, int rank, int flags, int* unit_begin, int* unit_end, double* est_seconds);

/* Memory estimate before allocation (Fig. 1 "estimate the required memory size").
 * Writes the bytes one rank needs into *bytes_per_gpu (host).  If budget_bytes > 0 and the estimate
 * exceeds it, returns LFM_ENOMEM and writes the name of the largest term into limiting_term
 * (host, len bytes, NUL-terminated). */
lfm_status lfm_plan_estimate(int nnum, int nz, int kh, int kw, int height, int width, int world, int flags,
                             size_t budget_bytes, size_t* bytes_per_gpu, char* limiting_term, size_t len);

/* Create a plan (one-time; "the PSF is evenly distributed to each card ... used directly for
 * the next reconstruction").
 *   psf_host   : host [nz][N][N][kh][kw] fp32, >= 0 (LFM_ENEG otherwise).  Only this rank's units are
 *                copied to the device.  Not retained.
 *   psf_t_host : NULL -> backward = exact adjoint of psf (C6).  Else host [nz][N][N][kh][kw] >= 0, the MATLAB
 *                lineage "Ht": backward(r)(z,p,q) = sum_{s,t} r(s,t) Ht[z][p%N][q%N](p-s+ch, q-t+cw), which
 *                equals the exact adjoint when Ht = rot180(psf) per kernel.  Not retained; costs a
 *                second set of transfer matrices / direct taps.
 *   nnum       : N, odd >= 1.  height, width divisible by N.  kh, kw odd.
 *   optics     : for the metric region (may be NULL: lfm_quality / auto mode then return LFM_EINVAL).
 *   dist       : NULL means single GPU.
 * Builds the coarse transfer matrices (frequency mode), the normalizer H^T 1 and the region. */
lfm_status lfm_plan_create(lfm_plan* out, const float* psf_host, const float* psf_t_host,
                           int nnum, int nz, int kh, int kw, int height, int width,
                           const lfm_optics* optics, const lfm_dist* dist, int flags, void* stream);

lfm_status lfm_plan_info(lfm_plan plan, lfm_info* info /* host */);

/* Process-wide cap on the device memory later lfm_plan_create calls may plan for (bytes; 0 = the device's free
 * memory, the default).  The hybrid planner keeps the frequency-path transfer matrices under it by moving planes
 * to the direct (tensor-core or CUDA-core) path; LFM_ENOMEM names the limiting term if that is not enough. */
lfm_status lfm_set_memory_limit(size_t bytes);

/* The units u = z*N*N + a1*N + a2 this plan's rank owns, [*unit_begin, *unit_end) (host ints).
 * Volumes at the boundary are the full [nz][H][W]; a rank reads / writes only its owned units' voxels. */
lfm_status lfm_plan_owned(lfm_plan plan, int* unit_begin, int* unit_end);

/* Destroys the plan and frees its device memory / communicator.  NULL is a no-op. */
void lfm_plan_destroy(lfm_plan plan);

/* Forward projection yhat = H x.
 *   x : device [nz][H][W] (only owned units read).   y : device [H][W] written; summed over ranks. */
lfm_status lfm_forward(lfm_plan plan, const float* x, float* y, void* stream);

/* Backward projection xhat = H^T y.
 *   y : device [H][W].   x : device [nz][H][W]; voxels of owned units written, others untouched. */
lfm_status lfm_backward(lfm_plan plan, const float* y, float* x, void* stream);

/* Normalizer H^T 1 into x (device [nz][H][W], owned units written). */
lfm_status lfm_normalizer(lfm_plan plan, float* x, void* stream);

/* One RL iteration without the stop rule: x_out = x_in * H^T(y/(max(H x_in,0)+eps)) / max(H^T 1, eps),
 * and, if entropy_host != NULL, the DCT entropy of max_z x_out (Eq. 12) into *entropy_host
 * (synchronises).  x_in, x_out: device [nz][H][W] (owned units; may alias).  y: device [H][W].
 * yhat_out: optional device [H][W] receiving H x_in (summed over ranks). */
lfm_status lfm_rl_step(lfm_plan plan, const float* y, const float* x_in, float* x_out, float eps,
                       int region, float* yhat_out, double* entropy_host, void* stream);

/* The RL loop with the DCT-entropy stop rule.
 *   y          : device [H][W], >= 0, not all zero.
 *   x          : device [nz][H][W].  In: x0 if policy->init_from_x.  Out: the argmax-E iterate on ALL
 *                voxels (gathered across ranks once at the end).
 *   best_iter, stop_iter : host outputs (1-based).
 *   series_host: host [max(n_iters, max_iters)] receiving E_1..E_stop.
 *   ms_host    : optional host [same] receiving per-iteration device milliseconds.
 * Auto mode reads one double per iteration to the host. */
lfm_status lfm_rl_iterate(lfm_plan plan, const float* y, float* x, const lfm_policy* policy,
                          int* best_iter, int* stop_iter, double* series_host, float* ms_host, void* stream);

/* Frame-batched lockstep RL for time-lapse data: F in {2,4,8,16} independent frames share every
 * pass over the transfer matrices (a (N^2 x units) x (units x F) complex GEMM per coarse frequency), each frame
 * with its own stop rule and argmax snapshot; frames that stop early are frozen.
 *   y : device [F][H][W];  x : device [F][nz][H][W] (in: x0 if policy->init_from_x; out: each frame's argmax iterate)
 *   best_iter, stop_iter : host [F];  series_host : host [F][max(n_iters, max_iters)];
 *   ms_host : optional host [max(...)] device ms per lockstep iteration.  RL update only. */
lfm_status lfm_rl_iterate_batch(lfm_plan plan, int frames, const float* y, float* x, const lfm_policy* policy,
                                int* best_iter, int* stop_iter, double* series_host, float* ms_host, void* stream);

/* End-to-end call with HOST buffers: copies y in (H2D), runs lfm_rl_iterate, copies the argmax-E
 * volume out (D2H).  y_host [H][W], x_host [nz][H][W] (in: x0 if init_from_x; out: x_best).
 * With a page-locked x_host on a single rank in auto mode, an improving iterate whose E gain over the previous one is
 * below 1 % (the curve flattening before the stop) is copied into x_host on a side stream while the next iteration
 * runs (skipped while a previous copy is still on the link), so the argmax is usually on the host when the loop stops
 * and the final copy is skipped; x_host may hold such an intermediate iterate during the call and holds x_best when
 * it returns.  Otherwise x_best is copied once after the loop.  (Developer switch LFM_HOST_MIRROR: every improving
 * iterate -- measured slower at c3: the copies take HBM bandwidth from the iteration.) */
lfm_status lfm_deconvolve_host(lfm_plan plan, const float* y_host, float* x_host, const lfm_policy* policy,
                               int* best_iter, int* stop_iter, double* series_host, float* ms_host, void* stream);

/* DCT entropy of max_z x (P:63 + Eq. 12).  x: device [nz][H][W]; max-projection reduced over ranks.
 * region: LFM_REGION_*.  *entropy: host. */
lfm_status lfm_quality(lfm_plan plan, const float* x, int region, double* entropy, void* stream);

/* Stand-alone DCT entropy of one image (Eq. 12 with Eqs. 1-11).  img: device [H][W] fp32.
 * nnum: N for Eqs. (7), (11).  Outputs (host): entropy, region sizes x_s, y_s. */
lfm_status lfm_dct_entropy(const float* img, int height, int width, int nnum, const lfm_optics* optics,
                           int region, double* entropy, int* x_s, int* y_s, void* stream);

/* ---- live per-stage timing (CUDA events on the plan's calls' stream) ----
 * Stages of one iteration: 0 r2c_x (a2), 1 fwd_mac (a3), 2 c2r_yhat (a4), 3 dir_fwd (direct planes, K9),
 * 4 allreduce_sum (C1), 5 r2c_ratio (a5), 6 bwd_mac (a6), 7 c2r_update (a7), 8 dir_bwd (direct planes + update),
 * 9 maxproj_allreduce (a7 z-max + C2), 10 metric (a8).
 * When enabled, lfm_rl_iterate records an event before each stage and after the last one and adds the
 * elapsed times after its per-iteration synchronisation.  `launches` counts this library's kernels. */
#define LFM_N_STAGES 11
typedef struct {
    double ms[LFM_N_STAGES];          /* summed device milliseconds per stage   */
    long long count[LFM_N_STAGES];    /* number of timed executions per stage   */
    long long launches;               /* kernels launched by the library so far */
    long long iterations;             /* RL iterations executed so far          */
    double kern_ms[4];                /* summed device ms of the dominant kernels, timed on the stream (or SM
                                         partition) that runs them: tcgen05 forward, forward MAC, tcgen05
                                         backward (+ its update), backward MAC                           */
    long long kern_count[4];
    long long d2h_bytes;              /* device -> host bytes of lfm_rl_iterate / lfm_deconvolve_host so far: the
                                         8-byte E_k reads, the argmax mirror copies and final volume copies      */
} lfm_profile_t;

/* enable != 0 turns per-stage event timing on.  Counters keep accumulating until read with reset. */
lfm_status lfm_profile(lfm_plan plan, int enable);
/* Copies the counters into *out (host); reset != 0 zeroes them afterwards. */
lfm_status lfm_profile_read(lfm_plan plan, lfm_profile_t* out, int reset);
/* Name of stage i (static string), or NULL. */
const char* lfm_profile_stage_name(int i);

#ifdef __cplusplus
}
#endif
#endif /* LFM_H_ */
