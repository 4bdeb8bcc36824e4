// lfm_capi.cu -- the C ABI declared in include/lfm.h: plan (transfer matrices, normalizer, region),
// projections, the RL loop with the DCT-entropy stop rule, and depth/phase sharding over NCCL.
// See DESIGN.md §2 (path and boundary) and §5 (kernels).
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <vector>

#include "lfm_internal.cuh"
#include "tc_sm100.cuh"

using namespace lfm;

namespace {

thread_local char g_err[1024] = "";

lfm_status fail(lfm_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}

#define CK(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return fail(LFM_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

#define NK(call)                                                                                  \
    do {                                                                                          \
        ncclResult_t r_ = (call);                                                                 \
        if (r_ != ncclSuccess) return fail(LFM_ENCCL, "%s failed: %s", #call, ncclGetErrorString(r_)); \
    } while (0)

#define ST(call)                              \
    do {                                      \
        lfm_status s_ = (call);               \
        if (s_ != LFM_OK) return s_;          \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline size_t round_up(size_t a, size_t b) { return (a + b - 1) / b * b; }

struct Region {
    int xs = 0, ys = 0;
    std::vector<int2> tri, rect;
};

// Eqs. (7), (11), (9)-(10), (6): P_u = d_ML/(Q N), d_psf = 1.22 lambda N / NA,
// X_S = clamp(ceil(P_u W / d_psf), 1, W), Y_S likewise with H (reading C10); triangle u X_S + v Y_S < X_S Y_S
// with u the height index < Y_S and v the width index < X_S (reading C11).
lfm_status make_region(const lfm_optics* o, int nnum, int H, int W, Region* r) {
    if (!o) return fail(LFM_EINVAL, "optics is NULL: the metric region needs Eqs. (7)-(11) inputs");
    if (!(o->wavelength_um > 0) || !(o->na > 0) || !(o->mla_pitch_um > 0) || !(o->magnification > 0))
        return fail(LFM_EINVAL, "optics fields must be > 0 (S:25)");
    if (o->na > 1.6) return fail(LFM_EINVAL, "optics.na must be <= 1.6 (S:27)");
    if (H < 2 || W < 2) return fail(LFM_EDIM, "image must be at least 2x2 for the metric (S:60)");
    const double pu = o->mla_pitch_um / (o->magnification * nnum);
    const double dpsf = 1.22 * o->wavelength_um * nnum / o->na;
    long long xs = (long long)std::ceil(pu * W / dpsf), ys = (long long)std::ceil(pu * H / dpsf);
    if (xs < 1) xs = 1;
    if (xs > W) xs = W;
    if (ys < 1) ys = 1;
    if (ys > H) ys = H;
    r->xs = (int)xs;
    r->ys = (int)ys;
    r->tri.clear();
    r->rect.clear();
    for (int u = 0; u < ys; ++u)
        for (int v = 0; v < xs; ++v) {
            r->rect.push_back(make_int2(u, v));
            if ((long long)u * xs + (long long)v * ys < xs * ys) r->tri.push_back(make_int2(u, v));
        }
    return LFM_OK;
}

// orthonormal DCT-II basis rows, Eqs. (2)-(4): C[u][x] = c(u,Z) cos((2x+1) pi u / (2Z))
void dct_rows(int Z, int count, std::vector<double>* out) {
    out->resize((size_t)count * Z);
    const double pi = 3.14159265358979323846;
    for (int u = 0; u < count; ++u) {
        const double c = (u == 0) ? 1.0 / std::sqrt((double)Z) : std::sqrt(2.0 / Z);
        for (int x = 0; x < Z; ++x) (*out)[(size_t)u * Z + x] = c * std::cos((2.0 * x + 1.0) * pi * u / (2.0 * Z));
    }
}

struct MetricDev {
    int H = 0, W = 0, xs = 0, ys = 0;
    double *Cr = nullptr, *Cw = nullptr, *T1 = nullptr, *rowsq = nullptr, *out = nullptr;
    int2* mem[2] = {nullptr, nullptr};
    int nmem[2] = {0, 0};
};

void metric_free(MetricDev* m) {
    cudaFree(m->Cr);
    cudaFree(m->Cw);
    cudaFree(m->T1);
    cudaFree(m->rowsq);
    cudaFree(m->out);
    cudaFree(m->mem[0]);
    cudaFree(m->mem[1]);
    *m = MetricDev();
}

lfm_status metric_alloc(MetricDev* m, const Region& r, int H, int W, cudaStream_t s, size_t* bytes) {
    m->H = H;
    m->W = W;
    m->xs = r.xs;
    m->ys = r.ys;
    std::vector<double> cr, cw;
    dct_rows(H, r.ys, &cr);
    dct_rows(W, r.xs, &cw);
    CK(cudaMalloc(&m->Cr, cr.size() * sizeof(double)));
    CK(cudaMalloc(&m->Cw, cw.size() * sizeof(double)));
    // T1 = (m C_W^T) column-major [xs][H], followed by the per-member entropy terms of launch_metric
    CK(cudaMalloc(&m->T1, ((size_t)H * r.xs + std::max(r.tri.size(), r.rect.size())) * sizeof(double)));
    CK(cudaMalloc(&m->rowsq, (size_t)H * sizeof(double)));
    CK(cudaMalloc(&m->out, 8 * sizeof(double)));
    CK(cudaMalloc(&m->mem[0], r.tri.size() * sizeof(int2)));
    CK(cudaMalloc(&m->mem[1], r.rect.size() * sizeof(int2)));
    m->nmem[0] = (int)r.tri.size();
    m->nmem[1] = (int)r.rect.size();
    CK(cudaMemcpyAsync(m->Cr, cr.data(), cr.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(m->Cw, cw.data(), cw.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(m->mem[0], r.tri.data(), r.tri.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(m->mem[1], r.rect.data(), r.rect.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));   // host vectors die here
    if (bytes)
        *bytes += (cr.size() + cw.size() + (size_t)H * r.xs + H + 8) * sizeof(double) +
                  (r.tri.size() + r.rect.size()) * sizeof(int2);
    return LFM_OK;
}

struct SizeTerms {
    size_t transfer, spectra, volumes, images, staging, metric;
    size_t total() const { return transfer + spectra + volumes + images + staging + metric; }
};

void unit_range(int nu_total, int world, int rank, int* b, int* e) {
    const int base = nu_total / world, extra = nu_total % world;
    *b = rank * base + (rank < extra ? rank : extra);
    *e = *b + base + (rank < extra ? 1 : 0);
}

struct Geo {
    int N, nz, kh, kw, H, W, nh, nw, ch, cw;
    int lcmin_h, lcmin_w, Lh, Lw, nk2, nkappa;
};

lfm_status make_geo(int nnum, int nz, int kh, int kw, int H, int W, bool direct, Geo* g) {
    if (nnum < 1 || nnum % 2 == 0) return fail(LFM_EDIM, "nnum=%d must be odd and >= 1 (S:26)", nnum);
    if (nz < 1) return fail(LFM_EDIM, "nz=%d must be >= 1", nz);
    if (kh < 1 || kw < 1 || kh % 2 == 0 || kw % 2 == 0) return fail(LFM_EDIM, "kernel %dx%d must have odd sides (S:192)", kh, kw);
    if (H < 1 || W < 1 || H % nnum || W % nnum)
        return fail(LFM_EDIM, "image %dx%d must be divisible by nnum=%d (S:188)", H, W, nnum);
    g->N = nnum;
    g->nz = nz;
    g->kh = kh;
    g->kw = kw;
    g->H = H;
    g->W = W;
    g->nh = H / nnum;
    g->nw = W / nnum;
    g->ch = (kh - 1) / 2;
    g->cw = (kw - 1) / 2;
    // alias-free coarse transform size n + ceil(c / N), rounded up to a 5-smooth length
    g->lcmin_h = g->nh + (g->ch + nnum - 1) / nnum;
    g->lcmin_w = g->nw + (g->cw + nnum - 1) / nnum;
    if (direct) {
        g->Lh = g->Lw = g->nk2 = g->nkappa = 0;
    } else {
        g->Lh = next_smooth(g->lcmin_h < 2 ? 2 : g->lcmin_h);
        g->Lw = next_smooth(g->lcmin_w < 2 ? 2 : g->lcmin_w);
        g->nk2 = g->Lw / 2 + 1;
        g->nkappa = g->Lh * g->nk2;
    }
    return LFM_OK;
}

SizeTerms size_terms(const Geo& g, int nu, int nu_total, int world, bool direct) {
    SizeTerms t{};
    const size_t N2 = (size_t)g.N * g.N;
    const size_t nu_pad = round_up((size_t)nu, 16);
    const size_t vol = (size_t)nu * g.nh * g.nw * sizeof(float);
    if (direct) {
        t.transfer = (size_t)nu * g.kh * g.kw * sizeof(float);
        t.spectra = 0;
        t.staging = 0;
    } else {
        t.transfer = (size_t)g.nkappa * N2 * nu_pad * sizeof(float2);
        t.spectra = 2 * (size_t)g.nkappa * nu_pad * sizeof(float2) + 2 * (size_t)g.nkappa * N2 * sizeof(float2);
        t.staging = (size_t)nu * g.kh * g.kw * sizeof(float);
    }
    t.volumes = 4 * vol + (world > 1 ? (size_t)nu_total * g.nh * g.nw * sizeof(float) : 0);
    t.images = 3 * (size_t)g.H * g.W * sizeof(float);
    t.metric = (size_t)g.H * 64 * sizeof(double) * 2 + (1 << 20);
    return t;
}

}  // namespace

struct lfm_plan_s {
    Geo geo{};
    XformGeom xg{};     // frequency-path transforms (nu = FFT units, umap)
    XformGeom xall{};   // every owned unit (layout conversion, max-projection, generic direct path)
    FftDesc fh{}, fw{};
    int rank = 0, world = 1;
    std::vector<int> rcut;   // rank r owns units [rcut[r], rcut[r+1])
    bool comm = false, direct = false;
    ncclComm_t nccl = nullptr;
    int u0 = 0, u1 = 0, nu = 0, nu_pad = 0, nu_total = 0;
    // hybrid plan: FFT units (frequency path) and direct planes (spatial path)
    int nu_fft = 0, nu_fft_pad = 16;
    int* umap = nullptr;        // [nu_fft] local unit index of FFT transform t
    std::vector<DirArgs> dgroups;   // SIMT direct planes grouped by tap-box size D (one launch per group)
    std::vector<TcDirArgs> tcf, tcb;   // tensor-core direct groups (forward / backward coefficient layouts)
    int n_tc_planes = 0;
    int mem_moved = 0;   // planes moved off the frequency path to fit the memory budget
    double tc_flops_exec = 0.0, tc_flops_alg = 0.0;   // per projection (lfm_info)
    double tc_active_frac = 0.0;                       // mean fraction of nonzero (chunk, tap row) windows
    int part_moved = 0;                                // tensor-core planes the partition-aware step moved to FFT
    SymState* sym = nullptr;                           // LFM_PLAN_SYMMETRIC: C1 over symmetric memory (kernels_sym.cu)
    // LFM_PLAN_FRAMES: transfer matrices split into fp16 hi / lo rows (M) plus a split transposed copy (MT, rows u of
    // bpitch complex) for the fp16 batched MACs (kernels_mac_f16.cu); the single-frame MACs are unavailable
    bool frames = false;
    float2* MT = nullptr;
    int bpitch = 0;
    MacF16Args mf_fwd{}, mf_bwd{};
    int* mf_eb = nullptr;                              // [2][32] per-frame source scale exponents (fwd, bwd)
    const void* mf_src[2] = {nullptr, nullptr};        // encoded source pointers / frame counts of mf_fwd / mf_bwd
    int mf_F[2] = {0, 0};
    // overlap-save tiled frequency path (LFM_PLAN_TILES): one group per coarse-tap range of the
    // frequency-path planes, each with transforms of tg.L points per axis over tg.ntile tiles; M (forward) and M^T
    // (backward) stored split as in FRAMES plans, both MACs on kind::f16 with the tiles as the GEMM's N
    // (kernels_mac_f16.cu, F >= ntile)
    struct TileGroup {
        TileGeom tg{};
        XformGeom xg{};            // the group's windows (L x L) and units (umap, nu, nu_pad)
        FftDesc fd{};
        float2* tw = nullptr;      // twiddles of L (warp kernels, M build)
        int* umap = nullptr;       // [nu] local unit index of the group's transform t
        float2 *M = nullptr, *MT = nullptr, *G = nullptr, *Xh = nullptr, *Y = nullptr, *R = nullptr;
        unsigned* tmax = nullptr;  // [2][32] per-tile |source| bounds (float bits) of the forward / backward MAC
        MacF16Args fwd{}, bwd{};
        int F = 0;
    };
    bool tiled = false;
    std::vector<TileGroup> tgs;
    double fft_alg_bytes = 0.0;   // per projection: algorithmic bytes of the frequency path's MAC (lfm_info)
    std::vector<void*> dallocs;     // device arrays owned by the direct groups
    int n_direct_planes = 0;
    float* dpart = nullptr;         // [max group planes][H][W] per-plane forward partials
    int num_sms = 148;
    float2 *tw_h = nullptr, *tw_w = nullptr;
    float2* M = nullptr;
    float* psf = nullptr;       // owned PSF slice (generic direct mode)
    float* psfb = nullptr;      // owned backward PSF slice = rot180(supplied Ht), or == psf (exact adjoint)
    float2* Mb = nullptr;       // backward transfer matrices (== M unless Ht is supplied)
    float* norm = nullptr;
    float* hty = nullptr;       // H^T y (ISRA), allocated on first use
    double* norm_sum = nullptr; // device scalar, summed over ranks
    float* xb[3] = {nullptr, nullptr, nullptr};
    float* xfull = nullptr;     // gather buffer (world > 1)
    float2 *G = nullptr, *Xh = nullptr, *Y = nullptr, *R = nullptr;
    float* yhat = nullptr;
    float* rimg = nullptr;
    unsigned* mproj = nullptr;
    double* partials = nullptr; // 3 * kParts
    double* stats = nullptr;    // 3
    double* host = nullptr;     // pinned 16 doubles (8, 9: the pipelined fixed loop's E_k slots)
    float *y_stage = nullptr, *x_stage = nullptr;   // lfm_deconvolve_host staging
    // lfm_deconvolve_host: every improving iterate is converted and copied to the host on a side stream while the
    // next iteration runs, so the call returns without a final 0.2-1.7 GB device-to-host copy
    cudaStream_t scopy = nullptr;
    cudaEvent_t evconv[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t evcopy = nullptr;   // end of the last mirror copy (a new one is skipped while it is in flight)
    // fixed-iteration host loop pipelined one iteration deep: the max-projection and the metric of iteration k run on
    // stream smet while iteration k + 1 runs on the caller's stream (rl_loop)
    cudaStream_t smet = nullptr;
    cudaEvent_t evupd[2] = {nullptr, nullptr}, evmet[2] = {nullptr, nullptr};
    // CUDA-graph replay of one iteration (LFM_PLAN_GRAPHS): one graph per (cur, next) buffer pair,
    // keyed also by the measurement pointer and the policy scalars baked into the captured launches
    bool graphs = false;
    struct GraphKey {
        int cur, nxt, region, update;
        const float* y;
        float eps;
    };
    std::vector<GraphKey> gkeys;
    std::vector<cudaGraphExec_t> gexec;
    // device-resident auto-stop loop (LFM_PLAN_DEVICE_LOOP): one graph = WHILE node over two unrolled
    // iterations (xb[0] -> xb[1] -> xb[0]), stop rule and argmax snapshot (into xb[2]) on the device
    bool dloop = false;
    struct LoopKey {
        const float* y;
        float eps;
        int region, update, mode, n_iters, min_iters, patience, max_iters;
    };
    std::vector<LoopKey> lkeys;
    std::vector<cudaGraphExec_t> lexec;
    LoopState* lstate = nullptr;
    double* lseries = nullptr;
    int lseries_cap = 0;
    // frame-batched forward MAC on tcgen05 (F >= 8), tensor map over M encoded on first use
    bool mac_tc_ready = false, mac_tc_off = false;
    int mac_tc_F = 0;
    MacTcArgs mac_tc{};
    // frame-batched backward MAC on tcgen05 (F = 8, 16), tensor maps re-encoded when the batch buffers change
    BmacTcArgs bmac_tc{};
    int bmac_F = 0;   // nonzero once the map is encoded
    // frame-batched lockstep buffers (lfm_rl_iterate_batch), capacity bcap frames
    int bcap = 0;
    float2 *bG = nullptr, *bXh = nullptr, *bY = nullptr, *bR = nullptr;
    float *bx = nullptr, *byhat = nullptr;
    unsigned* bmproj = nullptr;
    double *bent = nullptr, *bhost = nullptr;
    double *bmT1 = nullptr, *bmrs = nullptr;   // per-frame metric workspaces (launch_metric_batch)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // co-resident projections: the tensor-core direct kernel on a high-priority side stream, the
    // frequency-path MAC beside it on the caller's stream, one fork / join per projection
    struct Part {
        int sms_tc = 0, sms_mac = 0;                // SMs of the two sides
        CUgreenCtx gtc = nullptr, gmac = nullptr;   // green contexts over disjoint SM sets
        cudaStream_t stc = nullptr, smac = nullptr;
    };
    Part part[2];   // [forward, backward] projection; part[d].stc == nullptr: the two run one after the other
    cudaEvent_t evf = nullptr, evj = nullptr, evj2 = nullptr;
    cudaEvent_t kev[4][2] = {};   // kernel timers (lfm_profile_t.kern_ms)
    bool prof = false;
    cudaEvent_t pev[LFM_N_STAGES + 1] = {};
    lfm_profile_t pacc{};
    bool has_optics = false;
    lfm_optics optics{};
    Region region;
    MetricDev met;
    size_t transfer_bytes = 0, bytes = 0;
    double plan_ms = 0.0;
};

namespace {

constexpr int kParts = 296;
size_t g_mem_limit = 0;   // lfm_set_memory_limit (0: the device's free memory)

const char* kStageNames[LFM_N_STAGES] = {"r2c_x",      "fwd_mac",    "c2r_yhat", "dir_fwd",
                                         "allreduce_sum", "r2c_ratio", "bwd_mac", "c2r_update",
                                         "dir_bwd",    "maxproj_allreduce", "metric"};
enum { ST_R2C_X = 0, ST_FWD_MAC, ST_C2R_YHAT, ST_DIR_FWD, ST_ALLRED_SUM, ST_R2C_RATIO, ST_BWD_MAC, ST_C2R_UPD,
       ST_DIR_BWD, ST_MAXPROJ, ST_METRIC };

// records the start event of `stage` (stage == LFM_N_STAGES: end of the last stage) when profiling
inline lfm_status mark(lfm_plan p, int stage, cudaStream_t s) {
    if (!p->prof) return LFM_OK;
    CK(cudaEventRecord(p->pev[stage], s));
    return LFM_OK;
}

// ---- §5.5 SM partitions (green contexts; driver entry points fetched through the runtime, no -lcuda) ----
struct GreenApi {
    CUresult (*get_res)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
    CUresult (*split)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned) = nullptr;
    CUresult (*gen_desc)(CUdevResourceDesc*, CUdevResource*, unsigned) = nullptr;
    CUresult (*create)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
    CUresult (*destroy)(CUgreenCtx) = nullptr;
    CUresult (*stream)(CUstream*, CUgreenCtx, unsigned, int) = nullptr;
    bool ok = false;
};

const GreenApi& green_api() {
    static GreenApi a = [] {
        GreenApi g;
        cudaDriverEntryPointQueryResult q;
        auto get = [&](const char* n, void** f) {
            return cudaGetDriverEntryPoint(n, f, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess;
        };
        g.ok = get("cuDeviceGetDevResource", (void**)&g.get_res) && get("cuDevSmResourceSplitByCount", (void**)&g.split) &&
               get("cuDevResourceGenerateDesc", (void**)&g.gen_desc) && get("cuGreenCtxCreate", (void**)&g.create) &&
               get("cuGreenCtxDestroy", (void**)&g.destroy) && get("cuGreenCtxStreamCreate", (void**)&g.stream);
        return g;
    }();
    return a;
}

void green_free(lfm_plan p) {
    const GreenApi& g = green_api();
    for (auto& pt : p->part) {
        if (pt.stc) cudaStreamDestroy(pt.stc);
        if (pt.smac) cudaStreamDestroy(pt.smac);
        if (pt.gtc && g.ok) g.destroy(pt.gtc);
        if (pt.gmac && g.ok) g.destroy(pt.gmac);
        pt = lfm_plan_s::Part{};
    }
    for (cudaEvent_t* e : {&p->evf, &p->evj, &p->evj2}) {
        if (*e) cudaEventDestroy(*e);
        *e = nullptr;
    }
}

// split the device's SMs into a tensor-core side of >= want_tc SMs (rounded by the driver) and the rest for the
// frequency path; false (the projection then runs its two halves one after the other) if the driver cannot
bool green_split(lfm_plan p, int dev, int want_tc, lfm_plan_s::Part* out) {
    const GreenApi& g = green_api();
    if (!g.ok) return false;
    CUdevResource all{}, grp{}, rest{};
    if (g.get_res((CUdevice)dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return false;
    unsigned n = 1;
    if (g.split(&grp, &n, &all, &rest, 0, (unsigned)want_tc) != CUDA_SUCCESS || n != 1) return false;
    if (rest.sm.smCount < 8) return false;
    CUdevResourceDesc dt = nullptr, dm = nullptr;
    lfm_plan_s::Part pt;
    bool ok = g.gen_desc(&dt, &grp, 1) == CUDA_SUCCESS && g.gen_desc(&dm, &rest, 1) == CUDA_SUCCESS &&
              g.create(&pt.gtc, dt, (CUdevice)dev, CU_GREEN_CTX_DEFAULT_STREAM) == CUDA_SUCCESS &&
              g.create(&pt.gmac, dm, (CUdevice)dev, CU_GREEN_CTX_DEFAULT_STREAM) == CUDA_SUCCESS &&
              g.stream((CUstream*)&pt.stc, pt.gtc, CU_STREAM_NON_BLOCKING, 0) == CUDA_SUCCESS &&
              g.stream((CUstream*)&pt.smac, pt.gmac, CU_STREAM_NON_BLOCKING, 0) == CUDA_SUCCESS;
    for (cudaEvent_t* e : {&p->evf, &p->evj, &p->evj2})
        if (ok && !*e) ok = cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
        if (pt.stc) cudaStreamDestroy(pt.stc);
        if (pt.smac) cudaStreamDestroy(pt.smac);
        if (pt.gtc) g.destroy(pt.gtc);
        if (pt.gmac) g.destroy(pt.gmac);
        return false;
    }
    pt.sms_tc = (int)grp.sm.smCount;
    pt.sms_mac = (int)rest.sm.smCount;
    *out = pt;
    return true;
}

// kernel timer k (0 tc fwd, 1 mac fwd, 2 tc bwd, 3 mac bwd): start (e = 0) / end (e = 1) on stream s; a kernel
// that did not run this iteration (its plan has no such planes / units) leaves both events unrecorded
inline lfm_status kmark(lfm_plan p, int k, int e, cudaStream_t s) {
    if (!p->prof) return LFM_OK;
    CK(cudaEventRecord(p->kev[k][e], s));
    return LFM_OK;
}

// dev timing knob LFM_PART_SKIP (results are wrong with it set): 1 skips the tensor-core kernels, 2 the MACs, so that
// either half of a partitioned projection can be timed alone on its partition
int part_skip() {
    static const int v = getenv("LFM_PART_SKIP") ? atoi(getenv("LFM_PART_SKIP")) : 0;
    return v;
}

// dev A/B LFM_C2R_FULL: tiled plans run their C2R on the whole GPU after the join (default: inside the partition)
bool c2r_full() {
    static const bool v = getenv("LFM_C2R_FULL") != nullptr;
    return v;
}

// fork the caller's stream s onto the projection's two partition streams (*st tensor cores, *sm MAC)
lfm_status fork(lfm_plan p, const lfm_plan_s::Part& pt, cudaStream_t s, cudaStream_t* st, cudaStream_t* sm) {
    CK(cudaEventRecord(p->evf, s));
    CK(cudaStreamWaitEvent(pt.stc, p->evf, 0));
    CK(cudaStreamWaitEvent(pt.smac, p->evf, 0));
    *st = pt.stc;
    *sm = pt.smac;
    return LFM_OK;
}

// s waits for everything issued so far on the partition stream ps
lfm_status join(lfm_plan p, cudaStream_t ps, cudaEvent_t ev, cudaStream_t s) {
    (void)p;
    CK(cudaEventRecord(ev, ps));
    CK(cudaStreamWaitEvent(s, ev, 0));
    return LFM_OK;
}

lfm_status read_kernel_timers(lfm_plan p, int mask = 0xF) {
    mask &= part_skip() & 1 ? 0xA : 0xF;
    mask &= part_skip() & 2 ? 0x5 : 0xF;
    for (int k = 0; k < 4; ++k) {
        if (!((mask >> k) & 1)) continue;
        const bool ran = (k & 1) ? p->nu_fft > 0 : !(k < 2 ? p->tcf.empty() : p->tcb.empty());
        if (!ran) continue;
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, p->kev[k][0], p->kev[k][1]));
        p->pacc.kern_ms[k] += ms;
        p->pacc.kern_count[k] += 1;
    }
    return LFM_OK;
}

void plan_free(lfm_plan p) {
    if (!p) return;
    for (cudaGraphExec_t g : p->gexec) cudaGraphExecDestroy(g);
    for (cudaGraphExec_t g : p->lexec) cudaGraphExecDestroy(g);
    cudaFree(p->lstate);
    cudaFree(p->lseries);
    if (p->sym) sym_destroy(p->sym);
    cudaFree(p->MT);
    cudaFree(p->mf_eb);
    for (auto& gr : p->tgs) {
        for (void* q : {(void*)gr.tw, (void*)gr.umap, (void*)gr.M, (void*)gr.MT, (void*)gr.G, (void*)gr.Xh, (void*)gr.Y,
                        (void*)gr.R, (void*)gr.tmax})
            cudaFree(q);
    }
    if (p->nccl) ncclCommDestroy(p->nccl);
    cudaFree(p->tw_h);
    cudaFree(p->tw_w);
    cudaFree(p->umap);
    for (void* q : p->dallocs) cudaFree(q);
    cudaFree(p->dpart);
    if (p->Mb && p->Mb != p->M) cudaFree(p->Mb);
    cudaFree(p->M);
    if (p->psfb && p->psfb != p->psf) cudaFree(p->psfb);
    cudaFree(p->psf);
    cudaFree(p->norm);
    cudaFree(p->hty);
    cudaFree(p->norm_sum);
    for (auto& x : p->xb) cudaFree(x);
    cudaFree(p->xfull);
    cudaFree(p->G);
    cudaFree(p->Xh);
    cudaFree(p->Y);
    cudaFree(p->R);
    cudaFree(p->yhat);
    cudaFree(p->rimg);
    cudaFree(p->mproj);
    cudaFree(p->partials);
    cudaFree(p->stats);
    cudaFree(p->y_stage);
    cudaFree(p->x_stage);
    cudaFree(p->bG);
    cudaFree(p->bXh);
    cudaFree(p->bY);
    cudaFree(p->bR);
    cudaFree(p->bx);
    cudaFree(p->byhat);
    cudaFree(p->bmproj);
    cudaFree(p->bent);
    cudaFree(p->bmT1);
    cudaFree(p->bmrs);
    if (p->bhost) cudaFreeHost(p->bhost);
    if (p->host) cudaFreeHost(p->host);
    green_free(p);
    if (p->scopy) cudaStreamDestroy(p->scopy);
    if (p->evcopy) cudaEventDestroy(p->evcopy);
    if (p->smet) cudaStreamDestroy(p->smet);
    for (cudaEvent_t e : {p->evupd[0], p->evupd[1], p->evmet[0], p->evmet[1]})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : p->evconv)
        if (e) cudaEventDestroy(e);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    for (auto& e : p->pev)
        if (e) cudaEventDestroy(e);
    for (auto& kv : p->kev)
        for (auto& e : kv)
            if (e) cudaEventDestroy(e);
    metric_free(&p->met);
    delete p;
}

template <typename T>
lfm_status dalloc(lfm_plan p, T** ptr, size_t bytes, const char* what) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(ptr, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? LFM_ENOMEM : LFM_ECUDA, "cudaMalloc(%s, %zu bytes): %s", what,
                    bytes, cudaGetErrorString(e));
    }
    p->bytes += bytes;
    return LFM_OK;
}

lfm_status twiddles(int L, float2** out, lfm_plan p, cudaStream_t s) {
    std::vector<float2> t(L);
    const double pi = 3.14159265358979323846;
    for (int k = 0; k < L; ++k) {
        const double a = -2.0 * pi * k / L;
        t[k] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    ST(dalloc(p, out, L * sizeof(float2), "twiddles"));
    CK(cudaMemcpyAsync(*out, t.data(), L * sizeof(float2), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    return LFM_OK;
}

R2CArgs r2c_args(int src, const float* in, const float* in2, float eps, int ntrans, float2* out, long long ld) {
    R2CArgs a{};
    a.src = src;
    a.in = in;
    a.in2 = in2;
    a.eps = eps;
    a.ntrans = ntrans;
    a.out = out;
    a.out_ld = ld;
    a.cdiv = INT_MAX;
    a.cmul = 0;
    return a;
}

lfm_status allreduce(lfm_plan p, void* buf, size_t n, ncclDataType_t t, ncclRedOp_t op, cudaStream_t s) {
    if (!p->comm) return LFM_OK;
    NK(ncclAllReduce(buf, buf, n, t, op, p->nccl, s));
    return LFM_OK;
}

// yhat = H x (x polyphase, owned units) summed over ranks
// yhat = H x summed over ranks; x polyphase (owned units) or image layout [nz][H][W]
lfm_status op_forward_src(lfm_plan p, const float* x, bool image, float* ysum, cudaStream_t s) {
    const int N2 = p->geo.N * p->geo.N;
    // with a symmetric window the producers write this rank's partial image there and C1 sums it into ysum
    float* yimg = p->sym ? sym_buffer(p->sym, 0) : ysum;
    ST(mark(p, ST_R2C_X, s));
    if (p->direct) {
        const float* xp = x;
        if (image) {
            CK(launch_image_to_poly(x, p->xb[0], p->xall, p->u0, p->nu, s));
            xp = p->xb[0];
        }
        ST(mark(p, ST_FWD_MAC, s));
        ST(mark(p, ST_C2R_YHAT, s));
        ST(mark(p, ST_DIR_FWD, s));
        CK(launch_direct_fwd(xp, p->psf, yimg, p->xall, s));
        p->pacc.launches += 1;
    } else {
        // tensor-core planes: stage the source; FFT units: coarse transforms.  Then the two halves of the projection
        // -- tcgen05 kernel and frequency-path MAC + C2R -- run side by side on the plan's SM partitions (§5.5) or one
        // after the other on `s`; afterwards the direct planes' partial images are added onto the C2R output.
        // With partitions the staging of the tensor-core source and the coarse R2C run inside their halves (each on
        // its own partition, overlapping the other half) rather than on the whole GPU before the fork.
        const lfm_plan_s::Part& pt = p->part[0];
        const bool split = pt.stc != nullptr;
        static const bool prefork = getenv("LFM_STAGE_PREFORK") != nullptr;   // dev A/B: staging before the fork
        cudaStream_t st = s, sm = s;
        if (split && !prefork) ST(fork(p, pt, s, &st, &sm));
        for (const TcDirArgs& tg : p->tcf) CK(launch_tcdir_fwd(tg, x, image ? 1 : 0, yimg, 0, st, TC_PART_STAGE));
        if (p->nu_fft > 0 && p->tiled) {   // §5.6: window transforms of every (tile, unit), |window| bounds per tile
            for (auto& gr : p->tgs) {
                CK(cudaMemsetAsync(gr.tmax, 0, 32 * sizeof(unsigned), sm));
                R2CArgs a = r2c_args(image ? SRC_IMAGE : SRC_POLY, x, nullptr, 0.f, gr.tg.ntile * gr.xg.nu, gr.G, gr.xg.nu_pad);
                a.cdiv = gr.xg.nu;
                a.cmul = (long long)gr.xg.nkappa * gr.xg.nu_pad;
                CK(launch_r2c_tile(gr.xg, gr.tg, gr.tw, a, 0, gr.tmax, sm));
            }
        } else if (p->nu_fft > 0) {
            CK(launch_r2c(p->xg, p->fh, p->fw, p->tw_h, p->tw_w,
                          r2c_args(image ? SRC_IMAGE : SRC_POLY, x, nullptr, 0.f, p->nu_fft, p->G, p->nu_fft_pad), sm));
        }
        if (split && prefork) ST(fork(p, pt, s, &st, &sm));
        ST(mark(p, ST_FWD_MAC, s));
        if (!p->tcf.empty() && !(part_skip() & 1)) {
            ST(kmark(p, 0, 0, st));
            for (const TcDirArgs& tg : p->tcf) CK(launch_tcdir_fwd(tg, x, image ? 1 : 0, yimg, 0, st, TC_PART_MAIN));
            ST(kmark(p, 0, 1, st));
        }
        if (p->nu_fft > 0 && !(part_skip() & 2)) {
            ST(kmark(p, 1, 0, sm));
            if (p->tiled)
                for (auto& gr : p->tgs) CK(launch_mac_f16(gr.fwd, 1, gr.F, split ? pt.sms_mac : p->num_sms, sm));
            else
                CK(launch_fwd_mac(p->M, p->G, p->Y, p->geo.nkappa, N2, p->nu_fft_pad, split ? pt.sms_mac : p->num_sms,
                                  split, sm));
            ST(kmark(p, 1, 1, sm));
        }
        // join the MAC partition, then the C2R on the whole GPU (on the small MAC partition it would lengthen the
        // critical path), then the tensor-core partition.  Tiled plans (§5.6) run their C2R inside the partition.
        const bool c2r_in = split && p->tiled && !c2r_full();
        if (split && !c2r_in) ST(join(p, pt.smac, p->evj2, s));
        if (p->nu_fft > 0) {
            C2RArgs c{};
            c.dst = DST_IMAGE;
            c.in = p->Y;
            c.in_ld = N2;
            c.ntrans = N2;
            c.out = yimg;
            if (p->tiled) {
                for (size_t gi = 0; gi < p->tgs.size(); ++gi) {   // the groups' images summed in group order
                    const auto& gr = p->tgs[gi];
                    c.in = gr.Y;
                    c.ntrans = gr.tg.ntile * N2;
                    c.cdiv = N2;
                    c.cmul = (long long)gr.xg.nkappa * N2;
                    c.nsum = gr.fwd.ksplit;
                    c.in_sstride = gr.fwd.out_sstride;
                    c.accum = gi > 0;
                    CK(launch_c2r_tile(gr.xg, gr.tg, gr.tw, c, 0, c2r_in ? sm : s));
                }
            } else {
                CK(launch_c2r(p->xg, p->fh, p->fw, p->tw_h, p->tw_w, c, s));
            }
            p->pacc.launches += 3;
        }
        if (c2r_in) ST(join(p, pt.smac, p->evj2, s));
        if (split) ST(join(p, pt.stc, p->evj, s));
        ST(mark(p, ST_C2R_YHAT, s));
        ST(mark(p, ST_DIR_FWD, s));
        bool acc = p->nu_fft > 0;
        for (const TcDirArgs& tg : p->tcf) {
            CK(launch_tcdir_fwd(tg, x, image ? 1 : 0, yimg, acc ? 1 : 0, s, TC_PART_FINISH));
            p->pacc.launches += 3;
            acc = true;
        }
        for (const DirArgs& dg : p->dgroups) {
            CK(launch_dir_fwd(dg, x, image ? 1 : 0, p->dpart, yimg, acc ? 1 : 0, s));
            p->pacc.launches += 2;
            acc = true;
        }
        if (!acc) CK(cudaMemsetAsync(yimg, 0, (size_t)p->geo.H * p->geo.W * sizeof(float), s));
    }
    ST(mark(p, ST_ALLRED_SUM, s));
    if (p->sym) {
        CK(sym_reduce(p->sym, 0, ysum, s));
        p->pacc.launches += 1;
        return LFM_OK;
    }
    return allreduce(p, yimg, (size_t)p->geo.H * p->geo.W, ncclFloat, ncclSum, s);
}

lfm_status op_forward_poly(lfm_plan p, const float* xp, float* yimg, cudaStream_t s) {
    return op_forward_src(p, xp, /*image=*/false, yimg, s);
}

// backward projection of an image source into one of the C2R destinations
//   src: SRC_RATIO (img = y, img2 = yhat), SRC_ONES, SRC_IMAGE2D (img)
// aux: the update's second volume (nullptr -> the normalizer H^T 1; ISRA passes H^T y)
lfm_status op_backward(lfm_plan p, int src, const float* img, const float* img2, float eps, int dst, float* out,
                       const float* xold, cudaStream_t s, const float* aux = nullptr) {
    const int N2 = p->geo.N * p->geo.N;
    if (!aux) aux = p->norm;
    ST(mark(p, ST_R2C_RATIO, s));
    if (p->direct) {
        const size_t n = (size_t)p->geo.H * p->geo.W;
        const float* r = img;
        if (src == SRC_RATIO) {
            CK(launch_ratio(img, img2, p->rimg, n, eps, s));
            r = p->rimg;
            p->pacc.launches += 1;
        } else if (src == SRC_ONES) {
            CK(launch_fill(p->rimg, n, 1.0f, s));
            r = p->rimg;
            p->pacc.launches += 1;
        }
        ST(mark(p, ST_BWD_MAC, s));
        ST(mark(p, ST_C2R_UPD, s));
        ST(mark(p, ST_DIR_BWD, s));
        CK(launch_direct_bwd(r, p->psfb, out, dst, xold, aux, p->mproj, eps, p->xall, s));
        p->pacc.launches += 1;
        ST(mark(p, ST_MAXPROJ, s));
        return LFM_OK;
    }
    // as in the forward (§5.5); the two halves write disjoint units of `out`
    const lfm_plan_s::Part& pt = p->part[1];
    const bool split = pt.stc != nullptr;
    static const bool prefork = getenv("LFM_STAGE_PREFORK") != nullptr;
    cudaStream_t st = s, sm = s;
    if (split && !prefork) ST(fork(p, pt, s, &st, &sm));   // staging / R2C inside the halves, as in the forward
    for (const TcDirArgs& tg : p->tcb) CK(launch_tcdir_bwd(tg, src, img, img2, eps, dst, out, xold, aux, st, TC_PART_STAGE));
    if (p->nu_fft > 0 && p->tiled) {   // §5.6: windows of every (tile, output phase), R rows of bpitch
        // the ratio (or the plain image) once into output-phase planes, read row-contiguously by every tile group
        int gsrc = src;
        const float* gimg = img;
        if (src == SRC_RATIO || src == SRC_IMAGE2D) {
            CK(launch_image_phase_planes(img, src == SRC_RATIO ? img2 : nullptr, eps, p->rimg, p->geo.N, p->geo.H,
                                         p->geo.W, sm));
            p->pacc.launches += 1;
            gsrc = SRC_POLY;
            gimg = p->rimg;
        }
        for (auto& gr : p->tgs) {
            CK(cudaMemsetAsync(gr.tmax + 32, 0, 32 * sizeof(unsigned), sm));
            XformGeom gx = gr.xg;
            if (gsrc == SRC_POLY) gx.umap = nullptr;   // item = output phase b' -> plane b' of rimg
            R2CArgs a = r2c_args(gsrc, gimg, img2, eps, gr.tg.ntile * N2, gr.R, p->bpitch);
            a.cdiv = N2;
            a.cmul = (long long)gr.xg.nkappa * p->bpitch;
            CK(launch_r2c_tile(gx, gr.tg, gr.tw, a, 1, gr.tmax + 32, sm));
        }
    } else if (p->nu_fft > 0) {
        CK(launch_r2c(p->xg, p->fh, p->fw, p->tw_h, p->tw_w, r2c_args(src, img, img2, eps, N2, p->R, N2), sm));
    }
    if (split && prefork) ST(fork(p, pt, s, &st, &sm));
    ST(mark(p, ST_BWD_MAC, s));
    if (!p->tcb.empty() && !(part_skip() & 1)) {
        ST(kmark(p, 2, 0, st));
        for (const TcDirArgs& tg : p->tcb) {
            CK(launch_tcdir_bwd(tg, src, img, img2, eps, dst, out, xold, aux, st, TC_PART_MAIN));
            p->pacc.launches += (dst == DST_UPDATE || dst == DST_ISRA) ? 3 : 2;
        }
        ST(kmark(p, 2, 1, st));
    }
    if (p->nu_fft > 0 && !(part_skip() & 2)) {
        ST(kmark(p, 3, 0, sm));
        if (p->tiled)
            for (auto& gr : p->tgs) CK(launch_mac_f16(gr.bwd, 0, gr.F, split ? pt.sms_mac : p->num_sms, sm));
        else
            CK(launch_bwd_mac(p->Mb, p->R, p->Xh, p->geo.nkappa, N2, p->nu_fft_pad, sm));
        ST(kmark(p, 3, 1, sm));
    }
    const bool c2r_in = split && p->tiled && !c2r_full();   // as in the forward
    if (split && !c2r_in) ST(join(p, pt.smac, p->evj2, s));   // C2R + update on the whole GPU, as in the forward
    if (p->nu_fft > 0) {
        C2RArgs c{};
        c.dst = dst;
        c.in = p->Xh;
        c.in_ld = p->nu_fft_pad;
        c.ntrans = p->nu_fft;
        c.out = out;
        c.xold = xold;
        c.norm = aux;
        c.eps = eps;
        if (p->tiled) {
            for (const auto& gr : p->tgs) {   // disjoint units
                c.in = gr.Xh;
                c.in_ld = gr.xg.nu_pad;
                c.ntrans = gr.tg.ntile * gr.xg.nu;
                c.cdiv = gr.xg.nu;
                c.cmul = (long long)gr.xg.nkappa * gr.xg.nu_pad;
                CK(launch_c2r_tile(gr.xg, gr.tg, gr.tw, c, 1, c2r_in ? sm : s));
            }
        } else {
            CK(launch_c2r(p->xg, p->fh, p->fw, p->tw_h, p->tw_w, c, s));
        }
        p->pacc.launches += 3;
    }
    if (c2r_in) ST(join(p, pt.smac, p->evj2, s));
    if (split) ST(join(p, pt.stc, p->evj, s));
    ST(mark(p, ST_C2R_UPD, s));
    ST(mark(p, ST_DIR_BWD, s));
    for (const DirArgs& dg : p->dgroups) {
        CK(launch_dir_bwd(dg, src, img, img2, eps, dst, out, xold, aux, s));
        p->pacc.launches += 1;
    }
    ST(mark(p, ST_MAXPROJ, s));
    return LFM_OK;
}

lfm_status op_metric(lfm_plan p, int region, cudaStream_t s) {
    if (!p->has_optics) return fail(LFM_EINVAL, "plan was created without optics: the DCT-entropy metric needs them");
    const int ri = region == LFM_REGION_RECTANGLE ? 1 : 0;
    if (p->sym) {   // C2 in our own kernel over the symmetric window: the partial max-projection sits in slot 1
        CK(sym_reduce(p->sym, 1, p->mproj, s));
        p->pacc.launches += 1;
    } else {
        ST(allreduce(p, p->mproj, (size_t)p->geo.H * p->geo.W, ncclFloat, ncclMax, s));
    }
    ST(mark(p, ST_METRIC, s));
    CK(launch_metric(p->mproj, p->geo.H, p->geo.W, p->met.xs, p->met.ys, p->met.Cr, p->met.Cw, p->met.mem[ri],
                     p->met.nmem[ri], p->met.T1, p->met.rowsq, p->met.out, s));
    p->pacc.launches += 3;
    ST(mark(p, LFM_N_STAGES, s));
    return LFM_OK;
}

// one iteration on polyphase volumes, then the z max-projection and (optionally) the metric -> met.out[0]
//   RL   (C1): xn = xc * H^T(y/(max(H xc,0)+eps)) / max(H^T 1, eps)
//   ISRA (f3): xn = xc * H^T y / max(H^T H xc, eps)           (hty = H^T y, polyphase)
// a7 z max-projection of the new iterate, every pixel written (into the symmetric window's slot 1 when C2
// runs there), and optionally the metric (a8)
lfm_status op_tail(lfm_plan p, const float* xn, int region, bool metric, cudaStream_t s) {
    CK(launch_max_project_poly(xn, p->sym ? reinterpret_cast<unsigned*>(sym_buffer(p->sym, 1)) : p->mproj, p->xall, s));
    p->pacc.launches += 1;
    if (metric) ST(op_metric(p, region, s));
    return LFM_OK;
}

lfm_status op_step(lfm_plan p, const float* y, const float* xc, float* xn, float eps, int region, bool metric,
                   cudaStream_t s, int update = LFM_UPDATE_RL, const float* hty = nullptr, bool tail = true) {
    ST(op_forward_poly(p, xc, p->yhat, s));
    if (update == LFM_UPDATE_ISRA)
        ST(op_backward(p, SRC_IMAGE2D, p->yhat, nullptr, eps, DST_ISRA, xn, xc, s, hty));
    else
        ST(op_backward(p, SRC_RATIO, y, p->yhat, eps, DST_UPDATE, xn, xc, s));
    if (tail) ST(op_tail(p, xn, region, metric, s));
    return LFM_OK;
}

// f4: the whole iteration (transforms, MACs, direct planes, collectives, metric and the 8-byte D2H of E) as
// one CUDA graph, captured on first use for a (cur, next) buffer pair and replayed with a single launch.
lfm_status step_graph(lfm_plan p, const float* y, int cur, int nxt, const lfm_policy* pol, cudaStream_t s) {
    size_t gi = 0;
    for (; gi < p->gkeys.size(); ++gi) {
        const auto& k = p->gkeys[gi];
        if (k.cur == cur && k.nxt == nxt && k.y == y && k.eps == pol->eps && k.region == pol->region &&
            k.update == pol->update)
            break;
    }
    if (gi == p->gkeys.size()) {
        if (s == nullptr) return fail(LFM_EINVAL, "LFM_PLAN_GRAPHS needs a non-default stream (legacy stream cannot be captured)");
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        lfm_status st = op_step(p, y, p->xb[cur], p->xb[nxt], pol->eps, pol->region, true, s, pol->update, p->hty);
        cudaError_t ce = cudaSuccess;
        if (st == LFM_OK) ce = cudaMemcpyAsync(p->host, p->met.out, sizeof(double), cudaMemcpyDeviceToHost, s);
        cudaError_t ee = cudaStreamEndCapture(s, &graph);
        if (st != LFM_OK) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        if (ce != cudaSuccess || ee != cudaSuccess) {
            if (graph) cudaGraphDestroy(graph);
            return fail(LFM_ECUDA, "graph capture failed: %s", cudaGetErrorString(ce != cudaSuccess ? ce : ee));
        }
        cudaGraphExec_t exec = nullptr;
        cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) return fail(LFM_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ie));
        p->gkeys.push_back({cur, nxt, pol->region, pol->update, y, pol->eps});
        p->gexec.push_back(exec);
    }
    CK(cudaGraphLaunch(p->gexec[gi], s));
    return LFM_OK;
}


// one RL iteration xb[src] -> xb[dst] + device stop rule + argmax snapshot, captured into graph g
lfm_status capture_half(lfm_plan p, cudaGraph_t g, const float* y, const lfm_policy* pol, int cap, int src, int dst,
                        cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_second, int has_second,
                        cudaStream_t s) {
    const size_t vol = (size_t)p->nu * p->geo.nh * p->geo.nw;
    CK(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    lfm_status st = op_step(p, y, p->xb[src], p->xb[dst], pol->eps, pol->region, true, s, pol->update, p->hty);
    cudaError_t ce = cudaSuccess;
    if (st == LFM_OK) ce = launch_stop_rule(p->lstate, p->met.out, p->lseries, pol, cap, h_loop, h_second, has_second, s);
    if (st == LFM_OK && ce == cudaSuccess) ce = launch_cond_copy(p->lstate, p->xb[dst], p->xb[2], vol, s);
    cudaGraph_t out = nullptr;
    cudaError_t ee = cudaStreamEndCapture(s, &out);
    if (st != LFM_OK) return st;
    if (ce != cudaSuccess || ee != cudaSuccess)
        return fail(LFM_ECUDA, "loop capture failed: %s", cudaGetErrorString(ce != cudaSuccess ? ce : ee));
    return LFM_OK;
}

// the device-resident loop graph for (y, policy): WHILE(h) { it(0->1); IF(h2) { it(1->0) } }
lfm_status loop_graph(lfm_plan p, const float* y, const lfm_policy* pol, int cap, cudaGraphExec_t* exec_out,
                      cudaStream_t s) {
    for (size_t i = 0; i < p->lkeys.size(); ++i) {
        const auto& k = p->lkeys[i];
        if (k.y == y && k.eps == pol->eps && k.region == pol->region && k.update == pol->update && k.mode == pol->mode &&
            k.n_iters == pol->n_iters && k.min_iters == pol->min_iters && k.patience == pol->patience &&
            k.max_iters == pol->max_iters) {
            *exec_out = p->lexec[i];
            return LFM_OK;
        }
    }
    if (s == nullptr) return fail(LFM_EINVAL, "LFM_PLAN_DEVICE_LOOP needs a non-default stream (legacy stream cannot be captured)");
    cudaGraph_t G = nullptr;
    CK(cudaGraphCreate(&G, 0));
    auto bail = [&](lfm_status st) {
        cudaGraphDestroy(G);
        return st;
    };
#define LG(call)                                                                                      \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess) return bail(fail(LFM_ECUDA, "%s: %s", #call, cudaGetErrorString(e_))); \
    } while (0)
    cudaGraphConditionalHandle h_loop, h_second;
    LG(cudaGraphConditionalHandleCreate(&h_loop, G, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = h_loop;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    LG(cudaGraphAddNode(&wnode, G, nullptr, 0, &wp));
    cudaGraph_t W = wp.conditional.phGraph_out[0];
    LG(cudaGraphConditionalHandleCreate(&h_second, W, 0, cudaGraphCondAssignDefault));
    cudaGraph_t A = nullptr;
    LG(cudaGraphCreate(&A, 0));
    lfm_status st = capture_half(p, A, y, pol, cap, 0, 1, h_loop, h_second, 1, s);
    if (st != LFM_OK) {
        cudaGraphDestroy(A);
        return bail(st);
    }
    cudaGraphNode_t anode;
    cudaError_t ae = cudaGraphAddChildGraphNode(&anode, W, nullptr, 0, A);
    cudaGraphDestroy(A);
    LG(ae);
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = h_second;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    cudaGraphNode_t inode;
    LG(cudaGraphAddNode(&inode, W, &anode, 1, &ip));
    st = capture_half(p, ip.conditional.phGraph_out[0], y, pol, cap, 1, 0, h_loop, h_second, 0, s);
    if (st != LFM_OK) return bail(st);
    cudaGraphExec_t exec = nullptr;
    LG(cudaGraphInstantiate(&exec, G, 0));
#undef LG
    cudaGraphDestroy(G);
    p->lkeys.push_back({y, pol->eps, pol->region, pol->update, pol->mode, pol->n_iters, pol->min_iters, pol->patience,
                        pol->max_iters});
    p->lexec.push_back(exec);
    *exec_out = exec;
    return LFM_OK;
}

lfm_status check_policy(const lfm_policy* pol) {
    if (!pol) return fail(LFM_EINVAL, "policy is NULL");
    if (pol->mode != LFM_MODE_FIXED && pol->mode != LFM_MODE_AUTO) return fail(LFM_EINVAL, "policy.mode=%d", pol->mode);
    if (pol->mode == LFM_MODE_FIXED && pol->n_iters < 1) return fail(LFM_EINVAL, "policy.n_iters must be >= 1");
    if (pol->mode == LFM_MODE_AUTO && (pol->min_iters < 1 || pol->min_iters > pol->max_iters))
        return fail(LFM_EINVAL, "policy: need 1 <= min_iters <= max_iters (S:254)");
    if (pol->patience < 1) return fail(LFM_EINVAL, "policy.patience must be >= 1 (S:254)");
    if (!(pol->eps > 0.0f)) return fail(LFM_EINVAL, "policy.eps must be > 0");
    if (pol->region != LFM_REGION_TRIANGLE && pol->region != LFM_REGION_RECTANGLE)
        return fail(LFM_EINVAL, "policy.region=%d", pol->region);
    if (pol->update != LFM_UPDATE_RL && pol->update != LFM_UPDATE_ISRA) return fail(LFM_EINVAL, "policy.update=%d", pol->update);
    return LFM_OK;
}

// y validation -> sum(y) left in p->stats[0]
lfm_status check_y(lfm_plan p, const float* y, cudaStream_t s) {
    const size_t n = (size_t)p->geo.H * p->geo.W;
    CK(launch_sum_stats(y, n, p->partials, kParts, p->stats, s));
    CK(cudaMemcpyAsync(p->host, p->stats, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (!(p->host[1] >= 0.0)) return fail(LFM_ENEG, "measurement y has a negative (or NaN) entry: min=%g (S:270)", p->host[1]);
    if (!(p->host[2] > 0.0)) return fail(LFM_EZERO, "measurement y is all zero (S:288)");
    return LFM_OK;
}

lfm_status gather_to_image(lfm_plan p, const float* xp_local, float* x, cudaStream_t s) {
    if (!p->comm) {
        CK(launch_poly_to_image(xp_local, x, p->xall, p->u0, p->nu, s));
        return LFM_OK;
    }
    const size_t per = (size_t)p->geo.nh * p->geo.nw;
    NK(ncclGroupStart());
    for (int r = 0; r < p->world; ++r) {
        const int b = p->rcut[r], e = p->rcut[r + 1];
        if (e <= b) continue;
        ncclResult_t rr = ncclBroadcast(r == p->rank ? (const void*)xp_local : nullptr, p->xfull + (size_t)b * per,
                                        (size_t)(e - b) * per, ncclFloat, r, p->nccl, s);
        if (rr != ncclSuccess) {
            ncclGroupEnd();
            return fail(LFM_ENCCL, "ncclBroadcast: %s", ncclGetErrorString(rr));
        }
    }
    NK(ncclGroupEnd());
    CK(launch_poly_to_image(p->xfull, x, p->xall, 0, p->nu_total, s));
    return LFM_OK;
}


inline int floordiv(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }
inline int ceildiv(int a, int b) { return -floordiv(-a, b); }

// Tap box of the coarse kernels of one plane along one axis: for input phase a and output phase b the
// coarse taps d with PSF index k = b - a + c + N d inside the plane's non-zero support [k0, k1].
struct AxisBox {
    int D = 0, dmin = 0, dmax = 0;
    std::vector<int> dlo;   // [a][b]
};
AxisBox axis_box(int N, int c, int k0, int k1) {
    AxisBox bx;
    bx.dlo.assign((size_t)N * N, 0);
    bx.dmin = 1 << 30;
    bx.dmax = -(1 << 30);
    for (int a = 0; a < N; ++a)
        for (int b = 0; b < N; ++b) {
            const int lo = ceildiv(k0 - c - (b - a), N), hi = floordiv(k1 - c - (b - a), N);
            bx.dlo[(size_t)a * N + b] = lo;
            bx.D = std::max(bx.D, hi - lo + 1);
            bx.dmin = std::min(bx.dmin, lo);
            bx.dmax = std::max(bx.dmax, lo);
        }
    return bx;
}

// Planning constants of the hybrid cost model (per iteration, both projections):
//   frequency path  2 * units * N^2 * n_kappa * 8 B at kHbmBps, plus the coarse transforms;
//   direct path     2 * units * N^2 * D^2 * nh * nw * 2 flop at kDirFlops[D].
constexpr double kHbmBps = 7.0e12;
constexpr double kXformPerUnit = 9.0e-8;
const double kDirFlops[kDirMaxD + 1] = {1.0, 6.0e12, 14.0e12, 22.0e12, 26.0e12, 28.0e12};
// tensor-core direct path: achieved fraction of the tcgen05 floor (measured r01 at c3, staging and partial
// reduction included) and a fixed per-plane cost
constexpr double kTcEff = 0.68;
constexpr double kTcFixed = 5e-6;
constexpr double kSmClock = 1.965e9;
// SM partitions (§5.5), fitted to r01 measurements at c3 (scripts/gpu_part_sweep.sh, 88-120 tensor-core SMs) in
// terms of this cost model's own estimates (t_tc = 2.96 ms, 18.5 GB of transfer matrices per direction at c3):
//   tcgen05 side by side with a MAC on S SMs = kTcPartEff * kTcConc[d] * t_tc * N / S;
//   the MAC streams kMacSmBps[d] per SM alone (the whole GPU tops out at HBM), kMacConc[d] slower side by side,
//   its C2R (kC2rFull[d]) runs on the whole GPU after the join.
constexpr double kTcPartEff = 1.0;
constexpr double kTcConc[2] = {0.93, 0.95};   // warp-uniform MMA issue, 24-K-step drain groups (1.10, 1.16 before)
constexpr double kMacSmBps[2] = {92e9, 136e9};   // forward refitted r02 (f16 tensor side): 79 GB/s per SM side by side
constexpr double kMacConc[2] = {1.17, 1.12};
constexpr double kC2rFull[2] = {0.02e-3, 0.15e-3};
// HBM ceiling of a MAC partition (measured alone on 60-68 SMs: forward 6.3, backward 6.6 TB/s; side by side the
// backward still reaches 6.7 TB/s, hence the higher backward figure before kMacConc)
constexpr double kHbmPartBps[2] = {6.6e12, 7.5e12};

// predicted time of one direction (0 forward, 1 backward) of a projection whose tensor-core planes take t_tc on the
// whole GPU and whose frequency-path planes stream `bytes`: run one after the other, or side by side on the best SM
// partition (*best_s tensor-core SMs, 0 = one after the other)
double partition_time(double t_tc, double bytes, int d, int num_sms, int* best_s, double mac_rate_scale = 1.0) {
    const double serial = t_tc + bytes / kHbmBps + kC2rFull[d];
    double best = serial;
    *best_s = 0;
    if (t_tc <= 0 || bytes <= 0) return serial;
    for (int sm_tc = 16; sm_tc <= num_sms - 16; sm_tc += 8) {
        const int sm_mac = num_sms - sm_tc;
        const double t_tcp = kTcPartEff * kTcConc[d] * t_tc * num_sms / sm_tc;
        const double t_mac = kMacConc[d] * bytes / std::min(kHbmPartBps[d], kMacSmBps[d] * mac_rate_scale * sm_mac);
        const double t = std::max(t_tcp, t_mac) + kC2rFull[d];   // the C2R runs on the whole GPU after the join
        if (t < best) {
            best = t;
            *best_s = sm_tc;
        }
    }
    if (best >= 0.97 * serial) {   // not worth two green contexts
        *best_s = 0;
        return serial;
    }
    return best;
}

// ---- overlap-save tiles of the frequency path ----
// Per FFT unit and iteration: the split M (forward) and M^T (backward) streamed once each by the kind::f16 MACs,
// the tiles' spectra written by the R2C and read by the MAC (and the reverse), and the window transforms.
constexpr double kMacF16Bps = 5.3e12;        // kind::f16 tile MACs, HBM-bound (r02 c3 tiles: 5.25-5.45 TB/s)
constexpr double kXformPoint = 6.0e-12;      // whole-image transform seconds per point and direction (r02, L = 75)
constexpr double kXformPointTile = 4.5e-12;  // register-resident tile transforms, L <= 36 (r02, L = 27: 4.1e-12)
constexpr double kXformPointTileW = 7.5e-12; // warp-per-transform tile kernels, L > 36 (r02, L = 27: 7.5e-12)
constexpr double kPartMinShare = 0.18;     // smallest tensor-core share of a tiled projection that gets an SM partition
constexpr double kTcBwdLive = 1.25;         // tcgen05 backward / forward time live beside the tile half (r02: c3 1.23, c2 1.39)

// tile geometry for transform size L (ntile = 0: not possible) over coarse taps in [d1a, d1b] x [d2a, d2b]
TileGeom tile_geometry(const Geo& g, int L, int d1a, int d1b, int d2a, int d2b) {
    TileGeom t{};
    t.L = L;
    t.dmin1 = d1a;
    t.dmax1 = d1b;
    t.dmin2 = d2a;
    t.dmax2 = d2b;
    t.T1 = L - (t.dmax1 - t.dmin1);
    t.T2 = L - (t.dmax2 - t.dmin2);
    if (t.T1 < 1 || t.T2 < 1 || !tile_fft_size(L)) return TileGeom{};
    t.nty = (g.nh + t.T1 - 1) / t.T1;
    t.ntx = (g.nw + t.T2 - 1) / t.T2;
    t.ntile = t.nty * t.ntx;
    if (t.ntile > 32 || t.ntile < 2) return TileGeom{};
    return t;
}

double tile_unit_cost(const TileGeom& t, int N2) {
    const double nkap = (double)t.L * (t.L / 2 + 1);
    const double bpitch = (double)round_up((size_t)N2, 4);
    return nkap * (N2 + bpitch) * 8.0 / kMacF16Bps + 4.0 * t.ntile * nkap * 8.0 / kHbmBps +
           2.0 * (t.L <= 36 ? kXformPointTile : kXformPointTileW) * t.ntile * t.L * t.L;
}

double whole_unit_cost(const Geo& g, int N2) {
    return 2.0 * N2 * (double)g.nkappa * 8.0 / kHbmBps + 2.0 * kXformPoint * g.Lh * g.Lw;
}

// the cheapest tiling of coarse taps in [d1a, d1b] x [d2a, d2b] (ntile = 0: none possible, or LFM_PLAN_NO_TILES /
// FRAMES / DIRECT plans)
TileGeom choose_tiles(const Geo& g, int N2, int flags, int d1a, int d1b, int d2a, int d2b) {
    if ((flags & (LFM_PLAN_NO_TILES | LFM_PLAN_FRAMES | LFM_PLAN_DIRECT)) || N2 > 256) return TileGeom{};
    // the window offsets (forward outputs at dmax, backward at -dmin) need 0 in the tap range: a one-sided support
    // (an off-centre PSF) widens its range to the centre
    d1a = std::min(d1a, 0);
    d2a = std::min(d2a, 0);
    d1b = std::max(d1b, 0);
    d2b = std::max(d2b, 0);
    static const int cand[] = {16, 18, 20, 24, 25, 27, 30, 32, 36, 40, 45, 48};
    TileGeom best{};
    double best_c = 1e300;
    const char* ev = getenv("LFM_TILE_L");   // dev override of the transform size
    for (int L : cand) {
        if (ev && atoi(ev) != L) continue;
        const TileGeom t = tile_geometry(g, L, d1a, d1b, d2a, d2b);
        if (t.ntile == 0) continue;
        const double c = tile_unit_cost(t, N2);
        if (c < best_c) {
            best_c = c;
            best = t;
        }
    }
    return best;
}

// the same for a whole kh x kw kernel: coarse taps of every phase pair lie in [dmin, dmax] with N d + b - a + c in
// [0, k - 1] (reading of S:192's kernel centring); ntile = 0 also when whole-image transforms are
// cheaper by the cost model (the sharding model's view of the frequency path)
TileGeom choose_tiles(const Geo& g, int N2, int flags) {
    const TileGeom t = choose_tiles(g, N2, flags, ceildiv(-(g.N - 1) - g.ch, g.N), floordiv(g.kh - 1 + (g.N - 1) - g.ch, g.N),
                                    ceildiv(-(g.N - 1) - g.cw, g.N), floordiv(g.kw - 1 + (g.N - 1) - g.cw, g.N));
    if (t.ntile && !(flags & LFM_PLAN_TILES) && !(tile_unit_cost(t, N2) < 0.9 * whole_unit_cost(g, N2))) return TileGeom{};
    return t;
}

// SM partitions are used unless the plan runs the device-resident loop (its conditional graph body cannot hold
// kernels of other contexts), the driver lacks green contexts, or LFM_SERIAL is set (dev)
bool partitions_allowed(int flags) {
    return !(flags & (LFM_PLAN_DEVICE_LOOP | LFM_PLAN_FFT_ONLY | LFM_PLAN_DIRECT)) && !getenv("LFM_SERIAL") &&
           green_api().ok;
}

// tensor-core SMs for direction d, or 0 when one-after-the-other is predicted faster
int choose_partition(double t_tc, double bytes, int d, int num_sms, double mac_rate_scale) {
    const char* ev = getenv(d ? "LFM_TC_SMS_B" : "LFM_TC_SMS_F");   // dev override (0 = one after the other)
    if (ev) return atoi(ev);
    int best_s = 0;
    const double best = partition_time(t_tc, bytes, d, num_sms, &best_s, mac_rate_scale);
    if (getenv("LFM_PLAN_VERBOSE"))
        fprintf(stderr, "[lfm plan] direction %d: t_tc %.3f ms, MAC %.2f GB, predicted %.3f ms at %d tc SMs\n", d,
                t_tc * 1e3, bytes / 1e9, best * 1e3, best_s);
    return best_s;
}

// ---- cost-balanced sharding ----
// Per plane, as if one rank owned all of it: the path the hybrid cost model picks and its time per iteration.
// Frequency-path and CUDA-core planes cost in proportion to the units a rank owns; a tensor-core plane costs its
// whole-plane time whatever fraction a rank owns (the kernel runs every phase), so it is never split.
struct PlaneCost {
    double t;
    int atomic;
};

double tc_plane_time(const AxisBox& b1, const AxisBox& b2, const Geo& g, int N2, int num_sms) {
    const int T1 = b1.dmax - b1.dmin + b1.D, T2 = b2.dmax - b2.dmin + b2.D;
    const int Ntile = (int)round_up((size_t)N2, 16), ksteps = (N2 + 15) / 16;   // kind::f16 K-steps of 16 phases
    const int ptiles = (g.nh * (g.nw + T2 - 1) + 255) / 256;
    const double act = T1 >= 3 ? 1.0 - 1.0 / T1 : 1.0;   // edge tap rows: about half the chunks skipped
    const double pair_cycles = (double)ptiles * T1 * T2 * act * ksteps * 3.0 * (Ntile / 2);
    static const double tc_eff = getenv("LFM_TC_EFF") ? atof(getenv("LFM_TC_EFF")) : kTcEff;   // dev override
    return 2.0 * pair_cycles / ((num_sms / 2) * kSmClock * tc_eff) + kTcFixed;
}

std::vector<PlaneCost> plane_costs(const float* psf, int nnum, const Geo& g, int flags, int num_sms) {
    const int N2 = nnum * nnum, kh = g.kh, kw = g.kw;
    const size_t kk = (size_t)kh * kw;
    std::vector<PlaneCost> pc(g.nz);
    for (int z = 0; z < g.nz; ++z) {
        int k0 = kh, k1 = -1, j0 = kw, j1 = -1;
        for (int a = 0; a < N2; ++a) {
            const float* ker = psf + ((size_t)z * N2 + a) * kk;
            for (int i = 0; i < kh; ++i)
                for (int j = 0; j < kw; ++j)
                    if (ker[(size_t)i * kw + j] != 0.0f) {
                        k0 = std::min(k0, i);
                        k1 = std::max(k1, i);
                        j0 = std::min(j0, j);
                        j1 = std::max(j1, j);
                    }
        }
        if (k1 < 0) {
            k0 = k1 = g.ch;
            j0 = j1 = g.cw;
        }
        const AxisBox b1 = axis_box(nnum, g.ch, k0, k1), b2 = axis_box(nnum, g.cw, j0, j1);
        const int D = std::max(b1.D, b2.D);
        const int T2 = b2.dmax - b2.dmin + b2.D;
        const TileGeom tl = choose_tiles(g, N2, flags);   // the frequency path as the plan would build it (§5.6)
        const double t_fft = N2 * (tl.ntile ? tile_unit_cost(tl, N2) : whole_unit_cost(g, N2));
        const double t_dir = D <= kDirMaxD ? 2.0 * N2 * N2 * D * D * (double)g.nh * g.nw * 2.0 / kDirFlops[D] : 1e30;
        const bool tc_ok = !(flags & LFM_PLAN_NO_TC) && round_up((size_t)N2, 16) <= 256 && T2 <= 65;
        const double t_tc = tc_ok ? tc_plane_time(b1, b2, g, N2, num_sms) : 1e30;
        int mode;
        if (flags & LFM_PLAN_FFT_ONLY)
            mode = 0;
        else if (flags & LFM_PLAN_DIRECT)
            mode = (flags & LFM_PLAN_TC_DIRECT) && tc_ok ? 2 : 1;
        else {
            const double best = std::min(t_fft, std::min(t_dir, t_tc));
            mode = best == t_fft ? 0 : (best == t_tc ? 2 : 1);
        }
        pc[z].t = mode == 0 ? t_fft : (mode == 2 ? t_tc : (D <= kDirMaxD ? t_dir : t_fft));
        pc[z].atomic = mode == 2;
    }
    return pc;
}

// contiguous unit ranges [cut[r], cut[r+1]) whose estimated costs are as equal as the cut granularity allows:
// frequency-path / CUDA-core planes may be cut between any two units, tensor-core planes only at their borders
std::vector<int> balanced_cuts(const std::vector<PlaneCost>& pc, int N2, int world) {
    const int nz = (int)pc.size();
    double total = 0;
    for (const PlaneCost& c : pc) total += c.t;
    std::vector<int> cut(world + 1, 0);
    cut[world] = nz * N2;
    for (int r = 1; r < world; ++r) {
        const double target = total * r / world;
        double pre = 0;
        int u = nz * N2;
        for (int z = 0; z < nz; ++z) {
            if (pre + pc[z].t >= target) {
                if (pc[z].atomic)
                    u = (target - pre <= pre + pc[z].t - target) ? z * N2 : (z + 1) * N2;
                else
                    u = z * N2 + (int)std::lround((target - pre) / std::max(pc[z].t, 1e-30) * N2);
                break;
            }
            pre += pc[z].t;
        }
        cut[r] = std::max(cut[r - 1], std::min(u, nz * N2));
    }
    return cut;
}

double range_cost(const std::vector<PlaneCost>& pc, int N2, int b, int e) {
    double t = 0;
    for (int z = 0; z < (int)pc.size(); ++z) {
        const int lo = std::max(b, z * N2), hi = std::min(e, (z + 1) * N2);
        if (hi <= lo) continue;
        t += pc[z].atomic ? pc[z].t : pc[z].t * (hi - lo) / N2;
    }
    return t;
}

// §5.6: one tile group: window geometry tg over the local units `units`; builds its transfer matrices on the L x L
// grid (K1 on the window size), the split M / M^T of the kind::f16 MACs, its spectra buffers and MAC arguments
lfm_status build_tile_group(lfm_plan p, lfm_plan_s::TileGroup& gr, const TileGeom& tg, const std::vector<int>& units,
                            const XformGeom& xg_plan, bool has_ht, cudaStream_t s) {
    const int N2 = p->geo.N * p->geo.N;
    const int L = tg.L, nkap = L * (L / 2 + 1), nt = tg.ntile;
    const int nu = (int)units.size(), nu_pad = (int)round_up((size_t)nu, 16);
    gr.tg = tg;
    gr.xg = xg_plan;
    gr.xg.Lh = gr.xg.Lw = L;
    gr.xg.nk2 = L / 2 + 1;
    gr.xg.nkappa = nkap;
    gr.xg.nu = nu;
    gr.xg.nu_pad = nu_pad;
    if (!fft_factor(L, &gr.fd)) return fail(LFM_EUNSUPPORTED, "tile window %d is not 5-smooth", L);
    {
        std::vector<float2> t(L);
        for (int k = 0; k < L; ++k) {
            const double ang = -2.0 * 3.14159265358979323846 * k / L;
            t[k] = make_float2((float)std::cos(ang), (float)std::sin(ang));
        }
        ST(dalloc(p, &gr.tw, L * sizeof(float2), "tile twiddles"));
        CK(cudaMemcpy(gr.tw, t.data(), L * sizeof(float2), cudaMemcpyHostToDevice));
    }
    ST(dalloc(p, &gr.umap, nu * sizeof(int), "tile group unit map"));
    CK(cudaMemcpy(gr.umap, units.data(), nu * sizeof(int), cudaMemcpyHostToDevice));
    gr.xg.umap = gr.umap;
    const size_t mbytes = (size_t)nkap * N2 * nu_pad * sizeof(float2);
    const size_t mtb = (size_t)nkap * nu_pad * p->bpitch * sizeof(float2);
    const size_t gbytes = (size_t)nt * nkap * nu_pad * sizeof(float2);
    // forward MAC split along K so that every SM gets >= 16 (kappa, half, split) items (load balance); the partial
    // spectra are summed in split order by the C2R
    const int ksplit = std::max(1, std::min(8, (16 * p->num_sms + 2 * nkap - 1) / (2 * nkap)));
    ST(dalloc(p, &gr.M, mbytes, "transfer matrices (tiles)"));
    ST(dalloc(p, &gr.MT, mtb, "transposed transfer matrices (tiles)"));
    ST(dalloc(p, &gr.G, gbytes, "G spectra (tiles)"));
    ST(dalloc(p, &gr.Xh, gbytes, "Xh spectra (tiles)"));
    ST(dalloc(p, &gr.Y, (size_t)ksplit * nt * nkap * N2 * sizeof(float2), "Y spectra (tiles)"));
    ST(dalloc(p, &gr.R, (size_t)nt * nkap * p->bpitch * sizeof(float2), "R spectra (tiles)"));
    ST(dalloc(p, &gr.tmax, 64 * sizeof(unsigned), "tile scale bounds"));
    p->transfer_bytes += mbytes + mtb;
    CK(cudaMemsetAsync(gr.M, 0, mbytes, s));   // padding columns stay zero
    CK(cudaMemsetAsync(gr.G, 0, gbytes, s));
    CK(cudaMemsetAsync(gr.R, 0, (size_t)nt * nkap * p->bpitch * sizeof(float2), s));
    CK(cudaMemsetAsync(gr.tmax, 0, 64 * sizeof(unsigned), s));
    // K1 on the window grid: M[kappa][b'][t] = DFT_{L x L}(g_{u(t),b'}) (taps within the group's range: no wrap)
    R2CArgs a = r2c_args(SRC_KERNEL, p->psf, nullptr, 0.f, N2 * nu, gr.M, (long long)N2 * nu_pad);
    a.cdiv = nu;
    a.cmul = nu_pad;
    CK(launch_r2c(gr.xg, gr.fd, gr.fd, gr.tw, gr.tw, a, s));
    float2* Mb = gr.M;
    if (has_ht) {   // rot180(Ht): only its transposed split copy is kept
        ST(dalloc(p, &Mb, mbytes, "backward transfer matrices (tiles, temporary)"));
        CK(cudaMemsetAsync(Mb, 0, mbytes, s));
        R2CArgs ab = r2c_args(SRC_KERNEL, p->psfb, nullptr, 0.f, N2 * nu, Mb, (long long)N2 * nu_pad);
        ab.cdiv = nu;
        ab.cmul = nu_pad;
        CK(launch_r2c(gr.xg, gr.fd, gr.fd, gr.tw, gr.tw, ab, s));
    }
    // M (forward) and M^T (backward) split into scaled fp16 hi / lo rows as for FRAMES plans; the tiles' spectra G / R
    // are the MACs' frames, their |window| bounds the per-tile scales
    CK(mac_f16_prepare(gr.M, Mb, gr.MT, nkap, N2, nu_pad, p->bpitch, &gr.fwd, &gr.bwd, s));
    if (Mb != gr.M) {
        CK(cudaStreamSynchronize(s));
        cudaFree(Mb);
        p->bytes -= mbytes;
    }
    gr.F = nt <= 8 ? 8 : (nt <= 16 ? 16 : 32);
    CK(mac_f16_encode_src(&gr.fwd, 1, gr.G, (long long)nkap * nu_pad, gr.F, nt));
    CK(mac_f16_encode_src(&gr.bwd, 0, gr.R, (long long)nkap * p->bpitch, gr.F, nt));
    gr.fwd.bmax = gr.tmax;
    gr.fwd.out = gr.Y;
    gr.fwd.out_fstride = (long long)nkap * N2;
    gr.fwd.out_ld = N2;
    gr.fwd.ksplit = ksplit;
    gr.fwd.out_sstride = (long long)nt * nkap * N2;
    gr.bwd.bmax = gr.tmax + 32;
    gr.bwd.out = gr.Xh;
    gr.bwd.out_fstride = (long long)nkap * nu_pad;
    gr.bwd.out_ld = nu_pad;
    // algorithmic bytes of one projection's MAC (M or M^T of the real units + the tiles' spectra in and out)
    p->fft_alg_bytes += (double)nkap * N2 * nu * 8.0 + (double)nt * nkap * (nu + N2) * 8.0;
    return LFM_OK;
}

}  // namespace

// ================================================================================================
extern "C" {

lfm_policy lfm_policy_default(void) {
    lfm_policy p;
    p.mode = LFM_MODE_AUTO;
    p.n_iters = 10;
    p.max_iters = 50;
    p.min_iters = 2;
    p.patience = 1;
    p.eps = 1e-6f;
    p.region = LFM_REGION_TRIANGLE;
    p.init_from_x = 0;
    p.update = LFM_UPDATE_RL;
    return p;
}

const char* lfm_last_error(void) { return g_err; }

const char* lfm_version(void) { return "lfm-b200 0.1 (sm_100a; frequency-domain polyphase RL + fp64 DCT entropy)"; }

lfm_status lfm_comm_unique_id(unsigned char* id_out) {
    if (!id_out) return fail(LFM_EINVAL, "id_out is NULL");
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(id_out, &id, 128);
    return LFM_OK;
}

lfm_status lfm_partition_model(double t_tc_ms, double mac_bytes, int direction, int num_sms, double mac_rate_scale,
                               int* tc_sms, double* predicted_ms) {
    g_err[0] = 0;
    if (!tc_sms) return fail(LFM_EINVAL, "tc_sms is NULL");
    if (t_tc_ms < 0 || mac_bytes < 0 || num_sms < 32 || (direction != 0 && direction != 1) || !(mac_rate_scale > 0) ||
        mac_rate_scale > 1)
        return fail(LFM_EINVAL, "lfm_partition_model: t_tc_ms, mac_bytes >= 0, direction 0/1, num_sms >= 32, "
                                "0 < mac_rate_scale <= 1");
    int s = 0;
    const double t = partition_time(t_tc_ms * 1e-3, mac_bytes, direction, num_sms, &s, mac_rate_scale);
    *tc_sms = s;
    if (predicted_ms) *predicted_ms = t * 1e3;
    return LFM_OK;
}

lfm_status lfm_tile_model(int nnum, int height, int width, int d1a, int d1b, int d2a, int d2b, int flags, int* L,
                          int* T1, int* T2, int* ntile, double* cost_unit, double* cost_whole) {
    g_err[0] = 0;
    if (!L || !T1 || !T2 || !ntile) return fail(LFM_EINVAL, "NULL argument");
    if (d1a > d1b || d2a > d2b) return fail(LFM_EINVAL, "tap ranges [%d, %d] x [%d, %d]", d1a, d1b, d2a, d2b);
    const int r = std::max(std::max(-d1a, d1b), std::max(-d2a, d2b));
    Geo g;
    ST(make_geo(nnum, 1, nnum * (2 * r + 1), nnum * (2 * r + 1), height, width, false, &g));
    const TileGeom t = choose_tiles(g, nnum * nnum, flags, d1a, d1b, d2a, d2b);
    *L = t.ntile ? t.L : 0;
    *T1 = t.ntile ? t.T1 : 0;
    *T2 = t.ntile ? t.T2 : 0;
    *ntile = t.ntile;
    if (cost_unit) *cost_unit = t.ntile ? tile_unit_cost(t, nnum * nnum) : 0.0;
    if (cost_whole) *cost_whole = whole_unit_cost(g, nnum * nnum);
    return LFM_OK;
}

lfm_status lfm_shard_units(int nz, int nnum, int world, int rank, int* unit_begin, int* unit_end) {
    g_err[0] = 0;
    if (!unit_begin || !unit_end) return fail(LFM_EINVAL, "NULL argument");
    if (nz < 1 || nnum < 1 || world < 1 || rank < 0 || rank >= world)
        return fail(LFM_EINVAL, "nz=%d nnum=%d world=%d rank=%d", nz, nnum, world, rank);
    unit_range(nz * nnum * nnum, world, rank, unit_begin, unit_end);
    return LFM_OK;
}

lfm_status lfm_plan_estimate(int nnum, int nz, int kh, int kw, int height, int width, int world, int flags,
                             size_t budget_bytes, size_t* bytes_per_gpu, char* limiting_term, size_t len) {
    g_err[0] = 0;
    if (!bytes_per_gpu) return fail(LFM_EINVAL, "bytes_per_gpu is NULL");
    if (world < 1) return fail(LFM_EINVAL, "world=%d", world);
    const bool direct = (flags & LFM_PLAN_DIRECT) != 0;
    Geo g;
    ST(make_geo(nnum, nz, kh, kw, height, width, direct, &g));
    const int nu_total = nz * nnum * nnum;
    int b, e;
    unit_range(nu_total, world, 0, &b, &e);   // rank 0 owns the largest share
    SizeTerms t = size_terms(g, e - b, nu_total, world, direct);
    *bytes_per_gpu = t.total();
    const char* names[6] = {"transfer matrices", "spectra workspaces", "volumes", "images", "PSF staging", "metric"};
    const size_t vals[6] = {t.transfer, t.spectra, t.volumes, t.images, t.staging, t.metric};
    int best = 0;
    for (int i = 1; i < 6; ++i)
        if (vals[i] > vals[best]) best = i;
    if (limiting_term && len) snprintf(limiting_term, len, "%s (%zu bytes)", names[best], vals[best]);
    if (budget_bytes > 0 && *bytes_per_gpu > budget_bytes)
        return fail(LFM_ENOMEM, "estimate %zu bytes per GPU exceeds budget %zu; limiting term: %s (%zu bytes)",
                    *bytes_per_gpu, budget_bytes, names[best], vals[best]);
    return LFM_OK;
}

lfm_status lfm_plan_create(lfm_plan* out, const float* psf_host, const float* psf_t_host, int nnum, int nz, int kh,
                           int kw, int height, int width, const lfm_optics* optics, const lfm_dist* dist, int flags,
                           void* stream) {
    g_err[0] = 0;
    const auto t_start = std::chrono::steady_clock::now();
    if (!out) return fail(LFM_EINVAL, "out is NULL");
    *out = nullptr;
    if (!psf_host) return fail(LFM_EINVAL, "psf_host is NULL");
    if (flags & LFM_PLAN_FRAMES) {   // built for frame batches: every plane on the frequency path
        if (flags & (LFM_PLAN_DIRECT | LFM_PLAN_DEVICE_LOOP | LFM_PLAN_GRAPHS))
            return fail(LFM_EINVAL, "LFM_PLAN_FRAMES excludes LFM_PLAN_DIRECT / _DEVICE_LOOP / _GRAPHS");
        flags |= LFM_PLAN_FFT_ONLY;
    }
    Geo g;
    ST(make_geo(nnum, nz, kh, kw, height, width, /*direct=*/false, &g));
    int rank = 0, world = 1;
    if (dist) {
        rank = dist->rank;
        world = dist->world;
        if (world < 1 || rank < 0 || rank >= world) return fail(LFM_EINVAL, "dist rank=%d world=%d", rank, world);
    }
    cudaStream_t s = as_stream(stream);
    lfm_plan p = new lfm_plan_s();
    auto guard = [&](lfm_status st) {
        if (st != LFM_OK) plan_free(p);
        return st;
    };
#define PG(call)                                  \
    do {                                          \
        lfm_status s__ = (call);                  \
        if (s__ != LFM_OK) return guard(s__);     \
    } while (0)
#define CKG(call)                                                                                           \
    do {                                                                                                    \
        cudaError_t e_ = (call);                                                                            \
        if (e_ != cudaSuccess)                                                                              \
            return guard(fail(LFM_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__)); \
    } while (0)
    p->geo = g;
    p->graphs = (flags & LFM_PLAN_GRAPHS) != 0;
    p->dloop = (flags & LFM_PLAN_DEVICE_LOOP) != 0;
    p->mac_tc_off = (flags & LFM_PLAN_NO_TC) != 0;
    p->rank = rank;
    p->world = world;
    p->nu_total = nz * nnum * nnum;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev);
    // ownership: cost-balanced contiguous unit ranges (every rank computes all of them from the full PSF), or the
    // even split with LFM_PLAN_EVEN_SHARDS
    p->rcut.assign(world + 1, 0);
    if (world > 1 && !(flags & LFM_PLAN_EVEN_SHARDS)) {
        for (size_t i = 0, n = (size_t)p->nu_total * kh * kw; i < n; ++i)
            if (!(psf_host[i] >= 0.0f)) return guard(fail(LFM_ENEG, "psf has a negative (or NaN) entry at unit %zu (S:192)", i / ((size_t)kh * kw)));
        p->rcut = balanced_cuts(plane_costs(psf_host, nnum, g, flags, p->num_sms), nnum * nnum, world);
    } else {
        for (int r = 0; r < world; ++r) unit_range(p->nu_total, world, r, &p->rcut[r], &p->rcut[r + 1]);
    }
    p->u0 = p->rcut[rank];
    p->u1 = p->rcut[rank + 1];
    p->nu = p->u1 - p->u0;
    p->nu_pad = (int)round_up((size_t)(p->nu > 0 ? p->nu : 1), 16);
    // PSF validation over the owned slice
    const size_t kk = (size_t)kh * kw;
    // "at least one nonzero kernel per z": a plane that projects nothing is rejected (whole stack, so every
    // rank reaches the same verdict; the scan stops at a plane's first nonzero entry)
    for (int z = 0; z < nz; ++z) {
        const float* hz = psf_host + (size_t)z * nnum * nnum * kk;
        size_t i = 0;
        const size_t n = (size_t)nnum * nnum * kk;
        while (i < n && hz[i] == 0.0f) ++i;
        if (i == n) return guard(fail(LFM_EZERO, "psf plane z=%d is all zero: it projects nothing (S:192)", z));
    }
    const float* psf_own = psf_host + (size_t)p->u0 * kk;
    for (size_t i = 0, n = (size_t)p->nu * kk; i < n; ++i)
        if (!(psf_own[i] >= 0.0f)) return guard(fail(LFM_ENEG, "psf has a negative (or NaN) entry at unit %zu (S:192)", p->u0 + i / kk));
    // backward kernels: the exact adjoint uses psf itself (C6); a supplied Ht enters as rot180(Ht) so that
    // H^T r (z,p,q) = sum_s r(s) Ht[z][p%N][q%N](p - s + c) runs through the same adjoint machinery
    std::vector<float> psfb_host;
    const float* psfb_own = psf_own;
    if (psf_t_host) {
        psfb_host.resize((size_t)p->nu * kk);
        const float* ht_own = psf_t_host + (size_t)p->u0 * kk;
        for (size_t uu = 0; uu < (size_t)p->nu; ++uu)
            for (int i = 0; i < kh; ++i)
                for (int j = 0; j < kw; ++j) {
                    const float v = ht_own[uu * kk + (size_t)(kh - 1 - i) * kw + (kw - 1 - j)];
                    if (!(v >= 0.0f)) return guard(fail(LFM_ENEG, "psf_t has a negative (or NaN) entry at unit %zu", p->u0 + uu));
                    psfb_host[uu * kk + (size_t)i * kw + j] = v;
                }
        psfb_own = psfb_host.data();
    }
    if (optics) {
        PG(make_region(optics, nnum, height, width, &p->region));
        p->has_optics = true;
        p->optics = *optics;
    }
    // memory budget ("estimate the required memory size"): everything but the transfer matrices must fit now;
    // the hybrid planner below fits the transfer matrices into what remains (moving planes to the direct path)
    size_t mem_budget = 0, nonM_bytes = 0;
    {
        SizeTerms t = size_terms(g, p->nu, p->nu_total, world, (flags & LFM_PLAN_DIRECT) != 0);
        size_t free_b = 0, total_b = 0;
        CKG(cudaMemGetInfo(&free_b, &total_b));
        mem_budget = g_mem_limit > 0 ? std::min(g_mem_limit, free_b) : free_b;
        nonM_bytes = t.total() - t.transfer;
        if (nonM_bytes > mem_budget) {
            const char* names[5] = {"spectra workspaces", "volumes", "images", "PSF staging", "metric"};
            const size_t vals[5] = {t.spectra, t.volumes, t.images, t.staging, t.metric};
            int best = 0;
            for (int i = 1; i < 5; ++i)
                if (vals[i] > vals[best]) best = i;
            return guard(fail(LFM_ENOMEM, "plan needs %zu bytes on this GPU besides transfer matrices, %zu available; "
                              "limiting term: %s (%zu bytes)", nonM_bytes, mem_budget, names[best], vals[best]));
        }
    }
    if ((world > 1 && !(flags & LFM_PLAN_NO_COMM)) || (flags & LFM_PLAN_FORCE_COMM)) {
        if (!dist) return guard(fail(LFM_EINVAL, "LFM_PLAN_FORCE_COMM needs an lfm_dist with an NCCL unique id"));
        ncclUniqueId id;
        memcpy(&id, dist->nccl_id, 128);
        ncclResult_t r = ncclCommInitRank(&p->nccl, world, id, rank);
        if (r != ncclSuccess) return guard(fail(LFM_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)));
        p->comm = true;
        if (flags & LFM_PLAN_SYMMETRIC) {   // C1 over an NCCL symmetric window (collective: every rank passes the flag)
            char e[256];
            const lfm_status ss = sym_create(p->nccl, (size_t)height * width, getenv("LFM_SYM_NO_MULTIMEM") ? 0 : 1,
                                             &p->sym, e, sizeof(e));
            if (ss != LFM_OK) return guard(fail(ss, "LFM_PLAN_SYMMETRIC: %s", e));
        }
    }
    // geometry for the kernels
    XformGeom& xg = p->xg;
    xg.N = nnum;
    xg.H = height;
    xg.W = width;
    xg.nh = g.nh;
    xg.nw = g.nw;
    xg.nz = nz;
    xg.Lh = g.Lh;
    xg.Lw = g.Lw;
    xg.nk2 = g.nk2;
    xg.nkappa = g.nkappa;
    xg.unit0 = p->u0;
    xg.nu = p->nu;
    xg.nu_pad = p->nu_pad;
    xg.kh = kh;
    xg.kw = kw;
    xg.ch = g.ch;
    xg.cw = g.cw;
    xg.umap = nullptr;
    p->xall = xg;
    const int N2 = nnum * nnum;
    const size_t HW = (size_t)height * width;
    const size_t vol = (size_t)p->nu * g.nh * g.nw;
    // buffers
    for (auto& x : p->xb) PG(dalloc(p, &x, vol * sizeof(float), "volume"));
    PG(dalloc(p, &p->norm, vol * sizeof(float), "normalizer"));
    PG(dalloc(p, &p->norm_sum, 4 * sizeof(double), "norm_sum"));
    if (p->comm) PG(dalloc(p, &p->xfull, (size_t)p->nu_total * g.nh * g.nw * sizeof(float), "gather volume"));
    PG(dalloc(p, &p->yhat, HW * sizeof(float), "yhat"));
    PG(dalloc(p, &p->rimg, HW * sizeof(float), "ratio image"));
    PG(dalloc(p, &p->mproj, HW * sizeof(unsigned), "max projection"));
    PG(dalloc(p, &p->partials, 3 * kParts * sizeof(double), "partials"));
    PG(dalloc(p, &p->stats, 4 * sizeof(double), "stats"));
    CKG(cudaMallocHost(&p->host, 16 * sizeof(double)));
    CKG(cudaEventCreate(&p->ev0));
    CKG(cudaEventCreate(&p->ev1));
    // PSF slice of the owned units -> device ("the PSF is evenly distributed to each card")
    PG(dalloc(p, &p->psf, (size_t)p->nu * kk * sizeof(float), "psf slice"));
    if (p->nu > 0) CKG(cudaMemcpyAsync(p->psf, psf_own, (size_t)p->nu * kk * sizeof(float), cudaMemcpyHostToDevice, s));
    p->psfb = p->psf;
    if (psf_t_host) {
        PG(dalloc(p, &p->psfb, (size_t)p->nu * kk * sizeof(float), "backward psf slice"));
        if (p->nu > 0)
            CKG(cudaMemcpyAsync(p->psfb, psfb_own, (size_t)p->nu * kk * sizeof(float), cudaMemcpyHostToDevice, s));
        CKG(cudaStreamSynchronize(s));   // psfb_host is read by the copy
    }

    // ---- hybrid plan: per plane, the tap box of its coarse kernels and a cost model pick the
    //      direct path (D x D taps per phase pair) or the frequency path (streamed transfer matrices)
    std::vector<int> plane_direct(nz, 0), plane_D(nz, 0);
    std::vector<double> pt_fft(nz, 0.0), pt_alt(nz, 1e30), pm_fft(nz, 0.0), pm_alt(nz, 0.0);
    std::vector<int> p_alt(nz, 0);   // best direct alternative per plane (1 CUDA-core, 2 tensor-core, 0 none)
    std::vector<AxisBox> box1(nz), box2(nz);
    const int zb = p->nu > 0 ? p->u0 / N2 : 0, ze = p->nu > 0 ? (p->u1 - 1) / N2 : -1;
    // frequency path: whole-image transforms, or overlap-save tiles (§5.6) with the window geometry of each plane's own
    // coarse-tap range (planes with equal ranges share a tile group)
    std::vector<TileGeom> ptile(nz);
    std::vector<double> pt_whole(nz, 0.0), pm_whole(nz, 0.0), pt_tile(nz, 0.0), pm_tile(nz, 0.0), pt_dir(nz, 1e30),
        pt_tc(nz, 1e30);
    std::vector<int> ptc_ok(nz, 0);
    bool too_big = false;
    for (int z = zb; z <= ze; ++z) {
        int k0 = kh, k1 = -1, j0 = kw, j1 = -1;
        const int ub = std::max(p->u0, z * N2), ue = std::min(p->u1, (z + 1) * N2);
        for (int u = ub; u < ue; ++u)
            for (int w = 0; w < (psf_t_host ? 2 : 1); ++w) {
                const float* ker = (w ? psfb_own : psf_own) + (size_t)(u - p->u0) * kk;
                for (int i = 0; i < kh; ++i)
                    for (int j = 0; j < kw; ++j)
                        if (ker[(size_t)i * kw + j] != 0.0f) {
                            k0 = std::min(k0, i);
                            k1 = std::max(k1, i);
                            j0 = std::min(j0, j);
                            j1 = std::max(j1, j);
                        }
            }
        if (k1 < 0) {   // all-zero owned kernels: a single (zero) tap
            k0 = k1 = g.ch;
            j0 = j1 = g.cw;
        }
        box1[z] = axis_box(nnum, g.ch, k0, k1);
        box2[z] = axis_box(nnum, g.cw, j0, j1);
        const int D = std::max(box1[z].D, box2[z].D);
        plane_D[z] = D;
        const double units = ue - ub;
        pt_whole[z] = units * whole_unit_cost(g, N2);
        pm_whole[z] = units * (double)g.nkappa * N2 * sizeof(float2) * (psf_t_host ? 2 : 1);
        ptile[z] = choose_tiles(g, N2, flags, box1[z].dmin, box1[z].dmax + box1[z].D - 1, box2[z].dmin,
                                box2[z].dmax + box2[z].D - 1);
        if (ptile[z].ntile) {
            pt_tile[z] = units * tile_unit_cost(ptile[z], N2);
            pm_tile[z] = units * (double)ptile[z].L * (ptile[z].L / 2 + 1) * (N2 + round_up((size_t)N2, 4)) * 8.0;
        }
        const double t_dir = D <= kDirMaxD ? 2.0 * units * N2 * D * D * (double)g.nh * g.nw * 2.0 / kDirFlops[D] : 1e30;
        // tensor-core direct (kernels_tcdir.cu): per direction, CTA pairs over 256-pixel tiles of the padded grid,
        // every tap x K-step = 3 pair MMAs of Ntile/2 cycles (tcgen05 floor), at the measured efficiency
        const int T1 = box1[z].dmax - box1[z].dmin + box1[z].D, T2 = box2[z].dmax - box2[z].dmin + box2[z].D;
        const int Ntile = (int)round_up((size_t)N2, 16);
        const bool tc_ok = !(flags & LFM_PLAN_NO_TC) && Ntile <= 256 && T2 <= 65;
        const double t_tc = tc_ok ? tc_plane_time(box1[z], box2[z], g, N2, p->num_sms) : 1e30;   // whole plane
        pt_dir[z] = t_dir;
        pt_tc[z] = t_tc;
        ptc_ok[z] = tc_ok;
        // device bytes per plane on each path (memory-aware planning below)
        if (tc_ok && t_tc <= t_dir) {
            p_alt[z] = 2;
            pt_alt[z] = t_tc;
            const double lp = (double)g.nh * (g.nw + T2 - 1);
            pm_alt[z] = (double)T1 * T2 * ((N2 + 63) / 64) * 2 * Ntile * 64 * 2 * 2 + 2.0 * ((N2 + 63) / 64) * lp * 128 +
                        2.0 * height * width * 4;
        } else if (D <= kDirMaxD) {
            p_alt[z] = 1;
            pt_alt[z] = t_dir;
            pm_alt[z] = 2.0 * units * D * D * N2 * 4 + (double)height * width * 4;
        }
    }
    // tiles when every owned plane has a tiling and (LFM_PLAN_TILES, or the tiles beat whole-image transforms by 10 %
    // over the owned planes)
    bool use_tiles = zb <= ze;
    {
        double sw = 0.0, st = 0.0;
        for (int z = zb; z <= ze; ++z) {
            use_tiles &= ptile[z].ntile > 0;
            sw += pt_whole[z];
            st += pt_tile[z];
        }
        if (use_tiles && !(flags & LFM_PLAN_TILES) && !(st < 0.9 * sw)) use_tiles = false;
    }
    for (int z = zb; z <= ze; ++z) {
        pt_fft[z] = use_tiles ? pt_tile[z] : pt_whole[z];
        pm_fft[z] = use_tiles ? pm_tile[z] : pm_whole[z];
        int mode = 0;                            // 0 FFT, 1 SIMT direct, 2 tensor-core direct
        if (flags & LFM_PLAN_FFT_ONLY) {
            mode = 0;
        } else if (flags & LFM_PLAN_DIRECT) {
            mode = (flags & LFM_PLAN_TC_DIRECT) && ptc_ok[z] ? 2 : 1;
        } else {
            const double best = std::min(pt_fft[z], std::min(pt_dir[z], pt_tc[z]));
            mode = best == pt_fft[z] ? 0 : (best == pt_tc[z] ? 2 : 1);
        }
        plane_direct[z] = mode;
        if (mode == 1 && plane_D[z] > kDirMaxD) too_big = true;
    }
    // memory-aware planning: while the frequency-path planes' transfer matrices do not fit, move the plane whose
    // direct alternative costs the least extra time per byte saved
    p->mem_moved = 0;
    if (!(flags & (LFM_PLAN_FFT_ONLY | LFM_PLAN_DIRECT))) {
        auto need = [&]() {
            double b = 0;
            for (int z = zb; z <= ze; ++z) b += plane_direct[z] == 0 ? pm_fft[z] : pm_alt[z];
            return b;
        };
        const double avail = 0.94 * (double)(mem_budget - nonM_bytes);
        while (need() > avail) {
            int best = -1;
            double best_r = 1e300;
            for (int z = zb; z <= ze; ++z) {
                if (plane_direct[z] != 0 || p_alt[z] == 0 || pm_fft[z] <= pm_alt[z]) continue;
                const double r = (pt_alt[z] - pt_fft[z]) / (pm_fft[z] - pm_alt[z]);
                if (r < best_r) {
                    best_r = r;
                    best = z;
                }
            }
            if (best < 0) break;
            plane_direct[best] = p_alt[best];
            ++p->mem_moved;
        }
        if (need() > avail)
            return guard(fail(LFM_ENOMEM, "transfer matrices of the frequency-path planes need %.0f bytes, %.0f available "
                              "after moving %d planes to the direct path; limiting term: transfer matrices",
                              need(), avail, p->mem_moved));
    }
    // partition-aware refinement (§5.5): side by side on SM partitions a tensor-core plane costs SM time (its
    // whole-GPU time spread over the tensor-core partition), a frequency-path plane only its transfer bytes at a
    // partition SM's streaming rate -- far below the whole-GPU HBM rate the per-plane choice above assumed.  Planes
    // with the most tensor time per transfer byte move back to the frequency path while the predicted partitioned
    // iteration (both directions, partition_time, plus the coarse transforms of the added units) keeps improving and
    // the transfer matrices fit.
    p->part_moved = 0;
    // (LFM_PLAN_MOVE, dev: force the number of moved planes -- also without partitions, so that a serial profiling
    //  run sees the plane assignment of the partitioned plan)
    if ((partitions_allowed(flags) || getenv("LFM_PLAN_MOVE")) && !use_tiles &&
        !(flags & (LFM_PLAN_FFT_ONLY | LFM_PLAN_DIRECT | LFM_PLAN_NO_TC))) {
        bool simt = false;
        for (int z = zb; z <= ze; ++z) simt |= plane_direct[z] == 1;
        std::vector<int> cand;
        for (int z = zb; z <= ze; ++z)
            if (plane_direct[z] == 2 && pm_fft[z] > 0) cand.push_back(z);
        std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) { return pt_alt[a] / pm_fft[a] > pt_alt[b] / pm_fft[b]; });
        auto predict = [&](int k) {   // predicted seconds per iteration with the first k candidates on the FFT path
            double t_tc = 0.0, units_fft = 0.0;
            std::vector<int> mode(plane_direct);
            for (int i = 0; i < k; ++i) mode[cand[i]] = 0;
            for (int z = zb; z <= ze; ++z) {
                const double units = std::min<long long>(p->u1, (long long)(z + 1) * N2) - std::max<long long>(p->u0, (long long)z * N2);
                if (mode[z] == 2) t_tc += 0.5 * pt_alt[z];
                if (mode[z] == 0) units_fft += units;
            }
            const double bytes = units_fft * N2 * g.nkappa * 8.0;
            double t = kXformPerUnit * units_fft;
            for (int d = 0; d < 2; ++d) {
                const double gsm = round_up((size_t)std::max(units_fft, 1.0), 16) * 8.0 + 1024.0;
                const double scale = d == 0 ? std::min(4.0, std::floor(228.0 * 1024.0 / gsm)) / 4.0 : 1.0;
                int sdummy = 0;
                t += partition_time(t_tc, bytes, d, p->num_sms, &sdummy, scale);
            }
            double mem = 0;
            for (int z = zb; z <= ze; ++z) mem += mode[z] == 0 ? pm_fft[z] : pm_alt[z];
            return mem <= 0.94 * (double)(mem_budget - nonM_bytes) ? t : 1e30;
        };
        int best_k = 0;
        if (!simt && !cand.empty()) {
            double best_t = predict(0);
            for (int k = 1; k <= (int)cand.size(); ++k) {
                const double t = predict(k);
                if (t < best_t * 0.95) {   // the model's error is ~10 %: move only on a clear predicted gain
                    best_t = t;
                    best_k = k;
                }
            }
            if (const char* ev = getenv("LFM_PLAN_MOVE")) best_k = std::max(0, std::min((int)cand.size(), atoi(ev)));   // dev
            if (getenv("LFM_PLAN_VERBOSE"))
                fprintf(stderr, "[lfm plan] partition-aware: %d of %zu tensor-core planes to the frequency path "
                                "(predicted %.3f -> %.3f ms per iteration)\n",
                        best_k, cand.size(), predict(0) * 1e3, predict(best_k) * 1e3);
        }
        for (int i = 0; i < best_k; ++i) plane_direct[cand[i]] = 0;
        p->part_moved = best_k;
    }
    p->direct = too_big;   // all-direct request with boxes beyond kDirMaxD: the generic spatial kernels
    if (!p->direct) {
        // FFT units through a unit map (z-major order kept)
        std::vector<int> umap;
        for (int u = p->u0; u < p->u1; ++u)
            if (plane_direct[u / N2] == 0) umap.push_back(u - p->u0);
        p->nu_fft = (int)umap.size();
        p->nu_fft_pad = (int)round_up((size_t)std::max(p->nu_fft, 1), 16);
        if (p->nu_fft > 0) {
            PG(dalloc(p, &p->umap, umap.size() * sizeof(int), "unit map"));
            CKG(cudaMemcpyAsync(p->umap, umap.data(), umap.size() * sizeof(int), cudaMemcpyHostToDevice, s));
        }
        xg.nu = p->nu_fft;
        xg.nu_pad = p->nu_fft_pad;
        xg.umap = p->umap;
        // direct planes grouped by box size; taps g_z[b'][a][e] = h_{z,a}[b - a + c + N (dlo + e)] (both layouts)
        size_t coef_bytes = 0;
        for (int D = 1; D <= kDirMaxD; ++D) {
            std::vector<int> zl;
            for (int z = zb; z <= ze; ++z)
                if (plane_direct[z] == 1 && plane_D[z] == D) zl.push_back(z);
            if (zl.empty()) continue;
            const int nzd = (int)zl.size(), DD = D * D;
            std::vector<float> cf((size_t)nzd * N2 * DD * N2, 0.0f), cb((size_t)nzd * N2 * DD * N2, 0.0f);
            std::vector<int> dl((size_t)nzd * 2 * N2);
            DirArgs da{};
            da.dmin1 = da.dmin2 = 1 << 30;
            da.dmax1 = da.dmax2 = -(1 << 30);
            for (int zi = 0; zi < nzd; ++zi) {
                const int z = zl[zi];
                const AxisBox& B1 = box1[z];
                const AxisBox& B2 = box2[z];
                da.dmin1 = std::min(da.dmin1, B1.dmin);
                da.dmax1 = std::max(da.dmax1, B1.dmax);
                da.dmin2 = std::min(da.dmin2, B2.dmin);
                da.dmax2 = std::max(da.dmax2, B2.dmax);
                for (int q = 0; q < N2; ++q) {
                    dl[((size_t)zi * 2 + 0) * N2 + q] = B1.dlo[q];
                    dl[((size_t)zi * 2 + 1) * N2 + q] = B2.dlo[q];
                }
                for (int a = 0; a < N2; ++a) {
                    const int u = z * N2 + a;
                    if (u < p->u0 || u >= p->u1) continue;
                    const int a1 = a / nnum, a2 = a % nnum;
                    const float* ker = psf_host + (size_t)u * kk;
                    const float* kerb = psfb_own + (size_t)(u - p->u0) * kk;
                    for (int bq = 0; bq < N2; ++bq) {
                        const int b1 = bq / nnum, b2 = bq % nnum;
                        const int o1 = B1.dlo[(size_t)a1 * nnum + b1], o2 = B2.dlo[(size_t)a2 * nnum + b2];
                        for (int e1 = 0; e1 < D; ++e1) {
                            const int k1 = b1 - a1 + g.ch + nnum * (o1 + e1);
                            if (k1 < 0 || k1 >= kh) continue;
                            for (int e2 = 0; e2 < D; ++e2) {
                                const int k2 = b2 - a2 + g.cw + nnum * (o2 + e2);
                                if (k2 < 0 || k2 >= kw) continue;
                                cf[(((size_t)zi * N2 + a) * DD + e1 * D + e2) * N2 + bq] = ker[(size_t)k1 * kw + k2];
                                cb[(((size_t)zi * N2 + bq) * DD + e1 * D + e2) * N2 + a] = kerb[(size_t)k1 * kw + k2];
                            }
                        }
                    }
                }
            }
            int* dz = nullptr;
            float *dcf = nullptr, *dcb = nullptr;
            int* ddl = nullptr;
            PG(dalloc(p, &dz, zl.size() * sizeof(int), "direct plane list"));
            p->dallocs.push_back(dz);
            PG(dalloc(p, &dcf, cf.size() * sizeof(float), "direct taps (forward layout)"));
            p->dallocs.push_back(dcf);
            PG(dalloc(p, &dcb, cb.size() * sizeof(float), "direct taps (backward layout)"));
            p->dallocs.push_back(dcb);
            PG(dalloc(p, &ddl, dl.size() * sizeof(int), "direct box origins"));
            p->dallocs.push_back(ddl);
            CKG(cudaMemcpyAsync(dz, zl.data(), zl.size() * sizeof(int), cudaMemcpyHostToDevice, s));
            CKG(cudaMemcpyAsync(dcf, cf.data(), cf.size() * sizeof(float), cudaMemcpyHostToDevice, s));
            CKG(cudaMemcpyAsync(dcb, cb.data(), cb.size() * sizeof(float), cudaMemcpyHostToDevice, s));
            CKG(cudaMemcpyAsync(ddl, dl.data(), dl.size() * sizeof(int), cudaMemcpyHostToDevice, s));
            CKG(cudaStreamSynchronize(s));   // host vectors die at the end of this scope
            da.N = nnum;
            da.H = height;
            da.W = width;
            da.nh = g.nh;
            da.nw = g.nw;
            da.unit0 = p->u0;
            da.nu = p->nu;
            da.nzd = nzd;
            da.zlist = dz;
            da.D = D;
            da.coef_f = dcf;
            da.coef_b = dcb;
            da.dlo = ddl;
            p->dgroups.push_back(da);
            p->n_direct_planes += nzd;
            coef_bytes += 2 * cf.size() * sizeof(float);
        }
        // §5.5: with planes on both the tensor cores and the frequency path, each projection runs its two halves side
        // by side on disjoint SM partitions (green contexts) when the cost model says that beats running them one after
        // the other; the tensor-core schedule of each direction is laid out for its partition
        int tc_sms[2] = {p->num_sms, p->num_sms};
        if (partitions_allowed(flags)) {
            double t_tc = 0.0, units_fft = 0.0;
            int nsimt = 0;
            for (int z = zb; z <= ze; ++z) {
                const double units = std::min<long long>(p->u1, (long long)(z + 1) * N2) - std::max<long long>(p->u0, (long long)z * N2);
                if (plane_direct[z] == 2) t_tc += 0.5 * pt_alt[z];   // per direction
                if (plane_direct[z] == 0) units_fft += units;
                nsimt += plane_direct[z] == 1;
            }
            const double bytes = units_fft * N2 * g.nkappa * 8.0;   // M streamed once per direction
            // tiled frequency path (§5.6): its MAC (tensor cores, HBM-bound), transforms (SIMT) and the tensor-core
            // direct planes share the SMs in proportion to their modelled whole-GPU times (r02 c3 sweeps: the
            // proportional split, rounded to the driver's 8-SM steps, was the best step)
            double t_f = 0.0;   // per direction, the tiled frequency-path planes
            for (int z = zb; z <= ze; ++z)
                if (plane_direct[z] == 0) t_f += 0.5 * pt_fft[z];
            for (int d = 0; d < 2 && use_tiles && t_tc > 0 && units_fft > 0 && nsimt == 0; ++d) {
                // live beside the backward tile half (MAC + C2R / update) the tcgen05 backward runs slower than its
                // forward twin, which the whole-GPU model does not see (r02, c3 on 24 SMs: 1.70 vs 1.38 ms; c2 on 32:
                // 0.098 vs 0.070 ms; serialised on the whole GPU both 0.24 ms): weight its share accordingly (c3: the
                // backward partition 24 -> 32 SMs, 281 -> 288 it/s on one box)
                const double ttc = d ? kTcBwdLive * t_tc : t_tc;
                const double raw = p->num_sms * ttc / (ttc + t_f);
                // a small tensor-core share is not worth a partition: the tile half then loses more on its fewer SMs
                // than the overlap gains (c4, share 0.02: 38.4 it/s one after the other vs 36.0 on a forced 16-SM
                // partition; c3 forward, share 0.16: 298.5 it/s one after the other vs 291.4 partitioned, with the
                // backward (0.20) partitioned in both; c2, shares 0.22 / 0.26: 2163 partitioned vs 1841 not)
                int want = raw < kPartMinShare * p->num_sms ? 0 : (int)std::lround(raw / 8.0) * 8;
                if (want) want = std::max(16, std::min(p->num_sms - 16, want));
                if (const char* ev = getenv(d ? "LFM_TC_SMS_B" : "LFM_TC_SMS_F")) want = atoi(ev);   // dev override
                if (getenv("LFM_PLAN_VERBOSE"))
                    fprintf(stderr, "[lfm plan] tiles, direction %d: t_tc %.3f ms, t_freq %.3f ms -> %d tc SMs\n", d,
                            ttc * 1e3, t_f * 1e3, want);
                if (want > 0 && green_split(p, dev, want, &p->part[d])) tc_sms[d] = p->part[d].sms_tc;
            }
            for (int d = 0; d < 2 && !use_tiles && t_tc > 0 && bytes > 0 && nsimt == 0; ++d) {
                // the partition's forward MAC keeps four 8-warp CTAs per SM in flight while G[kappa] fits four times in
                // shared memory; fewer resident CTAs stream proportionally less (c4: 3 CTAs, ~81 GB/s per SM)
                const double gsm = round_up((size_t)std::max(units_fft, 1.0), 16) * 8.0 + 1024.0;
                const double scale = d == 0 ? std::min(4.0, std::floor(228.0 * 1024.0 / gsm)) / 4.0 : 1.0;
                const int want = choose_partition(t_tc, bytes, d, p->num_sms, scale);
                if (want > 0 && green_split(p, dev, want, &p->part[d])) tc_sms[d] = p->part[d].sms_tc;
            }
        }
        // tensor-core direct planes: one merged launch per direction (LPT schedule over (plane, tile) items)
        {
            std::vector<int> zl, d1a, d1b, d2a, d2b;
            for (int z = zb; z <= ze; ++z)
                if (plane_direct[z] == 2) {
                    zl.push_back(z);
                    d1a.push_back(box1[z].dmin);
                    d1b.push_back(box1[z].dmax + box1[z].D - 1);
                    d2a.push_back(box2[z].dmin);
                    d2b.push_back(box2[z].dmax + box2[z].D - 1);
                }
            if (!zl.empty()) {
                TcDirArgs ta{};
                ta.N = nnum;
                ta.H = height;
                ta.W = width;
                ta.nh = g.nh;
                ta.nw = g.nw;
                ta.unit0 = p->u0;
                ta.nu = p->nu;
                ta.nzd = (int)zl.size();
                int* dz = nullptr;
                PG(dalloc(p, &dz, zl.size() * sizeof(int), "tc plane list"));
                p->dallocs.push_back(dz);
                CKG(cudaMemcpyAsync(dz, zl.data(), zl.size() * sizeof(int), cudaMemcpyHostToDevice, s));
                ta.zlist = dz;
                TcDirArgs tb = ta;
                for (int w = 0; w < 2; ++w) {
                    TcDirArgs& t = w ? tb : ta;
                    std::vector<TcPlane> pls;
                    if (!tcdir_geometry(&t, !w, d1a.data(), d1b.data(), d2a.data(), d2b.data(), &pls, tc_sms[w]))
                        return guard(fail(LFM_EUNSUPPORTED, "tensor-core direct path needs Nnum^2 <= 256"));
                    uint16_t *cf = nullptr, *sr = nullptr;
                    float* pt = nullptr;
                    int* nzf = nullptr;
                    unsigned* am = nullptr;
                    const size_t nf = tcdir_coef_elems(t, pls), ns = tcdir_src_elems(t, !w), np = tcdir_part_floats(t, !w);
                    size_t ntile = 0;
                    for (const TcPlane& pl : pls) ntile += (size_t)pl.T1 * pl.T2 * t.nch;
                    PG(dalloc(p, &cf, nf * sizeof(uint16_t), "tc direct taps"));
                    p->dallocs.push_back(cf);
                    PG(dalloc(p, &sr, ns * sizeof(uint16_t), "tc direct staged source"));
                    p->dallocs.push_back(sr);
                    PG(dalloc(p, &am, ((size_t)t.nzd + 1) * sizeof(unsigned), "tc operand maxima"));
                    p->dallocs.push_back(am);
                    t.amax = am;   // [0]: the staged source's max (per launch); [1 + zi]: plane maxima (plan time)
                    {   // fp16 scale of each plane's coefficient tiles from its largest tap
                        CKG(cudaMemsetAsync(am, 0, ((size_t)t.nzd + 1) * sizeof(unsigned), s));
                        CKG(launch_tc_plane_amax(w ? p->psfb : p->psf, dz, t.nzd, N2, (int)kk, p->u0, p->nu, am + 1, s));
                        std::vector<unsigned> pm(t.nzd);
                        CKG(cudaMemcpyAsync(pm.data(), am + 1, t.nzd * sizeof(unsigned), cudaMemcpyDeviceToHost, s));
                        CKG(cudaStreamSynchronize(s));
                        for (int zi = 0; zi < t.nzd; ++zi) {
                            float f;
                            memcpy(&f, &pm[zi], sizeof(f));
                            pls[zi].bexp = tc::f16_scale_exp(f);
                        }
                    }
                    if (np) {
                        PG(dalloc(p, &pt, np * sizeof(float), "tc direct forward partials"));
                        p->dallocs.push_back(pt);
                    }
                    PG(dalloc(p, &nzf, ntile * sizeof(int), "tc tile flags"));
                    t.coef = cf;
                    t.src = sr;
                    t.part = pt;
                    // coefficient tiles + nonzero flags -> windows that can be skipped (edge tap rows x chunks)
                    for (int zi = 0; zi < t.nzd; ++zi)
                        CKG(launch_tcdir_coef(t, pls[zi], zi, zl[zi], w ? p->psfb : p->psf, kh, kw, g.ch, g.cw, !w, cf,
                                              nzf + pls[zi].coef_off / 2, s));
                    std::vector<int> flags_h(ntile), rowmask;
                    CKG(cudaMemcpyAsync(flags_h.data(), nzf, ntile * sizeof(int), cudaMemcpyDeviceToHost, s));
                    CKG(cudaStreamSynchronize(s));
                    cudaFree(nzf);
                    tcdir_window_masks(t, &pls, flags_h, &rowmask);
                    std::vector<int> ranges;
                    tcdir_ranges(t, flags_h, &ranges);
                    if (getenv("LFM_PLAN_VERBOSE")) {
                        double sn = 0, nzt = 0;
                        for (int r : ranges)
                            if (r) {
                                sn += r >> 16;
                                ++nzt;
                            }
                        fprintf(stderr, "[lfm plan] tc %s: %zu tiles, %.0f nonzero, mean MMA width %.1f of %d\n",
                                w ? "bwd" : "fwd", ranges.size(), nzt, nzt > 0 ? sn / nzt : 0.0, t.Ntile);
                    }
                    int* drg = nullptr;
                    PG(dalloc(p, &drg, ranges.size() * sizeof(int), "tc column ranges"));
                    p->dallocs.push_back(drg);
                    CKG(cudaMemcpyAsync(drg, ranges.data(), ranges.size() * sizeof(int), cudaMemcpyHostToDevice, s));
                    t.trange = drg;
                    std::vector<int> ioff, items;
                    tcdir_schedule(t, pls, &ioff, &items);
                    TcPlane* dpl = nullptr;
                    int *dio = nullptr, *dit = nullptr, *drm = nullptr;
                    PG(dalloc(p, &dpl, pls.size() * sizeof(TcPlane), "tc plane records"));
                    p->dallocs.push_back(dpl);
                    PG(dalloc(p, &drm, rowmask.size() * sizeof(int), "tc window masks"));
                    p->dallocs.push_back(drm);
                    PG(dalloc(p, &dio, ioff.size() * sizeof(int), "tc schedule"));
                    p->dallocs.push_back(dio);
                    PG(dalloc(p, &dit, items.size() * sizeof(int), "tc schedule"));
                    p->dallocs.push_back(dit);
                    CKG(cudaMemcpyAsync(dpl, pls.data(), pls.size() * sizeof(TcPlane), cudaMemcpyHostToDevice, s));
                    CKG(cudaMemcpyAsync(drm, rowmask.data(), rowmask.size() * sizeof(int), cudaMemcpyHostToDevice, s));
                    CKG(cudaMemcpyAsync(dio, ioff.data(), ioff.size() * sizeof(int), cudaMemcpyHostToDevice, s));
                    CKG(cudaMemcpyAsync(dit, items.data(), items.size() * sizeof(int), cudaMemcpyHostToDevice, s));
                    t.planes = dpl;
                    t.rowmask = drm;
                    t.item_off = dio;
                    t.items = dit;
                    CKG(tcdir_encode(&t, !w));
                    CKG(cudaStreamSynchronize(s));   // host vectors die at the end of this scope
                    coef_bytes += nf * sizeof(uint16_t);
                    if (!w)   // executed tensor flops of one projection: 3 pair MMAs (K = 16) per K-step of every nonzero window
                              // tap, over the tile's column range
                        for (size_t zi = 0; zi < pls.size(); ++zi) {
                            const TcPlane& pl = pls[zi];
                            double col_ks = 0;
                            int gk = 0;
                            for (int c = 0; c < t.nch; ++c)
                                for (int t1 = 0; t1 < pl.T1; ++t1) {
                                    if (!((rowmask[pl.mask_off + t1] >> c) & 1)) continue;
                                    for (int t2 = 0; t2 < pl.T2; ++t2) {
                                        const int ks = c == t.nch - 1 ? t.kst_last : 4;
                                        const int rg = ranges[(size_t)pl.coef_off / 2 + (size_t)(t1 * pl.T2 + t2) * t.nch + c];
                                        col_ks += (double)ks * (rg >> 16);
                                        gk += ks;
                                        if ((c * pl.T1 + t1 == pl.last_win && t2 == pl.T2 - 1) || gk + 4 > t.chain_k) gk = 0;
                                    }
                                }
                            p->tc_flops_exec += (double)t.tiles * col_ks * 3.0 * 2.0 * 256.0 * 16.0;
                            p->tc_active_frac += (double)pl.active_windows / (pl.T1 * t.nch) / pls.size();
                            const int z = zl[zi];
                            p->tc_flops_alg += 2.0 * (double)N2 * N2 * box1[z].D * box2[z].D * g.nh * g.nw;
                        }
                }
                p->tcf.push_back(ta);
                p->tcb.push_back(tb);
                p->n_tc_planes += ta.nzd;
                p->n_direct_planes += ta.nzd;
            }
        }
        p->transfer_bytes = coef_bytes;
        int maxg = 0;
        for (const DirArgs& dg : p->dgroups) maxg = std::max(maxg, dg.nzd);
        if (maxg > 0) PG(dalloc(p, &p->dpart, (size_t)maxg * HW * sizeof(float), "direct forward partials"));
        if (p->nu_fft > 0 && use_tiles) {
            // §5.6: one tile group per coarse-tap range of the frequency-path planes (z order kept inside a group)
            CKG(tile_fft_init());
            p->tiled = true;
            p->bpitch = (int)round_up((size_t)N2, 4);
            const std::vector<int>& umap_h = umap;   // the host unit map (the device copy may still be in flight on s)
            std::vector<int> gz;                 // first plane of each group (its tile geometry)
            std::vector<std::vector<int>> gunits;
            for (int t = 0; t < p->nu_fft; ++t) {
                const int z = (p->u0 + umap_h[t]) / N2;
                size_t gi = 0;
                for (; gi < gz.size(); ++gi) {
                    const TileGeom& a = ptile[gz[gi]];
                    const TileGeom& b = ptile[z];
                    if (a.dmin1 == b.dmin1 && a.dmax1 == b.dmax1 && a.dmin2 == b.dmin2 && a.dmax2 == b.dmax2) break;
                }
                if (gi == gz.size()) {
                    gz.push_back(z);
                    gunits.emplace_back();
                }
                gunits[gi].push_back(umap_h[t]);
            }
            p->tgs.resize(gz.size());
            for (size_t gi = 0; gi < gz.size(); ++gi)
                PG(build_tile_group(p, p->tgs[gi], ptile[gz[gi]], gunits[gi], xg, psf_t_host != nullptr, s));
        } else if (p->nu_fft > 0) {
            // whole-image transforms (Lh x Lw)
            const int Lh = g.Lh, Lw = g.Lw, nkap = g.nkappa;
            if (!fft_factor(Lh, &p->fh) || !fft_factor(Lw, &p->fw))
                return guard(fail(LFM_EUNSUPPORTED, "coarse transform sizes %dx%d are not 5-smooth", Lh, Lw));
            PG(twiddles(Lh, &p->tw_h, p, s));
            PG(twiddles(Lw, &p->tw_w, p, s));
            const size_t mbytes = (size_t)nkap * N2 * p->nu_fft_pad * sizeof(float2);
            p->transfer_bytes += mbytes;
            PG(dalloc(p, &p->M, mbytes, "transfer matrices"));
            PG(dalloc(p, &p->G, (size_t)nkap * p->nu_fft_pad * sizeof(float2), "G spectra"));
            PG(dalloc(p, &p->Xh, (size_t)nkap * p->nu_fft_pad * sizeof(float2), "Xh spectra"));
            PG(dalloc(p, &p->Y, (size_t)nkap * N2 * sizeof(float2), "Y spectra"));
            PG(dalloc(p, &p->R, (size_t)nkap * N2 * sizeof(float2), "R spectra"));
            CKG(cudaMemsetAsync(p->M, 0, mbytes, s));      // padding columns stay zero
            CKG(cudaMemsetAsync(p->G, 0, (size_t)nkap * p->nu_fft_pad * sizeof(float2), s));
            // K1: transfer matrices M[kappa][b'][t] = DFT_{Lh x Lw}(g_{u(t),b'}), g_{u,b'}[d] = h_u[b' - a + c + N d]
            R2CArgs a = r2c_args(SRC_KERNEL, p->psf, nullptr, 0.f, N2 * p->nu_fft, p->M, (long long)N2 * p->nu_fft_pad);
            a.cdiv = p->nu_fft;
            a.cmul = p->nu_fft_pad;
            CKG(launch_r2c(xg, p->fh, p->fw, p->tw_h, p->tw_w, a, s));
            p->Mb = p->M;
            if (psf_t_host) {   // second set of transfer matrices from rot180(Ht)
                p->transfer_bytes += mbytes;
                PG(dalloc(p, &p->Mb, mbytes, "backward transfer matrices"));
                CKG(cudaMemsetAsync(p->Mb, 0, mbytes, s));
                R2CArgs ab = r2c_args(SRC_KERNEL, p->psfb, nullptr, 0.f, N2 * p->nu_fft, p->Mb, (long long)N2 * p->nu_fft_pad);
                ab.cdiv = p->nu_fft;
                ab.cmul = p->nu_fft_pad;
                CKG(launch_r2c(xg, p->fh, p->fw, p->tw_h, p->tw_w, ab, s));
            }
            p->fft_alg_bytes = (double)g.nkappa * N2 * p->nu_fft * 8.0 + (double)g.nkappa * (p->nu_fft + N2) * 8.0;
        }
        CKG(cudaStreamSynchronize(s));
        if (p->psfb != p->psf) {
            cudaFree(p->psfb);
            p->bytes -= (size_t)p->nu * kk * sizeof(float);
        }
        cudaFree(p->psf);           // transfer matrices and direct taps replace the PSF
        p->bytes -= (size_t)p->nu * kk * sizeof(float);
        p->psf = nullptr;
        p->psfb = nullptr;
    } else {
        p->transfer_bytes = (size_t)p->nu * kk * sizeof(float);
    }
    // normalizer H^T 1, polyphase, and its global sum (for c0 = sum y / sum H^T 1, reading C2)
    PG(op_backward(p, SRC_ONES, nullptr, nullptr, 1.0f, DST_POLY, p->norm, nullptr, s));
    CKG(launch_sum_stats(p->norm, vol, p->partials, kParts, p->stats, s));
    CKG(cudaMemcpyAsync(p->norm_sum, p->stats, sizeof(double), cudaMemcpyDeviceToDevice, s));
    PG(allreduce(p, p->norm_sum, 1, ncclDouble, ncclSum, s));
    if (p->has_optics) PG(metric_alloc(&p->met, p->region, height, width, s, &p->bytes));
    CKG(cudaMemcpyAsync(p->host, p->norm_sum, sizeof(double), cudaMemcpyDeviceToHost, s));
    CKG(cudaStreamSynchronize(s));
    // c0 = sum y / sum H^T 1 (reading C2) needs sum H^T 1 > 0 (LFM_EZERO: "a PSF that projects nothing", lfm.h)
    if (!(p->host[0] > 0.0) || !std::isfinite(p->host[0]))
        return guard(fail(LFM_EZERO, "sum of H^T 1 = %g: the PSF projects nothing onto this %dx%d image", p->host[0],
                          height, width));
    if (flags & LFM_PLAN_FRAMES) {
        // after every single-frame use of M (the normalizer above): the transposed copy for the backward pass, then
        // both split in place into scaled fp16 hi / lo rows
        if (p->nu_fft <= 0 || N2 > 256) return guard(fail(LFM_EUNSUPPORTED, "LFM_PLAN_FRAMES needs frequency-path units and N^2 <= 256"));
        p->bpitch = (int)round_up((size_t)N2, 4);
        const size_t mtb = (size_t)g.nkappa * p->nu_fft_pad * p->bpitch * sizeof(float2);
        PG(dalloc(p, &p->MT, mtb, "transposed transfer matrices (LFM_PLAN_FRAMES)"));
        p->transfer_bytes += mtb;
        PG(dalloc(p, &p->mf_eb, 64 * sizeof(int), "frame scales"));
        CKG(mac_f16_prepare(p->M, p->Mb, p->MT, g.nkappa, N2, p->nu_fft_pad, p->bpitch, &p->mf_fwd, &p->mf_bwd, s));
        if (p->Mb != p->M) {   // a supplied Ht: its matrices live on only as the transposed copy
            cudaFree(p->Mb);
            p->bytes -= (size_t)g.nkappa * N2 * p->nu_fft_pad * sizeof(float2);
            p->transfer_bytes -= (size_t)g.nkappa * N2 * p->nu_fft_pad * sizeof(float2);
        }
        p->Mb = nullptr;
        p->frames = true;
    }
    p->plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    *out = p;
    return LFM_OK;
#undef PG
#undef CKG
}

lfm_status lfm_shard_units_balanced(const float* psf_host, int nnum, int nz, int kh, int kw, int height, int width,
                                    int world, int rank, int flags, int* unit_begin, int* unit_end, double* est_seconds) {
    g_err[0] = 0;
    if (!psf_host || !unit_begin || !unit_end) return fail(LFM_EINVAL, "NULL argument");
    if (world < 1 || rank < 0 || rank >= world) return fail(LFM_EINVAL, "rank=%d world=%d", rank, world);
    Geo g;
    ST(make_geo(nnum, nz, kh, kw, height, width, /*direct=*/false, &g));
    int num_sms = 148, dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();   // host-only use (no device): B200 defaults
        num_sms = 148;
    }
    const std::vector<PlaneCost> pc = plane_costs(psf_host, nnum, g, flags, num_sms);
    const int N2 = nnum * nnum;
    std::vector<int> cut(world + 1, 0);
    if (flags & LFM_PLAN_EVEN_SHARDS)
        for (int r = 0; r < world; ++r) unit_range(nz * N2, world, r, &cut[r], &cut[r + 1]);
    else
        cut = balanced_cuts(pc, N2, world);
    *unit_begin = cut[rank];
    *unit_end = cut[rank + 1];
    if (est_seconds) *est_seconds = range_cost(pc, N2, cut[rank], cut[rank + 1]);
    return LFM_OK;
}

lfm_status lfm_set_memory_limit(size_t bytes) {
    g_mem_limit = bytes;
    return LFM_OK;
}

lfm_status lfm_plan_owned(lfm_plan p, int* unit_begin, int* unit_end) {
    g_err[0] = 0;
    if (!p || !unit_begin || !unit_end) return fail(LFM_EINVAL, "NULL argument");
    *unit_begin = p->u0;
    *unit_end = p->u1;
    return LFM_OK;
}

lfm_status lfm_plan_info(lfm_plan p, lfm_info* info) {
    if (!p || !info) return fail(LFM_EINVAL, "NULL argument");
    info->nnum = p->geo.N;
    info->nz = p->geo.nz;
    info->kh = p->geo.kh;
    info->kw = p->geo.kw;
    info->height = p->geo.H;
    info->width = p->geo.W;
    info->unit_begin = p->u0;
    info->unit_end = p->u1;
    const lfm_plan_s::TileGroup* g0 = p->tiled ? &p->tgs[0] : nullptr;   // (tiled plans: the first group)
    info->fft_h = g0 ? g0->tg.L : p->geo.Lh;
    info->fft_w = g0 ? g0->tg.L : p->geo.Lw;
    info->lc_min_h = p->geo.lcmin_h;
    info->lc_min_w = p->geo.lcmin_w;
    info->n_kappa = g0 ? g0->xg.nkappa : p->geo.nkappa;
    info->tiles = g0 ? g0->tg.ntile : 0;
    info->tile_T1 = g0 ? g0->tg.T1 : 0;
    info->tile_T2 = g0 ? g0->tg.T2 : 0;
    info->tile_groups = (int)p->tgs.size();
    info->fft_bytes = p->fft_alg_bytes;
    info->units_padded = p->nu_fft_pad;
    info->x_s = p->region.xs;
    info->y_s = p->region.ys;
    info->direct = p->direct ? 1 : (p->nu_fft == 0 ? 1 : 0);
    info->direct_planes = p->direct ? p->geo.nz : p->n_direct_planes;
    info->fft_units = p->direct ? 0 : p->nu_fft;
    info->tc_planes = p->direct ? 0 : p->n_tc_planes;
    info->tc_flops_executed = p->direct ? 0.0 : p->tc_flops_exec;
    info->planes_moved_for_memory = p->mem_moved;
    for (int d = 0; d < 2; ++d) {
        info->partition_sms[d][0] = p->part[d].sms_tc;
        info->partition_sms[d][1] = p->part[d].sms_mac;
    }
    {
        info->c1_mode = p->sym ? 1 + sym_multimem(p->sym) : 0;
        info->tc_moved_to_fft = p->part_moved;
    }
    info->tc_flops_algorithmic = p->direct ? 0.0 : p->tc_flops_alg;
    info->transfer_bytes = p->transfer_bytes;
    info->device_bytes = p->bytes;
    info->plan_ms = p->plan_ms;
    return LFM_OK;
}

void lfm_plan_destroy(lfm_plan p) { plan_free(p); }

lfm_status lfm_forward(lfm_plan p, const float* x, float* y, void* stream) {
    g_err[0] = 0;
    if (!p || !x || !y) return fail(LFM_EINVAL, "NULL argument");
    if (p->frames) return fail(LFM_EUNSUPPORTED, "plan built for frame batches (LFM_PLAN_FRAMES): use lfm_rl_iterate_batch");
    return op_forward_src(p, x, /*image=*/true, y, as_stream(stream));
}

lfm_status lfm_backward(lfm_plan p, const float* y, float* x, void* stream) {
    g_err[0] = 0;
    if (!p || !x || !y) return fail(LFM_EINVAL, "NULL argument");
    if (p->frames) return fail(LFM_EUNSUPPORTED, "plan built for frame batches (LFM_PLAN_FRAMES): use lfm_rl_iterate_batch");
    return op_backward(p, SRC_IMAGE2D, y, nullptr, 1.0f, DST_VOLIMAGE, x, nullptr, as_stream(stream));
}

lfm_status lfm_normalizer(lfm_plan p, float* x, void* stream) {
    g_err[0] = 0;
    if (!p || !x) return fail(LFM_EINVAL, "NULL argument");
    CK(launch_poly_to_image(p->norm, x, p->xall, p->u0, p->nu, as_stream(stream)));
    return LFM_OK;
}

lfm_status lfm_rl_step(lfm_plan p, const float* y, const float* x_in, float* x_out, float eps, int region,
                       float* yhat_out, double* entropy_host, void* stream) {
    g_err[0] = 0;
    if (!p || !y || !x_in || !x_out) return fail(LFM_EINVAL, "NULL argument");
    if (p->frames) return fail(LFM_EUNSUPPORTED, "plan built for frame batches (LFM_PLAN_FRAMES): use lfm_rl_iterate_batch");
    if (!(eps > 0.0f)) return fail(LFM_EINVAL, "eps must be > 0");
    cudaStream_t s = as_stream(stream);
    CK(launch_image_to_poly(x_in, p->xb[0], p->xall, p->u0, p->nu, s));
    ST(op_step(p, y, p->xb[0], p->xb[1], eps, region, entropy_host != nullptr, s));
    if (yhat_out) CK(cudaMemcpyAsync(yhat_out, p->yhat, (size_t)p->geo.H * p->geo.W * sizeof(float), cudaMemcpyDeviceToDevice, s));
    CK(launch_poly_to_image(p->xb[1], x_out, p->xall, p->u0, p->nu, s));
    if (entropy_host) {
        CK(cudaMemcpyAsync(p->host, p->met.out, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        *entropy_host = p->host[0];
    }
    return LFM_OK;
}

lfm_status rl_loop(lfm_plan p, const float* y, float* x, const lfm_policy* pol, int* best_iter, int* stop_iter,
                   double* series_host, float* ms_host, cudaStream_t s, float* host_mirror, bool* mirrored);

lfm_status lfm_rl_iterate(lfm_plan p, const float* y, float* x, const lfm_policy* pol, int* best_iter, int* stop_iter,
                          double* series_host, float* ms_host, void* stream) {
    g_err[0] = 0;
    if (!p || !y || !x || !best_iter || !stop_iter || !series_host) return fail(LFM_EINVAL, "NULL argument");
    bool mirrored = false;
    return rl_loop(p, y, x, pol, best_iter, stop_iter, series_host, ms_host, as_stream(stream), nullptr, &mirrored);
}

// the RL loop; host_mirror (single rank, host loop only): each improving iterate is written to x (device, image
// layout) and copied to host_mirror on p->scopy while the next iteration runs; *mirrored tells whether host_mirror
// holds x_best on return (the caller then skips its own copy)
lfm_status rl_loop(lfm_plan p, const float* y, float* x, const lfm_policy* pol, int* best_iter, int* stop_iter,
                   double* series_host, float* ms_host, cudaStream_t s, float* host_mirror, bool* mirrored) {
    *mirrored = false;
    if (p->frames) return fail(LFM_EUNSUPPORTED, "plan built for frame batches (LFM_PLAN_FRAMES): use lfm_rl_iterate_batch");
    ST(check_policy(pol));
    if (!p->has_optics) return fail(LFM_EINVAL, "plan was created without optics: the stop rule needs the DCT-entropy metric");
    ST(check_y(p, y, s));
    const size_t vol = (size_t)p->nu * p->geo.nh * p->geo.nw;
    int cur = 0, best = -1;
    const bool isra = pol->update == LFM_UPDATE_ISRA;
    if (isra) {   // H^T y once per call (polyphase, owned units)
        if (!p->hty) ST(dalloc(p, &p->hty, vol * sizeof(float), "H^T y"));
        ST(op_backward(p, SRC_IMAGE2D, y, nullptr, 1.0f, DST_POLY, p->hty, nullptr, s));
    }
    if (pol->init_from_x) {
        CK(launch_image_to_poly(x, p->xb[cur], p->xall, p->u0, p->nu, s));
    } else if (isra) {
        CK(cudaMemcpyAsync(p->xb[cur], p->hty, vol * sizeof(float), cudaMemcpyDeviceToDevice, s));   // x0 = H^T y
    } else {
        CK(launch_fill_dev(p->xb[cur], vol, p->stats, p->norm_sum, s));   // c0 = sum y / sum H^T 1
    }
    const int cap = pol->mode == LFM_MODE_FIXED ? pol->n_iters : pol->max_iters;
    if (p->dloop && !p->prof) {
        // device-resident loop: one graph launch, no host round trip per iteration
        if (!p->lstate) ST(dalloc(p, &p->lstate, sizeof(LoopState), "loop state"));
        if (p->lseries_cap < cap) {
            cudaFree(p->lseries);
            p->lseries = nullptr;
            ST(dalloc(p, &p->lseries, (size_t)cap * sizeof(double), "loop series"));
            p->lseries_cap = cap;
            for (cudaGraphExec_t g : p->lexec) cudaGraphExecDestroy(g);   // captured the old series pointer
            p->lexec.clear();
            p->lkeys.clear();
        }
        cudaGraphExec_t exec = nullptr;
        ST(loop_graph(p, y, pol, cap, &exec, s));
        CK(launch_loop_reset(p->lstate, s));
        if (ms_host) CK(cudaEventRecord(p->ev0, s));
        CK(cudaGraphLaunch(exec, s));
        if (ms_host) CK(cudaEventRecord(p->ev1, s));
        LoopState hs;
        CK(cudaMemcpyAsync(&hs, p->lstate, sizeof(LoopState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaMemcpy(series_host, p->lseries, (size_t)hs.k * sizeof(double), cudaMemcpyDeviceToHost));
        if (ms_host) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
            for (int i = 0; i < hs.k; ++i) ms_host[i] = ms / hs.k;   // per-iteration average (one graph launch)
        }
        p->pacc.iterations += hs.k;
        // xb[2] holds the argmax iterate once some iteration improved E; if none did (e.g. NaN entropies) return the
        // last iterate, as the host loop does
        ST(gather_to_image(p, hs.best_k > 0 ? p->xb[2] : p->xb[(hs.k & 1) ? 1 : 0], x, s));
        CK(cudaStreamSynchronize(s));
        *best_iter = hs.best_k;
        *stop_iter = hs.k;
        return LFM_OK;
    }
    // fixed-iteration mode, one rank, no graphs / profiling / mirror: pipeline the host loop one iteration deep.
    // Iteration k + 1 is issued before E_k is read; its output buffer avoids x_k's and best_{k-1}'s, so whichever of
    // them E_k makes the argmax survives (three volume buffers suffice).  The max-projection and the metric of
    // iteration k run on p->smet beside iteration k + 1 (they only read x_k, which iteration k + 1 also only reads,
    // and x_k's buffer is rewritten at k + 2 at the earliest, after E_k -- hence its max-projection -- was waited for).
    static const bool no_pipe = getenv("LFM_NO_PIPELINE") != nullptr;   // dev A/B
    if (pol->mode == LFM_MODE_FIXED && !p->graphs && !p->prof && !p->comm && !host_mirror && !no_pipe) {
        if (!p->smet) {
            CK(cudaStreamCreateWithFlags(&p->smet, cudaStreamNonBlocking));
            for (auto* e : {&p->evupd[0], &p->evupd[1], &p->evmet[0], &p->evmet[1]})
                CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
        double best_e = -INFINITY;
        int best_k = 0, xk = cur;   // xk: the buffer of the newest iterate
        auto take = [&](int kk, int buf) -> lfm_status {   // E_kk of the iterate in buf: argmax bookkeeping
            CK(cudaEventSynchronize(p->evmet[kk & 1]));
            const double e = p->host[8 + (kk & 1)];
            series_host[kk - 1] = e;
            p->pacc.iterations += 1;
            if (e > best_e) {
                best_e = e;
                best_k = kk;
                best = buf;
            }
            return LFM_OK;
        };
        if (ms_host) CK(cudaEventRecord(p->ev0, s));
        int prev_buf = -1;
        for (int kk = 1; kk <= pol->n_iters; ++kk) {
            int nxt = 0;
            while (nxt == xk || nxt == best) ++nxt;
            ST(op_step(p, y, p->xb[xk], p->xb[nxt], pol->eps, pol->region, true, s, pol->update, p->hty, false));
            CK(cudaEventRecord(p->evupd[kk & 1], s));
            CK(cudaStreamWaitEvent(p->smet, p->evupd[kk & 1], 0));
            ST(op_tail(p, p->xb[nxt], pol->region, true, p->smet));
            CK(cudaMemcpyAsync(p->host + 8 + (kk & 1), p->met.out, sizeof(double), cudaMemcpyDeviceToHost, p->smet));
            CK(cudaEventRecord(p->evmet[kk & 1], p->smet));
            p->pacc.d2h_bytes += sizeof(double);
            if (kk > 1) ST(take(kk - 1, prev_buf));
            prev_buf = nxt;
            xk = nxt;
        }
        ST(take(pol->n_iters, prev_buf));
        CK(cudaStreamWaitEvent(s, p->evmet[pol->n_iters & 1], 0));   // the caller's stream sees the whole loop
        if (ms_host) {
            CK(cudaEventRecord(p->ev1, s));
            CK(cudaEventSynchronize(p->ev1));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
            for (int i = 0; i < pol->n_iters; ++i) ms_host[i] = ms / pol->n_iters;   // per-iteration average
        }
        if (best < 0) best = xk;
        ST(gather_to_image(p, p->xb[best], x, s));
        CK(cudaStreamSynchronize(s));
        *best_iter = best_k;
        *stop_iter = pol->n_iters;
        return LFM_OK;
    }
    const bool mirror = host_mirror && !p->comm;
    if (mirror && !p->scopy) {
        CK(cudaStreamCreateWithFlags(&p->scopy, cudaStreamNonBlocking));
        for (auto& e : p->evconv) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&p->evcopy, cudaEventDisableTiming));
    }
    // every exit path (errors included) drains the side stream first: no queued conversion or copy into the
    // caller's x / host_mirror may run after this call has returned (lfm.h: nothing is written after a failure)
    struct DrainOnExit {
        cudaStream_t st;
        ~DrainOnExit() {
            if (st) cudaStreamSynchronize(st);
        }
    } drain_guard{mirror ? p->scopy : nullptr};
    bool conv_pending[3] = {false, false, false};
    int mirrored_buf = -1;
    double best_e = -INFINITY, prev = 0.0;
    int decreases = 0, k = 0, best_k = 0;
    for (;;) {
        ++k;
        int nxt = 0;
        while (nxt == cur || nxt == best) ++nxt;
        if (conv_pending[nxt]) {   // the side stream may still read this buffer (an earlier best being mirrored)
            CK(cudaStreamWaitEvent(s, p->evconv[nxt], 0));
            conv_pending[nxt] = false;
        }
        if (ms_host) CK(cudaEventRecord(p->ev0, s));
        if (p->graphs && !p->prof) {
            ST(step_graph(p, y, cur, nxt, pol, s));
        } else {
            ST(op_step(p, y, p->xb[cur], p->xb[nxt], pol->eps, pol->region, true, s, pol->update, p->hty));
            CK(cudaMemcpyAsync(p->host, p->met.out, sizeof(double), cudaMemcpyDeviceToHost, s));
        }
        p->pacc.d2h_bytes += sizeof(double);
        if (ms_host) CK(cudaEventRecord(p->ev1, s));
        CK(cudaStreamSynchronize(s));
        const double e = p->host[0];
        series_host[k - 1] = e;
        p->pacc.iterations += 1;
        if (p->prof) {
            for (int st = 0; st < LFM_N_STAGES; ++st) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, p->pev[st], p->pev[st + 1]));
                p->pacc.ms[st] += ms;
                p->pacc.count[st] += 1;
            }
            ST(read_kernel_timers(p));
        }
        if (ms_host) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
            ms_host[k - 1] = ms;
        }
        // stop rule (reading C15): strict decreases counted, argmax with ties -> smallest k
        // (relative gain of E_k over E_{k-1}: the auto-stop curve flattening before its peak, see the mirror below)
        const double gain = k > 1 ? (e - prev) / std::max(std::fabs(e), 1e-300) : 1.0;
        if (k > 1 && e < prev)
            ++decreases;
        else
            decreases = 0;
        prev = e;
        if (e > best_e) {
            best_e = e;
            best_k = k;
            best = nxt;
            // iteration k is complete (synchronised above): convert + copy it on the side stream -- unless the previous
            // mirror copy is still in flight (the host link is slower than an iteration): then this iterate is skipped
            // and a later one (or the final copy after the loop) brings x_best
            // Which improving iterates are mirrored: in auto mode those after the curve has flattened (gain below
            // kMirrorGain: the stop is near, and the iterate the stop keeps is then usually on the host already when
            // the loop ends); every one with LFM_HOST_MIRROR (dev); none in fixed mode (x_best is copied after the loop)
            static const bool mirror_all = getenv("LFM_HOST_MIRROR") != nullptr;
            constexpr double kMirrorGain = 1e-2;
            const bool want = mirror && (mirror_all || (pol->mode != LFM_MODE_FIXED && gain < kMirrorGain));
            bool link_busy = false;
            if (want && mirrored_buf >= 0) {
                const cudaError_t q = cudaEventQuery(p->evcopy);
                if (q == cudaErrorNotReady) {
                    link_busy = true;
                    cudaGetLastError();   // (not an error)
                } else if (q != cudaSuccess) {
                    return fail(LFM_ECUDA, "mirror copy: %s", cudaGetErrorString(q));
                }
            }
            if (want && !link_busy) {
                ST(gather_to_image(p, p->xb[nxt], x, p->scopy));
                CK(cudaEventRecord(p->evconv[nxt], p->scopy));
                conv_pending[nxt] = true;
                CK(cudaMemcpyAsync(host_mirror, x, (size_t)p->geo.nz * p->geo.H * p->geo.W * sizeof(float),
                                   cudaMemcpyDeviceToHost, p->scopy));
                CK(cudaEventRecord(p->evcopy, p->scopy));
                p->pacc.d2h_bytes += (long long)p->geo.nz * p->geo.H * p->geo.W * sizeof(float);
                mirrored_buf = nxt;
                p->pacc.launches += 1;
            }
        }
        cur = nxt;
        bool stop;
        if (pol->mode == LFM_MODE_FIXED)
            stop = k >= pol->n_iters;
        else
            stop = (k >= pol->min_iters && decreases >= pol->patience) || k >= cap;
        if (stop) break;
    }
    if (best < 0) best = cur;
    if (mirror && mirrored_buf == best) {   // x and host_mirror already hold x_best once the side stream drains
        CK(cudaStreamSynchronize(p->scopy));
        *mirrored = true;
    } else {
        if (mirror) CK(cudaStreamSynchronize(p->scopy));   // no in-flight mirror may overwrite x after this point
        ST(gather_to_image(p, p->xb[best], x, s));
        CK(cudaStreamSynchronize(s));
    }
    *best_iter = best_k;
    *stop_iter = k;
    return LFM_OK;
}

lfm_status lfm_deconvolve_host(lfm_plan p, const float* y_host, float* x_host, const lfm_policy* pol, int* best_iter,
                               int* stop_iter, double* series_host, float* ms_host, void* stream) {
    g_err[0] = 0;
    if (!p || !y_host || !x_host) return fail(LFM_EINVAL, "NULL argument");
    ST(check_policy(pol));
    cudaStream_t s = as_stream(stream);
    const size_t HW = (size_t)p->geo.H * p->geo.W;
    const size_t V = (size_t)p->geo.nz * HW;
    if (!p->y_stage) ST(dalloc(p, &p->y_stage, HW * sizeof(float), "y staging"));
    if (!p->x_stage) ST(dalloc(p, &p->x_stage, V * sizeof(float), "x staging"));
    CK(cudaMemcpyAsync(p->y_stage, y_host, HW * sizeof(float), cudaMemcpyHostToDevice, s));
    if (pol->init_from_x) CK(cudaMemcpyAsync(p->x_stage, x_host, V * sizeof(float), cudaMemcpyHostToDevice, s));
    // the host loop mirrors each improving iterate into x_host while the next iteration runs (the device-resident
    // loop has no per-iteration host step: it copies once at the end)
    // (only into page-locked memory: a copy into pageable memory would block the host loop)
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, x_host) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();   // clear a possible error of the query
    bool mirrored = false;
    ST(rl_loop(p, p->y_stage, p->x_stage, pol, best_iter, stop_iter, series_host, ms_host, s,
               (p->dloop || !pinned) ? nullptr : x_host, &mirrored));
    if (!mirrored) {
        CK(cudaMemcpyAsync(x_host, p->x_stage, V * sizeof(float), cudaMemcpyDeviceToHost, s));
        p->pacc.d2h_bytes += (long long)V * sizeof(float);
    }
    CK(cudaStreamSynchronize(s));
    return LFM_OK;
}

lfm_status lfm_quality(lfm_plan p, const float* x, int region, double* entropy, void* stream) {
    g_err[0] = 0;
    if (!p || !x || !entropy) return fail(LFM_EINVAL, "NULL argument");
    if (region != LFM_REGION_TRIANGLE && region != LFM_REGION_RECTANGLE) return fail(LFM_EINVAL, "region=%d", region);
    cudaStream_t s = as_stream(stream);
    unsigned* mp = p->sym ? reinterpret_cast<unsigned*>(sym_buffer(p->sym, 1)) : p->mproj;   // op_metric's C2 input
    CK(cudaMemsetAsync(mp, 0, (size_t)p->geo.H * p->geo.W * sizeof(unsigned), s));
    CK(launch_max_project(x, mp, p->xall, s));
    ST(op_metric(p, region, s));
    CK(cudaMemcpyAsync(p->host, p->met.out, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *entropy = p->host[0];
    return LFM_OK;
}

lfm_status lfm_dct_entropy(const float* img, int height, int width, int nnum, const lfm_optics* optics, int region,
                           double* entropy, int* x_s, int* y_s, void* stream) {
    g_err[0] = 0;
    if (!img || !entropy) return fail(LFM_EINVAL, "NULL argument");
    if (nnum < 1) return fail(LFM_EINVAL, "nnum=%d", nnum);
    if (region != LFM_REGION_TRIANGLE && region != LFM_REGION_RECTANGLE) return fail(LFM_EINVAL, "region=%d", region);
    Region r;
    ST(make_region(optics, nnum, height, width, &r));
    cudaStream_t s = as_stream(stream);
    MetricDev m;
    lfm_status st = metric_alloc(&m, r, height, width, s, nullptr);
    if (st != LFM_OK) {
        metric_free(&m);
        return st;
    }
    const int ri = region == LFM_REGION_RECTANGLE ? 1 : 0;
    double h = 0.0;
    cudaError_t e = launch_metric(reinterpret_cast<const unsigned*>(img), height, width, m.xs, m.ys, m.Cr, m.Cw, m.mem[ri],
                                  m.nmem[ri], m.T1, m.rowsq, m.out, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, m.out, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    metric_free(&m);
    if (e != cudaSuccess) return fail(LFM_ECUDA, "lfm_dct_entropy: %s", cudaGetErrorString(e));
    *entropy = h;
    if (x_s) *x_s = r.xs;
    if (y_s) *y_s = r.ys;
    return LFM_OK;
}

lfm_status lfm_rl_iterate_batch(lfm_plan p, int frames, const float* y, float* x, const lfm_policy* pol, int* best_iter,
                                int* stop_iter, double* series_host, float* ms_host, void* stream) {
    g_err[0] = 0;
    if (!p || !y || !x || !best_iter || !stop_iter || !series_host) return fail(LFM_EINVAL, "NULL argument");
    if (p && p->frames ? (frames != 8 && frames != 16 && frames != 32)
                       : (frames != 2 && frames != 4 && frames != 8 && frames != 16))
        return fail(LFM_EINVAL, "frames=%d: the batched path takes 2, 4, 8 or 16 frames (LFM_PLAN_FRAMES plans: 8, 16 or "
                    "32; one frame: lfm_rl_iterate)", frames);
    ST(check_policy(pol));
    if (pol->update != LFM_UPDATE_RL) return fail(LFM_EUNSUPPORTED, "the batched path runs the RL update only");
    if (p->direct) return fail(LFM_EUNSUPPORTED, "the batched path needs a frequency / hybrid plan");
    if (p->geo.N * p->geo.N > 256) return fail(LFM_EUNSUPPORTED, "the batched forward MAC handles N^2 <= 256");
    if (!p->has_optics) return fail(LFM_EINVAL, "plan was created without optics: the stop rule needs the metric");
    cudaStream_t s = as_stream(stream);
    const int F = frames, N2 = p->geo.N * p->geo.N;
    const size_t HW = (size_t)p->geo.H * p->geo.W;
    if (p->tiled) {
        // a tiled plan (§5.6) already batches its tiles through the kind::f16 MACs: the frames run one after the other
        // through the single-frame loop (identical results to lfm_rl_iterate per frame); ms_host sums the frames'
        // k-th iterations
        const int sstride = std::max(pol->n_iters, pol->max_iters);
        std::vector<float> msf(ms_host ? sstride : 0, 0.0f);
        if (ms_host) std::fill(ms_host, ms_host + sstride, 0.0f);
        for (int f = 0; f < F; ++f) {
            bool mirrored = false;
            ST(rl_loop(p, y + f * HW, x + (size_t)f * p->geo.nz * HW, pol, best_iter + f, stop_iter + f,
                       series_host + (size_t)f * sstride, ms_host ? msf.data() : nullptr, s, nullptr, &mirrored));
            if (ms_host)
                for (int i = 0; i < stop_iter[f] && i < sstride; ++i) ms_host[i] += msf[i];
        }
        return LFM_OK;
    }
    const size_t vol = (size_t)p->nu * p->geo.nh * p->geo.nw;
    const long long sG = (long long)p->geo.nkappa * p->nu_fft_pad, sY = (long long)p->geo.nkappa * N2;
    const int rld = p->frames ? p->bpitch : N2;             // R row pitch (the fp16 MACs read R through a TMA map)
    const long long sR = (long long)p->geo.nkappa * rld;
    if (p->bcap < F) {   // (re)allocate the per-frame state
        cudaFree(p->bG); cudaFree(p->bXh); cudaFree(p->bY); cudaFree(p->bR); cudaFree(p->bx); cudaFree(p->byhat);
        cudaFree(p->bmproj); cudaFree(p->bent); cudaFree(p->bmT1); cudaFree(p->bmrs);
        if (p->bhost) cudaFreeHost(p->bhost);
        p->bG = p->bXh = p->bY = p->bR = nullptr;
        p->bx = p->byhat = nullptr;
        p->bmproj = nullptr;
        p->bent = p->bhost = nullptr;
        p->bmT1 = p->bmrs = nullptr;
        p->bcap = 0;
        if (p->nu_fft > 0) {
            ST(dalloc(p, &p->bG, (size_t)F * sG * sizeof(float2), "batch G spectra"));
            ST(dalloc(p, &p->bXh, (size_t)F * sG * sizeof(float2), "batch Xh spectra"));
            ST(dalloc(p, &p->bY, (size_t)F * sY * sizeof(float2), "batch Y spectra"));
            ST(dalloc(p, &p->bR, (size_t)F * sR * sizeof(float2), "batch R spectra"));
            CK(cudaMemsetAsync(p->bG, 0, (size_t)F * sG * sizeof(float2), s));   // padding columns stay zero
            CK(cudaMemsetAsync(p->bR, 0, (size_t)F * sR * sizeof(float2), s));
        }
        ST(dalloc(p, &p->bx, (size_t)3 * F * vol * sizeof(float), "batch volumes"));
        ST(dalloc(p, &p->byhat, (size_t)F * HW * sizeof(float), "batch yhat"));
        ST(dalloc(p, &p->bmproj, (size_t)F * HW * sizeof(unsigned), "batch max projections"));
        ST(dalloc(p, &p->bent, (size_t)2 * F * sizeof(double), "batch entropies"));
        {
            const int nmem = std::max(p->met.nmem[0], p->met.nmem[1]);
            ST(dalloc(p, &p->bmT1, (size_t)F * ((size_t)p->met.xs * p->geo.H + nmem) * sizeof(double), "batch metric T1"));
            ST(dalloc(p, &p->bmrs, (size_t)F * p->geo.H * sizeof(double), "batch metric rows"));
        }
        CK(cudaMallocHost(&p->bhost, (size_t)2 * F * sizeof(double)));
        p->bcap = F;
    }
    auto xbuf = [&](int f, int b) { return p->bx + ((size_t)f * 3 + b) * vol; };
    // validate every frame and initialise x0 (uniform c0_f = sum y_f / sum H^T 1, reading C2, or caller's x)
    for (int f = 0; f < F; ++f) {
        ST(check_y(p, y + (size_t)f * HW, s));
        if (pol->init_from_x)
            CK(launch_image_to_poly(x + (size_t)f * p->geo.nz * HW, xbuf(f, 0), p->xall, p->u0, p->nu, s));
        else
            CK(launch_fill_dev(xbuf(f, 0), vol, p->stats, p->norm_sum, s));
    }
    const int cap = pol->mode == LFM_MODE_FIXED ? pol->n_iters : pol->max_iters;
    const int sstride = std::max(pol->n_iters, pol->max_iters);   // series_host row stride (lfm.h)
    std::vector<int> cur(F, 0), best(F, -1), dec(F, 0), bestk(F, 0), stopped(F, 0);
    std::vector<double> prev(F, 0.0), beste(F, -INFINITY);
    int k = 0, active = F;
    while (active > 0) {
        ++k;
        std::vector<int> nxt(F, 0);
        for (int f = 0; f < F; ++f)
            while (nxt[f] == cur[f] || nxt[f] == best[f]) ++nxt[f];
        if (ms_host) CK(cudaEventRecord(p->ev0, s));
        // ---- forward: coarse transforms per frame, one batched pass over M, inverse per frame ----
        // (profile stages here are batch groups: r2c_x = all frames' transforms, fwd_mac = the batched pass,
        //  c2r_yhat = per-frame inverse + direct planes + ratio transform, bwd_mac, c2r_update = per-frame rest)
        ST(mark(p, ST_R2C_X, s));
        if (p->nu_fft > 0) {
            for (int f = 0; f < F; ++f)
                if (!stopped[f])
                    CK(launch_r2c(p->xg, p->fh, p->fw, p->tw_h, p->tw_w,
                                  r2c_args(SRC_POLY, xbuf(f, cur[f]), nullptr, 0.f, p->nu_fft, p->bG + f * sG, p->nu_fft_pad), s));
            ST(mark(p, ST_FWD_MAC, s));
            if (p->frames) {   // fp16 split transfer matrices, kind::f16 (kernels_mac_f16.cu)
                CK(launch_frame_scales(p->bG, sG, p->nu_fft_pad, F, p->mf_eb, s));
                if (p->mf_src[0] != p->bG || p->mf_F[0] != F) {
                    CK(mac_f16_encode_src(&p->mf_fwd, 1, p->bG, sG, F));
                    p->mf_src[0] = p->bG;
                    p->mf_F[0] = F;
                }
                p->mf_fwd.bexp = p->mf_eb;
                p->mf_fwd.out = p->bY;
                p->mf_fwd.out_fstride = sY;
                p->mf_fwd.out_ld = N2;
                ST(kmark(p, 1, 0, s));
                CK(launch_mac_f16(p->mf_fwd, 1, F, p->num_sms, s));
            } else if (!p->mac_tc_off && F >= 8 && N2 <= 256) {   // tcgen05 3xTF32 batched MAC
                if (!p->mac_tc_ready) {
                    p->mac_tc.nkappa = p->geo.nkappa;
                    p->mac_tc.N2 = N2;
                    p->mac_tc.nu_pad = p->nu_fft_pad;
                    CK(mac_tc_encode(&p->mac_tc, p->M));
                    p->mac_tc_ready = true;
                }
                if (p->mac_tc.G != p->bG || p->mac_tc.g_fstride != sG || p->mac_tc_F != F) {
                    CK(mac_tc_encode_g(&p->mac_tc, p->bG, sG, F));
                    p->mac_tc_F = F;
                }
                p->mac_tc.G = p->bG;
                p->mac_tc.g_fstride = sG;
                p->mac_tc.Y = p->bY;
                p->mac_tc.y_fstride = sY;
                ST(kmark(p, 1, 0, s));
                CK(launch_fwd_mac_batch_tc(p->mac_tc, F, p->num_sms, s));
            } else {
                ST(kmark(p, 1, 0, s));
                CK(launch_fwd_mac_batch(p->M, p->bG, sG, p->bY, sY, F, p->geo.nkappa, N2, p->nu_fft_pad, s));
            }
            ST(kmark(p, 1, 1, s));
            p->pacc.launches += 1;
        }
        ST(mark(p, ST_C2R_YHAT, s));
        for (int f = 0; f < F; ++f) {
            if (stopped[f]) continue;
            float* yimg = p->byhat + f * HW;
            bool acc = false;
            if (p->nu_fft > 0) {
                C2RArgs c{};
                c.dst = DST_IMAGE;
                c.in = p->bY + f * sY;
                c.in_ld = N2;
                c.ntrans = N2;
                c.out = yimg;
                CK(launch_c2r(p->xg, p->fh, p->fw, p->tw_h, p->tw_w, c, s));
                p->pacc.launches += 2;
                acc = true;
            }
            for (const TcDirArgs& tg : p->tcf) {
                CK(launch_tcdir_fwd(tg, xbuf(f, cur[f]), 0, yimg, acc ? 1 : 0, s));
                p->pacc.launches += 3;
                acc = true;
            }
            for (const DirArgs& dg : p->dgroups) {
                CK(launch_dir_fwd(dg, xbuf(f, cur[f]), 0, p->dpart, yimg, acc ? 1 : 0, s));
                acc = true;
            }
            ST(allreduce(p, yimg, HW, ncclFloat, ncclSum, s));
            if (p->nu_fft > 0)
                CK(launch_r2c(p->xg, p->fh, p->fw, p->tw_h, p->tw_w,
                              r2c_args(SRC_RATIO, y + f * HW, yimg, pol->eps, N2, p->bR + f * sR, rld), s));
        }
        // ---- backward: one batched pass over M^H, inverse + update per frame ----
        ST(mark(p, ST_DIR_FWD, s));   // (empty stages: the batch groups above hold their work)
        ST(mark(p, ST_ALLRED_SUM, s));
        ST(mark(p, ST_R2C_RATIO, s));
        ST(mark(p, ST_BWD_MAC, s));
        if (p->nu_fft > 0) {
            ST(kmark(p, 3, 0, s));
            static const bool bwd_simt = getenv("LFM_BWD_BATCH_SIMT") != nullptr;   // dev: CUDA-core batched backward
            if (p->frames) {   // fp16 split transposed transfer matrices, kind::f16
                CK(launch_frame_scales(p->bR, sR, rld, F, p->mf_eb + 32, s));
                if (p->mf_src[1] != p->bR || p->mf_F[1] != F) {
                    CK(mac_f16_encode_src(&p->mf_bwd, 0, p->bR, sR, F));
                    p->mf_src[1] = p->bR;
                    p->mf_F[1] = F;
                }
                p->mf_bwd.bexp = p->mf_eb + 32;
                p->mf_bwd.out = p->bXh;
                p->mf_bwd.out_fstride = sG;
                p->mf_bwd.out_ld = p->nu_fft_pad;
                CK(launch_mac_f16(p->mf_bwd, 0, F, p->num_sms, s));
            } else if (!p->mac_tc_off && (F == 8 || F == 16) && !bwd_simt) {   // tcgen05 3xTF32
                if (!p->bmac_F) {   // tensor map over the (backward) transfer matrices, once
                    p->bmac_tc.nkappa = p->geo.nkappa;
                    p->bmac_tc.N2 = N2;
                    p->bmac_tc.nu_pad = p->nu_fft_pad;
                    CK(bmac_tc_encode(&p->bmac_tc, p->Mb));
                    p->bmac_F = F;
                }
                p->bmac_tc.Xh = p->bXh;
                p->bmac_tc.x_fstride = sG;
                p->bmac_tc.R = p->bR;
                p->bmac_tc.r_fstride = sR;
                CK(launch_bwd_mac_batch_tc(p->bmac_tc, F, p->num_sms, s));
            } else {
                CK(launch_bwd_mac_batch(p->Mb, p->bR, sR, p->bXh, sG, F, p->geo.nkappa, N2, p->nu_fft_pad, s));
            }
            ST(kmark(p, 3, 1, s));
            p->pacc.launches += 1;
        }
        ST(mark(p, ST_C2R_UPD, s));
        for (int f = 0; f < F; ++f) {
            if (stopped[f]) continue;
            float* xo = xbuf(f, cur[f]);
            float* xn = xbuf(f, nxt[f]);
            if (p->nu_fft > 0) {
                C2RArgs c{};
                c.dst = DST_UPDATE;
                c.in = p->bXh + f * sG;
                c.in_ld = p->nu_fft_pad;
                c.ntrans = p->nu_fft;
                c.out = xn;
                c.xold = xo;
                c.norm = p->norm;
                c.eps = pol->eps;
                CK(launch_c2r(p->xg, p->fh, p->fw, p->tw_h, p->tw_w, c, s));
            }
            for (const TcDirArgs& tg : p->tcb) {
                CK(launch_tcdir_bwd(tg, SRC_RATIO, y + f * HW, p->byhat + f * HW, pol->eps, DST_UPDATE, xn, xo, p->norm, s));
                p->pacc.launches += 3;
            }
            for (const DirArgs& dg : p->dgroups)
                CK(launch_dir_bwd(dg, SRC_RATIO, y + f * HW, p->byhat + f * HW, pol->eps, DST_UPDATE, xn, xo, p->norm, s));
        }
        // a7 / C2 / a8 of every frame in one launch each: the max-projections (frame f from its new slot; a stopped
        // frame's slot is re-projected and ignored), one collective over all frames, the batched metric
        {
            FrameSel sel{};
            for (int f = 0; f < F; ++f) sel.b[f] = stopped[f] ? cur[f] : nxt[f];
            CK(launch_max_project_poly_batch(p->bx, vol, sel, F, p->bmproj, p->xall, s));
            ST(allreduce(p, p->bmproj, (size_t)F * HW, ncclFloat, ncclMax, s));
            const int ri = pol->region == LFM_REGION_RECTANGLE ? 1 : 0;
            CK(launch_metric_batch(p->bmproj, F, p->geo.H, p->geo.W, p->met.xs, p->met.ys, p->met.Cr, p->met.Cw,
                                   p->met.mem[ri], p->met.nmem[ri], p->bmT1, p->bmrs, p->bent, s));
            p->pacc.launches += 4;
        }
        ST(mark(p, ST_DIR_BWD, s));
        ST(mark(p, ST_MAXPROJ, s));
        ST(mark(p, ST_METRIC, s));
        ST(mark(p, LFM_N_STAGES, s));
        if (ms_host) CK(cudaEventRecord(p->ev1, s));
        CK(cudaMemcpyAsync(p->bhost, p->bent, 2 * F * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (p->prof) {
            for (int st = 0; st < LFM_N_STAGES; ++st) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, p->pev[st], p->pev[st + 1]));
                p->pacc.ms[st] += ms;
                p->pacc.count[st] += 1;
            }
            ST(read_kernel_timers(p, 0xA));   // the batched MACs (tensor-core planes run per frame)
        }
        if (ms_host) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
            ms_host[k - 1] = ms;
        }
        p->pacc.iterations += active;
        for (int f = 0; f < F; ++f) {
            if (stopped[f]) continue;
            const double e = p->bhost[2 * f];
            series_host[(size_t)f * sstride + k - 1] = e;
            if (k > 1 && e < prev[f])
                ++dec[f];
            else
                dec[f] = 0;
            prev[f] = e;
            if (e > beste[f]) {
                beste[f] = e;
                bestk[f] = k;
                best[f] = nxt[f];
            }
            cur[f] = nxt[f];
            const bool stop = pol->mode == LFM_MODE_FIXED
                                  ? k >= pol->n_iters
                                  : ((k >= pol->min_iters && dec[f] >= pol->patience) || k >= cap);
            if (stop) {
                stopped[f] = 1;
                stop_iter[f] = k;
                best_iter[f] = bestk[f];
                --active;
            }
        }
    }
    for (int f = 0; f < F; ++f)
        ST(gather_to_image(p, xbuf(f, best[f] < 0 ? cur[f] : best[f]), x + (size_t)f * p->geo.nz * HW, s));
    CK(cudaStreamSynchronize(s));
    return LFM_OK;
}

lfm_status lfm_profile(lfm_plan p, int enable) {
    if (!p) return fail(LFM_EINVAL, "plan is NULL");
    if (enable && !p->pev[0]) {
        for (auto& e : p->pev) CK(cudaEventCreate(&e));
        for (auto& kv : p->kev)
            for (auto& e : kv) CK(cudaEventCreate(&e));
    }
    if (enable && !p->has_optics) return fail(LFM_EINVAL, "profiling times lfm_rl_iterate, which needs optics");
    p->prof = enable != 0;
    return LFM_OK;
}

lfm_status lfm_profile_read(lfm_plan p, lfm_profile_t* out, int reset) {
    if (!p || !out) return fail(LFM_EINVAL, "NULL argument");
    *out = p->pacc;
    if (reset) p->pacc = lfm_profile_t{};
    return LFM_OK;
}

const char* lfm_profile_stage_name(int i) { return (i >= 0 && i < LFM_N_STAGES) ? kStageNames[i] : nullptr; }

}  // extern "C"
