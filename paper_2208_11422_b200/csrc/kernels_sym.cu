// kernels_sym.cu -- C1 (the forward projection's sum over ranks) as our own kernel over NCCL symmetric
// memory instead of ncclAllReduce (LFM_PLAN_SYMMETRIC; SURVEY f4 "NVLS multimem allreduce").
//
// Every rank writes its partial image yhat_r into a window registered with ncclCommWindowRegister
// (NCCL_WIN_COLL_SYMMETRIC): the same offset on every GPU of the NVLink domain, reachable by peer loads (LSA pointers)
// and, where the switch supports NVLS, through one multicast address.  One kernel then
//   1. waits on an LSA barrier (every rank's producers -- C2R, tcgen05 reduction, direct planes -- have finished; the
//      barrier's release / acquire orders their writes before the loads below),
//   2. forms yhat = sum_r yhat_r for its slice of pixels:
//        multimem: one `multimem.ld_reduce.add.v4.f32` per 16 bytes -- the NVSwitch adds the ranks' values and returns
//                  the sum (NVLS in-switch reduction);
//        lsa:      a load from every peer's window in rank order and an fp32 sum in that fixed order (deterministic,
//                  P2P over NVLink);
//      and writes it to the rank's local yhat (the ratio / update consumers read that),
//   3. waits on the barrier again, so no rank overwrites its partial (next iteration) while a peer may still read it.
// Every rank computes the full sum (each reads H*W floats): at c3 4 MB per rank and iteration over NVLink.
#include <nccl.h>
#include <nccl_device.h>

#include <cstdio>

#include "lfm_internal.cuh"

namespace lfm {

template <bool MM>
__global__ void __launch_bounds__(256) sym_sum_kernel(ncclDevComm comm, ncclWindow_t win, size_t n, float* __restrict__ out) {
    ncclCoopCta cta;
    ncclLsaBarrierSession<ncclCoopCta> bar(cta, comm, ncclTeamTagLsa(), blockIdx.x, MM);
    bar.sync(cta, cuda::memory_order_acq_rel);   // every rank's partial image is complete
    const int P = comm.lsaSize;
    const size_t n4 = n / 4;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 v;
        if constexpr (MM) {
            const float4* mc = reinterpret_cast<const float4*>(ncclGetLsaMultimemPointer(win, 0, comm));
            asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "l"(mc + i)
                         : "memory");
        } else {
            v = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int r = 0; r < P; ++r) {   // rank order: the sum does not depend on timing
                const float4 t = reinterpret_cast<const float4*>(ncclGetLsaPointer(win, 0, r))[i];
                v.x += t.x;
                v.y += t.y;
                v.z += t.z;
                v.w += t.w;
            }
        }
        reinterpret_cast<float4*>(out)[i] = v;
    }
    for (size_t i = 4 * n4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {   // tail
        float v = 0.f;
        for (int r = 0; r < P; ++r) v += reinterpret_cast<const float*>(ncclGetLsaPointer(win, 0, r))[i];
        out[i] = v;
    }
    bar.sync(cta, cuda::memory_order_acq_rel);   // every rank has read every partial
}

struct SymState {
    ncclComm_t comm = nullptr;
    void* buf = nullptr;           // ncclMemAlloc'd, registered window (this rank's partial image)
    size_t bytes = 0, n = 0;
    ncclWindow_t win = nullptr;
    ncclDevComm dcomm{};
    bool dcomm_ok = false;
    int multimem = 0, blocks = 0;
};

// plan-time setup (collective over the communicator): symmetric buffer for n floats, window, and a device communicator
// with one LSA barrier per block; multimem is requested when asked for and falls back to peer loads when NCCL refuses
lfm_status sym_create(ncclComm_t comm, size_t n, int want_multimem, SymState** out, char* err, size_t errlen) {
    SymState* st = new SymState();
    st->comm = comm;
    st->n = n;
    st->bytes = (n * sizeof(float) + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
    st->blocks = 132;
    ncclResult_t r = ncclMemAlloc(&st->buf, st->bytes);
    if (r == ncclSuccess) r = ncclCommWindowRegister(comm, st->buf, st->bytes, &st->win, NCCL_WIN_COLL_SYMMETRIC);
    if (r != ncclSuccess) {
        snprintf(err, errlen, "symmetric window: %s", ncclGetErrorString(r));
        sym_destroy(st);
        return LFM_ENCCL;
    }
    for (int mm = want_multimem ? 1 : 0; mm >= 0; --mm) {
        ncclDevCommRequirements req{};
        req.lsaBarrierCount = st->blocks;
        req.lsaMultimem = mm != 0;
        r = ncclDevCommCreate(comm, &req, &st->dcomm);
        if (r == ncclSuccess) {
            st->dcomm_ok = true;
            st->multimem = mm;
            break;
        }
    }
    if (!st->dcomm_ok) {
        snprintf(err, errlen, "ncclDevCommCreate: %s", ncclGetErrorString(r));
        sym_destroy(st);
        return LFM_ENCCL;
    }
    cudaMemset(st->buf, 0, st->bytes);
    *out = st;
    return LFM_OK;
}

float* sym_buffer(SymState* st) { return st ? reinterpret_cast<float*>(st->buf) : nullptr; }
int sym_multimem(const SymState* st) { return st ? st->multimem : 0; }

// out[0..n) = sum over ranks of every rank's sym_buffer (see the header comment)
cudaError_t sym_sum(SymState* st, float* out, cudaStream_t s) {
    if (st->multimem)
        sym_sum_kernel<true><<<st->blocks, 256, 0, s>>>(st->dcomm, st->win, st->n, out);
    else
        sym_sum_kernel<false><<<st->blocks, 256, 0, s>>>(st->dcomm, st->win, st->n, out);
    return cudaGetLastError();
}

void sym_destroy(SymState* st) {
    if (!st) return;
    if (st->dcomm_ok) ncclDevCommDestroy(st->comm, &st->dcomm);
    if (st->win) ncclCommWindowDeregister(st->comm, st->win);
    if (st->buf) ncclMemFree(st->buf);
    delete st;
}

}  // namespace lfm
