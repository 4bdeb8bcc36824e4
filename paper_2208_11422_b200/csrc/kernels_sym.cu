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

// OP 0: C1, float sum of the partial images; OP 1: C2, max of the partial max-projections (non-negative floats as
// uint32 bits: their order is the float order, and max is exact, so every rank's E_k and stop decision agree)
template <bool MM, int OP>
__global__ void __launch_bounds__(256) sym_reduce_kernel(ncclDevComm comm, ncclWindow_t win, size_t off, size_t n,
                                                         float* __restrict__ out) {
    ncclCoopCta cta;
    ncclLsaBarrierSession<ncclCoopCta> bar(cta, comm, ncclTeamTagLsa(), blockIdx.x, MM);
    bar.sync(cta, cuda::memory_order_acq_rel);   // every rank's partial is complete
    const int P = comm.lsaSize;
    const size_t n4 = n / 4;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        uint4 v;
        if constexpr (MM) {
            const uint4* mc = reinterpret_cast<const uint4*>(static_cast<char*>(ncclGetLsaMultimemPointer(win, 0, comm)) + off);
            if constexpr (OP == 0)
                asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "l"(mc + i)
                             : "memory");
            else {   // no vector form for the integer max: four scalar in-switch reductions
                const unsigned* mu = reinterpret_cast<const unsigned*>(mc + i);
                asm volatile("multimem.ld_reduce.relaxed.sys.global.max.u32 %0, [%1];" : "=r"(v.x) : "l"(mu) : "memory");
                asm volatile("multimem.ld_reduce.relaxed.sys.global.max.u32 %0, [%1];" : "=r"(v.y) : "l"(mu + 1) : "memory");
                asm volatile("multimem.ld_reduce.relaxed.sys.global.max.u32 %0, [%1];" : "=r"(v.z) : "l"(mu + 2) : "memory");
                asm volatile("multimem.ld_reduce.relaxed.sys.global.max.u32 %0, [%1];" : "=r"(v.w) : "l"(mu + 3) : "memory");
            }
        } else {
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
            uint4 m = make_uint4(0u, 0u, 0u, 0u);
            for (int r = 0; r < P; ++r) {   // rank order: the sum does not depend on timing
                const char* base = static_cast<const char*>(ncclGetLsaPointer(win, 0, r)) + off;
                if constexpr (OP == 0) {
                    const float4 t = reinterpret_cast<const float4*>(base)[i];
                    a.x += t.x;
                    a.y += t.y;
                    a.z += t.z;
                    a.w += t.w;
                } else {
                    const uint4 t = reinterpret_cast<const uint4*>(base)[i];
                    m.x = max(m.x, t.x);
                    m.y = max(m.y, t.y);
                    m.z = max(m.z, t.z);
                    m.w = max(m.w, t.w);
                }
            }
            if constexpr (OP == 0)
                v = make_uint4(__float_as_uint(a.x), __float_as_uint(a.y), __float_as_uint(a.z), __float_as_uint(a.w));
            else
                v = m;
        }
        reinterpret_cast<uint4*>(out)[i] = v;
    }
    for (size_t i = 4 * n4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {   // tail
        float a = 0.f;
        unsigned m = 0u;
        for (int r = 0; r < P; ++r) {
            const char* base = static_cast<const char*>(ncclGetLsaPointer(win, 0, r)) + off;
            if constexpr (OP == 0)
                a += reinterpret_cast<const float*>(base)[i];
            else
                m = max(m, reinterpret_cast<const unsigned*>(base)[i]);
        }
        reinterpret_cast<unsigned*>(out)[i] = OP == 0 ? __float_as_uint(a) : m;
    }
    bar.sync(cta, cuda::memory_order_acq_rel);   // every rank has read every partial
}

struct SymState {
    ncclComm_t comm = nullptr;
    void* buf = nullptr;           // ncclMemAlloc'd, registered window: slot 0 the partial image, slot 1 the partial
                                   // max-projection, each `slot` bytes
    size_t bytes = 0, n = 0, slot = 0;
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
    st->slot = (n * sizeof(float) + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
    st->bytes = 2 * st->slot;
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
    cudaDeviceSynchronize();   // the plan's streams may be non-blocking: the zeroed window must be visible to them
    *out = st;
    return LFM_OK;
}

float* sym_buffer(SymState* st, int slot) {
    return st ? reinterpret_cast<float*>(static_cast<char*>(st->buf) + (size_t)slot * st->slot) : nullptr;
}
int sym_multimem(const SymState* st) { return st ? st->multimem : 0; }

// out[0..n) = sum over ranks of every rank's slot 0 (C1) / max over ranks of slot 1 (C2); see the header comment
cudaError_t sym_reduce(SymState* st, int op, void* out, cudaStream_t s) {
    float* o = static_cast<float*>(out);
    const size_t off = op ? st->slot : 0;
    if (st->multimem) {
        if (op) sym_reduce_kernel<true, 1><<<st->blocks, 256, 0, s>>>(st->dcomm, st->win, off, st->n, o);
        else sym_reduce_kernel<true, 0><<<st->blocks, 256, 0, s>>>(st->dcomm, st->win, off, st->n, o);
    } else {
        if (op) sym_reduce_kernel<false, 1><<<st->blocks, 256, 0, s>>>(st->dcomm, st->win, off, st->n, o);
        else sym_reduce_kernel<false, 0><<<st->blocks, 256, 0, s>>>(st->dcomm, st->win, off, st->n, o);
    }
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
