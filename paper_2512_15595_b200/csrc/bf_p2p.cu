// bf_p2p.cu -- OR-merge of per-rank partial filters over peer memory
// (construction's exchange step).  NCCL has no bitwise-OR
// reduction, so E1/E2 (paper_2512_15595_b200/dist.py) move the partials with
// NCCL into staging buffers and fold them in a second pass.  Here the
// exchange and the OR are ONE kernel over NVLink: every rank maps every
// peer's filter (CUDA IPC), rank r loads its 1/P slice of all P partials
// directly from the peers' HBM (P independent 16-byte loads in flight per
// element), ORs them, and stores the result into all P filters -- a
// reduce-scatter by OR fused with the all-gather, no staging, no fold pass.
// Per rank and merge: (P-1)/P*M bytes read from peers and (P-1)/P*M written
// to peers (E2 moves the same bytes but through two collectives, a P*M/P
// staging buffer and a separate fold over it).
#include <cuda_runtime.h>
#include <string.h>

#include "../../include/bf.h"
#include "bf_internal.h"

namespace bf {

struct PeerPtrs {
    uint4* p[BF_P2P_MAX_RANKS];
};

__device__ __forceinline__ uint4 ld_cg16(const uint4* a)
{
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a));
    return v;
}
__device__ __forceinline__ void st_cg16(uint4* a, uint4 v)
{
    asm volatile("st.global.cg.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// 16-byte elements [lo, hi) of every peer's filter: OR of all P, stored back
// into all P.  Then the 4-byte tail words [tlo, thi) (bytes not a multiple of
// 16; only the last rank has any).  P is small (<= 16); UNR elements per
// thread per step keep UNR*P loads in flight.
template <int UNR>
__global__ void __launch_bounds__(256) p2p_or_kernel(PeerPtrs pp, uint32_t P, uint64_t lo, uint64_t hi,
                                                    uint64_t tlo, uint64_t thi)
{
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = lo + tid; base < hi; base += nth * UNR) {
        uint4 v[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) v[u] = make_uint4(0, 0, 0, 0);
        for (uint32_t q = 0; q < P; ++q) {
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const uint64_t i = base + (uint64_t)u * nth;
                if (i < hi) {
                    const uint4 x = ld_cg16(pp.p[q] + i);
                    v[u].x |= x.x;
                    v[u].y |= x.y;
                    v[u].z |= x.z;
                    v[u].w |= x.w;
                }
            }
        }
        for (uint32_t q = 0; q < P; ++q) {
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const uint64_t i = base + (uint64_t)u * nth;
                if (i < hi) st_cg16(pp.p[q] + i, v[u]);
            }
        }
    }
    for (uint64_t w = tlo + tid; w < thi; w += nth) {
        uint32_t v = 0;
        for (uint32_t q = 0; q < P; ++q) v |= ((volatile const uint32_t*)pp.p[q])[w];
        for (uint32_t q = 0; q < P; ++q) ((volatile uint32_t*)pp.p[q])[w] = v;
    }
    __threadfence_system();  // peer stores performed before the kernel is seen complete
}

}  // namespace bf

using namespace bf;

extern "C" {

int bf_ipc_handle(const void* dev_ptr, void* handle_out)
{
    if (!dev_ptr || !handle_out) return report_error(BF_EINVAL, "bf_ipc_handle", "null pointer");
    cudaIpcMemHandle_t h;
    static_assert(sizeof(h) <= BF_IPC_HANDLE_BYTES, "IPC handle size");
    cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return report_error(BF_ECUDA, "bf_ipc_handle: cudaIpcGetMemHandle", cudaGetErrorString(e));
    }
    memset(handle_out, 0, BF_IPC_HANDLE_BYTES);
    memcpy(handle_out, &h, sizeof h);
    return BF_OK;
}

int bf_ipc_open(const void* handle, void** dev_ptr_out)
{
    if (!handle || !dev_ptr_out) return report_error(BF_EINVAL, "bf_ipc_open", "null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *dev_ptr_out = nullptr;
        return report_error(BF_ECUDA, "bf_ipc_open: cudaIpcOpenMemHandle", cudaGetErrorString(e));
    }
    return BF_OK;
}

int bf_ipc_close(void* dev_ptr)
{
    if (!dev_ptr) return BF_OK;
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return report_error(BF_ECUDA, "bf_ipc_close: cudaIpcCloseMemHandle", cudaGetErrorString(e));
    }
    return BF_OK;
}

int bf_p2p_or_merge(void* const* peers, uint32_t nranks, uint32_t rank, uint64_t bytes, void* stream)
{
    if (!peers || nranks < 1 || nranks > BF_P2P_MAX_RANKS || rank >= nranks)
        return report_error(BF_EINVAL, "bf_p2p_or_merge", "need 1 <= nranks <= BF_P2P_MAX_RANKS, rank < nranks");
    if (bytes % 4) return report_error(BF_EINVAL, "bf_p2p_or_merge", "bytes must be a multiple of 4");
    PeerPtrs pp;
    memset(&pp, 0, sizeof pp);
    for (uint32_t q = 0; q < nranks; ++q) {
        if (!peers[q] || ((uintptr_t)peers[q] & 15))
            return report_error(BF_EINVAL, "bf_p2p_or_merge", "peer pointers must be non-null and 16-byte aligned");
        pp.p[q] = (uint4*)peers[q];
    }
    if (bytes == 0 || nranks == 1) return BF_OK;  // nothing to exchange
    const uint64_t n16 = bytes / 16;
    const uint64_t lo = n16 * rank / nranks, hi = n16 * (rank + 1) / nranks;
    uint64_t tlo = 0, thi = 0;  // 4-byte tail words past the last 16-byte element
    if (rank == nranks - 1) {
        tlo = n16 * 4;
        thi = bytes / 4;
    }
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    constexpr int UNR = 4;
    uint64_t want = (hi - lo + 256 * UNR - 1) / (256 * UNR);
    uint64_t grid = want < (uint64_t)nsm * 4 ? want : (uint64_t)nsm * 4;
    if (grid < 1) grid = 1;
    p2p_or_kernel<UNR><<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(pp, nranks, lo, hi, tlo, thi);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return report_error(BF_ECUDA, "bf_p2p_or_merge launch", cudaGetErrorString(e));
    count_launch();
    return BF_OK;
}

}  // extern "C"
