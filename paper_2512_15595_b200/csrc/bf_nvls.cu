// bf_nvls.cu -- in-switch OR merge of partial filters over NVLink SHARP
// (SURVEY 8(e) E4, NEXT N4): every rank binds its own physical buffer to one
// multicast object; a kernel on rank r reads its 1/P slice through the
// multicast address with multimem.ld_reduce.or (the NVSwitch ORs the P
// copies) and writes the result back with multimem.st (the switch broadcasts
// it to every rank's copy).  No OR-fold pass over P staged copies, no
// all-to-all: each rank moves M/P in and M/P out over NVLink.
//
// Driver entry points are fetched at run time (cudaGetDriverEntryPoint) so
// the library keeps no link-time dependency on libcuda.
#include <cuda.h>
#include <cuda_runtime.h>
#include <string.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <new>

#include "../../include/bf.h"
#include "bf_internal.h"

namespace bf {

#define BF_DRV(name) static decltype(&name) p_##name = nullptr;
BF_DRV(cuMulticastGetGranularity)
BF_DRV(cuMulticastCreate)
BF_DRV(cuMulticastAddDevice)
BF_DRV(cuMulticastBindMem)
BF_DRV(cuMulticastUnbind)
BF_DRV(cuMemCreate)
BF_DRV(cuMemRelease)
BF_DRV(cuMemAddressReserve)
BF_DRV(cuMemAddressFree)
BF_DRV(cuMemMap)
BF_DRV(cuMemUnmap)
BF_DRV(cuMemSetAccess)
BF_DRV(cuMemExportToShareableHandle)
BF_DRV(cuMemImportFromShareableHandle)
BF_DRV(cuGetErrorString)
#undef BF_DRV

static bool load_driver()
{
    static int state = 0;  // 0 unknown, 1 ok, -1 missing
    if (state) return state > 0;
    bool ok = true;
#define BF_GET(name)                                                                                 \
    {                                                                                                \
        cudaDriverEntryPointQueryResult q;                                                           \
        void* fp = nullptr;                                                                          \
        if (cudaGetDriverEntryPoint(#name, &fp, cudaEnableDefault, &q) != cudaSuccess || !fp) ok = false; \
        p_##name = (decltype(p_##name))fp;                                                           \
    }
    BF_GET(cuMulticastGetGranularity)
    BF_GET(cuMulticastCreate)
    BF_GET(cuMulticastAddDevice)
    BF_GET(cuMulticastBindMem)
    BF_GET(cuMulticastUnbind)
    BF_GET(cuMemCreate)
    BF_GET(cuMemRelease)
    BF_GET(cuMemAddressReserve)
    BF_GET(cuMemAddressFree)
    BF_GET(cuMemMap)
    BF_GET(cuMemUnmap)
    BF_GET(cuMemSetAccess)
    BF_GET(cuMemExportToShareableHandle)
    BF_GET(cuMemImportFromShareableHandle)
    BF_GET(cuGetErrorString)
#undef BF_GET
    state = ok ? 1 : -1;
    return ok;
}

// multimem.ld_reduce / multimem.st are scalar for .or (ptxas rejects .v4 with
// .or): 8 bytes per instruction, grid-stride over the slice
__global__ void __launch_bounds__(256) nvls_or_kernel(unsigned long long* mc, uint64_t lo8, uint64_t hi8)
{
    constexpr int U = 4;  // switch round trips in flight per thread
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = lo8 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < hi8; i += U * stride) {
        unsigned long long v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            asm volatile("multimem.ld_reduce.relaxed.sys.global.or.b64 %0, [%1];"
                         : "=l"(v[u])
                         : "l"(mc + i + u * stride)
                         : "memory");
#pragma unroll
        for (int u = 0; u < U; ++u)
            asm volatile("multimem.st.relaxed.sys.global.b64 [%0], %1;" ::"l"(mc + i + u * stride), "l"(v[u]) : "memory");
    }
    for (; i < hi8; i += stride) {
        unsigned long long v;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.or.b64 %0, [%1];" : "=l"(v) : "l"(mc + i) : "memory");
        asm volatile("multimem.st.relaxed.sys.global.b64 [%0], %1;" ::"l"(mc + i), "l"(v) : "memory");
    }
}

}  // namespace bf

using namespace bf;

struct bf_mcast {
    int device;
    uint32_t nranks;
    uint64_t size;  // rounded to the multicast granularity
    CUmemGenericAllocationHandle mc_handle, mem_handle;
    CUdeviceptr uc_ptr, mc_ptr;
    int htype;
    int export_fd = -1;
    bool added, bound, uc_mapped, mc_mapped;
};

static int drv_fail(CUresult r, const char* what)
{
    const char* s = nullptr;
    if (p_cuGetErrorString) p_cuGetErrorString(r, &s);
    return report_error(BF_ECUDA, what, s ? s : "driver error");
}

extern "C" {

static CUmemAllocationHandleType htype(int t)
{
    return t == BF_MCAST_FABRIC ? CU_MEM_HANDLE_TYPE_FABRIC : CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
}

int bf_mcast_create(uint64_t bytes, uint32_t nranks, int handle_type, int exporter, void* handle,
                    bf_mcast** out)
{
    if (!out || !handle || bytes == 0 || nranks < 1 || (handle_type != BF_MCAST_FABRIC && handle_type != BF_MCAST_POSIX_FD))
        return report_error(BF_EINVAL, "bf_mcast_create", "bad arguments");
    if (!load_driver()) return report_error(BF_EUNSUPPORTED, "bf_mcast_create", "driver multicast API missing");
    int dev = 0;
    cudaGetDevice(&dev);
    cudaFree(nullptr);  // make sure the primary context exists
    int mc_ok = 0;
    cudaDeviceGetAttribute(&mc_ok, (cudaDeviceAttr)CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    if (!mc_ok) return report_error(BF_EUNSUPPORTED, "bf_mcast_create", "device has no multicast support");
    bf_mcast* m = new (std::nothrow) bf_mcast();
    if (!m) return report_error(BF_ENOMEM, "bf_mcast_create", "host allocation");
    m->device = dev;
    m->nranks = nranks;
    m->htype = handle_type;
    CUmulticastObjectProp prop;
    memset(&prop, 0, sizeof prop);
    prop.numDevices = nranks;
    prop.handleTypes = htype(handle_type);
    prop.size = bytes;
    size_t gran = 0;
    CUresult r = p_cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS) {
        delete m;
        return drv_fail(r, "cuMulticastGetGranularity");
    }
    m->size = (bytes + gran - 1) / gran * gran;
    prop.size = m->size;
    if (exporter) {
        r = p_cuMulticastCreate(&m->mc_handle, &prop);
        if (r == CUDA_SUCCESS) {
            if (handle_type == BF_MCAST_FABRIC) {
                r = p_cuMemExportToShareableHandle(handle, m->mc_handle, CU_MEM_HANDLE_TYPE_FABRIC, 0);
            } else {
                int fd = -1;
                r = p_cuMemExportToShareableHandle(&fd, m->mc_handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
                int32_t blob[2] = {(int32_t)getpid(), fd};
                memset(handle, 0, BF_MCAST_HANDLE_BYTES);
                memcpy(handle, blob, sizeof blob);
                m->export_fd = fd;
            }
        }
    } else if (handle_type == BF_MCAST_FABRIC) {
        r = p_cuMemImportFromShareableHandle(&m->mc_handle, handle, CU_MEM_HANDLE_TYPE_FABRIC);
    } else {
        // the exporter's fd lives in its process: duplicate it into ours
        int32_t blob[2];
        memcpy(blob, handle, sizeof blob);
        int pidfd = (int)syscall(SYS_pidfd_open, blob[0], 0);
        int fd = pidfd < 0 ? -1 : (int)syscall(SYS_pidfd_getfd, pidfd, blob[1], 0);
        if (pidfd >= 0) close(pidfd);
        if (fd < 0) {
            delete m;
            return report_error(BF_ECUDA, "bf_mcast_create", "pidfd_getfd failed (exporter fd not reachable)");
        }
        r = p_cuMemImportFromShareableHandle(&m->mc_handle, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
        close(fd);
    }
    if (r != CUDA_SUCCESS) {
        if (m->mc_handle) p_cuMemRelease(m->mc_handle);
        if (m->export_fd >= 0) close(m->export_fd);
        delete m;
        return drv_fail(r, exporter ? "cuMulticastCreate/export" : "cuMemImportFromShareableHandle");
    }
    *out = m;
    return BF_OK;
}

int bf_mcast_add_device(bf_mcast* m)
{
    if (!m) return report_error(BF_EINVAL, "bf_mcast_add_device", "null");
    CUresult r = p_cuMulticastAddDevice(m->mc_handle, (CUdevice)m->device);
    if (r != CUDA_SUCCESS) return drv_fail(r, "cuMulticastAddDevice");
    m->added = true;
    return BF_OK;
}

int bf_mcast_bind(bf_mcast* m, void** uc_ptr)
{
    if (!m || !uc_ptr || !m->added) return report_error(BF_EINVAL, "bf_mcast_bind", "add the device first");
    CUmemAllocationProp ap;
    memset(&ap, 0, sizeof ap);
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = m->device;
    ap.requestedHandleTypes = htype(m->htype);
    CUresult r = p_cuMemCreate(&m->mem_handle, m->size, &ap, 0);
    if (r != CUDA_SUCCESS) return drv_fail(r, "cuMemCreate");
    r = p_cuMulticastBindMem(m->mc_handle, 0, m->mem_handle, 0, m->size, 0);
    if (r != CUDA_SUCCESS) return drv_fail(r, "cuMulticastBindMem");
    m->bound = true;
    CUmemAccessDesc acc;
    memset(&acc, 0, sizeof acc);
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = m->device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    // unicast view of the local copy
    if ((r = p_cuMemAddressReserve(&m->uc_ptr, m->size, 0, 0, 0)) != CUDA_SUCCESS) return drv_fail(r, "reserve uc");
    if ((r = p_cuMemMap(m->uc_ptr, m->size, 0, m->mem_handle, 0)) != CUDA_SUCCESS) return drv_fail(r, "map uc");
    if ((r = p_cuMemSetAccess(m->uc_ptr, m->size, &acc, 1)) != CUDA_SUCCESS) return drv_fail(r, "access uc");
    m->uc_mapped = true;
    // multicast view (every rank's copy at once)
    if ((r = p_cuMemAddressReserve(&m->mc_ptr, m->size, 0, 0, 0)) != CUDA_SUCCESS) return drv_fail(r, "reserve mc");
    if ((r = p_cuMemMap(m->mc_ptr, m->size, 0, m->mc_handle, 0)) != CUDA_SUCCESS) return drv_fail(r, "map mc");
    if ((r = p_cuMemSetAccess(m->mc_ptr, m->size, &acc, 1)) != CUDA_SUCCESS) return drv_fail(r, "access mc");
    m->mc_mapped = true;
    *uc_ptr = (void*)m->uc_ptr;
    return BF_OK;
}

int bf_mcast_or_reduce(bf_mcast* m, uint32_t rank, uint64_t bytes, void* stream)
{
    if (!m || !m->mc_mapped || rank >= m->nranks || bytes > m->size || (bytes & 7))
        return report_error(BF_EINVAL, "bf_mcast_or_reduce", "bad arguments");
    const uint64_t n8 = bytes / 8;
    const uint64_t lo = n8 * rank / m->nranks, hi = n8 * (rank + 1) / m->nranks;
    if (hi > lo) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device);
        nvls_or_kernel<<<4 * sms, 256, 0, (cudaStream_t)stream>>>((unsigned long long*)m->mc_ptr, lo, hi);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return report_error(BF_ECUDA, "nvls_or_kernel launch", cudaGetErrorString(e));
        count_launch();
    }
    return BF_OK;
}

int bf_mcast_mc_ptr(bf_mcast* m, void** mc_ptr, uint64_t* size)
{
    if (!m || !m->mc_mapped) return report_error(BF_EINVAL, "bf_mcast_mc_ptr", "not bound");
    if (mc_ptr) *mc_ptr = (void*)m->mc_ptr;
    if (size) *size = m->size;
    return BF_OK;
}

void bf_mcast_destroy(bf_mcast* m)
{
    if (!m || !load_driver()) return;
    if (m->mc_mapped) {
        p_cuMemUnmap(m->mc_ptr, m->size);
        p_cuMemAddressFree(m->mc_ptr, m->size);
    }
    if (m->uc_mapped) {
        p_cuMemUnmap(m->uc_ptr, m->size);
        p_cuMemAddressFree(m->uc_ptr, m->size);
    }
    if (m->bound) p_cuMulticastUnbind(m->mc_handle, (CUdevice)m->device, 0, m->size);
    if (m->mem_handle) p_cuMemRelease(m->mem_handle);
    if (m->mc_handle) p_cuMemRelease(m->mc_handle);
    if (m->export_fd >= 0) close(m->export_fd);
    delete m;
}

}  // extern "C"
