"""Probe which multicast object properties the driver accepts on this box."""
from cuda.bindings import driver as d
import torch
torch.cuda.init(); torch.zeros(1, device="cuda")
H = d.CUmemAllocationHandleType
for nd in (1, 2, 8):
    for ht in (H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, H.CU_MEM_HANDLE_TYPE_FABRIC, H.CU_MEM_HANDLE_TYPE_NONE):
        p = d.CUmulticastObjectProp()
        p.numDevices = nd
        p.handleTypes = ht
        p.size = 1 << 21
        e, g = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        e2, gm = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        p.size = max(int(g), 1 << 21)
        e3, h = d.cuMulticastCreate(p)
        ex = None
        if e3 == d.CUresult.CUDA_SUCCESS and ht == H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR:
            ex = d.cuMemExportToShareableHandle(h, ht, 0)[0]
        if e3 == d.CUresult.CUDA_SUCCESS and ht != H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR and ht != H.CU_MEM_HANDLE_TYPE_NONE:
            ex = d.cuMemExportToShareableHandle(h, ht, 0)[0]
        ad = None
        if e3 == d.CUresult.CUDA_SUCCESS:
            ad = d.cuMulticastAddDevice(h, 0)[0]
        print(f"nd={nd} ht={ht.name} gran={e.name}:{int(g)} min={int(gm)} create={e3.name} export={ex} add={ad}", flush=True)
