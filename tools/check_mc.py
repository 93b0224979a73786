import torch
from cuda.bindings import driver as cu
cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED", "CU_DEVICE_ATTRIBUTE_L2_CACHE_SIZE",
             "CU_DEVICE_ATTRIBUTE_MAX_PERSISTING_L2_CACHE_SIZE"):
    a = getattr(cu.CUdevice_attribute, name, None)
    print(name, cu.cuDeviceGetAttribute(a, dev) if a is not None else "n/a")
print(torch.cuda.get_device_properties(0))
