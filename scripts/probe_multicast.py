"""Probe the driver's multicast object support on this box (cuda-python): granularities and which
cuMulticastCreate property combinations succeed."""
from cuda.bindings import driver as d

d.cuInit(0)
err, dev = d.cuDeviceGet(0)
err, ctx = d.cuDevicePrimaryCtxRetain(dev)
d.cuCtxSetCurrent(ctx)
print("multicast supported", d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
for ht_name in ("CU_MEM_HANDLE_TYPE_NONE", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_FABRIC"):
    for nd in (1, 2):
        p = d.CUmulticastObjectProp()
        p.numDevices = nd
        p.handleTypes = getattr(d.CUmemAllocationHandleType, ht_name)
        p.size = 2 << 20
        e1, gmin = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        e2, grec = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        p.size = max(gmin if e1 == 0 else 0, 2 << 20)
        e3, h = d.cuMulticastCreate(p)
        print(ht_name, "devices", nd, "gran", e1, gmin, e2, grec, "size", p.size, "create", e3)
        if e3 == d.CUresult.CUDA_SUCCESS:
            e4 = d.cuMulticastAddDevice(h, dev)
            print("   add device", e4)
            d.cuMemRelease(h)
