"""Probe which multicast-object properties this driver accepts (dev script)."""
from cuda.bindings import driver as drv
drv.cuInit(0)
err, dev = drv.cuDeviceGet(0)
err, ctx = drv.cuDevicePrimaryCtxRetain(dev)
drv.cuCtxSetCurrent(ctx)
H = drv.CUmemAllocationHandleType
for nd in (1, 2):
    for ht in (H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, H.CU_MEM_HANDLE_TYPE_FABRIC):
        for size in (2 << 20, 512 << 20):
            p = drv.CUmulticastObjectProp()
            p.numDevices = nd
            p.handleTypes = ht
            p.flags = 0
            p.size = size
            e1, g = drv.cuMulticastGetGranularity(p, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
            e2, g2 = drv.cuMulticastGetGranularity(p, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
            e3, h = drv.cuMulticastCreate(p)
            print(nd, ht, size, e1, g, e2, g2, e3)
