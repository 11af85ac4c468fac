"""Probe: can this box create, bind and map an NVLink SHARP (NVLS) multicast object across its GPUs?
One process, every visible GPU, cuda-python driver bindings. Prints one line per step."""
import sys

from cuda.bindings import driver as cu


def chk(r, what):
    err = r[0] if isinstance(r, tuple) else r
    if err != cu.CUresult.CUDA_SUCCESS:
        print(f"{what}: {err}")
        sys.exit(0)
    return r[1:] if isinstance(r, tuple) and len(r) > 2 else (r[1] if isinstance(r, tuple) and len(r) == 2 else None)


chk(cu.cuInit(0), "cuInit")
n = chk(cu.cuDeviceGetCount(), "count")
devs = [chk(cu.cuDeviceGet(i), "dev") for i in range(n)]
for d in devs:
    ms = chk(cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d), "attr")
    print("device", int(d), "multicast supported:", ms)
prop = cu.CUmulticastObjectProp()
prop.numDevices = n
prop.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
prop.size = 1 << 21
gran = chk(cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED),
           "granularity")
print("granularity", gran)
prop.size = max(gran, 1 << 21)
mc = chk(cu.cuMulticastCreate(prop), "cuMulticastCreate")
print("created")
for d in devs:
    chk(cu.cuMulticastAddDevice(mc, d), "cuMulticastAddDevice")
print("added", n)
ctxs = []
for d in devs:
    ctx = chk(cu.cuDevicePrimaryCtxRetain(d), "ctx")
    chk(cu.cuCtxSetCurrent(ctx), "setctx")
    ap = cu.CUmemAllocationProp()
    ap.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    ap.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    ap.location.id = int(d)
    ap.requestedHandleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
    mem = chk(cu.cuMemCreate(prop.size, ap, 0), "cuMemCreate")
    chk(cu.cuMulticastBindMem(mc, 0, mem, 0, prop.size, 0), "cuMulticastBindMem")
    print("bound device", int(d))
print("MULTICAST OK")
