"""Probe: does this B200 box support NVLS multicast objects (cuMulticast*) for one device?
Prints one JSON line.  Used to decide whether the multimem exchange path can be tested on the
1-GPU gpurun boxes."""
import json

from cuda.bindings import driver as d


def ok(r):
    err = r[0] if isinstance(r, tuple) else r
    return err == d.CUresult.CUDA_SUCCESS, (r[1:] if isinstance(r, tuple) else ())


out = {}
d.cuInit(0)
_, dev = d.cuDeviceGet(0)
_, ctx = d.cuDevicePrimaryCtxRetain(dev)
d.cuCtxSetCurrent(ctx)
for a in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED",
          "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED"):
    r = d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, a), dev)
    out[a] = int(r[1]) if r[0] == d.CUresult.CUDA_SUCCESS else str(r[0])
try:
    prop = d.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
    prop.size = 2 << 20
    r = d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
    out["mc_granularity"] = int(r[1]) if r[0] == d.CUresult.CUDA_SUCCESS else str(r[0])
    g = int(r[1]) if r[0] == d.CUresult.CUDA_SUCCESS else (2 << 20)
    prop.size = g
    r = d.cuMulticastCreate(prop)
    out["mc_create"] = str(r[0])
    if r[0] == d.CUresult.CUDA_SUCCESS:
        mc = r[1]
        out["mc_add_device"] = str(d.cuMulticastAddDevice(mc, dev)[0])
        ap = d.CUmemAllocationProp()
        ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = 0
        ap.requestedHandleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        r2 = d.cuMemCreate(g, ap, 0)
        out["mem_create"] = str(r2[0])
        if r2[0] == d.CUresult.CUDA_SUCCESS:
            out["mc_bind"] = str(d.cuMulticastBindMem(mc, 0, r2[1], 0, g, 0)[0])
            r3 = d.cuMemAddressReserve(g, g, 0, 0)
            out["va_reserve"] = str(r3[0])
            if r3[0] == d.CUresult.CUDA_SUCCESS:
                out["mc_map"] = str(d.cuMemMap(r3[1], g, 0, mc, 0)[0])
            r4 = d.cuMemExportToShareableHandle(mc, d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0)
            out["mc_export_fd"] = str(r4[0])
except Exception as e:  # noqa: BLE001
    out["exception"] = repr(e)
print(json.dumps(out))
