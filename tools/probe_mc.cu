// Probe: can this box create / bind / map a CUDA multicast object (NVLS) for one device?
#include <cuda.h>
#include <cstdio>
int main() {
  cuInit(0);
  CUdevice dev; cuDeviceGet(&dev, 0);
  CUcontext ctx; cuDevicePrimaryCtxRetain(&ctx, dev); cuCtxSetCurrent(ctx);
  int v = 0;
  cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  printf("multicast supported %d\n", v);
  unsigned long long types[] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC};
  for (int t = 0; t < 3; t++) {
    CUmulticastObjectProp p = {};
    p.numDevices = 1;
    p.handleTypes = types[t];
    p.size = 2 << 20;
    size_t g = 0;
    CUresult r = cuMulticastGetGranularity(&g, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    const char *s = nullptr; cuGetErrorName(r, &s);
    printf("type %llu granularity %zu (%s)\n", types[t], g, s);
    CUmemGenericAllocationHandle mc;
    r = cuMulticastCreate(&mc, &p);
    cuGetErrorName(r, &s);
    printf("type %llu create: %s\n", types[t], s);
    if (r != CUDA_SUCCESS) continue;
    r = cuMulticastAddDevice(mc, dev); cuGetErrorName(r, &s); printf("  add device: %s\n", s);
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
    ap.requestedHandleTypes = (CUmemAllocationHandleType)types[t];
    CUmemGenericAllocationHandle mh;
    r = cuMemCreate(&mh, p.size, &ap, 0); cuGetErrorName(r, &s); printf("  mem create: %s\n", s);
    r = cuMulticastBindMem(mc, 0, mh, 0, p.size, 0); cuGetErrorName(r, &s); printf("  bind: %s\n", s);
    CUdeviceptr va; r = cuMemAddressReserve(&va, p.size, p.size, 0, 0); cuGetErrorName(r, &s); printf("  reserve: %s\n", s);
    r = cuMemMap(va, p.size, 0, mc, 0); cuGetErrorName(r, &s); printf("  map mc: %s\n", s);
    CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    r = cuMemSetAccess(va, p.size, &ad, 1); cuGetErrorName(r, &s); printf("  set access: %s\n", s);
  }
  return 0;
}
