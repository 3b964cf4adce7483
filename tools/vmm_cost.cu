// vmm_cost.cu — host cost of the VMM calls behind one pool segment
// (cuMemCreate / AddressReserve / Map / SetAccess) as the number of live
// mappings grows, with and without a POSIX-FD-exportable handle.  Probe.
// nvcc -O2 -o /tmp/vmm_cost tools/vmm_cost.cu -lcuda
#include <cuda.h>
#include <chrono>
#include <cstdio>
#include <vector>
static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
int main(int argc, char **argv) {
  cuInit(0);
  CUdevice dev;
  cuDeviceGet(&dev, 0);
  CUcontext ctx;
  cuDevicePrimaryCtxRetain(&ctx, dev);
  cuCtxSetCurrent(ctx);
  const size_t sz = (argc > 1 ? atoll(argv[1]) : 10) << 20;
  for (int shareable = 0; shareable < 2; ++shareable) {
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = 0;
    if (shareable) prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
    const size_t phys = (sz + gran - 1) / gran * gran;
    std::vector<std::pair<CUdeviceptr, CUmemGenericAllocationHandle>> live;
    double t[4] = {0, 0, 0, 0};
    for (int i = 0; i < 600; ++i) {
      CUmemGenericAllocationHandle h;
      CUdeviceptr va;
      double a = now_us();
      cuMemCreate(&h, phys, &prop, 0);
      double b = now_us();
      cuMemAddressReserve(&va, phys, gran, 0, 0);
      double c = now_us();
      cuMemMap(va, phys, 0, h, 0);
      double d = now_us();
      CUmemAccessDesc acc{};
      acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      acc.location.id = 0;
      acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
      cuMemSetAccess(va, phys, &acc, 1);
      double e = now_us();
      t[0] += b - a; t[1] += c - b; t[2] += d - c; t[3] += e - d;
      live.emplace_back(va, h);
      if ((i + 1) % 100 == 0) {
        printf("{\"shareable\":%d,\"seg_MiB\":%zu,\"live\":%d,\"create_us\":%.1f,\"reserve_us\":%.1f,\"map_us\":%.1f,\"setaccess_us\":%.1f}\n",
               shareable, phys >> 20, i + 1, t[0] / 100, t[1] / 100, t[2] / 100, t[3] / 100);
        t[0] = t[1] = t[2] = t[3] = 0;
      }
    }
    double a = now_us();
    for (auto &p : live) { cuMemUnmap(p.first, phys); cuMemAddressFree(p.first, phys); cuMemRelease(p.second); }
    printf("{\"shareable\":%d,\"release_all_us_per_seg\":%.1f}\n", shareable, (now_us() - a) / live.size());
  }
  return 0;
}
