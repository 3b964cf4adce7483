// probe_mc.cu — does this box support NVSwitch multicast objects, and does a
// one-device multicast team work (cuMulticastCreate / AddDevice / BindMem /
// map the MC address / multimem.st from a kernel / read back through the
// unicast mapping)?  (probe, not product code)
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/probe_mc.cu -o /tmp/probe_mc -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char *s; cuGetErrorString(r_, &s); \
  printf("{\"step\":\"%s\",\"error\":\"%s\"}\n", #x, s); return 1; } } while (0)

__global__ void mc_store(uint4 *mc, const uint4 *src, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = src[i];
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
  }
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  int mc = 0, ndev = 0;
  cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  cudaGetDeviceCount(&ndev);
  printf("{\"multicast_supported\":%d,\"devices\":%d}\n", mc, ndev);
  if (!mc) return 0;
  cudaSetDevice(0);
  cudaFree(0);
  const size_t want = 64ull << 20;
  CUmulticastObjectProp p;
  memset(&p, 0, sizeof p);
  p.numDevices = 1;
  p.size = want;
  p.handleTypes = getenv("MC_HT") ? (CUmemAllocationHandleType)atoi(getenv("MC_HT")) : CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CK(cuMulticastGetGranularity(&gran, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  p.size = (want + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle mh;
  CK(cuMulticastCreate(&mh, &p));
  CK(cuMulticastAddDevice(mh, dev));
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof ap);
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t ugran = 0;
  CK(cuMemGetAllocationGranularity(&ugran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  CUmemGenericAllocationHandle ph;
  CK(cuMemCreate(&ph, p.size, &ap, 0));
  CK(cuMulticastBindMem(mh, 0, ph, 0, p.size, 0));
  CUdeviceptr uva, mva;
  CK(cuMemAddressReserve(&uva, p.size, 0, 0, 0));
  CK(cuMemMap(uva, p.size, 0, ph, 0));
  CUmemAccessDesc ad;
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uva, p.size, &ad, 1));
  CK(cuMemAddressReserve(&mva, p.size, 0, 0, 0));
  CK(cuMemMap(mva, p.size, 0, mh, 0));
  CK(cuMemSetAccess(mva, p.size, &ad, 1));
  std::vector<uint32_t> h(want / 4);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint32_t)(i * 2654435761u) | (i % 7 == 0 ? 0x7FC00001u : 0u);
  void *src;
  cudaMalloc(&src, want);
  cudaMemcpy(src, h.data(), want, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mc_store<<<148 * 4, 256>>>((uint4 *)mva, (const uint4 *)src, want / 16);
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) mc_store<<<148 * 4, 256>>>((uint4 *)mva, (const uint4 *)src, want / 16);
  cudaEventRecord(e1);
  cudaError_t ke = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<uint32_t> back(want / 4);
  cudaMemcpy(back.data(), (void *)uva, want, cudaMemcpyDeviceToHost);
  printf("{\"kernel\":\"%s\",\"bytes_equal\":%s,\"GBps_write\":%.1f}\n", cudaGetErrorString(ke),
         memcmp(back.data(), h.data(), want) == 0 ? "true" : "false", 10.0 * want / (ms * 1e-3) / 1e9);
  return 0;
}
