// api_cost.cu — host-side cost of the CUDA runtime calls on the submit path
// (event record / query / elapsed, stream wait, kernel launch, async copy).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/api_cost tools/api_cost.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

__global__ void noop(int *p) {
  if (p && threadIdx.x == 1024) *p = 0;
}
__global__ void stamp(unsigned long long *out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  cudaSetDevice(0);
  cudaFree(0);
  const int N = 2000;
  cudaStream_t s, s2;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  std::vector<cudaEvent_t> ev(N), evn(N);
  for (int i = 0; i < N; ++i) {
    cudaEventCreate(&ev[i]);
    cudaEventCreateWithFlags(&evn[i], cudaEventDisableTiming);
  }
  int *d;
  cudaMalloc(&d, 1 << 20);
  unsigned long long *hs;
  cudaHostAlloc(&hs, 4096, cudaHostAllocMapped);
  unsigned long long *ds;
  cudaHostGetDevicePointer(&ds, hs, 0);
  void *hp;
  cudaMallocHost(&hp, 1 << 20);
  double t0;
#define MEASURE(name, ...)                        \
  cudaDeviceSynchronize();                        \
  t0 = now_us();                                  \
  for (int i = 0; i < N; ++i) { __VA_ARGS__; }         \
  printf("%-34s %8.3f us\n", name, (now_us() - t0) / N);
  MEASURE("cudaEventRecord (timing)", cudaEventRecord(ev[i], s));
  MEASURE("cudaEventRecord (no timing)", cudaEventRecord(evn[i], s));
  cudaDeviceSynchronize();
  MEASURE("cudaEventQuery (done)", cudaEventQuery(ev[i]));
  float ms;
  MEASURE("cudaEventElapsedTime", cudaEventElapsedTime(&ms, ev[0], ev[i]));
  MEASURE("cudaStreamWaitEvent", cudaStreamWaitEvent(s2, ev[i], 0));
  MEASURE("noop<<<1,32>>>", noop<<<1, 32, 0, s>>>(d));
  MEASURE("noop<<<148,256>>>", noop<<<148, 256, 0, s>>>(d));
  MEASURE("stamp<<<1,1>>> (globaltimer)", stamp<<<1, 1, 0, s>>>(ds + (i & 255)));
  MEASURE("cudaMemcpyAsync D2H 4KiB", cudaMemcpyAsync(hp, d, 4096, cudaMemcpyDeviceToHost, s));
  MEASURE("cudaMemcpyAsync D2D 4KiB", cudaMemcpyAsync(d + 4096, d, 4096, cudaMemcpyDeviceToDevice, s));
  MEASURE("cudaLaunchHostFunc", cudaLaunchHostFunc(s, [](void *) {}, nullptr));
  MEASURE("cudaFuncSetAttribute (smem 198K)",
          cudaFuncSetAttribute(noop, cudaFuncAttributeMaxDynamicSharedMemorySize, 198 * 1024));
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1, 32, 4);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = 198 * 1024;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 4;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MEASURE("cudaLaunchKernelEx cluster4 198K", cudaLaunchKernelEx(&cfg, noop, d));
    cudaDeviceSynchronize();
    // device time per launch of back-to-back cluster launches
    cudaEventRecord(ev[0], s);
    for (int i = 0; i < 200; ++i) cudaLaunchKernelEx(&cfg, noop, d);
    cudaEventRecord(ev[1], s);
    cudaEventSynchronize(ev[1]);
    cudaEventElapsedTime(&ms, ev[0], ev[1]);
    printf("%-34s %8.3f us\n", "device: cluster4 198K noop each", ms * 1e3 / 200);
    cfg.numAttrs = 0;
    cudaEventRecord(ev[0], s);
    for (int i = 0; i < 200; ++i) cudaLaunchKernelEx(&cfg, noop, d);
    cudaEventRecord(ev[1], s);
    cudaEventSynchronize(ev[1]);
    cudaEventElapsedTime(&ms, ev[0], ev[1]);
    printf("%-34s %8.3f us\n", "device: 198K noop (no cluster) each", ms * 1e3 / 200);
  }
  // globaltimer vs host clock: resolution and offset stability
  cudaDeviceSynchronize();
  for (int k = 0; k < 5; ++k) {
    double h0 = now_us();
    stamp<<<1, 1, 0, s>>>(ds);
    cudaStreamSynchronize(s);
    double h1 = now_us();
    printf("globaltimer %llu ns, host mid %.1f us, round trip %.1f us\n", *(volatile unsigned long long *)hs,
           (h0 + h1) / 2, h1 - h0);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
