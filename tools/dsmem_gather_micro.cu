// dsmem_gather_micro.cu -- random 4-B gathers from distributed shared memory
// (x spread over a cluster's CTAs, ld.shared::cluster) vs the L2 gather
// ceiling.  Decides whether spmv can keep CSR and read x from the cluster.
// (probe, not product code)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/dsmem_gather_micro.cu -o /tmp/dg
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t hsh(uint32_t v) {
  v ^= v >> 16; v *= 0x7feb352dU; v ^= v >> 15; v *= 0x846ca68bU; v ^= v >> 16; return v;
}
__device__ __forceinline__ uint32_t cluster_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// each CTA holds `per` floats; gathers pick a random global index in [0, per*CS)
template <int CS, bool LOCAL_ONLY>
__global__ void dsmem_gather(const float *x, int per, int gathers_per_thread, float *out) {
  extern __shared__ float sm[];
  for (int i = threadIdx.x; i < per; i += blockDim.x) sm[i] = x[cluster_rank() * per + i];
  cluster_sync();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  float s = 0;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < gathers_per_thread; k += 4) {
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint32_t idx = hsh(t * 7919u + k + u) % (uint32_t)(per * CS);
      uint32_t rank = LOCAL_ONLY ? cluster_rank() : idx / per, off = idx % per;
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base + 4 * off), "r"(rank));
      asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v[u]) : "r"(ra));
    }
    s += (v[0] + v[1]) + (v[2] + v[3]);
  }
  cluster_sync();
  if (s == 1234.5f) out[t] = s;
}
template <int CS, bool LO>
void run(const char *name, const float *x, float *out, int per, int blocks, int threads, int g) {
  auto k = dsmem_gather<CS, LO>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, per * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = per * 4;
  cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = CS; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.attrs = a; cfg.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::vector<float> ts;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    cudaError_t le = cudaLaunchKernelEx(&cfg, k, x, per, g, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    if (le != cudaSuccess) { printf("{\"case\":\"%s\",\"error\":\"%s\"}\n", name, cudaGetErrorString(le)); return; }
    float ms; cudaEventElapsedTime(&ms, e0, e1); ts.push_back(ms * 1e3f);
  }
  std::sort(ts.begin(), ts.end());
  double n = (double)blocks * threads * g;
  printf("{\"case\":\"%s\",\"cluster\":%d,\"KiB_per_cta\":%d,\"blocks\":%d,\"us\":%.2f,\"G_gathers_per_s\":%.1f,\"err\":\"%s\"}\n", name,
         CS, per * 4 / 1024, blocks, ts[2], n / ts[2] / 1e3, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  float *x, *out; cudaMalloc(&x, 64 << 20); cudaMemset(x, 0, 64 << 20); cudaMalloc(&out, 64 << 20);
  const int g = 64;  // gathers per thread
  // 16.7 M gathers total in each case where possible
  run<16, false>("dsmem16_random", x, out, 56 * 1024, 144, 1024, 112);
  run<16, true>("dsmem16_local_only", x, out, 56 * 1024, 144, 1024, 112);
  run<8, false>("dsmem8_random", x, out, 56 * 1024, 144, 1024, 112);
  run<4, false>("dsmem4_random", x, out, 56 * 1024, 144, 1024, 112);
  run<2, false>("dsmem2_random", x, out, 56 * 1024, 148, 1024, 112);
  run<1, false>("smem_local", x, out, 56 * 1024, 148, 1024, 112);
  (void)g;
  return 0;
}
