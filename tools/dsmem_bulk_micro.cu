// dsmem_bulk_micro.cu -- smem -> peer smem bandwidth inside a cluster with the
// bulk-copy engine (cp.async.bulk.shared::cluster.shared::cta, mbarrier
// complete_tx on the receiver) vs LSU remote loads (ld.shared::cluster.v4):
// the split-K exchange of the tcgen05 sgemm (4 CTAs, each sending three 32 KB
// quarter-tiles and receiving three).  (probe, not product code)
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/dsmem_bulk_micro.cu -o /tmp/db
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t rank_() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
constexpr int Q = 32 * 1024;   // one quarter-tile
template <int NZ, bool BULK>
__global__ void exch(float *out, int reps) {
  extern __shared__ __align__(128) unsigned char sm[];   // [NZ quarters of my partial][NZ-1 receive slots]
  __shared__ uint64_t bar;
  const uint32_t me = rank_();
  for (int i = threadIdx.x; i < NZ * Q / 4; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = (float)(me + 1);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  csync();
  float acc = 0;
  for (int r = 0; r < reps; ++r) {
    if (BULK) {
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"((NZ - 1) * Q) : "memory");
      }
      csync();   // every receiver armed (and done reading last round's slots)
      if (threadIdx.x < NZ && threadIdx.x != me) {
        const uint32_t q = threadIdx.x;
        const uint32_t slot = me < q ? me : me - 1;   // my slot index at receiver q
        uint32_t dst, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(sa(sm + NZ * Q + slot * Q)), "r"(q));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(sa(&bar)), "r"(q));
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "r"(sa(sm + q * Q)), "r"(Q), "r"(rb)
                     : "memory");
      }
      asm volatile("{\n.reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(
                       sa(&bar)), "r"(r & 1)
                   : "memory");
      // sum own quarter + received slots (local smem)
      for (int i = threadIdx.x; i < Q / 16; i += blockDim.x) {
        float4 v = reinterpret_cast<const float4 *>(sm + me * Q)[i];
        for (int k = 0; k < NZ - 1; ++k) {
          float4 w = reinterpret_cast<const float4 *>(sm + NZ * Q + k * Q)[i];
          v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
        }
        acc += v.x + v.y + v.z + v.w;
      }
      if (threadIdx.x < NZ) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    } else {
      csync();
      for (int i = threadIdx.x; i < Q / 16; i += blockDim.x) {
        float4 v = make_float4(0, 0, 0, 0);
        for (int q = 0; q < NZ; ++q) {
          uint32_t ra;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(sa(sm + me * Q + i * 16)), "r"(q));
          float4 w;
          asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(w.x), "=f"(w.y), "=f"(w.z), "=f"(w.w) : "r"(ra));
          v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
        }
        acc += v.x + v.y + v.z + v.w;
      }
    }
    csync();
  }
  if (acc == 1234.5f) out[blockIdx.x] = acc;
}
template <int NZ, bool BULK>
void run(const char *name, float *out, int reps) {
  auto k = exch<NZ, BULK>;
  const int smem = (2 * NZ - 1) * Q;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(128); cfg.blockDim = dim3(192); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = NZ; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.attrs = a; cfg.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::vector<float> ts;
  for (int rr = 0; rr < 5; ++rr) {
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k, out, reps);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ts.push_back(ms * 1e3f);
  }
  std::sort(ts.begin(), ts.end());
  const double bytes_in_per_cta = (double)(NZ - 1) * Q * reps;
  printf("{\"case\":\"%s\",\"cluster\":%d,\"reps\":%d,\"us\":%.2f,\"us_per_exchange\":%.2f,\"GBps_in_per_sm\":%.1f,\"err\":\"%s\"}\n",
         name, NZ, reps, ts[2], ts[2] / reps, bytes_in_per_cta / (ts[2] / 1e6) / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  float *out; cudaMalloc(&out, 4096);
  run<4, true>("bulk_push_then_local_sum", out, 50);
  run<4, false>("lsu_remote_pull_sum", out, 50);
  run<2, true>("bulk_push_then_local_sum", out, 50);
  run<2, false>("lsu_remote_pull_sum", out, 50);
  return 0;
}
