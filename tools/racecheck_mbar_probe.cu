// racecheck_mbar_probe.cu -- does compute-sanitizer racecheck model the
// mbarrier handoff of a bulk copy (cp.async.bulk -> complete_tx -> try_wait)
// and of a plain st.shared released by mbarrier.arrive?  One producer lane,
// 4 consumer warps, ONE use of the buffer (no reuse, so no WAR at all): any
// hazard reported here is one racecheck cannot see through.  (probe)
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/racecheck_mbar_probe.cu -o /tmp/rp
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void probe(const float *x, float *out, int tail) {
  __shared__ __align__(128) float buf[1024 + 4];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 128) {   // producer (warp 4)
    if (tail) buf[1024] = x[1024];   // plain store, released by the arrive below
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(4096) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(buf)),
                 "l"(x), "r"(4096), "r"(sa(&bar))
                 : "memory");
  } else if (threadIdx.x < 128) {
    asm volatile("{\n.reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}" ::"r"(
                     sa(&bar))
                 : "memory");
    float s = 0;
    for (int i = threadIdx.x; i < 1024; i += 128) s += buf[i];
    if (tail) s += buf[1024];
    out[threadIdx.x] = s;
  }
}
int main() {
  float *x, *out;
  cudaMalloc(&x, 8192); cudaMalloc(&out, 4096); cudaMemset(x, 0, 8192);
  probe<<<1, 160>>>(x, out, 0);
  probe<<<1, 160>>>(x, out, 1);
  printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
