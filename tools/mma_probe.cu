// mma_probe.cu — issue rate of tcgen05.mma kind::tf32 (M128 x N x K8) with
// operands already in shared memory (probe, not product code): one CTA per
// SM, a single thread issues `iters` MMAs back to back on the same smem
// tiles, then one commit; the kernel time / (iters x CTAs) gives clk per MMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_probe.cu -o /tmp/mma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int BN, int KIND>   // KIND 0: tf32 (K=8), 1: f16/bf16 (K=16)
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long *clk_out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < (128 + BN) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(base)[i] = 0x3f800000u;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t tmem = tslot;
    const uint32_t idesc = (1u << 4) | ((KIND == 0 ? 2u : 1u) << 7) | ((KIND == 0 ? 2u : 1u) << 10) |
                           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = desc_sw128(smem_u32(base)), db = desc_sw128(smem_u32(base + 128 * 128));
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t a = da + (uint64_t)(2 * (i & 3)), b = db + (uint64_t)(2 * (i & 3));
      if (KIND == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(a), "l"(b), "r"(idesc), "r"(i));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(a), "l"(b), "r"(idesc), "r"(i));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
                     smem_u32(&bar))
                 : "memory");
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *clk_out = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(BN));
}

template <int BN, int KIND>
void run(const char *name, int sms) {
  const int iters = 4096;
  const int smem = (128 + BN) * 128 + 2048;
  cudaFuncSetAttribute(mma_loop<BN, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long *d;
  cudaMalloc(&d, 8);
  mma_loop<BN, KIND><<<sms, 128, smem>>>(64, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_loop<BN, KIND><<<sms, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long clk = 0;
  cudaMemcpy(&clk, d, 8, cudaMemcpyDeviceToHost);
  const double flop = 2.0 * 128 * BN * (KIND == 0 ? 8 : 16) * iters * sms;
  printf("{\"mma\":\"%s\",\"N\":%d,\"err\":\"%s\",\"clk_per_mma\":%.1f,\"TFLOPs\":%.1f}\n", name, BN,
         cudaGetErrorString(err), (double)clk / iters, flop / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<256, 0>("tf32 M128 K8", sms);
  run<128, 0>("tf32 M128 K8", sms);
  run<256, 1>("bf16 M128 K16", sms);
  return 0;
}
