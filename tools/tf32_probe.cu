// tf32_probe.cu — how does tcgen05.mma kind::tf32 read an fp32 operand whose
// low 13 mantissa bits are not zero?  (probe, not product code)
//
// A is 128 x 32 fp32 (one K-major SWIZZLE_128B tile), B is 64 x 32; one MMA
// with K = 8.  Row r of A holds x_r at k = 0 and zeros elsewhere; B holds 1.0
// at (n = 0, k = 0).  D[r][0] = T(x_r) where T is the hardware's fp32 -> tf32
// reading.  x = 1 + f*u with u = 2^-10 (the tf32 ulp at 1):
//   f      trunc   rne     rna
//   0.75   1       1+u     1+u
//   0.5    1       1       1+u
//   1.5    1+u     1+2u    1+2u
//   0.25   1       1       1
// The 3xTF32 sgemm needs to know T to form lo = x - T(x) without rewriting x.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tf32_probe.cu -o /tmp/tf32_probe
#include <cstdio>
#include <cstdint>
#include <cstring>
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
// element (r, k) of a K-major SWIZZLE_128B tile of 32-fp32 rows
__device__ __forceinline__ int sw_off(int r, int k) { return r * 128 + (((k >> 2) ^ (r & 7)) << 4) + (k & 3) * 4; }

__global__ void __launch_bounds__(128, 1) probe(const float *xa, float *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~(uintptr_t)1023);
  uint8_t *sa = base, *sb = base + 128 * 128;
  for (int i = threadIdx.x; i < (128 + 64) * 32; i += blockDim.x) reinterpret_cast<float *>(base)[i] = 0.f;
  __syncthreads();
  const int r = threadIdx.x;
  *reinterpret_cast<float *>(sa + sw_off(r, 0)) = xa[r];
  if (r == 0) *reinterpret_cast<float *>(sb + sw_off(0, 0)) = 1.0f;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(64));
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
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                 "l"(desc_sw128(smem_u32(sa))), "l"(desc_sw128(smem_u32(sb))), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
                   smem_u32(&bar))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  out[r] = __uint_as_float(v);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
  const double u = 1.0 / 1024;
  const double fr[4] = {0.75, 0.5, 1.5, 0.25};
  float hx[128];
  for (int r = 0; r < 128; ++r) {
    const double f = fr[r & 3];
    hx[r] = (float)((r & 4) ? -(1.0 + f * u) : (1.0 + f * u));
  }
  float *dx, *dout;
  cudaMalloc(&dx, sizeof hx);
  cudaMalloc(&dout, sizeof hx);
  cudaMemcpy(dx, hx, sizeof hx, cudaMemcpyHostToDevice);
  const int smem = (128 + 64) * 128 + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dx, dout);
  cudaError_t err = cudaDeviceSynchronize();
  float ho[128];
  cudaMemcpy(ho, dout, sizeof ho, cudaMemcpyDeviceToHost);
  // classify
  int votes[3] = {0, 0, 0};   // trunc, rne, rna
  for (int r = 0; r < 8; ++r) {
    const double f = fr[r & 3], s = (r & 4) ? -1.0 : 1.0;
    const double t = 1.0 + (double)(int)f * u;
    const double rne = 1.0 + u * (f == 0.5 ? 0.0 : (f == 1.5 ? 2.0 : (f > 0.5 ? 1.0 : 0.0)));
    const double rna = 1.0 + u * (f >= 1.5 ? 2.0 : (f >= 0.5 ? 1.0 : 0.0));
    const double got = ho[r] * s;
    votes[0] += got == t;
    votes[1] += got == rne;
    votes[2] += got == rna;
    printf("{\"x\": %.10f, \"got\": %.10f}\n", (double)hx[r], (double)ho[r]);
  }
  printf("{\"probe\": \"tf32_operand_read\", \"err\": \"%s\", \"trunc\": %d, \"rne\": %d, \"rna\": %d, \"of\": 8}\n",
         cudaGetErrorString(err), votes[0], votes[1], votes[2]);
  return 0;
}
