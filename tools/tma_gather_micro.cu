// tma_gather_micro.cu -- random 16-B row gathers through the TMA unit
// (cp.async.bulk.tensor.2d.tile::gather4: 4 rows per instruction) vs the
// L1TEX random-gather ceiling (~262 G 4-B gathers/s, one 128-B line
// wavefront per clock per SM).  x (4 MiB) viewed as [1 Mi/4 rows x 4 floats].
// (probe, not product code)
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/tma_gather_micro.cu -o /tmp/tg -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t hsh(uint32_t v) {
  v ^= v >> 16; v *= 0x7feb352dU; v ^= v >> 15; v *= 0x846ca68bU; v ^= v >> 16; return v;
}
// every issuing lane: `per` gather4 ops into its own 1 KiB smem slice, 128-B aligned slots
// (rewritten; a throughput probe)
__global__ void tma_gather(const __grid_constant__ CUtensorMap map, int per, uint32_t rows_mask, int issuers,
                           float *out) {
  __shared__ __align__(128) float buf[32][256];
  __shared__ uint64_t bar[32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool issuer = lane == 0 && w < issuers;
  if (issuer) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[w])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (issuer) {
    const uint32_t base = (blockIdx.x * 32 + w) * 7919u;
    const int batch = 16;   // 16 gather4 (1 KiB) in flight per issuer per round
    for (int r = 0; r < per; r += batch) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[w])), "r"(batch * 64) : "memory");
      for (int k = 0; k < batch; ++k) {
        const uint32_t s0 = base + (uint32_t)(r + k) * 4u;
        const int r0 = hsh(s0) & rows_mask, r1 = hsh(s0 + 1) & rows_mask, r2 = hsh(s0 + 2) & rows_mask,
                  r3 = hsh(s0 + 3) & rows_mask;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(sa(&buf[w][(k % 8) * 32])),
            "l"(&map), "r"(sa(&bar[w])), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
            : "memory");
      }
      asm volatile("{\n.reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(
                       sa(&bar[w])), "r"((r / batch) & 1)
                   : "memory");
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && buf[0][0] == 1234.5f) out[blockIdx.x] = buf[1][1];
}

int main() {
  const int n = 1 << 20;
  float *x, *out;
  cudaMalloc(&x, n * 4); cudaMemset(x, 0, n * 4); cudaMalloc(&out, 1 << 20);
  CUtensorMap map;
  cuuint64_t dims[2] = {4, (cuuint64_t)n / 4};
  cuuint64_t strides[1] = {16};
  cuuint32_t box[2] = {4, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { const char *s; cuGetErrorString(r, &s); printf("{\"encode\":\"%s\"}\n", s); return 1; }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int issuers : {1, 2, 4, 8, 16, 32}) {
    const int per = 4096 / issuers * 4;   // gather4 ops per issuer; 16 Ki gather4 per CTA
    std::vector<float> v;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      tma_gather<<<sms, 1024>>>(map, per, (uint32_t)(n / 4 - 1), issuers, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); v.push_back(ms * 1e3f);
    }
    std::sort(v.begin(), v.end());
    const double rows = (double)sms * issuers * per * 4;
    printf("{\"issuers_per_cta\":%d,\"us\":%.2f,\"G_rows_per_s\":%.1f,\"err\":\"%s\"}\n", issuers, v[2],
           rows / v[2] / 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
