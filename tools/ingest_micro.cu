// ingest_micro.cu -- how fast can every SM pull the same L2-resident array
// into shared memory (cp.async.bulk, double-buffered chunks)?  Decides whether
// a column-blocked spmv (x chunks staged in smem, gathers from smem) can beat
// the ~260 G/s random-gather ceiling of spmv4.  Also: random 4-B gathers from
// smem.  (probe, not product code)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/ingest_micro.cu -o /tmp/im
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint32_t hsh(uint32_t v) {
  v ^= v >> 16; v *= 0x7feb352dU; v ^= v >> 15; v *= 0x846ca68bU; v ^= v >> 16; return v;
}

// each CTA streams `total` bytes of x (starting at an offset per CTA group) in
// CHUNK-byte pieces through NBUF buffers; GATHERS random smem reads per thread
// per chunk model the work done on each chunk.
template <int NBUF>
__global__ void __launch_bounds__(256) ingest(const char *x, size_t xbytes, uint32_t chunk, size_t total, int gathers,
                                              float *out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t bar[NBUF];
  const int nchunks = (int)(total / chunk);
  const size_t base = ((size_t)blockIdx.x * total) % xbytes;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NBUF; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < NBUF && i < nchunks; ++i) {
      mbar_expect(&bar[i], chunk);
      bulk_g2s(sm + (size_t)i * chunk, x + (base + (size_t)i * chunk) % xbytes, chunk, &bar[i]);
    }
  float s = 0;
  const uint32_t fmask = chunk / 4 - 1;
  for (int c = 0; c < nchunks; ++c) {
    const int b = c % NBUF;
    mbar_wait(&bar[b], (c / NBUF) & 1);
    const float *xs = (const float *)(sm + (size_t)b * chunk);
    for (int g = 0; g < gathers; ++g) s += xs[hsh(threadIdx.x * 977 + g * 131 + c) & fmask];
    __syncthreads();
    if (threadIdx.x == 0 && c + NBUF < nchunks) {
      mbar_expect(&bar[b], chunk);
      bulk_g2s(sm + (size_t)b * chunk, x + (base + (size_t)(c + NBUF) * chunk) % xbytes, chunk, &bar[b]);
    }
  }
  if (s == 1234.5f) out[blockIdx.x] = s;
}

int main() {
  const size_t xbytes = 4 << 20;
  char *x; float *out;
  cudaMalloc(&x, xbytes); cudaMemset(x, 0, xbytes); cudaMalloc(&out, 4096);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char *name, auto kern, int ctas, uint32_t chunk, int nbuf, size_t total, int gathers) {
    size_t smem = (size_t)chunk * nbuf;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    std::vector<float> v;
    for (int r = 0; r < 7; ++r) {
      cudaEventRecord(a);
      kern<<<ctas, 256, smem>>>(x, xbytes, chunk, total, gathers, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); v.push_back(ms * 1e3f);
    }
    std::sort(v.begin(), v.end());
    float us = v[3];
    double per_sm = (double)total / us / 1e3;
    double gps = (double)ctas * 256.0 * gathers * (total / chunk) / us / 1e3;
    printf("{\"case\":\"%s\",\"ctas\":%d,\"chunk_KiB\":%u,\"nbuf\":%d,\"MiB_per_cta\":%.2f,\"gathers_per_thread_per_chunk\":%d,"
           "\"us\":%.2f,\"GBps_per_sm\":%.1f,\"GBps_total\":%.0f,\"G_smem_gathers_per_s\":%.1f,\"err\":\"%s\"}\n",
           name, ctas, chunk >> 10, nbuf, total / 1048576.0, gathers, us, per_sm, per_sm * ctas, gps,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (size_t mib : {1, 2, 4}) {
    run("ingest2", ingest<2>, sms, 64 << 10, 2, mib << 20, 0);
    run("ingest3", ingest<3>, sms, 64 << 10, 3, mib << 20, 0);
    run("ingest2_96K", ingest<2>, sms, 96 << 10, 2, mib << 20, 0);
    run("ingest4_32K", ingest<4>, sms, 32 << 10, 4, mib << 20, 0);
  }
  // ingest + gathers: 113K nnz per CTA spread over the chunks (1M rows x16 / 148)
  for (size_t mib : {1, 2, 4}) {
    int chunks = (int)((mib << 20) / (64 << 10));
    int g = (int)(16.0 * (1 << 20) / sms / 256 / chunks + 0.5);
    run("ingest3_gather", ingest<3>, sms, 64 << 10, 3, mib << 20, std::max(1, g));
  }
  // pure smem gathers (one chunk resident, many gathers)
  run("smem_gather_only", ingest<2>, sms, 64 << 10, 2, 128 << 10, 221);
  return 0;
}
