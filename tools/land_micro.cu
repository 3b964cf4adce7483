// land_micro.cu — standalone probe of copy+checksum kernel designs for `land`
// (not product code).  Times, on one HBM-resident buffer of the bench probe's
// size, several ways of moving S bytes and checksumming them:
//   memcpy      cudaMemcpyAsync D2D (copy engines)
//   copy_u4     SM grid-stride uint4 copy, no checksum
//   land_u4     the product land kernel (kLandU = 4), identity layout
//   sum_u8      grid-stride copy + checksum, 8 vectors per lane in flight
//   tma_reg     cp.async.bulk global->smem ring, checksum + STG.128 from registers
//   tma_bulk    cp.async.bulk global->smem ring, checksum from smem, bulk store back
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//        -I paper_2404_14691_b200/csrc tools/land_micro.cu -o tools/land_micro
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#include "checksum.cuh"
namespace sage {
struct __align__(16) LandItem {
  unsigned long long dst_vec0;
  long long src_rel0;
  long long data0;
  unsigned int nvec;
  unsigned int pad_;
};
struct Gpu { int sm_count; };
#include "land_kernels.cuh"
}  // namespace sage
using namespace sage;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void copy_u4(const uint4 *__restrict__ s, uint4 *__restrict__ d, unsigned long long n) {
  unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = __ldg(s + i), b = __ldg(s + i + stride), c = __ldg(s + i + 2 * stride), e = __ldg(s + i + 3 * stride);
    d[i] = a; d[i + stride] = b; d[i + 2 * stride] = c; d[i + 3 * stride] = e;
  }
  for (; i < n; i += stride) d[i] = __ldg(s + i);
}

template <int U, int CS = 0>
__global__ void __launch_bounds__(256) sum_u(const uint4 *__restrict__ s, uint4 *__restrict__ d, unsigned long long n,
                                             unsigned long long *acc_out) {
  unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long acc = 0;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = CS & 2 ? __ldcs(s + i + u * stride) : __ldg(s + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (CS & 1) __stcs(d + i + u * stride, v[u]); else d[i + u * stride] = v[u];
      acc += vec_sum(v[u], 2 * (i + u * stride));
    }
  }
  for (; i < n; i += stride) { uint4 v = __ldg(s + i); d[i] = v; acc += vec_sum(v, 2 * i); }
  block_reduce_add(acc, acc_out);
}

// ---------------------------------------------------------------- TMA ring ---
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }

constexpr int TB = 256;
template <int STAGES, int SBYTES, bool BULK_STORE>
__global__ void __launch_bounds__(TB, 1) tma_land(const uint8_t *__restrict__ s, uint8_t *__restrict__ d,
                                                  unsigned long long bytes, unsigned long long *acc_out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[STAGES];
  const unsigned long long units = (bytes + SBYTES - 1) / SBYTES;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long first = blockIdx.x;
  const unsigned long long step = gridDim.x;
  auto issue = [&](unsigned long long u, int st) {
    unsigned long long off = u * SBYTES;
    uint32_t nb = (uint32_t)min((unsigned long long)SBYTES, bytes - off);
    mbar_expect_tx(&full[st], nb);
    bulk_g2s(sm + st * SBYTES, s + off, nb, &full[st]);
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < STAGES; ++k)
      if (first + k * step < units) issue(first + k * step, k);
  unsigned long long acc = 0;
  int k = 0;
  for (unsigned long long u = first; u < units; u += step, ++k) {
    const int st = k % STAGES;
    mbar_wait(&full[st], (k / STAGES) & 1);
    unsigned long long off = u * SBYTES;
    uint32_t nb = (uint32_t)min((unsigned long long)SBYTES, bytes - off);
    const uint4 *q = reinterpret_cast<const uint4 *>(sm + st * SBYTES);
    uint4 *dq = reinterpret_cast<uint4 *>(d + off);
    for (uint32_t v = threadIdx.x; v < nb / 16; v += TB) {
      uint4 x = q[v];
      if (!BULK_STORE) dq[v] = x;
      acc += vec_sum(x, (off / 8) + 2ull * v);
    }
    if (BULK_STORE) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        bulk_s2g(d + off, sm + st * SBYTES, nb);
        bulk_commit();
        bulk_wait_read<0>();
      }
    }
    __syncthreads();  // everyone done reading stage st
    if (threadIdx.x == 0 && u + STAGES * step < units) issue(u + STAGES * step, st);
  }
  if (BULK_STORE && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  block_reduce_add(acc, acc_out);
}

int main(int argc, char **argv) {
  const unsigned long long S = argc > 1 ? strtoull(argv[1], 0, 0) : 138412288ull;
  int sm = 0;
  CK(cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0));
  uint8_t *src, *dst, *flush;
  unsigned long long *acc;
  const size_t FL = 512ull << 20;
  CK(cudaMalloc(&src, S + 4096));
  CK(cudaMalloc(&dst, S + 4096));
  CK(cudaMalloc(&flush, FL));
  CK(cudaMalloc(&acc, 64));
  std::vector<uint8_t> h(S);
  for (size_t i = 0; i < S; ++i) h[i] = (uint8_t)(i * 2654435761u >> 13);
  CK(cudaMemcpy(src, h.data(), S, cudaMemcpyHostToDevice));
  const unsigned long long want = host_checksum(h.data(), S);
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  // identity layout: one item
  LandItem item{0, 0, (long long)S, (unsigned)(S / 16), 0};
  uint32_t prefix[2] = {0, (uint32_t)(S / 16)};
  LandItem *d_item;
  uint32_t *d_prefix;
  unsigned int *d_done;
  CK(cudaMalloc(&d_item, sizeof(item)));
  CK(cudaMalloc(&d_prefix, sizeof(prefix)));
  CK(cudaMalloc(&d_done, 16));
  CK(cudaMemset(d_done, 0, 16));
  CK(cudaMemcpy(d_item, &item, sizeof(item), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_prefix, prefix, sizeof(prefix), cudaMemcpyHostToDevice));
  Gpu G{sm};

  auto run = [&](const char *name, auto fn, bool check, int reps = 20, bool flush_between = false) {
    for (int w = 0; w < 3; ++w) { CK(cudaMemsetAsync(acc, 0, 8, st)); fn(); }
    float best = 1e30f, tot = 0;
    for (int r = 0; r < reps; ++r) {
      if (flush_between) CK(cudaMemsetAsync(flush, r, FL, st));
      CK(cudaMemsetAsync(acc, 0, 8, st));
      CK(cudaEventRecord(e0, st));
      fn();
      CK(cudaEventRecord(e1, st));
      CK(cudaStreamSynchronize(st));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
      tot += ms;
    }
    CK(cudaGetLastError());
    unsigned long long got = 0;
    CK(cudaMemcpy(&got, acc, 8, cudaMemcpyDeviceToHost));
    const double gbs = 2.0 * S / (tot / reps * 1e-3) / 1e9;
    printf("{\"kernel\":\"%s\",\"bytes\":%llu,\"mean_us\":%.2f,\"best_us\":%.2f,\"GBps_mean\":%.1f,\"GBps_best\":%.1f,"
           "\"checksum_ok\":%s,\"flush\":%s}\n",
           name, S, tot / reps * 1e3, best * 1e3, gbs, 2.0 * S / (best * 1e-3) / 1e9,
           check ? (got == want ? "true" : "false") : "null", flush_between ? "true" : "false");
  };
  for (int fl = 0; fl < 2; ++fl) {
    bool F = fl == 1;
    run("memcpy", [&] { CK(cudaMemcpyAsync(dst, src, S, cudaMemcpyDeviceToDevice, st)); }, false, 20, F);
    run("copy_u4", [&] { copy_u4<<<sm * 8, 256, 0, st>>>((const uint4 *)src, (uint4 *)dst, S / 16); }, false, 20, F);
    run("land_u4", [&] {
      LandArgs a{d_item, d_prefix, 1, (uint32_t)(S / 16), src, S, dst, acc, d_done, nullptr};
      land_kernel<<<land_grid(&G, (uint32_t)(S / 16)), kLandThreads, 0, st>>>(a);
    }, true, 20, F);
    for (int sh : {4, 7}) {   // misaligned source runs (funnel-shift paths)
      LandItem it2{0, 0, (long long)(S - 16), (unsigned)(S / 16), 0};
      CK(cudaMemcpy(d_item, &it2, sizeof(it2), cudaMemcpyHostToDevice));
      char nm[32];
      snprintf(nm, sizeof nm, "land_sh%d", sh);
      run(nm, [&] {
        LandArgs a{d_item, d_prefix, 1, (uint32_t)(S / 16), src + sh, S - 16, dst, acc, d_done, nullptr};
        land_kernel<<<land_grid(&G, (uint32_t)(S / 16)), kLandThreads, 0, st>>>(a);
      }, false, 20, F);
      CK(cudaMemcpy(d_item, &item, sizeof(item), cudaMemcpyHostToDevice));
    }
    if (getenv("LM_SHORT")) continue;
    run("sum_u4", [&] { sum_u<4><<<sm * 4, 256, 0, st>>>((const uint4 *)src, (uint4 *)dst, S / 16, acc); }, true, 20, F);
    run("sum_u8", [&] { sum_u<8><<<sm * 4, 256, 0, st>>>((const uint4 *)src, (uint4 *)dst, S / 16, acc); }, true, 20, F);
    run("sum_u8_g8", [&] { sum_u<8><<<sm * 8, 256, 0, st>>>((const uint4 *)src, (uint4 *)dst, S / 16, acc); }, true, 20, F);
    run("sum_u4_stcs", [&] { sum_u<4, 1><<<sm * 4, 256, 0, st>>>((const uint4 *)src, (uint4 *)dst, S / 16, acc); }, true, 20, F);
    run("sum_u4_ldcs_stcs", [&] { sum_u<4, 3><<<sm * 4, 256, 0, st>>>((const uint4 *)src, (uint4 *)dst, S / 16, acc); }, true, 20, F);
    run("sum_u8_stcs", [&] { sum_u<8, 1><<<sm * 4, 256, 0, st>>>((const uint4 *)src, (uint4 *)dst, S / 16, acc); }, true, 20, F);
    run("sum_u8_ldcs", [&] { sum_u<8, 2><<<sm * 4, 256, 0, st>>>((const uint4 *)src, (uint4 *)dst, S / 16, acc); }, true, 20, F);
    run("sum_u8_b2", [&] { sum_u<8><<<sm * 2, 256, 0, st>>>((const uint4 *)src, (uint4 *)dst, S / 16, acc); }, true, 20, F);
    run("sum_u16_b4", [&] { sum_u<16><<<sm * 4, 256, 0, st>>>((const uint4 *)src, (uint4 *)dst, S / 16, acc); }, true, 20, F);
#define TMA(ST, SB, BS, BPS)                                                                                   \
    {                                                                                                          \
      auto k = tma_land<ST, SB, BS>;                                                                           \
      CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * SB));                       \
      run("tma_" #ST "x" #SB "_" #BS "_b" #BPS, [&] { k<<<sm * BPS, TB, ST * SB, st>>>(src, dst, S, acc); }, true, 20, F); \
    }
    TMA(4, 16384, false, 1)
  }
  return 0;
}
