// gather_micro.cu -- what bounds spmv4 (cfg-2: 1 Mi rows x 16 random columns,
// x 4 MiB)?  Times random 4-B gathers from an L2-resident array with and
// without the col/val streams, with cache hints, and the streams alone.
// (probe, not product code)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/gather_micro.cu -o /tmp/gm
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t hsh(uint32_t v) {
  v ^= v >> 16; v *= 0x7feb352dU; v ^= v >> 15; v *= 0x846ca68bU; v ^= v >> 16; return v;
}
template <int MODE>
__device__ __forceinline__ float ldx(const float *p) {
  float r;
  if (MODE == 0) r = __ldg(p);
  else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  else asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
// pure gathers, hashed indices (no index stream)
template <int MODE>
__global__ void __launch_bounds__(256) gather_hash(const float *x, uint32_t mask, float *out, int n, int per) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  float s = 0;
  for (int k = 0; k < per; ++k) s += ldx<MODE>(x + (hsh(t * per + k) & mask));
  if (s == 12345.f) out[t] = s;
}
// spmv-shaped: stream col + val (16 B per lane per step), gather x
template <int MODE, int STREAM_HINT>
__global__ void __launch_bounds__(256) spmv_like(const int *col, const float *val, const float *x, float *y, int rows) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = g >> 2, sub = g & 3;
  float s = 0;
  if (row < rows) {
    const int k = row * 16 + 4 * sub;
    int4 c; float4 v;
    if (STREAM_HINT == 0) { c = __ldg((const int4 *)(col + k)); v = __ldg((const float4 *)(val + k)); }
    else {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "l"(col + k), "l"(pol));
      asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(val + k), "l"(pol));
    }
    s = fmaf(v.x, ldx<MODE>(x + c.x), s); s = fmaf(v.y, ldx<MODE>(x + c.y), s);
    s = fmaf(v.z, ldx<MODE>(x + c.z), s); s = fmaf(v.w, ldx<MODE>(x + c.w), s);
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  if (row < rows && sub == 0) y[row] = s;
}
// streams only (no gather): col + val summed
__global__ void __launch_bounds__(256) stream_only(const int *col, const float *val, float *y, int rows) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = g >> 2, sub = g & 3;
  float s = 0;
  if (row < rows) {
    const int k = row * 16 + 4 * sub;
    int4 c = __ldg((const int4 *)(col + k)); float4 v = __ldg((const float4 *)(val + k));
    s = v.x * c.x + v.y * c.y + v.z * c.z + v.w * c.w;
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  if (row < rows && sub == 0) y[row] = s;
}
// flush L2
__global__ void scrub(float *p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] += 1.f;
}

template <typename F>
static float timeit(F f, float *flush, size_t nflush, bool do_flush) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<float> v;
  for (int r = 0; r < 7; ++r) {
    if (do_flush) scrub<<<148 * 8, 256>>>(flush, nflush);
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); v.push_back(ms * 1e3f);
  }
  std::sort(v.begin(), v.end());
  return v[3];
}
#include <algorithm>
int main() {
  const int rows = 1 << 20, nnz = rows * 16;
  int *col; float *val, *x, *y, *big, *out;
  cudaMalloc(&col, nnz * 4); cudaMalloc(&val, nnz * 4); cudaMalloc(&x, (64 << 20)); cudaMalloc(&y, rows * 4);
  cudaMalloc(&out, 64 << 20);
  size_t nflush = 256ull << 20; cudaMalloc(&big, nflush * 4);
  std::vector<int> h(nnz); uint32_t s = 1;
  for (int i = 0; i < nnz; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) % rows; }
  cudaMemcpy(col, h.data(), nnz * 4, cudaMemcpyHostToDevice);
  cudaMemset(val, 0, nnz * 4); cudaMemset(x, 0, 64 << 20);
  const int blocks = rows * 4 / 256;
  auto P = [&](const char *name, float us, double gathers, double bytes) {
    printf("{\"case\":\"%s\",\"us\":%.2f,\"G_gathers_per_s\":%.1f,\"stream_GBps\":%.0f}\n", name, us, gathers / us / 1e3,
           bytes / us / 1e3);
  };
  // pure gathers: 16.7 M from 4 MiB, then 1 MiB / 16 MiB / 64 MiB arrays
  for (int lg : {18, 20, 22, 24}) {
    uint32_t mask = (1u << lg) - 1;
    char nm[64];
    snprintf(nm, 64, "hash_gather_ldg_%dMiB", (4 << lg) >> 20);
    P(nm, timeit([&] { gather_hash<0><<<blocks, 256>>>(x, mask, out, nnz, 4); }, big, nflush, false), nnz, 0);
    snprintf(nm, 64, "hash_gather_noalloc_%dMiB", (4 << lg) >> 20);
    P(nm, timeit([&] { gather_hash<1><<<blocks, 256>>>(x, mask, out, nnz, 4); }, big, nflush, false), nnz, 0);
    snprintf(nm, 64, "hash_gather_cg_%dMiB", (4 << lg) >> 20);
    P(nm, timeit([&] { gather_hash<2><<<blocks, 256>>>(x, mask, out, nnz, 4); }, big, nflush, false), nnz, 0);
  }
  for (int fl = 0; fl < 2; ++fl) {
    const char *sfx = fl ? "_l2cold" : "_l2warm";
    char nm[64];
    snprintf(nm, 64, "stream_only%s", sfx);
    P(nm, timeit([&] { stream_only<<<blocks, 256>>>(col, val, y, rows); }, big, nflush, fl), 0, 8.0 * nnz);
    snprintf(nm, 64, "spmv_ldg%s", sfx);
    P(nm, timeit([&] { spmv_like<0, 0><<<blocks, 256>>>(col, val, x, y, rows); }, big, nflush, fl), nnz, 8.0 * nnz);
    snprintf(nm, 64, "spmv_noalloc%s", sfx);
    P(nm, timeit([&] { spmv_like<1, 0><<<blocks, 256>>>(col, val, x, y, rows); }, big, nflush, fl), nnz, 8.0 * nnz);
    snprintf(nm, 64, "spmv_ldg_stream_evict_first%s", sfx);
    P(nm, timeit([&] { spmv_like<0, 1><<<blocks, 256>>>(col, val, x, y, rows); }, big, nflush, fl), nnz, 8.0 * nnz);
    snprintf(nm, 64, "spmv_noalloc_stream_evict_first%s", sfx);
    P(nm, timeit([&] { spmv_like<1, 1><<<blocks, 256>>>(col, val, x, y, rows); }, big, nflush, fl), nnz, 8.0 * nnz);
  }
  printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
