// checksum.cuh — the segment content checksum (spec: oracle/sage_oracle.c),
// device and host forms.  64-bit word p of the landed segment:
//   k = (u32)p*0x9E3779B1 ^ (u32)(p>>32)*0x85EBCA77
//   a = lo ^ k, b = hi ^ (k + 0x7F4A7C15), term = a*b + (b<<32 | a), sum mod 2^64
#pragma once
#include <cstdint>
#include <cstring>

namespace sage {

__host__ __device__ __forceinline__ unsigned long long pair_term(uint32_t lo, uint32_t hi, uint32_t k) {
  uint32_t a = lo ^ k, b = hi ^ (k + 0x7F4A7C15u);
  return (unsigned long long)a * b + (((unsigned long long)b << 32) | a);
}
// one 16-byte vector starting at 64-bit word p0 (p0 even)
__host__ __device__ __forceinline__ unsigned long long vec_sum(uint4 v, unsigned long long p0) {
  uint32_t khi = (uint32_t)(p0 >> 32) * 0x85EBCA77u;
  uint32_t m = (uint32_t)p0 * 0x9E3779B1u;
  return pair_term(v.x, v.y, m ^ khi) + pair_term(v.z, v.w, (m + 0x9E3779B1u) ^ khi);
}
// host: checksum of `bytes` (multiple of 16) at 64-bit word base p0 (even)
inline uint64_t host_checksum(const uint8_t *p, uint64_t bytes, uint64_t p0 = 0) {
  uint64_t s = 0;
  for (uint64_t i = 0; i + 16 <= bytes; i += 16) {
    uint4 v;
    memcpy(&v, p + i, 16);
    s += vec_sum(v, p0 + i / 8);
  }
  return s;
}

#ifdef __CUDACC__
__device__ __forceinline__ void block_reduce_add(unsigned long long v, unsigned long long *out) {
  __shared__ unsigned long long red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int nw = (blockDim.x + 31) >> 5;
    v = lane < nw ? red[lane] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && v) atomicAdd(out, v);
  }
}
#endif

}  // namespace sage
