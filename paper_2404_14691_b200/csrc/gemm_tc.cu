// gemm_tc.cu — the sgemm function body on the 5th-gen tensor cores.
//
// C[M,N] (fp32, row-major) = A[M,K] . BT[N,K]^T, with A the function's
// shared read-only weights (landed segment) and BT the invocation input,
// both fp32 and K-contiguous (Parboil's sgemm also takes the second operand
// transposed, "matrix2t").  The MMA runs as tcgen05.mma kind::tf32 with the
// fp32 accumulator in TMEM.
//
// Structure (one 128 x BN output tile per CTA, 6 warps):
//   warp 0      TMA producer: A/BT K-blocks (32 fp32 = one 128-B swizzle
//               row) into a STAGES-deep smem ring, mbarrier complete_tx
//   warp 1      TMEM allocator + single-thread MMA issuer: 4 x
//               tcgen05.mma (K = 8 each) per K-block, tcgen05.commit frees
//               the smem slot; a final commit signals the epilogue
//   warps 2-5   epilogue: tcgen05.ld 32x32b.x32 -> registers -> global
// Cluster variant (MC): CTAs that own vertically adjacent M tiles of the same
// N tile and K range run as a 2-CTA cluster.  Each loads its own A block and
// HALF of the shared B block, multicast by TMA into both CTAs' smem, so the
// L2 -> SM traffic for B halves (this skinny GEMM re-reads B once per M
// tile).  A slot is refilled only when BOTH CTAs' MMAs have read it: each
// MMA thread commits to the slot's empty barrier in both CTAs (count 2).
// Operands use the canonical K-major SWIZZLE_128B layout: 8-row x 128-B
// core groups 1024 B apart (SBO = 64 x 16 B), start address advanced by
// 32 B per K = 8 step inside the swizzle atom.
//
// FP32 accuracy (3xTF32, the default): a TF32 operand keeps 10 of fp32's 23
// mantissa bits, so one pass has a relative error of ~2^-11 per product --
// far outside rtol 1e-3 on a K = 4096 dot product near cancellation.  Each
// operand x is split as x = hi + lo with hi = x with its low 13 mantissa
// bits cleared (exactly a TF32 value) and lo = x - hi (exact in fp32, |lo| <
// 2^-10 |x|), and the tile product is accumulated as
//     A.B ~= A_hi.B_hi + A_hi.B_lo + A_lo.B_hi
// (the dropped A_lo.B_lo term is < 2^-20 relative; lo's own TF32 reading
// adds < 2^-21).  The split happens in shared memory: the epilogue warps,
// idle during the K loop, convert each landed stage (lo into a second
// buffer of the same swizzled layout; the transform is elementwise, so the
// swizzle needs no decoding) and release it to the MMA issuer through a
// second mbarrier.  X3 = 1 keeps the landed x as "hi": valid because the
// tensor core reads a TF32 operand with the low 13 bits ignored
// (tools/tf32_probe.cu measures this); X3 = 2 also rewrites hi in place
// (one more shared-memory store per element, correct under any reading).
#include "common.h"

#include <cudaTypedefs.h>

namespace sage {

// phase timestamps per CTA (tools/gemm_phases.cu builds with SAGE_GEMM_TRACE)
#ifdef SAGE_GEMM_TRACE
__device__ unsigned long long g_gemm_trace[1024 * 12];
__device__ __forceinline__ void gemm_mark(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (cta < 1024) g_gemm_trace[cta * 12 + slot] = t;
}
#else
__device__ __forceinline__ void gemm_mark(int) {}
#endif

constexpr int TC_BM = 128;        // UMMA M (rows of A / C per CTA)
constexpr int TC_BK = 32;         // fp32 elements per K-block = 128 bytes
// smem ring depth per N tile: as many 128-B K-blocks as fit in ~200 KB
template <int BN>
constexpr int tc_stages() { return BN >= 256 ? 4 : BN >= 128 ? 6 : 8; }
constexpr int TC_THREADS = 192;
// 3xTF32: eight converter warps (2..9) split each stage -- four could not keep
// the tensor pipe fed (ncu: the split's smem loads dominated the stalls,
// tensor pipe 13% active, profiles/r2_sgemm_x3_ncu.txt); warps 2..5 are the epilogue
constexpr int TC_CONV_WARPS_X3 = 8;
template <int X3>
__host__ __device__ constexpr int tc_threads() { return X3 ? 64 + 32 * TC_CONV_WARPS_X3 : TC_THREADS; }

template <int BN, int X3 = 0, bool PAIR = false>
struct TcSmem {
  static constexpr int A_BYTES = TC_BM * TC_BK * 4;   // 16 KB
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * TC_BK * 4;   // PAIR: this CTA's half of B
  static constexpr int RAW = A_BYTES + B_BYTES;
  static constexpr int STAGE = X3 ? 2 * RAW : RAW;     // 3xTF32: + lo copies of both tiles
  static constexpr int STAGES = X3 ? (192 * 1024) / STAGE : tc_stages<BN>();
  static constexpr int TOTAL = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(STAGES >= 2, "smem ring needs two stages");
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// a barrier other CTAs of the cluster arrive on (release.cluster)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// arrive on the barrier at the same smem offset in cluster CTA `rank`
__device__ __forceinline__ void mbar_arrive_remote(uint64_t *bar, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// canonical K-major SWIZZLE_128B smem descriptor (version 1, SBO = 1024 B)
__device__ __forceinline__ uint64_t kmajor_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);       // start address  [0,14)
  d |= (uint64_t)1 << 16;                         // LBO (unused for swizzled K-major) [16,30)
  d |= (uint64_t)(1024 >> 4) << 32;               // SBO: 8-row groups 1024 B apart [32,46)
  d |= (uint64_t)1 << 46;                         // version = 1 (Blackwell) [46,48)
  d |= (uint64_t)2 << 61;                         // layout: SWIZZLE_128B [61,64)
  return d;
}
// instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = BN
template <int BN, int UM = TC_BM>
__device__ __forceinline__ uint32_t tf32_idesc() {
  return (1u << 4)                 // c_format = F32
         | (2u << 7)               // a_format = TF32
         | (2u << 10)              // b_format = TF32
         | ((uint32_t)(BN >> 3) << 17)
         | ((uint32_t)(UM >> 4) << 24);
}

// hi = x with the low 13 mantissa bits cleared (a TF32 value); lo = x - hi exactly
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// 3xTF32 split of one landed stage (X3 > 0): NT converter threads, float4 granularity
template <int X3, int NT>
__device__ __forceinline__ void split_tile(uint8_t *raw, uint8_t *lo, int bytes, int t) {
  float4 *r4 = reinterpret_cast<float4 *>(raw), *l4 = reinterpret_cast<float4 *>(lo);
  constexpr int U = 4;
  for (int i0 = t; i0 < bytes / 16; i0 += NT * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * NT < bytes / 16) v[u] = r4[i0 + u * NT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i0 + u * NT >= bytes / 16) break;
      const float4 h = make_float4(tf32_hi(v[u].x), tf32_hi(v[u].y), tf32_hi(v[u].z), tf32_hi(v[u].w));
      l4[i0 + u * NT] = make_float4(v[u].x - h.x, v[u].y - h.y, v[u].z - h.z, v[u].w - h.w);
      if constexpr (X3 == 2) r4[i0 + u * NT] = h;
    }
  }
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// CTA pair (PAIR): one M = 256 MMA across the two SMs of a TPC; the leader
// issues it, reading A rows [0,128) + B rows [0,BN/2) from its smem and the
// peer's A rows [128,256) + B rows [BN/2,BN) from the peer's (same offsets)
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// PAIR: CTAs (2j, 2j+1) of a cluster -- adjacent along x, where the driver
// forms pairs for a cta_group::2 kernel -- own M tiles 2j, 2j+1 of one 256-row
// pair tile.  Each loads its A rows and its HALF of B (BN/2 rows) with its
// own TMA + full barrier, and (3xTF32) splits its own stage; the converters
// of both CTAs arrive on the LEADER's conv barrier (count 2 x warps), the
// leader issues tcgen05.mma.cta_group::2 (M = 256, N = BN) and commits to
// the empty / tmem_full barriers of both CTAs (multicast).  Per SM: half of
// B's smem, TMA and split traffic, so a 3xTF32 stage is 64 KB and the ring
// holds 3 stages instead of 2.  Each CTA's TMEM holds its 128 rows.
template <int BN, bool MC = false, bool CR = false, int X3 = 0, bool PAIR = false>
__global__ void __launch_bounds__(tc_threads<X3>(), 1)
    sgemm_tf32_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, float *C,
                      int M, int N, int K) {
  static_assert(!(PAIR && MC), "PAIR and B-multicast clusters are exclusive");
  using S = TcSmem<BN, X3, PAIR>;
  constexpr int TC_STAGES = S::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t *sA = smem;                                  // STAGES x A_BYTES
  uint8_t *sB = smem + TC_STAGES * S::A_BYTES;         // STAGES x B_BYTES
  uint8_t *sAl = smem + TC_STAGES * S::RAW;            // X3: STAGES x A_BYTES (lo parts)
  uint8_t *sBl = sAl + TC_STAGES * S::A_BYTES;         // X3: STAGES x B_BYTES
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + TC_STAGES * S::STAGE);
  uint64_t *empty = full + TC_STAGES;
  uint64_t *conv = empty + TC_STAGES;                  // X3: stage split, 4 converter warps
  uint64_t *tmem_full = conv + TC_STAGES;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) gemm_mark(0);
  // PAIR: M tiles along x (the driver forms CTA pairs along the cluster's x)
  const int m0 = (PAIR ? blockIdx.x : blockIdx.y) * TC_BM, n0 = (PAIR ? blockIdx.y : blockIdx.x) * BN;
  // split-K: CTA z covers K-blocks [z*kblocks, (z+1)*kblocks) and adds its
  // partial tile into C (zeroed by the host) with vector reductions
  const int kblocks = K / TC_BK / gridDim.z;
  const int kb0 = blockIdx.z * kblocks;
  const bool split = gridDim.z > 1;
  uint32_t crank = 0;
  if constexpr (MC || PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const uint32_t prank = PAIR ? (crank & 1u) : 0u;   // 0: pair leader (issues the MMAs)
  const uint32_t leader_rank = crank & ~1u;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < TC_STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], MC ? 2 : 1);   // MC: both CTAs' MMAs must release a slot
        mbar_init(&conv[s], PAIR ? 2 * TC_CONV_WARPS_X3 : TC_CONV_WARPS_X3);   // PAIR: both CTAs' converters
      }
      mbar_init(tmem_full, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // TMEM: BN fp32 columns x 128 lanes for the accumulator
    if constexpr (PAIR) {   // both CTAs' warp 1, same smem slot
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(BN < 32 ? 32 : BN));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(BN < 32 ? 32 : BN));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (MC || PAIR) cluster_sync_all();   // the peer's barriers exist before any multicast lands
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) gemm_mark(1);

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer ----
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % TC_STAGES, round = kb / TC_STAGES;
        mbar_wait(&empty[s], (round & 1) ^ 1);
        mbar_expect_tx(&full[s], S::RAW);   // the TMA bytes (3xTF32 lo buffers are written by the converter)
        tma_load_2d(sA + s * S::A_BYTES, &mapA, &full[s], (kb0 + kb) * TC_BK, m0);
        if constexpr (MC)   // this CTA's half of B, into both CTAs (same smem offset)
          tma_load_2d_mc(sB + s * S::B_BYTES + crank * (S::B_BYTES / 2), &mapB, &full[s], (kb0 + kb) * TC_BK,
                         n0 + (int)crank * (BN / 2), (uint16_t)0x3);
        else
          tma_load_2d(sB + s * S::B_BYTES, &mapB, &full[s], (kb0 + kb) * TC_BK, n0 + (int)prank * (BN / 2));
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && prank == 0) {
      // ---- MMA issuer (single thread; PAIR: the leader CTA's only) ----
      const uint32_t idesc = tf32_idesc<BN, PAIR ? 2 * TC_BM : TC_BM>();
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % TC_STAGES, round = kb / TC_STAGES;
        if constexpr (PAIR) mbar_wait_cluster(&conv[s], round & 1);
        else mbar_wait(X3 ? &conv[s] : &full[s], round & 1);
        if (kb == 0) gemm_mark(2);
        if (kb == kblocks / 2) gemm_mark(3);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = kmajor_sw128_desc(smem_u32(sA + s * S::A_BYTES));
        const uint64_t db = kmajor_sw128_desc(smem_u32(sB + s * S::B_BYTES));
        const uint64_t dal = kmajor_sw128_desc(smem_u32(sAl + s * S::A_BYTES));
        const uint64_t dbl = kmajor_sw128_desc(smem_u32(sBl + s * S::B_BYTES));
#pragma unroll
        for (int k = 0; k < TC_BK / 8; ++k) {
          // advance 32 B (8 tf32) along K inside the 128-B swizzle row: +2 in 16-B units
          const uint64_t a = da + (uint64_t)(2 * k), b = db + (uint64_t)(2 * k);
          const uint32_t acc = (kb | k) ? 1u : 0u;
          if constexpr (X3 && PAIR) {
            mma_tf32_pair(tmem, dal + (uint64_t)(2 * k), b, idesc, acc);
            mma_tf32_pair(tmem, a, dbl + (uint64_t)(2 * k), idesc, 1u);
            mma_tf32_pair(tmem, a, b, idesc, 1u);
          } else if constexpr (X3) {
            // correction terms first (smallest magnitudes), then hi.hi
            mma_tf32(tmem, dal + (uint64_t)(2 * k), b, idesc, acc);
            mma_tf32(tmem, a, dbl + (uint64_t)(2 * k), idesc, 1u);
            mma_tf32(tmem, a, b, idesc, 1u);
          } else if constexpr (PAIR) {
            mma_tf32_pair(tmem, a, b, idesc, acc);
          } else {
            mma_tf32(tmem, a, b, idesc, acc);
          }
        }
        // free the smem slot once these MMAs have read it (MC: in both CTAs,
        // whose producers both write into it)
        if constexpr (PAIR)
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&empty[s])),
              "h"((uint16_t)(0x3u << leader_rank))
              : "memory");
        else if constexpr (MC)
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&empty[s])),
              "h"((uint16_t)0x3)
              : "memory");
        else
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(&empty[s]))
                       : "memory");
      }
      gemm_mark(4);
      if constexpr (PAIR)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(tmem_full)),
            "h"((uint16_t)(0x3u << leader_rank))
            : "memory");
      else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(tmem_full))
                     : "memory");
    }
  } else {
    if constexpr (X3 > 0) {
      // ---- 3xTF32 split: warps 2..9 convert each landed stage ----
      constexpr int NT = 32 * TC_CONV_WARPS_X3;
      const int t = threadIdx.x - 64;
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % TC_STAGES, round = kb / TC_STAGES;
        mbar_wait(&full[s], round & 1);
        split_tile<X3, NT>(sA + s * S::A_BYTES, sAl + s * S::A_BYTES, S::A_BYTES, t);
        split_tile<X3, NT>(sB + s * S::B_BYTES, sBl + s * S::B_BYTES, S::B_BYTES, t);
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        if constexpr (PAIR) asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
        else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_remote(&conv[s], leader_rank);   // the leader's MMA reads both halves
          else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&conv[s])) : "memory");
        }
      }
    }
    // ---- epilogue: warps 2..5 own TMEM lane quadrants (warp % 4) ----
    if (warp < 6) mbar_wait(tmem_full, 0);
    if (warp == 2 && lane == 0) gemm_mark(5);
  }
  if (warp >= 2 && warp < 6) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quad = warp & 3;
    const int row = m0 + quad * 32 + lane;
    float *crow = C + (size_t)row * N + n0;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)c;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if constexpr (CR) {
        // split-K partial -> this CTA's smem (the drained operand ring),
        // rows padded by 16 B so a warp's 16-B stores hit distinct banks
        float4 *prow = reinterpret_cast<float4 *>(smem + (size_t)(quad * 32 + lane) * (BN * 4 + 16) + c * 4);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          prow[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
      } else if (row < M) {
        float4 *dst = reinterpret_cast<float4 *>(crow + c);
        if (split) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + j), "f"(__uint_as_float(r[4 * j])),
                         "f"(__uint_as_float(r[4 * j + 1])), "f"(__uint_as_float(r[4 * j + 2])),
                         "f"(__uint_as_float(r[4 * j + 3]))
                         : "memory");
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                 __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
        }
      }
    }
  }
  if constexpr (CR) {
    // split-K reduction over the cluster (the gridDim.z CTAs of one tile):
    // CTA z sums rows [z*R, (z+1)*R) of every CTA's partial through DSMEM and
    // stores them -- no atomics and no zeroed C (saves the memset launch;
    // in-kernel it is ~1.5 us slower than red.add, profiles/r1_sgemm_mc_ab.txt)
    if (threadIdx.x == 64) gemm_mark(7);
    cluster_sync_all();    // every partial is in its CTA's smem
    if (threadIdx.x == 64) gemm_mark(8);
    {
      // every warp of the CTA (the producer, MMA and converter warps are idle now)
      constexpr int NT = tc_threads<X3>();
      const int nz = (int)gridDim.z, rows = TC_BM / nz, t = threadIdx.x;
      const int r0 = (int)blockIdx.z * rows;
      constexpr int U = 4;   // outputs per thread in flight, each summing up to 8 partials
      for (int f0 = t; f0 < rows * (BN / 4); f0 += NT * U) {
        float4 acc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        // four partials x U outputs: 16 independent remote loads in flight
        // before any add (one DSMEM round trip per group, not one per partial)
        for (int q0 = 0; q0 < nz; q0 += 4) {
          float4 v[4][U];
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const int q = q0 + qq;
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int f = f0 + u * NT;
              const int row = r0 + f / (BN / 4), c4 = f % (BN / 4);
              const uint32_t la = smem_u32(smem + (size_t)row * (BN * 4 + 16) + c4 * 16);
              uint32_t ra;
              // split-K peers: cluster rank q (PAIR: the same pair slot of pair q)
              asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(PAIR ? prank + 2u * q : (uint32_t)q));
              if (q < nz && f < rows * (BN / 4))
                asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(v[qq][u].x), "=f"(v[qq][u].y), "=f"(v[qq][u].z), "=f"(v[qq][u].w)
                             : "r"(ra));
              else
                v[qq][u] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
#pragma unroll
          for (int qq = 0; qq < 4; ++qq)
#pragma unroll
            for (int u = 0; u < U; ++u) {
              acc[u].x += v[qq][u].x; acc[u].y += v[qq][u].y; acc[u].z += v[qq][u].z; acc[u].w += v[qq][u].w;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int f = f0 + u * NT;
          const int row = r0 + f / (BN / 4), c4 = f % (BN / 4);
          if (f < rows * (BN / 4) && m0 + row < M)
            *reinterpret_cast<float4 *>(C + (size_t)(m0 + row) * N + n0 + 4 * c4) = acc[u];
        }
      }
    }
    if (threadIdx.x == 64) gemm_mark(9);
    cluster_sync_all();   // peers are done reading this CTA's partial
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) gemm_mark(6);
  if constexpr (PAIR) cluster_sync_all();   // both CTAs are done with the pair's TMEM
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN < 32 ? 32 : BN));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN < 32 ? 32 : BN));
  }
  // MC: the peer may still signal this CTA's empty barriers / land multicast
  // bytes in its smem until it is done; neither CTA exits before both are
  if constexpr (MC) cluster_sync_all();
}

// ------------------------------------------------------------ stream-K ----
// 3xTF32, one CTA per SM: the (tile, K-block) units of the whole GEMM -- for
// the cfg-2 shape 32 tiles x 128 K-blocks -- are cut into equal contiguous
// ranges, one per CTA, so every SM of the GPU runs K-blocks (the split-K
// grid above uses 128 of 148).  A range spans at most two tiles (range <
// K-blocks per tile); each segment accumulates in its own TMEM half and is
// added into C (zeroed by the host) with vector reductions.  No clusters:
// in a busy burst a CTA needs one free SM, not four in one GPC.
template <int BN>
__global__ void __launch_bounds__(tc_threads<1>(), 1)
    sgemm_x3_sk_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, float *C,
                       int M, int N, int K, int units_per_cta) {
  using S = TcSmem<BN, 1>;
  constexpr int ST = S::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t *sA = smem, *sB = smem + ST * S::A_BYTES;
  uint8_t *sAl = smem + ST * S::RAW, *sBl = sAl + ST * S::A_BYTES;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + ST * S::STAGE);
  uint64_t *empty = full + ST;
  uint64_t *conv = empty + ST;
  uint64_t *tmem_full = conv + ST;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kblk = K / TC_BK, ntn = N / BN;
  const int total = (M / TC_BM) * ntn * kblk;
  const int u0 = blockIdx.x * units_per_cta;
  const int u1 = min(total, u0 + units_per_cta);
  const int nu = u1 - u0;
  if (nu <= 0) return;   // (the host sizes the grid so this does not happen)
  const int t0 = u0 / kblk;                // first tile; a second one starts at unit (t0 + 1) * kblk
  const int split_u = min(u1, (t0 + 1) * kblk);
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < ST; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], 1);
        mbar_init(&conv[i], TC_CONV_WARPS_X3);
      }
      mbar_init(tmem_full, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      for (int j = 0; j < nu; ++j) {
        const int u = u0 + j, t = u / kblk, kb = u - t * kblk;
        const int m0 = (t / ntn) * TC_BM, n0 = (t % ntn) * BN;
        const int st = j % ST, round = j / ST;
        mbar_wait(&empty[st], (round & 1) ^ 1);
        mbar_expect_tx(&full[st], S::RAW);
        tma_load_2d(sA + st * S::A_BYTES, &mapA, &full[st], kb * TC_BK, m0);
        tma_load_2d(sB + st * S::B_BYTES, &mapB, &full[st], kb * TC_BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = tf32_idesc<BN>();
      for (int j = 0; j < nu; ++j) {
        const int u = u0 + j;
        const int st = j % ST, round = j / ST;
        mbar_wait(&conv[st], round & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc_t = tmem + (u >= split_u ? (uint32_t)BN : 0u);   // segment's TMEM half
        const bool first = (u == u0) || (u == split_u);
        const uint64_t da = kmajor_sw128_desc(smem_u32(sA + st * S::A_BYTES));
        const uint64_t db = kmajor_sw128_desc(smem_u32(sB + st * S::B_BYTES));
        const uint64_t dal = kmajor_sw128_desc(smem_u32(sAl + st * S::A_BYTES));
        const uint64_t dbl = kmajor_sw128_desc(smem_u32(sBl + st * S::B_BYTES));
#pragma unroll
        for (int k = 0; k < TC_BK / 8; ++k) {
          const uint64_t a = da + (uint64_t)(2 * k), b = db + (uint64_t)(2 * k);
          const uint32_t acc = (first && k == 0) ? 0u : 1u;
          mma_tf32(acc_t, dal + (uint64_t)(2 * k), b, idesc, acc);
          mma_tf32(acc_t, a, dbl + (uint64_t)(2 * k), idesc, 1u);
          mma_tf32(acc_t, a, b, idesc, 1u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&empty[st]))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(tmem_full))
                   : "memory");
    }
  } else {
    constexpr int NT = 32 * TC_CONV_WARPS_X3;
    const int t = threadIdx.x - 64;
    for (int j = 0; j < nu; ++j) {
      const int st = j % ST, round = j / ST;
      mbar_wait(&full[st], round & 1);
      split_tile<1, NT>(sA + st * S::A_BYTES, sAl + st * S::A_BYTES, S::A_BYTES, t);
      split_tile<1, NT>(sB + st * S::B_BYTES, sBl + st * S::B_BYTES, S::B_BYTES, t);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&conv[st])) : "memory");
    }
    if (warp < 6) mbar_wait(tmem_full, 0);
  }
  if (warp >= 2 && warp < 6) {
    // ---- epilogue: each segment's partial tile, added into C ----
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quad = warp & 3;
    const int nseg = u1 > split_u ? 2 : 1;
    for (int sg = 0; sg < nseg; ++sg) {
      const int tile = t0 + sg;
      const int row = (tile / ntn) * TC_BM + quad * 32 + lane, n0 = (tile % ntn) * BN;
      float *crow = C + (size_t)row * N + n0;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(sg * BN + c);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < M) {
          float4 *dst = reinterpret_cast<float4 *>(crow + c);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + q), "f"(__uint_as_float(r[4 * q])),
                         "f"(__uint_as_float(r[4 * q + 1])), "f"(__uint_as_float(r[4 * q + 2])),
                         "f"(__uint_as_float(r[4 * q + 3]))
                         : "memory");
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
  }
}

// ------------------------------------------------------------------ host -----
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int encode_kmajor(CUtensorMap *map, const void *base, uint64_t rows, uint64_t k, uint32_t box_rows) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return fail(SAGE_ECUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  cuuint64_t dims[2] = {k, rows};
  cuuint64_t strides[1] = {k * 4};
  cuuint32_t box[2] = {TC_BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuTensorMapEncodeTiled");
  return SAGE_OK;
}

static int sm_count_of(int dev) {
  static int counts[64] = {0};
  if (dev < 0 || dev >= 64) return 148;
  if (!counts[dev]) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    counts[dev] = n;
  }
  return counts[dev];
}

// SAGE_SGEMM_MC=1 (opt-in): 2-CTA clusters with B multicast.  Off by default:
// on the cfg-2 shape (4096 x 256 x 4096) it measured 29.1 vs 27.1 us; ncu
// shows both variants latency-bound (DRAM 37%, L2 34-36%, SM 32% of peak),
// so halving B's L2 traffic buys nothing (profiles/r1_sgemm_mc_ab.txt)
static bool sgemm_mc_enabled() {
  static const bool on = [] { const char *e = getenv("SAGE_SGEMM_MC"); return e && atoi(e) != 0; }();
  return on;
}

template <int BN, bool MC, bool CR, int X3, bool PAIR = false>
static int launch_tc_kernel(const CUtensorMap &ma, const CUtensorMap &mb, float *C, int M, int N, int K, int split,
                            cudaStream_t s) {
  using S = TcSmem<BN, X3, PAIR>;
  auto kern = sgemm_tf32_kernel<BN, MC, CR, X3, PAIR>;
  // the smem opt-in is per device and context (FixedGSL instances launch from
  // fresh contexts): cheap, so set it on every launch
  SAGE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::TOTAL));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = PAIR ? dim3(M / TC_BM, N / BN, split) : dim3(N / BN, M / TC_BM, split);
  cfg.blockDim = dim3(tc_threads<X3>());
  cfg.dynamicSmemBytes = S::TOTAL;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (MC || CR || PAIR) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PAIR ? 2 : 1;
    attr[0].val.clusterDim.y = MC ? 2 : 1;
    attr[0].val.clusterDim.z = CR ? split : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  SAGE_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mb, C, M, N, K));
  return SAGE_OK;
}

// SAGE_SGEMM_PAIR=1 (opt-in): the CTA-pair (cta_group::2) 3xTF32 kernel.
// Off by default: on the cfg-2 shape its K loop takes as long as the 1-CTA
// kernel's (36.4 vs 36.6 us -- both issue the tensor pipe at the TF32 rate,
// 1.14 us per 3-pass K-block), and clusters of 2 x split = 8 CTAs at ~198 KB
// of smem do not all co-schedule in one wave (tools/call_pair.sh phase trace:
// the last clusters start 48 us late), so the kernel takes 2x as long
static bool sgemm_pair_enabled() {
  static const bool on = [] { const char *e = getenv("SAGE_SGEMM_PAIR"); return e && atoi(e) != 0; }();
  return on;
}

// SAGE_SGEMM_SK=1 (opt-in): the stream-K 3xTF32 kernel over every SM.  Off
// by default: measured 51.3 vs 49.2 us back to back (the memset launch and
// the red.add epilogue of up to two partial tiles per CTA outweigh the 12%
// shorter K range), and slower inside the cfg-2 burst (tools/call_sk.sh)
static bool sgemm_sk_enabled() {
  static const bool on = [] { const char *e = getenv("SAGE_SGEMM_SK"); return e && atoi(e) != 0; }();
  return on;
}

template <int BN>
static int launch_sk(const float *A, const float *BT, float *C, int M, int N, int K, cudaStream_t s, int sms) {
  CUtensorMap ma, mb;
  SAGE_TRY(encode_kmajor(&ma, A, (uint64_t)M, (uint64_t)K, TC_BM));
  SAGE_TRY(encode_kmajor(&mb, BT, (uint64_t)N, (uint64_t)K, BN));
  const int kblk = K / TC_BK, total = (M / TC_BM) * (N / BN) * kblk;
  int per = (total + sms - 1) / sms;
  if (per > kblk) per = kblk;   // a range must not span more than two tiles
  const int grid = (total + per - 1) / per;
  SAGE_CUDA(cudaMemsetAsync(C, 0, (size_t)M * N * 4, s));
  using S = TcSmem<BN, 1>;
  SAGE_CUDA(cudaFuncSetAttribute(sgemm_x3_sk_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::TOTAL));
  sgemm_x3_sk_kernel<BN><<<grid, tc_threads<1>(), S::TOTAL, s>>>(ma, mb, C, M, N, K, per);
  SAGE_CUDA(cudaGetLastError());
  return SAGE_OK;
}

template <int BN, int X3>
static int launch_tc(const float *A, const float *BT, float *C, int M, int N, int K, cudaStream_t s) {
  if constexpr (X3 == 1 && BN == 256) {
    if (sgemm_sk_enabled()) {
      int dev = 0;
      cudaGetDevice(&dev);
      return launch_sk<BN>(A, BT, C, M, N, K, s, sm_count_of(dev));
    }
  }
  // 2-CTA clusters along M when the M tiles pair up
  const bool mc = sgemm_mc_enabled() && (M / TC_BM) % 2 == 0;
  // split K so the grid covers the SMs: a skinny GEMM (N <= 256) has only
  // M/128 full-width tiles; splitting K keeps every A element read once
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = sm_count_of(dev);
  const int tiles = (N / BN) * (M / TC_BM), kblk = K / TC_BK;
  int split = 1;
  while (split * 2 * tiles <= sms && kblk % (split * 2) == 0 && kblk / (split * 2) >= 8) split *= 2;
  // split-K partials are reduced inside the cluster of the split CTAs (DSMEM)
  // unless disabled (SAGE_SGEMM_CR=0) or B-multicast clusters are requested
  static const bool cr_on = [] { const char *e = getenv("SAGE_SGEMM_CR"); return !(e && atoi(e) == 0); }();
  const bool cr = cr_on && !mc && split > 1 && split <= 8 && TC_BM % split == 0;
  // CTA pairs: 3xTF32 at BN = 256, M tiles pairing up, cluster (1, 2, split) within the portable 8
  const bool pair = X3 == 1 && BN == 256 && !mc && sgemm_pair_enabled() && (M / TC_BM) % 2 == 0 &&
                    2 * (cr ? split : 1) <= 8;
  CUtensorMap ma, mb;
  SAGE_TRY(encode_kmajor(&ma, A, (uint64_t)M, (uint64_t)K, TC_BM));
  SAGE_TRY(encode_kmajor(&mb, BT, (uint64_t)N, (uint64_t)K, (mc || pair) ? BN / 2 : BN));
  if (split > 1 && !cr) SAGE_CUDA(cudaMemsetAsync(C, 0, (size_t)M * N * 4, s));
  int rc;
  if constexpr (X3 == 1 && BN == 256) {
    if (pair) {
      rc = cr ? launch_tc_kernel<BN, false, true, X3, true>(ma, mb, C, M, N, K, split, s)
              : launch_tc_kernel<BN, false, false, X3, true>(ma, mb, C, M, N, K, split, s);
      if (rc != SAGE_OK) return rc;
      SAGE_CUDA(cudaGetLastError());
      return SAGE_OK;
    }
  }
  rc = mc ? launch_tc_kernel<BN, true, false, X3>(ma, mb, C, M, N, K, split, s)
       : cr ? launch_tc_kernel<BN, false, true, X3>(ma, mb, C, M, N, K, split, s)
            : launch_tc_kernel<BN, false, false, X3>(ma, mb, C, M, N, K, split, s);
  if (rc != SAGE_OK) return rc;
  SAGE_CUDA(cudaGetLastError());
  return SAGE_OK;
}

// SAGE_SGEMM_PASSES: 3 (default) = 3xTF32, FP32-accurate, with the landed x
// used as hi (X3 = 1); 4 = 3xTF32 with hi rewritten in place (X3 = 2);
// 1 = single-pass TF32 (diagnostics: the round-1 kernel)
int sgemm_passes() {
  static const int v = [] { const char *e = getenv("SAGE_SGEMM_PASSES"); return e ? atoi(e) : 3; }();
  return v;
}

template <int X3>
static int sgemm_tc_x(const float *A, const float *BT, float *C, int M, int N, int K, cudaStream_t s) {
  // widest N tile that divides N: A (the shared weights, the dominant
  // operand of these skinny GEMMs) is then streamed through smem once
  static const int force_bn = [] { const char *e = getenv("SAGE_SGEMM_BN"); return e ? atoi(e) : 0; }();
  if (force_bn == 64) return launch_tc<64, X3>(A, BT, C, M, N, K, s);       // diagnostics: tile sweep
  if (force_bn == 128 && N % 128 == 0) return launch_tc<128, X3>(A, BT, C, M, N, K, s);
  if (N % 256 == 0) return launch_tc<256, X3>(A, BT, C, M, N, K, s);
  if (N % 128 == 0) return launch_tc<128, X3>(A, BT, C, M, N, K, s);
  return launch_tc<64, X3>(A, BT, C, M, N, K, s);
}

// M % 128 == 0, N % 64 == 0, K % 32 == 0, 16-B aligned operands
int sgemm_tc(const float *A, const float *BT, float *C, int M, int N, int K, cudaStream_t s) {
  if (M <= 0 || N <= 0 || K <= 0 || M % TC_BM || N % 64 || K % TC_BK)
    return fail(SAGE_EINVAL, "sgemm (tcgen05): M % 128, N % 64 and K % 32 must be 0");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(BT) | reinterpret_cast<uintptr_t>(C)) & 15)
    return fail(SAGE_EINVAL, "sgemm (tcgen05): operands must be 16-byte aligned");
  const int p = sgemm_passes();
  if (p == 1) return sgemm_tc_x<0>(A, BT, C, M, N, K, s);
  if (p == 4) return sgemm_tc_x<2>(A, BT, C, M, N, K, s);
  return sgemm_tc_x<1>(A, BT, C, M, N, K, s);
}

// module-load the sgemm kernels of the configured precision (a fresh
// FixedGSL context loads only what its body needs)
template <int X3>
static int touch_x() {
  cudaFuncAttributes a;
  if constexpr (X3 == 1) {
    SAGE_CUDA(cudaFuncGetAttributes(&a, sgemm_x3_sk_kernel<256>));
    SAGE_CUDA(cudaFuncGetAttributes(&a, sgemm_tf32_kernel<256, false, true, X3, true>));
    SAGE_CUDA(cudaFuncGetAttributes(&a, sgemm_tf32_kernel<256, false, false, X3, true>));
  }
  SAGE_CUDA(cudaFuncGetAttributes(&a, sgemm_tf32_kernel<256, false, true, X3>));
  SAGE_CUDA(cudaFuncGetAttributes(&a, sgemm_tf32_kernel<256, false, false, X3>));
  SAGE_CUDA(cudaFuncGetAttributes(&a, sgemm_tf32_kernel<128, false, true, X3>));
  SAGE_CUDA(cudaFuncGetAttributes(&a, sgemm_tf32_kernel<64, false, true, X3>));
  return SAGE_OK;
}
int touch_tc_kernels() {
  const int p = sgemm_passes();
  return p == 1 ? touch_x<0>() : p == 4 ? touch_x<2>() : touch_x<1>();
}

}  // namespace sage
