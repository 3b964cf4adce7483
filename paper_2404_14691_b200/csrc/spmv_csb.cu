// spmv_csb.cu — y = A.x over the column-sliced block format (CSB) of
// parboil.spmv(fmt="csb").
//
// Why a second format: CSR spmv on the cfg-2 shape (1 Mi rows x 16 random
// columns, x 4 MiB) is bound by random 4-B gathers from L2: ~0.9 distinct-
// sector loads per clock per SM, 262 G/s on the whole GPU (the GATHER body,
// tools/gather_micro.cu), whatever the array size or cache hint.  Gathers
// from shared memory run at ~926 G/s (tools/ingest_micro.cu).  CSB stores
// the matrix so that every CTA sees x one shared-memory-sized chunk at a time:
//
//   rows   -> G row groups of R rows          (one CTA row of the grid)
//   cols   -> S slices of SC columns           (S CTAs of a row group = one
//             cluster; their partial y's are summed over DSMEM at the end)
//   slice  -> CH chunks of CW columns          (the x chunk TMA-bulk-copied
//             into shared memory through an NS-deep ring)
//   chunk  -> W sub-buckets, one per consumer warp: warp w owns a fixed row
//             range of the group, so no two warps ever update the same row
//
// Entries of a sub-bucket are (idx, val) pairs, idx = row_local << 17 |
// col_in_chunk, sorted by row; a bucket (g, s, c) is padded with SKIP
// entries (idx = 0xFFFFFFFF) to a 16-B multiple so one bulk copy moves it.
// offsets[(b * W + w)] is the first entry of sub-bucket (b, w), b = (g * S +
// s) * CH + c; offsets[NB * W] ends the array.
//
// Per CTA: 1 producer warp (one elected lane issues the bulk copies of the
// x chunk and the bucket's entries onto a full barrier) + W = 16 consumer
// warps (wait full, gather from the staged x, add into the CTA's y partial
// in shared memory; every consumer thread fences the async proxy and arrives
// on empty -- racecheck-clean, profiles/r1_spmv_csb_sanitizer.txt).  A warp's rows are its own and one
// row's entries inside a 32-entry window are merged in lane order, so every
// sum has a fixed order (sm_100 has no native shared fp32 atomic add: it
// would be a CAS loop); slices are summed in rank order.  Repeated launches
// are bit-identical; the order differs from CSR's sequential one, so the
// results agree with it to fp32 rounding.
#include "common.h"

namespace sage {
namespace {

constexpr int kCsbWarps = 16;                  // consumer warps (W)
constexpr int kCsbThreads = (kCsbWarps + 1) * 32;
constexpr uint32_t kCsbSkip = 0xFFFFFFFFu;
constexpr int kCsbColBits = 17;
constexpr uint32_t kCsbSmem = 227u * 1024u - 128u;   // dynamic smem a CTA may use (static: barriers)

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mb_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect_arrive(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "CSB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra CSB_WAIT_%=;\n}\n" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_to_smem(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ uint2 lds_u2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float lds_f(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_f(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float dsmem_load(const float *local, uint32_t rank) {
  uint32_t remote;
  float v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_addr(local)), "r"(rank));
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
  return v;
}

struct CsbShape {
  int rows, cols, R, S, NS, SC, CW, CH, G, Emax;
  uint32_t ys_bytes, tbl_bytes, stage_bytes;   // y partial; offsets table; one stage = x chunk + entries
};

constexpr int kCsbMaxStages = 8;
constexpr int kCsbU = 4;   // 32-entry windows in flight per consumer warp

// kMode 0: pair merge + segmented shuffle sums for longer runs (default);
// diagnostics (SAGE_CSB_MODE): 1 shared-memory atomicAdd per entry, 2 the
// chunk feed alone, 3 gathers + products without the y updates (2 and 3
// give wrong results)
template <int kMode>
__global__ void __launch_bounds__(kCsbThreads, 1)
    spmv_csb_kernel(const uint32_t *__restrict__ off, const uint2 *__restrict__ ent, const float *__restrict__ x,
                    float *__restrict__ y, CsbShape sh) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[kCsbMaxStages], empty[kCsbMaxStages];
  float *ys = reinterpret_cast<float *>(smem);
  const uint32_t ys_a = smem_addr(ys);
  uint32_t *tbl = reinterpret_cast<uint32_t *>(smem + sh.ys_bytes);   // this CTA's CH * W + 1 offsets
  const int s = blockIdx.x % sh.S, g = blockIdx.x / sh.S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *stages = smem + sh.ys_bytes + sh.tbl_bytes;
  // row groups start their slice at staggered chunks: 74 CTAs reading the
  // same x chunk at once would queue on the same L2 lines
  const int c_first = (int)(((long long)g * sh.CH) / sh.G);
  auto chunk_at = [&](int k) { return (c_first + k) % sh.CH; };
  auto stage_x = [&](int st) { return reinterpret_cast<float *>(stages + (size_t)st * sh.stage_bytes); };
  auto stage_e = [&](int st) { return reinterpret_cast<uint2 *>(stages + (size_t)st * sh.stage_bytes + 4u * sh.CW); };
  if (threadIdx.x == 0) {
    for (int i = 0; i < sh.NS; ++i) {
      mb_init(&full[i], 1);
      mb_init(&empty[i], kCsbWarps * 32);   // every consumer thread releases its own reads
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const size_t t0 = (size_t)(g * sh.S + s) * sh.CH * kCsbWarps;
  const int ntbl = sh.CH * kCsbWarps + 1;
  for (int i = threadIdx.x; i < ntbl; i += kCsbThreads) tbl[i] = __ldg(off + t0 + i);
  for (int r = threadIdx.x; r < sh.R; r += kCsbThreads) ys[r] = 0.f;
  __syncthreads();

  if (warp == kCsbWarps) {
    // ---- producer: x chunk + the bucket's entries, one bulk copy each ----
    if (lane == 0) {
      const long long slice_end = min((long long)(s + 1) * sh.SC, (long long)sh.cols);
      for (int k = 0, st = 0, ph = 0; k < sh.CH; ++k) {
        const int c = chunk_at(k);
        if (k >= sh.NS) mb_wait(&empty[st], ph ^ 1);
        const long long col0 = (long long)s * sh.SC + (long long)c * sh.CW;
        const int ncols = (int)max(0LL, min((long long)sh.CW, slice_end - col0));
        const uint32_t xb16 = (uint32_t)(ncols * 4) & ~15u;
        const uint32_t e0 = tbl[c * kCsbWarps], e1 = tbl[(c + 1) * kCsbWarps];
        const uint32_t eb = (e1 - e0) * 8u;
        float *xs = stage_x(st);
        for (int t = (int)(xb16 / 4); t < ncols; ++t) xs[t] = __ldg(x + col0 + t);   // <16-B tail, plain stores
        mb_expect_arrive(&full[st], xb16 + eb);    // release: the tail stores are visible to the waiters
        if (xb16) bulk_to_smem(xs, x + col0, xb16, &full[st]);
        if (eb) bulk_to_smem(stage_e(st), ent + e0, eb, &full[st]);
        if (++st == sh.NS) {
          st = 0;
          ph ^= 1;
        }
      }
    }
  } else {
    // ---- consumers: warp `warp` owns sub-bucket (b, warp) of every chunk ----
    for (int k = 0, st = 0, ph = 0; k < sh.CH; ++k) {
      const int c = chunk_at(k);
      const uint32_t base = tbl[c * kCsbWarps];
      const uint32_t lo = tbl[c * kCsbWarps + warp] - base, hi = tbl[c * kCsbWarps + warp + 1] - base;
      mb_wait(&full[st], ph);
      const float *xs = stage_x(st);
      const uint2 *es = stage_e(st);
      if (kMode == 2) {
        // diagnostic (SAGE_CSB_MODE=2): the feed alone, no arithmetic
      } else if (kMode == 3) {
        // diagnostic: gathers + products only, one sum per lane (wrong results)
        const uint32_t xs_a = smem_addr(xs), es_a = smem_addr(es);
        float acc = 0.f;
#pragma unroll 4
        for (uint32_t e = lo + lane; e < hi; e += 32) {
          const uint2 en = lds_u2(es_a + 8u * e);
          if (en.x != kCsbSkip) acc += __uint_as_float(en.y) * lds_f(xs_a + 4u * (en.x & ((1u << kCsbColBits) - 1)));
        }
        if (acc == 1234.5f) ys[lane] = acc;
      } else if (kMode == 1) {
        // shared-memory atomic add per entry (a CAS loop on sm_100)
#pragma unroll 4
        for (uint32_t e = lo + lane; e < hi; e += 32) {
          const uint2 en = es[e];
          if (en.x != kCsbSkip)
            atomicAdd(ys + (en.x >> kCsbColBits), __uint_as_float(en.y) * xs[en.x & ((1u << kCsbColBits) - 1)]);
        }
      } else {
        // sorted rows, kCsbU windows of 32 entries per step (independent
        // load / multiply / merge chains; the y updates then go window by
        // window).  Runs of one row are adjacent and short (a row has ~0.2
        // entries per chunk on the cfg-2 shape): pairs merge with one
        // shuffle, a window holding a run of 3+ takes the full segmented scan.
        const uint32_t xs_a = smem_addr(xs), es_a = smem_addr(es);
        for (uint32_t w0 = lo; w0 < hi; w0 += 32 * kCsbU) {
          uint32_t key[kCsbU];
          float v[kCsbU];
#pragma unroll
          for (int u = 0; u < kCsbU; ++u) {
            const uint32_t e = w0 + 32 * u + lane;
            key[u] = kCsbSkip;
            v[u] = 0.f;
            if (e < hi) {
              const uint2 en = lds_u2(es_a + 8u * e);
              if (en.x != kCsbSkip) {
                key[u] = en.x >> kCsbColBits;
                v[u] = __uint_as_float(en.y) * lds_f(xs_a + 4u * (en.x & ((1u << kCsbColBits) - 1)));
              }
            }
          }
          bool head[kCsbU];
#pragma unroll
          for (int u = 0; u < kCsbU; ++u) {
            const uint32_t nxt = __shfl_down_sync(0xffffffffu, key[u], 1);
            const float nv = __shfl_down_sync(0xffffffffu, v[u], 1);
            const bool pair = lane < 31 && nxt == key[u] && key[u] != kCsbSkip;
            const bool pair_next = __shfl_down_sync(0xffffffffu, pair, 1);
            if (!__any_sync(0xffffffffu, pair && lane < 30 && pair_next)) {
              if (pair) v[u] += nv;
            } else {
#pragma unroll
              for (int d = 1; d < 32; d <<= 1) {
                const float vv = __shfl_down_sync(0xffffffffu, v[u], d);
                const uint32_t kk = __shfl_down_sync(0xffffffffu, key[u], d);
                if (lane + d < 32 && kk == key[u]) v[u] += vv;
              }
            }
            const uint32_t prev = __shfl_up_sync(0xffffffffu, key[u], 1);
            head[u] = (lane == 0 || prev != key[u]) && key[u] != kCsbSkip;
          }
#pragma unroll
          for (int u = 0; u < kCsbU; ++u) {
            if (head[u]) {
              const uint32_t ya = ys_a + 4u * key[u];
              sts_f(ya, lds_f(ya) + v[u]);
            }
            __syncwarp();
          }
        }
      }
      // the stage's next fill is an async-proxy (bulk copy) write: order this
      // thread's generic-proxy reads of it before its release
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mb_arrive(&empty[st]);
      if (++st == sh.NS) {
        st = 0;
        ph ^= 1;
      }
    }
  }
  __syncthreads();
  // ---- y = sum of the S slices' partials (rank order), rows split by rank ----
  const long long row0 = (long long)g * sh.R;
  if (sh.S == 1) {
    for (int r = threadIdx.x; r < sh.R && row0 + r < sh.rows; r += kCsbThreads) y[row0 + r] = ys[r];
  } else {
    cluster_sync();
    const int per = (sh.R + sh.S - 1) / sh.S;
    const int lo = s * per, hi = min(sh.R, lo + per);
    for (int r = lo + threadIdx.x; r < hi && row0 + r < sh.rows; r += kCsbThreads) {
      float acc = dsmem_load(ys + r, 0);
      for (int q = 1; q < sh.S; ++q) acc += dsmem_load(ys + r, (uint32_t)q);
      y[row0 + r] = acc;
    }
    cluster_sync();   // peers may still read this CTA's partial
  }
}

}  // namespace

int spmv_csb(const sage_body_desc *b, cudaStream_t st, int sm_count) {
  (void)sm_count;
  CsbShape sh{};
  sh.rows = (int)b->args[0];
  sh.cols = (int)b->args[1];
  const uint64_t o_off = (uint64_t)b->args[2], o_ent = (uint64_t)b->args[3];
  sh.R = (int)b->args[4];
  sh.CW = (int)b->args[5];
  sh.Emax = (int)b->args[6];
  sh.S = (int)(b->args[7] & 0xf);
  sh.NS = (int)((b->args[7] >> 4) & 0xf);
  if (sh.rows <= 0 || sh.cols <= 0 || sh.R <= 0 || sh.R >= (1 << (32 - kCsbColBits)) || sh.CW <= 0 ||
      sh.CW % 4 || sh.CW > (1 << kCsbColBits) || sh.Emax < 0 || sh.S < 1 || sh.S > 8 || sh.NS < 2 ||
      sh.NS > kCsbMaxStages)
    return fail(SAGE_EINVAL, "spmv_csb: bad format parameters");
  sh.G = (sh.rows + sh.R - 1) / sh.R;
  sh.SC = ((sh.cols + sh.S - 1) / sh.S + 3) / 4 * 4;
  sh.CH = (sh.SC + sh.CW - 1) / sh.CW;
  sh.ys_bytes = ((uint32_t)sh.R * 4u + 127u) & ~127u;
  sh.tbl_bytes = ((uint32_t)(sh.CH * kCsbWarps + 1) * 4u + 127u) & ~127u;
  sh.stage_bytes = ((uint32_t)sh.CW * 4u + (uint32_t)sh.Emax * 8u + 127u) & ~127u;
  const uint64_t nb = (uint64_t)sh.G * sh.S * sh.CH;
  const uint64_t smem = (uint64_t)sh.ys_bytes + sh.tbl_bytes + (uint64_t)sh.NS * sh.stage_bytes;
  if (smem > kCsbSmem) return fail(SAGE_EINVAL, "spmv_csb: format needs more shared memory than a CTA has");
  if (o_off + 4 * (nb * kCsbWarps + 1) > b->ro_bytes || o_ent > b->ro_bytes || ((b->ro + o_ent) & 15) ||
      ((b->ro + o_off) & 3) || (uint64_t)sh.cols * 4 > b->input_bytes || (uint64_t)sh.rows * 4 > b->out_bytes ||
      (b->input & 15))
    return fail(SAGE_EINVAL, "spmv_csb: buffers too small or misaligned");
  static const int mode = [] { const char *e = getenv("SAGE_CSB_MODE"); return e ? atoi(e) : 0; }();
  auto kern = mode == 1   ? spmv_csb_kernel<1>
              : mode == 2 ? spmv_csb_kernel<2>
              : mode == 3 ? spmv_csb_kernel<3>
                          : spmv_csb_kernel<0>;
  SAGE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(sh.G * sh.S));
  cfg.blockDim = dim3(kCsbThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)sh.S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SAGE_CUDA(cudaLaunchKernelEx(&cfg, kern, (const uint32_t *)(b->ro + o_off),
                               (const uint2 *)(b->ro + o_ent), (const float *)b->input, (float *)b->out, sh));
  return SAGE_OK;
}

int touch_csb_kernel() {
  cudaFuncAttributes a;
  SAGE_CUDA(cudaFuncGetAttributes(&a, spmv_csb_kernel<0>));
  SAGE_CUDA(cudaFuncGetAttributes(&a, spmv_csb_kernel<1>));
  SAGE_CUDA(cudaFuncGetAttributes(&a, spmv_csb_kernel<2>));
  SAGE_CUDA(cudaFuncGetAttributes(&a, spmv_csb_kernel<3>));
  return SAGE_OK;
}

}  // namespace sage
