/*
 * sage_oracle.c — CPU restatement of the SAGE data-plane byte arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker / the CPU reference arm.  The product path
 * (paper_2404_14691_b200/, libsagedp.so) never links or calls it.
 *
 * What it restates
 *   The reference (pkg/src/gslsim) models a read-only load as bytes pushed
 *   through a channel (functions.py:257-268, resources.py:137-149) and never
 *   materialises data.  The real plane lands a packed "DB" record
 *   (ref PAPER.md:345-347, Request/Data with RO type) into a segment whose
 *   tensors sit at 16-byte aligned offsets, and computes a 64-bit content
 *   checksum so the sharing manager can verify/deduplicate segments
 *   (sharing.py:136-177 decides WHO loads; this decides WHAT was loaded).
 *   Parity status: segment contents and checksums have no reference golden
 *   vectors (SURVEY.md §8c "parity unpinned" rows); this file is the
 *   specification, and tests/golden/ pins it with committed vectors.
 *
 * Checksum (order independent, so any GPU reduction tree is bit exact),
 * over the 64-bit little-endian words of the LANDED segment (its size is a
 * multiple of 16):
 *   lo_p, hi_p = low / high 32-bit halves of word p
 *   k_p = (uint32)p * 0x9E3779B1 ^ (uint32)(p >> 32) * 0x85EBCA77
 *   a_p = lo_p ^ k_p            b_p = hi_p ^ (k_p + 0x7F4A7C15)
 *   sum = Σ_p  a_p * b_p + (b_p << 32 | a_p)      (64-bit products, mod 2^64)
 *   One 32x32->64 multiply per 8 bytes keeps the land kernel HBM-bound; the
 *   linear term keeps every single-word change visible even when a_p*b_p = 0.
 *
 * Land (unpack):  seg[dst_off[i] + b] = packed[src_off[i] + b] for b < len[i];
 *   every other segment byte is zero.
 *
 * Host-only loading path (the CPU baseline of BASELINE.md "CPU-baseline
 * plan" item 2): per invocation copy the DB record into a private buffer,
 * unpack it through the layout and checksum it, fanned out over T threads.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

static inline uint64_t pair_term(uint32_t lo, uint32_t hi, uint64_t p) {
  uint32_t k = (uint32_t)p * 0x9E3779B1u ^ (uint32_t)(p >> 32) * 0x85EBCA77u;
  uint32_t a = lo ^ k, b = hi ^ (k + 0x7F4A7C15u);
  return (uint64_t)a * (uint64_t)b + (((uint64_t)b << 32) | a);
}

/* checksum of `bytes` (multiple of 8) starting at 64-bit word index word_base */
uint64_t oracle_checksum(const uint8_t *p, uint64_t bytes, uint64_t word_base) {
  /* one 64-bit load per word: this form vectorises (AVX2 vpmuludq) */
  uint64_t s = 0, n = bytes / 8;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t w;
    memcpy(&w, p + 8 * i, 8);
    const uint64_t q = word_base + i;
    const uint32_t k = (uint32_t)q * 0x9E3779B1u ^ (uint32_t)(q >> 32) * 0x85EBCA77u;
    const uint32_t a = (uint32_t)w ^ k, b = (uint32_t)(w >> 32) ^ (k + 0x7F4A7C15u);
    s += (uint64_t)a * b + (((uint64_t)b << 32) | a);
  }
  return s;
}

/* validate a layout; 0 ok, -1 bad */
int oracle_layout_check(const uint64_t *src_off, const uint64_t *dst_off, const uint64_t *len,
                        uint32_t n, uint64_t packed_bytes, uint64_t seg_bytes) {
  if (seg_bytes % 16) return -1;
  for (uint32_t i = 0; i < n; ++i) {
    if (dst_off[i] % 16) return -1;
    if (i == 0 && dst_off[0] != 0) return -1;
    if (src_off[i] + len[i] > packed_bytes || src_off[i] + len[i] < src_off[i]) return -1;
    uint64_t end = dst_off[i] + len[i];
    uint64_t lim = (i + 1 < n) ? dst_off[i + 1] : seg_bytes;
    if (end > lim) return -1;
    if (i + 1 < n && dst_off[i + 1] < dst_off[i]) return -1;
  }
  return 0;
}

/* unpack packed -> seg (seg_bytes, zero padded); returns the checksum */
uint64_t oracle_land(const uint8_t *packed, const uint64_t *src_off, const uint64_t *dst_off,
                     const uint64_t *len, uint32_t n, uint8_t *seg, uint64_t seg_bytes) {
  uint64_t cur = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (dst_off[i] > cur) memset(seg + cur, 0, dst_off[i] - cur);
    memcpy(seg + dst_off[i], packed + src_off[i], len[i]);
    cur = dst_off[i] + len[i];
  }
  if (seg_bytes > cur) memset(seg + cur, 0, seg_bytes - cur);
  return oracle_checksum(seg, seg_bytes, 0);
}

/* ---- host-only loading path, multi-threaded (CPU baseline) ---------------- */
typedef struct {
  const uint8_t *db;
  const uint64_t *src_off, *dst_off, *len;
  uint32_t n;
  uint64_t packed_bytes, seg_bytes;
  int n_inv;
  uint8_t **scratch;      /* per thread: private host copy + landed segment */
  uint64_t *sums;         /* per invocation checksum out */
  int next;
  pthread_mutex_t mu;
} hostpath_job;

typedef struct { hostpath_job *job; int tid; } hostpath_arg;

static void *hostpath_worker(void *argp) {
  hostpath_arg *a = (hostpath_arg *)argp;
  hostpath_job *J = a->job;
  uint8_t *priv = J->scratch[a->tid];
  uint8_t *seg = priv + ((J->packed_bytes + 63) & ~(uint64_t)63);
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int i = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (i >= J->n_inv) break;
    memcpy(priv, J->db, J->packed_bytes);                       /* CPU_LOAD: DB -> host  */
    J->sums[i] = oracle_land(priv, J->src_off, J->dst_off, J->len, J->n, seg, J->seg_bytes);
  }
  return NULL;
}

/* Run n_inv independent host-only loads of one DB record on `threads`
 * threads.  Returns 0, or -1 on allocation failure.                          */
int oracle_hostpath_run(const uint8_t *db, const uint64_t *src_off, const uint64_t *dst_off,
                        const uint64_t *len, uint32_t n, uint64_t packed_bytes,
                        uint64_t seg_bytes, int n_inv, int threads, uint64_t *sums) {
  if (threads < 1) threads = 1;
  hostpath_job J = {db, src_off, dst_off, len, n, packed_bytes, seg_bytes, n_inv, NULL, sums, 0,
                    PTHREAD_MUTEX_INITIALIZER};
  J.scratch = (uint8_t **)calloc((size_t)threads, sizeof(uint8_t *));
  pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
  hostpath_arg *args = (hostpath_arg *)calloc((size_t)threads, sizeof(hostpath_arg));
  int rc = 0;
  if (!J.scratch || !th || !args) { rc = -1; goto out; }
  for (int t = 0; t < threads; ++t) {
    J.scratch[t] = (uint8_t *)malloc(((packed_bytes + 63) & ~(uint64_t)63) + seg_bytes + 64);
    if (!J.scratch[t]) { rc = -1; goto out; }
    memset(J.scratch[t], 0, ((packed_bytes + 63) & ~(uint64_t)63) + seg_bytes + 64);  /* fault in */
  }
  for (int t = 0; t < threads; ++t) {
    args[t].job = &J; args[t].tid = t;
    pthread_create(&th[t], NULL, hostpath_worker, &args[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
out:
  if (J.scratch) for (int t = 0; t < threads; ++t) free(J.scratch[t]);
  free(J.scratch); free(th); free(args);
  return rc;
}

/* ---- the host-only path as a CPU serving process would run it ------------
 * One invocation on one core: CPU_LOAD (DB record -> the invocation's private
 * host buffer), then ONE pass that unpacks and checksums together: each
 * landed 64-bit word is loaded from the private copy, stored into the
 * segment and folded into the checksum while in registers (the loop
 * vectorises with AVX2).  Same bytes and checksum as oracle_land.            */
static inline uint64_t term64(uint64_t w, uint64_t q) {
  const uint32_t k = (uint32_t)q * 0x9E3779B1u ^ (uint32_t)(q >> 32) * 0x85EBCA77u;
  const uint32_t a = (uint32_t)w ^ k, b = (uint32_t)(w >> 32) ^ (k + 0x7F4A7C15u);
  return (uint64_t)a * b + (((uint64_t)b << 32) | a);
}
static uint64_t copy_run(uint8_t *restrict dst, const uint8_t *restrict src, uint64_t nwords, uint64_t q0) {
  uint64_t s = 0;
  for (uint64_t k = 0; k < nwords; ++k) {
    uint64_t w;
    memcpy(&w, src + 8 * k, 8);
    memcpy(dst + 8 * k, &w, 8);
    s += term64(w, q0 + k);
  }
  return s;
}
static uint64_t zero_run(uint8_t *dst, uint64_t nwords, uint64_t q0) {
  memset(dst, 0, 8 * nwords);
  uint64_t s = 0;
  for (uint64_t k = 0; k < nwords; ++k) s += term64(0, q0 + k);
  return s;
}
uint64_t oracle_load_into(const uint8_t *db, const uint64_t *src_off, const uint64_t *dst_off,
                          const uint64_t *len, uint32_t n, uint64_t packed_bytes, uint8_t *priv, uint8_t *seg,
                          uint64_t seg_bytes) {
  memcpy(priv, db, packed_bytes);
  uint64_t s = 0, cur = 0;   /* cur: word-aligned landed position */
  for (uint32_t i = 0; i < n; ++i) {
    const uint64_t d0 = dst_off[i], d1 = d0 + len[i];   /* d0 is 16-B aligned (layout invariant) */
    if (len[i] == 0) continue;
    s += zero_run(seg + cur, (d0 - cur) / 8, cur / 8);
    const uint64_t full = len[i] / 8;
    s += copy_run(seg + d0, priv + src_off[i], full, d0 / 8);
    cur = d0 + 8 * full;
    if (d1 > cur) {            /* the tensor's last bytes + zero padding to the word end */
      uint64_t w = 0;
      memcpy(&w, priv + src_off[i] + 8 * full, d1 - cur);
      memcpy(seg + cur, &w, 8);
      s += term64(w, cur / 8);
      cur += 8;
    }
  }
  s += zero_run(seg + cur, (seg_bytes - cur) / 8, cur / 8);
  return s;
}

/* aggregate memcpy rate (GB/s, read + write bytes) of `threads` threads each
 * copying its own `bytes` buffer `reps` times: the host memory roofline    */
typedef struct { uint8_t *a, *b; uint64_t bytes; int reps; } memcpy_arg;
static void *memcpy_worker(void *p) {
  memcpy_arg *m = (memcpy_arg *)p;
  for (int r = 0; r < m->reps; ++r) memcpy(m->b, m->a, m->bytes);
  return NULL;
}
#include <time.h>
double oracle_memcpy_rate(uint64_t bytes, int threads, int reps) {
  if (threads < 1) threads = 1;
  memcpy_arg *args = (memcpy_arg *)calloc((size_t)threads, sizeof(memcpy_arg));
  pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
  double gbs = -1;
  int ok = args && th;
  for (int t = 0; ok && t < threads; ++t) {
    args[t].a = (uint8_t *)malloc(bytes);
    args[t].b = (uint8_t *)malloc(bytes);
    if (!args[t].a || !args[t].b) { ok = 0; break; }
    memset(args[t].a, 1, bytes);
    memset(args[t].b, 0, bytes);
    args[t].bytes = bytes;
    args[t].reps = reps;
  }
  if (ok) {
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, memcpy_worker, &args[t]);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    const double s = (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec);
    gbs = 2.0 * (double)bytes * reps * threads / s / 1e9;
  }
  for (int t = 0; args && t < threads; ++t) { free(args[t].a); free(args[t].b); }
  free(args); free(th);
  return gbs;
}
