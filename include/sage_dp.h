/*
 * sage_dp.h — C-ABI of the B200-native SAGE data plane (libsagedp.so).
 *
 * The reference (arxiv 2404.14691, pkg/src/gslsim) has no native code and no FFI:
 * its data plane exists only as a model.  Each entry point below replaces one
 * modelled seam of that simulator; the file:line it replaces is cited on the
 * declaration (paths relative to /root/reference/pkg/src/gslsim/).  The Python
 * host layer (paper_2404_14691_b200/) keeps the reference's registration /
 * invocation API and calls these through ctypes.
 *
 * Conventions
 *   - every call returns int status: SAGE_OK (0) or a negative SAGE_E* code;
 *     no C++ exception crosses the ABI; sage_last_error() gives the message
 *     (thread-local).
 *   - handles are opaque uint64 (0 is never a valid handle).
 *   - device pointers travel as uint64; host pointers as void*.
 *   - the library owns device memory, pinned staging, streams and events;
 *     the caller owns host source buffers until the op's end event completes.
 *   - completions are POLLED (sage_event_poll); the library never calls back
 *     into the host language.
 *   - all times are microseconds on the library clock (CLOCK_MONOTONIC,
 *     epoch = sage_init); device event times are converted onto it.
 */
#ifndef SAGE_DP_H
#define SAGE_DP_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAGE_ABI_VERSION 1

/* ---- status codes -------------------------------------------------------- */
#define SAGE_OK          0
#define SAGE_EINVAL     -1  /* bad argument (reference: ValueError)                     */
#define SAGE_ENOMEM     -2  /* pool budget exceeded (reference: resources.Denied value) */
#define SAGE_ECUDA      -3  /* CUDA driver/runtime error                                */
#define SAGE_ENOTREADY  -4  /* event/op not complete yet (poll again)                   */
#define SAGE_ESTATE     -5  /* double/unknown free, not initialised (SimulationError)   */
#define SAGE_ECHECKSUM  -6  /* landed bytes do not match the expected checksum          */
#define SAGE_ENODEV     -7  /* no such GPU / no GPU visible                              */

typedef uint64_t sage_handle;

/* ---- lifecycle ----------------------------------------------------------- *
 * Replaces Simulation.__init__'s device state (simulation.py:99-159): one
 * pool + staging rings + copy/land/host streams per GPU.                      */
#define SAGE_INIT_PEER_ACCESS  0x1u   /* map every pool segment for all GPUs (fan-out) */
#define SAGE_INIT_SHARE_DEVICE 0x2u   /* n_gpus logical planes on fewer physical devices
                                         (logical g -> device g % visible): exercises the
                                         multi-GPU control plane + peer lands on one GPU */
int         sage_init(int n_gpus, uint64_t pool_bytes_per_gpu, uint64_t staging_bytes,
                      uint64_t chunk_bytes, uint32_t flags);
int         sage_shutdown(void);
const char *sage_last_error(void);
int         sage_abi_version(void);
int         sage_device_count(int *n);
/* physical CUDA device of logical GPU `gpu` (device offset / shared planes applied) */
int         sage_gpu_device(int gpu, int *dev);
int64_t     sage_now_us(void);
/* the clock's epoch on CLOCK_MONOTONIC (ns): a host reads the library clock
 * without a call as (clock_gettime(CLOCK_MONOTONIC) - epoch_ns) / 1000       */
int64_t     sage_clock_epoch_ns(void);
/* host threads used for the CPU_LOAD memcpy fan-out (default 8) */
int         sage_set_host_threads(int n);

/* ---- memory pool ----------------------------------------------------------
 * Replaces MemoryLedger.try_alloc / free / usage_by_class / fits
 * (resources.py:271-337) and round_up_umb (resources.py:36-40).  Segments are
 * cuMemCreate physical allocations mapped with cuMemMap; the ledger charges
 * round_up(bytes, granularity) against the per-GPU budget exactly like the
 * reference (granularity 0 = exact), while the physical mapping is rounded to
 * the VMM page (2 MiB).  A refused allocation returns SAGE_ENOMEM and writes
 * the shortfall (the reference's Denied.shortfall_umb, in bytes).            */
#define SAGE_CLASS_CONTEXT         0
#define SAGE_CLASS_READ_ONLY       1
#define SAGE_CLASS_WRITABLE        2
#define SAGE_CLASS_INSTANCE_FIXED  3
#define SAGE_ALLOC_ACCOUNT_ONLY    0x100  /* OR into cls: charge the ledger, map nothing
                                             (FixedGSL instances allocate in their own context) */
#define SAGE_ALLOC_UNACCOUNTED     0x200  /* OR into cls: map without charging the ledger
                                             (runtime scratch: staging for oversized inputs) */
int sage_pool_configure(int gpu, uint64_t capacity_bytes, uint64_t granularity_bytes);
int sage_pool_alloc(int gpu, uint64_t bytes, int cls, sage_handle *h, uint64_t *dptr,
                    uint64_t *shortfall);
int sage_pool_free(sage_handle h);
/* ledger release now (the reference frees at once, sharing.py:217-229), the
 * physical pages once `ev` completes (a D2H / kernel may still read them)   */
int sage_pool_free_after(sage_handle h, sage_handle ev);
/* ... after every event in evs (e.g. the cache D2H and peer lands reading the
 * segment over NVLink from other GPUs)                                       */
int sage_pool_free_after_n(sage_handle h, const sage_handle *evs, int n);
int sage_pool_effective(int gpu, uint64_t bytes, uint64_t *effective);
int sage_pool_usage(int gpu, uint64_t by_class[4], uint64_t *ledger_total,
                    uint64_t *physical_total, uint64_t *capacity);
/* give the pages of freed segments back to the device: the size-keyed cache
 * of mapped free segments and every chunk (private writable segments are
 * carved from 1 GiB chunks) none of whose pieces is live; what a cuMemCreate
 * that finds the HBM full does by itself.  *released: bytes unmapped.
 * (new: the reference's ledger holds no pages, resources.py:271-337)      */
int sage_pool_trim(int gpu, uint64_t *released);
/* map an existing segment into another GPU's address space is implicit when
 * SAGE_INIT_PEER_ACCESS is set; this returns the (shared) VA               */
int sage_pool_dptr(sage_handle h, uint64_t *dptr, uint64_t *bytes);

/* ---- cross-process sharing (the paper's memory daemon -> function engines,
 * PAPER.md:279-281, 358-379): a segment's physical pages
 * leave as a POSIX file descriptor (pass it over a Unix socket, SCM_RIGHTS)
 * and are mapped zero-copy into another process on the same GPU.           */
int sage_pool_export(sage_handle h, int *fd, uint64_t *phys_bytes);
int sage_segment_import(int gpu, int fd, uint64_t phys_bytes, sage_handle *h, uint64_t *dptr);
int sage_segment_unimport(sage_handle h);   /* no device work may still read the mapping */
/* cross-process device-side dependencies: an interprocess event recorded
 * after `after` (ipc_handle receives its 64-byte cudaIpcEventHandle); the
 * other process opens it and waits on it like any event (stream waits only) */
int sage_ipc_event_export(sage_handle after, sage_handle *ev, void *ipc_handle);
int sage_ipc_event_open(int gpu, const void *ipc_handle, sage_handle *ev);

/* ---- pinned host buffers (the Stage-2 CPU read-only cache, sharing.py:226-228) */
int sage_host_alloc(uint64_t bytes, sage_handle *h, void **ptr);
int sage_host_free(sage_handle h);
/* pin an existing host range (the memory daemon's host-side DB store): loads
 * from it skip the staging memcpy and DMA straight from it                  */
int sage_host_register(void *ptr, uint64_t bytes);
int sage_host_unregister(void *ptr);

/* ---- segment layouts ------------------------------------------------------
 * A layout maps a PACKED host stream (tensors back to back at arbitrary byte
 * offsets, the "DB" record of ref PAPER.md:345-347 Request/Data) onto the
 * landed segment (each tensor at a 16-B aligned offset, zero padding between
 * extents).  dst_off must be ascending, dst_off[0] == 0, 16-B aligned, with
 * dst_off[i] + len[i] <= dst_off[i+1]; src_off[i] + len[i] <= packed_bytes;
 * seg_bytes is a multiple of 16.  n == 0 is the empty segment.              */
int sage_layout_create(const uint64_t *src_off, const uint64_t *dst_off, const uint64_t *len,
                       uint32_t n, uint64_t packed_bytes, uint64_t seg_bytes, sage_handle *layout);
int sage_layout_destroy(sage_handle layout);
/* number of land launches (chunks) a load of this layout takes */
int sage_layout_chunks(sage_handle layout, uint32_t *n_chunks);
/* the checksum a packed record will have once landed (host unpack + checksum):
 * the registration-time content key of the deduplicating sharing manager    */
int sage_layout_checksum(sage_handle layout, const void *packed, uint64_t packed_bytes, uint64_t *checksum);

/* ---- events ---------------------------------------------------------------
 * Every asynchronous op returns an END event; stage begin/end times are read
 * back from events.  Replaces Token.subscribe / set_ready
 * (functions.py:281-301): a follower's SYNC_WAIT is a device-side wait on the
 * leader's END event — no host hop.                                          */
int sage_event_query(sage_handle ev);                  /* SAGE_OK or SAGE_ENOTREADY */
int sage_event_sync(sage_handle ev);
int sage_event_time(sage_handle ev, int64_t *t_us);    /* completion time, library clock */
int sage_event_release(sage_handle ev);
/* a second, independently released handle on the same event (keep a stage
 * END alive past the invocation that owns it: peer readers of a segment)   */
int sage_event_alias(sage_handle ev, sage_handle *out);
/* poll n events; done[i] = 1 when complete.  Blocks up to timeout_us until at
 * least one is complete.  Returns the number complete (>= 0) or an error.    */
int sage_event_poll(const sage_handle *evs, int n, uint8_t *done, int64_t timeout_us);

/* ---- streams / context pool -----------------------------------------------
 * Replaces the GPU_CTX stage node (functions.py:258-264, 285.1 ms at :59).
 * SAGE: a slot of the pre-created stream pool of the (already live) primary
 * context.  FixedGSL: sage_fixedgsl_submit creates a fresh context per
 * invocation (cuCtxCreate), the honest serial baseline.                       */
int sage_ctx_acquire(int gpu, sage_handle *slot);
int sage_ctx_release(sage_handle slot);
/* bind a function context segment on the slot's stream (zero its header and
 * publish the function's descriptor); waits on `wait` events first          */
int sage_ctx_bind(sage_handle slot, uint64_t ctx_dptr, uint64_t ctx_bytes,
                  const sage_handle *wait, int n_wait, sage_handle *begin_ev,
                  sage_handle *end_ev);
/* make the slot's stream wait for events (the SYNC_WAIT node)                */
int sage_stream_wait(sage_handle slot, const sage_handle *evs, int n);
/* SYNC_WAIT as one call: begin event, device-side wait on evs, end event     */
int sage_sync_wait(sage_handle slot, const sage_handle *evs, int n, sage_handle *begin_ev, sage_handle *end_ev);
int sage_slot_record(sage_handle slot, sage_handle *ev);
/* the slot's cudaStream_t (as an integer) so a DNN framework can enqueue a
 * function body (ResNet-50 via PyTorch) on the invocation's stream          */
int sage_slot_stream(sage_handle slot, uint64_t *stream);

/* ---- loads ----------------------------------------------------------------
 * Replaces the CPU_LOAD -> GPU_LOAD chain (functions.py:257-268) and
 * Channel.begin_transfer (resources.py:137-149): the packed host stream goes
 * through the pinned staging ring (CPU memcpy fan-out = CPU_LOAD), chunked
 * double-buffered H2D on the copy engine (= GPU_LOAD) and the sm_100a `land`
 * kernel (unpack + 64-bit content checksum) into dst.                        */
#define SAGE_LOAD_SRC_PINNED   0x1u  /* src is pinned/registered: skip the staging memcpy */
#define SAGE_LOAD_SRC_DEVICE   0x2u  /* src is a device pointer (HBM-resident): no PCIe   */
#define SAGE_LOAD_SRC_PEER     0x4u  /* src is a device pointer on another GPU: NVLink    */
#define SAGE_LOAD_NO_VERIFY    0x8u  /* identity loads from pinned memory or this GPU's HBM:
                                        one DMA / D2D copy, no checksum pass (private
                                        payloads; shared segments always verify)           */
typedef struct {
  int32_t gpu;
  uint32_t flags;
  uint64_t dst;              /* device pointer of the landed segment                  */
  sage_handle layout;        /* 0 = identity: dst gets the packed bytes, padded to 16 */
  const void *src;           /* packed stream (host, or device address cast to ptr)   */
  uint64_t src_bytes;        /* must equal the layout's packed_bytes                  */
  const sage_handle *wait;   /* events the load must wait for (serial plans)          */
  int32_t n_wait;
  int32_t src_gpu;           /* SAGE_LOAD_SRC_PEER: owner GPU of src                  */
} sage_load_desc;
typedef struct {
  int64_t cpu_begin_us, cpu_end_us;   /* CPU_LOAD (staging memcpy); -1 if none        */
  int64_t gpu_begin_us, gpu_end_us;   /* GPU_LOAD (first copy .. last land)          */
  uint64_t host_bytes;                /* bytes memcpy'd into pinned staging          */
  uint64_t link_bytes;                /* bytes over PCIe (or NVLink for PEER)        */
  uint64_t landed_bytes;              /* segment bytes written by land               */
  uint64_t checksum;                  /* content checksum of the landed segment      */
  uint32_t chunks;
  int32_t status;
} sage_load_info;
int sage_segment_load(const sage_load_desc *d, sage_handle *load, sage_handle *end_ev);
int sage_load_info_get(sage_handle load, sage_load_info *out);   /* ENOTREADY until done */
/* CPU_LOAD alone (serial plans): memcpy the DB record into a pinned host
 * buffer on the GPU's host stream after `wait`; begin/end are host-completed
 * device-ordered events                                                      */
int sage_host_load(int gpu, void *pinned_dst, const void *src, uint64_t bytes, const sage_handle *wait,
                   int n_wait, sage_handle *begin_ev, sage_handle *end_ev);
int sage_load_release(sage_handle load);
/* recompute the checksum of a landed segment on the device (verify / dedup) */
int sage_segment_checksum(int gpu, uint64_t dptr, uint64_t bytes, uint64_t *checksum);
/* D2H a landed segment into a pinned host buffer on the copy stream
 * (Stage1 -> Stage2 read-only cache, sharing.py:217-229)                     */
int sage_d2h_cache(int gpu, uint64_t src_dptr, void *host_dst, uint64_t bytes,
                   const sage_handle *wait, int n_wait, sage_handle *end_ev);
/* peer copy of a landed segment to another GPU over NVLink (fan-out)         */
int sage_fanout(int src_gpu, uint64_t src_dptr, int dst_gpu, uint64_t dst_dptr, uint64_t bytes,
                const sage_handle *wait, int n_wait, sage_handle *end_ev);
/* what the box offers for the one-to-many step (simulation.py:113-115 is the
 * shared host channel it replaces): peer reachability per plane, and whether
 * an NVSwitch multicast object can be made (why not, if not)               */
typedef struct {
  int32_t n_gpus, n_devices;
  uint32_t peer_mask[32];        /* bit h of [g]: plane g reaches plane h's pages     */
  int32_t multicast_attr;        /* every device reports MULTICAST_SUPPORTED          */
  int32_t multicast;             /* a multicast object over all devices was created   */
  uint64_t multicast_granularity;
  char why[160];
} sage_fanout_caps_t;
int sage_fanout_caps(sage_fanout_caps_t *out);
/* one segment into up to 32 destination allocations (pool handles, one per
 * GPU): NVLS multicast (multimem.st through a multicast object binding every
 * destination's pages, one pass over the source) when every destination is
 * on its own device and the box allows it, else copy-engine peer copies    */
#define SAGE_BCAST_P2P_ONLY        0x1u
#define SAGE_BCAST_PATH_P2P        0
#define SAGE_BCAST_PATH_MULTICAST  1
typedef struct {
  int32_t src_gpu, n_dst;
  uint64_t src_dptr, bytes;      /* bytes: multiple of 16                            */
  int32_t dst_gpu[32];
  sage_handle dst_alloc[32];
  uint32_t flags;
  int32_t path;                  /* out: SAGE_BCAST_PATH_*                            */
} sage_bcast_desc;
int sage_fanout_broadcast(sage_bcast_desc *d, const sage_handle *wait, int n_wait, sage_handle *end_ev);

/* ---- function bodies (the COMPUTE node, functions.py:276) ----------------- */
#define SAGE_BODY_TOUCH    0  /* read RO + input, write a digest (synthetic functions) */
#define SAGE_BODY_SGEMM    1  /* C[M,N] = A[M,K] . B[K,N], A = RO, fp32 in / TF32 MMA   */
#define SAGE_BODY_STENCIL  2  /* 7-point 3-D Jacobi, coefficients RO, fp32               */
#define SAGE_BODY_SPMV     3  /* CSR y = A.x, A = RO, fp32                              */
#define SAGE_BODY_SPIN     4  /* occupy the SMs for args[0] microseconds                */
#define SAGE_BODY_SGEMM_F32 5 /* the SGEMM on SIMT fp32 cores (exact-fp32 variant)      */
#define SAGE_BODY_SPMV_CSB 7  /* y = A.x, A = RO in the column-sliced block format of
                                 parboil.spmv(fmt="csb"); args = {rows, cols, offsets
                                 offset, entries offset, R, CW, Emax, S | nnz << 8}   */
#define SAGE_BODY_RESNET50 8  /* the registered ResNet-50 program (args[0] = sage_net_create
                                 handle); out = logits then the workspace              */
#define SAGE_BODY_GATHER   6  /* diagnostic: args[0] random 4-B gathers from the input
                                 (a power-of-two float array), the ceiling spmv's x
                                 gathers run against; writes 16 B                   */
/* SGEMM: C[M,N] = A[M,K] . BT[N,K]^T, fp32 in memory, tcgen05 kind::tf32 MMAs
 * with fp32 accumulation in TMEM; args = {M, N, K}; input = BT (K-contiguous,
 * Parboil's "matrix2t")                                                       */
typedef struct {
  int32_t body;
  int32_t pad_;
  uint64_t ro;        /* landed read-only segment (device)              */
  uint64_t input;     /* landed input (device)                          */
  uint64_t out;       /* writable output (device)                       */
  uint64_t ro_bytes, input_bytes, out_bytes;
  int64_t  args[8];   /* body-specific shape parameters                 */
} sage_body_desc;
/* the same with the node's predecessors' END events waited on first         */
int sage_launch_after(sage_handle slot, const sage_handle *wait, int n_wait, const sage_body_desc *b,
                      sage_handle *begin_ev, sage_handle *end_ev);
int sage_return_after(sage_handle slot, const sage_handle *wait, int n_wait, uint64_t src_dptr, void *dst,
                      uint64_t bytes, sage_handle *begin_ev, sage_handle *end_ev);
int sage_launch(sage_handle slot, const sage_body_desc *b, sage_handle *begin_ev,
                sage_handle *end_ev);
/* D2H the result on the slot's stream (the RETURN node)                      */
int sage_return(sage_handle slot, uint64_t src_dptr, void *host_dst, uint64_t bytes,
                sage_handle *begin_ev, sage_handle *end_ev);

/* ---- one invocation in one call (the Parallel-plan fast path) ----------------
 * Replaces the per-node walk of PlanExecution (functions.py:341-433) for the
 * Parallel DAG: GPU_CTX bind ‖ (CPU_LOAD -> GPU_LOAD of RO + input) -> SYNC_WAIT
 * -> COMPUTE -> RETURN, enqueued with device-side dependencies in one call.
 * Stage times, bytes and checksums come back in one collect call.           */
#define SAGE_INV_CTX      0x01u   /* bind ctx_dptr (leader / private context)       */
#define SAGE_INV_RO       0x02u   /* land the read-only segment                     */
#define SAGE_INV_INPUT    0x04u   /* land the invocation input                      */
#define SAGE_INV_SYNC     0x08u   /* SYNC_WAIT on `wait` (leader tokens)             */
#define SAGE_INV_RET_HOST 0x10u   /* ret_dst is host memory: the D2H leaves the slot
                                     stream for a return stream (PCIe overlap)      */
#define SAGE_INV_VERIFY_INPUT 0x20u /* checksum the landed input too (off: the input is
                                     private to the invocation; only shared segments
                                     must be verified, north_star)                  */
#define SAGE_SRC_HOST      0      /* pageable host: staging memcpy (CPU_LOAD) + H2D */
#define SAGE_SRC_PINNED    1      /* pinned host: H2D only                          */
#define SAGE_SRC_HBM       2      /* device-resident source: land from HBM          */
#define SAGE_SRC_PEER      3      /* another GPU's landed segment: land over NVLink */
typedef struct {
  int32_t gpu;
  uint32_t flags;
  uint64_t ctx_dptr, ctx_bytes;
  int32_t ro_kind, ro_src_gpu;
  sage_handle ro_layout;          /* 0 = identity (cache reload / peer copy)        */
  const void *ro_src;
  uint64_t ro_src_bytes, ro_dst;
  sage_handle ro_wait[2];         /* e.g. the Stage-2 cache D2H, a peer's token     */
  int32_t n_ro_wait;
  int32_t in_kind;
  const void *in_src;
  uint64_t in_bytes, in_dst;
  sage_handle wait[4];            /* SYNC_WAIT: leader RO / ctx END events, and the
                                     compute-gate predecessor (ComputeGate)          */
  int32_t n_wait;
  int32_t pad_;
  sage_body_desc body;            /* COMPUTE                                        */
  uint64_t ret_src;               /* RETURN: D2H (or D2D) ret_bytes to ret_dst      */
  void *ret_dst;
  uint64_t ret_bytes;
} sage_invoke_desc;
typedef struct {
  int64_t t[16];                  /* begin/end per reference Stage (cf. FixedGSL info) */
  uint64_t host_bytes, link_bytes;
  uint64_t ro_checksum, in_checksum;
  int64_t ro_landed_us;           /* -1 if no RO load                               */
  int32_t status, pad_;
} sage_invoke_info;
/* ro_end / ctx_end (may be null) receive borrowed handles of the RO-landed and
 * context-bound events, valid until sage_invoke_release                      */
int sage_invoke(const sage_invoke_desc *d, sage_handle *inv, sage_handle *done_ev, sage_handle *ro_end,
                sage_handle *ctx_end);
int sage_invoke_collect(sage_handle inv, sage_invoke_info *out);   /* ENOTREADY until done */
/* Finished invocations in completion order: up to `max` handles into `out`,
 * waiting up to timeout_us for the first.  Returns the count (>= 0).  The
 * device signals completion with a host function on the slot stream; the
 * library's completion thread has already resolved every stage time, so the
 * following sage_invoke_collect is a copy.  (Replaces polling each
 * invocation's done event: PlanExecution completion, functions.py:420-433.) */
int sage_invoke_ready(sage_handle *out, int max, int64_t timeout_us);
int sage_invoke_release(sage_handle inv);

/* ---- FixedGSL serial baseline (policies.py:102-126, functions.py:261-267) ---
 * One invocation = fresh cuCtxCreate + cudaMalloc + pageable synchronous
 * per-tensor cudaMemcpy + body + D2H + context teardown, run on a library
 * worker thread; completion is polled through its end event.                 */
#define SAGE_INSTANCE_THREAD   0  /* a fresh context on a library worker thread        */
#define SAGE_INSTANCE_PROCESS  1  /* a fresh OS process per instance (sage_instance_worker) */
#define SAGE_INSTANCE_POOLED   2  /* DGSF: run in a pre-created context (no GPU_CTX)    */
typedef struct {
  int32_t gpu;
  int32_t mode;                  /* SAGE_INSTANCE_*                                  */
  sage_handle layout;            /* RO layout (0 = identity)                         */
  const void *ro_src; uint64_t ro_src_bytes;
  const void *input;  uint64_t input_bytes;
  uint64_t alloc_bytes;          /* device bytes the instance reserves (1 GiB-rounded) */
  sage_body_desc body;           /* ro/input/out pointers are filled in by the worker */
  void *result; uint64_t result_bytes;
  sage_handle ctx;               /* SAGE_INSTANCE_POOLED: from sage_instance_ctx_create */
} sage_fixedgsl_desc;
typedef struct {
  int64_t t[16];                 /* begin/end per reference Stage (functions.py:164-176
                                    order: container,cpu_ctx,cpu_load,gpu_ctx,gpu_load,
                                    sync_wait,compute,return); -1 = absent            */
  uint64_t checksum;             /* checksum of the RO bytes as loaded                */
  int64_t teardown_us;           /* cuCtxDestroy time (after completion)              */
  int32_t status;
  int32_t pad_;
} sage_fixedgsl_info;
int sage_fixedgsl_submit(const sage_fixedgsl_desc *d, sage_handle *job, sage_handle *end_ev);
int sage_fixedgsl_info_get(sage_handle job, sage_fixedgsl_info *out);
int sage_fixedgsl_release(sage_handle job);
/* DGSF's pre-created contexts (policies.py:163-179): a real cuCtxCreate made at
 * registration with the body's kernels loaded; one job at a time runs in it  */
int sage_instance_ctx_create(int gpu, int body, sage_handle *ctx);
int sage_instance_ctx_destroy(sage_handle ctx);
/* the entry of an instance process (SAGE_INSTANCE_PROCESS): sage_instance_worker
 * calls it with the memfd of its region; not for other callers               */
int sage_instance_child(int fd);

/* ---- measurement ------------------------------------------------------------
 * Live kernel timing for the roofline: when enabled, every land / body launch
 * is bracketed by CUDA events on the stream it is launched on; stats_get
 * resolves them and reports launches, summed device time and algorithmic
 * bytes (land: packed bytes read + segment bytes written).                    */
#define SAGE_KERNEL_LAND     0
#define SAGE_KERNEL_TOUCH    1
#define SAGE_KERNEL_SGEMM    2
#define SAGE_KERNEL_STENCIL  3
#define SAGE_KERNEL_SPMV     4
#define SAGE_KERNEL_VERIFY   5   /* direct-path checksum of DMA'd identity loads */
#define SAGE_KERNEL_GATHER   6   /* SAGE_BODY_GATHER; work = gathers               */
#define SAGE_KERNEL_KINDS    7
int sage_stats_enable(int on);
int sage_stats_reset(void);
int sage_stats_get(int gpu, int kind, uint64_t *launches, double *total_us, uint64_t *bytes);
/* drain every stream of a GPU; record a timing marker on its idle aux stream */
int sage_device_sync(int gpu);
int sage_mark(int gpu, sage_handle *ev);
/* elapsed µs between two completed events of the same GPU (device clock) */
int sage_event_elapsed(sage_handle a, sage_handle b, double *us);

/* ---- ResNet-50 convolution (tcgen05 implicit GEMM, BF16) -------------------
 * One convolution of NHWC bf16 activations with OHWI bf16 filters read in
 * place, fp32 accumulation in TMEM, epilogue y = acc * scale + bias
 * (+ residual) (ReLU), bf16 NHWC out; scale / bias fold batch-norm from its
 * bf16 parameters (scale = gamma * rsqrt(var + eps), bias = beta - mean *
 * scale; gamma == 0 pointer: identity).  SAGE_CONV_C4: the input is NHWC with
 * 4 channels (conv1's 3 padded) and the filter is [Cout][ceil(R*S/16)*64].
 * Replaces the COMPUTE delay of the resnet50 record (functions.py:154, :276). */
#define SAGE_CONV_NHWC  0
#define SAGE_CONV_C4    1
/* SAGE_CONV_S2D: the stem (7x7 stride 2 pad 3 over 3 channels) as a stride-1
 * 4x4 convolution over its 2x2 space-to-depth input: NHWC with 16 channels
 * (dr, ds, c; c padded to 4) of (H/2, W/2) pixels, filter [Cout][4][4][16]
 * with w'[a][b][dr][ds][c] = w[2a+dr-1][2b+ds-1][c] (zero outside 7x7),
 * cin = 16, r = s = 4, stride 1, pad 2; the output has the input's size.
 * Every K-block is one filter row of 4 taps x 16 channels = 128 B per pixel,
 * so the gather is the regular layers' coalesced one.                      */
#define SAGE_CONV_S2D   2
typedef struct {
  uint64_t x, w, out, residual;             /* device pointers (residual 0 = none) */
  uint64_t bn_gamma, bn_beta, bn_mean, bn_var;
  float bn_eps;
  int32_t n, h, w_, cin, cout, r, s, stride, pad, relu, mode, pad_;
} sage_conv_desc;
int sage_conv(sage_handle slot, const sage_conv_desc *d);

/* ---- ResNet-50 body: a registered program of native kernels --------------
 * Ops address the landed RO segment by offset (filters OHWI bf16, batch-norm
 * bf16, classifier) and buffers by id: SAGE_NET_BUF_INPUT (the request image,
 * NHWC bf16), SAGE_NET_BUF_OUT (the fp32 logits), SAGE_NET_BUF_WS0 + i (the
 * invocation's workspace, laid out after the logits in its writable segment).
 * Launched as body SAGE_BODY_RESNET50 with args[0] = the network handle.   */
#define SAGE_NET_PAD_INPUT  1   /* NHWC3 -> NHWC4 (the stem's C4 gather)       */
#define SAGE_NET_CONV       2   /* sage_conv on (src, filter, BN, res) -> dst  */
#define SAGE_NET_MAXPOOL    3   /* 3x3 stride 2 pad 1                           */
#define SAGE_NET_POOL_FC    4   /* avg pool into buffer `res` + classifier -> dst (fp32) */
#define SAGE_NET_S2D_INPUT  5   /* NHWC3 (h, w) -> 2x2 space-to-depth NHWC16 (h/2, w/2) (SAGE_CONV_S2D stem) */
#define SAGE_NET_BUF_INPUT  0
#define SAGE_NET_BUF_OUT    1
#define SAGE_NET_BUF_WS0    2
typedef struct {
  int32_t kind, src, dst, res;               /* buffer ids (res -1: none)        */
  uint64_t w_off, g_off, b_off, m_off, v_off; /* RO offsets (g_off = ~0: no BN)   */
  float eps;
  int32_t n, h, w, cin, cout, r, s, stride, pad, relu, mode;
} sage_net_op;
int sage_net_create(const sage_net_op *ops, int n_ops, const uint64_t *buf_bytes, int n_bufs, sage_handle *net,
                    uint64_t *workspace_bytes);
int sage_net_destroy(sage_handle net);

/* ---- sharing manager: the native resident table ----------------------------
 * Replaces SharingManager's resident dict and its state machine
 * (sharing.py:103-335): warmth classification (:115-125), delta sizes
 * (:126-134), leader election by allocation (:136-177), the refcounted
 * release (:181-196), the four-stage timed decay (:217-246), eviction
 * (:248-263), victim choice under pressure (:271-298) and the invariant sweep
 * (:305-335); plus a content index for deduplicating identical RO records.
 * Host code: usable without a GPU.  The caller owns the ledger allocations and
 * the engine timers and executes each returned step (sharing.py).           */
#define SAGE_SHARE_RO           0x1u   /* ro_sharing (policies.py:29)                  */
#define SAGE_SHARE_CTX          0x2u   /* ctx_sharing                                   */
#define SAGE_SHARE_MULTI_STAGE  0x4u   /* multi_stage_exit                              */
#define SAGE_FN_HAS_RO          0x1u   /* fn_flags: ro_mem_mb > 0                        */
#define SAGE_WARMTH_COLD        0      /* WarmthClass order (functions.py:23-41)        */
#define SAGE_WARMTH_STAGE4      1
#define SAGE_WARMTH_STAGE3      2
#define SAGE_WARMTH_STAGE2      3
#define SAGE_WARMTH_STAGE1_HOT  4
#define SAGE_RES_ACTIVE         0      /* ResidentState (sharing.py:30-36)              */
#define SAGE_RES_STAGE1         1
#define SAGE_RES_STAGE2         2
#define SAGE_RES_STAGE3         3
#define SAGE_RES_STAGE4         4
#define SAGE_TOKEN_RO           0
#define SAGE_TOKEN_CTX          1
typedef struct {
  int32_t warmth;
  uint8_t shared_ro, shared_ctx, wait_ro, wait_ctx;
  uint8_t leader_ro, leader_ctx;     /* this admission allocates the shared segment   */
  uint8_t timer_cancelled;           /* a decay timer was pending: cancel the engine's */
  uint8_t new_resident;
  uint64_t alloc_ro, alloc_ctx;      /* bytes of new shared segments to allocate      */
  uint64_t resident;                 /* resident id (0 in a preview of none)          */
} sage_share_grant;
/* step actions, executed by the caller in this order */
#define SAGE_STEP_CACHE_RO     0x01u  /* allocate the host RO cache (+ D2H of the held segment) */
#define SAGE_STEP_FREE_RO      0x02u  /* free the GPU RO segment (after the cache D2H / readers) */
#define SAGE_STEP_FREE_CTX     0x04u
#define SAGE_STEP_DROP_CACHE   0x08u
#define SAGE_STEP_EVICT        0x10u  /* the resident is gone                          */
#define SAGE_STEP_GPU_FREED    0x20u  /* wake the GPU's queue (policies.on_memory_freed) */
#define SAGE_STEP_ARM          0x40u  /* schedule the decay timer (deadline_us, timer_gen) */
typedef struct {
  uint32_t actions;
  int32_t state_before, state_after;
  uint32_t timer_gen;
  uint8_t timer_cancelled, _pad[7];
  int64_t deadline_us;
  uint64_t resident;
} sage_share_step;
#define SAGE_HOLD_RO         0x1u
#define SAGE_HOLD_CTX        0x2u
#define SAGE_HOLD_CACHE      0x4u
#define SAGE_HOLD_CPU_CTX    0x8u
#define SAGE_HOLD_CONTAINER  0x10u
typedef struct {
  uint64_t resident;
  int32_t fn, gpu, state;
  uint32_t active, holds, timer_gen;
  uint64_t ro_bytes, ctx_bytes;
  int64_t last_activity_us, deadline_us;
  uint32_t has_checksum, _pad;
  uint64_t checksum;
} sage_resident_info;
int sage_share_create(int n_gpus, uint32_t flags, int64_t keep_alive_us, const int64_t intervals_us[4],
                      sage_handle *tab);
int sage_share_destroy(sage_handle tab);
int sage_share_preview(sage_handle tab, int32_t fn, int gpu, uint64_t ro_bytes, uint64_t ctx_bytes,
                       uint32_t fn_flags, sage_share_grant *g);                /* sharing.py:108-134 */
int sage_share_admit(sage_handle tab, int32_t fn, int gpu, uint64_t ro_bytes, uint64_t ctx_bytes,
                     uint32_t fn_flags, int64_t now_us, sage_share_grant *g);  /* sharing.py:136-177 */
/* preview + capacity check + admit in one call (policies.py:286-297 + the
 * admit): the shared segments this admission would lead plus extra_bytes of
 * private ones, rounded up to granularity as one request, must fit in
 * avail_bytes (< 0: unlimited).  Refused: SAGE_ENOMEM, *g holds the preview,
 * the table is unchanged (the caller demotes and calls sage_share_admit).
 * opts SAGE_ADMIT_DEFER_RO_LEADER: an admission that would lead a new RO
 * segment returns SAGE_ADMIT_DEFERRED (> 0) with the preview, table unchanged
 * (content dedup: the caller looks for identical landed content first).     */
#define SAGE_ADMIT_DEFER_RO_LEADER 0x1u
#define SAGE_ADMIT_DEFERRED        1
int sage_share_admit_within(sage_handle tab, int32_t fn, int gpu, uint64_t ro_bytes, uint64_t ctx_bytes,
                            uint32_t fn_flags, int64_t now_us, int64_t avail_bytes, uint64_t extra_bytes,
                            uint64_t granularity, uint32_t opts, sage_share_grant *g);
/* attach the leader's stage END event to a token (ev != 0) or mark it ready  */
int sage_share_token(sage_handle tab, uint64_t resident, int kind, sage_handle ev);
int sage_share_token_ready(sage_handle tab, uint64_t resident, int kind, int *ready);
int sage_share_release(sage_handle tab, int32_t fn, int gpu, int64_t now_us,
                       sage_share_step *out);                                  /* sharing.py:181-196 */
/* the decay timer (resident, timer_gen) fired                                */
int sage_share_expire(sage_handle tab, uint64_t resident, uint32_t timer_gen, int64_t now_us,
                      sage_share_step *out);                                   /* sharing.py:203-246 */
int sage_share_victim(sage_handle tab, int gpu, int32_t exclude_fn, uint64_t *resident); /* :288-298 */
int sage_share_demote(sage_handle tab, uint64_t resident, int64_t now_us,
                      sage_share_step *out);                                   /* sharing.py:271-286 */
int sage_share_evict(sage_handle tab, uint64_t resident, sage_share_step *out); /* sharing.py:248-263 */
int sage_share_info(sage_handle tab, uint64_t resident, sage_resident_info *out);
int sage_share_lookup(sage_handle tab, int32_t fn, int gpu, uint64_t *resident);
int sage_share_list(sage_handle tab, uint64_t *ids, int cap, int *n);
int sage_share_ro_loads(sage_handle tab, int32_t fn, int gpu, uint32_t *n);  /* sharing.py:174-175 */
/* content index: a landed RO segment's checksum; lookup of another function's
 * resident segment with the same content on a GPU (token ready)             */
int sage_share_set_checksum(sage_handle tab, uint64_t resident, uint64_t checksum);
int sage_share_find_content(sage_handle tab, int gpu, uint64_t checksum, int32_t exclude_fn,
                            uint64_t *resident);
int sage_share_check(sage_handle tab);                                         /* sharing.py:305-335 */

/* ---- test support (never on the product path) ------------------------------
 * Runs the chunk planner and the land byte semantics on the host so the
 * planner can be checked against the oracle without a GPU.                   */
int sage_debug_emulate_land(sage_handle layout, const void *packed, uint64_t packed_bytes, void *seg_out,
                            uint64_t chunk_bytes, uint64_t *checksum);

#ifdef __cplusplus
}
#endif
#endif /* SAGE_DP_H */
