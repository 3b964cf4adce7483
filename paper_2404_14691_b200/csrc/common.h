// common.h — internals shared by the libsagedp translation units.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only: ranges cost a pointer test unless a profiler attaches

#include <pthread.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/sage_dp.h"

namespace sage {

// host-side NVTX range for a data-plane phase (issue, load, body launch):
// visible in nsys / ncu timelines, no cost without a profiler attached
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

// ---------------------------------------------------------------- errors ----
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);
int cu_fail(CUresult r, const char *what);

#define SAGE_CUDA(call)                                   \
  do {                                                    \
    cudaError_t e__ = (call);                             \
    if (e__ != cudaSuccess) return ::sage::cuda_fail(e__, #call); \
  } while (0)
#define SAGE_CU(call)                                     \
  do {                                                    \
    CUresult r__ = (call);                                \
    if (r__ != CUDA_SUCCESS) return ::sage::cu_fail(r__, #call); \
  } while (0)
#define SAGE_TRY(call)                                    \
  do {                                                    \
    int rc__ = (call);                                    \
    if (rc__ != SAGE_OK) return rc__;                     \
  } while (0)

// ------------------------------------------------------- driver entry pts ---
struct Driver {
  PFN_cuMemCreate_v10020 MemCreate = nullptr;
  PFN_cuMemRelease_v10020 MemRelease = nullptr;
  PFN_cuMemAddressReserve_v10020 MemAddressReserve = nullptr;
  PFN_cuMemAddressFree_v10020 MemAddressFree = nullptr;
  PFN_cuMemMap_v10020 MemMap = nullptr;
  PFN_cuMemUnmap_v10020 MemUnmap = nullptr;
  PFN_cuMemSetAccess_v10020 MemSetAccess = nullptr;
  PFN_cuMemGetAllocationGranularity_v10020 MemGetAllocationGranularity = nullptr;
  PFN_cuCtxCreate_v3020 CtxCreate = nullptr;
  PFN_cuCtxDestroy_v4000 CtxDestroy = nullptr;
  PFN_cuCtxSetCurrent_v4000 CtxSetCurrent = nullptr;
  PFN_cuCtxGetCurrent_v4000 CtxGetCurrent = nullptr;
  PFN_cuDevicePrimaryCtxRetain_v7000 DevicePrimaryCtxRetain = nullptr;
  PFN_cuMemExportToShareableHandle_v10020 MemExportToShareableHandle = nullptr;
  PFN_cuMemImportFromShareableHandle_v10020 MemImportFromShareableHandle = nullptr;
};
extern Driver drv;
int load_driver();

// ------------------------------------------------------------------ clock ---
int64_t host_now_us();   // CLOCK_MONOTONIC µs since sage_init

// ---------------------------------------------------------------- handles ---
enum class Kind : uint8_t { Event = 1, Slot, Alloc, Host, Layout, Load, Job, Inv };
inline sage_handle make_handle(Kind k, uint64_t id) { return ((uint64_t)k << 56) | id; }
inline Kind handle_kind(sage_handle h) { return (Kind)(h >> 56); }

// --------------------------------------------------------------- events -----
struct Event {
  int gpu = -1;
  cudaEvent_t ev = nullptr;      // device event (null for host jobs)
  std::atomic<int> host_done{0}; // host job completion (FixedGSL)
  int64_t host_time = -1;        // host job completion time
  std::atomic<bool> recorded{false};
  std::atomic<bool> pending{false}; // created for an invocation not yet issued (invoke.cu):
                                    // queries report "not ready", waits block until recorded
  std::atomic<int> refs{1};      // handles naming this event (event_alias)
  std::atomic<bool> done{false}; // sticky completion (skips re-queries)
  int64_t t_cache = INT64_MIN;   // host-clock time once resolved
  bool ipc = false;              // interprocess event (no timing; destroyed, never pooled)
};
int event_new(int gpu, sage_handle *h, Event **out);        // device event
int event_new_host(sage_handle *h, Event **out);            // host-completed event
// a second handle on the same recorded event (a stage boundary shared by the
// stage that ends and the one that begins there); released independently
int event_alias(sage_handle src, sage_handle *out);
Event *event_get(sage_handle h);
int event_record(Event *e, cudaStream_t s);
int event_time_us(Event *e, int64_t *t);                    // requires completion
int event_query(Event *e);                                  // SAGE_OK / SAGE_ENOTREADY
// block until a pending event has been recorded by the issuer; ESTATE for an
// event that was never recorded and is not pending
int event_await_recorded(Event *e);

// --------------------------------------------------------------- per GPU ----
struct Layout;

struct ChunkScratch {  // per-load device accumulator + pinned result
  unsigned long long *d_acc = nullptr;   // ring of accumulators on device
  unsigned int *d_done = nullptr;        // ring of finished-block counters
  unsigned long long *h_res = nullptr;   // mapped pinned results (host view)
  unsigned long long *d_res = nullptr;   // ... device view
  uint32_t n = 0;
  std::atomic<uint64_t> next{0};
  // a slot belongs to one load from open to release: its result must not be
  // overwritten by a later load while the first is still unread
  std::vector<uint8_t> busy;
  std::mutex mu;
};

struct Gpu {
  int id = -1;                            // logical GPU (the runtime's index)
  int dev = -1;                           // physical CUDA device it runs on
  int sm_count = 0;
  CUcontext primary = nullptr;
  cudaStream_t copy = nullptr, land = nullptr, host = nullptr, d2h = nullptr, aux = nullptr;
  cudaStream_t direct = nullptr;          // pinned identity loads: back-to-back DMAs, off the ring
  cudaStream_t verify = nullptr;          // ... and their checksum pass, so DMAs never wait on it
  cudaEvent_t ev_dma = nullptr;           // direct -> verify hand-off (re-recorded under load_mu)
  std::vector<cudaStream_t> slots;        // pre-created stream pool (the "context pool")
  std::vector<cudaStream_t> rets;         // RETURN copy streams (empty: copy on the slot stream)
  cudaEvent_t ev_ret = nullptr;           // slot -> return stream hand-off (under ret_mu)
  uint64_t ret_seq = 0;
  std::mutex ret_mu;
  std::vector<int> slot_free;             // free slot indices
  std::mutex slot_mu;
  // staging rings
  uint32_t ring = 0;
  uint64_t chunk = 0;
  uint8_t *pin = nullptr;                 // ring * (chunk + 64) pinned
  uint8_t *dstage = nullptr;              // ring * (chunk + 64) device
  std::vector<cudaEvent_t> ev_cpu, ev_h2d, ev_land;  // per ring slot
  uint64_t chunk_seq = 0;                 // global chunk sequence (ring position)
  std::mutex load_mu;                     // serialises load enqueue (ring order)
  ChunkScratch scratch;
  // clock anchor (see clock_anchor_refresh)
  cudaStream_t clock = nullptr;           // dedicated top-priority stream, never loaded
  cudaStream_t ipc = nullptr;             // records interprocess events (fan-out to other processes)
  std::mutex ipc_mu;
  cudaEvent_t anchor_trial = nullptr;
  cudaEvent_t anchor = nullptr;
  int64_t anchor_us = 0;
  std::mutex anchor_mu;
  // pool
  struct Pool *pool = nullptr;
  // misc scratch for checksum verify
  unsigned long long *d_verify = nullptr;
  // live kernel timing
  struct StatRec { int kind; cudaEvent_t b, e; uint64_t bytes; };
  std::mutex stat_mu;
  std::vector<StatRec> stat_pending;
  std::vector<cudaEvent_t> stat_free;
  uint64_t stat_count[8] = {0}, stat_bytes[8] = {0};
  double stat_us[8] = {0};
};

struct State {
  bool up = false;
  int n_gpus = 0;
  uint64_t chunk = 8ull << 20;
  uint32_t flags = 0;
  std::vector<std::unique_ptr<Gpu>> gpus;
  int host_threads = 8;
  int n_devices = 1;                      // physical devices visible at init
};
extern State st;
Gpu *gpu_get(int g);
// physical device of logical GPU g (identity unless SAGE_INIT_SHARE_DEVICE
// folds several logical planes onto fewer devices)
inline int dev_of(int g) {
  return (g >= 0 && g < (int)st.gpus.size() && st.gpus[g]) ? st.gpus[g]->dev : g;
}
int require_up();

// device->host clock anchor (core.cu); call with G->anchor_mu held
void clock_anchor_refresh(Gpu *G, bool force = false);

// host memcpy fan-out pool (CPU_LOAD)
void parallel_memcpy(void *dst, const void *src, size_t bytes);
void pool_threads_start(int n);
void pool_threads_stop();

// pool internals (pool.cu)
int pool_alloc_phys(sage_handle h, CUmemGenericAllocationHandle *ph, uint64_t *phys, uint64_t *dptr, int *gpu);
int pool_create(Gpu *g, uint64_t capacity);
void pool_destroy(Gpu *g);

// device state (pool.cu)
int gpu_setup(int id, uint64_t pool_bytes, uint64_t staging_bytes, uint64_t chunk);
void gpu_teardown(Gpu *G);
int slot_stream(sage_handle h, Gpu **G, cudaStream_t *s);
int wait_events(cudaStream_t s, const sage_handle *w, int n);
// bodies (bodies.cu)
int launch_body(const sage_body_desc *b, cudaStream_t s, int sm_count);
int launch_timed(Gpu *G, cudaStream_t s, const sage_body_desc *b);   // + live kernel stats
// RETURN copy after `prev` (the boundary event just recorded on slot stream
// s, or 0): on s, or -- a D2H (host_dst) with G->rets configured -- on a
// return stream
// pre_end (optional): a pre-created event to record as the END (the caller
// gets an alias of it)
int return_enqueue(Gpu *G, cudaStream_t s, sage_handle prev, uint64_t src, void *dst, uint64_t bytes,
                   bool host_dst, sage_handle *begin_ev, sage_handle *end_ev, sage_handle pre_end = 0);
int touch_body_kernels(int body);   // module-load one body's kernels into the current context
int64_t host_epoch_us();            // CLOCK_MONOTONIC µs of the library epoch (sage_init)
int64_t mono_us();                  // CLOCK_MONOTONIC µs (absolute)
// tcgen05 GEMM (gemm_tc.cu)
int sgemm_tc(const float *A, const float *BT, float *C, int M, int N, int K, cudaStream_t s);
int touch_tc_kernels();
// tcgen05 implicit-GEMM convolution (conv_tc.cu)
struct ConvFrame {                  // graph mode: buffers read from a device frame
  const uint64_t *frame;
  int x_sel, res_sel, out_sel;      // frame slots (res_sel < 0: no residual)
  uint64_t x_off, res_off, out_off;
};
int conv_bf16(const sage_conv_desc *d, cudaStream_t s, int sms, const ConvFrame *f);
int conv_optin_all();
int touch_conv_kernels();
// the ResNet-50 program body (resnet.cu)
int net_run(const sage_body_desc *b, cudaStream_t s, int sms);
void nets_release_graphs();   // sage_shutdown: captured programs die with the device state
int touch_net_kernels();
// column-sliced block spmv (spmv_csb.cu)
int spmv_csb(const sage_body_desc *b, cudaStream_t s, int sm_count);
int touch_csb_kernel();

// invocations (invoke.cu): stop the completion thread, drop live records
void invoke_shutdown();
// wait until the invocation issuer has enqueued everything submitted for
// `gpu` (-1: every GPU)
void issuer_drain(int gpu);

// sage_segment_load with an optional pre-created END event (land.cu)
int segment_load(const sage_load_desc *d, sage_handle *load_out, sage_handle *end_ev, sage_handle pre_end);
// ... in pieces: open validates, creates the events and applies the waits;
// a load that is not staged through the ring completes inside open (*cur ==
// nullptr, handles out).  Otherwise each step enqueues chunks until `budget`
// link bytes moved (piece_ev: recorded after the piece's last H2D) and the
// last one sets *done and hands out the handles.
struct LoadCursor;
int segment_load_open(const sage_load_desc *d, sage_handle pre_end, LoadCursor **cur, sage_handle *load_out,
                      sage_handle *end_ev);
int segment_load_step(LoadCursor *c, uint64_t budget, uint64_t *bytes, sage_handle *piece_ev, bool *done,
                      sage_handle *load_out, sage_handle *end_ev);
void segment_load_close(LoadCursor *c);

// layouts (land.cu)
int layouts_destroy_all();

// live kernel timing (core.cu): bracket a launch on its stream when enabled
bool stats_on();
cudaEvent_t stat_begin(Gpu *G, cudaStream_t s);
void stat_end(Gpu *G, cudaStream_t s, int kind, cudaEvent_t b, uint64_t bytes);
void stats_clear_gpu(Gpu *G);

}  // namespace sage
