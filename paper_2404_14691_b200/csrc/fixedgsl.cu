// fixedgsl.cu — the FixedGSL serial baseline on real hardware.
//
// Reference: InstancePolicy (policies.py:102-126) admits one size-fixed
// instance per invocation and runs the SERIAL plan
// (functions.py:261-267): CPU ctx -> CPU load -> GPU ctx -> GPU load ->
// compute -> return, each stage after the previous.  Here every stage is the
// real operation a container-per-function deployment performs:
//   CPU_CTX   host-side instance state
//   CPU_LOAD  malloc + memcpy of the DB record into the instance's private
//             (pageable) host memory
//   GPU_CTX   cuCtxCreate of a fresh context + module load
//   GPU_LOAD  cudaMalloc of the instance reservation + one synchronous
//             pageable cudaMemcpy per tensor + the input
//   COMPUTE   the body kernel, synchronised
//   RETURN    synchronous D2H of the result
// then the context is destroyed (timed separately as teardown).
#include "common.h"
#include "checksum.cuh"

#include <chrono>

namespace sage {

struct Job {
  sage_fixedgsl_desc d;
  sage_fixedgsl_info info;
  Event *ev = nullptr;
  std::atomic<int> done{0};
  std::vector<uint64_t> src_off, dst_off, len;  // layout copy (tensor list)
  uint64_t seg = 0;
};

static std::mutex g_job_mu;
static std::unordered_map<uint64_t, Job *> g_jobs;
static std::atomic<uint64_t> g_job_next{1};
static std::mutex g_sem_mu;
static std::condition_variable g_sem_cv;
static int g_running = 0;
static const int kMaxConcurrent = 32;

extern int layout_tensors(sage_handle h, std::vector<uint64_t> *src, std::vector<uint64_t> *dst,
                          std::vector<uint64_t> *len, uint64_t *packed, uint64_t *seg);

static void stamp(Job *J, int stage, bool end) { J->info.t[2 * stage + (end ? 1 : 0)] = host_now_us(); }

static int run_job(Job *J) {
  const sage_fixedgsl_desc &d = J->d;
  enum { CPU_CTX = 1, CPU_LOAD = 2, GPU_CTX = 3, GPU_LOAD = 4, COMPUTE = 6, RET = 7 };
  // CPU_CTX
  stamp(J, CPU_CTX, false);
  std::vector<uint8_t> input_copy;
  stamp(J, CPU_CTX, true);
  // CPU_LOAD: the instance reads its data from the DB into private memory
  stamp(J, CPU_LOAD, false);
  uint8_t *priv = (uint8_t *)malloc(d.ro_src_bytes ? d.ro_src_bytes : 1);
  if (!priv) return fail(SAGE_ENOMEM, "fixedgsl: host malloc");
  if (d.ro_src_bytes) memcpy(priv, d.ro_src, d.ro_src_bytes);
  stamp(J, CPU_LOAD, true);
  // GPU_CTX: a fresh context (what a cold container pays)
  stamp(J, GPU_CTX, false);
  CUcontext ctx = nullptr;
  CUresult r = drv.CtxCreate(&ctx, 0, (CUdevice)dev_of(d.gpu));
  if (r != CUDA_SUCCESS) { free(priv); return cu_fail(r, "cuCtxCreate"); }
  drv.CtxSetCurrent(ctx);
  int rc = touch_all_kernels();
  stamp(J, GPU_CTX, true);
  uint8_t *dmem = nullptr;
  if (rc == SAGE_OK) {
    // GPU_LOAD: reservation + per-tensor synchronous pageable copies
    stamp(J, GPU_LOAD, false);
    uint64_t ro_b = J->seg, in_b = (d.input_bytes + 255) & ~255ull, out_b = (d.body.out_bytes + 255) & ~255ull;
    uint64_t need = ((ro_b + 255) & ~255ull) + in_b + out_b;
    uint64_t bytes = std::max<uint64_t>(d.alloc_bytes, need);
    cudaError_t e = cudaMalloc(&dmem, bytes);
    if (e != cudaSuccess) rc = cuda_fail(e, "fixedgsl cudaMalloc");
    uint8_t *ro = dmem, *in = dmem + ((ro_b + 255) & ~255ull), *out = in + in_b;
    if (rc == SAGE_OK && ro_b) e = cudaMemset(ro, 0, ro_b);
    for (size_t i = 0; rc == SAGE_OK && i < J->len.size(); ++i)
      if (J->len[i] && (e = cudaMemcpy(ro + J->dst_off[i], priv + J->src_off[i], J->len[i], cudaMemcpyHostToDevice)) != cudaSuccess)
        rc = cuda_fail(e, "fixedgsl cudaMemcpy");
    if (rc == SAGE_OK && in_b && (e = cudaMemset(in, 0, in_b)) != cudaSuccess) rc = cuda_fail(e, "fixedgsl memset");
    if (rc == SAGE_OK && d.input_bytes && (e = cudaMemcpy(in, d.input, d.input_bytes, cudaMemcpyHostToDevice)) != cudaSuccess)
      rc = cuda_fail(e, "fixedgsl input cudaMemcpy");
    stamp(J, GPU_LOAD, true);
    // COMPUTE
    if (rc == SAGE_OK) {
      stamp(J, COMPUTE, false);
      sage_body_desc b = d.body;
      b.ro = (uint64_t)ro; b.ro_bytes = ro_b;
      b.input = (uint64_t)in; b.input_bytes = (d.input_bytes + 15) & ~15ull;
      b.out = (uint64_t)out; b.out_bytes = d.body.out_bytes;
      rc = launch_body(&b, 0, gpu_get(d.gpu)->sm_count);
      if (rc == SAGE_OK && (e = cudaDeviceSynchronize()) != cudaSuccess) rc = cuda_fail(e, "fixedgsl compute");
      stamp(J, COMPUTE, true);
    }
    // RETURN
    if (rc == SAGE_OK) {
      stamp(J, RET, false);
      if (d.result_bytes && (e = cudaMemcpy(d.result, out, d.result_bytes, cudaMemcpyDeviceToHost)) != cudaSuccess)
        rc = cuda_fail(e, "fixedgsl return");
      stamp(J, RET, true);
    }
    // verification only (outside every stage): checksum of what was loaded
    if (rc == SAGE_OK && ro_b) {
      std::vector<uint8_t> host(ro_b);
      if (cudaMemcpy(host.data(), ro, ro_b, cudaMemcpyDeviceToHost) == cudaSuccess)
        J->info.checksum = host_checksum(host.data(), ro_b);
    }
  }
  // teardown (after completion; reported separately)
  int64_t t0 = host_now_us();
  if (dmem) cudaFree(dmem);
  drv.CtxSetCurrent(nullptr);
  drv.CtxDestroy(ctx);
  J->info.teardown_us = host_now_us() - t0;
  free(priv);
  return rc;
}

static void job_thread(Job *J) {
  {
    std::unique_lock<std::mutex> lk(g_sem_mu);
    g_sem_cv.wait(lk, [] { return g_running < kMaxConcurrent; });
    ++g_running;
  }
  int rc = run_job(J);
  J->info.status = rc;
  {
    std::lock_guard<std::mutex> lk(g_sem_mu);
    --g_running;
  }
  g_sem_cv.notify_one();
  // the caller may release the end event as soon as it reads complete, and
  // the job only after `done`: publish the event first
  Event *ev = J->ev;
  ev->host_time = host_now_us();
  J->done.store(1, std::memory_order_release);
  ev->host_done.store(1, std::memory_order_release);
}

}  // namespace sage

using namespace sage;

extern "C" {

int sage_fixedgsl_submit(const sage_fixedgsl_desc *d, sage_handle *job, sage_handle *end_ev) {
  SAGE_TRY(require_up());
  if (!d || !job || !end_ev) return fail(SAGE_EINVAL, "fixedgsl_submit: null argument");
  if (!gpu_get(d->gpu)) return fail(SAGE_ENODEV, "fixedgsl_submit: bad gpu");
  auto *J = new Job();
  J->d = *d;
  for (int i = 0; i < 16; ++i) J->info.t[i] = -1;
  J->info.status = SAGE_ENOTREADY;
  if (d->layout) {
    uint64_t packed = 0;
    int rc = layout_tensors(d->layout, &J->src_off, &J->dst_off, &J->len, &packed, &J->seg);
    if (rc != SAGE_OK) { delete J; return rc; }
    if (packed != d->ro_src_bytes) { delete J; return fail(SAGE_EINVAL, "fixedgsl: ro_src_bytes != layout packed"); }
  } else if (d->ro_src_bytes) {
    J->src_off = {0}; J->dst_off = {0}; J->len = {d->ro_src_bytes};
    J->seg = (d->ro_src_bytes + 15) & ~15ull;
  }
  SAGE_TRY(event_new_host(end_ev, &J->ev));
  uint64_t id = g_job_next++;
  {
    std::lock_guard<std::mutex> lk(g_job_mu);
    g_jobs[id] = J;
  }
  *job = make_handle(Kind::Job, id);
  std::thread(job_thread, J).detach();
  return SAGE_OK;
}

int sage_fixedgsl_info_get(sage_handle h, sage_fixedgsl_info *out) {
  if (handle_kind(h) != Kind::Job || !out) return fail(SAGE_EINVAL, "not a job handle");
  std::lock_guard<std::mutex> lk(g_job_mu);
  auto it = g_jobs.find(h & ((1ull << 56) - 1));
  if (it == g_jobs.end()) return fail(SAGE_ESTATE, "unknown job");
  if (!it->second->done.load(std::memory_order_acquire)) return SAGE_ENOTREADY;
  *out = it->second->info;
  return SAGE_OK;
}

int sage_fixedgsl_release(sage_handle h) {
  if (handle_kind(h) != Kind::Job) return fail(SAGE_EINVAL, "not a job handle");
  Job *J;
  {
    std::lock_guard<std::mutex> lk(g_job_mu);
    auto it = g_jobs.find(h & ((1ull << 56) - 1));
    if (it == g_jobs.end()) return fail(SAGE_ESTATE, "double or unknown job release");
    J = it->second;
    if (!J->done.load()) return fail(SAGE_ESTATE, "job still running");
    g_jobs.erase(it);
  }
  delete J;
  return SAGE_OK;
}

}  // extern "C"
