// fixedgsl.cu — instance-per-invocation baselines on real hardware: FixedGSL
// (a fresh context per invocation) and DGSF (a pool of pre-created contexts).
//
// Reference: InstancePolicy (policies.py:102-126) admits one size-fixed
// instance per invocation and runs the SERIAL plan (functions.py:261-267):
// CPU ctx -> CPU load -> GPU ctx -> GPU load -> compute -> return, each stage
// after the previous; PoolPolicy (DGSF, policies.py:129-276) runs the same
// chain without GPU_CTX in one of N contexts pre-created per (function, GPU).
// Every stage here is the real operation of a container-per-function
// deployment:
//   CPU_CTX   thread mode: host-side instance state; process mode: the
//             instance's own OS process starting (posix_spawn .. main)
//   CPU_LOAD  malloc + memcpy of the DB record into the instance's private
//             (pageable) host memory
//   GPU_CTX   cuCtxCreate of a fresh context + module load of this body's
//             kernels only (process mode: + driver initialisation)
//   GPU_LOAD  cudaMalloc of the instance reservation + one synchronous
//             pageable cudaMemcpy per tensor + the input
//   COMPUTE   the body kernel, synchronised
//   RETURN    synchronous D2H of the result
// then the context is destroyed (timed separately as teardown).
//
// Modes (sage_fixedgsl_desc.mode):
//   SAGE_INSTANCE_THREAD   the instance runs on a library worker thread of
//                          this process (many instances share one driver
//                          instance and its locks)
//   SAGE_INSTANCE_PROCESS  one OS process per instance (sage_instance_worker,
//                          next to libsagedp.so): the DB record, the input and
//                          the result travel through a memfd the instance maps
//   SAGE_INSTANCE_POOLED   DGSF: the job runs in a context made at
//                          registration by sage_instance_ctx_create; no
//                          GPU_CTX stage, no teardown
#include "common.h"
#include "checksum.cuh"

#include <dlfcn.h>
#include <spawn.h>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>

extern char **environ;

namespace sage {

enum { ST_CPU_CTX = 1, ST_CPU_LOAD = 2, ST_GPU_CTX = 3, ST_GPU_LOAD = 4, ST_COMPUTE = 6, ST_RET = 7 };

// what one instance needs, wherever it runs; times are absolute monotonic µs
struct InstanceWork {
  int dev = 0;
  const uint8_t *db = nullptr;
  uint64_t db_bytes = 0;
  const uint8_t *input = nullptr;
  uint64_t input_bytes = 0;
  uint64_t alloc_bytes = 0, seg = 0;
  const uint64_t *src_off = nullptr, *dst_off = nullptr, *len = nullptr;
  uint32_t n = 0;
  sage_body_desc body{};
  uint8_t *result = nullptr;
  uint64_t result_bytes = 0;
  CUcontext pooled = nullptr;     // DGSF: run here, keep it
  bool init_driver = false;       // a fresh process: driver initialisation is part of GPU_CTX
  int64_t *t = nullptr;           // [16] stage stamps (absolute µs)
  uint64_t checksum = 0;
  int64_t teardown_us = 0;
};

// the serial chain from CPU_LOAD on (CPU_CTX is stamped by the caller)
static int run_instance(InstanceWork &W) {
  auto stamp = [&](int st, bool end) { W.t[2 * st + (end ? 1 : 0)] = mono_us(); };
  stamp(ST_CPU_LOAD, false);
  uint8_t *priv = (uint8_t *)malloc(W.db_bytes ? W.db_bytes : 1);
  if (!priv) return fail(SAGE_ENOMEM, "instance: host malloc");
  if (W.db_bytes) memcpy(priv, W.db, W.db_bytes);
  stamp(ST_CPU_LOAD, true);
  CUcontext ctx = W.pooled, prev = nullptr;
  int rc = SAGE_OK;
  if (!ctx) stamp(ST_GPU_CTX, false);
  if (W.init_driver) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= W.dev) {
      free(priv);
      return fail(SAGE_ENODEV, "instance: no CUDA device");
    }
    if ((rc = load_driver()) != SAGE_OK) { free(priv); return rc; }
  }
  drv.CtxGetCurrent(&prev);
  if (!ctx) {
    CUresult r = drv.CtxCreate(&ctx, 0, (CUdevice)W.dev);
    if (r != CUDA_SUCCESS) { free(priv); return cu_fail(r, "cuCtxCreate"); }
    drv.CtxSetCurrent(ctx);
    rc = touch_body_kernels(W.body.body);
    stamp(ST_GPU_CTX, true);
  } else {
    drv.CtxSetCurrent(ctx);
  }
  uint8_t *dmem = nullptr;
  if (rc == SAGE_OK) {
    stamp(ST_GPU_LOAD, false);
    const uint64_t ro_b = W.seg, in_b = (W.input_bytes + 255) & ~255ull, out_b = (W.body.out_bytes + 255) & ~255ull;
    const uint64_t need = ((ro_b + 255) & ~255ull) + in_b + out_b;
    cudaError_t e = cudaMalloc(&dmem, std::max<uint64_t>(W.alloc_bytes, need));
    if (e != cudaSuccess) rc = cuda_fail(e, "instance cudaMalloc");
    uint8_t *ro = dmem, *in = dmem + ((ro_b + 255) & ~255ull), *out = in + in_b;
    if (rc == SAGE_OK && ro_b && (e = cudaMemset(ro, 0, ro_b)) != cudaSuccess) rc = cuda_fail(e, "instance memset");
    for (uint32_t i = 0; rc == SAGE_OK && i < W.n; ++i)
      if (W.len[i] && (e = cudaMemcpy(ro + W.dst_off[i], priv + W.src_off[i], W.len[i], cudaMemcpyHostToDevice)) !=
                          cudaSuccess)
        rc = cuda_fail(e, "instance cudaMemcpy");
    if (rc == SAGE_OK && in_b && (e = cudaMemset(in, 0, in_b)) != cudaSuccess) rc = cuda_fail(e, "instance memset");
    if (rc == SAGE_OK && W.input_bytes &&
        (e = cudaMemcpy(in, W.input, W.input_bytes, cudaMemcpyHostToDevice)) != cudaSuccess)
      rc = cuda_fail(e, "instance input cudaMemcpy");
    stamp(ST_GPU_LOAD, true);
    if (rc == SAGE_OK) {
      stamp(ST_COMPUTE, false);
      sage_body_desc b = W.body;
      b.ro = (uint64_t)ro; b.ro_bytes = ro_b;
      b.input = (uint64_t)in; b.input_bytes = (W.input_bytes + 15) & ~15ull;
      b.out = (uint64_t)out;
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, W.dev);
      rc = launch_body(&b, 0, sms);
      if (rc == SAGE_OK && (e = cudaDeviceSynchronize()) != cudaSuccess) rc = cuda_fail(e, "instance compute");
      stamp(ST_COMPUTE, true);
    }
    if (rc == SAGE_OK) {
      stamp(ST_RET, false);
      if (W.result_bytes && (e = cudaMemcpy(W.result, out, W.result_bytes, cudaMemcpyDeviceToHost)) != cudaSuccess)
        rc = cuda_fail(e, "instance return");
      stamp(ST_RET, true);
    }
    // verification only, outside every stage: checksum of what was loaded
    if (rc == SAGE_OK && ro_b) {
      std::vector<uint8_t> host(ro_b);
      if (cudaMemcpy(host.data(), ro, ro_b, cudaMemcpyDeviceToHost) == cudaSuccess)
        W.checksum = host_checksum(host.data(), ro_b);
    }
  }
  const int64_t t0 = mono_us();
  if (dmem) cudaFree(dmem);
  if (!W.pooled) {
    drv.CtxSetCurrent(nullptr);
    drv.CtxDestroy(ctx);
  }
  drv.CtxSetCurrent(prev);
  W.teardown_us = mono_us() - t0;
  free(priv);
  return rc;
}

// ------------------------------------------------------------ process mode ---
// The shared region an instance process maps (memfd): header, tensor table,
// DB record, input, result.
struct InstShm {
  uint64_t magic;
  int32_t dev, status;
  uint32_t n, pad_;
  uint64_t db_bytes, input_bytes, alloc_bytes, seg, result_bytes;
  sage_body_desc body;
  uint64_t off_tab, off_db, off_input, off_result, total;
  int64_t t[16];
  uint64_t checksum;
  int64_t teardown_us;
  char err[256];
};
static const uint64_t kShmMagic = 0x5341474549535431ull;   // "SAGEIST1"

static std::string worker_path() {
  Dl_info info{};
  if (!dladdr((void *)&worker_path, &info) || !info.dli_fname) return "";
  std::string p(info.dli_fname);
  const size_t slash = p.rfind('/');
  return (slash == std::string::npos ? std::string(".") : p.substr(0, slash)) + "/sage_instance_worker";
}

// ------------------------------------------------------------------- jobs ---
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
static std::condition_variable &g_sem_cv = *new std::condition_variable;   // never destroyed (exit with jobs parked)
static int g_running = 0;
static const int kMaxConcurrent = 32;

extern int layout_tensors(sage_handle h, std::vector<uint64_t> *src, std::vector<uint64_t> *dst,
                          std::vector<uint64_t> *len, uint64_t *packed, uint64_t *seg);

struct InstCtx {
  int gpu = -1;
  CUcontext ctx = nullptr;
  std::atomic<bool> busy{false};
};
static std::mutex g_ictx_mu;
static std::unordered_map<uint64_t, InstCtx *> g_ictx;
static uint64_t g_ictx_next = 1;
constexpr uint8_t kCtxKind = 0x22;

static InstCtx *ictx_get(sage_handle h) {
  if ((h >> 56) != kCtxKind) return nullptr;
  std::lock_guard<std::mutex> lk(g_ictx_mu);
  auto it = g_ictx.find(h & ((1ull << 56) - 1));
  return it == g_ictx.end() ? nullptr : it->second;
}

static void fill_work(Job *J, InstanceWork &W, int64_t *t) {
  const sage_fixedgsl_desc &d = J->d;
  W.dev = dev_of(d.gpu);
  W.db = (const uint8_t *)d.ro_src;
  W.db_bytes = d.ro_src_bytes;
  W.input = (const uint8_t *)d.input;
  W.input_bytes = d.input_bytes;
  W.alloc_bytes = d.alloc_bytes;
  W.seg = J->seg;
  W.src_off = J->src_off.data();
  W.dst_off = J->dst_off.data();
  W.len = J->len.data();
  W.n = (uint32_t)J->len.size();
  W.body = d.body;
  W.result = (uint8_t *)d.result;
  W.result_bytes = d.result_bytes;
  W.t = t;
}

static int run_in_process(Job *J, int64_t *t) {
  const sage_fixedgsl_desc &d = J->d;
  const std::string exe = worker_path();
  if (exe.empty() || access(exe.c_str(), X_OK) != 0)
    return fail(SAGE_ESTATE, "process-per-instance: sage_instance_worker is not built next to libsagedp.so");
  const uint32_t n = (uint32_t)J->len.size();
  auto a64 = [](uint64_t v) { return (v + 63) & ~63ull; };
  const uint64_t off_tab = a64(sizeof(InstShm)), off_db = a64(off_tab + 24ull * n), off_in = a64(off_db + d.ro_src_bytes),
                 off_res = a64(off_in + d.input_bytes), total = a64(off_res + d.result_bytes);
  const int fd = memfd_create("sage-instance", 0);
  if (fd < 0) return fail(SAGE_ESTATE, "memfd_create failed");
  if (ftruncate(fd, (off_t)total) != 0) { close(fd); return fail(SAGE_ENOMEM, "instance region: ftruncate"); }
  void *map = mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  if (map == MAP_FAILED) { close(fd); return fail(SAGE_ENOMEM, "instance region: mmap"); }
  auto *H = (InstShm *)map;
  memset(H, 0, sizeof *H);
  H->magic = kShmMagic;
  H->dev = dev_of(d.gpu);
  H->n = n;
  H->db_bytes = d.ro_src_bytes;
  H->input_bytes = d.input_bytes;
  H->alloc_bytes = d.alloc_bytes;
  H->seg = J->seg;
  H->result_bytes = d.result_bytes;
  H->body = d.body;
  H->off_tab = off_tab; H->off_db = off_db; H->off_input = off_in; H->off_result = off_res; H->total = total;
  H->status = SAGE_ENOTREADY;
  for (int i = 0; i < 16; ++i) H->t[i] = -1;
  uint64_t *tab = (uint64_t *)((uint8_t *)map + off_tab);
  for (uint32_t i = 0; i < n; ++i) {
    tab[3 * i] = J->src_off[i];
    tab[3 * i + 1] = J->dst_off[i];
    tab[3 * i + 2] = J->len[i];
  }
  // the DB and the request are in place before the instance exists
  if (d.ro_src_bytes) memcpy((uint8_t *)map + off_db, d.ro_src, d.ro_src_bytes);
  if (d.input_bytes) memcpy((uint8_t *)map + off_in, d.input, d.input_bytes);
  char fdarg[32];
  snprintf(fdarg, sizeof fdarg, "%d", fd);
  char *argv[] = {const_cast<char *>(exe.c_str()), fdarg, nullptr};
  pid_t pid = 0;
  t[2 * ST_CPU_CTX] = mono_us();   // the instance process starts: its CPU context
  int rc = posix_spawn(&pid, exe.c_str(), nullptr, nullptr, argv, environ);
  if (rc != 0) {
    munmap(map, total);
    close(fd);
    return fail(SAGE_ESTATE, "posix_spawn of sage_instance_worker failed");
  }
  int wst = 0;
  while (waitpid(pid, &wst, 0) < 0 && errno == EINTR) {
  }
  int status = H->status;
  if (!WIFEXITED(wst) && status == SAGE_ENOTREADY) status = fail(SAGE_ESTATE, "instance process died");
  else if (status != SAGE_OK) status = fail(status, std::string("instance process: ") + H->err);
  for (int i = 2 * ST_CPU_LOAD; i < 16; ++i) t[i] = H->t[i];
  t[2 * ST_CPU_CTX + 1] = H->t[2 * ST_CPU_CTX + 1];
  J->info.checksum = H->checksum;
  J->info.teardown_us = H->teardown_us;
  if (status == SAGE_OK && d.result_bytes) memcpy(d.result, (uint8_t *)map + off_res, d.result_bytes);
  munmap(map, total);
  close(fd);
  return status;
}

static int run_job(Job *J) {
  const sage_fixedgsl_desc &d = J->d;
  int64_t t[16];
  for (int i = 0; i < 16; ++i) t[i] = -1;
  int rc;
  if (d.mode == SAGE_INSTANCE_PROCESS) {
    rc = run_in_process(J, t);
  } else {
    InstanceWork W;
    fill_work(J, W, t);
    t[2 * ST_CPU_CTX] = mono_us();
    t[2 * ST_CPU_CTX + 1] = mono_us();   // in-process: the instance state is a host struct
    InstCtx *C = nullptr;
    if (d.mode == SAGE_INSTANCE_POOLED) {
      C = ictx_get(d.ctx);
      if (!C) return fail(SAGE_ESTATE, "pooled instance: unknown context");
      if (C->busy.exchange(true)) return fail(SAGE_ESTATE, "pooled instance: context already in use");
      W.pooled = C->ctx;
    }
    rc = run_instance(W);
    if (C) C->busy.store(false);
    J->info.checksum = W.checksum;
    J->info.teardown_us = W.teardown_us;
  }
  const int64_t epoch = host_epoch_us();
  for (int i = 0; i < 16; ++i) J->info.t[i] = t[i] >= 0 ? t[i] - epoch : -1;
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
  if (d->mode < SAGE_INSTANCE_THREAD || d->mode > SAGE_INSTANCE_POOLED)
    return fail(SAGE_EINVAL, "fixedgsl_submit: unknown instance mode");
  if (d->mode == SAGE_INSTANCE_POOLED && !ictx_get(d->ctx))
    return fail(SAGE_EINVAL, "fixedgsl_submit: pooled mode needs a context from sage_instance_ctx_create");
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

// DGSF: a real CUDA context made now (registration time) with the body's
// kernels loaded into it; jobs submitted in SAGE_INSTANCE_POOLED mode run in it
int sage_instance_ctx_create(int gpu, int body, sage_handle *h) {
  SAGE_TRY(require_up());
  if (!h) return fail(SAGE_EINVAL, "instance_ctx_create: null out");
  if (!gpu_get(gpu)) return fail(SAGE_ENODEV, "instance_ctx_create: bad gpu");
  CUcontext prev = nullptr, ctx = nullptr;
  drv.CtxGetCurrent(&prev);
  CUresult r = drv.CtxCreate(&ctx, 0, (CUdevice)dev_of(gpu));
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuCtxCreate (pre-created context)");
  drv.CtxSetCurrent(ctx);
  int rc = touch_body_kernels(body);
  drv.CtxSetCurrent(prev);
  if (rc != SAGE_OK) {
    drv.CtxDestroy(ctx);
    return rc;
  }
  auto *C = new InstCtx();
  C->gpu = gpu;
  C->ctx = ctx;
  std::lock_guard<std::mutex> lk(g_ictx_mu);
  const uint64_t id = g_ictx_next++;
  g_ictx[id] = C;
  *h = ((uint64_t)kCtxKind << 56) | id;
  return SAGE_OK;
}

int sage_instance_ctx_destroy(sage_handle h) {
  InstCtx *C;
  {
    std::lock_guard<std::mutex> lk(g_ictx_mu);
    auto it = g_ictx.find(h & ((1ull << 56) - 1));
    if ((h >> 56) != kCtxKind || it == g_ictx.end()) return fail(SAGE_ESTATE, "instance_ctx_destroy: unknown context");
    C = it->second;
    if (C->busy.load()) return fail(SAGE_ESTATE, "instance_ctx_destroy: context in use");
    g_ictx.erase(it);
  }
  CUcontext prev = nullptr;
  drv.CtxGetCurrent(&prev);
  drv.CtxDestroy(C->ctx);
  if (prev != C->ctx) drv.CtxSetCurrent(prev);
  delete C;
  return SAGE_OK;
}

// the body of one instance process (sage_instance_worker): map the region,
// run the serial chain, write stamps / checksum / status back, exit
int sage_instance_child(int fd) {
  InstShm probe{};
  if (pread(fd, &probe, sizeof probe, 0) != (ssize_t)sizeof probe || probe.magic != kShmMagic) return 2;
  void *map = mmap(nullptr, probe.total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  if (map == MAP_FAILED) return 3;
  auto *H = (InstShm *)map;
  H->t[2 * ST_CPU_CTX + 1] = mono_us();   // the instance process is up
  int rc = SAGE_OK;
  {
    const uint64_t *tab = (const uint64_t *)((uint8_t *)map + H->off_tab);
    std::vector<uint64_t> src(H->n), dst(H->n), len(H->n);
    for (uint32_t i = 0; i < H->n; ++i) {
      src[i] = tab[3 * i];
      dst[i] = tab[3 * i + 1];
      len[i] = tab[3 * i + 2];
    }
    InstanceWork W;
    W.dev = H->dev;
    W.db = (const uint8_t *)map + H->off_db;
    W.db_bytes = H->db_bytes;
    W.input = (const uint8_t *)map + H->off_input;
    W.input_bytes = H->input_bytes;
    W.alloc_bytes = H->alloc_bytes;
    W.seg = H->seg;
    W.src_off = src.data();
    W.dst_off = dst.data();
    W.len = len.data();
    W.n = H->n;
    W.body = H->body;
    W.result = (uint8_t *)map + H->off_result;
    W.result_bytes = H->result_bytes;
    W.t = H->t;
    W.init_driver = true;
    rc = run_instance(W);
    H->checksum = W.checksum;
    H->teardown_us = W.teardown_us;
  }
  if (rc != SAGE_OK) snprintf(H->err, sizeof H->err, "%s", sage_last_error());
  H->status = rc;
  munmap(map, probe.total);
  return rc == SAGE_OK ? 0 : 1;
}

}  // extern "C"
