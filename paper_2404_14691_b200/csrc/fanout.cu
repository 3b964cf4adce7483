// fanout.cu — one landed segment to the other GPUs of the box over NVLink.
//
// The reference has no GPU-to-GPU path: every GPU pulls its own copy through
// the one shared host channel (simulation.py:113-115), which is the loading
// contention SAGE removes.  Here a segment crosses PCIe once (the home GPU's
// land) and then goes GPU to GPU:
//   multicast  an NVSwitch multicast object (cuMulticastCreate) binds every
//              destination's physical pages; one kernel on the home GPU reads
//              the home copy and stores it through the multicast address with
//              multimem.st -- the switch replicates each store to all bound
//              GPUs (one pass over the source, NVLS)
//   p2p        fallback when multicast objects cannot be made (no fabric
//              manager / NVSwitch team, a single device, or a plane sharing
//              its device): one copy-engine peer copy per destination
// sage_fanout_caps reports what the box supports and why not, so callers and
// the bench line say which path ran.
#include "common.h"

#include <algorithm>

namespace sage {

__global__ void mc_broadcast_kernel(uint4 *mc, const uint4 *__restrict__ src, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = src[i];
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
  }
}

struct McDriver {
  PFN_cuMulticastCreate_v12010 Create = nullptr;
  PFN_cuMulticastAddDevice_v12010 AddDevice = nullptr;
  PFN_cuMulticastBindMem_v12010 BindMem = nullptr;
  PFN_cuMulticastUnbind_v12010 Unbind = nullptr;
  PFN_cuMulticastGetGranularity_v12010 Granularity = nullptr;
  PFN_cuDeviceGetAttribute_v2000 DevAttr = nullptr;
  bool loaded = false;
};
static McDriver mcd;

template <class F>
static bool mc_entry(const char *name, F *fn) {
  cudaDriverEntryPointQueryResult q;
  void *p = nullptr;
  if (cudaGetDriverEntryPointByVersion(name, &p, 12010, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}

static bool mc_load() {
  if (mcd.loaded) return mcd.Create != nullptr;
  mcd.loaded = true;
  bool ok = mc_entry("cuMulticastCreate", &mcd.Create) && mc_entry("cuMulticastAddDevice", &mcd.AddDevice) &&
            mc_entry("cuMulticastBindMem", &mcd.BindMem) && mc_entry("cuMulticastUnbind", &mcd.Unbind) &&
            mc_entry("cuMulticastGetGranularity", &mcd.Granularity) &&
            mc_entry("cuDeviceGetAttribute", &mcd.DevAttr);
  if (!ok) mcd.Create = nullptr;
  return ok;
}

// try to make a multicast object over `devs` (distinct physical devices);
// on success *out holds it (the caller binds, maps and releases)
static CUresult mc_make(const std::vector<int> &devs, uint64_t bytes, CUmemGenericAllocationHandle *out,
                        size_t *gran) {
  CUmulticastObjectProp prop{};
  prop.numDevices = (unsigned)devs.size();
  prop.size = bytes;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
  size_t g = 0;
  CUresult r = mcd.Granularity(&g, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS) return r;
  prop.size = (bytes + g - 1) / g * g;
  r = mcd.Create(out, &prop);
  if (r != CUDA_SUCCESS) return r;
  for (int d : devs)
    if ((r = mcd.AddDevice(*out, (CUdevice)d)) != CUDA_SUCCESS) {
      drv.MemRelease(*out);
      return r;
    }
  *gran = g;
  return CUDA_SUCCESS;
}

}  // namespace sage

using namespace sage;

extern "C" int sage_fanout_caps(sage_fanout_caps_t *out) {
  SAGE_TRY(require_up());
  if (!out) return fail(SAGE_EINVAL, "fanout_caps: null out");
  memset(out, 0, sizeof *out);
  out->n_gpus = st.n_gpus;
  std::vector<int> devs;
  for (int g = 0; g < st.n_gpus && g < 32; ++g) {
    const int d = dev_of(g);
    if (std::find(devs.begin(), devs.end(), d) == devs.end()) devs.push_back(d);
    for (int h = 0; h < st.n_gpus && h < 32; ++h) {
      const int e = dev_of(h);
      int can = d == e;   // planes sharing a device reach each other's pages directly
      if (d != e) cudaDeviceCanAccessPeer(&can, d, e);
      if (can) out->peer_mask[g] |= 1u << h;
    }
  }
  out->n_devices = (int)devs.size();
  if (!mc_load()) {
    snprintf(out->why, sizeof out->why, "multicast driver entry points unavailable");
    return SAGE_OK;
  }
  int sup = 1;
  for (int d : devs) {
    int v = 0;
    mcd.DevAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)d);
    sup &= v != 0;
  }
  out->multicast_attr = sup;
  if (!sup) {
    snprintf(out->why, sizeof out->why, "a device reports CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 0");
    return SAGE_OK;
  }
  if ((int)devs.size() < 2 || (int)devs.size() != st.n_gpus) {
    snprintf(out->why, sizeof out->why, "multicast needs one plane per distinct device (%d planes, %d devices)",
             st.n_gpus, (int)devs.size());
    return SAGE_OK;
  }
  CUmemGenericAllocationHandle h = 0;
  size_t gran = 0;
  CUresult r = mc_make(devs, 2ull << 20, &h, &gran);
  if (r != CUDA_SUCCESS) {
    snprintf(out->why, sizeof out->why,
             "cuMulticastCreate/AddDevice: CUresult %d (no NVSwitch team or fabric manager visible)", (int)r);
    return SAGE_OK;
  }
  drv.MemRelease(h);
  out->multicast = 1;
  out->multicast_granularity = gran;
  snprintf(out->why, sizeof out->why, "ok");
  return SAGE_OK;
}

// the segment at src (src_gpu) into every destination allocation: multicast
// when possible (and not refused by flags), else peer copies; *end_ev
// completes when every copy has landed
extern "C" int sage_fanout_broadcast(sage_bcast_desc *d, const sage_handle *wait, int n_wait, sage_handle *end_ev) {
  SAGE_TRY(require_up());
  if (!d || !end_ev || d->n_dst < 1 || d->n_dst > 32 || !d->bytes || (d->bytes & 15) || (d->src_dptr & 15))
    return fail(SAGE_EINVAL, "fanout_broadcast: bad descriptor (1..32 destinations, 16-B aligned bytes)");
  Gpu *S = gpu_get(d->src_gpu);
  if (!S) return fail(SAGE_ENODEV, "fanout_broadcast: bad source gpu");
  std::vector<uint64_t> dptr(d->n_dst), phys(d->n_dst);
  std::vector<CUmemGenericAllocationHandle> ph(d->n_dst);
  std::vector<int> devs;
  for (int i = 0; i < d->n_dst; ++i) {
    int g = -1;
    SAGE_TRY(pool_alloc_phys(d->dst_alloc[i], &ph[i], &phys[i], &dptr[i], &g));
    if (g != d->dst_gpu[i]) return fail(SAGE_EINVAL, "fanout_broadcast: allocation is not on its destination gpu");
    if (phys[i] < d->bytes) return fail(SAGE_EINVAL, "fanout_broadcast: destination smaller than the segment");
    const int dv = dev_of(g);
    if (std::find(devs.begin(), devs.end(), dv) == devs.end()) devs.push_back(dv);
  }
  cudaSetDevice(S->dev);
  cudaStream_t s = S->aux;
  SAGE_TRY(wait_events(s, wait, n_wait));
  Event *E;
  SAGE_TRY(event_new(d->src_gpu, end_ev, &E));
  d->path = SAGE_BCAST_PATH_P2P;
  bool mc_ok = !(d->flags & SAGE_BCAST_P2P_ONLY) && mc_load() && (int)devs.size() == d->n_dst && d->n_dst >= 1 &&
               std::find(devs.begin(), devs.end(), S->dev) != devs.end();
  if (mc_ok) {
    // every destination on its own device and the home among them: bind
    // their pages to one multicast object and write them all in one pass
    CUmemGenericAllocationHandle mc = 0;
    size_t gran = 0;
    const uint64_t size = *std::min_element(phys.begin(), phys.end());
    CUresult r = mc_make(devs, size, &mc, &gran);
    const uint64_t span = size / gran * gran;
    if (r == CUDA_SUCCESS && span >= d->bytes) {
      int bound = 0;
      for (; bound < d->n_dst && r == CUDA_SUCCESS; ++bound) r = mcd.BindMem(mc, 0, ph[bound], 0, span, 0);
      CUdeviceptr va = 0;
      if (r == CUDA_SUCCESS) r = drv.MemAddressReserve(&va, span, gran, 0, 0);
      if (r == CUDA_SUCCESS) r = drv.MemMap(va, span, 0, mc, 0);
      if (r == CUDA_SUCCESS) {
        CUmemAccessDesc a{};
        a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        a.location.id = S->dev;
        a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        r = drv.MemSetAccess(va, span, &a, 1);
      }
      if (r == CUDA_SUCCESS) {
        const uint64_t n = d->bytes / 16;
        const int blocks = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)S->sm_count * 4);
        mc_broadcast_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<uint4 *>(va),
                                                   reinterpret_cast<const uint4 *>(d->src_dptr), n);
        if (cudaGetLastError() == cudaSuccess) {
          SAGE_TRY(event_record(E, s));
          cudaStreamSynchronize(s);   // the mapping dies with this call
          d->path = SAGE_BCAST_PATH_MULTICAST;
        }
      }
      if (va) {
        drv.MemUnmap(va, span);
        drv.MemAddressFree(va, span);
      }
      for (int i = 0; i < d->n_dst; ++i) mcd.Unbind(mc, (CUdevice)dev_of(d->dst_gpu[i]), 0, span);
    }
    if (mc) drv.MemRelease(mc);
    if (d->path == SAGE_BCAST_PATH_MULTICAST) return SAGE_OK;
  }
  // p2p fallback: one copy-engine peer copy per destination
  for (int i = 0; i < d->n_dst; ++i) {
    const int dv = dev_of(d->dst_gpu[i]);
    if (dv == S->dev)
      SAGE_CUDA(cudaMemcpyAsync((void *)dptr[i], (const void *)d->src_dptr, d->bytes, cudaMemcpyDeviceToDevice, s));
    else
      SAGE_CUDA(cudaMemcpyPeerAsync((void *)dptr[i], dv, (const void *)d->src_dptr, S->dev, d->bytes, s));
  }
  return event_record(E, s);
}
