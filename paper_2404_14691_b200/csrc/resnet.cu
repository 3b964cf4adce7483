// resnet.cu — the ResNet-50 function body as a program of native kernels.
//
// The reference models resnet50's COMPUTE as a fixed 24.3 ms delay
// (functions.py:154, :276).  Here the body is a registered "network program"
// (sage_net_create): an ordered list of operations over the landed RO
// segment (filters, batch-norm parameters and the classifier, addressed by
// their offsets in the segment) and the invocation's writable segment (the
// request image, the logits and the activation workspace).  One invocation's
// COMPUTE runs the program on its stream:
//   S2D_INPUT   NHWC 3-channel image -> 2x2 space-to-depth, 16 channels (the
//               stem as a 4x4 stride-1 conv, SAGE_CONV_S2D); PAD_INPUT -> 4
//               channels for the older C4 stem
//   CONV        tcgen05 implicit GEMM (conv_tc.cu), BN / residual / ReLU fused
//   MAXPOOL     3x3 stride 2 pad 1 (the stem)
//   POOL_FC     global average pool + the 1000-way classifier, fp32 logits
// No PyTorch, no cuDNN: the BF16 ResNet-50 record runs on these kernels only.
//
// Launch: 57 kernels per forward would cost ~0.45 ms of host time on the
// issuing thread, so the program is captured once per (landed segment,
// context) as CUDA graphs whose kernels read their activation buffers from a
// device-side FRAME {input, logits, workspace}.  An invocation then costs two
// launches: a one-thread kernel writing its frame, and the graph.  Launches
// of one executable graph serialise, so up to SAGE_NET_INSTANCES graphs (each with
// its own frame) serve concurrent invocations; an instance is reused after
// its previous run's completion event (device-side wait).
// SAGE_NET_GRAPHS=0 launches the ops one by one with direct pointers.
#include "common.h"

#include <cuda_bf16.h>

#include <map>

namespace sage {

struct BufRef {        // a buffer: frame[sel] + off on the device, or `direct`
  int sel;
  uint64_t off, direct;
};
__device__ __forceinline__ uint64_t resolve(const uint64_t *frame, const BufRef &r) {
  return frame ? frame[r.sel] + r.off : r.direct;
}

// NHWC bf16 [P, 3] -> [P, 4] (zero fourth channel)
__global__ void pad_c4_kernel(const uint64_t *frame, BufRef src, BufRef dst, long long pix) {
  const __nv_bfloat16 *in = reinterpret_cast<const __nv_bfloat16 *>(resolve(frame, src));
  uint2 *out = reinterpret_cast<uint2 *>(resolve(frame, dst));
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < pix; i += (long long)gridDim.x * blockDim.x) {
    const __nv_bfloat16 *s = in + 3 * i;
    __nv_bfloat162 lo = __halves2bfloat162(s[0], s[1]);
    __nv_bfloat162 hi = __halves2bfloat162(s[2], __float2bfloat16(0.f));
    uint2 v;
    v.x = *reinterpret_cast<uint32_t *>(&lo);
    v.y = *reinterpret_cast<uint32_t *>(&hi);
    out[i] = v;
  }
}

// NHWC bf16 [N, H, W, 3] -> 2x2 space-to-depth [N, H/2, W/2, 16]: channel
// (dr * 2 + ds) * 4 + c of output pixel (i, j) is input (2i + dr, 2j + ds, c),
// c = 3 zero (the SAGE_CONV_S2D stem); one thread = one output pixel (32 B)
__global__ void s2d_kernel(const uint64_t *frame, BufRef src, BufRef dst, int N, int H, int W) {
  const __nv_bfloat16 *in = reinterpret_cast<const __nv_bfloat16 *>(resolve(frame, src));
  uint4 *out = reinterpret_cast<uint4 *>(resolve(frame, dst));
  const int H2 = H / 2, W2 = W / 2;
  const long long total = (long long)N * H2 * W2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i % W2);
    const long long t = i / W2;
    const int r = (int)(t % H2), n = (int)(t / H2);
    __nv_bfloat16 v[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int dr = q >> 1, ds = q & 1;
      const __nv_bfloat16 *p = in + ((size_t)(n * H + 2 * r + dr) * W + 2 * j + ds) * 3;
      v[4 * q] = p[0];
      v[4 * q + 1] = p[1];
      v[4 * q + 2] = p[2];
      v[4 * q + 3] = __float2bfloat16(0.f);
    }
    out[2 * i] = *reinterpret_cast<const uint4 *>(&v[0]);
    out[2 * i + 1] = *reinterpret_cast<const uint4 *>(&v[8]);
  }
}

// 3x3 stride-2 pad-1 max pool over NHWC bf16; one thread = 8 channels of one output pixel
__global__ void maxpool_kernel(const uint64_t *frame, BufRef src, BufRef dst, int N, int H, int W, int C, int P,
                               int Q) {
  const __nv_bfloat16 *in = reinterpret_cast<const __nv_bfloat16 *>(resolve(frame, src));
  __nv_bfloat16 *out = reinterpret_cast<__nv_bfloat16 *>(resolve(frame, dst));
  const int c8 = C / 8;
  const long long total = (long long)N * P * Q * c8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int cg = (int)(i % c8);
    long long t = i / c8;
    const int q = (int)(t % Q);
    t /= Q;
    const int p = (int)(t % P);
    const int n = (int)(t / P);
    // all nine window loads in flight at once; out-of-image taps read as
    // bf16 -inf (0xFF80), which never wins the max
    uint4 v[9];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int ih = 2 * p - 1 + r;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int iw = 2 * q - 1 + s;
        v[3 * r + s] = (ih >= 0 && ih < H && iw >= 0 && iw < W)
                           ? __ldg(reinterpret_cast<const uint4 *>(in + ((size_t)(n * H + ih) * W + iw) * C + cg * 8))
                           : make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
      }
    }
    float m[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) m[e] = -INFINITY;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v[k]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h[e]);
        m[2 * e] = fmaxf(m[2 * e], f.x);
        m[2 * e + 1] = fmaxf(m[2 * e + 1], f.y);
      }
    }
    uint4 o;
    __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(m[2 * e], m[2 * e + 1]);
    *reinterpret_cast<uint4 *>(out + ((size_t)(n * P + p) * Q + q) * C + cg * 8) = o;
  }
}

// global average pool: [N, HW, C] bf16 -> [N, C] fp32
// feat[n, c] = mean over HW of in[n, :, c]: a block per (sample, 256
// channels), each lane owns 8 channels (one 16-B vector per pixel) and the 8
// warps split the pixels; partial sums meet in shared memory
constexpr int kPoolWarps = 8;
__global__ void __launch_bounds__(256) avgpool_kernel(const uint64_t *frame, BufRef src, BufRef dst, int HW, int C) {
  const __nv_bfloat16 *in = reinterpret_cast<const __nv_bfloat16 *>(resolve(frame, src));
  float *feat = reinterpret_cast<float *>(resolve(frame, dst));
  __shared__ float part[kPoolWarps][256];
  const int n = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 256 + lane * 8;
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c < C) {
    const __nv_bfloat16 *p = in + (size_t)n * HW * C + c;
#pragma unroll 4
    for (int i = warp; i < HW; i += kPoolWarps) {
      const uint4 v = __ldg(reinterpret_cast<const uint4 *>(p + (size_t)i * C));
      const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(h[k]);
        s[2 * k] += f.x;
        s[2 * k + 1] += f.y;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) part[warp][lane * 8 + k] = s[k];
  __syncthreads();
  const int cc = blockIdx.x * 256 + threadIdx.x;
  if (cc < C) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < kPoolWarps; ++w) t += part[w][threadIdx.x];
    feat[(size_t)n * C + cc] = t / (float)HW;
  }
}

// logits[n, j] = feat[n] . W[j] + b[j]: kFcSplit warps per class j, each
// over a quarter of the channels (lane l: channels q*C/4 + 128 i + 4 l), for
// up to 8 samples at a time with their feature loads all in flight; the
// quarters meet in shared memory.  4000 short warps instead of 1000 long ones
// (one warp per class ran a 3.2k-instruction dependent chain: 22 us under ncu)
constexpr int kFcMaxC = 2048, kFcSplit = 4, kFcNB = 8;
__global__ void __launch_bounds__(256, 4) fc_kernel(const uint64_t *frame, BufRef src, BufRef dst,
                                                 const __nv_bfloat16 *__restrict__ w,
                                                 const __nv_bfloat16 *__restrict__ b, int N, int C, int J) {
  const float *feat = reinterpret_cast<const float *>(resolve(frame, src));
  float *out = reinterpret_cast<float *>(resolve(frame, dst));
  __shared__ float part[8][kFcNB];
  const int bw = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + bw, cls = gw / kFcSplit, q = gw % kFcSplit;
  const bool active = cls < J;
  constexpr int IT = kFcMaxC / kFcSplit / 128;
  const int span = C / kFcSplit, iters = span / 128;   // C % 512 == 0, C <= kFcMaxC (net_create)
  const size_t c0 = (size_t)q * span + lane * 4;
  uint2 wv[IT];
#pragma unroll
  for (int i = 0; i < IT; ++i)
    wv[i] = (active && i < iters) ? __ldg(reinterpret_cast<const uint2 *>(w + (size_t)cls * C + c0 + i * 128))
                                  : make_uint2(0u, 0u);
  for (int n0 = 0; n0 < N; n0 += kFcNB) {
    const int nb = min(kFcNB, N - n0);
    float s[kFcNB];
#pragma unroll
    for (int k = 0; k < kFcNB; ++k) s[k] = 0.f;
    if (active) {
#pragma unroll
      for (int i = 0; i < IT; ++i) {
        if (i < iters) {
          const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&wv[i]);
          const float2 w0 = __bfloat1622float2(h[0]), w1 = __bfloat1622float2(h[1]);
#pragma unroll
          for (int k = 0; k < kFcNB; ++k) {
            if (k < nb) {
              const float4 f = __ldg(reinterpret_cast<const float4 *>(feat + (size_t)(n0 + k) * C + c0 + i * 128));
              s[k] += w0.x * f.x + w0.y * f.y + w1.x * f.z + w1.y * f.w;
            }
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kFcNB; ++k)
#pragma unroll
      for (int o = 16; o; o >>= 1) s[k] += __shfl_xor_sync(0xffffffffu, s[k], o);
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < kFcNB; ++k) part[bw][k] = s[k];
    }
    __syncthreads();
    if (active && q == 0 && lane < nb) {
      float v = __bfloat162float(b[cls]);
#pragma unroll
      for (int k = 0; k < kFcSplit; ++k) v += part[bw + k][lane];
      out[(size_t)(n0 + lane) * J + cls] = v;
    }
    __syncthreads();
  }
}

// one invocation's frame: where its buffers are
__global__ void set_frame_kernel(uint64_t *frame, uint64_t input, uint64_t out, uint64_t ws) {
  if (threadIdx.x == 0) {
    frame[0] = input;
    frame[1] = out;
    frame[2] = ws;
  }
}

// concurrent runs of one program over one segment (SAGE_NET_INSTANCES, default 16)
static int instances() {
  static const int n = [] { const char *e = getenv("SAGE_NET_INSTANCES"); return e ? std::max(1, atoi(e)) : 16; }();
  return n;
}

struct GraphInst {
  cudaGraphExec_t exec = nullptr;
  uint64_t *frame = nullptr;      // device: {input, logits, workspace}
  cudaEvent_t done = nullptr;     // end of this instance's last run
  bool used = false;
};
struct GraphSet {                 // the instances of one (segment, context)
  std::vector<GraphInst> inst;
  uint64_t next = 0;
};

struct Net {
  std::vector<sage_net_op> ops;
  std::vector<uint64_t> buf_off;     // workspace offsets of buffers 2..
  uint64_t workspace = 0;
  std::mutex mu;
  std::map<std::pair<uint64_t, CUcontext>, GraphSet> graphs;
  cudaStream_t capture = nullptr;
};
static std::mutex g_net_mu;
static std::unordered_map<uint64_t, Net *> g_nets;
static uint64_t g_net_next = 1;
constexpr uint8_t kNetKind = 0x23;

static Net *net_get(uint64_t h) {
  if ((h >> 56) != kNetKind) return nullptr;
  std::lock_guard<std::mutex> lk(g_net_mu);
  auto it = g_nets.find(h & ((1ull << 56) - 1));
  return it == g_nets.end() ? nullptr : it->second;
}

static int grid_for(long long n, int sms) {
  return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, (long long)sms * 16));
}

// enqueue the program on s.  frame != null: buffers come from the device
// frame (graph capture); else from base[3] = {input, logits, workspace}.
static int enqueue_ops(Net *net, uint64_t ro, const uint64_t *frame, const uint64_t base[3], cudaStream_t s, int sms) {
  auto ref = [&](int id, BufRef *r) -> bool {
    if (id == SAGE_NET_BUF_INPUT) *r = {0, 0, base[0]};
    else if (id == SAGE_NET_BUF_OUT) *r = {1, 0, base[1]};
    else if (id >= SAGE_NET_BUF_WS0 && id - SAGE_NET_BUF_WS0 < (int)net->buf_off.size()) {
      const uint64_t off = net->buf_off[id - SAGE_NET_BUF_WS0];
      *r = {2, off, base[2] + off};
    } else {
      return false;
    }
    return true;
  };
  for (const sage_net_op &op : net->ops) {
    BufRef src, dst, res{};
    if (!ref(op.src, &src) || !ref(op.dst, &dst) || (op.res >= 0 && !ref(op.res, &res)))
      return fail(SAGE_EINVAL, "resnet body: op names an unknown buffer");
    switch (op.kind) {
      case SAGE_NET_PAD_INPUT: {
        const long long pix = (long long)op.n * op.h * op.w;
        pad_c4_kernel<<<grid_for(pix, sms), 256, 0, s>>>(frame, src, dst, pix);
        break;
      }
      case SAGE_NET_S2D_INPUT: {
        if ((op.h | op.w) & 1) return fail(SAGE_EINVAL, "resnet body: S2D_INPUT needs even height and width");
        const long long pix = (long long)op.n * (op.h / 2) * (op.w / 2);
        s2d_kernel<<<grid_for(pix, sms), 256, 0, s>>>(frame, src, dst, op.n, op.h, op.w);
        break;
      }
      case SAGE_NET_CONV: {
        sage_conv_desc d{};
        d.x = frame ? 16 : src.direct;        // direct pointers only validate alignment in frame mode
        d.out = frame ? 16 : dst.direct;
        d.residual = op.res >= 0 ? (frame ? 16 : res.direct) : 0;
        d.w = ro + op.w_off;
        if (op.g_off != UINT64_MAX) {
          d.bn_gamma = ro + op.g_off;
          d.bn_beta = ro + op.b_off;
          d.bn_mean = ro + op.m_off;
          d.bn_var = ro + op.v_off;
        }
        d.bn_eps = op.eps;
        d.n = op.n; d.h = op.h; d.w_ = op.w; d.cin = op.cin; d.cout = op.cout;
        d.r = op.r; d.s = op.s; d.stride = op.stride; d.pad = op.pad; d.relu = op.relu; d.mode = op.mode;
        if (frame) {
          ConvFrame f{frame, src.sel, op.res >= 0 ? res.sel : -1, dst.sel, src.off, res.off, dst.off};
          SAGE_TRY(conv_bf16(&d, s, sms, &f));
        } else {
          SAGE_TRY(conv_bf16(&d, s, sms, nullptr));
        }
        continue;
      }
      case SAGE_NET_MAXPOOL: {
        const int P = (op.h + 2 - 3) / 2 + 1, Q = (op.w + 2 - 3) / 2 + 1;
        maxpool_kernel<<<grid_for((long long)op.n * P * Q * op.cin / 8, sms), 256, 0, s>>>(frame, src, dst, op.n,
                                                                                          op.h, op.w, op.cin, P, Q);
        break;
      }
      case SAGE_NET_POOL_FC: {
        if (op.res < 0) return fail(SAGE_EINVAL, "resnet body: POOL_FC needs a feature buffer");
        avgpool_kernel<<<dim3((op.cin + 255) / 256, op.n), 256, 0, s>>>(frame, src, res, op.h * op.w, op.cin);
        fc_kernel<<<(op.cout * kFcSplit * 32 + 255) / 256, 256, 0, s>>>(frame, res, dst, (const __nv_bfloat16 *)(ro + op.w_off),
                                                              (const __nv_bfloat16 *)(ro + op.b_off), op.n, op.cin,
                                                              op.cout);
        break;
      }
      default:
        return fail(SAGE_EINVAL, "resnet body: unknown op kind");
    }
    SAGE_CUDA(cudaGetLastError());
  }
  return SAGE_OK;
}

static bool graphs_enabled() {
  static const bool on = [] { const char *e = getenv("SAGE_NET_GRAPHS"); return !(e && atoi(e) == 0); }();
  return on;
}

// capture one instance of the program over segment `ro` (net->mu held)
static int capture_instance(Net *net, uint64_t ro, int sms, GraphInst *gi) {
  SAGE_TRY(conv_optin_all());   // attributes are not settable while capturing
  SAGE_CUDA(cudaMalloc(&gi->frame, 4 * sizeof(uint64_t)));
  SAGE_CUDA(cudaEventCreateWithFlags(&gi->done, cudaEventDisableTiming));
  if (!net->capture) SAGE_CUDA(cudaStreamCreateWithFlags(&net->capture, cudaStreamNonBlocking));
  SAGE_CUDA(cudaStreamBeginCapture(net->capture, cudaStreamCaptureModeThreadLocal));
  const uint64_t none[3] = {0, 0, 0};
  int rc = enqueue_ops(net, ro, gi->frame, none, net->capture, sms);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(net->capture, &g);
  if (rc != SAGE_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture (resnet program)");
  e = cudaGraphInstantiate(&gi->exec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate (resnet program)");
  return SAGE_OK;
}

// run a registered network on stream s: ro = landed segment, input = request
// image, out = logits followed by the workspace (b->out_bytes covers logits)
int net_run(const sage_body_desc *b, cudaStream_t s, int sms) {
  Net *net = net_get((uint64_t)b->args[0]);
  if (!net) return fail(SAGE_EINVAL, "resnet body: unknown network handle");
  const uint64_t ws = (b->out + b->out_bytes + 255) & ~255ull;
  if (!graphs_enabled()) {
    const uint64_t base[3] = {b->input, b->out, ws};
    return enqueue_ops(net, b->ro, nullptr, base, s, sms);
  }
  CUcontext ctx = nullptr;
  drv.CtxGetCurrent(&ctx);
  std::lock_guard<std::mutex> lk(net->mu);
  GraphSet &set = net->graphs[{b->ro, ctx}];
  // an idle instance, else a new one (up to instances()), else round robin
  GraphInst *gi = nullptr;
  for (auto &x : set.inst)
    if (!x.used || cudaEventQuery(x.done) == cudaSuccess) {
      gi = &x;
      break;
    }
  if (!gi && (int)set.inst.size() < instances()) {
    set.inst.emplace_back();
    gi = &set.inst.back();
    int rc = capture_instance(net, b->ro, sms, gi);
    if (rc != SAGE_OK) {
      set.inst.pop_back();
      return rc;
    }
  }
  if (!gi) gi = &set.inst[set.next++ % set.inst.size()];
  if (gi->used) SAGE_CUDA(cudaStreamWaitEvent(s, gi->done, 0));   // its frame is free once its last run ended
  set_frame_kernel<<<1, 32, 0, s>>>(gi->frame, b->input, b->out, ws);
  SAGE_CUDA(cudaGetLastError());
  SAGE_CUDA(cudaGraphLaunch(gi->exec, s));
  SAGE_CUDA(cudaEventRecord(gi->done, s));
  gi->used = true;
  return SAGE_OK;
}

int touch_net_kernels() {
  cudaFuncAttributes a;
  SAGE_CUDA(cudaFuncGetAttributes(&a, pad_c4_kernel));
  SAGE_CUDA(cudaFuncGetAttributes(&a, s2d_kernel));
  SAGE_CUDA(cudaFuncGetAttributes(&a, maxpool_kernel));
  SAGE_CUDA(cudaFuncGetAttributes(&a, avgpool_kernel));
  SAGE_CUDA(cudaFuncGetAttributes(&a, fc_kernel));
  SAGE_CUDA(cudaFuncGetAttributes(&a, set_frame_kernel));
  return touch_conv_kernels();
}

static void net_drop_graphs(Net *N) {
  std::lock_guard<std::mutex> lk(N->mu);
  for (auto &kv : N->graphs)
    for (auto &gi : kv.second.inst) {
      if (gi.done) {
        cudaEventSynchronize(gi.done);
        cudaEventDestroy(gi.done);
      }
      if (gi.exec) cudaGraphExecDestroy(gi.exec);
      if (gi.frame) cudaFree(gi.frame);
    }
  N->graphs.clear();
  if (N->capture) cudaStreamDestroy(N->capture);
  N->capture = nullptr;
}

static void net_free(Net *N) {
  net_drop_graphs(N);
  delete N;
}

void nets_release_graphs() {
  std::lock_guard<std::mutex> lk(g_net_mu);
  for (auto &kv : g_nets) net_drop_graphs(kv.second);
}

}  // namespace sage

using namespace sage;

extern "C" int sage_net_create(const sage_net_op *ops, int n_ops, const uint64_t *buf_bytes, int n_bufs,
                               sage_handle *net, uint64_t *workspace_bytes) {
  if (!ops || n_ops <= 0 || n_bufs < 0 || (n_bufs && !buf_bytes) || !net)
    return fail(SAGE_EINVAL, "net_create: bad arguments");
  auto *N = new Net();
  N->ops.assign(ops, ops + n_ops);
  uint64_t off = 0;
  for (int i = 0; i < n_bufs; ++i) {
    N->buf_off.push_back(off);
    off += (buf_bytes[i] + 255) & ~255ull;
  }
  N->workspace = off;
  for (const sage_net_op &op : N->ops) {
    if (op.kind < SAGE_NET_PAD_INPUT || op.kind > SAGE_NET_S2D_INPUT) {
      delete N;
      return fail(SAGE_EINVAL, "net_create: unknown op kind");
    }
    if (op.kind == SAGE_NET_POOL_FC && (op.cin % 512 || op.cin > kFcMaxC || op.cin <= 0)) {
      delete N;
      return fail(SAGE_EINVAL, "net_create: POOL_FC needs a multiple of 512 features, at most 2048");
    }
  }
  std::lock_guard<std::mutex> lk(g_net_mu);
  const uint64_t id = g_net_next++;
  g_nets[id] = N;
  *net = ((uint64_t)kNetKind << 56) | id;
  if (workspace_bytes) *workspace_bytes = off;
  return SAGE_OK;
}

extern "C" int sage_net_destroy(sage_handle net) {
  Net *N;
  {
    std::lock_guard<std::mutex> lk(g_net_mu);
    auto it = g_nets.find(net & ((1ull << 56) - 1));
    if ((net >> 56) != kNetKind || it == g_nets.end()) return fail(SAGE_ESTATE, "net_destroy: unknown network");
    N = it->second;
    g_nets.erase(it);
  }
  net_free(N);
  return SAGE_OK;
}
