// sgemm_host_cost.cu — host cost of one sgemm_tc launch and of its parts
// (tensor-map encode, smem opt-in, cluster launch).  Probe, not product code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include
//      tools/sgemm_host_cost.cu -o /tmp/sgemm_host_cost -lcuda
#include "../paper_2404_14691_b200/csrc/common.h"
#include <chrono>
#include <cstdio>
namespace sage {
int fail(int code, const std::string &msg) { fprintf(stderr, "fail %d %s\n", code, msg.c_str()); return code; }
int cuda_fail(cudaError_t e, const char *what) { fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e)); return -3; }
int cu_fail(CUresult r, const char *what) { fprintf(stderr, "%s: %d\n", what, (int)r); return -3; }
}  // namespace sage
#include "../paper_2404_14691_b200/csrc/gemm_tc.cu"

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
int main() {
  const int M = 4096, N = 256, K = 4096, R = 200;
  float *A, *B, *C;
  cudaMalloc(&A, (size_t)M * K * 4);
  cudaMalloc(&B, (size_t)N * K * 4);
  cudaMalloc(&C, (size_t)M * N * 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int i = 0; i < 5; ++i) sage::sgemm_tc(A, B, C, M, N, K, s);
  cudaDeviceSynchronize();
  double t0 = now_us();
  for (int i = 0; i < R; ++i) sage::sgemm_tc(A, B, C, M, N, K, s);
  double t1 = now_us();
  cudaDeviceSynchronize();
  double t2 = now_us();
  printf("sgemm_tc host call      %8.2f us  (device drain %8.2f us per launch)\n", (t1 - t0) / R, (t2 - t0) / R);
  CUtensorMap ma;
  t0 = now_us();
  for (int i = 0; i < R; ++i) sage::encode_kmajor(&ma, A, M, K, 128);
  printf("encode_kmajor           %8.2f us\n", (now_us() - t0) / R);
  int dev;
  t0 = now_us();
  for (int i = 0; i < R; ++i) cudaGetDevice(&dev);
  printf("cudaGetDevice           %8.2f us\n", (now_us() - t0) / R);
  t0 = now_us();
  for (int i = 0; i < R; ++i)
    cudaFuncSetAttribute(sage::sgemm_tf32_kernel<256, false, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         sage::TcSmem<256, 1>::TOTAL);
  printf("cudaFuncSetAttribute    %8.2f us\n", (now_us() - t0) / R);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
