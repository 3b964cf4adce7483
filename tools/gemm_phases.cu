// gemm_phases.cu — where does a tcgen05 sgemm CTA spend its time?  Builds
// gemm_tc.cu with SAGE_GEMM_TRACE (globaltimer marks per CTA) and runs the
// cfg-2 shape (probe, not product code).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DSAGE_GEMM_TRACE
//      tools/gemm_phases.cu -o /tmp/gemm_phases -lcuda
#include "../paper_2404_14691_b200/csrc/common.h"
#include <algorithm>
#include <cstdio>
#include <vector>
namespace sage {
int fail(int code, const std::string &msg) { fprintf(stderr, "fail %d %s\n", code, msg.c_str()); return code; }
int cuda_fail(cudaError_t e, const char *what) { fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e)); return -3; }
int cu_fail(CUresult r, const char *what) { fprintf(stderr, "%s: %d\n", what, (int)r); return -3; }
}  // namespace sage
#include "../paper_2404_14691_b200/csrc/gemm_tc.cu"

int main() {
  const int M = 4096, N = 256, K = 4096;
  float *A, *B, *C;
  cudaMalloc(&A, (size_t)M * K * 4);
  cudaMalloc(&B, (size_t)N * K * 4);
  cudaMalloc(&C, (size_t)M * N * 4);
  cudaMemset(A, 0, (size_t)M * K * 4);
  cudaMemset(B, 0, (size_t)N * K * 4);
  for (int i = 0; i < 5; ++i) sage::sgemm_tc(A, B, C, M, N, K, 0);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> tr(1024 * 12);
  cudaMemcpyFromSymbol(tr.data(), sage::g_gemm_trace, tr.size() * 8);
  unsigned long long t0 = ~0ull, tend = 0;
  int ctas = 0;
  for (int c = 0; c < 1024; ++c)
    if (tr[c * 12 + 0]) { t0 = std::min(t0, tr[c * 12 + 0]); tend = std::max(tend, tr[c * 12 + 6]); ++ctas; }
  const char *names[10] = {"start", "setup done", "first K-block landed", "half K-blocks landed", "last MMA issued",
                           "accumulator ready", "epilogue done", "partial in smem", "cluster synced",
                           "rows reduced"};
  printf("%d CTAs, kernel span %.2f us (first start -> last epilogue end)\n", ctas, (tend - t0) / 1e3);
  for (int k = 0; k < 10; ++k) {
    std::vector<double> v;
    for (int c = 0; c < 1024; ++c)
      if (tr[c * 12 + 0] && tr[c * 12 + k]) v.push_back((tr[c * 12 + k] - t0) / 1e3);
    if (v.empty()) continue;
    std::sort(v.begin(), v.end());
    printf("  %-22s min %7.2f  median %7.2f  max %7.2f us\n", names[k], v.front(), v[v.size() / 2], v.back());
  }
  return 0;
}
