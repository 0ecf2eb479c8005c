// Latency of one fused-pivot CTA (k_pivot_blk, SPD; k_pivot_lu_blk, LU) vs n
// = m + r on an idle B200: 20 independent copies in one launch (20 SMs, no
// contention), CUDA events around the launch, best of 5.  The upper
// levels' waves hold 1-50 such nodes, so the per-node latency is the wave time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1510_07363_b200/csrc -o pivot_lat pivot_lat.cu
#include <cstdio>
#include <vector>
#include <cstring>
#include <cuda_runtime.h>
#include "kernels.cuh"
using namespace lorasp;
int main() {
  cudaFuncSetAttribute(k_pivot_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, 215 * 1024);
  cudaFuncSetAttribute(k_pivot_lu_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, 215 * 1024);
  int ns[] = {32, 48, 64, 96, 128, 160};
  const int NC = 20;
  double *K, *K0; int *st; PivTask *dt;
  cudaMalloc(&K, (size_t)NC * 160 * 160 * 8 * 2); cudaMalloc(&K0, (size_t)NC * 160 * 160 * 8 * 2);
  cudaMalloc(&st, 64); cudaMalloc(&dt, NC * sizeof(PivTask));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("{");
  for (int q = 0; q < 6; ++q) {
    const int n = ns[q], r = n / 4, m = n - r;
    std::vector<double> h((size_t)n * n * 2, 0.0);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        double v = (i == j) ? (i < m ? 4.0 : 0.0) : ((i < m && j < m && (i - j == 1 || j - i == 1)) ? -1.0 : 0.0);
        if (i >= m && j < m && (i - m) == (j % r)) v = 0.3;   // V^T rows
        if (j >= m && i < m && (j - m) == (i % r)) v = 0.3;
        h[i + (size_t)j * n] = v;
      }
    for (int c = 0; c < NC; ++c) cudaMemcpy(K0 + (size_t)c * 2 * n * n, h.data(), (size_t)n * n * 8, cudaMemcpyHostToDevice);
    float best[2] = {1e9f, 1e9f};
    for (int kind = 0; kind < 2; ++kind) {
      std::vector<PivTask> ts(NC);
      for (int c = 0; c < NC; ++c) {
        PivTask t{};
        t.F = K + (size_t)c * 2 * n * n; t.ld = n; t.m = m; t.r = r; t.node = c; t.F2 = t.F + (size_t)n * n;
        ts[c] = t;
      }
      cudaMemcpy(dt, ts.data(), NC * sizeof(PivTask), cudaMemcpyHostToDevice);
      for (int it = 0; it < 6; ++it) {
        cudaMemcpy(K, K0, (size_t)NC * 2 * n * n * 8, cudaMemcpyDeviceToDevice);
        cudaMemset(st, 0, 64);
        cudaEventRecord(e0);
        if (kind == 0) k_pivot_blk<<<NC, 512, pivb_smem_bytes(n)>>>(dt, st);
        else k_pivot_lu_blk<<<NC, 512, pivb_smem_bytes(n)>>>(dt, st);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it > 0 && ms < best[kind]) best[kind] = ms;
      }
      int hs[4];
      cudaMemcpy(hs, st, 16, cudaMemcpyDeviceToHost);
      double gr; memcpy(&gr, hs + 2, 8);
      if (hs[0]) printf("\"status_n%d_kind%d\": [%d, %d, %g], ", n, kind, hs[0], hs[1], gr);
    }
    printf("%s\"n%d\": {\"spd_us\": %.1f, \"lu_us\": %.1f}", q ? ", " : "", n, best[0] * 1e3, best[1] * 1e3);
  }
  printf("}\n");
  return 0;
}
