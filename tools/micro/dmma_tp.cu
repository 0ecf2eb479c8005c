// FP64 tensor-core (DMMA, mma.sync ... .f64) vs FP64 FMA-pipe (DFMA) throughput
// on B200, whole GPU (north_star item 3: "Schur GEMMs on FP64 DMMA tensor cores
// only for block sizes where ncu shows the tensor pipe beating the FMA path").
//   dfma   : every thread runs 8 independent DFMA chains          (2 flops / DFMA)
//   m8n8k4 : every warp runs 4 independent accumulators of mma.sync.m8n8k4.f64
//            (8*8*4*2 = 512 flops / warp instruction)
//   m16n8k16: mma.sync.m16n8k16.f64 (sm_90+ shape, 4096 flops / warp instruction)
// Grid = 148 SMs x 4 CTAs x 256 threads; CUDA-event timed; TFLOP/s printed.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double *out, double a, double b, int n) {
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = a + j + threadIdx.x;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], b, a);
  double r = 0;
  for (int j = 0; j < 8; ++j) r += x[j];
  if (r == 12345.0) out[threadIdx.x] = r;
}

__global__ void k_m8n8k4(double *out, double a, int n) {
  double A = a + threadIdx.x, B = a * 0.5;
  double c[4][2];
  for (int j = 0; j < 4; ++j) c[j][0] = c[j][1] = 0.0;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(A), "d"(B));
  }
  double r = 0;
  for (int j = 0; j < 4; ++j) r += c[j][0] + c[j][1];
  if (r == 12345.0) out[threadIdx.x] = r;
}

__global__ void k_m16n8k16(double *out, double a, int n) {
  double A[8], B[4];
  for (int j = 0; j < 8; ++j) A[j] = a + j + threadIdx.x;
  for (int j = 0; j < 4; ++j) B[j] = a * 0.5 + j;
  double c[2][4];
  for (int j = 0; j < 2; ++j)
    for (int q = 0; q < 4; ++q) c[j][q] = 0.0;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
          "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
          : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
          : "d"(A[0]), "d"(A[1]), "d"(A[2]), "d"(A[3]), "d"(A[4]), "d"(A[5]), "d"(A[6]), "d"(A[7]), "d"(B[0]),
            "d"(B[1]), "d"(B[2]), "d"(B[3]));
  }
  double r = 0;
  for (int j = 0; j < 2; ++j)
    for (int q = 0; q < 4; ++q) r += c[j][q];
  if (r == 12345.0) out[threadIdx.x] = r;
}

int main() {
  double *o;
  cudaMalloc(&o, 1 << 20);
  const int grid = 148 * 4, block = 256, n = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const double warps = grid * (block / 32.0);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_dfma<<<grid, block>>>(o, 0.5, 0.999, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fd = 2.0 * 8 * n * (double)grid * block;
    cudaEventRecord(e0);
    k_m8n8k4<<<grid, block>>>(o, 0.5, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms2;
    cudaEventElapsedTime(&ms2, e0, e1);
    const double f2 = 512.0 * 4 * n * warps;
    cudaEventRecord(e0);
    k_m16n8k16<<<grid, block>>>(o, 0.5, n / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms3;
    cudaEventElapsedTime(&ms3, e0, e1);
    const double f3 = 4096.0 * 2 * (n / 4) * warps;
    if (rep)
      printf("{\"dfma_tflops\": %.2f, \"dmma_m8n8k4_tflops\": %.2f, \"dmma_m16n8k16_tflops\": %.2f, \"err\": \"%s\"}\n",
             fd / ms / 1e9, f2 / ms2 / 1e9, f3 / ms3 / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
