// Does a PDL-launched kernel see the scalar its single-CTA predecessor wrote?
// Chain per step k: k_part (296 CTAs: partial sums of x . y) -> k_final (1 CTA:
// s = sum of partials) -> k_axpy (y -= s * x / |x|^2), all launched with
// programmatic stream serialization; each kernel triggers at entry and waits
// (griddepcontrol.wait) before touching memory.  Compared with the same chain
// launched plainly: both must give the same |y|^2 (measured: identical, so this
// isolated chain does not reproduce the GMRES anomaly noted in DESIGN.md 6b).
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ void enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__global__ void k_part(int n, const double *x, const double *y, double *part) {
  enter();
  __shared__ double red[8];
  double s = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s += x[i] * y[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}
__global__ void k_final(const double *part, int np, double *out) {
  enter();
  __shared__ double red[8];
  double s = 0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < 8; ++w) t += red[w];
    *out = t;
  }
}
__global__ void k_axpy(int n, const double *s, const double *x, double *y) {
  enter();
  const double a = -*s;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = a * x[i] + y[i];
}
template <typename... KArgs, typename... Args>
void launch(bool pdl, void (*k)(KArgs...), int g, int b, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g);
  cfg.blockDim = dim3(b);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
int main() {
  const int n = 1 << 16, NV = 8, steps = 8;
  double *X, *y, *part, *sc;
  cudaMalloc(&X, sizeof(double) * n * NV);
  cudaMalloc(&y, sizeof(double) * n);
  cudaMalloc(&part, sizeof(double) * 512);
  cudaMalloc(&sc, sizeof(double) * 64);
  std::vector<double> hx(n * NV), hy(n);
  // orthonormal-ish basis vectors: disjoint supports, unit norm
  for (int v = 0; v < NV; ++v)
    for (int i = 0; i < n; ++i) hx[v * n + i] = ((i % NV) == v) ? 1.0 / sqrt((double)n / NV) : 0.0;
  for (int i = 0; i < n; ++i) hy[i] = 1.0 + 0.001 * (i % 97);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaMemcpy(X, hx.data(), sizeof(double) * n * NV, cudaMemcpyHostToDevice);
    cudaMemcpy(y, hy.data(), sizeof(double) * n, cudaMemcpyHostToDevice);
    for (int s = 0; s < steps; ++s)
      for (int v = 0; v < NV; ++v) {   // y -= (x_v . y) x_v  for every basis vector
        launch(pdl, k_part, 296, 256, st, n, (const double *)(X + (size_t)v * n), (const double *)y, part);
        launch(pdl, k_final, 1, 256, st, (const double *)part, 296, sc + v);
        launch(pdl, k_axpy, 592, 256, st, n, (const double *)(sc + v), (const double *)(X + (size_t)v * n), y);
      }
    cudaStreamSynchronize(st);
    std::vector<double> out(n);
    cudaMemcpy(out.data(), y, sizeof(double) * n, cudaMemcpyDeviceToHost);
    double nrm = 0;
    for (double v : out) nrm += v * v;
    printf("%s: |y|^2 after the projections = %.15e  err=%s\n", pdl ? "PDL " : "plain",
           nrm, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
