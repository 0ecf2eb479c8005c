// What the division-free Sturm step costs on one warp: the bare two-term
// recurrence, + sign counting, + per-block renormalisation, + loads.
#include <cstdio>
#include <cuda_runtime.h>
// lagged sign count (the pair (p_{i-2}, p_{i-1}) is compared while p_i's DFMA
// is in flight), next block's (d, e2) loaded during the current block
__device__ __forceinline__ int sturm_lag(const double2 *__restrict__ de, int nblk, double x) {
  double pa = 1.0, pb = 1.0, s = 1.0;
  int c = 0;
  double2 nx[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) nx[u] = de[u];
  for (int b = 0; b < nblk; ++b) {
    double dx[8], ee[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      dx[u] = nx[u].x - x;
      ee[u] = nx[u].y;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) nx[u] = de[(8 * b + 8 + u) & 511];
    dx[0] *= s;
    ee[0] *= s;
    ee[1] *= s;
    double sn = 1.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double p = fma(dx[u], pb, -ee[u] * pa);
      c += (int)(((unsigned)__double2hiint(pa) ^ (unsigned)__double2hiint(pb)) >> 31);
      pa = pb;
      pb = p;
      if (u == 5) {
        const double amax = fmax(fabs(pa), fabs(pb));
        const int ex = (__double2hiint(amax) >> 20) & 0x7ff;
        sn = __hiloint2double((2046 - ex) << 20, 0);
      }
    }
    s = sn;
  }
  c += (int)(((unsigned)__double2hiint(pa) ^ (unsigned)__double2hiint(pb)) >> 31);
  return c;
}
template <int MODE>
__global__ void k(const double2 *g, int nblk, double x0, double *out, long long *cyc) {
  __shared__ double2 de[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) de[i] = g[i & 63];
  __syncthreads();
  double dx[8], ee[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    dx[u] = de[u].x - x0 - 1e-3 * threadIdx.x;
    ee[u] = de[u].y;
  }
  double pa = 1.0, pb = 1.0, s = 1.0;
  unsigned hb = 0x3ff00000u;
  int c = 0;
  long long t0 = clock64();
  if (MODE == 4) {
    for (int rr = 0; rr < nblk / 8; ++rr) c += sturm_lag(de, 8, x0 + 1e-9 * c);
  } else
  for (int b = 0; b < nblk; ++b) {
    if (MODE >= 3) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double2 t = de[(8 * b + u) & 511];
        dx[u] = t.x - x0;
        ee[u] = t.y;
      }
    }
    double sn = 1.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double cu = (MODE >= 2 && u == 0) ? dx[u] * s : dx[u];
      const double p = fma(cu, pb, -ee[u] * pa);
      if (MODE >= 1) {
        const unsigned hp = (unsigned)__double2hiint(p);
        c += (int)((hp ^ hb) >> 31);
        hb = hp;
      }
      pa = pb;
      pb = p;
      if (MODE >= 2 && u == 5) {
        const double amax = fmax(fabs(pa), fabs(pb));
        const int ex = (__double2hiint(amax) >> 20) & 0x7ff;
        sn = __hiloint2double((2046 - ex) << 20, 0);
      }
    }
    if (MODE >= 2) s = sn;
    else if ((b & 7) == 7) { pa *= 1e-30; pb *= 1e-30; }
  }
  out[threadIdx.x] = pa + pb + c;
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double2 h[64];
  for (int i = 0; i < 64; ++i) h[i] = make_double2(0.5 * __builtin_sin(i * 1.3), 0.09 * __builtin_cos(i * 0.7) * __builtin_cos(i * 0.7));
  double2 *g;
  double *o;
  long long *c, hc;
  cudaMalloc(&g, sizeof(h));
  cudaMalloc(&o, 8192);
  cudaMalloc(&c, 8);
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  const int nb = 1000;
  const char *nm[] = {"bare recurrence", "+ sign count", "+ renormalise", "+ smem loads", "lagged+prefetch"};
  for (int thr : {32, 128, 256}) {
    for (int M = 0; M < 5; ++M) {
      for (int rep = 0; rep < 2; ++rep) {
        if (M == 0) k<0><<<1, thr>>>(g, nb, 0.1, o, c);
        if (M == 1) k<1><<<1, thr>>>(g, nb, 0.1, o, c);
        if (M == 2) k<2><<<1, thr>>>(g, nb, 0.1, o, c);
        if (M == 3) k<3><<<1, thr>>>(g, nb, 0.1, o, c);
        if (M == 4) k<4><<<1, thr>>>(g, nb, 0.1, o, c);
      }
      cudaDeviceSynchronize();
      cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
      printf("threads %3d %-16s %.1f cycles / step\n", thr, nm[M], hc / (8.0 * nb));
    }
  }
  return 0;
}
