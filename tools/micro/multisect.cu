// Cycles of the eigenvalue phase pieces from kernels.cuh on one SM: sturm_count
// alone (24 counts per lane) and grp_multisect<4> over all m eigenvalues, for
// 128 / 256 / 512 threads, m = 40 (a random scaled tridiagonal).
#include <cstdio>
#include "../../paper_1510_07363_b200/csrc/kernels.cuh"
using namespace lorasp;
// candidate: (d_i, e2_{i-1}) pairs as double2, the next block's 8 pairs loaded
// into registers while the current block runs
__device__ __forceinline__ int sturm_b(const double2 *__restrict__ de, int m, double x) {
  double pa = 1.0, pb = 1.0, s = 1.0;
  unsigned hb = (unsigned)__double2hiint(pb);
  int c = 0;
  bool dead = false;
  double2 cur[8], nxt[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) cur[u] = de[u];
  for (int i0 = 0; i0 < m; i0 += 8) {
    if (i0 + 8 < m) {
#pragma unroll
      for (int u = 0; u < 8; ++u) nxt[u] = de[i0 + 8 + u];
    }
    double dx[8], ee[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      dx[u] = cur[u].x - x;
      ee[u] = cur[u].y;
    }
    dx[0] *= s;
    ee[0] *= s;
    ee[1] *= s;
    double sn = 1.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double p = fma(dx[u], pb, -ee[u] * pa);
      const unsigned hp = (unsigned)__double2hiint(p);
      c += (int)((hp ^ hb) >> 31);
      hb = hp;
      pa = pb;
      pb = p;
      if (u == 5) {
        const double amax = fmax(fabs(pa), fabs(pb));
        const int ex = (__double2hiint(amax) >> 20) & 0x7ff;
        sn = __hiloint2double((2046 - ex) << 20, 0);
      }
    }
    dead |= (pa == 0.0) && (pb == 0.0);
    s = sn;
#pragma unroll
    for (int u = 0; u < 8; ++u) cur[u] = nxt[u];
  }
  return dead ? -1 : c;
}
template <int MODE>
__global__ void k(const double *dg, const double *eg, int m, int reps, double *out, long long *cyc) {
  __shared__ double d[136], e2[136], lam[136];
  __shared__ double2 de[136];
  for (int i = threadIdx.x; i < 136; i += blockDim.x) {
    d[i] = i < m ? dg[i] : 4.0;
    e2[i] = i < m - 1 ? eg[i] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 136; i += blockDim.x) de[i] = make_double2(d[i], i == 0 ? 0.0 : e2[i - 1]);
  __syncthreads();
  long long t0 = clock64();
  int acc = 0;
  for (int r = 0; r < reps; ++r) {
    if (MODE == 0) {
      for (int q = 0; q < 24; ++q) acc += sturm_count(d, e2, m, -1.0 + 2.0 * (threadIdx.x + q) / 600.0 + 1e-3 * acc, 0.0);
    } else if (MODE == 2) {
      for (int q = 0; q < 24; ++q) acc += sturm_b(de, m, -1.0 + 2.0 * (threadIdx.x + q) / 600.0 + 1e-3 * acc);
    } else {
      grp_multisect<4>(d, e2, m, 0, m, -1.2, 1.2, 0.0, lam, 1.0);
    }
  }
  if (MODE != 1) lam[threadIdx.x % 136] = acc;
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = acc + lam[threadIdx.x % 136];
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  const int m = 40;
  double hd[136], he[136];
  for (int i = 0; i < 136; ++i) {
    hd[i] = 0.5 * __builtin_sin(i * 1.3);
    he[i] = 0.3 * __builtin_cos(i * 0.7);
    he[i] *= he[i];
  }
  double *dd, *de, *o;
  long long *c, h;
  cudaMalloc(&dd, sizeof(hd));
  cudaMalloc(&de, sizeof(he));
  cudaMalloc(&o, 8192);
  cudaMalloc(&c, 8);
  cudaMemcpy(dd, hd, sizeof(hd), cudaMemcpyHostToDevice);
  cudaMemcpy(de, he, sizeof(he), cudaMemcpyHostToDevice);
  for (int thr : {32, 128, 160, 256, 512}) {
    for (int rep = 0; rep < 2; ++rep) k<0><<<1, thr>>>(dd, de, m, 4, o, c);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("threads %3d: sturm_count %.1f cycles per step\n", thr, h / (4.0 * 24 * m));
    for (int rep = 0; rep < 2; ++rep) k<1><<<1, thr>>>(dd, de, m, 4, o, c);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("threads %3d: grp_multisect<4> all %d eigenvalues: %.0f cycles\n", thr, m, h / 4.0);
    for (int rep = 0; rep < 2; ++rep) k<2><<<1, thr>>>(dd, de, m, 4, o, c);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("threads %3d: sturm_b %.1f cycles per step\n", thr, h / (4.0 * 24 * m));
  }
  return 0;
}
