// Cycles per step of the division-free Sturm count (kernels.cuh sturm_count)
// with d / e2 in shared memory, 256 threads on one SM, m = 40.  Variants:
//  0: as in kernels.cuh (8-step blocks, loads inside the block)
//  1: the next block's d / e2 prefetched into registers during the current one
//  2: d / e2 interleaved (one 16-byte load per step) + prefetch
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__device__ __forceinline__ int count(const double *__restrict__ d, const double *__restrict__ e2,
                                     const double2 *__restrict__ de, int m, double x) {
  const double *e2m = e2 - 1;
  double p0 = 1.0, p1 = 1.0;
  int c = 0;
  bool zero = false;
  if (V == 0 || V >= 3) {
    unsigned zmask = 0xffffffffu;
    for (int i0 = 0; i0 < m; i0 += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u;
        const double ee = (i == 0) ? 0.0 : e2m[i];
        const double p2 = fma(d[i] - x, p1, -ee * p0);
        const long long b2 = __double_as_longlong(p2), b1 = __double_as_longlong(p1);
        if (V == 0) zero |= (b2 << 1) == 0;
        if (V == 4) zmask = min(zmask, (unsigned)__double2hiint(p2) & 0x7ff00000u);   // 0: zero or subnormal
        if (V == 4) c += (int)((unsigned)(__double2hiint(p2) ^ __double2hiint(p1)) >> 31);
        else c += (int)((unsigned long long)(b2 ^ b1) >> 63);
        p0 = p1;
        p1 = p2;
      }
      const double a = fmax(fabs(p0), fabs(p1));
      const long long ex = ((__double_as_longlong(a) >> 52) & 0x7ff) - 1023;
      const double sc = __longlong_as_double((long long)(1023 - ex) << 52);
      p0 *= sc;
      p1 *= sc;
      if (V == 4 && zmask == 0) zero = true;
    }
  } else {
    double dn[8], en[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (V == 1) {
        dn[u] = d[u];
        en[u] = u == 0 ? 0.0 : e2m[u];
      } else {
        double2 t = de[u];
        dn[u] = t.x;
        en[u] = t.y;
      }
    }
    for (int i0 = 0; i0 < m; i0 += 8) {
      double dc[8], ec[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        dc[u] = dn[u] - x;
        ec[u] = en[u];
      }
      if (i0 + 8 < m) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (V == 1) {
            dn[u] = d[i0 + 8 + u];
            en[u] = e2m[i0 + 8 + u];
          } else {
            double2 t = de[i0 + 8 + u];
            dn[u] = t.x;
            en[u] = t.y;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double p2 = fma(dc[u], p1, -ec[u] * p0);
        const long long b2 = __double_as_longlong(p2), b1 = __double_as_longlong(p1);
        zero |= (b2 << 1) == 0;
        c += (int)((unsigned long long)(b2 ^ b1) >> 63);
        p0 = p1;
        p1 = p2;
      }
      const double a = fmax(fabs(p0), fabs(p1));
      const long long ex = ((__double_as_longlong(a) >> 52) & 0x7ff) - 1023;
      const double sc = __longlong_as_double((long long)(1023 - ex) << 52);
      p0 *= sc;
      p1 *= sc;
    }
  }
  return zero ? -1 : c;
}

// NX interleaved counts per thread (independent chains hide the FP64 latency)
template <int NX>
__device__ __forceinline__ void count_multi(const double *__restrict__ d, const double *__restrict__ e2, int m,
                                           const double *x, int *c) {
  const double *e2m = e2 - 1;
  double p0[NX], p1[NX];
  bool zero = false;
#pragma unroll
  for (int j = 0; j < NX; ++j) {
    p0[j] = p1[j] = 1.0;
    c[j] = 0;
  }
  for (int i0 = 0; i0 < m; i0 += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u;
      const double ee = (i == 0) ? 0.0 : e2m[i];
      const double di = d[i];
#pragma unroll
      for (int j = 0; j < NX; ++j) {
        const double p2 = fma(di - x[j], p1[j], -ee * p0[j]);
        const long long b2 = __double_as_longlong(p2), b1 = __double_as_longlong(p1[j]);
        zero |= (b2 << 1) == 0;
        c[j] += (int)((unsigned long long)(b2 ^ b1) >> 63);
        p0[j] = p1[j];
        p1[j] = p2;
      }
    }
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      const double a = fmax(fabs(p0[j]), fabs(p1[j]));
      const long long ex = ((__double_as_longlong(a) >> 52) & 0x7ff) - 1023;
      const double sc = __longlong_as_double((long long)(1023 - ex) << 52);
      p0[j] *= sc;
      p1[j] *= sc;
    }
  }
  if (zero) c[0] = -1;
}
template <int NX>
__global__ void __launch_bounds__(256, 1) km(const double *dg, const double *eg, int m, int rounds, int *out,
                                               long long *cyc) {
  __shared__ double d[128], e2[128];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    d[i] = i < m ? dg[i] : 4.0;
    e2[i] = i < m - 1 ? eg[i] : 0.0;
  }
  __syncthreads();
  double lo = -1.0, hi = 1.0;
  int acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    double x[NX];
    int c[NX];
#pragma unroll
    for (int j = 0; j < NX; ++j) x[j] = lo + (hi - lo) * (threadIdx.x * NX + j + 1) * (1.0 / 1025.0);
    count_multi<NX>(d, e2, m, x, c);
#pragma unroll
    for (int j = 0; j < NX; ++j) acc += c[j];
    if (c[0] > m / 2) hi = x[0]; else lo = x[0] - 1e-3;
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int V>
__global__ void __launch_bounds__(256, 1) k(const double *dg, const double *eg, int m, int rounds, int *out,
                                              long long *cyc) {
  __shared__ double d[128], e2[128];
  __shared__ double2 de[128];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    d[i] = i < m ? dg[i] : 4.0;
    e2[i] = i < m - 1 ? eg[i] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 128; i += blockDim.x) de[i] = make_double2(d[i], i == 0 ? 0.0 : e2[i - 1]);
  __syncthreads();
  double lo = -1.0, hi = 1.0;
  int acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const double x = lo + (hi - lo) * (threadIdx.x + 1) / 257.0;
    const int c = count<V>(d, e2, de, m, x);
    acc += c;
    if (c > m / 2) hi = x; else lo = x - 1e-3;
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  const int m = 40, rounds = 200;
  double hd[128], he[128];
  for (int i = 0; i < 128; ++i) {
    hd[i] = 0.5 * __builtin_sin(i * 1.3);
    he[i] = 0.3 * __builtin_cos(i * 0.7);
    he[i] *= he[i];
  }
  double *dd, *de;
  int *o;
  long long *c, h;
  cudaMalloc(&dd, 1024);
  cudaMalloc(&de, 1024);
  cudaMalloc(&o, 4096);
  cudaMalloc(&c, 8);
  cudaMemcpy(dd, hd, 1024, cudaMemcpyHostToDevice);
  cudaMemcpy(de, he, 1024, cudaMemcpyHostToDevice);
  for (int v = 0; v < 8; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      if (v == 0) k<0><<<1, 256>>>(dd, de, m, rounds, o, c);
      if (v == 1) k<1><<<1, 256>>>(dd, de, m, rounds, o, c);
      if (v == 2) k<2><<<1, 256>>>(dd, de, m, rounds, o, c);
      if (v == 3) k<3><<<1, 256>>>(dd, de, m, rounds, o, c);
      if (v == 4) k<4><<<1, 256>>>(dd, de, m, rounds, o, c);
      if (v == 5) k<0><<<1, 128>>>(dd, de, m, rounds, o, c);
      if (v == 6) k<0><<<1, 32>>>(dd, de, m, rounds, o, c);
      if (v == 7) k<1><<<1, 32>>>(dd, de, m, rounds, o, c);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("variant %d: %.1f cycles / Sturm step (m = %d)\n", v, h / (double)rounds / m, m);
  }
  for (int nx = 1; nx <= 4; ++nx) {
    for (int thr = 128; thr <= 256; thr += 128) {
      for (int rep = 0; rep < 2; ++rep) {
        if (nx == 1) km<1><<<1, thr>>>(dd, de, m, rounds, o, c);
        if (nx == 2) km<2><<<1, thr>>>(dd, de, m, rounds, o, c);
        if (nx == 3) km<3><<<1, thr>>>(dd, de, m, rounds, o, c);
        if (nx == 4) km<4><<<1, thr>>>(dd, de, m, rounds, o, c);
      }
      cudaDeviceSynchronize();
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("NX %d, %d threads: %.1f cycles per step of all NX chains\n", nx, thr, h / (double)rounds / m);
    }
  }
  return 0;
}
