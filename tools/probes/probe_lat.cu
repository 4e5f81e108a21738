// FP64 latency probe: dependent chains of DFMA / DADD / DMUL / DDIV / DSQRT and SHFL on one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  double x = a + threadIdx.x * 1e-9, y = b;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-3);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, y);
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __ddiv_rn(x, y) + 1.0;
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dsqrt_rn(x) + 1.0;
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fmax(x, y * (double)i);
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = t1 - t0;
  out[threadIdx.x] = x;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 64 * 8);
  const int n = 4096;
  lat<<<1, 32>>>(out, cyc, 1.0, 0.9999999, n);
  lat<<<1, 32>>>(out, cyc, 1.0, 0.9999999, n);
  long long h[8]; cudaMemcpy(h, cyc, 7 * 8, cudaMemcpyDeviceToHost);
  const char* names[] = {"DFMA", "DADD", "DMUL", "DDIV+DADD", "DSQRT+DADD", "SHFL64+DADD", "DMNMX(+DMUL)"};
  for (int i = 0; i < 7; ++i) printf("%-14s %.1f cycles/op (dependent chain, 1 warp)\n", names[i], (double)h[i] / n);
  // throughput with 4 warps on one SM sub-partition each
  return 0;
}
