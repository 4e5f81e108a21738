// Cycle cost of one p64_apply + p64_norm_after on register and shared-memory columns.
#include <cstdio>
#include "../../paper_1208_2451_b200/csrc/panel64.cuh"
__global__ void k_apply(double* out, long long* cyc, int nwarps_active) {
  extern __shared__ double sd[];
  __shared__ double vs[64];
  const int t = threadIdx.x, g = t & 1;
  double rr[P64_E];
  for (int e = 0; e < P64_E; ++e) rr[e] = 1.0 + 1e-3 * e + 1e-6 * t;
  for (int e = 0; e < P64_E; ++e) sd[e * P64_T + t] = 2.0 + 1e-3 * e + 1e-6 * t;
  if (t < 64) vs[t] = 0.01 * t;
  __syncthreads();
  RegCol xr{rr};
  SmemCol xs{sd + t};
  double key = 0;
  long long c0 = clock64();
  if ((t >> 5) < nwarps_active) {
    for (int k = 0; k < 64; ++k) {
      p64_apply(xr, g, k, vs, 1e-3, true);
      key += p64_norm_after(xr, g, k);
    }
  }
  long long c1 = clock64();
  if ((t >> 5) < nwarps_active) {
    for (int k = 0; k < 64; ++k) {
      p64_apply(xs, g, k, vs, 1e-3, true);
      key += p64_norm_after(xs, g, k);
    }
  }
  long long c2 = clock64();
  if (t == 0) { cyc[0] = c1 - c0; cyc[1] = c2 - c1; }
  for (int e = 0; e < P64_E; ++e) key += rr[e];
  out[t] = key;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 64);
  cudaFuncSetAttribute(k_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  for (int nw : {1, 4, 16}) {
    k_apply<<<1, 512, P64_E * P64_T * 8>>>(out, cyc, nw);
    k_apply<<<1, 512, P64_E * P64_T * 8>>>(out, cyc, nw);
    long long h[2]; cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
    printf("active warps %2d: register column %.0f cycles/step, smem column %.0f cycles/step (%s)\n", nw, h[0] / 64.0, h[1] / 64.0, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
