// Cycle cost of one panel1 step body (p1_apply_kb + p1_next_key) on register columns,
// per k, with 1..8 active warps per CTA (1 CTA, 256 threads).
#include <cstdio>
#include "../../paper_1208_2451_b200/csrc/panel1.cuh"
__global__ void __launch_bounds__(256, 1) k_apply(double* out, long long* cyc, int nwarps_active) {
  __shared__ double vs[64];
  const int t = threadIdx.x;
  double rr[P1_H];
  for (int e = 0; e < P1_H; ++e) rr[e] = 1.0 + 1e-3 * e + 1e-6 * t;
  if (t < 64) vs[t] = 0.01 * t;
  __syncthreads();
  const P1Reg xr{rr};
  const uint32_t vsa = (uint32_t)__cvta_generic_to_shared(vs);
  double key = 0;
  for (int k = 0; k < 64; ++k) {
    __syncthreads();
    long long c0 = clock64();
    if ((t >> 5) < nwarps_active) {
      const int r = k & 7;
#define AP(KBC) { p1_apply_kb<KBC>(xr, vsa, 1e-3, true); key += p1_next_key<KBC>(xr, r); }
      P1_DISPATCH(k >> 3, AP)
    }
    __syncthreads();
    long long c1 = clock64();
    if (t == 0) cyc[k] = c1 - c0;
    if (t == 5) {
      const int r = k & 7;
#define CD(KBC) key += p1_sumsq<KBC, true>(xr, r, key);
      P1_DISPATCH(k >> 3, CD)
    }
    __syncthreads();
    long long c2 = clock64();
    if (t == 0) cyc[64 + k] = c2 - c1;
  }
  for (int e = 0; e < P1_H; ++e) key += rr[e];
  out[t] = key;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 128 * 8);
  long long h[128];
  for (int rep = 0; rep < 2; ++rep)
  for (int nw : {1, 4, 8}) {
    k_apply<<<1, 256>>>(out, cyc, nw);
    cudaMemcpy(h, cyc, 128 * 8, cudaMemcpyDeviceToHost);
    long long s = 0; for (int k = 0; k < 64; ++k) s += h[k];
    long long s2 = 0; for (int k = 0; k < 64; ++k) s2 += h[64 + k];
    printf("   lone-lane sumsq after apply: mean %lld; k=0 %lld k=1 %lld k=7 %lld k=8 %lld k=16 %lld\n", s2 / 64, h[64], h[65], h[71], h[72], h[80]);
    printf("rep %d apply+norm nw=%d: mean %lld cyc/step; k=0 %lld k=1 %lld k=7 %lld k=8 %lld k=16 %lld k=32 %lld k=48 %lld k=62 %lld\n", rep, nw, s / 64, h[0], h[1], h[7], h[8], h[16], h[32], h[48], h[62]);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
