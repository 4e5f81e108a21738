// Latency of the current p1_candidate (single lane), warm vs after touching a lot of other code.
#include <cstdio>
#include "../../paper_1208_2451_b200/csrc/panel1.cuh"
__global__ void __launch_bounds__(256, 1) k(double* out, long long* cyc, int wl, int steps) {
  __shared__ __align__(16) double wp[64];
  __shared__ P1Rec rec;
  const int t = threadIdx.x, lane = t & 31;
  double rr[P1_H];
  for (int e = 0; e < P1_H; ++e) rr[e] = 1.0 + 1e-3 * e + 1e-6 * t;
  const P1Reg xr{rr};
  double acc = 0.0;
  for (int kk = 0; kk < steps; ++kk) {
    const int r = kk & 7, L = 7 - (kk >> 3);
    __syncwarp();
    long long c0 = clock64();
    if (lane == wl) {
      int skip; double alpha, beta;
      p1_candidate(xr, r, L, 0, 2.0 + kk, wp, skip, alpha, beta);
      rec.alpha = alpha; rec.beta = beta; rec.skip = skip;
    }
    __syncwarp();
    long long c1 = clock64();
    acc += rec.alpha;
    if (t == 0) cyc[kk] = c1 - c0;
  }
  out[t] = acc + wp[3];
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 64 * 8);
  long long h[64];
  k<<<1, 32>>>(out, cyc, 5, 64);
  cudaMemcpy(h, cyc, 64 * 8, cudaMemcpyDeviceToHost);
  long long s = 0; for (int i = 0; i < 64; ++i) s += h[i];
  printf("candidate warm loop: mean %lld; k=0 %lld k=1 %lld k=8 %lld k=9 %lld k=40 %lld\n", s / 64, h[0], h[1], h[8], h[9], h[40]);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
