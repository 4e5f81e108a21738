// Cost of pieces of the panel1 candidate-reflector sequence on one warp, in isolation.
#include <cstdio>
#include "../../paper_1208_2451_b200/csrc/panel1.cuh"
__global__ void __launch_bounds__(256, 1) k_cand(double* out, long long* cyc, int wl, int KBr) {
  __shared__ double wp[64 * 32];
  const int t = threadIdx.x, lane = t & 31;
  double rr[P1_H];
  for (int e = 0; e < P1_H; ++e) rr[e] = 1.0 + 1e-3 * e + 1e-6 * t;
  double acc = 0;
  for (int rep = 0; rep < 4; ++rep) {
    const int KB = KBr, k = 8 * KB;
    __syncwarp();
    long long c0 = clock64();
    if (lane == wl) {
#define P1_PUB(KBC) _Pragma("unroll") for (int i = 8 * (KBC); i < P1_H; ++i) wp[i] = rr[i];
      P1_DISPATCH(KB, P1_PUB)
#undef P1_PUB
    }
    __syncwarp();
    long long c1 = clock64();
    if (lane == wl) {
#pragma unroll
      for (int i = 32; i < P1_H; ++i) wp[i] = rr[i] + 1.0;
    }
    __syncwarp();
    long long c2 = clock64();
#pragma unroll
    for (int i = 32; i < P1_H; ++i) wp[i * 32 + lane] = rr[i] + 2.0;
    __syncwarp();
    long long c3 = clock64();
    const double xk = wp[k];
    const double vtv = p1_warp_sumsq(wp + k, 64 - k, xk);
    long long c4 = clock64();
    double key = 0;
    if (lane == wl) {
#define P1_SS(KBC) key = p1_sumsq<KBC, true>(xr_dummy, 0, xk);
      const P1Reg xr{rr};
      switch (KB) { case 0: key = p1_sumsq<0, true>(xr, 0, xk); break; default: key = p1_sumsq<4, true>(xr, 0, xk); break; }
    }
    key = __shfl_sync(0xffffffffu, key, wl);
    long long c5 = clock64();
    acc += vtv + key;
    if (t == 0 && rep == 3) { cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; cyc[3] = c4 - c3; cyc[4] = c5 - c4; }
  }
  out[t] = acc;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 64 * 8);
  long long h[8];
  for (int KB : {0, 4}) {
    k_cand<<<1, 32>>>(out, cyc, 5, KB);
    cudaMemcpy(h, cyc, 5 * 8, cudaMemcpyDeviceToHost);
    printf("KB=%d switch-copy %lld | static copy 32 %lld | full-warp copy 32 %lld | warp_sumsq %lld | lane sumsq %lld cycles\n", KB, h[0], h[1], h[2], h[3], h[4]);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
