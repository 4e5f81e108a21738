// Register-update issue rate on one warp: x[i] -= v[i]*w (separate mul/sub or FMA), NE elements.
#include <cstdio>
template <int NE, int FMA>
__global__ void __launch_bounds__(256, 1) k(double* out, long long* cyc, double w0, int n) {
  const int t = threadIdx.x;
  double x[NE], v[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) { x[i] = t + i; v[i] = 1e-3 * (i + t); }
  double w = w0;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < NE; ++i) x[i] = FMA ? fma(-v[i], w, x[i]) : __dsub_rn(x[i], __dmul_rn(v[i], w));
    w = w * 0.999 + x[5] * 1e-30;
  }
  long long t1 = clock64();
  if (t == 0) cyc[0] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int i = 0; i < NE; ++i) s += x[i] + v[i];
  out[t] = s;
}
template <int NE, int FMA>
void run(double* out, long long* cyc, int nw) {
  long long h; const int n = 1000;
  for (int r = 0; r < 2; ++r) k<NE, FMA><<<1, 32 * nw>>>(out, cyc, 1.0, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double ins = (double)NE * (FMA ? 1 : 2);
  printf("NE=%2d %s warps=%d: %.0f cyc/pass, %.3f DP instr/cycle/warp\n", NE, FMA ? "fma    " : "mul+sub", nw, (double)h / n, ins * n / h);
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8192 * 8); cudaMalloc(&cyc, 64);
  run<16, 0>(out, cyc, 1); run<32, 0>(out, cyc, 1); run<64, 0>(out, cyc, 1);
  run<16, 1>(out, cyc, 1); run<32, 1>(out, cyc, 1); run<64, 1>(out, cyc, 1);
  run<64, 0>(out, cyc, 4); run<64, 0>(out, cyc, 8);
  return 0;
}
