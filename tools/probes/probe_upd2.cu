// x[64] in registers, update x -= v*w with v from: shared memory / compile-time constants; 1 warp.
#include <cstdio>
#include <cstdint>
template <int NE, int VMODE>
__global__ void __launch_bounds__(256, 1) k(double* out, long long* cyc, double w0, int n) {
  __shared__ __align__(16) double vs[64];
  const int t = threadIdx.x;
  double x[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) x[i] = t + i;
  if (t < 64) vs[t] = 1e-3 * t;
  __syncthreads();
  double w = w0;
  const double2* vp = reinterpret_cast<const double2*>(vs);
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < NE / 2; ++i) {
      double2 q;
      if (VMODE == 0) q = vp[i];
      else if (VMODE == 1) q = make_double2(1e-3 * (2 * i + 1), 1e-3 * (2 * i + 2));
      else {
        // volatile shared loads: not hoisted, placed where written
        const uint32_t a = (uint32_t)__cvta_generic_to_shared(vs) + 16 * i;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(q.x), "=d"(q.y) : "r"(a));
      }
      if (VMODE == 3) {
        x[2 * i] = fma(-q.x, w, x[2 * i]);
        x[2 * i + 1] = fma(-q.y, w, x[2 * i + 1]);
      } else {
        x[2 * i] = __dsub_rn(x[2 * i], __dmul_rn(q.x, w));
        x[2 * i + 1] = __dsub_rn(x[2 * i + 1], __dmul_rn(q.y, w));
      }
    }
    w = w * 0.999 + x[5] * 1e-30;
  }
  long long t1 = clock64();
  if (t == 0) cyc[0] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int i = 0; i < NE; ++i) s += x[i];
  out[t] = s;
}
template <int NE, int VM>
void run(double* out, long long* cyc) {
  long long h; const int n = 1000;
  for (int r = 0; r < 2; ++r) k<NE, VM><<<1, 32>>>(out, cyc, 1.0, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("NE=%2d vmode=%d: %.0f cyc/pass, %.3f DP instr/cycle\n", NE, VM, (double)h / n, (VM == 3 ? 1.0 : 2.0) * NE * n / h);
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8192 * 8); cudaMalloc(&cyc, 64);
  run<48, 0>(out, cyc); run<56, 0>(out, cyc); run<60, 0>(out, cyc); run<64, 0>(out, cyc);
  run<64, 2>(out, cyc); run<64, 3>(out, cyc);
  return 0;
}
