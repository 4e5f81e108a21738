// 64-element dot with 4/8 accumulators: v from registers / shared (volatile LDS.128) / shared (plain); 1 warp.
#include <cstdio>
#include <cstdint>
template <int MODE, int NACC>
__global__ void __launch_bounds__(256, 1) k(double* out, long long* cyc, int n) {
  __shared__ __align__(16) double vs[64];
  const int t = threadIdx.x;
  double x[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) x[i] = t + i;
  if (t < 64) vs[t] = 1e-3 * t;
  __syncthreads();
  const uint32_t va = (uint32_t)__cvta_generic_to_shared(vs);
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
    double d[NACC];
#pragma unroll
    for (int a = 0; a < NACC; ++a) d[a] = 0.0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      double2 v;
      if (MODE == 0) v = make_double2(1e-3 * (2 * i) + acc, 1e-3 * (2 * i + 1));
      else if (MODE == 1) asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(va + 16 * i));
      else v = reinterpret_cast<const double2*>(vs)[i];
      d[(2 * i) % NACC] = fma(v.x, x[2 * i], d[(2 * i) % NACC]);
      d[(2 * i + 1) % NACC] = fma(v.y, x[2 * i + 1], d[(2 * i + 1) % NACC]);
    }
    double s = 0;
#pragma unroll
    for (int a = 0; a < NACC; ++a) s += d[a];
    acc += s * 1e-30;
  }
  long long t1 = clock64();
  if (t == 0) cyc[0] = t1 - t0;
  double s = acc;
#pragma unroll
  for (int i = 0; i < 64; ++i) s += x[i];
  out[t] = s;
}
template <int M, int A>
void run(double* out, long long* cyc) {
  long long h; const int n = 1000;
  for (int r = 0; r < 2; ++r) k<M, A><<<1, 32>>>(out, cyc, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dot64 mode=%d nacc=%d: %.0f cyc/pass\n", M, A, (double)h / n);
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8192 * 8); cudaMalloc(&cyc, 64);
  run<0, 4>(out, cyc); run<1, 4>(out, cyc); run<2, 4>(out, cyc);
  run<0, 8>(out, cyc); run<1, 8>(out, cyc); run<2, 8>(out, cyc);
  return 0;
}
