// Validate fast correctly-rounded division q = a/b via a correctly rounded
// reciprocal y = RN(1/b) and one FMA correction (Markstein), against __ddiv_rn.
#include <cstdio>
#include <cstdint>
#include <curand_kernel.h>
__device__ __forceinline__ double fdiv(double a, double b, double y) {
  const double q = __dmul_rn(a, y);
  const double r = fma(-b, q, a);
  return fma(r, y, q);
}
__global__ void check(unsigned long long* bad, unsigned long long seed, int iters, int mode) {
  curandStatePhilox4_32_10_t st;
  curand_init(seed, blockIdx.x * blockDim.x + threadIdx.x, 0, &st);
  unsigned long long nb = 0;
  for (int i = 0; i < iters; ++i) {
    double a, b;
    if (mode == 0) { a = curand_normal_double(&st); b = curand_normal_double(&st); }
    else if (mode == 1) { a = curand_uniform_double(&st) * 2 - 1; b = curand_uniform_double(&st) * 1e-3; }
    else {  // random bit patterns in a moderate exponent range
      unsigned long long ua = ((unsigned long long)curand(&st) << 32) | curand(&st);
      unsigned long long ub = ((unsigned long long)curand(&st) << 32) | curand(&st);
      ua = (ua & 0x800FFFFFFFFFFFFFull) | ((unsigned long long)(1023 + (int)(curand(&st) % 200) - 100) << 52);
      ub = (ub & 0x800FFFFFFFFFFFFFull) | ((unsigned long long)(1023 + (int)(curand(&st) % 200) - 100) << 52);
      a = __longlong_as_double(ua); b = __longlong_as_double(ub);
    }
    const double y = __drcp_rn(b);
    const double q = fdiv(a, b, y);
    const double ref = __ddiv_rn(a, b);
    if (__double_as_longlong(q) != __double_as_longlong(ref)) ++nb;
  }
  atomicAdd(bad, nb);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(d, 0, 8);
    const int blocks = 148 * 8, threads = 256, iters = 1000;
    check<<<blocks, threads>>>(d, 1234 + mode, iters, mode);
    unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("mode %d: %llu mismatches out of %llu (%s)\n", mode, h, (unsigned long long)blocks * threads * iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
