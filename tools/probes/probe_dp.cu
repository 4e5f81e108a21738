// FP64 issue rates: independent DADD / DMUL / DFMA / mixed mul+sub chains, 1..8 warps per SM.
#include <cstdio>
template <int OP>
__global__ void thr(double* out, long long* cyc, double y, int n) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (OP == 0) x[i] = __dadd_rn(x[i], y);
      if (OP == 1) x[i] = __dmul_rn(x[i], y);
      if (OP == 2) x[i] = fma(x[i], y, 1e-3);
      if (OP == 3) x[i] = __dsub_rn(x[i], __dmul_rn(y, x[(i + 1) & 15]));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  out[threadIdx.x] = s;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8192 * 8); cudaMalloc(&cyc, 64);
  long long h; const int n = 2048;
  const char* nm[] = {"DADD", "DMUL", "DFMA", "DMUL+DSUB pairs"};
  for (int op = 0; op < 4; ++op)
    for (int nw : {1, 2, 4, 8, 16}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (op == 0) thr<0><<<1, 32 * nw>>>(out, cyc, 1.0000001, n);
        if (op == 1) thr<1><<<1, 32 * nw>>>(out, cyc, 1.0000001, n);
        if (op == 2) thr<2><<<1, 32 * nw>>>(out, cyc, 1.0000001, n);
        if (op == 3) thr<3><<<1, 32 * nw>>>(out, cyc, 1.0000001, n);
      }
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double instr = (double)n * 16 * nw * (op == 3 ? 2 : 1);
      printf("%-16s warps=%2d: %.3f warp-instr/cycle/SM\n", nm[op], nw, instr / h);
    }
  return 0;
}
