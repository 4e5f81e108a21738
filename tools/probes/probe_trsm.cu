// Isolated timing of trsm variants (L21 = (R11^-1 R12)^T, bsel = 64, p rows), with bit comparison.
#include <cstdio>
#include <vector>
#include <cstring>
#include <cstdint>
__device__ unsigned long long g_stamp[8];
#define TC_STAMP(k) do { if (blockIdx.x == 0 && threadIdx.x == 0) { unsigned long long _t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t)); g_stamp[k] = _t; } } while (0)
#include "../../paper_1208_2451_b200/csrc/tri64.cuh"
int main(int argc, char** argv) {
  const int64_t p = argc > 1 ? atoll(argv[1]) : 8192;
  const int b = 64;
  std::vector<double> R((size_t)b * p);
  srand(3);
  for (int i = 0; i < b; ++i)
    for (int64_t q = 0; q < p; ++q) R[(size_t)i * p + q] = (q == i ? 4.0 : 0.0) + (q >= i ? (rand() / (double)RAND_MAX - 0.5) : 0.0);
  double *Rd, *L1, *L2, *cand, *fro; long long* cf; DevState* st;
  const int64_t ldl = p;
  cudaMalloc(&Rd, R.size() * 8); cudaMalloc(&L1, (size_t)b * ldl * 8); cudaMalloc(&L2, (size_t)b * ldl * 8);
  cudaMalloc(&cand, 4096 * 8); cudaMalloc(&cf, 4096 * 8);
  cudaMalloc(&fro, 8); cudaMalloc(&st, sizeof(DevState)); cudaMemset(st, 0, sizeof(DevState));
  double one = 1.0; cudaMemcpy(fro, &one, 8, cudaMemcpyHostToDevice);
  cudaMemcpy(Rd, R.data(), R.size() * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(trsm_w_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int64_t ncol = p - b;
  auto timeit = [&](const char* name, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-10s %8.1f us  (%s)\n", name, ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
  };
  const size_t dynw = (((size_t)b * (b + 1) / 2 + 1) / 2 * 2 + (size_t)b * TTCP) * 8;
  timeit("trsm_w<2>", [&] { trsm_w_kernel<2><<<(int)std::min<int64_t>(2048, (ncol + TTC - 1) / TTC), TW_WARPS * 32, dynw>>>(Rd, p, b, L1, ldl, cand, cf, st, 0, fro, -1, -1); });
  timeit("trsm_c", [&] { trsm_c_kernel<<<(int)std::min<int64_t>(2048, (ncol + TC_COLS - 1) / TC_COLS), TC_T, 0>>>(Rd, p, b, L2, ldl, cand, cf, st, 0, fro, -1, -1); });
  { std::vector<double> h1((size_t)b * ldl), h2((size_t)b * ldl);
    cudaMemcpy(h1.data(), L1, h1.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), L2, h2.size() * 8, cudaMemcpyDeviceToHost);
    size_t diff = 0;
    for (int i = 0; i < b; ++i) for (int64_t c = 0; c < ncol; ++c) diff += memcmp(&h1[i * ldl + c], &h2[i * ldl + c], 8) != 0;
    printf("trsm_c bitwise differences: %zu\n", diff); }
  { unsigned long long h[8]; cudaMemcpyFromSymbol(h, g_stamp, sizeof(h));
    printf("stamps (ns from start): load %llu check-done %llu stage %llu  loop %llu  reduce %llu\n", h[4]-h[0], h[5]-h[0], h[1]-h[0], h[2]-h[1], h[3]-h[2]); }
  return 0;
}
