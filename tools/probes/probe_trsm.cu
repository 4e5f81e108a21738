// Isolated timing of trsm variants (L21 = (R11^-1 R12)^T, bsel = 64, p rows), with bit comparison.
#include <cstdio>
#include <vector>
#include <cstring>
#include "../../paper_1208_2451_b200/csrc/tri64.cuh"
int main() {
  const int64_t p = 8192;
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
  timeit("trsm_v", [&] { trsm_v_kernel<<<(int)std::min<int64_t>(2048, (ncol + TV_COLS - 1) / TV_COLS), TV_T, 0>>>(Rd, p, b, L2, ldl, cand, cf, st, 0, fro, -1, -1); });
  std::vector<double> h1((size_t)b * ldl), h2((size_t)b * ldl);
  cudaMemcpy(h1.data(), L1, h1.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), L2, h2.size() * 8, cudaMemcpyDeviceToHost);
  size_t diff = 0;
  for (int i = 0; i < b; ++i) for (int64_t c = 0; c < ncol; ++c) diff += memcmp(&h1[i * ldl + c], &h2[i * ldl + c], 8) != 0;
  printf("bitwise differences: %zu\n", diff);
  return 0;
}
