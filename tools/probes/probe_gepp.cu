// Per-phase timeline of the register GEPP kernel (copy of lsolve.cuh's gepp_reg_kernel with marks).
#include <cstdio>
#include <vector>
#include "../../paper_1208_2451_b200/csrc/lsolve.cuh"
__global__ void __launch_bounds__(GR_T, 1) gepp_probe(long long* tl, const double* src, int64_t ld, const int32_t* rowmap, int b,
                                                          double* D, int32_t* piv, int32_t* gperm, DevState* st,
                                                          int panel) {
  __shared__ double colk[2][64];
  __shared__ __align__(16) double prow[64], krow[64];
  __shared__ int s_gp[64];
  __shared__ double red[40];
  if (prrp_failed(st)) return;
  const int t = threadIdx.x, lane = t & 31;
  const int i = t >> 2, q = t & 3;
  double a[16];
  double mx = 0.0;
  {
    const bool rowok = i < b;
    const int64_t row = rowok ? (rowmap ? rowmap[i] : i) : 0;
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int j = 16 * q + s;
      a[s] = rowok && j < b ? src[row * ld + j] : 0.0;
      mx = fmax(mx, fabs(a[s]));
    }
  }
  if (t < 64) s_gp[t] = t;
  __syncthreads();
  for (int k = 0; k < b; ++k) {
    if (t == 0) tl[k * 8 + 0] = clock64();
    const int ks = k & 15, kq = k >> 4, cb = k & 1;
    // 1. column k, rows >= k, published by its owners
    double ak = a[0];
#pragma unroll
    for (int s = 1; s < 16; ++s)
      if (s == ks) ak = a[s];
    if (q == kq && i < b) colk[cb][i] = ak;
    if (t == 0) tl[k * 8 + 1] = clock64();
    __syncthreads();
    if (t == 0) tl[k * 8 + 2] = clock64();
    // 2. first-max pivot (every warp, redundantly)
    double best = -1.0;
    int bi = INT_MAX;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int r = k + lane + 32 * u;
      if (r < b) {
        const double v = fabs(colk[cb][r]);
        if (v > best) { best = v; bi = r; }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (best == 0.0) {
      if (t == 0) prrp_set_error(st, PRRP_ERR_SINGULAR_MATRIX, panel, -1, k, 0.0);
      return;
    }
    const int pv = bi;
    if (t == 0) tl[k * 8 + 3] = clock64();
    // 3. rows k and pv trade places through shared memory
    if (i == pv) {
#pragma unroll
      for (int s = 0; s < 16; s += 2) *reinterpret_cast<double2*>(&prow[16 * q + s]) = make_double2(a[s], a[s + 1]);
    }
    if (i == k && pv != k) {
#pragma unroll
      for (int s = 0; s < 16; s += 2) *reinterpret_cast<double2*>(&krow[16 * q + s]) = make_double2(a[s], a[s + 1]);
    }
    if (t == 0) {
      piv[k] = pv;
      if (pv != k) { const int g = s_gp[k]; s_gp[k] = s_gp[pv]; s_gp[pv] = g; }
    }
    if (t == 0) tl[k * 8 + 4] = clock64();
    __syncthreads();
    if (t == 0) tl[k * 8 + 5] = clock64();
    if (pv != k) {
      if (i == k) {
#pragma unroll
        for (int s = 0; s < 16; ++s) a[s] = prow[16 * q + s];
      } else if (i == pv) {
#pragma unroll
        for (int s = 0; s < 16; ++s) a[s] = krow[16 * q + s];
      }
    }
    // 4. multiplier and rank-1 update of rows k+1 .. b-1
    if (i > k && i < b) {
      const double ckk = colk[cb][pv];
      const double cik = colk[cb][i == pv ? k : i];
      const double l = div_fast(cik, ckk, __drcp_rn(ckk));
      // columns >= b are zero in a[] and prow[]: updating them is exact and harmless
      if (16 * q > k) {
#pragma unroll
        for (int s = 0; s < 16; s += 2) {
          const double2 pr = *reinterpret_cast<const double2*>(&prow[16 * q + s]);
          a[s] = sub_rn(a[s], mul_rn(l, pr.x));
          a[s + 1] = sub_rn(a[s + 1], mul_rn(l, pr.y));
          const double m0 = fabs(a[s]), m1 = fabs(a[s + 1]);
          const double m01 = m0 > m1 ? m0 : m1;
          mx = m01 > mx ? m01 : mx;
        }
      } else if (16 * q + 15 >= k) {
#pragma unroll
        for (int s = 0; s < 16; ++s) {
          const int j = 16 * q + s;
          if (j == k) a[s] = l;
          if (j > k) {
            a[s] = sub_rn(a[s], mul_rn(l, prow[j]));
            const double m0 = fabs(a[s]);
            mx = m0 > mx ? m0 : mx;
          }
        }
      }
    }
    if (t == 0) tl[k * 8 + 6] = clock64();
  }
  __syncthreads();
  if (i < b) {
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int j = 16 * q + s;
      if (j < b) D[(int64_t)i * b + j] = a[s];
    }
  }
  if (t < b) gperm[t] = s_gp[t];
  const double m = block_max(mx, red);
  if (t == 0) atomic_max_abs(&st->finish_max, m);
}


int main() {
  const int b = 64;
  std::vector<double> h(b * b);
  srand(1);
  for (auto& v : h) v = rand() / (double)RAND_MAX - 0.5;
  double *A, *D; int *piv, *gp; DevState* st; long long* tl;
  cudaMalloc(&A, b * b * 8); cudaMalloc(&D, b * b * 8); cudaMalloc(&piv, 256); cudaMalloc(&gp, 256);
  cudaMalloc(&st, sizeof(DevState)); cudaMemset(st, 0, sizeof(DevState)); cudaMalloc(&tl, 64 * 8 * 8);
  cudaMemcpy(A, h.data(), b * b * 8, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) gepp_probe<<<1, GR_T>>>(tl, A, b, nullptr, b, D, piv, gp, st, 0);
  cudaDeviceSynchronize();
  std::vector<long long> T(64 * 8);
  cudaMemcpy(T.data(), tl, 64 * 8 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"select+sts", "bar1", "argmax", "swap-write", "bar2", "update"};
  double acc[6] = {0};
  for (int k = 0; k < 64; ++k) for (int m = 0; m < 6; ++m) acc[m] += T[k * 8 + m + 1] - T[k * 8 + m];
  for (int m = 0; m < 6; ++m) printf("%s %.0f  ", nm[m], acc[m] / 64);
  printf("\nstep total %.0f cycles; k=1: ", (double)(T[63 * 8 + 6] - T[0]) / 64);
  for (int m = 0; m < 6; ++m) printf("%lld ", T[8 + m + 1] - T[8 + m]);
  printf("\n%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
