// Warp-per-column triangular kernels for panel widths b <= 128.
//
// One warp owns one column (lane l holds rows l, l+32, ... : NR = b/32 rows
// per lane in registers); the sequential dimension runs as a short runtime
// loop whose pivot value is broadcast with one shuffle.  Code stays small
// (no 2000-line unrolled bodies thrashing the instruction cache) and every
// element sees exactly the reference's sequence of operations:
//
//   trsm_w_kernel      L21 = (R11^-1 R12)^T  matcore.trsm_upper (matcore.py:78-94):
//                      for i = b-1..0: x_i /= u_ii; x_l -= u_li x_i (l < i)
//   compose_w_kernel   L21 <- L21[:,p] L11   matcore.matmul     (matcore.py:41-51):
//                      y_j = fma chain over k = j..b-1 from +0
//   blockrow_w_kernel  GEPP finish of the block row (gepp.py:53-60):
//                      x_i -= l_ik x_k for i > k, k increasing; running max
#pragma once
#include "lsolve.cuh"

#define TW_WARPS 8                  // warps per block
#define T64_B 64                    // kept for the driver's b == 64 checks
#define T64_TW (TW_WARPS * 32)

template <int NR>
__global__ void __launch_bounds__(TW_WARPS * 32) trsm_w_kernel(const double* __restrict__ Rbuf, int64_t p, int bsel,
                                                              double* L21, int64_t ldl, double* cand,
                                                              long long* cand_flat, DevState* st, int panel) {
  extern __shared__ __align__(16) double r11[];     // packed upper, bsel(bsel+1)/2
  __shared__ double red_d[33];
  __shared__ long long red_l[33];
  if (prrp_failed(st)) return;
  load_r11(Rbuf, p, bsel, r11);
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) r11_checks(r11, bsel, st->fro, st, panel, true);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ncol = p - bsel;
  double worst = -1.0;
  long long wflat = LLONG_MAX;
  for (int64_t jj = (int64_t)blockIdx.x * TW_WARPS + warp; jj < ncol; jj += (int64_t)gridDim.x * TW_WARPS) {
    const int64_t pos = bsel + jj;
    double x[NR];
#pragma unroll
    for (int u = 0; u < NR; ++u) {
      const int i = lane + 32 * u;
      x[u] = i < bsel ? Rbuf[(int64_t)i * p + pos] : 0.0;
    }
    for (int i = bsel - 1; i >= 0; --i) {
      const int ou = i >> 5, ol = i & 31;
      double xi = 0.0;
#pragma unroll
      for (int u = 0; u < NR; ++u)
        if (u == ou) xi = x[u];
      xi = __shfl_sync(0xffffffffu, xi, ol);
      xi = div_rn(xi, r11[upk(i, i)]);
      const double* rc = r11 + upk(0, i);
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int l = lane + 32 * u;
        if (l < i) x[u] = sub_rn(x[u], mul_rn(rc[l], xi));
        else if (l == i) x[u] = xi;
      }
    }
#pragma unroll
    for (int u = 0; u < NR; ++u) {
      const int i = lane + 32 * u;
      if (i < bsel) {
        L21[(int64_t)i * ldl + jj] = x[u];
        const double ax = fabs(x[u]);
        const long long fl = (long long)i * ncol + jj;
        if (ax > worst || (ax == worst && fl < wflat)) { worst = ax; wflat = fl; }
      }
    }
  }
  reduce_worst(worst, wflat, red_d, red_l);
  if (threadIdx.x == 0) { cand[blockIdx.x] = worst; cand_flat[blockIdx.x] = wflat; }
}

// out[r][j] = sum_{k >= j} L21[r][gperm[k]] * L11[k][j]
template <int NR>
__global__ void __launch_bounds__(TW_WARPS * 32) compose_w_kernel(const double* __restrict__ L21, int64_t ldl,
                                                                 int64_t M, int b, const double* __restrict__ D,
                                                                 const int32_t* gperm, double* out, int64_t ldo,
                                                                 DevState* st) {
  extern __shared__ __align__(16) double lt[];   // lt[k*b + j] = L11[k][j] (unit lower)
  __shared__ int s_gp[PRRP_MAXH];
  if (prrp_failed(st)) return;
  const int t = threadIdx.x;
  for (int i = t; i < b; i += blockDim.x) s_gp[i] = gperm[i];
  for (int e = t; e < b * b; e += blockDim.x) {
    const int k = e / b, j = e % b;
    lt[e] = k > j ? D[e] : (k == j ? 1.0 : 0.0);
  }
  __syncthreads();
  const int lane = t & 31, warp = t >> 5;
  for (int64_t r = (int64_t)blockIdx.x * TW_WARPS + warp; r < M; r += (int64_t)gridDim.x * TW_WARPS) {
    double xv[NR], acc[NR];
#pragma unroll
    for (int u = 0; u < NR; ++u) {
      const int k = lane + 32 * u;
      xv[u] = k < b ? L21[(int64_t)s_gp[k] * ldl + r] : 0.0;
      acc[u] = 0.0;
    }
    for (int k = 0; k < b; ++k) {
      double xk = 0.0;
#pragma unroll
      for (int u = 0; u < NR; ++u)
        if (u == (k >> 5)) xk = xv[u];
      xk = __shfl_sync(0xffffffffu, xk, k & 31);
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int j = lane + 32 * u;
        if (j <= k && j < b) acc[u] = fma(xk, lt[k * b + j], acc[u]);
      }
    }
    double* o = out + r * ldo;
#pragma unroll
    for (int u = 0; u < NR; ++u) {
      const int j = lane + 32 * u;
      if (j < b) o[j] = acc[u];
    }
  }
}

// Block-row finish (see blockrow_kernel): warp per column.
template <int NR>
__global__ void __launch_bounds__(TW_WARPS * 32) blockrow_w_kernel(double* A, int64_t lda, int64_t col0, int b,
                                                                  int64_t n, const double* __restrict__ D,
                                                                  const int32_t* gperm, int64_t* p, DevState* st) {
  extern __shared__ __align__(16) double lc[];   // lc[k*b + i] = L11[i][k] (column k contiguous)
  __shared__ int s_gp[PRRP_MAXH];
  __shared__ int64_t s_p[PRRP_MAXH];
  __shared__ double red[40];
  if (prrp_failed(st)) return;
  const int t = threadIdx.x;
  for (int i = t; i < b; i += blockDim.x) s_gp[i] = gperm[i];
  for (int e = t; e < b * b; e += blockDim.x) {
    const int i = e / b, k = e % b;
    lc[k * b + i] = D[e];
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int i = t; i < b; i += blockDim.x) s_p[i] = p[col0 + s_gp[i]];
    __syncthreads();
    for (int i = t; i < b; i += blockDim.x) p[col0 + i] = s_p[i];
  }
  const int lane = t & 31, warp = t >> 5;
  double mx = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * TW_WARPS + warp; j < n; j += (int64_t)gridDim.x * TW_WARPS) {
    double x[NR];
    if (j >= col0 && j < col0 + b) {
      const int jc = (int)(j - col0);
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int i = lane + 32 * u;
        if (i < b) x[u] = D[i * b + jc];
      }
    } else {
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int i = lane + 32 * u;
        x[u] = i < b ? A[(col0 + s_gp[i]) * lda + j] : 0.0;
      }
      if (j >= col0 + b) {
#pragma unroll
        for (int u = 0; u < NR; ++u) mx = fmax(mx, fabs(x[u]));
        for (int k = 0; k + 1 < b; ++k) {
          double xk = 0.0;
#pragma unroll
          for (int u = 0; u < NR; ++u)
            if (u == (k >> 5)) xk = x[u];
          xk = __shfl_sync(0xffffffffu, xk, k & 31);
          const double* lk = lc + k * b;
#pragma unroll
          for (int u = 0; u < NR; ++u) {
            const int i = lane + 32 * u;
            if (i > k && i < b) {
              x[u] = sub_rn(x[u], mul_rn(lk[i], xk));
              mx = fmax(mx, fabs(x[u]));
            }
          }
        }
      }
    }
    // the whole column is read before any row is written (the same warp owns it)
    __syncwarp();
#pragma unroll
    for (int u = 0; u < NR; ++u) {
      const int i = lane + 32 * u;
      if (i < b) A[(col0 + i) * lda + j] = x[u];
    }
  }
  const double m = block_max(mx, red);
  if (t == 0 && m > 0.0) atomic_max_abs(&st->finish_max, m);
}
