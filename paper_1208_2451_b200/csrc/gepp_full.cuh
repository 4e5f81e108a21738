// gepp_factor for any shape (gepp.py:39-65), unblocked like the reference:
// per step k one pivot launch (first max of |column k| at or below the
// diagonal, row interchange over all n columns + row order) and one update
// launch (multipliers c[q,k] / c[k,k] by true division, then c[q,j] -=
// l_q * c[k,j] with the product rounded first, running max of the live
// trailing block).  HBM-bound: (m-k)(n-k) elements read and written per step.
#pragma once
#include "common.cuh"

__global__ void __launch_bounds__(1024) gf_pivot_kernel(double* A, int64_t lda, int64_t m, int64_t n, int64_t k,
                                                        int64_t* perm, DevState* st) {
  __shared__ unsigned long long s_best[32];
  __shared__ long long s_bi[32];
  if (prrp_failed(st)) return;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  // np.argmax order on |column k|: keys are the bit patterns of |x| (monotone
  // for non-negative doubles) with every NaN mapped above +inf, so the first
  // NaN wins like numpy's argmax; ties go to the smaller row.
  unsigned long long best = 0ull;
  long long bi = LLONG_MAX;
  for (int64_t q = k + t; q < m; q += blockDim.x) {
    const double x = fabs(A[q * lda + k]);
    const unsigned long long v = isnan(x) ? 0x7FF8000000000000ull : (unsigned long long)__double_as_longlong(x);
    if (v > best || (v == best && q < bi)) { best = v; bi = q; }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  if (lane == 0) { s_best[wid] = best; s_bi[wid] = bi; }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    best = lane < nw ? s_best[lane] : 0ull;
    bi = lane < nw ? s_bi[lane] : LLONG_MAX;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) {
      // an exactly zero pivot column (or an empty one) is singular (gepp.py:49-51)
      const bool sing = best == 0ull || bi < k || bi >= m;
      s_bi[0] = sing ? -1 : bi;
      if (sing) prrp_set_error(st, PRRP_ERR_SINGULAR_MATRIX, -1, -1, (int)k, 0.0);
    }
  }
  __syncthreads();
  const long long pv = s_bi[0];
  if (pv < 0 || pv == k) return;
  for (int64_t j = t; j < n; j += blockDim.x) {
    const double a = A[k * lda + j];
    A[k * lda + j] = A[pv * lda + j];
    A[pv * lda + j] = a;
  }
  if (t == 0) {
    const int64_t p = perm[k];
    perm[k] = perm[pv];
    perm[pv] = p;
  }
}

#define GF_ROWS 8
__global__ void __launch_bounds__(256) gf_update_kernel(double* A, int64_t lda, int64_t m, int64_t n, int64_t k,
                                                        DevState* st) {
  __shared__ double s_l[GF_ROWS];
  __shared__ double red[40];
  if (prrp_failed(st)) return;
  const int t = threadIdx.x;
  const double d = A[k * lda + k];
  const int64_t w = n - k - 1;
  double mx = 0.0;
  for (int64_t q0 = k + 1 + (int64_t)blockIdx.x * GF_ROWS; q0 < m; q0 += (int64_t)gridDim.x * GF_ROWS) {
    const int nr = (int)min((int64_t)GF_ROWS, m - q0);
    __syncthreads();
    if (t < nr) {
      const double l = div_rn(A[(q0 + t) * lda + k], d);
      A[(q0 + t) * lda + k] = l;
      s_l[t] = l;
    }
    __syncthreads();
    if (w > 0) {
      // all GF_ROWS loads in flight before the stores (the compiler cannot
      // reorder a load past a store to A)
      for (int64_t j = k + 1 + t; j < n; j += blockDim.x) {
        const double u = A[k * lda + j];
        double v[GF_ROWS];
#pragma unroll
        for (int r = 0; r < GF_ROWS; ++r) v[r] = r < nr ? A[(q0 + r) * lda + j] : 0.0;
#pragma unroll
        for (int r = 0; r < GF_ROWS; ++r)
          if (r < nr) {
            v[r] = sub_rn(v[r], mul_rn(s_l[r], u));
            A[(q0 + r) * lda + j] = v[r];
            mx = fmax(mx, fabs(v[r]));
          }
      }
    }
  }
  const double mm = block_max(mx, red);
  if (t == 0 && mm > 0.0) atomic_max_abs(&st->inter_max, mm);
}
