// Verification and solve kernels on the packed L\U factors:
//
//   rel. factorization error  metrics.rel_factorization_error (metrics.py:56-63):
//                             ||Pi A - L U||_F / ||A||_F.  Pi A is gathered into
//                             a work matrix, L U is subtracted one 64-wide
//                             k-block at a time with the DMMA Schur kernel
//                             (L block: unit lower diagonal block made explicit,
//                             U block: zeros below its diagonal), then two
//                             sum-of-squares reductions.
//   luprrp_solve              luprrp.py:204-214: y = L^-1 (P b) (unit lower),
//                             x = U^-1 y (true division), blocked by 64 rows:
//                             a 16-threads-per-row GEMV against the solved
//                             part, then a one-warp triangular solve of the
//                             diagonal block.  One CTA per right-hand side.
#pragma once
#include "common.cuh"

// C[i][j] = A[perm[i]][j], i < m, j < n (row-major)
__global__ void gather_rows_kernel(const double* __restrict__ A, int64_t lda, const int64_t* __restrict__ perm, int64_t m,
                                   int64_t n, double* __restrict__ C, int64_t ldc) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    C[i * ldc + j] = A[perm[i] * lda + j];
  }
}

// K-major M x Kp block of L for k-block [k0, k0+kb): rows r >= k0 of the
// packed factors; the diagonal block is unit lower (1 on the diagonal, 0 above).
__global__ void build_lk_kernel(const double* __restrict__ LU, int64_t ldlu, int64_t m, int64_t k0, int kb, int Kp,
                                double* __restrict__ Lk, int64_t ldlk) {
  const int64_t M = m - k0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M * Kp; e += (int64_t)gridDim.x * blockDim.x) {
    const int kk = (int)(e / M);
    const int64_t r = e - (int64_t)kk * M;
    double v = 0.0;
    if (kk < kb) v = r > kk ? LU[(k0 + r) * ldlu + k0 + kk] : (r == kk ? 1.0 : 0.0);
    Lk[(int64_t)kk * ldlk + r] = v;
  }
}

// Kp x N row-major block of U for k-block [k0, k0+kb): zeros below its diagonal.
__global__ void build_uk_kernel(const double* __restrict__ LU, int64_t ldlu, int64_t n, int64_t k0, int kb, int Kp,
                                double* __restrict__ Uk, int64_t lduk) {
  const int64_t N = n - k0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N * Kp; e += (int64_t)gridDim.x * blockDim.x) {
    const int kk = (int)(e / N);
    const int64_t c = e - (int64_t)kk * N;
    Uk[(int64_t)kk * lduk + c] = (kk < kb && c >= kk) ? LU[(k0 + kk) * ldlu + k0 + c] : 0.0;
  }
}

// out += sum of squares of X (m x n row-major); two-level: block partials then one atomic per block
__global__ void sumsq_kernel(const double* __restrict__ X, int64_t ldx, int64_t m, int64_t n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    const double v = X[i * ldx + j];
    s = fma(v, v, s);
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) atomicAdd(out, s);
  }
}

#define LS_T 1024
// x = U^-1 L^-1 (P b) for one right-hand side per CTA (column-major B, X).
__global__ void __launch_bounds__(LS_T) lu_solve_kernel(const double* __restrict__ LU, int64_t ldlu, int64_t n,
                                                       const int64_t* __restrict__ perm, const double* __restrict__ Bm,
                                                       int64_t ldb, double* X, int64_t ldx, DevState* st) {
  __shared__ double tb[64];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const double* b = Bm + (int64_t)blockIdx.x * ldb;
  double* x = X + (int64_t)blockIdx.x * ldx;
  for (int64_t i = t; i < n; i += LS_T) x[i] = b[perm[i]];
  __syncthreads();
  const int r = t >> 4, q = t & 15;
  // forward substitution with the unit lower factor
  for (int64_t i0 = 0; i0 < n; i0 += 64) {
    const int nb = (int)min((int64_t)64, n - i0);
    double acc = 0.0;
    if (r < nb) {
      const double* row = LU + (i0 + r) * ldlu;
      for (int64_t c = q; c < i0; c += 16) acc = fma(row[c], x[c], acc);
    }
    for (int o = 8; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (q == 0 && r < nb) tb[r] = x[i0 + r] - acc;
    __syncthreads();
    if (warp == 0) {
      double y0 = lane < nb ? tb[lane] : 0.0, y1 = lane + 32 < nb ? tb[lane + 32] : 0.0;
      for (int rr = 0; rr < nb; ++rr) {
        const double yr = __shfl_sync(0xffffffffu, rr < 32 ? y0 : y1, rr & 31);
        if (lane > rr && lane < nb) y0 -= LU[(i0 + lane) * ldlu + i0 + rr] * yr;
        if (lane + 32 > rr && lane + 32 < nb) y1 -= LU[(i0 + lane + 32) * ldlu + i0 + rr] * yr;
      }
      if (lane < nb) x[i0 + lane] = y0;
      if (lane + 32 < nb) x[i0 + lane + 32] = y1;
    }
    __syncthreads();
  }
  // back substitution with the upper factor
  const int64_t nblk = (n + 63) / 64;
  for (int64_t bi = nblk - 1; bi >= 0; --bi) {
    const int64_t i0 = bi * 64;
    const int nb = (int)min((int64_t)64, n - i0);
    double acc = 0.0;
    if (r < nb) {
      const double* row = LU + (i0 + r) * ldlu;
      for (int64_t c = i0 + nb + q; c < n; c += 16) acc = fma(row[c], x[c], acc);
    }
    for (int o = 8; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (q == 0 && r < nb) tb[r] = x[i0 + r] - acc;
    __syncthreads();
    if (warp == 0) {
      double y0 = lane < nb ? tb[lane] : 0.0, y1 = lane + 32 < nb ? tb[lane + 32] : 0.0;
      for (int rr = nb - 1; rr >= 0; --rr) {
        const double d = LU[(i0 + rr) * ldlu + i0 + rr];
        if (d == 0.0) {
          if (lane == 0) prrp_set_error(st, PRRP_ERR_SINGULAR_FACTOR, -1, (int)(i0 + rr), -1, 0.0);
        }
        double v = __shfl_sync(0xffffffffu, rr < 32 ? y0 : y1, rr & 31);
        v = div_rn(v, d);
        if (lane == (rr & 31)) {
          if (rr < 32) y0 = v;
          else y1 = v;
        }
        if (lane < rr && lane < nb) y0 -= LU[(i0 + lane) * ldlu + i0 + rr] * v;
        if (lane + 32 < rr && lane + 32 < nb) y1 -= LU[(i0 + lane + 32) * ldlu + i0 + rr] * v;
      }
      if (lane < nb) x[i0 + lane] = y0;
      if (lane + 32 < nb) x[i0 + lane + 32] = y1;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Stability measurements (metrics.py:65-145).
//
// residual_extended (metrics.py:75-92): r = rhs - A x accumulated in twice
// working precision, exactly the reference's recipe per row i, j ascending:
//   p, pe = two_prod(A[i,j], -x[j])   (Veltkamp split, 2^27 + 1)
//   s, se = two_sum(s, p)             (Knuth)
//   comp += pe + se;   r_i = s + comp
// Every operation is rounded on its own (no FMA contraction), so the result
// is bit-identical to the numpy elementwise evaluation.  One thread per row;
// x staged through shared memory.
// ---------------------------------------------------------------------------
#define RX_T 128
#define RX_XC 2048
__device__ __forceinline__ void two_prod_rn(double a, double b, double& p, double& e) {
  const double split = 134217729.0;
  p = mul_rn(a, b);
  const double ca = mul_rn(split, a);
  const double ah = sub_rn(ca, sub_rn(ca, a));
  const double al = sub_rn(a, ah);
  const double cb = mul_rn(split, b);
  const double bh = sub_rn(cb, sub_rn(cb, b));
  const double bl = sub_rn(b, bh);
  e = add_rn(add_rn(add_rn(sub_rn(mul_rn(ah, bh), p), mul_rn(ah, bl)), mul_rn(al, bh)), mul_rn(al, bl));
}

__device__ __forceinline__ void two_sum_rn(double a, double b, double& s, double& e) {
  s = add_rn(a, b);
  const double bb = sub_rn(s, a);
  e = add_rn(sub_rn(a, sub_rn(s, bb)), sub_rn(b, bb));
}

__global__ void __launch_bounds__(RX_T) residual_ext_kernel(const double* __restrict__ A, int64_t lda, int64_t m,
                                                            int64_t n, const double* __restrict__ x,
                                                            const double* __restrict__ rhs, double* __restrict__ r) {
  __shared__ double xs[RX_XC];
  const int64_t i = (int64_t)blockIdx.x * RX_T + threadIdx.x;
  double s = i < m ? rhs[i] : 0.0, comp = 0.0;
  for (int64_t j0 = 0; j0 < n; j0 += RX_XC) {
    const int nc = (int)min((int64_t)RX_XC, n - j0);
    __syncthreads();
    for (int c = threadIdx.x; c < nc; c += RX_T) xs[c] = -x[j0 + c];
    __syncthreads();
    if (i < m) {
      const double* row = A + i * lda + j0;
      for (int c = 0; c < nc; ++c) {
        double p, pe, se;
        two_prod_rn(row[c], xs[c], p, pe);
        two_sum_rn(s, p, s, se);
        comp = add_rn(comp, add_rn(pe, se));
      }
    }
  }
  if (i < m) r[i] = add_rn(s, comp);
}

// column sums of |A| (||A||_1 = max), one thread per column (coalesced rows)
__global__ void abs_colsum_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                                  double* __restrict__ colabs) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double s = 0.0;
  for (int64_t i = 0; i < m; ++i) s += fabs(A[i * lda + j]);
  colabs[j] = s;
}

// row sums of |A| and of |A| |x| (||A||_inf, the componentwise denominator),
// one warp per row
__global__ void abs_rowsum_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                                  const double* __restrict__ x, double* rowabs, double* absax) {
  const int lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= m) return;
  double s = 0.0, t = 0.0;
  const double* row = A + i * lda;
  for (int64_t j = lane; j < n; j += 32) {
    const double a = fabs(row[j]);
    s += a;
    if (x) t = fma(a, fabs(x[j]), t);
  }
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  if (lane == 0) {
    if (rowabs) rowabs[i] = s;
    if (absax) absax[i] = t;
  }
}
