// Row-level data movement and the per-column finish kernels.
//
//   permute_kernel   luprrp._permute_tail (luprrp.py:98-104): the panel
//                    permutation moves <= 2b rows (+2 per swap-loop
//                    interchange); only those rows are moved, whole rows of
//                    the packed L\U storage (L part and trailing part), plus
//                    the global row order.  Pure data movement.
//   blockrow_kernel  luprrp._gepp_finish (luprrp.py:107-127) for the block
//                    row: L part rows permuted by the GEPP order, diagonal
//                    block written from the single-CTA GEPP, every trailing
//                    column eliminated with the same pivots / multipliers
//                    (gepp.py:53-60: swap, c -= l * c_k product-then-subtract)
//                    and its running max folded into finish_max.
//   compose_kernel   L21 <- L21[:, perm] @ L11 with matcore.matmul's rounding
//                    (matcore.py:41-51: accumulation from zero in increasing k,
//                    one FMA per k, which is what BLAS dger does on FMA hosts).
#pragma once
#include "common.cuh"

__global__ void iota_kernel(int64_t* p, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = i;
}

// max|A| over an m x n row-major matrix into st->orig_max / inter_max / finish_max
__global__ void maxabs_kernel(const double* A, int64_t lda, int64_t m, int64_t n, DevState* st) {
  __shared__ double red[40];
  double mx = 0.0;
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    mx = fmax(mx, fabs(A[i * lda + j]));
  }
  mx = block_max(mx, red);
  if (threadIdx.x == 0) {
    atomic_max_abs(&st->orig_max, mx);
    atomic_max_abs(&st->inter_max, mx);
    atomic_max_abs(&st->finish_max, mx);
  }
}

#define PERM_CW 16              // columns per block
#define PERM_MAXROWS 1536       // moved rows staged in shared memory (192 KB)

// moved: pairs (dst pos, src pos) relative to row0.  Block x handles columns
// [x*CW, x*CW+CW) of every moved row: gather all sources, then scatter.
__global__ void __launch_bounds__(256) permute_kernel(double* A, int64_t lda, int64_t row0, int64_t ncols,
                                                      const int32_t* moved, int64_t* p, DevState* st, int panel) {
  extern __shared__ __align__(16) double tmp[];
  if (prrp_failed(st)) return;
  const int cnt = st->moved;
  if (cnt == 0) return;
  if (cnt > PERM_MAXROWS) {
    if (blockIdx.x == 0 && threadIdx.x == 0)
      prrp_set_error(st, PRRP_ERR_UNSUPPORTED, panel, -1, -1, 0.0);
    return;
  }
  const int64_t c0 = (int64_t)blockIdx.x * PERM_CW;
  const int cw = (int)min((int64_t)PERM_CW, ncols - c0);
  for (int e = threadIdx.x; e < cnt * PERM_CW; e += blockDim.x) {
    const int r = e / PERM_CW, cc = e % PERM_CW;
    if (cc < cw) tmp[e] = A[(row0 + moved[2 * r + 1]) * lda + c0 + cc];
  }
  __shared__ int64_t ptmp[PERM_MAXROWS];
  if (blockIdx.x == 0)
    for (int r = threadIdx.x; r < cnt; r += blockDim.x) ptmp[r] = p[row0 + moved[2 * r + 1]];
  __syncthreads();
  for (int e = threadIdx.x; e < cnt * PERM_CW; e += blockDim.x) {
    const int r = e / PERM_CW, cc = e % PERM_CW;
    if (cc < cw) A[(row0 + moved[2 * r]) * lda + c0 + cc] = tmp[e];
  }
  if (blockIdx.x == 0)
    for (int r = threadIdx.x; r < cnt; r += blockDim.x) p[row0 + moved[2 * r]] = ptmp[r];
}

// Column-range variant for the look-ahead schedule: the moved rows of one
// panel, columns [c_lo, c_hi) only (three launches on three streams cover
// the panel + next panel, the trailing columns and the L part); the pair
// count comes from moved_cnt (double-buffered per panel).  Blocks stage up
// to PC_CAP doubles: cpb = min(32, PC_CAP / cnt) columns per pass.  The
// launch with p != nullptr also moves the global row order.
#define PC_CAP 4096
#define PC_ROWS 1024
__global__ void __launch_bounds__(256) permute_cols_kernel(double* A, int64_t lda, int64_t row0, int64_t c_lo,
                                                          int64_t c_hi, const int32_t* moved, const int32_t* moved_cnt,
                                                          int64_t* p, DevState* st, int panel) {
  __shared__ __align__(16) double tmp[PC_CAP];
  __shared__ int64_t srow[PC_ROWS], drow[PC_ROWS];   // source / destination row offsets (elements)
  if (prrp_failed(st)) return;
  const int cnt = *moved_cnt;
  if (cnt == 0) return;
  if (cnt > PC_ROWS) {
    if (blockIdx.x == 0 && threadIdx.x == 0) prrp_set_error(st, PRRP_ERR_UNSUPPORTED, panel, -1, -1, 0.0);
    return;
  }
  const int t = threadIdx.x;
  for (int r = t; r < cnt; r += blockDim.x) {
    srow[r] = (row0 + moved[2 * r + 1]) * lda;
    drow[r] = (row0 + moved[2 * r]) * lda;
  }
  __syncthreads();
  const int cpb = min(32, PC_CAP / cnt);
  for (int64_t c0 = c_lo + (int64_t)blockIdx.x * cpb; c0 < c_hi; c0 += (int64_t)gridDim.x * cpb) {
    const int cw = (int)min((int64_t)cpb, c_hi - c0);
    const int tot = cnt * cw;
    // 8 independent loads in flight per thread, then the staging stores
    for (int e0 = t; e0 < tot; e0 += 8 * blockDim.x) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        const int r = e / cw, cc = e - r * cw;
        v[u] = e < tot ? A[srow[r] + c0 + cc] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        if (e < tot) tmp[e] = v[u];
      }
    }
    __syncthreads();
    for (int e = t; e < tot; e += blockDim.x) {
      const int r = e / cw, cc = e - r * cw;
      A[drow[r] + c0 + cc] = tmp[e];
    }
    __syncthreads();
  }
  if (p && blockIdx.x == 0) {
    int64_t* pt = reinterpret_cast<int64_t*>(tmp);
    for (int r = t; r < cnt; r += blockDim.x) pt[r] = p[row0 + moved[2 * r + 1]];
    __syncthreads();
    for (int r = t; r < cnt; r += blockDim.x) p[row0 + moved[2 * r]] = pt[r];
  }
}

// Block row finish.  Columns [0, col0): rows col0.. permuted by gperm.
// Columns [col0, col0+b): packed L11\U11 from D.  Columns [col0+b, n):
// pivots + elimination with L11 (strictly lower part of D), running max.
#define BR_TW 64
__global__ void __launch_bounds__(BR_TW) blockrow_kernel(double* A, int64_t lda, int64_t col0, int b, int64_t n,
                                                        const double* D, const int32_t* piv, const int32_t* gperm,
                                                        int64_t* p, DevState* st) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[40];
  __shared__ int s_piv[PRRP_MAXH], s_gp[PRRP_MAXH];
  __shared__ int64_t s_p[PRRP_MAXH];
  if (prrp_failed(st)) return;
  double* L = sm;                       // b x b (row-major) copy of D
  double* xs = sm + b * b;              // b x BR_TW column tile
  const int t = threadIdx.x;
  for (int i = t; i < b; i += blockDim.x) { s_piv[i] = piv[i]; s_gp[i] = gperm[i]; }
  const int64_t j = (int64_t)blockIdx.x * BR_TW + t;
  const bool on = j < n;
  const bool trailing = on && j >= col0 + b;
  if (blockIdx.x * (int64_t)BR_TW + BR_TW > col0 + b)   // this block has trailing columns
    for (int e = t; e < b * b; e += blockDim.x) L[e] = D[e];
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int i = t; i < b; i += blockDim.x) s_p[i] = p[col0 + s_gp[i]];
    __syncthreads();
    for (int i = t; i < b; i += blockDim.x) p[col0 + i] = s_p[i];
  }
  double mx = 0.0;
  if (on && j < col0) {
    for (int i = 0; i < b; ++i) xs[i * BR_TW + t] = A[(col0 + s_gp[i]) * lda + j];
    for (int i = 0; i < b; ++i) A[(col0 + i) * lda + j] = xs[i * BR_TW + t];
  } else if (on && j < col0 + b) {
    const int jc = (int)(j - col0);
    for (int i = 0; i < b; ++i) A[(col0 + i) * lda + j] = D[i * b + jc];
  } else if (trailing) {
    // Rows carry their multipliers through later interchanges, so replaying
    // the reference's step-by-step elimination equals: gather the rows in
    // their final order, then eliminate with the final L11 column by column
    // (same multiplier, same pivot value, same update order per element).
    for (int i = 0; i < b; ++i) {
      const double v = A[(col0 + s_gp[i]) * lda + j];
      xs[i * BR_TW + t] = v;
      mx = fmax(mx, fabs(v));
    }
    for (int k = 0; k < b; ++k) {
      if (k + 1 < b) {
        const double xk = xs[k * BR_TW + t];
        for (int i = k + 1; i < b; ++i) {
          const double v = sub_rn(xs[i * BR_TW + t], mul_rn(L[i * b + k], xk));
          xs[i * BR_TW + t] = v;
          mx = fmax(mx, fabs(v));
        }
      }
    }
    for (int i = 0; i < b; ++i) A[(col0 + i) * lda + j] = xs[i * BR_TW + t];
  }
  const double m = block_max(mx, red);
  if (t == 0 && m > 0.0) atomic_max_abs(&st->finish_max, m);
}

// compose: out[r][j] = sum_k L21[r][gperm[k]] * L11[k][j], fma chain from 0 in
// increasing k.  L21 column-major (ldl), out row-major rows of A.
__global__ void __launch_bounds__(128) compose_kernel(const double* L21, int64_t ldl, int64_t M, int b,
                                                        const double* D, const int32_t* gperm, double* out,
                                                        int64_t ldo, DevState* st) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_gp[PRRP_MAXH];
  if (prrp_failed(st)) return;
  double* L = sm;                     // unit lower L11, b x b row-major
  double* xs = sm + b * b;            // b x TW
  const int TW = blockDim.x;
  const int t = threadIdx.x;
  for (int i = t; i < b; i += blockDim.x) s_gp[i] = gperm[i];
  for (int e = t; e < b * b; e += blockDim.x) {
    const int k = e / b, jj = e % b;
    L[e] = k > jj ? D[e] : (k == jj ? 1.0 : 0.0);
  }
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * TW + t;
  if (r >= M) return;
  for (int k = 0; k < b; ++k) xs[k * TW + t] = L21[(int64_t)s_gp[k] * ldl + r];
  double* o = out + r * ldo;
  for (int jc = 0; jc < b; jc += 8) {
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < b; ++k) {
      const double x = xs[k * TW + t];
      const double* lr = L + k * b + jc;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (jc + q < b) acc[q] = fma(x, lr[q], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (jc + q < b) o[jc + q] = acc[q];
  }
}
