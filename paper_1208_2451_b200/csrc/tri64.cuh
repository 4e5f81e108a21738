// Warp-per-column triangular kernels for panel widths b <= 128.
//
// A block stages a tile of TC = 32 columns (coalesced global loads into a
// padded shared tile); each warp then owns one column at a time (lane l holds
// rows l, l+32, ... : NR = ceil(b/32) rows per lane in registers) and runs the
// sequential dimension as a short runtime loop whose pivot value is broadcast
// with one shuffle.  Results go back through the tile for coalesced stores.
// Every element sees exactly the reference's sequence of operations:
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
#define TC 32                       // columns per tile
#define TCP (TC + 1)                // padded tile pitch
#define T64_B 64
#define T64_TW (TW_WARPS * 32)

template <int NR>
__device__ __forceinline__ double lane_pick(const double (&x)[NR], int row) {
  double v = 0.0;
#pragma unroll
  for (int u = 0; u < NR; ++u)
    if (u == (row >> 5)) v = x[u];
  return __shfl_sync(0xffffffffu, v, row & 31);
}

// trsm tile: one column per warp (latency-bound chain of bsel divisions)
#define TTC TW_WARPS
#define TTCP (TTC + 1)

template <int NR>
__global__ void __launch_bounds__(TW_WARPS * 32) trsm_w_kernel(const double* __restrict__ Rbuf, int64_t p, int bsel,
                                                              double* L21, int64_t ldl, double* cand,
                                                              long long* cand_flat, DevState* st, int panel,
                                                              const double* fro, int tl, int ti) {
  extern __shared__ __align__(16) double sm[];
  double* r11 = sm;                                    // packed upper, bsel(bsel+1)/2
  double* tile = sm + ((bsel * (bsel + 1) / 2 + 1) & ~1);   // bsel x TTCP
  __shared__ double red_d[33];
  __shared__ long long red_l[33];
  __shared__ double rcp[PRRP_MAXH];
  if (prrp_failed(st)) return;
  load_r11(Rbuf, p, bsel, r11);
  __syncthreads();
  for (int i = threadIdx.x; i < bsel; i += blockDim.x) rcp[i] = __drcp_rn(r11[upk(i, i)]);
  if (blockIdx.x == 0 && threadIdx.x == 0) r11_checks(r11, bsel, *fro, st, panel, true, tl, ti);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t ncol = p - bsel;
  double worst = -1.0;
  long long wflat = LLONG_MAX;
  for (int64_t c0 = (int64_t)blockIdx.x * TTC; c0 < ncol; c0 += (int64_t)gridDim.x * TTC) {
    const int tc = (int)min((int64_t)TTC, ncol - c0);
    for (int e = t; e < bsel * TTC; e += blockDim.x) {
      const int i = e / TTC, cc = e % TTC;
      if (cc < tc) tile[i * TTCP + cc] = Rbuf[(int64_t)i * p + bsel + c0 + cc];
    }
    __syncthreads();
    for (int cc = warp; cc < tc; cc += TW_WARPS) {
      double x[NR];
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int i = lane + 32 * u;
        x[u] = i < bsel ? tile[i * TTCP + cc] : 0.0;
      }
      for (int i = bsel - 1; i >= 0; --i) {
        const double xi = div_fast(lane_pick(x, i), r11[upk(i, i)], rcp[i]);
        const double* rc = r11 + upk(0, i);
#pragma unroll
        for (int u = 0; u < NR; ++u) {
          const int l = lane + 32 * u;
          if (l < i) x[u] = sub_rn(x[u], mul_rn(rc[l], xi));
          else if (l == i) x[u] = xi;
        }
      }
      const int64_t jj = c0 + cc;
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int i = lane + 32 * u;
        if (i < bsel) {
          tile[i * TTCP + cc] = x[u];
          const double ax = fabs(x[u]);
          const long long fl = (long long)i * ncol + jj;
          if (ax > worst || (ax == worst && fl < wflat)) { worst = ax; wflat = fl; }
        }
      }
    }
    __syncthreads();
    for (int e = t; e < bsel * TTC; e += blockDim.x) {
      const int i = e / TTC, cc = e % TTC;
      if (cc < tc) L21[(int64_t)i * ldl + c0 + cc] = tile[i * TTCP + cc];
    }
    __syncthreads();
  }
  reduce_worst(worst, wflat, red_d, red_l);
  if (threadIdx.x == 0) { cand[blockIdx.x] = worst; cand_flat[blockIdx.x] = wflat; }
}

// trsm, four columns per warp (8 lanes per column; lane j of a group holds
// rows j, j+8, ..., j+56 in registers).  Per step i (descending): the owner
// lane's value is broadcast within the group, every lane divides it
// (div_fast = true division), and each lane updates its rows l < i with the
// reference's product-then-subtract (matcore.py:78-94).  ~10 instructions per
// column-step instead of ~80 for a warp per column.  Requires bsel <= 64.
#define TV_WARPS 8
#define TV_T (TV_WARPS * 32)
#define TV_COLS (TV_WARPS * 4)
__global__ void __launch_bounds__(TV_T) trsm_v_kernel(const double* __restrict__ Rbuf, int64_t p, int bsel,
                                                      double* L21, int64_t ldl, double* cand, long long* cand_flat,
                                                      DevState* st, int panel, const double* fro, int tl, int ti) {
  __shared__ double r11[64 * 65 / 2];
  __shared__ double rcp[64], dg[64];
  __shared__ double red_d[33];
  __shared__ long long red_l[33];
  if (prrp_failed(st)) return;
  load_r11(Rbuf, p, bsel, r11);
  __syncthreads();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int i = t; i < bsel; i += blockDim.x) {
    dg[i] = r11[upk(i, i)];
    rcp[i] = __drcp_rn(dg[i]);
  }
  if (blockIdx.x == 0 && t == 0) r11_checks(r11, bsel, *fro, st, panel, true, tl, ti);
  __syncthreads();
  const int64_t ncol = p - bsel;
  const int g = lane >> 3, j = lane & 7;
  const unsigned gmask = 0xffu << (8 * g);
  double worst = -1.0;
  long long wflat = LLONG_MAX;
  for (int64_t cb = ((int64_t)blockIdx.x * TV_WARPS + warp) * 4; cb < ncol; cb += (int64_t)gridDim.x * TV_COLS) {
    const int64_t c = cb + g;
    const bool on = c < ncol;
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int row = j + 8 * q;
      x[q] = (on && row < bsel) ? Rbuf[(int64_t)row * p + bsel + c] : 0.0;
    }
#pragma unroll 1
    for (int i = bsel - 1; i >= 0; --i) {
      // x[i >> 3] by a select tree (a dynamic index would put x in local memory)
      const int qi = i >> 3;
      const bool b0 = qi & 1, b1 = qi & 2, b2 = qi & 4;
      const double s01 = b0 ? x[1] : x[0], s23 = b0 ? x[3] : x[2];
      const double s45 = b0 ? x[5] : x[4], s67 = b0 ? x[7] : x[6];
      const double s03 = b1 ? s23 : s01, s47 = b1 ? s67 : s45;
      const double xo = b2 ? s47 : s03;
      double xi = __shfl_sync(0xffffffffu, xo, (lane & ~7) | (i & 7));
      xi = div_fast(xi, dg[i], rcp[i]);
      const double* u = r11 + i * (i + 1) / 2;   // column i of R11, rows 0..i-1
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int row = j + 8 * q;
        if (row < i) x[q] = sub_rn(x[q], mul_rn(u[row], xi));
        else if (row == i) x[q] = xi;
      }
    }
    (void)gmask;
    if (on) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int row = j + 8 * q;
        if (row < bsel) {
          L21[(int64_t)row * ldl + c] = x[q];
          const double ax = fabs(x[q]);
          const long long fl = (long long)row * ncol + c;
          if (ax > worst || (ax == worst && fl < wflat)) { worst = ax; wflat = fl; }
        }
      }
    }
  }
  reduce_worst(worst, wflat, red_d, red_l);
  if (t == 0) { cand[blockIdx.x] = worst; cand_flat[blockIdx.x] = wflat; }
}

// out[r][j] = sum_{k >= j} L21[r][gperm[k]] * L11[k][j]
template <int NR>
__global__ void __launch_bounds__(TW_WARPS * 32) compose_w_kernel(const double* __restrict__ L21, int64_t ldl,
                                                                 int64_t M, int b, const double* __restrict__ D,
                                                                 const int32_t* gperm, double* out, int64_t ldo,
                                                                 DevState* st) {
  extern __shared__ __align__(16) double sm[];
  double* lt = sm;                       // lt[k*b + j] = L11[k][j] (unit lower)
  double* tile = sm + b * b;             // b x TCP: tile[k][r] = L21[r][gperm[k]]
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
  for (int64_t r0 = (int64_t)blockIdx.x * TC; r0 < M; r0 += (int64_t)gridDim.x * TC) {
    const int tr = (int)min((int64_t)TC, M - r0);
    for (int e = t; e < b * TC; e += blockDim.x) {
      const int k = e / TC, rr = e % TC;
      if (rr < tr) tile[k * TCP + rr] = L21[(int64_t)s_gp[k] * ldl + r0 + rr];
    }
    __syncthreads();
    for (int rr = warp; rr < tr; rr += TW_WARPS) {
      double xv[NR], acc[NR];
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int k = lane + 32 * u;
        xv[u] = k < b ? tile[k * TCP + rr] : 0.0;
        acc[u] = 0.0;
      }
      for (int k = 0; k < b; ++k) {
        const double xk = lane_pick(xv, k);
        const double* lk = lt + k * b;
#pragma unroll
        for (int u = 0; u < NR; ++u) {
          const int j = lane + 32 * u;
          if (j <= k) acc[u] = fma(xk, lk[j], acc[u]);
        }
      }
      double* o = out + (r0 + rr) * ldo;
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int j = lane + 32 * u;
        if (j < b) o[j] = acc[u];
      }
    }
    __syncthreads();
  }
}

// Block-row finish (see blockrow_kernel): columns [0, col0) permuted by the
// GEPP order, [col0, col0+b) from D, [col0+b, n) eliminated.
template <int NR>
__global__ void __launch_bounds__(TW_WARPS * 32) blockrow_w_kernel(double* A, int64_t lda, int64_t col0, int b,
                                                                  int64_t n, const double* __restrict__ D,
                                                                  const int32_t* gperm, int64_t* p, DevState* st) {
  extern __shared__ __align__(16) double sm[];
  double* lc = sm;                       // lc[k*b + i] = L11[i][k] (column k contiguous)
  double* tile = sm + b * b;             // b x TCP
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
  for (int64_t c0 = (int64_t)blockIdx.x * TC; c0 < n; c0 += (int64_t)gridDim.x * TC) {
    const int tc = (int)min((int64_t)TC, n - c0);
    // stage: rows in final GEPP order (L part and trailing part), D for the diagonal block
    for (int e = t; e < b * TC; e += blockDim.x) {
      const int i = e / TC, cc = e % TC;
      if (cc >= tc) continue;
      const int64_t j = c0 + cc;
      tile[i * TCP + cc] = (j >= col0 && j < col0 + b) ? D[i * b + (j - col0)] : A[(col0 + s_gp[i]) * lda + j];
    }
    __syncthreads();
    for (int cc = warp; cc < tc; cc += TW_WARPS) {
      const int64_t j = c0 + cc;
      if (j < col0 + b) continue;                      // L part / diagonal block: data movement only
      double x[NR];
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int i = lane + 32 * u;
        x[u] = i < b ? tile[i * TCP + cc] : 0.0;
        mx = fmax(mx, fabs(x[u]));
      }
      for (int k = 0; k + 1 < b; ++k) {
        const double xk = lane_pick(x, k);
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
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int i = lane + 32 * u;
        if (i < b) tile[i * TCP + cc] = x[u];
      }
    }
    __syncthreads();
    for (int e = t; e < b * TC; e += blockDim.x) {
      const int i = e / TC, cc = e % TC;
      if (cc < tc) A[(col0 + i) * lda + c0 + cc] = tile[i * TCP + cc];
    }
    __syncthreads();
  }
  const double m = block_max(mx, red);
  if (t == 0 && m > 0.0) atomic_max_abs(&st->finish_max, m);
}
