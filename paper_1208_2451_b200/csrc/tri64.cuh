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
                                                              const double* fro, int tl, int ti,
                                                              const int32_t* live, int32_t* want) {
  extern __shared__ __align__(16) double sm[];
  double* r11 = sm;                                    // packed upper, bsel(bsel+1)/2
  double* tile = sm + ((bsel * (bsel + 1) / 2 + 1) & ~1);   // bsel x TTCP
  __shared__ double red_d[33];
  __shared__ long long red_l[33];
  __shared__ double rcp[PRRP_MAXH];
  if (prrp_failed(st) || (live && *live <= bsel)) return;
  load_r11(Rbuf, p, bsel, r11);
  __syncthreads();
  for (int i = threadIdx.x; i < bsel; i += blockDim.x) rcp[i] = __drcp_rn(r11[upk(i, i)]);
  if (blockIdx.x == 0 && threadIdx.x < 32)
    r11_checks_warp([&](int k) { return r11[upk(k, k)]; }, bsel, *fro, st, panel, true, tl, ti, want);
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

// trsm in 8-row chunks, four columns per warp (8 lanes per column, lane j
// holds rows j + 8q in registers).  Chunk k (rows 8k..8k+7, descending) is one register
// x[k] per lane: its 8x8 triangle is solved with a shuffle per step, which
// leaves the 8 solved values in registers of every lane of the group; rows of
// the chunks q < k then take their 8 product-then-subtract updates in step
// order with one 16-byte shared load per two multipliers.  Per element the
// operation sequence is exactly matcore.trsm_upper's (matcore.py:78-94):
// x_l -= u_li x_i for i = b-1 .. l+1, then x_l /= u_ll.  The divisions use the
// reciprocal form and are range-checked once per column group; a group that
// saw an out-of-range quotient is redone with IEEE divisions.
// R11 is padded to 8-row chunks with an identity tail (x = 0 rows): the padded
// updates are x_l - 0*0, which leave every x_l (including -0 and NaN) unchanged.
#define TC_WARPS 8
#define TC_T (TC_WARPS * 32)
#define TC_COLS (TC_WARPS * 4)
#define TC_UP 66   // padded R11 row pitch: 8 consecutive rows hit 8 distinct 16-byte bank groups

#ifndef TC_STAMP
#define TC_STAMP(k)
#endif

// NQ = 8-row chunks per column (8: b <= 64, 16: b <= 128), UP = padded R11 pitch
template <bool EXACT, int NQ, int UP>
__device__ __forceinline__ bool trsm_c_column(double (&x)[NQ], const double* __restrict__ us,
                                              const double* __restrict__ dg, const double* __restrict__ rc, int nk,
                                              int lane) {
  const int j = lane & 7;
  bool bad = false;
#pragma unroll 1
  for (int k = nk - 1; k >= 0; --k) {
    double v = x[0];
#pragma unroll
    for (int q = 1; q < NQ; ++q)
      if (q == k) v = x[q];
    const double2* ur = reinterpret_cast<const double2*>(us + (8 * k + j) * UP + 8 * k);
    const double2* dr = reinterpret_cast<const double2*>(dg + 8 * k);
    const double2* rr = reinterpret_cast<const double2*>(rc + 8 * k);
    double ut[8], dk[8], rk[8], xs[8];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const double2 a = ur[s], d = dr[s], r = rr[s];
      ut[2 * s] = a.x; ut[2 * s + 1] = a.y;
      dk[2 * s] = d.x; dk[2 * s + 1] = d.y;
      rk[2 * s] = r.x; rk[2 * s + 1] = r.y;
    }
#pragma unroll
    for (int s = 7; s >= 0; --s) {
      const double a = __shfl_sync(0xffffffffu, v, (lane & ~7) | s);
      double xi;
      if (EXACT) {
        xi = __ddiv_rn(a, dk[s]);
      } else {
        const double q0 = __dmul_rn(a, rk[s]);
        xi = fma(fma(-dk[s], q0, a), rk[s], q0);
        const double aq = fabs(xi);
        bad |= !(aq < 1e300 && (aq > 1e-290 || a == 0.0));
      }
      xs[s] = xi;
      if (j < s) v = sub_rn(v, mul_rn(ut[s], xi));
      else if (j == s) v = xi;
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (q == k) x[q] = v;
#pragma unroll
    for (int q = 0; q < NQ - 1; ++q) {
      if (q < k) {
        const double2* uq = reinterpret_cast<const double2*>(us + (8 * q + j) * UP + 8 * k);
        double u[8];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const double2 a = uq[s];
          u[2 * s] = a.x; u[2 * s + 1] = a.y;
        }
#pragma unroll
        for (int s = 7; s >= 0; --s) x[q] = sub_rn(x[q], mul_rn(u[s], xs[s]));
      }
    }
  }
  return bad;
}

template <int NQ, int UP>
__device__ __forceinline__ void trsm_c_body(double* us, double* dg, double* rc, double* red_d, long long* red_l,
                                            const double* __restrict__ Rbuf, int64_t p, int bsel, double* L21,
                                            int64_t ldl, double* cand, long long* cand_flat, DevState* st, int panel,
                                            const double* fro, int tl, int ti, int32_t* want) {
  constexpr int BW = 8 * NQ;   // padded R11 width
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nk = (bsel + 7) >> 3, bp = nk * 8;
  TC_STAMP(0);
  const double frov = (blockIdx.x == 0 && t < 32) ? *fro : 0.0;   // issued before the staging loads
  // padded R11: upper triangle of the first bsel rows, identity on [bsel, bp)
  for (int base = t; base < bp * BW; base += 8 * TC_T) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = base + u * TC_T, l = e / BW, i = e % BW;
      v[u] = (e < bp * BW && l < bsel && i >= l && i < bsel) ? Rbuf[(int64_t)l * p + i] : (l == i ? 1.0 : 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = base + u * TC_T, l = e / BW, i = e % BW;
      if (e < bp * BW) us[l * UP + i] = v[u];
    }
  }
  __syncthreads();
  TC_STAMP(4);
  for (int i = t; i < bp; i += TC_T) {
    dg[i] = us[i * UP + i];
    rc[i] = __drcp_rn(dg[i]);
  }
  if (blockIdx.x == 0 && t < 32)
    r11_checks_warp([&](int k) { return us[k * UP + k]; }, bsel, frov, st, panel, true, tl, ti, want);
  TC_STAMP(5);
  __syncthreads();
  TC_STAMP(1);
  const int64_t ncol = p - bsel;
  const int g = lane >> 3, j = lane & 7;
  double worst = -1.0;
  long long wflat = LLONG_MAX;
  for (int64_t cb = ((int64_t)blockIdx.x * TC_WARPS + warp) * 4; cb < ncol; cb += (int64_t)gridDim.x * TC_COLS) {
    const int64_t c = cb + g;
    const bool on = c < ncol;
    double x[NQ];
    auto load = [&] {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int row = j + 8 * q;
        x[q] = (on && row < bsel) ? Rbuf[(int64_t)row * p + bsel + c] : 0.0;
      }
    };
    load();
    if (__any_sync(0xffffffffu, trsm_c_column<false, NQ, UP>(x, us, dg, rc, nk, lane))) {
      load();
      trsm_c_column<true, NQ, UP>(x, us, dg, rc, nk, lane);
    }
    if (on) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
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
  TC_STAMP(2);
  reduce_worst(worst, wflat, red_d, red_l);
  if (t == 0) { cand[blockIdx.x] = worst; cand_flat[blockIdx.x] = wflat; }
  TC_STAMP(3);
}

__global__ void __launch_bounds__(TC_T) trsm_c_kernel(const double* __restrict__ Rbuf, int64_t p, int bsel,
                                                      double* L21, int64_t ldl, double* cand, long long* cand_flat,
                                                      DevState* st, int panel, const double* fro, int tl, int ti,
                                                      const int32_t* live, int32_t* want) {
  __shared__ __align__(16) double us[64 * TC_UP];
  __shared__ __align__(16) double dg[64], rc[64];
  __shared__ double red_d[33];
  __shared__ long long red_l[33];
  if (prrp_failed(st) || (live && *live <= bsel)) return;
  trsm_c_body<8, TC_UP>(us, dg, rc, red_d, red_l, Rbuf, p, bsel, L21, ldl, cand, cand_flat, st, panel, fro, tl, ti,
                        want);
}

// b in (64, 128]: 16 chunks per column, R11 (128 x TC_UP2) in dynamic shared memory
#define TC_UP2 130
constexpr size_t kTrsmC2Smem = (size_t)(128 * TC_UP2 + 2 * 128) * 8;
__global__ void __launch_bounds__(TC_T) trsm_c2_kernel(const double* __restrict__ Rbuf, int64_t p, int bsel,
                                                       double* L21, int64_t ldl, double* cand, long long* cand_flat,
                                                       DevState* st, int panel, const double* fro, int tl, int ti,
                                                       const int32_t* live, int32_t* want) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ double red_d[33];
  __shared__ long long red_l[33];
  if (prrp_failed(st) || (live && *live <= bsel)) return;
  trsm_c_body<16, TC_UP2>(dsm, dsm + 128 * TC_UP2, dsm + 128 * TC_UP2 + 128, red_d, red_l, Rbuf, p, bsel, L21, ldl,
                          cand, cand_flat, st, panel, fro, tl, ti, want);
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

// Block-row finish, thread per column (b a multiple of 8).  The warp-per-
// column form above keeps half its lanes idle (row i > k) and pays a shuffle
// per pivot step: 0.59 ms per panel at config 5 on the fin stream, which is
// close to the critical path there.  Here a thread owns one column of the
// block row in shared memory (tile[i][c], conflict free) and walks it
// LEFT-looking in blocks of 8 pivots: the 8 pivot rows of a block are
// finished in registers, then every row below receives the block's 8
// updates, eight rows at a time (eight independent chains per thread).  Per
// element the operation sequence is unchanged -- x_i -= l_ik x_k for k = 0, 1,
// ... in increasing order, product rounded, then subtracted (gepp.py:57-59)
// -- so the result and the running maximum (every intermediate value, the
// reference's observe_finish) are bit-identical to the warp-per-column
// kernel.  L11's strictly lower part is staged per pivot block:
// lt[off(kb) + (i - 8 kb) * 8 + kk] = L11[i][8 kb + kk], read as broadcasts.
#define BX_TC 128                     // columns (threads) per tile
__host__ __device__ inline int bx_off(int kb, int b) { return 8 * (kb * b - 4 * kb * (kb - 1)); }
__host__ __device__ inline size_t bx_smem(int b) {
  return ((size_t)bx_off(b / 8, b) + (size_t)b * BX_TC) * 8;
}
__global__ void __launch_bounds__(BX_TC) blockrow_x_kernel(double* A, int64_t lda, int64_t col0, int b, int64_t n,
                                                           const double* __restrict__ D, const int32_t* gperm,
                                                           int64_t* p, DevState* st, int64_t bl, int nr, int rk) {
  extern __shared__ __align__(16) double sm[];
  const int nkb = b >> 3;
  double* lt = sm;                                 // per-block strictly lower L11
  double* tile = sm + bx_off(nkb, b);              // b x BX_TC
  __shared__ int s_gp[PRRP_MAXH];
  __shared__ int64_t s_p[PRRP_MAXH];
  __shared__ double red[40];
  if (prrp_failed(st)) return;
  const int t = threadIdx.x;
  for (int i = t; i < b; i += blockDim.x) s_gp[i] = gperm[i];
  for (int kb = 0; kb < nkb; ++kb) {
    const int rows = b - 8 * kb;
    double* dst = lt + bx_off(kb, b);
    for (int e0 = t; e0 < rows * 8; e0 += 8 * blockDim.x) {      // 8 independent loads in flight
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        const int i = 8 * kb + e / 8, k = 8 * kb + (e & 7);
        v[u] = (e < rows * 8 && i > k) ? D[i * b + k] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        if (e < rows * 8) dst[e] = v[u];
      }
    }
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int i = t; i < b; i += blockDim.x) s_p[i] = p[col0 + s_gp[i]];
    __syncthreads();
    for (int i = t; i < b; i += blockDim.x) p[col0 + i] = s_p[i];
  }
  double mx = 0.0;
  for (int64_t c0 = (int64_t)blockIdx.x * BX_TC; c0 < n; c0 += (int64_t)gridDim.x * BX_TC) {
    const int tc = (int)min((int64_t)BX_TC, n - c0);
    // stage: rows in final GEPP order (L part and trailing part), D for the
    // diagonal block; thread = column, 8 independent row loads in flight
    if (t < tc) {
      const int64_t j = c0 + t;
      const int64_t g = nr == 1 ? j : ((j / bl) * nr + rk) * bl + j % bl;
      const bool diag = g >= col0 && g < col0 + b;
      for (int i0 = 0; i0 < b; i0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = diag ? D[(i0 + u) * b + (g - col0)] : A[(col0 + s_gp[i0 + u]) * lda + j];
#pragma unroll
        for (int u = 0; u < 8; ++u) tile[(i0 + u) * BX_TC + t] = v[u];
      }
    }
    __syncthreads();
    if (t < tc) {
      const int64_t j = c0 + t;
      const int64_t g = nr == 1 ? j : ((j / bl) * nr + rk) * bl + j % bl;
      if (g >= col0 + b) {                           // trailing column: eliminate
        double* col = tile + t;
        // eight running maxima (one per row chain: a single one would be a
        // dependency chain through every update), merged after the column;
        // a > m ? a : m ignores NaN like fmax (m starts at 0).  (Keeping them
        // as bit patterns on the integer pipe was measured no faster.)
        double m8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#define BX_MAX(m, a) { const double a_ = fabs(a); m = a_ > m ? a_ : m; }
        for (int i = 0; i < b; i += 8) {
#pragma unroll
          for (int r = 0; r < 8; ++r) BX_MAX(m8[r], col[(i + r) * BX_TC]);
        }
        for (int kb = 0; kb < nkb; ++kb) {
          const double* lb = lt + bx_off(kb, b);     // rows 8 kb .. b-1, 8 entries each
          double x[8];
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) x[kk] = col[(8 * kb + kk) * BX_TC];
          // the block's own rows
#pragma unroll
          for (int kk = 0; kk < 7; ++kk) {
#pragma unroll
            for (int ii = kk + 1; ii < 8; ++ii) {
              x[ii] = sub_rn(x[ii], mul_rn(lb[ii * 8 + kk], x[kk]));
              BX_MAX(m8[ii], x[ii]);
            }
          }
#pragma unroll
          for (int kk = 1; kk < 8; ++kk) col[(8 * kb + kk) * BX_TC] = x[kk];
          // the rows below, eight at a time (eight independent chains)
          for (int i0 = 8 * kb + 8; i0 < b; i0 += 8) {
            const double* l8 = lb + (i0 - 8 * kb) * 8;
            double v[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = col[(i0 + r) * BX_TC];
#pragma unroll
            for (int kk = 0; kk < 8; kk += 2) {
              double2 l2[8];
#pragma unroll
              for (int r = 0; r < 8; ++r) l2[r] = *reinterpret_cast<const double2*>(l8 + r * 8 + kk);
#pragma unroll
              for (int r = 0; r < 8; ++r) {
                v[r] = sub_rn(v[r], mul_rn(l2[r].x, x[kk]));
                BX_MAX(m8[r], v[r]);
              }
#pragma unroll
              for (int r = 0; r < 8; ++r) {
                v[r] = sub_rn(v[r], mul_rn(l2[r].y, x[kk + 1]));
                BX_MAX(m8[r], v[r]);
              }
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) col[(i0 + r) * BX_TC] = v[r];
          }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) mx = m8[r] > mx ? m8[r] : mx;
#undef BX_MAX
      }
    }
    __syncthreads();
    if (t < tc) {
      for (int i0 = 0; i0 < b; i0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = tile[(i0 + u) * BX_TC + t];
#pragma unroll
        for (int u = 0; u < 8; ++u) A[(col0 + i0 + u) * lda + c0 + t] = v[u];
      }
    }
    __syncthreads();
  }
  const double m = block_max(mx, red);
  if (t == 0 && m > 0.0) atomic_max_abs(&st->finish_max, m);
}

// Operands of the DMMA compose (launch_compose_w): Lneg[k][r] = -L21[r][gperm[k]]
// (column-major, ld), Bm = unit-lower L11 from the packed D (row-major b x b),
// and the output block zeroed (the Schur kernel computes out - Lneg Bm).
__global__ void compose_prep_kernel(const double* __restrict__ L21, int64_t ldl, int64_t M, int b,
                                    const double* __restrict__ D, const int32_t* __restrict__ gperm, double* Lneg,
                                    int64_t ld, double* Bm, double* out, int64_t ldo, const DevState* st) {
  if (prrp_failed(st)) return;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = t0; e < M * b; e += nt) {
    const int k = (int)(e / M);
    const int64_t r = e % M;
    Lneg[(int64_t)k * ld + r] = -L21[(int64_t)gperm[k] * ldl + r];
  }
  for (int64_t e = t0; e < M * b; e += nt) {
    const int64_t r = e / b;
    const int j = (int)(e % b);
    out[r * ldo + j] = 0.0;
  }
  for (int64_t e = t0; e < (int64_t)b * b; e += nt) {
    const int k = (int)(e / b), j = (int)(e % b);
    Bm[e] = k > j ? D[e] : (k == j ? 1.0 : 0.0);
  }
}

// Block-row finish (see blockrow_kernel): columns [0, col0) permuted by the
// GEPP order, [col0, col0+b) from D, [col0+b, n) eliminated.
// Columns are local indices c < n; their global index (which decides the L
// part / diagonal block / trailing role) is g = ((c / bl) nr + rk) bl + c % bl
// -- a column block-cyclic layout over nr ranks (rank rk, block bl); the
// single-GPU driver passes nr = 1, rk = 0 (g = c).
template <int NR>
__global__ void __launch_bounds__(TW_WARPS * 32) blockrow_w_kernel(double* A, int64_t lda, int64_t col0, int b,
                                                                  int64_t n, const double* __restrict__ D,
                                                                  const int32_t* gperm, int64_t* p, DevState* st,
                                                                  int64_t bl, int nr, int rk) {
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
      const int64_t g = nr == 1 ? j : ((j / bl) * nr + rk) * bl + j % bl;
      tile[i * TCP + cc] = (g >= col0 && g < col0 + b) ? D[i * b + (g - col0)] : A[(col0 + s_gp[i]) * lda + j];
    }
    __syncthreads();
    for (int cc = warp; cc < tc; cc += TW_WARPS) {
      const int64_t j = c0 + cc;
      const int64_t g = nr == 1 ? j : ((j / bl) * nr + rk) * bl + j % bl;
      if (g < col0 + b) continue;                      // L part / diagonal block: data movement only
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
