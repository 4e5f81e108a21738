// calu_factor: tournament pivoting with a GEPP selector (tournament.py:299-359).
//
// Per panel of width bj over the trailing rows [col0, m):
//   gepp_node_kernel   one CTA per tournament node of a level: gather the
//                      node's member rows (panel columns only), run partial
//                      pivoting on them (gepp.py:39-65: first max wins,
//                      true division, product then subtraction), pass on the
//                      rows chosen before the first zero pivot
//                      (tournament.py:142-150), add the node's flop charge
//                      (tournament.py:220-234, times 3 to stay integral).
//   gepp_tail_order_kernel  the new order of the trailing rows: the single
//                      node's own order, else [pivots, rest ascending]
//                      (tournament.py:176-177, 214-215); RankDeficient when
//                      the root passes on fewer than bj rows.
//   tail_gather/scatter_kernel  luprrp._permute_tail (luprrp.py:98-104) on
//                      whole rows of the packed L\U storage + the row order
//                      (only rows whose position changes move).
//   (GEPP of the block row: the LU_PRRP finish kernels, without the compose)
//   trsm_right_kernel  L21 = A21 U11^-1 in matcore.trsm_upper_right's order
//                      (matcore.py:97-113): x_ik = (a_ik - x_i0 u_0k - ... -
//                      x_i,k-1 u_k-1,k) / u_kk, products rounded before each
//                      subtraction; also writes L21 column-major for the
//                      trailing update and folds max|L21| into pmm.
//   (trailing update: the DMMA Schur kernels, bit-identical to rank_update)
#pragma once
#include "common.cuh"

#define GN_T 1024

struct GeppLevel {
  const double* panel;      // A + col0*lda + col0: rows x bj, row-major (lda)
  int64_t lda;
  int bj;
  int mode;                 // 0 binary leaves, 1 binary merge, 2 flat first block, 3 flat step
  int64_t rows;             // trailing rows of the panel
  int64_t p_eff;            // leaves: number of leaf blocks
  int64_t nprev;            // merges: number of child candidate lists
  int64_t lo, hi;           // flat: the block's row range
  const int32_t* cand_in;   // [node][bj] candidates (panel-relative rows)
  const int32_t* cnt_in;
  int32_t* cand_out;
  int32_t* cnt_out;
  int32_t* order_full;      // single-node level: the node's full order (rows entries)
  double* wscratch;         // global fallback for the node's working rows
  int32_t* oscratch;        // global fallback for the node's order
  unsigned long long* chg3; // this panel's 3x tournament charge
  int smem_bytes;           // dynamic shared memory of the launch
  DevState* st;
  int panel_no;
};

// Member q of node `node` (panel-relative row).
__device__ __forceinline__ int64_t gn_member(const GeppLevel& g, int node, int64_t q, int64_t lo, int ca) {
  if (g.mode == 0) return lo + q;
  if (g.mode == 2) return q;
  if (g.mode == 1) return q < ca ? g.cand_in[(2 * node) * g.bj + q] : g.cand_in[(2 * node + 1) * g.bj + (q - ca)];
  return q < ca ? g.cand_in[q] : g.lo + (q - ca);
}

// SM: the node's rows live in shared memory (the launch guarantees they fit),
// so the sweeps compile to LDS/STS instead of generic loads
template <bool SM>
__global__ void __launch_bounds__(GN_T, 1) gepp_node_kernel(GeppLevel g) {
  extern __shared__ __align__(16) double gsm[];
  __shared__ double s_best[32];
  __shared__ int s_bi[32];
  __shared__ int s_stop;
  if (prrp_failed(g.st)) return;
  const int node = blockIdx.x, t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int bj = g.bj;
  int64_t lo = 0, r = 0;
  int ca = 0;
  if (g.mode == 0) {
    const int64_t base = g.rows / g.p_eff, extra = g.rows % g.p_eff;
    lo = node * base + min((int64_t)node, extra);
    r = base + (node < extra ? 1 : 0);
  } else if (g.mode == 1) {
    if (2 * node + 1 >= g.nprev) {   // odd node promoted unmerged
      const int c = g.cnt_in[2 * node];
      for (int q = t; q < c; q += blockDim.x) g.cand_out[node * bj + q] = g.cand_in[(2 * node) * bj + q];
      if (t == 0) g.cnt_out[node] = c;
      return;
    }
    ca = g.cnt_in[2 * node];
    r = ca + g.cnt_in[2 * node + 1];
  } else if (g.mode == 2) {
    r = g.hi;
  } else {
    ca = g.cnt_in[0];
    r = ca + (g.hi - g.lo);
  }
  const bool single = g.order_full != nullptr;
  if (r <= bj) {   // too few rows to select from: all pass (tournament.py:129-130)
    for (int64_t q = t; q < r; q += blockDim.x) g.cand_out[node * bj + q] = (int32_t)gn_member(g, node, q, lo, ca);
    if (t == 0) g.cnt_out[node] = (int)r;
    return;
  }
  // working rows: shared memory when they fit, else the node's global slot.
  // Rows never move: ord[q] = the working row at position q (the swaps of
  // gepp.py:52-54 permute ord only).
  double* W;
  int32_t* ord;
  if (SM) {
    W = gsm;
    ord = reinterpret_cast<int32_t*>(gsm + (size_t)r * bj);
  } else {
    const int64_t off = g.mode == 0 ? lo : (g.mode == 1 ? (int64_t)node * 2 * bj : 0);
    W = g.wscratch + off * bj;
    ord = single ? g.order_full : g.oscratch + off;
  }
  const int R = (int)r;
  for (int q = t / bj; q < R; q += blockDim.x / bj) {   // blockDim.x % bj need not be 0: tail below
    const int j = t % bj;
    if (t < (int)(blockDim.x / bj) * bj) W[(int64_t)q * bj + j] = g.panel[gn_member(g, node, q, lo, ca) * g.lda + j];
  }
  for (int q = t; q < R; q += blockDim.x) ord[q] = q;
  if (t == 0) {
    s_stop = bj;
    atomicAdd(g.chg3, (unsigned long long)(3 * r * bj * bj - (int64_t)bj * bj * bj));
  }
  // thread (rg, tc): column tc of positions rg, rg + RG, ...
  const int CW = (bj + 31) & ~31, RG = blockDim.x / CW, tc = t % CW, rg = t / CW;
  __syncthreads();
  double best = -1.0;
  int bi = INT_MAX;
  if (tc == 0)
    for (int q = rg; q < R; q += RG) {
      const double v = fabs(W[(int64_t)q * bj]);
      if (v > best) { best = v; bi = q; }
    }
  for (int k = 0; k < bj; ++k) {
    // first maximum of |column k| over positions >= k (gepp.py:48-49); the
    // partials come from the previous step's update of column k
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(ob, oi, best, bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) { s_best[wid] = best; s_bi[wid] = bi; }
    __syncthreads();
    if (wid == 0) {
      const int nw = blockDim.x >> 5;
      best = lane < nw ? s_best[lane] : -1.0;
      bi = lane < nw ? s_bi[lane] : INT_MAX;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (better(ob, oi, best, bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) {
        if (!(best > 0.0)) {
          s_stop = k;   // SingularMatrix(column=k): keep the k rows chosen
        } else if (bi != k) {
          const int32_t o = ord[k];
          ord[k] = ord[bi];
          ord[bi] = o;
        }
      }
    }
    __syncthreads();
    if (s_stop == k) break;
    const int64_t pk = (int64_t)ord[k] * bj;
    const double d = W[pk + k];
    const double rd = __drcp_rn(d);
    const int j = tc;
    const bool active = j > k && j < bj;
    const double u = active ? W[pk + j] : 0.0;
    best = -1.0;
    bi = INT_MAX;
    const int wbase = tc - lane;   // the warp's first column (warp-uniform)
    if (wbase + 31 > k && wbase < bj) {
      const bool next = j == k + 1;
      // 32 positions at a time: lane s fetches row ord[q_s] and its
      // multiplier c[q_s, k] / c[k, k] once, the warp then sweeps the rows
      for (int q0 = k + 1 + rg; q0 < R; q0 += 32 * RG) {
        const int ql = q0 + lane * RG;
        int64_t pl = 0;
        double ll = 0.0;
        if (ql < R) {
          pl = (int64_t)ord[ql] * bj;
          ll = div_fast(W[pl + k], d, rd);
        }
        const int nq = min(32, (R - q0 + RG - 1) / RG);
        // four rows per pass: loads first, then the updates and stores
        for (int sq = 0; sq < nq; sq += 4) {
          int64_t p[4];
          double l[4], w[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            p[x] = __shfl_sync(0xffffffffu, pl, (sq + x) & 31);
            l[x] = __shfl_sync(0xffffffffu, ll, (sq + x) & 31);
          }
          if (active) {
#pragma unroll
            for (int x = 0; x < 4; ++x) w[x] = sq + x < nq ? W[p[x] + j] : 0.0;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              if (sq + x < nq) {
                const double v = sub_rn(w[x], mul_rn(l[x], u));   // c[q, j] - l * c[k, j]
                W[p[x] + j] = v;
                if (next) {
                  const double av = fabs(v);
                  if (av > best) { best = av; bi = q0 + (sq + x) * RG; }
                }
              }
            }
          }
        }
      }
    }
  }
  const int cnt = s_stop;
  for (int q = t; q < cnt; q += blockDim.x) g.cand_out[node * bj + q] = (int32_t)gn_member(g, node, ord[q], lo, ca);
  if (single && ord != g.order_full)
    for (int q = t; q < R; q += blockDim.x) g.order_full[q] = ord[q];
  if (t == 0) g.cnt_out[node] = cnt;
}

// New order of the trailing rows (perm_rel[i] = old position of the row that
// lands at position i) + the rank check.  One block.
__global__ void __launch_bounds__(1024) gepp_tail_order_kernel(const int32_t* piv, const int32_t* cnt, int bj,
                                                              int64_t rows, const int32_t* order_full,
                                                              int32_t* mark, int32_t* perm_rel, DevState* st,
                                                              int panel) {
  __shared__ int s_w[32];
  __shared__ int64_t s_run;
  if (prrp_failed(st)) return;
  const int c = *cnt;
  if (c < bj) {
    if (threadIdx.x == 0) prrp_set_error(st, PRRP_ERR_RANK_DEFICIENT, panel, c, -1, 0.0);
    return;
  }
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  if (order_full) {
    for (int64_t i = t; i < rows; i += blockDim.x) perm_rel[i] = order_full[i];
    return;
  }
  for (int64_t i = t; i < rows; i += blockDim.x) mark[i] = 0;
  __syncthreads();
  for (int q = t; q < bj; q += blockDim.x) {
    mark[piv[q]] = 1;
    perm_rel[q] = piv[q];
  }
  if (t == 0) s_run = 0;
  __syncthreads();
  for (int64_t base = 0; base < rows; base += blockDim.x) {
    const int64_t i = base + t;
    const bool keep = i < rows && mark[i] == 0;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_w[wid] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < wid) before += s_w[w];
      total += s_w[w];
    }
    if (keep) perm_rel[bj + s_run + before + __popc(bal & ((1u << lane) - 1u))] = (int32_t)i;
    __syncthreads();
    if (t == 0) s_run += total;
    __syncthreads();
  }
}

// Row moves of the trailing rows, columns [c0, c1): gather into buf (one row
// per block iteration), then scatter back; rows that keep their position are
// skipped.  The launch with c0 == 0 also moves the global row order.
__global__ void __launch_bounds__(256) tail_gather_kernel(const double* A, int64_t lda, int64_t row0, int64_t rows,
                                                          int64_t c0, int64_t c1, const int32_t* perm_rel,
                                                          const int64_t* p, double* buf, int64_t* pbuf,
                                                          const DevState* st) {
  if (prrp_failed(st)) return;
  const int64_t w = c1 - c0;
  for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
    const int64_t src = perm_rel[i];
    if (src == i) continue;
    const double* s = A + (row0 + src) * lda + c0;
    double* d = buf + i * w;
    for (int64_t j = threadIdx.x; j < w; j += blockDim.x) d[j] = s[j];
    if (pbuf && threadIdx.x == 0) pbuf[i] = p[row0 + src];
  }
}

__global__ void __launch_bounds__(256) tail_scatter_kernel(double* A, int64_t lda, int64_t row0, int64_t rows,
                                                           int64_t c0, int64_t c1, const int32_t* perm_rel,
                                                           int64_t* p, const double* buf, const int64_t* pbuf,
                                                           const DevState* st) {
  if (prrp_failed(st)) return;
  const int64_t w = c1 - c0;
  for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
    if (perm_rel[i] == i) continue;
    double* d = A + (row0 + i) * lda + c0;
    const double* s = buf + i * w;
    for (int64_t j = threadIdx.x; j < w; j += blockDim.x) d[j] = s[j];
    if (pbuf && threadIdx.x == 0) p[row0 + i] = pbuf[i];
  }
}

// L21 = A21 U11^-1, one row per thread.  A21: rows [r0, r0+M), columns
// [col0, col0+bj) of A; U11 from the packed diagonal block (upper part).
// Dynamic smem: bj*bj (U) + bj*blockDim.x (row values, column-interleaved).
__global__ void trsm_right_kernel(double* A, int64_t lda, int64_t col0, int bj, int64_t r0, int64_t M, double* Lcm,
                                  int64_t ldl, DevState* st) {
  extern __shared__ __align__(16) double tsm[];
  __shared__ double red[40];
  __shared__ double rinv[PRRP_MAXH];
  if (prrp_failed(st)) return;
  double* U = tsm;
  double* xs = tsm + (size_t)bj * bj;
  const int TW = blockDim.x, t = threadIdx.x;
  for (int e = t; e < bj * bj; e += TW) {
    const int i = e / bj, j = e - i * bj;
    U[e] = j >= i ? A[(col0 + i) * lda + col0 + j] : 0.0;
  }
  __syncthreads();
  for (int i = t; i < bj; i += TW) rinv[i] = __drcp_rn(U[i * bj + i]);
  __syncthreads();
  double mx = 0.0;
  for (int64_t base = (int64_t)blockIdx.x * TW; base < M; base += (int64_t)gridDim.x * TW) {
    const int64_t i = base + t;
    if (i < M) {
      double* row = A + (r0 + i) * lda + col0;
      for (int k = 0; k < bj; ++k) xs[k * TW + t] = row[k];
      // column j final, then pushed into columns > j: each x_ik still sees
      // its subtractions in increasing j before its division
      for (int jj = 0; jj < bj; ++jj) {
        const double x = div_fast(xs[jj * TW + t], U[jj * bj + jj], rinv[jj]);
        xs[jj * TW + t] = x;
        mx = fmax(mx, fabs(x));
        for (int k = jj + 1; k < bj; ++k) xs[k * TW + t] = sub_rn(xs[k * TW + t], mul_rn(x, U[jj * bj + k]));
      }
      for (int k = 0; k < bj; ++k) {
        const double x = xs[k * TW + t];
        row[k] = x;
        Lcm[(int64_t)k * ldl + i] = x;
      }
    }
  }
  const double m = block_max(mx, red);
  if (t == 0 && m > 0.0) atomic_max_abs(&st->pmm, m);
}

__global__ void widen_kernel(const int32_t* src, int64_t n, int64_t* dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// trsm_right_kernel for bj <= 64 with the row in registers (same arithmetic
// and order); U11 and the reciprocals of its diagonal in shared memory.
__global__ void __launch_bounds__(128) trsm_right_reg_kernel(double* A, int64_t lda, int64_t col0, int bj, int64_t r0,
                                                             int64_t M, double* Lcm, int64_t ldl, DevState* st) {
  __shared__ double U[64 * 64];
  __shared__ double rinv[64];
  __shared__ double red[40];
  if (prrp_failed(st)) return;
  const int t = threadIdx.x;
  for (int e = t; e < 64 * 64; e += blockDim.x) {
    const int i = e >> 6, j = e & 63;
    U[e] = (i < bj && j < bj && j >= i) ? A[(col0 + i) * lda + col0 + j] : 0.0;
  }
  __syncthreads();
  for (int i = t; i < 64; i += blockDim.x) rinv[i] = i < bj ? __drcp_rn(U[i * 64 + i]) : 0.0;
  __syncthreads();
  double mx = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + t; i < M; i += (int64_t)gridDim.x * blockDim.x) {
    double* row = A + (r0 + i) * lda + col0;
    double x[64];
#pragma unroll
    for (int k = 0; k < 64; ++k) x[k] = k < bj ? row[k] : 0.0;
#pragma unroll
    for (int jj = 0; jj < 64; ++jj) {
      if (jj < bj) {
        const double xj = div_fast(x[jj], U[jj * 64 + jj], rinv[jj]);
        x[jj] = xj;
        mx = fmax(mx, fabs(xj));
#pragma unroll
        for (int k = jj + 1; k < 64; ++k) x[k] = sub_rn(x[k], mul_rn(xj, U[jj * 64 + k]));
      }
    }
#pragma unroll
    for (int k = 0; k < 64; ++k)
      if (k < bj) {
        row[k] = x[k];
        Lcm[(int64_t)k * ldl + i] = x[k];
      }
  }
  const double m = block_max(mx, red);
  if (t == 0 && m > 0.0) atomic_max_abs(&st->pmm, m);
}
