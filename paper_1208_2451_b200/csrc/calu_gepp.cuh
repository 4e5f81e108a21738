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
  // working rows: shared memory when they fit, else the node's global slot
  const size_t need = (size_t)r * bj * 8 + (size_t)r * 4;
  double* W;
  int32_t* ord;
  if (need <= (size_t)g.smem_bytes) {
    W = gsm;
    ord = reinterpret_cast<int32_t*>(gsm + (size_t)r * bj);
  } else {
    const int64_t off = g.mode == 0 ? lo : (g.mode == 1 ? (int64_t)node * 2 * bj : 0);
    W = g.wscratch + off * bj;
    ord = single ? g.order_full : g.oscratch + off;
  }
  for (int64_t e = t; e < r * bj; e += blockDim.x) {
    const int64_t q = e / bj;
    const int j = (int)(e - q * bj);
    W[e] = g.panel[gn_member(g, node, q, lo, ca) * g.lda + j];
  }
  for (int64_t q = t; q < r; q += blockDim.x) ord[q] = (int32_t)q;
  if (t == 0) {
    s_stop = bj;
    atomicAdd(g.chg3, (unsigned long long)(3 * r * bj * bj - (int64_t)bj * bj * bj));
  }
  __syncthreads();
  for (int k = 0; k < bj; ++k) {
    // first maximum of |W[q][k]|, q >= k (gepp.py:48-49)
    double best = -1.0;
    int bi = INT_MAX;
    for (int64_t q = k + t; q < r; q += blockDim.x) {
      const double v = fabs(W[q * bj + k]);
      if (v > best) { best = v; bi = (int)q; }
    }
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
        s_bi[0] = bi;
        if (best == 0.0) s_stop = k;   // SingularMatrix(column=k): keep the k rows chosen
      }
    }
    __syncthreads();
    if (s_stop == k) break;
    const int pv = s_bi[0];
    if (pv != k) {
      for (int j = t; j < bj; j += blockDim.x) {
        const double a = W[(int64_t)k * bj + j];
        W[(int64_t)k * bj + j] = W[(int64_t)pv * bj + j];
        W[(int64_t)pv * bj + j] = a;
      }
      if (t == 0) { const int32_t o = ord[k]; ord[k] = ord[pv]; ord[pv] = o; }
    }
    __syncthreads();
    const double d = W[(int64_t)k * bj + k];
    for (int64_t q = k + 1 + t; q < r; q += blockDim.x) W[q * bj + k] = div_rn(W[q * bj + k], d);
    __syncthreads();
    const int w = bj - k - 1;
    if (w > 0) {
      const int64_t tot = (r - k - 1) * w;
      for (int64_t e = t; e < tot; e += blockDim.x) {
        const int64_t q = k + 1 + e / w;
        const int j = k + 1 + (int)(e % w);
        W[q * bj + j] = sub_rn(W[q * bj + j], mul_rn(W[q * bj + k], W[(int64_t)k * bj + j]));
      }
    }
    __syncthreads();
  }
  const int cnt = s_stop;
  for (int q = t; q < cnt; q += blockDim.x) g.cand_out[node * bj + q] = (int32_t)gn_member(g, node, ord[q], lo, ca);
  if (single && ord != g.order_full)
    for (int64_t q = t; q < r; q += blockDim.x) g.order_full[q] = ord[q];
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
  if (prrp_failed(st)) return;
  double* U = tsm;
  double* xs = tsm + (size_t)bj * bj;
  const int TW = blockDim.x, t = threadIdx.x;
  for (int e = t; e < bj * bj; e += TW) {
    const int i = e / bj, j = e - i * bj;
    U[e] = j >= i ? A[(col0 + i) * lda + col0 + j] : 0.0;
  }
  __syncthreads();
  double mx = 0.0;
  for (int64_t base = (int64_t)blockIdx.x * TW; base < M; base += (int64_t)gridDim.x * TW) {
    const int64_t i = base + t;
    if (i < M) {
      double* row = A + (r0 + i) * lda + col0;
      for (int k = 0; k < bj; ++k) xs[k * TW + t] = row[k];
      for (int k = 0; k < bj; ++k) {
        double x = xs[k * TW + t];
        for (int j = 0; j < k; ++j) x = sub_rn(x, mul_rn(xs[j * TW + t], U[j * bj + k]));
        x = div_rn(x, U[k * bj + k]);
        xs[k * TW + t] = x;
        mx = fmax(mx, fabs(x));
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
