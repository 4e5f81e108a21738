// CALU_PRRP: tournament pivoting over a binary tree of strong RRQRs
// (tournament.py:155-217, 237-296) on the device.
//
// Rows stay in PHYSICAL slots; the factorization's logical row order of the
// trailing region is kept in pos2row (logical position -> physical row).
// Per panel only the b pivot rows move (into slots col0..col0+b, in selection
// order) and the rows they displace take the vacated slots, so the stable
// partition "[pivots, rest ascending]" (tournament.py:214-215) costs O(b) row
// moves instead of O(rows).  Leaves are contiguous LOGICAL blocks
// (tournament.py:64-88); every node is the same cluster QRCP engine fed with
// an index list.  L21 is produced in logical order and scattered to physical
// slots for the Schur update.  Once a panel is finished its rows sit at
// slots == logical positions, so the factors need no final gather (m == n).
#pragma once
#include "lsolve.cuh"

// node input rows for a merge level: lpos_in[node][0..2b) = [left child's
// candidates, right child's candidates] (panel-relative logical positions),
// rowidx = physical rows.  A child that was rank deficient passes fewer than
// b candidates (tournament.py:131-137): the members then close up and the
// unused tail is dead (-1: a zero row, never selected); live_out = members.
__global__ void calu_merge_inputs_kernel(const int32_t* cands, const int32_t* ccnt, int b, int nchild,
                                         int32_t* lpos_in, int64_t* rowidx, int32_t* live_out,
                                         const int64_t* pos2row, int64_t col0, int stride, const DevState* st) {
  if (prrp_failed(st)) return;     // the children may not have run: their outputs are not indices
  const int node = blockIdx.x;
  const int cl = ccnt[2 * node];
  const int cr = 2 * node + 1 < nchild ? ccnt[2 * node + 1] : 0;
  for (int t = threadIdx.x; t < 2 * b; t += blockDim.x) {
    int32_t lp = -1;
    if (t < cl) lp = cands[(2 * node) * b + t];
    else if (t < cl + cr) lp = cands[(2 * node + 1) * b + (t - cl)];
    lpos_in[node * stride + t] = lp;
    rowidx[node * stride + t] = lp >= 0 ? pos2row[col0 + lp] : -1;
  }
  if (threadIdx.x == 0) live_out[node] = cl + cr;
}

// selected candidates of each node: cands_out[node][q] = lpos(node, perm[q]),
// q < cnt_out[node] = wants[node] (b, fewer after a rank-deficient retry, or
// the members of a merge node that passed them through).
// Leaves (lpos_in == nullptr): lpos(node, j) = leaf_lo[node] + j.
__global__ void calu_select_kernel(const int32_t* const* perms, const int32_t* lpos_in, const int64_t* leaf_lo,
                                   int b, const int32_t* wants, const int32_t* lives, int merge, int32_t* cands_out,
                                   int32_t* cnt_out, int stride, const DevState* st) {
  if (prrp_failed(st)) return;
  const int node = blockIdx.x;
  const int32_t* perm = perms[node];
  const int cnt = min(wants[node], b);
  for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
    const int32_t j = perm[q];
    cands_out[node * b + q] = lpos_in ? lpos_in[node * stride + j] : (int32_t)(leaf_lo[node] + j);
  }
  if (threadIdx.x == 0) cnt_out[node] = cnt;
  (void)lives;
  (void)merge;
}

// Reorder the trailing region [col0, col0+rows) after the tournament.
//   order_mode 0 ("tournament"): new logical order = [pivots (selection
//     order), remaining positions ascending]                (tournament.py:214-215)
//   order_mode 1 ("single node"): new logical order = the node's own full
//     QRCP order perm_full[pos] (tournament.py:176-177)
// Physically the pivots move to slots col0..col0+b-1, displaced rows take
// the vacated slots.  Outputs: new pos2row, moved list (dst slot, src slot
// relative to col0) for permute_kernel, log2phys[t] = physical slot of
// logical position b+t (for scattering L21).  One block.
__global__ void __launch_bounds__(1024) calu_reorder_kernel(const int32_t* pivots, const int32_t* pivot_cnt,
                                                            const int32_t* perm_full, int order_mode, int b,
                                                            int64_t rows, int64_t col0, int64_t* pos2row,
                                                            int64_t* scratch /* 3*rows */, int32_t* moved,
                                                            int32_t* moved_cnt, int32_t* log2phys, DevState* st,
                                                            int panel) {
  __shared__ int s_cnt[33];
  __shared__ int64_t pv_slot[PRRP_MAXH], vsl[PRRP_MAXH];
  __shared__ int dsl[PRRP_MAXH], s_np, s_nd;
  if (prrp_failed(st)) return;
  // the tournament supplied fewer than b independent rows (tournament.py:210-213)
  if (order_mode == 0 && *pivot_cnt < b) {
    if (threadIdx.x == 0) prrp_set_error(st, PRRP_ERR_RANK_DEFICIENT, panel, *pivot_cnt, -1, 0.0);
    return;
  }
  const int t = threadIdx.x, T = blockDim.x;
  int64_t* oldp = scratch;                 // old pos2row (relative slots)
  int64_t* flag = scratch + rows;          // per logical position: pivot rank + 1, else 0
  int64_t* slot_pivot = scratch + 2 * rows;  // per relative slot: 1 if it holds a pivot row
  for (int64_t i = t; i < rows; i += T) {
    oldp[i] = pos2row[col0 + i] - col0;
    flag[i] = 0;
    slot_pivot[i] = 0;
  }
  __syncthreads();
  // pivots as logical positions
  for (int q = t; q < b; q += T) {
    const int32_t lp = order_mode == 0 ? pivots[q] : perm_full[q];
    flag[lp] = q + 1;
    pv_slot[q] = oldp[lp];
    slot_pivot[oldp[lp]] = 1;
  }
  __syncthreads();
  // displaced rows: slots < b not holding a pivot (increasing); vacated slots:
  // pivot rows' slots >= b (increasing); paired in that order (deterministic).
  // Ranks by counting (b <= 128 threads, O(b) each).
  if (t < b) {
    const int64_t sv = pv_slot[t];
    if (sv >= b) {
      int rk = 0;
      for (int q = 0; q < b; ++q) rk += pv_slot[q] >= b && pv_slot[q] < sv;
      vsl[rk] = sv;
    }
    if (!slot_pivot[t]) {
      int rk = 0;
      for (int q = 0; q < t; ++q) rk += !slot_pivot[q];
      dsl[rk] = t;
    }
  }
  // pivot moves (slot q <- src) in q order: compaction by counting
  if (t < b) {
    const bool mv = pv_slot[t] != t;
    if (mv) {
      int rk = 0;
      for (int q = 0; q < t; ++q) rk += pv_slot[q] != q;
      moved[2 * rk] = t;
      moved[2 * rk + 1] = (int32_t)pv_slot[t];
    }
  }
  if (t == 0) {
    int np = 0, nd = 0;
    for (int q = 0; q < b; ++q) np += pv_slot[q] != q;
    for (int q = 0; q < b; ++q) nd += !slot_pivot[q];     // = number of vacated slots
    s_np = np;
    s_nd = nd;
  }
  __syncthreads();
  {
    const int nd = s_nd;
    if (t < nd) {
      moved[2 * (s_np + t)] = (int32_t)vsl[t];
      moved[2 * (s_np + t) + 1] = dsl[t];
      // the row that was in slot dsl[t] now lives in vsl[t]
      slot_pivot[dsl[t]] = -(vsl[t] + 2);
    }
    if (t == 0) {
      st->moved = s_np + nd;
      if (moved_cnt) *moved_cnt = s_np + nd;
    }
  }
  __syncthreads();
  // new logical order
  if (order_mode == 1) {
    for (int64_t i = t; i < rows; i += T) {
      const int32_t lp = perm_full[i];
      int64_t s = oldp[lp];
      if (i < b) s = i;
      else if (s < b) s = -slot_pivot[s] - 2;
      pos2row[col0 + i] = col0 + s;
      if (i >= b) log2phys[i - b] = (int32_t)s;
    }
    return;
  }
  // order_mode 0: pivots first, then non-pivots by ascending old logical position
  for (int q = t; q < b; q += T) pos2row[col0 + q] = col0 + q;
  // block-wide exclusive scan over non-pivot flags, in chunks
  const int64_t per_t = (rows + T - 1) / T;
  const int64_t lo = t * per_t, hi = min(rows, lo + per_t);
  int cnt = 0;
  for (int64_t i = lo; i < hi; ++i) cnt += flag[i] == 0;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((t & 31) >= o) incl += y;
  }
  if ((t & 31) == 31) s_cnt[t >> 5] = incl;
  __syncthreads();
  if (t < 32) {
    const int nw = (T + 31) >> 5;
    int v = t < nw ? s_cnt[t] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (t >= o) v += y;
    }
    s_cnt[t] = v;
  }
  __syncthreads();
  int64_t np = b + incl - cnt + ((t >> 5) ? s_cnt[(t >> 5) - 1] : 0);
  for (int64_t i = lo; i < hi; ++i) {
    if (flag[i] != 0) continue;
    int64_t s = oldp[i];
    if (s < b) s = -slot_pivot[s] - 2;
    pos2row[col0 + np] = col0 + s;
    log2phys[np - b] = (int32_t)s;
    ++np;
  }
}

// R12 of the unpivoted Householder QR of the permuted panel transpose
// (tournament.py:271; pivoted_qr.py:64-71): the reflectors are fixed by the
// b pivot columns (QR of A11^T, log `refl`), so every non-pivot column gets
// the same b reflector applications the full householder_qr performs on it.
// Warp per column; lanes own rows lane, lane+32, ...; output Rbuf[i*p + b + t]
// for logical position b + t (row pos2row[col0 + b + t]).
template <int NR>
__global__ void __launch_bounds__(256) calu_apply_refl_kernel(const double* A, int64_t lda, int64_t col0, int b,
                                                              int64_t rows, const int64_t* pos2row,
                                                              const double* refl, double* Rbuf, DevState* st) {
  extern __shared__ __align__(16) double rf[];    // b x (b+1)
  if (prrp_failed(st)) return;
  for (int e = threadIdx.x; e < b * (b + 1); e += blockDim.x) rf[e] = refl[e];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t ncol = rows - b;
  for (int64_t t = (int64_t)blockIdx.x * nw + warp; t < ncol; t += (int64_t)gridDim.x * nw) {
    const int64_t row = pos2row[col0 + b + t];
    const double* src = A + row * lda + col0;
    double x[NR];
#pragma unroll
    for (int u = 0; u < NR; ++u) {
      const int i = lane + 32 * u;
      x[u] = i < b ? src[i] : 0.0;
    }
    for (int k = 0; k < b; ++k) {
      const double* v = rf + k * (b + 1);
      const double beta = v[b];
      if (beta == 0.0) continue;          // skipped reflector (pivoted_qr.py:47-54)
      double d = 0.0;
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int i = lane + 32 * u;
        if (i >= k && i < b) d = fma(v[i], x[u], d);
      }
      for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      const double w = mul_rn(beta, d);
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int i = lane + 32 * u;
        if (i >= k && i < b) x[u] = sub_rn(x[u], mul_rn(v[i], w));
      }
    }
#pragma unroll
    for (int u = 0; u < NR; ++u) {
      const int i = lane + 32 * u;
      if (i < b) Rbuf[(int64_t)i * rows + b + t] = x[u];
    }
  }
}

// copy R11 (b x b, row stride pb) of a small QR into the leading block of Rbuf (stride p)
__global__ void calu_copy_r11_kernel(const double* Rsmall, int b, double* Rbuf, int64_t p) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < b * b; e += gridDim.x * blockDim.x) {
    const int i = e / b, q = e % b;
    Rbuf[(int64_t)i * p + q] = Rsmall[(int64_t)i * b + q];
  }
}

// L21 (logical order, column-major ldl) -> physical slot order (column-major ldl2)
__global__ void calu_scatter_l21_kernel(const double* Lsrc, int64_t ldl, const int32_t* log2phys, int64_t M, int b,
                                        int64_t bslot, double* Ldst, int64_t ldd, const DevState* st) {
  if (prrp_failed(st)) return;     // the reorder that writes log2phys may have been skipped
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M * b; e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e / M);
    const int64_t t = e % M;
    Ldst[(int64_t)k * ldd + (log2phys[t] - bslot)] = Lsrc[(int64_t)k * ldl + t];
  }
}

// panel statistics for a tournament panel: multiplier max from the trsm
// candidates, swap count = sum over the tree's nodes
__global__ void calu_stats_kernel(const double* cand, int ncand, const int32_t* node_swaps, int nnodes,
                                  int32_t* swaps_dev, int panel, DevState* st) {
  __shared__ double red[40];
  if (prrp_failed(st)) return;
  double mx = -1.0;
  for (int i = threadIdx.x; i < ncand; i += blockDim.x) mx = fmax(mx, cand[i]);
  mx = block_max(mx, red);
  if (threadIdx.x == 0) {
    if (ncand > 0) atomic_max_abs(&st->pmm, mx);
    int s = 0;
    for (int i = 0; i < nnodes; ++i) s += node_swaps[i];
    swaps_dev[panel] = s;
  }
}

// m > n: rows n..m-1 are the unfinished tail; gather them into logical order
__global__ void calu_tail_gather_kernel(const double* A, int64_t lda, int64_t n, const int64_t* pos2row, int64_t m,
                                        double* tmp, const int64_t* porig, int64_t* ptmp) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (m - n) * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n, c = e % n;
    tmp[e] = A[pos2row[n + r] * lda + c];
    if (c == 0) ptmp[r] = porig[pos2row[n + r]];
  }
}

// leaf_lo[i] = first logical row of leaf i (contiguous blocks, first `extra`
// blocks one row larger: tournament.py:64-73) -- written on the device so the
// panel loop never waits for a pageable host copy
__global__ void calu_leaf_lo_kernel(int64_t* leaf_lo, int64_t p_eff, int64_t base, int64_t extra) {
  const int64_t i = threadIdx.x;
  for (int64_t j = i; j < p_eff; j += blockDim.x) leaf_lo[j] = j * base + min(j, extra);
}

// A21 of the permuted panel, transposed: out[k * ldo + t] = A[rowof[t], col0 + k]
// for t < ncol, k < b (32 rows per block through a padded shared tile)
__global__ void __launch_bounds__(256) calu_gather_t_kernel(const double* A, int64_t lda, int64_t col0, int b,
                                                           int64_t ncol, const int64_t* rowof, double* out,
                                                           int64_t ldo, const DevState* st) {
  if (prrp_failed(st)) return;
  extern __shared__ double tile[];   // b x 33
  const int64_t t0 = (int64_t)blockIdx.x * 32;
  const int nt = (int)min((int64_t)32, ncol - t0);
  for (int e = threadIdx.x; e < 32 * b; e += blockDim.x) {
    const int tl = e / b, k = e % b;
    if (tl < nt) tile[k * 33 + tl] = A[rowof[t0 + tl] * lda + col0 + k];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * b; e += blockDim.x) {
    const int k = e / 32, tl = e % 32;
    if (tl < nt) out[(int64_t)k * ldo + t0 + tl] = tile[k * 33 + tl];
  }
}

// L = -Q^T (column-major b x b) of a logged unpivoted QR, Q^T = H_{b-1} ... H_0:
// the identity's columns are transformed by the reflectors in log order.  A
// team of 8 threads owns a column (thread q keeps rows 8u + q, 16 values for
// b = 128), 16 columns per 128-thread CTA, ceil(b / 16) CTAs, so a reflector
// step is 2 x 16 FMAs and three shuffles per thread instead of a 128-row
// pass (the two-threads-per-column single-CTA form took 0.28 ms per panel
// on the CALU critical path).
// Reflector log: refl[k*(b+1) + i] = v_i (zero for i < k),
// refl[k*(b+1) + b] = beta (0: step skipped).
__global__ void __launch_bounds__(128) calu_form_negqt_kernel(const double* refl, int b, double* L) {
  extern __shared__ __align__(16) double rf[];   // b x (b + 1)
  for (int e0 = threadIdx.x; e0 < b * (b + 1); e0 += 8 * blockDim.x) {   // 8 independent loads in flight
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      v[u] = e < b * (b + 1) ? refl[e] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < b * (b + 1)) rf[e] = v[u];
    }
  }
  __syncthreads();
  const int j = blockIdx.x * 16 + (threadIdx.x >> 3), q = threadIdx.x & 7;
  const bool on = j < b;
  double m[PRRP_MAXH / 8];
#pragma unroll
  for (int u = 0; u < PRRP_MAXH / 8; ++u) m[u] = (on && 8 * u + q == j) ? 1.0 : 0.0;
  const int nu = (b + 7) >> 3;
  for (int k = 0; k < b; ++k) {
    const double* v = rf + k * (b + 1);
    const double beta = v[b];
    if (beta == 0.0) continue;                    // uniform
    const int u0 = k >> 3;                        // v is zero above row k
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int u = 0; u < PRRP_MAXH / 8; ++u) {
      if (u >= u0 && u < nu) {
        const int i = 8 * u + q;
        const double vi = i < b ? v[i] : 0.0;
        if (u & 1) d1 = fma(vi, m[u], d1);
        else d0 = fma(vi, m[u], d0);
      }
    }
    double dot = d0 + d1;
    dot += __shfl_xor_sync(0xffffffffu, dot, 1);
    dot += __shfl_xor_sync(0xffffffffu, dot, 2);
    dot += __shfl_xor_sync(0xffffffffu, dot, 4);
    const double w = beta * dot;
#pragma unroll
    for (int u = 0; u < PRRP_MAXH / 8; ++u) {
      if (u >= u0 && u < nu) {
        const int i = 8 * u + q;
        const double vi = i < b ? v[i] : 0.0;
        m[u] = fma(-vi, w, m[u]);
      }
    }
  }
  if (on) {
#pragma unroll
    for (int u = 0; u < PRRP_MAXH / 8; ++u) {
      const int i = 8 * u + q;
      if (i < b) L[i + (int64_t)j * b] = -m[u];
    }
  }
}

// flat-tree node inputs: members = [the candidates (b, fewer after a
// rank-deficient node), block rows lo .. lo+len), dead rows after them
__global__ void calu_flat_inputs_kernel(const int32_t* cands, const int32_t* ccnt, int b, int64_t lo, int len,
                                        int32_t* lpos_in, int64_t* rowidx, int32_t* live_out,
                                        const int64_t* pos2row, int64_t col0, const DevState* st) {
  if (prrp_failed(st)) return;
  const int c = ccnt[0];
  for (int t = threadIdx.x; t < b + len; t += blockDim.x) {
    int32_t lp = -1;
    if (t < c) lp = cands[t];
    else if (t < c + len) lp = (int32_t)(lo + (t - c));
    lpos_in[t] = lp;
    rowidx[t] = lp >= 0 ? pos2row[col0 + lp] : -1;
  }
  if (threadIdx.x == 0) live_out[0] = c + len;
}

// The unpivoted QR of the permuted panel (tournament.py:271) comes from the
// tournament's ROOT node when that node ran its QRCP: the root's first b
// pivot columns are the winners in selection order -- the columns of A11^T
// -- and a Householder reflector depends only on its own pivot column, so the
// root's leading R block and its first b logged reflectors are exactly the
// QR of A11^T (after swap-loop interchanges the root's R and log were
// recomputed from scratch in the final order).  Copies them, and sets
// final_live = 0 so the separate final-QR launch returns at once; a root
// that passed its members through (live <= b) leaves final_live large and
// that launch runs.
__global__ void calu_root_qr_kernel(const int32_t* root_live, int b, const double* root_R, int64_t root_p,
                                    const double* root_refl, double* Rsmall, double* refl, int32_t* final_live,
                                    const DevState* st) {
  if (prrp_failed(st)) return;
  const bool ran = *root_live > b;
  if (blockIdx.x == 0 && threadIdx.x == 0) *final_live = ran ? 0 : INT_MAX;
  if (!ran) return;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int e = t0; e < b * b; e += nt) {
    const int i = e / b, q = e - i * b;
    Rsmall[e] = root_R[(int64_t)i * root_p + q];
  }
  for (int e = t0; e < b * (b + 1); e += nt) refl[e] = root_refl[e];
}
