// Multiplier block L21 = (R11^-1 R12)^T, the strong-RRQR tau test and swap
// loop, and the partial-pivoting finish of the b x b diagonal block.
//
// Reference semantics:
//   matcore.trsm_upper      matcore.py:78-94   axpy back substitution from the
//                           last row, TRUE division x_i /= u_ii, then
//                           x_l -= u_li * x_i (product, then subtraction);
//                           exact-zero diagonal -> SingularFactor(index)
//   pivoted_qr._check_rank  pivoted_qr.py:101-105  |R[k,k]| < 2^-52 ||A||_F
//   pivoted_qr.strong_rrqr  pivoted_qr.py:113-147  while max|lt| > tau: swap
//                           the row-major first argmax (i, j) -> perm[i] <->
//                           perm[b+j], QR from scratch, re-check; cap
//                           ceil(2 b log p / log tau) + 10 (swap_cap :108-110)
//   gepp.gepp_factor        gepp.py:39-65   first-max pivot in column k,
//                           SingularMatrix(column) on an exact zero, true
//                           division, product-then-subtract rank-1 update,
//                           running max of the trailing block after each step
// Every operation above is reproduced element for element, so given the same
// R (resp. the same block) the outputs are bit-identical to the reference.
#pragma once
#include "panel.cuh"

#define TRSM_TW 128   // columns (threads) per trsm block

// packed upper triangle of R11, column q holds rows 0..q
__device__ __forceinline__ int upk(int i, int q) { return q * (q + 1) / 2 + i; }

__device__ void load_r11(const double* Rbuf, int64_t p, int bsel, double* r11) {
  // 8 independent loads in flight per thread (the loop is L2-latency bound)
  const int T = blockDim.x, tot = bsel * bsel;
  for (int base = threadIdx.x; base < tot; base += 8 * T) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * T;
      const int i = idx / bsel, q = idx - i * bsel;
      v[u] = (idx < tot && i <= q) ? Rbuf[(int64_t)i * p + q] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * T;
      const int i = idx / bsel, q = idx - i * bsel;
      if (idx < tot && i <= q) r11[upk(i, q)] = v[u];
    }
  }
}

// Rank check then singular-diagonal check (in the reference's order).
// Returns 0 when the block is usable.
__device__ int r11_checks(const double* r11, int bsel, double fro, DevState* st, int panel, bool report,
                          int tl = -1, int ti = -1) {
  for (int k = 0; k < bsel; ++k) {
    if (fabs(r11[upk(k, k)]) < PRRP_EPS * fro) {
      if (report) prrp_set_error(st, PRRP_ERR_RANK_DEFICIENT, panel, k, -1, 0.0, tl, ti);
      return 1;
    }
  }
  for (int i = bsel - 1; i >= 0; --i) {
    if (r11[upk(i, i)] == 0.0) {
      if (report) prrp_set_error(st, PRRP_ERR_SINGULAR_FACTOR, panel, i, -1, 0.0, tl, ti);
      return 1;
    }
  }
  return 0;
}

// r11_checks by one warp (ballots over the diagonal; same codes and indices):
// the first k with |r_kk| < eps*fro, else the last i with r_ii == 0.
// want != nullptr (a CALU tournament node, tournament.py:131-137): a rank
// failure is not an error; the node retries with want = the failing index,
// so it is recorded there (else want = bsel).
template <typename Diag>
__device__ int r11_checks_warp(Diag diag, int bsel, double fro, DevState* st, int panel, bool report, int tl = -1,
                               int ti = -1, int32_t* want = nullptr) {
  const int lane = threadIdx.x & 31;
  const double thr = PRRP_EPS * fro;
  int first_rank = -1, last_zero = -1;
  for (int k0 = 0; k0 < bsel; k0 += 32) {
    const int k = k0 + lane;
    const double d = k < bsel ? diag(k) : 1.0;
    const unsigned br = __ballot_sync(0xffffffffu, k < bsel && fabs(d) < thr);
    const unsigned bz = __ballot_sync(0xffffffffu, k < bsel && d == 0.0);
    if (br && first_rank < 0) first_rank = k0 + __ffs(br) - 1;
    if (bz) last_zero = k0 + 31 - __clz(bz);
  }
  if (first_rank >= 0) {
    if (report && lane == 0) {
      if (want) *want = first_rank;
      else prrp_set_error(st, PRRP_ERR_RANK_DEFICIENT, panel, first_rank, -1, 0.0, tl, ti);
    }
    return 1;
  }
  if (last_zero >= 0) {
    if (report && lane == 0) prrp_set_error(st, PRRP_ERR_SINGULAR_FACTOR, panel, last_zero, -1, 0.0, tl, ti);
    return 1;
  }
  if (report && lane == 0 && want) *want = bsel;
  return 0;
}

// Solve R11 x = R12[:, pos] for the positions [q0, q0 + blockDim.x) and write
// L21 (column-major, row pos - bsel).  Tracks the worst |x| with its
// row-major flat index in lt = R11^-1 R12 (bsel x (p - bsel)).
__device__ void trsm_tile(const double* Rbuf, int64_t p, int bsel, const double* r11, double* xs, int TW,
                          int64_t q0, double* L21, int64_t ldl, double& worst, long long& wflat) {
  const int t = threadIdx.x;
  const int64_t pos = q0 + t;
  const bool on = t < TW && pos < p;
  if (on)
    for (int i = 0; i < bsel; ++i) xs[i * TW + t] = Rbuf[(int64_t)i * p + pos];
  if (!on) return;
  for (int i = bsel - 1; i >= 0; --i) {
    const double xi = div_rn(xs[i * TW + t], r11[upk(i, i)]);
    xs[i * TW + t] = xi;
    const double* rc = r11 + upk(0, i);
    for (int l = 0; l < i; ++l) xs[l * TW + t] = sub_rn(xs[l * TW + t], mul_rn(rc[l], xi));
  }
  const int64_t jj = pos - bsel;
  const int64_t ncol = p - bsel;
  for (int i = 0; i < bsel; ++i) {
    const double x = xs[i * TW + t];
    L21[(int64_t)i * ldl + jj] = x;
    const double ax = fabs(x);
    const long long fl = (long long)i * ncol + jj;
    if (ax > worst || (ax == worst && fl < wflat)) { worst = ax; wflat = fl; }
  }
}

__device__ void reduce_worst(double& worst, long long& wflat, double* red_d, long long* red_l) {
  for (int o = 16; o; o >>= 1) {
    const double ow = __shfl_xor_sync(0xffffffffu, worst, o);
    const long long of = __shfl_xor_sync(0xffffffffu, wflat, o);
    if (ow > worst || (ow == worst && of < wflat)) { worst = ow; wflat = of; }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (l == 0) { red_d[w] = worst; red_l[w] = wflat; }
  __syncthreads();
  if (w == 0) {
    worst = l < nw ? red_d[l] : -1.0;
    wflat = l < nw ? red_l[l] : LLONG_MAX;
    for (int o = 16; o; o >>= 1) {
      const double ow = __shfl_xor_sync(0xffffffffu, worst, o);
      const long long of = __shfl_xor_sync(0xffffffffu, wflat, o);
      if (ow > worst || (ow == worst && of < wflat)) { worst = ow; wflat = of; }
    }
    if (l == 0) { red_d[32] = worst; red_l[32] = wflat; }
  }
  __syncthreads();
  worst = red_d[32];
  wflat = red_l[32];
}

// All-SM multiplier kernel (fast path): block b solves positions
// [bsel + b*TW, ...).  Block 0 performs the rank / singular checks.
__global__ void __launch_bounds__(TRSM_TW) trsm_kernel(const double* Rbuf, int64_t p, int bsel, double* L21,
                                                      int64_t ldl, double* cand, long long* cand_flat,
                                                      DevState* st, int panel, const double* fro, int tl, int ti,
                                                      const int32_t* live, int32_t* want) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red_d[33];
  __shared__ long long red_l[33];
  if (prrp_failed(st) || (live && *live <= bsel)) return;
  double* r11 = sm;
  double* xs = sm + bsel * (bsel + 1) / 2;
  load_r11(Rbuf, p, bsel, r11);
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x < 32)
    r11_checks_warp([&](int k) { return r11[upk(k, k)]; }, bsel, *fro, st, panel, true, tl, ti, want);
  double worst = -1.0;
  long long wflat = LLONG_MAX;
  trsm_tile(Rbuf, p, bsel, r11, xs, blockDim.x, bsel + (int64_t)blockIdx.x * blockDim.x, L21, ldl, worst, wflat);
  reduce_worst(worst, wflat, red_d, red_l);
  if (threadIdx.x == 0) { cand[blockIdx.x] = worst; cand_flat[blockIdx.x] = wflat; }
}

// ---------------------------------------------------------------------------
// GEPP of the b x b diagonal block (gepp.py:39-65 restricted to the block's
// columns; the trailing columns of the block row are finished per column by
// blockrow_kernel with the same multipliers and pivots).
// src row q of the block: src + (rowmap ? rowmap[q] : q) * ld, b entries.
// Output: D (b x b row-major packed L\U), piv[k] (row exchanged at step k),
// gperm (final order of the block rows).  Single CTA.
// ---------------------------------------------------------------------------
__device__ void gepp_diag(const double* src, int64_t ld, const int32_t* rowmap, int b, double* c /* smem b*b */,
                          double* D, int32_t* piv, int32_t* gperm, DevState* st, int panel, double* red) {
  // thread j owns column j for the swaps and the rank-1 updates (consecutive
  // threads touch consecutive words: no bank conflicts, no index division);
  // warp 0 runs the first-max pivot search of column k.
  const int t = threadIdx.x, T = blockDim.x;
  const int bp = b + 1;   // odd pitch: row and column walks are both bank-conflict free
  __shared__ int s_piv;
  __shared__ double s_colmax;
  __shared__ int s_gp[PRRP_MAXH];
  double mx = 0.0;
  for (int i = 0; i < b; ++i) {
    const int64_t row = rowmap ? rowmap[i] : i;
    for (int j = t; j < b; j += T) {
      const double v = src[row * ld + j];
      c[i * bp + j] = v;
      mx = fmax(mx, fabs(v));
    }
  }
  if (t < b) s_gp[t] = t;
  __syncthreads();
  for (int k = 0; k < b; ++k) {
    if (t < 32) {
      double best = -1.0;
      int bi = INT_MAX;
      for (int i = k + t; i < b; i += 32) {
        const double v = fabs(c[i * bp + k]);
        if (v > best) { best = v; bi = i; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (t == 0) { s_piv = bi; s_colmax = best; }
    }
    __syncthreads();
    const int pv = s_piv;
    if (s_colmax == 0.0) {
      if (t == 0) prrp_set_error(st, PRRP_ERR_SINGULAR_MATRIX, panel, -1, k, 0.0);
      return;
    }
    if (pv != k) {
      for (int j = t; j < b; j += T) {
        const double x = c[k * bp + j];
        c[k * bp + j] = c[pv * bp + j];
        c[pv * bp + j] = x;
      }
      if (t == 0) { const int g = s_gp[k]; s_gp[k] = s_gp[pv]; s_gp[pv] = g; }
    }
    if (t == 0) piv[k] = pv;
    __syncthreads();
    if (k + 1 < b) {
      const double ckk = c[k * bp + k];
      const double yk = __drcp_rn(ckk);
      for (int i = k + 1 + t; i < b; i += T) c[i * bp + k] = div_fast(c[i * bp + k], ckk, yk);
      __syncthreads();
      // column j = k + 1 + (t % W) and every H-th 8-row chunk below the pivot,
      // W = min(T, 128) column threads x H = T / W row groups (each element is
      // updated once per step whatever the split: same bits)
      const int W = T < 128 ? T : 128, H = T / W;
      const int tj = t % W, th = t / W;
      if (th < H) {
        for (int j = k + 1 + tj; j < b; j += W) {
          const double ckj = c[k * bp + j];
          int i = k + 1 + 8 * th;
          for (; i + 8 <= b; i += 8 * H) {       // batch the loads: no smem load->store chains
            double cv[8], lv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) { cv[u] = c[(i + u) * bp + j]; lv[u] = c[(i + u) * bp + k]; }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              cv[u] = sub_rn(cv[u], mul_rn(lv[u], ckj));
              mx = fmax(mx, fabs(cv[u]));
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) c[(i + u) * bp + j] = cv[u];
          }
          // the partial chunk at the bottom belongs to the group whose turn it is
          if (i < b) {
            for (; i < b; ++i) {
              const double v = sub_rn(c[i * bp + j], mul_rn(c[i * bp + k], ckj));
              c[i * bp + j] = v;
              mx = fmax(mx, fabs(v));
            }
          }
        }
      }
    }
    __syncthreads();
  }
  for (int idx = t; idx < b * b; idx += T) D[idx] = c[(idx / b) * bp + idx % b];
  if (t < b) gperm[t] = s_gp[t];
  const double m = block_max(mx, red);
  if (t == 0) atomic_max_abs(&st->finish_max, m);
}

__global__ void __launch_bounds__(1024) gepp_diag_kernel(const double* src, int64_t ld, const int32_t* rowmap, int b,
                                                          double* D, int32_t* piv, int32_t* gperm, DevState* st,
                                                          int panel) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[40];
  if (prrp_failed(st)) return;
  gepp_diag(src, ld, rowmap, b, sm, D, piv, gperm, st, panel, red);
}

// Register GEPP of a b x b block, b <= B = 64 or 128 (gepp.py:39-65, same
// arithmetic as gepp_diag).  B * B/16 threads (256 / 1024): thread (i, q) =
// (t / (B/16), t % (B/16)) holds row i, columns 16q .. 16q+15 in registers.  Per step: the owners of column k
// publish it, every warp finds the first-max pivot redundantly, the pivot
// row and row k trade places through shared memory, and each thread updates
// its 16 entries (product, then subtraction).  Two barriers per step.
#define GR_T 256
template <int B>
__global__ void __launch_bounds__(B * (B / 16), 1) gepp_reg_kernel(const double* src, int64_t ld, const int32_t* rowmap,
                                                                   int b, double* D, int32_t* piv, int32_t* gperm,
                                                                   DevState* st, int panel) {
  constexpr int QN = B / 16;
  __shared__ double colk[2][B];
  __shared__ __align__(16) double prow[B], krow[B];
  __shared__ int s_gp[B];
  __shared__ double red[40];
  if (prrp_failed(st)) return;
  const int t = threadIdx.x, lane = t & 31;
  const int i = t / QN, q = t % QN;
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
  if (t < B) s_gp[t] = t;
  __syncthreads();
  for (int k = 0; k < b; ++k) {
    const int ks = k & 15, kq = k >> 4, cb = k & 1;
    // 1. column k, rows >= k, published by its owners
    double ak = a[0];
#pragma unroll
    for (int s = 1; s < 16; ++s)
      if (s == ks) ak = a[s];
    if (q == kq && i < b) colk[cb][i] = ak;
    __syncthreads();
    // 2. first-max pivot (every warp, redundantly)
    double best = -1.0;
    int bi = INT_MAX;
#pragma unroll
    for (int u = 0; u < B / 32; ++u) {
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
    __syncthreads();
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

// ---------------------------------------------------------------------------
// Finalize a panel after the fast multiplier kernel: reduce the candidates,
// run the strong-RRQR swap loop if the tau bound is violated (rare; QR from
// scratch + multipliers inside the cluster), record the swap count and the
// multiplier max, compact the moved-row list and factor the diagonal block.
// ---------------------------------------------------------------------------
struct FinalizeArgs {
  PanelArgs pa;
  int swap_cap;
  double* D;
  int32_t* piv;
  int32_t* gperm;
  int32_t* swaps_dev;     // per-panel swap counts (device)
  int do_gepp;
};

__global__ void __launch_bounds__(1024, 1) panel_finalize_kernel(FinalizeArgs f) {
  extern __shared__ __align__(16) double dyn_smem[];
  __shared__ PanelShared S;
  __shared__ double red_d[33];
  __shared__ long long red_l[33];
  __shared__ double s_worst;
  __shared__ long long s_flat;
  __shared__ int s_cnt[33];
  cg::cluster_group cl = cg::this_cluster();
  const PanelArgs& a = f.pa;
  __shared__ int s_failed;
  if (cluster_failed(a.st, &s_failed)) return;
  const int c = (int)cl.block_rank(), C = (int)cl.num_blocks();
  const int t = threadIdx.x;

  // a tournament merge node whose children passed <= bsel rows in total
  // selects nothing: its members go up as they are (tournament.py:128-129)
  if (node_passes(a)) {
    if (c == 0) {
      for (int64_t q = t; q < a.p; q += blockDim.x) a.perm[q] = (int32_t)q;
      if (t == 0) {
        *a.want = *a.live;
        f.swaps_dev[a.swap_slot] = 0;
        if (a.node_rows) a.node_rows[a.swap_slot] = *a.live;
      }
    }
    return;
  }

  // Multipliers lt = R11^-1 R12 for a leading block of bs rows over this
  // cluster (tiles strided by CTA), then the cluster-wide worst |lt| with its
  // row-major flat index.  Returns the first rank-deficient diagonal (node
  // mode: the caller retries with fewer rows) or -1; other failures are
  // reported and return -2.
  double worst = -1.0;
  long long wflat = LLONG_MAX;
  auto cluster_multipliers = [&](int bs) -> int {
    double* r11 = dyn_smem;
    double* xs = dyn_smem + bs * (bs + 1) / 2;
    load_r11(a.Rbuf, a.p, bs, r11);
    __syncthreads();
    if (a.want) {
      for (int k = 0; k < bs; ++k)
        if (fabs(r11[upk(k, k)]) < PRRP_EPS * *a.fro) return k;
    }
    if (r11_checks(r11, bs, *a.fro, a.st, a.panel_id, c == 0 && t == 0, a.tree_level, a.tree_index)) return -2;
    worst = -1.0;
    wflat = LLONG_MAX;
    const int64_t nc = a.p - bs;
    const int TW = min((int)blockDim.x, bs > 64 ? 64 : 128);
    const int64_t ntile = (nc + TW - 1) / TW;
    for (int64_t tile = c; tile < ntile; tile += C) {
      trsm_tile(a.Rbuf, a.p, bs, r11, xs, TW, bs + tile * TW, a.L21, a.ldl, worst, wflat);
      __syncthreads();
    }
    reduce_worst(worst, wflat, red_d, red_l);
    if (t == 0) { S.red[0] = worst; S.rec[0].pos = wflat; }
    cl.sync();
    if (t < 32) {
      double w = -1.0;
      long long fl = LLONG_MAX;
      if (t < C) {
        w = *cl.map_shared_rank(&S.red[0], t);
        fl = cl.map_shared_rank(&S.rec[0], t)->pos;
      }
      for (int o = 16; o; o >>= 1) {
        const double ow = __shfl_xor_sync(0xffffffffu, w, o);
        const long long of = __shfl_xor_sync(0xffffffffu, fl, o);
        if (ow > w || (ow == w && of < fl)) { w = ow; fl = of; }
      }
      if (t == 0) { s_worst = w; s_flat = fl; }
    }
    __syncthreads();
    worst = s_worst;
    wflat = s_flat;
    cl.sync();   // the next use of S / dyn_smem may overwrite what other CTAs still read
    return -1;
  };

  int bs = a.bsel;
  int swaps = 0;
  if (a.want && *a.want < a.bsel) {
    // rank-deficient tournament node (tournament.py:131-137): the reference
    // retries strong_rrqr with want = the failing index; the QRCP is the same,
    // so only the multipliers (and a possible swap loop) are redone
    bs = *a.want;
    while (bs > 0) {
      const int k = cluster_multipliers(bs);
      if (k == -2) return;
      if (k < 0) break;
      bs = k;
    }
  } else {
    // reduce the fast-path candidates
    for (int i = t; i < a.ncand; i += blockDim.x) {
      const double w = a.cand[i];
      const long long fl = a.cand_flat[i];
      if (w > worst || (w == worst && fl < wflat)) { worst = w; wflat = fl; }
    }
    reduce_worst(worst, wflat, red_d, red_l);
  }

  // the strong-RRQR interchange loop (pivoted_qr.py:129-144) with leading block bs
  while (bs > 0 && a.p - bs > 0 && worst > a.tau) {
    const int64_t ncol = a.p - bs;
    if (swaps >= f.swap_cap) {
      if (c == 0 && t == 0)
        prrp_set_error(a.st, PRRP_ERR_NONCONVERGENCE, a.panel_id, -1, -1, worst, a.tree_level, a.tree_index);
      return;
    }
    const int i = (int)(wflat / ncol);
    const int64_t jj = wflat % ncol;
    cl.sync();
    if (c == 0 && t == 0) {
      const int32_t x = a.perm[i];
      a.perm[i] = a.perm[bs + jj];
      a.perm[bs + jj] = x;
    }
    cl.sync();
    engine_run(a, 1, a.perm, dyn_smem, S);
    cl.sync();
    const int k = cluster_multipliers(bs);
    if (k == -2) return;
    if (k >= 0) {
      // node: the re-check after a swap failed at k -> a fresh strong RRQR with
      // want = k (the column-pivoted QR from scratch, then its multipliers)
      bs = k;
      swaps = 0;
      engine_run(a, 0, a.perm, dyn_smem, S);
      cl.sync();
      while (bs > 0) {
        const int k2 = cluster_multipliers(bs);
        if (k2 == -2) return;
        if (k2 < 0) break;
        bs = k2;
      }
      continue;
    }
    ++swaps;
  }
  const int64_t ncol = a.p - bs;
  cl.sync();
  if (c != 0) return;

  if (t == 0) {
    f.swaps_dev[a.swap_slot] = swaps;
    a.st->swaps = swaps;
    if (a.want) *a.want = bs;
    if (a.node_rows) a.node_rows[a.swap_slot] = (int32_t)(a.live ? *a.live : a.p);
    // tournament nodes (tree_level >= 0) select rows only; the panel's
    // multiplier statistic comes from its final L21 (tournament.py:274)
    if (ncol > 0 && a.tree_level < 0) atomic_max_abs(&a.st->pmm, worst);
  }
  // compact the moved positions (pos -> src j with j != pos), deterministic order
  {
    const int T = blockDim.x;
    const int64_t per_t = (a.p + T - 1) / T;
    const int64_t lo = t * per_t, hi = min(a.p, lo + per_t);
    int cnt = 0;
    for (int64_t q = lo; q < hi; ++q) cnt += a.perm[q] != q;
    // block exclusive scan of cnt
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
      s_cnt[t] = v;   // inclusive per-warp totals
    }
    __syncthreads();
    int off = incl - cnt + ((t >> 5) ? s_cnt[(t >> 5) - 1] : 0);
    for (int64_t q = lo; q < hi; ++q) {
      const int32_t j = a.perm[q];
      if (j != q) { a.moved[2 * off] = (int32_t)q; a.moved[2 * off + 1] = j; ++off; }
    }
    if (t == blockDim.x - 1) {
      a.st->moved = off;
      if (a.moved_cnt) *a.moved_cnt = off;
    }
  }
  __syncthreads();
  if (f.do_gepp) {
    __shared__ double red[40];
    gepp_diag(a.src, a.ld, a.perm, a.h, dyn_smem, f.D, f.piv, f.gperm, a.st, a.panel_id, red);
  }
}
