// Register-resident panel QRCP engine for panel width h = 64 (BASELINE
// config 2 headline shape).  Same arithmetic contract as panel.cuh
// (pivoted_qr.py:43-87), re-organised for latency:
//
//  * a column of the transposed panel (one panel row, 64 doubles) is owned by
//    a PAIR of threads; thread g holds the rows whose slot (row & 7) lies in
//    [4g, 4g+4) — 32 doubles in registers — so numpy's 8-accumulator pairwise
//    norm chains never cross threads;
//  * each thread pair owns two columns: one in registers, one in shared
//    memory (same slot layout), i.e. 512 columns per CTA, 8192 per
//    16-CTA cluster, with no global-memory spill;
//  * every step costs one CTA barrier + one cluster barrier + one CTA barrier:
//    CTA-best records are pushed into every CTA's shared memory (DSMEM stores)
//    before the cluster barrier, so only the winner's column is fetched
//    remotely after it.
#pragma once
#include "panel.cuh"

#define P64_H 64
#define P64_G 2
#define P64_E 32            // elements per thread (H / G)
#define P64_SL 4            // slots per thread (8 / G)
#define P64_T 512           // threads per CTA
#define P64_GROUPS (P64_T / P64_G)
#define P64_MAXCOLS (2 * P64_GROUPS)   // columns per CTA

struct P64Rec {
  double key;
  long long pos;
  int jl;
  int pad;
};

struct P64Shared {
  double pub[2][P64_H];
  double xs[P64_H];
  double vs[P64_H];
  P64Rec recall[2][PRRP_CLUSTER_MAX];
  P64Rec wbest[P64_T / 32];
  double fro_warp[P64_T / 32];
  double fro_cta[PRRP_CLUSTER_MAX];
  double beta, alpha;
  int skip;
  int wc, wjl;
  long long wpos;
};

// row of element e held by thread g
__device__ __forceinline__ constexpr int p64_row(int e, int g) {
  return 8 * (e / P64_SL) + g * P64_SL + (e % P64_SL);
}

// numpy pairwise sum of squares of rows k+1 .. 63 of this column.  Called by
// every lane of the warp (full-mask shuffles); both lanes of a pair return
// the same bits.  Blocks of 8 rows entirely above row k+1 are skipped with a
// warp-uniform branch.
template <class X>
__device__ __forceinline__ double p64_norm_after(X& x, int g, int k) {
  const int n = P64_H - k - 1;
  const int rem = n < 8 ? n : (n & 7);
  const int lim = P64_H - rem;
  const int kb = (k + 1) >> 3;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  double l0 = 0.0, l1 = 0.0, l2 = 0.0, l3 = 0.0;
#pragma unroll
  for (int B = 0; B < 8; ++B) {
    if (B < kb) continue;
#pragma unroll
    for (int u = 0; u < P64_SL; ++u) {
      const int e = B * P64_SL + u;
      const int i = p64_row(e, g);
      const double v = x(e);
      const double sq = mul_rn(v, v);
      const bool in = i >= k + 1 && i < lim;
      if (u == 0) a0 = in ? add_rn(a0, sq) : a0;
      if (u == 1) a1 = in ? add_rn(a1, sq) : a1;
      if (u == 2) a2 = in ? add_rn(a2, sq) : a2;
      if (u == 3) a3 = in ? add_rn(a3, sq) : a3;
      if (B == 7) {
        const bool tl = i >= lim;
        if (u == 0) l0 = tl ? sq : 0.0;
        if (u == 1) l1 = tl ? sq : 0.0;
        if (u == 2) l2 = tl ? sq : 0.0;
        if (u == 3) l3 = tl ? sq : 0.0;
      }
    }
  }
  // slot sums S0..S7 and last-block squares L0..L7 into both lanes of the pair
  // partner lane (lane ^ 1) holds the other four slots; g selects which half is ours
  const bool hi = (threadIdx.x & 1) != 0;
  const double b0 = __shfl_xor_sync(0xffffffffu, a0, 1), b1 = __shfl_xor_sync(0xffffffffu, a1, 1);
  const double b2 = __shfl_xor_sync(0xffffffffu, a2, 1), b3 = __shfl_xor_sync(0xffffffffu, a3, 1);
  const double m0 = __shfl_xor_sync(0xffffffffu, l0, 1), m1 = __shfl_xor_sync(0xffffffffu, l1, 1);
  const double m2 = __shfl_xor_sync(0xffffffffu, l2, 1), m3 = __shfl_xor_sync(0xffffffffu, l3, 1);
  const double S0 = hi ? b0 : a0, S1 = hi ? b1 : a1, S2 = hi ? b2 : a2, S3 = hi ? b3 : a3;
  const double S4 = hi ? a0 : b0, S5 = hi ? a1 : b1, S6 = hi ? a2 : b2, S7 = hi ? a3 : b3;
  const double L0 = hi ? m0 : l0, L1 = hi ? m1 : l1, L2 = hi ? m2 : l2, L3 = hi ? m3 : l3;
  const double L4 = hi ? l0 : m0, L5 = hi ? l1 : m1, L6 = hi ? l2 : m2, L7 = hi ? l3 : m3;
  double res = -0.0;
  if (n >= 8) {
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) with r_j = S[(j + o) & 7], o = (k+1) & 7
    const int o = (k + 1) & 7;
    double r0 = S0, r1 = S1, r2 = S2, r3 = S3, r4 = S4, r5 = S5, r6 = S6, r7 = S7;
#define P64_ROT(c, s0, s1, s2, s3, s4, s5, s6, s7)                                     \
  {                                                                                    \
    const double t0 = c ? s0 : r0, t1 = c ? s1 : r1, t2 = c ? s2 : r2, t3 = c ? s3 : r3; \
    const double t4 = c ? s4 : r4, t5 = c ? s5 : r5, t6 = c ? s6 : r6, t7 = c ? s7 : r7; \
    r0 = t0; r1 = t1; r2 = t2; r3 = t3; r4 = t4; r5 = t5; r6 = t6; r7 = t7;              \
  }
    P64_ROT((o & 1) != 0, r1, r2, r3, r4, r5, r6, r7, r0)
    P64_ROT((o & 2) != 0, r2, r3, r4, r5, r6, r7, r0, r1)
    P64_ROT((o & 4) != 0, r4, r5, r6, r7, r0, r1, r2, r3)
#undef P64_ROT
    res = add_rn(add_rn(add_rn(r0, r1), add_rn(r2, r3)), add_rn(add_rn(r4, r5), add_rn(r6, r7)));
  }
  // sequential remainder: last-block rows 64-rem .. 63 (slots 8-rem .. 7)
  if (rem >= 8) res = add_rn(res, L0);
  if (rem >= 7) res = add_rn(res, L1);
  if (rem >= 6) res = add_rn(res, L2);
  if (rem >= 5) res = add_rn(res, L3);
  if (rem >= 4) res = add_rn(res, L4);
  if (rem >= 3) res = add_rn(res, L5);
  if (rem >= 2) res = add_rn(res, L6);
  if (rem >= 1) res = add_rn(res, L7);
  return res;
}

// Apply reflector k (v, beta) to one column held as x(e) (rows i(e) >= k).
// Called by every lane; `act` false turns the update into an exact no-op
// (w = 0: x - v*0 == x, and the +0 rows of finished pivot columns stay +0).
template <class X>
__device__ __forceinline__ void p64_apply(X& x, int g, int k, const double* vs, double beta, bool act) {
  const int kb = k >> 3;
  double d0 = 0.0, d1 = 0.0;
#pragma unroll
  for (int B = 0; B < 8; ++B) {
    if (B < kb) continue;
#pragma unroll
    for (int u = 0; u < P64_SL; ++u) {
      const int e = B * P64_SL + u;
      const int i = p64_row(e, g);
      if (i >= k) {
        if (u & 1) d1 = fma(vs[i], x(e), d1);
        else d0 = fma(vs[i], x(e), d0);
      }
    }
  }
  double dot = d0 + d1;
  dot = dot + __shfl_xor_sync(0xffffffffu, dot, 1);
  const double w = act ? mul_rn(beta, dot) : 0.0;
#pragma unroll
  for (int B = 0; B < 8; ++B) {
    if (B < kb) continue;
#pragma unroll
    for (int u = 0; u < P64_SL; ++u) {
      const int e = B * P64_SL + u;
      const int i = p64_row(e, g);
      if (i >= k) x(e) = sub_rn(x(e), mul_rn(vs[i], w));
    }
  }
}

struct RegCol {
  double (&r)[P64_E];
  __device__ __forceinline__ double& operator()(int e) const { return r[e]; }
};
struct SmemCol {
  double* s;   // element e at s[e * P64_T]
  __device__ __forceinline__ double& operator()(int e) const { return s[e * P64_T]; }
};

__global__ void __launch_bounds__(P64_T, 1) panel_qrcp64_kernel(PanelArgs a) {
  extern __shared__ __align__(16) double sdata[];      // P64_E x P64_T smem columns
  __shared__ P64Shared S;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ int s_failed;
  if (node_passes(a) || cluster_failed(a.st, &s_failed)) return;
  const int C = (int)cl.num_blocks();
  const int c = (int)cl.block_rank();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int q = t / P64_G, g = t % P64_G;
  const int mode = a.mode;
  const int64_t j0 = (int64_t)c * a.per;
  const int nl = (int)max((int64_t)0, min(a.per, a.p - j0));
  // local column ids: register column q, shared column P64_GROUPS + q
  const int jl_r = q, jl_s = P64_GROUPS + q;
  const bool on_r = jl_r < nl, on_s = jl_s < nl;

  double rr[P64_E];
  RegCol xr{rr};
  SmemCol xsm{sdata + t};
  // shared-memory columns exist (and dynamic smem is allocated) iff per > groups
  const bool has_s = a.per > P64_GROUPS;
  auto src_row = [&](int jl) -> const double* {
    const int64_t qq = j0 + jl;
    const int64_t j = mode == 0 ? qq : (int64_t)a.perm[qq];
    const int64_t row = a.rowidx ? a.rowidx[j] : j;
    return member_row(a.src, a.ld, row);
  };
  if (on_r) {
    const double* s = src_row(jl_r);
#pragma unroll
    for (int e = 0; e < P64_E; ++e) rr[e] = s[p64_row(e, g)];
  } else {
#pragma unroll
    for (int e = 0; e < P64_E; ++e) rr[e] = 0.0;
  }
  if (has_s) {
    if (on_s) {
      const double* s = src_row(jl_s);
#pragma unroll
      for (int e = 0; e < P64_E; ++e) xsm(e) = s[p64_row(e, g)];
    } else {
#pragma unroll
      for (int e = 0; e < P64_E; ++e) xsm(e) = 0.0;
    }
  }
  long long pos_r = j0 + jl_r, pos_s = j0 + jl_s;
  double key_r = -1.0, key_s = -1.0, fro = 0.0;
  if (mode == 0) {
    const double nr = p64_norm_after(xr, g, -1);
    if (on_r) { key_r = nr; fro += nr; }
    if (has_s) {
      const double ns = p64_norm_after(xsm, g, -1);
      if (on_s) { key_s = ns; fro += ns; }
    }
  } else {
    key_r = pos_r == 0 ? 1.0 : -1.0;
    key_s = pos_s == 0 ? 1.0 : -1.0;
  }
  if (mode == 0) {
    // ||panel||_F^2 partials: one lane per pair counts its columns
    double f = g == 0 ? fro : 0.0;
    for (int o = 16; o; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
    if (lane == 0) S.fro_warp[warp] = f;
  }
  if (!on_r) key_r = -1.0;
  if (!on_s) key_s = -1.0;
  __syncthreads();
  if (mode == 0 && t == 0) {
    double f = 0.0;
    for (int w = 0; w < P64_T / 32; ++w) f += S.fro_warp[w];
    for (int r = 0; r < C; ++r) *cl.map_shared_rank(&S.fro_cta[c], r) = f;
  }

#ifdef PRRP_P64_PROF
  const bool prof = a.prof && c == 0 && t == 0;
#else
  constexpr bool prof = false;
#endif
  long long pr_red = 0, pr_pub = 0, pr_refl = 0, pr_app = 0, pt = prof ? clock64() : 0;
  const long long p_start = pt;
  for (int k = 0; k < a.steps; ++k) {
    const int buf = k & 1;
    if (prof) { const long long n = clock64(); pr_app += n - pt; pt = n; }
    // ---- thread / warp / CTA best among active columns
    double bk = -INFINITY;
    long long bp = LLONG_MAX;
    int bj = -1;
    if (on_r && pos_r >= k && better(key_r, pos_r, bk, bp)) { bk = key_r; bp = pos_r; bj = jl_r; }
    if (on_s && pos_s >= k && better(key_s, pos_s, bk, bp)) { bk = key_s; bp = pos_s; bj = jl_s; }
    for (int o = 16; o; o >>= 1) {
      const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const long long op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (better(ok, op, bk, bp)) { bk = ok; bp = op; bj = oj; }
    }
    if (lane == 0) { S.wbest[warp].key = bk; S.wbest[warp].pos = bp; S.wbest[warp].jl = bj; }
    __syncthreads();
    if (prof) { const long long n = clock64(); pr_red += n - pt; pt = n; }
    {
      P64Rec r = lane < P64_T / 32 ? S.wbest[lane] : P64Rec{-INFINITY, LLONG_MAX, -1, 0};
      for (int o = 16; o; o >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, r.key, o);
        const long long op = __shfl_xor_sync(0xffffffffu, r.pos, o);
        const int oj = __shfl_xor_sync(0xffffffffu, r.jl, o);
        if (better(ok, op, r.key, r.pos)) { r.key = ok; r.pos = op; r.jl = oj; }
      }
      // owners of the CTA-best column publish rows k..63
      if (r.jl >= 0 && (r.jl == jl_r || r.jl == jl_s) && (r.jl % P64_GROUPS) == q) {
        if (r.jl == jl_r) {
#pragma unroll
          for (int e = 0; e < P64_E; ++e) { const int i = p64_row(e, g); if (i >= k) S.pub[buf][i] = rr[e]; }
        } else {
#pragma unroll
          for (int e = 0; e < P64_E; ++e) { const int i = p64_row(e, g); if (i >= k) S.pub[buf][i] = xsm(e); }
        }
      }
      if (t < C) {   // push this CTA's record into every CTA of the cluster
        P64Rec* dst = cl.map_shared_rank(&S.recall[buf][c], t);
        *dst = r;
      }
    }
    cl.sync();
    if (prof) { const long long n = clock64(); pr_pub += n - pt; pt = n; }

    // ---- warp 0: winner, its column, the reflector
    if (warp == 0) {
      P64Rec r = lane < C ? S.recall[buf][lane] : P64Rec{-INFINITY, LLONG_MAX, -1, 0};
      int rc = lane < C ? lane : -1;
      for (int o = 16; o; o >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, r.key, o);
        const long long op = __shfl_xor_sync(0xffffffffu, r.pos, o);
        const int oj = __shfl_xor_sync(0xffffffffu, r.jl, o);
        const int oc = __shfl_xor_sync(0xffffffffu, rc, o);
        if (better(ok, op, r.key, r.pos)) { r.key = ok; r.pos = op; r.jl = oj; rc = oc; }
      }
      const double* rpub = cl.map_shared_rank(&S.pub[buf][0], rc);
      for (int i = k + lane; i < P64_H; i += 32) S.xs[i] = rpub[i];
      if (k == 0 && mode == 0 && c == 0) {
        double f = lane < C ? S.fro_cta[lane] : 0.0;
        for (int o = 16; o; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
        if (lane == 0) *a.fro = sqrt(f);
      }
      __syncwarp();
      const int L = P64_H - k;
      // mode 0: the winner's key IS (x*x).sum() over rows k..63 in numpy's
      // pairwise order (same elements, same order as _reflect's normx)
      const double normx = __dsqrt_rn(mode == 0 ? r.key : warp_pairwise_sq(S.xs + k, L));
      int skip = normx == 0.0;
      double alpha = 0.0, beta = 0.0;
      if (!skip) {
        alpha = S.xs[k] >= 0.0 ? -normx : normx;
        for (int i = k + lane; i < P64_H; i += 32) S.vs[i] = (i == k) ? sub_rn(S.xs[k], alpha) : S.xs[i];
        __syncwarp();
        const double vtv = warp_pairwise_sq(S.vs + k, L);
        if (vtv == 0.0) skip = 1;
        else beta = div_rn(2.0, vtv);
      }
      if (lane == 0) {
        S.skip = skip; S.alpha = alpha; S.beta = beta;
        S.wc = rc; S.wjl = r.jl; S.wpos = r.pos;
      }
      if (a.refl && c == 0) {
        double* lg = a.refl + (int64_t)k * (P64_H + 1);
        for (int i = lane; i < P64_H; i += 32) lg[i] = (skip || i < k) ? 0.0 : S.vs[i];
        if (lane == 0) lg[P64_H] = skip ? 0.0 : beta;
      }
    }
    __syncthreads();
    if (prof) { const long long n = clock64(); pr_refl += n - pt; pt = n; }

    // ---- apply reflector k, norms for step k+1 (warp-uniform control flow)
    const int skip = S.skip;
    const double beta = S.beta, alpha = S.alpha;
    const bool mine = S.wc == c;
    const int wjl = S.wjl;
    const long long wpos = S.wpos;
    // warps whose columns are all absent or finished skip the work (warp-uniform)
    if (__any_sync(0xffffffffu, on_r && pos_r >= k)) {
      const bool live = on_r && pos_r >= k;
      const bool win = live && mine && wjl == jl_r;
      if (live && !win && pos_r == k) pos_r = wpos;        // displaced by the interchange
      p64_apply(xr, g, k, S.vs, beta, live && !win && !skip);
      if (win) {
        pos_r = k;
        if (!skip) {
#pragma unroll
          for (int e = 0; e < P64_E; ++e) {
            const int i = p64_row(e, g);
            if (i == k) rr[e] = alpha;
            else if (i > k) rr[e] = 0.0;
          }
        }
      }
      if (mode == 0) {
        const double nk = p64_norm_after(xr, g, k);
        key_r = (live && !win) ? nk : -1.0;
      } else {
        key_r = pos_r == k + 1 ? 1.0 : -1.0;
      }
    }
    if (has_s && __any_sync(0xffffffffu, on_s && pos_s >= k)) {
      const bool live = on_s && pos_s >= k;
      const bool win = live && mine && wjl == jl_s;
      if (live && !win && pos_s == k) pos_s = wpos;
      p64_apply(xsm, g, k, S.vs, beta, live && !win && !skip);
      if (win) {
        pos_s = k;
        if (!skip) {
#pragma unroll
          for (int e = 0; e < P64_E; ++e) {
            const int i = p64_row(e, g);
            if (i == k) xsm(e) = alpha;
            else if (i > k) xsm(e) = 0.0;
          }
        }
      }
      if (mode == 0) {
        const double nk = p64_norm_after(xsm, g, k);
        key_s = (live && !win) ? nk : -1.0;
      } else {
        key_s = pos_s == k + 1 ? 1.0 : -1.0;
      }
    }
  }
  if (prof) {
    const long long n = clock64();
    pr_app += n - pt;
    a.prof[0] += pr_red; a.prof[1] += pr_pub; a.prof[2] += pr_refl; a.prof[3] += pr_app;
    a.prof[4] += n - p_start; a.prof[5] += 1;
  }
  cl.sync();
  // ---- R by position, column order
  if (on_r) {
#pragma unroll
    for (int e = 0; e < P64_E; ++e) a.Rbuf[(int64_t)p64_row(e, g) * a.p + pos_r] = rr[e];
    if (g == 0) {
      const int64_t qq = j0 + jl_r;
      a.perm[pos_r] = (int32_t)(mode == 0 ? qq : (int64_t)a.perm[qq]);
    }
  }
  if (on_s) {
#pragma unroll
    for (int e = 0; e < P64_E; ++e) a.Rbuf[(int64_t)p64_row(e, g) * a.p + pos_s] = xsm(e);
    if (g == 0) {
      const int64_t qq = j0 + jl_s;
      a.perm[pos_s] = (int32_t)(mode == 0 ? qq : (int64_t)a.perm[qq]);
    }
  }
}
