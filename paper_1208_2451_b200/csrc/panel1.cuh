// Thread-per-column panel QRCP engine for panel width h = 64 (the BASELINE
// config-2 shape).  Arithmetic contract identical to panel.cuh
// (pivoted_qr.py:43-87); organisation chosen for FP64 issue efficiency:
//
//  * one thread owns one column of the transposed panel (one panel row, 64
//    doubles) entirely in REGISTERS with static indices: row i is element i,
//    numpy's pairwise slot of row i is i & 7, so the dot, the rank-1 update
//    and the 8-accumulator norm need no shuffles and no index arithmetic;
//  * a thread may own a second column in shared memory ([row][thread]
//    layout, ld.shared/st.shared), i.e. up to 2*P1_T columns per CTA and
//    12288 per 16-CTA cluster;
//  * per step: warp reduce -> CTA barrier -> every warp reduces the warp
//    bests -> records pushed into every CTA (DSMEM stores) -> cluster barrier
//    -> warp 0 fetches the winner column and builds the reflector -> CTA
//    barrier -> apply.
#pragma once
#include "panel.cuh"

#define P1_H 64
#define P1_T 384                 // threads per CTA (register budget: <= 170 regs)
#define P1_MAXCOLS (2 * P1_T)

struct P1Rec {
  double key;
  long long pos;
  int jl;
  int pad;
};

struct P1Shared {
  double pub[2][P1_H];
  double xs[P1_H];
  double vs[P1_H];
  P1Rec recall[2][PRRP_CLUSTER_MAX];
  P1Rec wbest[P1_T / 32];
  double fro_warp[P1_T / 32];
  double fro_cta[PRRP_CLUSTER_MAX];
  double beta, alpha;
  int skip;
  int wc, wjl;
  long long wpos;
};

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_f64(uint32_t addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;" :: "r"(addr), "d"(v) : "memory");
}

struct P1Reg {
  double (&r)[P1_H];
  __device__ __forceinline__ double ld(int i) const { return r[i]; }
  __device__ __forceinline__ void st(int i, double v) const { r[i] = v; }
};
struct P1Smem {
  uint32_t base;   // shared address of element 0; element i at base + i * P1_T * 8
  __device__ __forceinline__ double ld(int i) const { return lds_f64(base + (uint32_t)i * (P1_T * 8)); }
  __device__ __forceinline__ void st(int i, double v) const { sts_f64(base + (uint32_t)i * (P1_T * 8), v); }
};

// numpy pairwise sum of squares of rows k+1 .. 63 (k = -1: the whole column).
// Blocks of 8 rows are classified with warp-uniform branches (k is uniform):
// blocks above row k+1 are skipped, interior blocks run unpredicated, only the
// boundary block and the last block carry per-row predicates.
template <class X>
__device__ __forceinline__ double p1_norm(const X& x, int k) {
  const int n = P1_H - k - 1;
  const int rem = n < 8 ? n : (n & 7);
  const int lim = P1_H - rem;
  const int kb = (k + 1) >> 3;
  double S[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) S[s] = 0.0;
#pragma unroll
  for (int B = 0; B < 8; ++B) {
    if (B < kb) continue;
    if (B > kb && B < 7) {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const double v = x.ld(8 * B + s);
        S[s] = add_rn(S[s], mul_rn(v, v));
      }
    } else {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int i = 8 * B + s;
        if (i >= k + 1 && i < lim) {
          const double v = x.ld(i);
          S[s] = add_rn(S[s], mul_rn(v, v));
        }
      }
    }
  }
  double res = -0.0;
  if (n >= 8) {
    const int o = (k + 1) & 7;   // logical accumulator j is slot (j + o) & 7
    double r0 = S[0], r1 = S[1], r2 = S[2], r3 = S[3], r4 = S[4], r5 = S[5], r6 = S[6], r7 = S[7];
#define P1_ROT(c, s0, s1, s2, s3, s4, s5, s6, s7)                                      \
  {                                                                                    \
    const double t0 = c ? s0 : r0, t1 = c ? s1 : r1, t2 = c ? s2 : r2, t3 = c ? s3 : r3; \
    const double t4 = c ? s4 : r4, t5 = c ? s5 : r5, t6 = c ? s6 : r6, t7 = c ? s7 : r7; \
    r0 = t0; r1 = t1; r2 = t2; r3 = t3; r4 = t4; r5 = t5; r6 = t6; r7 = t7;              \
  }
    if (o & 1) P1_ROT(true, r1, r2, r3, r4, r5, r6, r7, r0)
    if (o & 2) P1_ROT(true, r2, r3, r4, r5, r6, r7, r0, r1)
    if (o & 4) P1_ROT(true, r4, r5, r6, r7, r0, r1, r2, r3)
#undef P1_ROT
    res = add_rn(add_rn(add_rn(r0, r1), add_rn(r2, r3)), add_rn(add_rn(r4, r5), add_rn(r6, r7)));
  }
  // sequential remainder: rows 64-rem .. 63 of the last block (squares recomputed)
#pragma unroll
  for (int s = 0; s < 8; ++s)
    if (s >= 8 - rem) {
      const double v = x.ld(56 + s);
      res = add_rn(res, mul_rn(v, v));
    }
  return res;
}

// apply reflector k; act == false is an exact no-op (w = 0)
template <class X>
__device__ __forceinline__ void p1_apply(const X& x, int k, const double* vs, double beta, bool act) {
  const int kb = k >> 3;
  double d[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int B = 0; B < 8; ++B) {
    if (B < kb) continue;
    if (B > kb) {
#pragma unroll
      for (int s = 0; s < 8; ++s) d[s & 3] = fma(vs[8 * B + s], x.ld(8 * B + s), d[s & 3]);
    } else {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int i = 8 * B + s;
        if (i >= k) d[s & 3] = fma(vs[i], x.ld(i), d[s & 3]);
      }
    }
  }
  const double dot = (d[0] + d[1]) + (d[2] + d[3]);
  const double w = act ? mul_rn(beta, dot) : 0.0;
#pragma unroll
  for (int B = 0; B < 8; ++B) {
    if (B < kb) continue;
    if (B > kb) {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int i = 8 * B + s;
        x.st(i, sub_rn(x.ld(i), mul_rn(vs[i], w)));
      }
    } else {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int i = 8 * B + s;
        if (i >= k) x.st(i, sub_rn(x.ld(i), mul_rn(vs[i], w)));
      }
    }
  }
}

template <class X>
__device__ __forceinline__ void p1_set_pivot(const X& x, int k, double alpha) {
#pragma unroll
  for (int i = 0; i < P1_H; ++i) {
    if (i == k) x.st(i, alpha);
    else if (i > k) x.st(i, 0.0);
  }
}

__global__ void __launch_bounds__(P1_T, 1) panel_qrcp1_kernel(PanelArgs a) {
  extern __shared__ __align__(16) double sdata[];      // P1_H x P1_T shared columns
  __shared__ P1Shared S;
  cg::cluster_group cl = cg::this_cluster();
  if (prrp_failed(a.st)) return;
  const int C = (int)cl.num_blocks();
  const int c = (int)cl.block_rank();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  constexpr int NW = P1_T / 32;
  const int mode = a.mode;
  const int64_t j0 = (int64_t)c * a.per;
  const int nl = (int)max((int64_t)0, min(a.per, a.p - j0));
  const int jl_r = t, jl_s = P1_T + t;
  const bool on_r = jl_r < nl, on_s = jl_s < nl;
  const bool has_s = nl > P1_T;      // CTA-uniform

  double rr[P1_H];
  const P1Reg xr{rr};
  const P1Smem xsm{(uint32_t)__cvta_generic_to_shared(sdata + t)};
  auto src_row = [&](int jl) -> const double* {
    const int64_t qq = j0 + jl;
    const int64_t j = mode == 0 ? qq : (int64_t)a.perm[qq];
    const int64_t row = a.rowidx ? a.rowidx[j] : j;
    return a.src + row * a.ld;
  };
  if (on_r) {
    const double2* s = reinterpret_cast<const double2*>(src_row(jl_r));
#pragma unroll
    for (int i = 0; i < P1_H / 2; ++i) { const double2 v = s[i]; rr[2 * i] = v.x; rr[2 * i + 1] = v.y; }
  } else {
#pragma unroll
    for (int i = 0; i < P1_H; ++i) rr[i] = 0.0;
  }
  if (has_s) {
    if (on_s) {
      const double* s = src_row(jl_s);
#pragma unroll
      for (int i = 0; i < P1_H; ++i) xsm.st(i, s[i]);
    } else {
#pragma unroll
      for (int i = 0; i < P1_H; ++i) xsm.st(i, 0.0);
    }
  }
  long long pos_r = j0 + jl_r, pos_s = j0 + jl_s;
  double key_r = -1.0, key_s = -1.0, fro = 0.0;
  if (mode == 0) {
    if (on_r) { key_r = p1_norm(xr, -1); fro += key_r; }
    if (has_s && on_s) { key_s = p1_norm(xsm, -1); fro += key_s; }
    for (int o = 16; o; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
    if (lane == 0) S.fro_warp[warp] = fro;
  } else {
    key_r = on_r && pos_r == 0 ? 1.0 : -1.0;
    key_s = on_s && pos_s == 0 ? 1.0 : -1.0;
  }
  __syncthreads();
  if (mode == 0 && t == 0) {
    double f = 0.0;
    for (int w = 0; w < NW; ++w) f += S.fro_warp[w];
    for (int r = 0; r < C; ++r) *cl.map_shared_rank(&S.fro_cta[c], r) = f;
  }

#ifdef PRRP_P64_PROF
  const bool prof = a.prof && c == 0 && t == 0;
#else
  constexpr bool prof = false;
#endif
  long long pr[4] = {0, 0, 0, 0}, pt = prof ? clock64() : 0;
  const long long p_start = pt;
#define P1_MARK(slot) if (prof) { const long long nn = clock64(); pr[slot] += nn - pt; pt = nn; }
  for (int k = 0; k < a.steps; ++k) {
    const int buf = k & 1;
    P1_MARK(3)
    // ---- warp best, then CTA best (every warp reduces the warp bests redundantly)
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
    P1_MARK(0)
    {
      P1Rec r = lane < NW ? S.wbest[lane] : P1Rec{-INFINITY, LLONG_MAX, -1, 0};
      for (int o = 16; o; o >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, r.key, o);
        const long long op = __shfl_xor_sync(0xffffffffu, r.pos, o);
        const int oj = __shfl_xor_sync(0xffffffffu, r.jl, o);
        if (better(ok, op, r.key, r.pos)) { r.key = ok; r.pos = op; r.jl = oj; }
      }
      if (r.jl >= 0 && r.jl == jl_r) {
#pragma unroll
        for (int i = 0; i < P1_H; ++i) if (i >= k) S.pub[buf][i] = rr[i];
      } else if (r.jl >= 0 && r.jl == jl_s) {
        for (int i = k; i < P1_H; ++i) S.pub[buf][i] = xsm.ld(i);
      }
      if (t < C) *cl.map_shared_rank(&S.recall[buf][c], t) = r;
    }
    cl.sync();
    P1_MARK(1)

    // ---- warp 0: winner, its column, the reflector
    if (warp == 0) {
      P1Rec r = lane < C ? S.recall[buf][lane] : P1Rec{-INFINITY, LLONG_MAX, -1, 0};
      int rc = lane < C ? lane : -1;
      for (int o = 16; o; o >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, r.key, o);
        const long long op = __shfl_xor_sync(0xffffffffu, r.pos, o);
        const int oj = __shfl_xor_sync(0xffffffffu, r.jl, o);
        const int oc = __shfl_xor_sync(0xffffffffu, rc, o);
        if (better(ok, op, r.key, r.pos)) { r.key = ok; r.pos = op; r.jl = oj; rc = oc; }
      }
      const double* rpub = cl.map_shared_rank(&S.pub[buf][0], rc);
      const double x0 = k + lane < P1_H ? rpub[k + lane] : 0.0;
      const double x1 = k + lane + 32 < P1_H ? rpub[k + lane + 32] : 0.0;
      if (k + lane < P1_H) S.xs[k + lane] = x0;
      if (k + lane + 32 < P1_H) S.xs[k + lane + 32] = x1;
      if (k == 0 && mode == 0 && c == 0) {
        double f = lane < C ? S.fro_cta[lane] : 0.0;
        for (int o = 16; o; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
        if (lane == 0) *a.fro = sqrt(f);
      }
      __syncwarp();
      const int L = P1_H - k;
      // mode 0: the winner's key IS (x*x).sum() over rows k..63 in numpy's order
      const double normx = __dsqrt_rn(mode == 0 ? r.key : warp_pairwise_sq(S.xs + k, L));
      int skip = normx == 0.0;
      double alpha = 0.0, beta = 0.0;
      if (!skip) {
        const double xk = __shfl_sync(0xffffffffu, x0, 0);
        alpha = xk >= 0.0 ? -normx : normx;
        if (k + lane < P1_H) S.vs[k + lane] = lane == 0 ? sub_rn(xk, alpha) : x0;
        if (k + lane + 32 < P1_H) S.vs[k + lane + 32] = x1;
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
        double* lg = a.refl + (int64_t)k * (P1_H + 1);
        for (int i = lane; i < P1_H; i += 32) lg[i] = (skip || i < k) ? 0.0 : S.vs[i];
        if (lane == 0) lg[P1_H] = skip ? 0.0 : beta;
      }
    }
    __syncthreads();
    P1_MARK(2)

    // ---- apply reflector k, norms for step k+1
    const int skip = S.skip;
    const double beta = S.beta, alpha = S.alpha;
    const bool mine = S.wc == c;
    const int wjl = S.wjl;
    const long long wpos = S.wpos;
    if (__any_sync(0xffffffffu, on_r && pos_r >= k)) {
      const bool live = on_r && pos_r >= k;
      const bool win = live && mine && wjl == jl_r;
      if (live && !win && pos_r == k) pos_r = wpos;
      p1_apply(xr, k, S.vs, beta, live && !win && !skip);
      if (win) {
        pos_r = k;
        if (!skip) p1_set_pivot(xr, k, alpha);
      }
      if (mode == 0) {
        const double nk = p1_norm(xr, k);
        key_r = (live && !win) ? nk : -1.0;
      } else {
        key_r = (live && pos_r == k + 1) ? 1.0 : -1.0;
      }
    }
    if (has_s && __any_sync(0xffffffffu, on_s && pos_s >= k)) {
      const bool live = on_s && pos_s >= k;
      const bool win = live && mine && wjl == jl_s;
      if (live && !win && pos_s == k) pos_s = wpos;
      p1_apply(xsm, k, S.vs, beta, live && !win && !skip);
      if (win) {
        pos_s = k;
        if (!skip) p1_set_pivot(xsm, k, alpha);
      }
      if (mode == 0) {
        const double nk = p1_norm(xsm, k);
        key_s = (live && !win) ? nk : -1.0;
      } else {
        key_s = (live && pos_s == k + 1) ? 1.0 : -1.0;
      }
    }
  }
  if (prof) {
    const long long nn = clock64();
    pr[3] += nn - pt;
    a.prof[0] += pr[0]; a.prof[1] += pr[1]; a.prof[2] += pr[2]; a.prof[3] += pr[3];
    a.prof[4] += nn - p_start; a.prof[5] += 1;
  }
#undef P1_MARK
  cl.sync();
  // ---- R by position, column order
  if (on_r) {
#pragma unroll
    for (int i = 0; i < P1_H; ++i) a.Rbuf[(int64_t)i * a.p + pos_r] = rr[i];
    const int64_t qq = j0 + jl_r;
    a.perm[pos_r] = (int32_t)(mode == 0 ? qq : (int64_t)a.perm[qq]);
  }
  if (on_s) {
    for (int i = 0; i < P1_H; ++i) a.Rbuf[(int64_t)i * a.p + pos_s] = xsm.ld(i);
    const int64_t qq = j0 + jl_s;
    a.perm[pos_s] = (int32_t)(mode == 0 ? qq : (int64_t)a.perm[qq]);
  }
}
