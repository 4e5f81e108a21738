// Latency-oriented panel QRCP engine for panels of at most 2048 columns
// (tournament merge nodes 2b x b, the CALU final QR b x b, short leaves and
// the late LU_PRRP panels).  Same arithmetic contract as panel.cuh
// (pivoted_qr.py:43-87): exact numpy-pairwise column norms, first-max
// argmax, the reflector of the winning column with numpy-pairwise v'v,
// w = beta (v' x), x -= v w (product rounded, then subtracted).
//
// Layout: a TEAM of 8 threads owns one column; thread q of a team keeps
// rows i = 8u + q (u < NR) in registers, so a column of h <= 128 rows costs
// 16 doubles per thread; a CTA holds 128 columns (h <= 64, 1024 threads) or
// 64 (h <= 128, 512 threads), a cluster of C <= 16 CTAs C times that.  The numpy pairwise order is
// kept exactly: at step k the relative row index t = i - k of thread q is
// congruent to (q - k) mod 8, so each thread holds exactly one of the eight
// pairwise slots; the slots are combined in numpy's order
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) with three shuffles whose partner
// lanes follow the rotation, and the n % 8 trailing terms are added in row
// order.  Per step:
//   A  every team's (key, position) -> warp best; the warp's best team
//      publishes its column (double-buffered by step parity)
//   B  warp 0: CTA best record; cluster barrier
//   C  warp 0: the cluster winner (DSMEM), its column, alpha, v, v'v, beta,
//      the reflector log; CTA barrier
//   D  every other active team: dot (8-lane butterfly), update, next key
// The per-thread work per step is ~NR elements instead of the thread-per-
// column engines' h, so the dependent chain per step is short.
#pragma once
#include "panel.cuh"

#define PT_G 8                    // threads per column
#define PT_NW 32                  // warps per CTA at most
// threads per CTA: 1024 (128 columns) while a thread's rows fit 64
// registers, 512 (64 columns, 128-register budget) for h > 64
template <int NR> struct PTCfg { static constexpr int T = (NR > 8 || NR <= 4) ? 512 : 1024; };

struct PTRec {
  double key;
  long long pos;
  int warp;                       // publishing warp in its CTA
  int pad;
};

struct PTShared {
  double wpub[2][PT_NW][PRRP_MAXH];
  double vs[PRRP_MAXH];
  double xs[PRRP_MAXH];
  PTRec wrec[PT_NW];
  PTRec rec[2];
  double red[PT_NW];
  double fro_part;
  double beta, alpha;
  int skip;
  int wc, ww;
  long long wpos;
};

__device__ __forceinline__ bool pt_better(double ka, long long pa, double kb, long long pb) {
  return ka > kb || (ka == kb && pa < pb);
}

// numpy-pairwise sum over rows [base, h) of squares of the team's column;
// thread q holds rows 8u + q.  Result in every thread of the team.
template <int NR>
__device__ __forceinline__ double pt_pairwise_sq(const double (&x)[NR], int q, int base, int h, int lane0) {
  const int n = h - base;
  const int n8 = n >= 8 ? n - (n % 8) : 0;
  const int s = (q - base) & 7;            // this thread's slot
  double acc = -0.0, tail = 0.0;
  bool has_tail = false;
#pragma unroll
  for (int u = 0; u < NR; ++u) {
    const int t = 8 * u + q - base;
    if (t >= 0 && t < n8) acc = add_rn(acc, sq_rn(x[u]));
    else if (t >= n8 && t < n) { tail = sq_rn(x[u]); has_tail = true; }
  }
  (void)has_tail;
  double res = -0.0;
  if (n >= 8) {
    // slots s and s^m live in lanes lane0 + ((s ^ m) + base) & 7
    double r = acc;
    r = add_rn(r, __shfl_sync(0xffffffffu, r, lane0 + (((s ^ 1) + base) & 7)));
    r = add_rn(r, __shfl_sync(0xffffffffu, r, lane0 + (((s ^ 2) + base) & 7)));
    r = add_rn(r, __shfl_sync(0xffffffffu, r, lane0 + (((s ^ 4) + base) & 7)));
    res = r;
  }
  // trailing terms t = n8 .. n-1 in order; term n8 + i sits in slot i's thread
  const int nt = n - n8;
#pragma unroll
  for (int i = 0; i < 7; ++i) {
    const double v = __shfl_sync(0xffffffffu, tail, lane0 + ((i + base) & 7));
    if (i < nt) res = add_rn(res, v);
  }
  return res;
}

template <int NR>
__global__ void __launch_bounds__(PTCfg<NR>::T, 1) panel_team_kernel(PanelArgs a) {
  constexpr int PT_T = PTCfg<NR>::T, PT_COLS = PT_T / PT_G, NWC = PT_T / 32;
  extern __shared__ __align__(16) double pt_dyn[];
  PTShared& S = *reinterpret_cast<PTShared*>(pt_dyn);
  cg::cluster_group cl = cg::this_cluster();
  if (node_passes(a)) return;                          // uniform over the cluster (read-only input)
  const int C = (int)cl.num_blocks();
  const int c = (int)cl.block_rank();
  __shared__ int s_failed;
  if (cluster_failed(a.st, &s_failed)) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int team = t >> 3, q = t & 7, lane0 = lane & ~7;
  const int h = a.h;
  const int mode = a.mode;
  const int64_t p = a.p;
  const int64_t myq = (int64_t)c * PT_COLS + team;    // initial position
  const bool on = myq < p;
  long long pos = on ? myq : LLONG_MAX;
  int64_t jcol = 0;                                   // the column this team holds
  double x[NR];
  {
    if (on) {
      jcol = mode == 0 ? myq : (int64_t)a.perm[myq];
      const int64_t row = a.rowidx ? a.rowidx[jcol] : jcol;
      const double* src = member_row(a.src, a.ld, row);
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int i = 8 * u + q;
        x[u] = i < h ? src[i] : 0.0;
      }
    } else {
#pragma unroll
      for (int u = 0; u < NR; ++u) x[u] = 0.0;
    }
  }
  double key = -1.0;
  if (mode == 0) {
    const double nrm = pt_pairwise_sq<NR>(x, q, 0, h, lane0);
    key = on ? nrm : -1.0;
    // ||panel||_F^2: per column, per warp, per CTA, per cluster
    double f = (on && q == 0) ? nrm : 0.0;
    for (int o = 16; o; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
    if (lane == 0) S.red[warp] = f;
    __syncthreads();
    if (t == 0) {
      double s = 0.0;
      for (int w = 0; w < NWC; ++w) s += S.red[w];
      S.fro_part = s;
    }
  } else {
    key = (on && pos == 0) ? 1.0 : -1.0;
  }

  for (int k = 0; k < a.steps; ++k) {
    const int buf = k & 1;
    // ---- A: warp best (teams are 8-lane groups), its column published
    {
      double bk = (on && pos >= k) ? key : -1.0;
      long long bp = (on && pos >= k) ? pos : LLONG_MAX;
      int bt = team;
#pragma unroll
      for (int o = 8; o < 32; o <<= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
        const long long op = __shfl_xor_sync(0xffffffffu, bp, o);
        const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
        if (pt_better(ok, op, bk, bp)) { bk = ok; bp = op; bt = ot; }
      }
      if (bt == team && bp != LLONG_MAX) {
#pragma unroll
        for (int u = 0; u < NR; ++u) {
          const int i = 8 * u + q;
          if (i >= k && i < h) S.wpub[buf][warp][i] = x[u];
        }
      }
      if (lane == 0) { S.wrec[warp].key = bk; S.wrec[warp].pos = bp; S.wrec[warp].warp = warp; }
    }
    __syncthreads();
    // ---- B: CTA best
    if (warp == 0) {
      PTRec r = lane < NWC ? S.wrec[lane] : PTRec{-1.0, LLONG_MAX, 0, 0};
      for (int o = 16; o; o >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, r.key, o);
        const long long op = __shfl_xor_sync(0xffffffffu, r.pos, o);
        const int ow = __shfl_xor_sync(0xffffffffu, r.warp, o);
        if (pt_better(ok, op, r.key, r.pos)) { r.key = ok; r.pos = op; r.warp = ow; }
      }
      if (lane == 0) S.rec[buf] = r;
    }
    if (C > 1) cl.sync(); else __syncthreads();
    // ---- C: the cluster winner and its reflector (warp 0)
    if (warp == 0) {
      PTRec r{-1.0, LLONG_MAX, -1, 0};
      int rc = -1;
      if (lane < C) {
        r = C > 1 ? *cl.map_shared_rank(&S.rec[buf], lane) : S.rec[buf];
        rc = lane;
      }
      for (int o = 16; o; o >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, r.key, o);
        const long long op = __shfl_xor_sync(0xffffffffu, r.pos, o);
        const int ow = __shfl_xor_sync(0xffffffffu, r.warp, o);
        const int oc = __shfl_xor_sync(0xffffffffu, rc, o);
        if (pt_better(ok, op, r.key, r.pos)) { r.key = ok; r.pos = op; r.warp = ow; rc = oc; }
      }
      const double* rpub = C > 1 ? cl.map_shared_rank(&S.wpub[buf][r.warp][0], rc) : &S.wpub[buf][r.warp][0];
      for (int i = k + lane; i < h; i += 32) S.xs[i] = rpub[i];
      if (k == 0 && mode == 0 && c == 0) {
        double f = 0.0;
        if (lane < C) f = C > 1 ? *cl.map_shared_rank(&S.fro_part, lane) : S.fro_part;
        for (int o = 16; o; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
        if (lane == 0) *a.fro = sqrt(f);
      }
      __syncwarp();
      const int L = h - k;
      const double nx2 = mode == 0 ? r.key : warp_pairwise_sq(S.xs + k, L);
      const double normx = __dsqrt_rn(nx2);
      int skip = normx == 0.0;
      double alpha = 0.0, beta = 0.0;
      if (!skip) {
        alpha = S.xs[k] >= 0.0 ? -normx : normx;
        for (int i = k + lane; i < h; i += 32) S.vs[i] = (i == k) ? sub_rn(S.xs[k], alpha) : S.xs[i];
        __syncwarp();
        const double vtv = warp_pairwise_sq(S.vs + k, L);
        if (vtv == 0.0) skip = 1;
        else beta = div_rn(2.0, vtv);
      }
      if (lane == 0) {
        S.skip = skip; S.alpha = alpha; S.beta = beta;
        S.wc = rc; S.ww = r.warp; S.wpos = r.pos;
      }
      if (a.refl && c == 0) {
        double* lg = a.refl + (int64_t)k * (h + 1);
        for (int i = lane; i < h; i += 32) lg[i] = (skip || i < k) ? 0.0 : S.vs[i];
        if (lane == 0) lg[h] = skip ? 0.0 : beta;
      }
    }
    __syncthreads();
    // ---- D: apply reflector k, next keys
    const int skip = S.skip;
    const double beta = S.beta, alpha = S.alpha;
    const long long wpos = S.wpos;
    const bool active = on && pos >= k;
    const bool winner = active && pos == wpos;        // positions are unique over the cluster
    // dot products: every lane takes part in the team butterfly (shuffles
    // outside divergent code), inactive lanes contribute zeros
    double d0 = 0.0, d1 = 0.0;
    if (active && !winner && !skip) {
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int i = 8 * u + q;
        if (i >= k && i < h) {
          if (u & 1) d1 = fma(S.vs[i], x[u], d1);
          else d0 = fma(S.vs[i], x[u], d0);
        }
      }
    }
    double d = d0 + d1;
    d += __shfl_xor_sync(0xffffffffu, d, 1);
    d += __shfl_xor_sync(0xffffffffu, d, 2);
    d += __shfl_xor_sync(0xffffffffu, d, 4);
    if (active) {
      if (winner) {                                   // the pivot column moves to position k
        pos = k;
        if (!skip) {
#pragma unroll
          for (int u = 0; u < NR; ++u) {
            const int i = 8 * u + q;
            if (i == k) x[u] = alpha;
            else if (i > k) x[u] = 0.0;
          }
        }
        key = -1.0;
      } else {
        if (pos == k) pos = wpos;                     // displaced by the interchange
        if (!skip) {
          const double w = mul_rn(beta, d);
#pragma unroll
          for (int u = 0; u < NR; ++u) {
            const int i = 8 * u + q;
            if (i >= k && i < h) x[u] = sub_rn(x[u], mul_rn(S.vs[i], w));
          }
        }
      }
    }
    if (mode == 0) {
      const double nk = pt_pairwise_sq<NR>(x, q, k + 1, h, lane0);
      if (on && pos > k) key = nk;
    } else {
      key = (on && pos == k + 1) ? 1.0 : -1.0;
    }
  }
  if (C > 1) cl.sync();
  // ---- R (by position) and the column order
  if (on) {
#pragma unroll
    for (int u = 0; u < NR; ++u) {
      const int i = 8 * u + q;
      if (i < h) a.Rbuf[(int64_t)i * p + pos] = x[u];
    }
    if (q == 0) a.perm[pos] = (int32_t)jcol;
  }
}

constexpr size_t kPTSmem = sizeof(PTShared);
