// Panel strong-RRQR engine: Householder QR with column pivoting of the h x p
// transposed panel A_panel^T, run by ONE thread-block cluster (<= 16 CTAs on
// one GPC) so that the b sequential pivot steps synchronise through the
// hardware cluster barrier and distributed shared memory instead of global
// memory.
//
// Reference semantics (pivoted_qr.py):
//   qr_column_pivoting  :74-87   exact column norms recomputed every step,
//                                first maximum wins (ties -> lowest position)
//   _reflect            :43-61   alpha = -sign(x0)||x||, v = x - alpha e1,
//                                beta = 2/v'v, w = beta * (v' R), R -= v w',
//                                R[k,k] = alpha, R[k+1:,k] = 0; skipped when
//                                ||x|| == 0 or v'v == 0
//   householder_qr      :64-71   the same steps with the pivot order fixed
// The norms and the reflector sums use numpy's pairwise order bit for bit
// (pairwise_sum); squares and outer-product updates are rounded separately
// (no FMA contraction), as numpy computes them.  The dot products v'R play
// the role of OpenBLAS dgemv and use a fixed 8-accumulator order (any order
// is within the reference's own cross-BLAS rounding envelope).
//
// Storage: CTA c owns columns [c*per, c*per + nl).  Each column (one panel
// row, h doubles) lives in shared memory as column jl of an h x capPad array
// (thread-per-column access is bank-conflict free); columns beyond `cap`
// spill to an L2-resident global scratch with the same layout.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

namespace cg = cooperative_groups;

#define PRRP_MAXCPT 4          // columns per thread
#define PRRP_CLUSTER_MAX 16

struct PanelArgs {
  const double* src;        // panel row j: src[row(j)*ld + 0..h)
  int64_t ld;
  const int64_t* rowidx;    // optional: row(j) = rowidx[j]; else row(j) = j
  int h;                    // transposed-panel rows (panel width), <= 128
  int64_t p;                // transposed-panel columns (panel rows)
  int bsel;                 // leading block for the strong RRQR (<= h)
  int steps;                // min(h, p)
  int mode;                 // 0 = pivoted (QRCP); 1 = fixed order given by perm (pos -> j)
  int32_t* perm;            // mode 1 input and always output: pos -> j
  double* Rbuf;             // out: h x p, Rbuf[i*p + pos]
  double* refl;             // optional out: steps x (h+1) reflector log (v, beta)
  double* ovf;              // overflow scratch (C * h * ovpad doubles)
  int64_t per;              // columns per CTA
  int cap;                  // columns per CTA kept in shared memory
  int cap_pad;              // odd pitch of the shared column array
  int64_t ovpad;            // pitch of the overflow array (>= per - cap)
  DevState* st;
  int panel_id;
  // finalize / swap-loop inputs
  double tau;
  const double* cand;       // per-block worst |lt| from the trsm kernel
  const long long* cand_flat;
  int ncand;
  double* L21;              // (p - bsel) x bsel column-major (ldl)
  int64_t ldl;
  int32_t* swaps_out;       // host-visible per-panel swap count (device pointer)
  int32_t* moved;           // out: compact list of moved positions (dst pos, src j) pairs
  int32_t* moved_cnt;       // optional out: number of moved pairs (besides DevState::moved)
  long long* prof;          // optional: per-phase clock64 totals of CTA 0 (diagnostics)
  int swap_slot;            // index into swaps_dev for this node's swap count
  int tree_level, tree_index;   // CALU tournament node (error payload), -1 otherwise
  double* fro;              // out (mode 0): ||panel||_F of this node
  // panel2 multi-cluster mode (mode 0 only): ngroups clusters exchange their
  // winners through global memory each step
  int ngroups;              // 0/1: one cluster
  double* xg;               // 2 x ngroups x P2_XS doubles (step-parity slots)
  unsigned long long* xflag;   // ngroups flags: epoch + k + 1 once group g published step k
  unsigned long long epoch;
  int fused_ak;             // panel2: fused apply + next-key pass over the shared rows
  // CALU tournament nodes (tournament.py:118-152); all nullptr elsewhere
  const int32_t* live;      // members actually present (<= p; the rest are dead zero rows);
                            // live <= bsel: the node passes its members through unselected
  int32_t* want;            // out: rows the node selects (< bsel after a rank-deficient retry)
  int32_t* node_rows;       // out (per node slot, like swaps_out): live member count
};

// "this node passes its members through" (tournament.py:128-129: idx.shape[0] <= b)
__device__ __forceinline__ bool node_passes(const PanelArgs& a) { return a.live && *a.live <= a.bsel; }

// The run-state error flag read consistently by every CTA of a cluster: a
// concurrent kernel (another tournament node, the look-ahead streams) may
// set it between the CTAs' own reads, and a CTA that returned early would
// leave the others waiting at a cluster barrier.  CTA 0 reads, one cluster
// barrier, everyone follows; a failed cluster passes a second barrier so
// CTA 0's flag stays readable until all have read it.  `flag` is a shared
// int of the calling kernel.  Returns true when the kernel must return.
__device__ __forceinline__ bool cluster_failed(const DevState* st, int* flag) {
  cg::cluster_group cl = cg::this_cluster();
  if (cl.num_blocks() == 1) return prrp_failed(st);
  if (threadIdx.x == 0) *flag = prrp_failed(st);
  cl.sync();
  const int f = *cl.map_shared_rank(flag, 0);
  if (f) cl.sync();
  return f != 0;
}

struct Rec {
  double key;
  long long pos;
  int jl;
  int pad;
};

struct PanelShared {
  double pub[2][PRRP_MAXH];
  double xs[PRRP_MAXH];
  double vs[PRRP_MAXH];
  Rec rec[2];
  Rec wbest[32];
  double red[40];
  double fro_part;
  double beta, alpha;
  int skip;
  int wc, wjl;
  long long wpos;
};

__device__ __forceinline__ double sq_rn(double x) { return mul_rn(x, x); }

// pairwise sum of squares of x[0..n) by one warp (result broadcast to all lanes)
__device__ __forceinline__ double warp_pairwise_sq(const double* x, int n) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  if (n < 8) {
    if (lane == 0) {
      s = -0.0;
      for (int i = 0; i < n; ++i) s = add_rn(s, sq_rn(x[i]));
    }
  } else {
    const int full = n - (n % 8);
    double r = 0.0;
    if (lane < 8) {
      // loads first (independent), then the dependent chain
      double v[PRRP_MAXH / 8];
#pragma unroll
      for (int u = 0; u < PRRP_MAXH / 8; ++u) {
        const int i = lane + 8 * u;
        v[u] = i < full ? x[i] : 0.0;
      }
      r = sq_rn(v[0]);
#pragma unroll
      for (int u = 1; u < PRRP_MAXH / 8; ++u)
        if (lane + 8 * u < full) r = add_rn(r, sq_rn(v[u]));
    }
    r = add_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = add_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = add_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
    if (lane == 0) {
      for (int i = full; i < n; ++i) r = add_rn(r, sq_rn(x[i]));
      s = r;
    }
  }
  return __shfl_sync(0xffffffffu, s, 0);
}

struct ColRef {
  double* base;
  int64_t stride;
  __device__ __forceinline__ double& operator[](int i) const { return base[(int64_t)i * stride]; }
};

__device__ __forceinline__ ColRef col_ref(const PanelArgs& a, double* sdata, int c, int jl) {
  if (jl < a.cap) return ColRef{sdata + jl, (int64_t)a.cap_pad};
  return ColRef{a.ovf + (int64_t)c * a.h * a.ovpad + (jl - a.cap), a.ovpad};
}

// Run the QR steps over the cluster.  On exit Rbuf/perm hold R (by position)
// and the column order; st->fro holds ||panel||_F (mode 0 only).
__device__ void engine_run(const PanelArgs& a, int mode, const int32_t* perm_in,
                           double* sdata, PanelShared& S) {
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks();
  const int c = (int)cl.block_rank();
  const int T = blockDim.x, t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5, nwarp = (T + 31) >> 5;
  const int h = a.h;
  const int64_t j0 = (int64_t)c * a.per;
  const int nl = (int)max((int64_t)0, min(a.per, a.p - j0));

  // ---- load: one warp per panel row, lanes over the h entries (coalesced)
  for (int jl = warp; jl < nl; jl += nwarp) {
    const int64_t q = j0 + jl;
    const int64_t j = mode == 0 ? q : (int64_t)perm_in[q];
    const int64_t row = a.rowidx ? a.rowidx[j] : j;
    const double* s = member_row(a.src, a.ld, row);
    ColRef col = col_ref(a, sdata, c, jl);
    for (int i = lane; i < h; i += 32) col[i] = s[i];
  }
  __syncthreads();

  long long pos[PRRP_MAXCPT];
  double key[PRRP_MAXCPT];
  double fro_part = 0.0;
#pragma unroll
  for (int u = 0; u < PRRP_MAXCPT; ++u) {
    const int jl = t + u * T;
    pos[u] = j0 + jl;
    key[u] = -1.0;
    if (jl < nl) {
      ColRef col = col_ref(a, sdata, c, jl);
      const double nrm = pairwise_sum(h, [&](int i) { return sq_rn(col[i]); });
      fro_part += nrm;
      key[u] = mode == 0 ? nrm : (pos[u] == 0 ? 1.0 : -1.0);
    }
  }
  if (mode == 0) {
    // cluster-wide ||panel||_F^2 (summation order: per column, per thread, per block)
    for (int o = 16; o; o >>= 1) fro_part += __shfl_xor_sync(0xffffffffu, fro_part, o);
    if (lane == 0) S.red[warp] = fro_part;
    __syncthreads();
    if (t == 0) {
      double f = 0.0;
      for (int w = 0; w < nwarp; ++w) f += S.red[w];
      S.fro_part = f;
    }
  }

  for (int k = 0; k < a.steps; ++k) {
    const int buf = k & 1;
    // ---- CTA best among active columns (pos >= k)
    double bk = -INFINITY;
    long long bp = LLONG_MAX;
    int bj = -1;
#pragma unroll
    for (int u = 0; u < PRRP_MAXCPT; ++u) {
      const int jl = t + u * T;
      if (jl < nl && pos[u] >= k && better(key[u], pos[u], bk, bp)) { bk = key[u]; bp = pos[u]; bj = jl; }
    }
    for (int o = 16; o; o >>= 1) {
      const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const long long op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (better(ok, op, bk, bp)) { bk = ok; bp = op; bj = oj; }
    }
    if (lane == 0) { S.wbest[warp].key = bk; S.wbest[warp].pos = bp; S.wbest[warp].jl = bj; }
    __syncthreads();
    if (warp == 0) {
      Rec r = lane < nwarp ? S.wbest[lane] : Rec{-INFINITY, LLONG_MAX, -1, 0};
      for (int o = 16; o; o >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, r.key, o);
        const long long op = __shfl_xor_sync(0xffffffffu, r.pos, o);
        const int oj = __shfl_xor_sync(0xffffffffu, r.jl, o);
        if (better(ok, op, r.key, r.pos)) { r.key = ok; r.pos = op; r.jl = oj; }
      }
      if (lane == 0) S.rec[buf] = r;
      if (r.jl >= 0) {
        ColRef col = col_ref(a, sdata, c, r.jl);
        for (int i = k + lane; i < h; i += 32) S.pub[buf][i] = col[i];
      }
    }
    cl.sync();

    // ---- warp 0: agree on the winner, fetch its column, build the reflector
    if (warp == 0) {
      Rec r{-INFINITY, LLONG_MAX, -1, 0};
      int rc = -1;
      if (lane < C) {
        const Rec* rr = cl.map_shared_rank(&S.rec[buf], lane);
        r = *rr;
        rc = lane;
      }
      for (int o = 16; o; o >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, r.key, o);
        const long long op = __shfl_xor_sync(0xffffffffu, r.pos, o);
        const int oj = __shfl_xor_sync(0xffffffffu, r.jl, o);
        const int oc = __shfl_xor_sync(0xffffffffu, rc, o);
        if (better(ok, op, r.key, r.pos)) { r.key = ok; r.pos = op; r.jl = oj; rc = oc; }
      }
      const double* rpub = cl.map_shared_rank(&S.pub[buf][0], rc);
      for (int i = k + lane; i < h; i += 32) S.xs[i] = rpub[i];
      if (k == 0 && mode == 0 && c == 0) {
        double f = 0.0;
        if (lane < C) f = *cl.map_shared_rank(&S.fro_part, lane);
        for (int o = 16; o; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
        if (lane == 0) *a.fro = sqrt(f);
      }
      __syncwarp();
      const int L = h - k;
      const double nx2 = warp_pairwise_sq(S.xs + k, L);
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
        S.wc = rc; S.wjl = r.jl; S.wpos = r.pos;
      }
      if (a.refl && c == 0) {
        double* lg = a.refl + (int64_t)k * (h + 1);
        for (int i = lane; i < h; i += 32) lg[i] = (skip || i < k) ? 0.0 : S.vs[i];
        if (lane == 0) lg[h] = skip ? 0.0 : beta;
      }
    }
    __syncthreads();

    // ---- apply reflector k to every active column, then norms for step k+1
    const int skip = S.skip;
    const double beta = S.beta, alpha = S.alpha;
    const int wc = S.wc, wjl = S.wjl;
    const long long wpos = S.wpos;
    const double* vs = S.vs;
#pragma unroll
    for (int u = 0; u < PRRP_MAXCPT; ++u) {
      const int jl = t + u * T;
      if (jl >= nl || pos[u] < k) continue;
      ColRef col = col_ref(a, sdata, c, jl);
      if (c == wc && jl == wjl) {               // the pivot column moves to position k
        pos[u] = k;
        if (!skip) {
          col[k] = alpha;
          for (int i = k + 1; i < h; ++i) col[i] = 0.0;
        }
        continue;
      }
      if (pos[u] == k) pos[u] = wpos;           // column displaced by the interchange
      double w = 0.0;
      if (!skip) {
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0, a7 = 0;
        int i = k;
        for (; i + 8 <= h; i += 8) {
          a0 = fma(vs[i + 0], col[i + 0], a0); a1 = fma(vs[i + 1], col[i + 1], a1);
          a2 = fma(vs[i + 2], col[i + 2], a2); a3 = fma(vs[i + 3], col[i + 3], a3);
          a4 = fma(vs[i + 4], col[i + 4], a4); a5 = fma(vs[i + 5], col[i + 5], a5);
          a6 = fma(vs[i + 6], col[i + 6], a6); a7 = fma(vs[i + 7], col[i + 7], a7);
        }
        for (; i < h; ++i) a0 = fma(vs[i], col[i], a0);
        const double dot = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
        w = mul_rn(beta, dot);
        col[k] = sub_rn(col[k], mul_rn(vs[k], w));
      }
      if (mode == 0) {
        const int base = k + 1;
        if (!skip) {
          key[u] = pairwise_sum(h - base, [&](int ii) {
            const int i = base + ii;
            const double x = sub_rn(col[i], mul_rn(vs[i], w));
            col[i] = x;
            return sq_rn(x);
          });
        } else {
          key[u] = pairwise_sum(h - base, [&](int ii) { return sq_rn(col[base + ii]); });
        }
      } else {
        if (!skip)
          for (int i = k + 1; i < h; ++i) col[i] = sub_rn(col[i], mul_rn(vs[i], w));
        key[u] = pos[u] == k + 1 ? 1.0 : -1.0;
      }
    }
  }
  cl.sync();

  // ---- write R (by position) and the column order
#pragma unroll
  for (int u = 0; u < PRRP_MAXCPT; ++u) {
    const int jl = t + u * T;
    if (jl >= nl) continue;
    ColRef col = col_ref(a, sdata, c, jl);
    const int64_t q = j0 + jl;
    const int64_t j = mode == 0 ? q : (int64_t)perm_in[q];
    for (int i = 0; i < h; ++i) a.Rbuf[(int64_t)i * a.p + pos[u]] = col[i];
    a.perm[pos[u]] = (int32_t)j;
  }
}

__global__ void __launch_bounds__(1024, 1) panel_qrcp_kernel(PanelArgs a) {
  extern __shared__ __align__(16) double dyn_smem[];
  __shared__ PanelShared S;
  __shared__ int s_failed;
  if (node_passes(a) || cluster_failed(a.st, &s_failed)) return;
  engine_run(a, a.mode, a.perm, dyn_smem, S);
}
