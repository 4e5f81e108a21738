// Thread-per-column panel QRCP engine for panel width h = 128 (BASELINE
// configs 2b and 5: LU_PRRP b = 128, CALU_PRRP tournament leaves and merge
// nodes, the CALU final QR).  Same arithmetic contract as panel.cuh /
// panel1.cuh (pivoted_qr.py:43-87) and the same per-step organisation as
// panel1.cuh (warp argmax -> the warp's best column builds its reflector ->
// CTA argmax -> 48-byte record pushed into every CTA with st.async ->
// cluster argmax -> the winner's v pulled once per CTA -> apply + next keys).
//
// A 128-double column does not fit one thread's registers, so a column is
// split: a 64-row REGISTER WINDOW plus the rows below it in shared memory
// ([row][thread] layout, conflict free).  The window is shifted like
// panel1's: during steps 8*KB .. 8*KB+7 register element i is absolute row
// 8*KB + i, rows 8*KB+64 .. 127 are in shared memory; at every block
// boundary the finished rows go to the global row-save area and 8 rows move
// from shared memory into the window.  From step 64 on, the column is
// entirely in registers.  One column per thread, <= 256 per CTA, <= 4096 per
// 16-CTA cluster.  Taller panels (LU_PRRP b = 128, p <= 8192) run as
// `ngroups` co-resident clusters: each cluster's winner CTA publishes its
// record and reflector to a global step-parity slot and releases a flag
// (epoch + k + 1); every CTA acquires the other groups' flags, takes the
// lexicographic best (largest key, then lowest global position) and, if it
// lies in another cluster, loads that reflector from L2.
#pragma once
#include "panel1.cuh"

#define P2_H 128
#define P2_W 64                  // register window
#define P2_T 256
#define P2_NW (P2_T / 32)
#define P2_RS (P2_T * 8)         // shared row stride (bytes)
#define P2_XS 136                // global exchange slot: 8 record doubles + 128 v
#ifndef P2_UNR
#define P2_UNR 1                 // unroll of the shared-memory block loops (ILP across blocks)
#endif
constexpr int kP2Unr = P2_UNR;

struct P2Shared {
  double wpub[2][P2_NW][P2_H];
  double vs[P2_H];
  P1Rec wrec[2][P2_NW];
  P1Rec rec[2][PRRP_CLUSTER_MAX];
  unsigned long long bar[2];
  double fro_warp[P2_NW];
  double alog[P2_H];
  int slog[P2_H];
  double fro;
  int failed;
  int gwin;                 // multi-cluster: group of the global winner
  double grec[8];           // its record (key, pos, alpha, beta, fro, jl|skip)
  double gx[4][P2_XS];      // staged remote records + reflectors (<= 4 groups)
};

// element i (relative to row 8*KB) of a split column: i < 64 in registers,
// i >= 64 at sb + (i - 64) * P2_RS (sb = the thread's shared row 8*KB)
struct P2Col {
  double (&r)[P2_W];
  uint32_t sb;
  __device__ __forceinline__ double ld(int i) const { return i < P2_W ? r[i] : lds_f64(sb + (uint32_t)(i - P2_W) * P2_RS); }
  __device__ __forceinline__ void st(int i, double v) const {
    if (i < P2_W) r[i] = v;
    else sts_f64(sb + (uint32_t)(i - P2_W) * P2_RS, v);
  }
};

// numpy pairwise sum of squares of all 128 rows (16 full 8-groups, no remainder)
__device__ __forceinline__ double p2_norm_full(const P2Col& x) {
  double S[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) S[s] = sq_rn(x.ld(s));
#pragma unroll
  for (int B = 1; B < 8; ++B)
#pragma unroll
    for (int s = 0; s < 8; ++s) S[s] = add_rn(S[s], sq_rn(x.ld(8 * B + s)));
#pragma unroll 1
  for (int B = 8; B < 16; ++B)
#pragma unroll
    for (int s = 0; s < 8; ++s) S[s] = add_rn(S[s], sq_rn(x.ld(8 * B + s)));
  return add_rn(add_rn(add_rn(S[0], S[1]), add_rn(S[2], S[3])), add_rn(add_rn(S[4], S[5]), add_rn(S[6], S[7])));
}

// numpy pairwise sum of squares of the relative rows r0 .. 8L+7 (p1_sumsq
// for up to 16 blocks: register blocks unrolled, shared blocks rolled)
__device__ __forceinline__ double p2_sumsq(const P2Col& x, int r0, int L) {
  if (L == 0 && r0 > 0) {
    double res = -0.0;
#pragma unroll
    for (int s = 1; s < 8; ++s)
      if (s >= r0) res = add_rn(res, sq_rn(x.ld(s)));
    return res;
  }
  double S[8], T[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const double q = sq_rn(x.ld(s));
    S[s] = s >= r0 ? q : 0.0;
    T[s] = 0.0;
  }
#pragma unroll
  for (int B = 1; B < 8; ++B) {
    if (B > L) break;
    if (B < L) {
#pragma unroll
      for (int s = 0; s < 8; ++s) S[s] = add_rn(S[s], sq_rn(x.ld(8 * B + s)));
    } else {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        T[s] = sq_rn(x.ld(8 * B + s));
        if (s < r0) S[s] = add_rn(S[s], T[s]);
      }
    }
  }
#pragma unroll kP2Unr
  for (int B = 8; B <= L; ++B) {
    const uint32_t a = x.sb + (uint32_t)(8 * B - P2_W) * P2_RS;
    double q[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) q[s] = sq_rn(lds_f64(a + (uint32_t)s * P2_RS));
    if (B < L) {
#pragma unroll
      for (int s = 0; s < 8; ++s) S[s] = add_rn(S[s], q[s]);
    } else {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        T[s] = q[s];
        if (s < r0) S[s] = add_rn(S[s], T[s]);
      }
    }
  }
  if (L == 0) return p1_combine(S, 0);
  double res = p1_combine(S, r0 & 7);
#pragma unroll
  for (int s = 0; s < 8; ++s)
    if (s >= r0) res = add_rn(res, T[s]);
  return res;
}

// apply reflector k (relative pivot row r = k & 7) on blocks 0..L
__device__ __forceinline__ void p2_apply(const P2Col& x, const double* vp, double beta, bool act, int L) {
  const uint32_t va = (uint32_t)__cvta_generic_to_shared(vp);
  double d[4];
#pragma unroll
  for (int B = 0; B < 8; ++B) {
    if (B > L) break;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const double2 v = lds2_f64(va + 64 * B + 16 * h);
      const int s = 2 * h;
      if (B == 0 && s < 4) {
        d[s] = mul_rn(v.x, x.ld(s));
        d[s + 1] = mul_rn(v.y, x.ld(s + 1));
      } else {
        d[s & 3] = fma(v.x, x.ld(8 * B + s), d[s & 3]);
        d[(s + 1) & 3] = fma(v.y, x.ld(8 * B + s + 1), d[(s + 1) & 3]);
      }
    }
  }
#pragma unroll kP2Unr
  for (int B = 8; B <= L; ++B) {
    const uint32_t a = x.sb + (uint32_t)(8 * B - P2_W) * P2_RS;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const double2 v = lds2_f64(va + 64 * B + 16 * h);
      d[(2 * h) & 3] = fma(v.x, lds_f64(a + (uint32_t)(2 * h) * P2_RS), d[(2 * h) & 3]);
      d[(2 * h + 1) & 3] = fma(v.y, lds_f64(a + (uint32_t)(2 * h + 1) * P2_RS), d[(2 * h + 1) & 3]);
    }
  }
  const double dot = (d[0] + d[1]) + (d[2] + d[3]);
  const double nw = act ? -mul_rn(beta, dot) : 0.0;
#pragma unroll
  for (int B = 0; B < 8; ++B) {
    if (B > L) break;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const double2 v = lds2_f64(va + 64 * B + 16 * h);
      const int s = 8 * B + 2 * h;
      x.r[s] = fma(v.x, nw, x.r[s]);
      x.r[s + 1] = fma(v.y, nw, x.r[s + 1]);
    }
  }
  if (!act) return;
#pragma unroll kP2Unr
  for (int B = 8; B <= L; ++B) {
    const uint32_t a = x.sb + (uint32_t)(8 * B - P2_W) * P2_RS;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const double2 v = lds2_f64(va + 64 * B + 16 * h);
      const uint32_t a0 = a + (uint32_t)(2 * h) * P2_RS;
      sts_f64(a0, fma(v.x, nw, lds_f64(a0)));
      sts_f64(a0 + P2_RS, fma(v.y, nw, lds_f64(a0 + P2_RS)));
    }
  }
}

// apply reflector k and compute the next key (p2_sumsq of the relative rows
// r0 .. 8L+7) in one pass over the shared rows, for L >= 8 (shared rows
// present): the register rows are updated and squared first, then every
// shared row is loaded once, updated, stored and squared, so the pairwise
// accumulation order is p2_sumsq's (blocks in increasing order).
__device__ __forceinline__ double p2_apply_key(const P2Col& x, const double* vp, double beta, bool act,
                                               bool do_apply, int L, int r0) {
  const uint32_t va = (uint32_t)__cvta_generic_to_shared(vp);
  double nw = 0.0;
  if (do_apply) {
    double d[4];
#pragma unroll
    for (int B = 0; B < 8; ++B) {
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 v = lds2_f64(va + 64 * B + 16 * h);
        const int s = 2 * h;
        if (B == 0 && s < 4) {
          d[s] = mul_rn(v.x, x.ld(s));
          d[s + 1] = mul_rn(v.y, x.ld(s + 1));
        } else {
          d[s & 3] = fma(v.x, x.ld(8 * B + s), d[s & 3]);
          d[(s + 1) & 3] = fma(v.y, x.ld(8 * B + s + 1), d[(s + 1) & 3]);
        }
      }
    }
#pragma unroll 1
    for (int B = 8; B <= L; ++B) {
      const uint32_t a = x.sb + (uint32_t)(8 * B - P2_W) * P2_RS;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 v = lds2_f64(va + 64 * B + 16 * h);
        d[(2 * h) & 3] = fma(v.x, lds_f64(a + (uint32_t)(2 * h) * P2_RS), d[(2 * h) & 3]);
        d[(2 * h + 1) & 3] = fma(v.y, lds_f64(a + (uint32_t)(2 * h + 1) * P2_RS), d[(2 * h + 1) & 3]);
      }
    }
    const double dot = (d[0] + d[1]) + (d[2] + d[3]);
    nw = act ? -mul_rn(beta, dot) : 0.0;
#pragma unroll
    for (int B = 0; B < 8; ++B) {
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 v = lds2_f64(va + 64 * B + 16 * h);
        const int s = 8 * B + 2 * h;
        x.r[s] = fma(v.x, nw, x.r[s]);
        x.r[s + 1] = fma(v.y, nw, x.r[s + 1]);
      }
    }
  }
  const bool upd = do_apply && act;
  double S[8], T[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const double q = sq_rn(x.ld(s));
    S[s] = s >= r0 ? q : 0.0;
    T[s] = 0.0;
  }
#pragma unroll
  for (int B = 1; B < 8; ++B)
#pragma unroll
    for (int s = 0; s < 8; ++s) S[s] = add_rn(S[s], sq_rn(x.ld(8 * B + s)));
#pragma unroll 1
  for (int B = 8; B <= L; ++B) {
    const uint32_t a = x.sb + (uint32_t)(8 * B - P2_W) * P2_RS;
    double q[8];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const uint32_t a0 = a + (uint32_t)(2 * h) * P2_RS;
      double x0 = lds_f64(a0), x1 = lds_f64(a0 + P2_RS);
      if (upd) {
        const double2 v = lds2_f64(va + 64 * B + 16 * h);
        x0 = fma(v.x, nw, x0);
        x1 = fma(v.y, nw, x1);
        sts_f64(a0, x0);
        sts_f64(a0 + P2_RS, x1);
      }
      q[2 * h] = sq_rn(x0);
      q[2 * h + 1] = sq_rn(x1);
    }
    if (B < L) {
#pragma unroll
      for (int s = 0; s < 8; ++s) S[s] = add_rn(S[s], q[s]);
    } else {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        T[s] = q[s];
        if (s < r0) S[s] = add_rn(S[s], T[s]);
      }
    }
  }
  double res = p1_combine(S, r0 & 7);
#pragma unroll
  for (int s = 0; s < 8; ++s)
    if (s >= r0) res = add_rn(res, T[s]);
  return res;
}

// the warp's best column builds its reflector (p1_candidate for the split column)
// (copy_smem = false: the shared-memory rows of v are copied by the whole warp
// afterwards, p2_copy_smem_rows)
__device__ __forceinline__ void p2_candidate(const P2Col& x, int r, int L, int mode, double key, double* wp,
                                             int& skip, double& alpha, double& beta, bool copy_smem = true) {
  double xk = x.ld(0);
#pragma unroll
  for (int s = 1; s < 8; ++s)
    if (s == r) xk = x.ld(s);
  const double normx = __dsqrt_rn(mode == 0 ? key : p2_sumsq(x, r, L));
  skip = normx == 0.0;
  alpha = xk >= 0.0 ? -normx : normx;
  const double vk = sub_rn(xk, alpha);
  double2* w2 = reinterpret_cast<double2*>(wp);
#pragma unroll
  for (int s = 0; s < 8; s += 2) {
    const double a0 = s < r ? 0.0 : (s == r ? vk : x.ld(s));
    const double a1 = s + 1 < r ? 0.0 : (s + 1 == r ? vk : x.ld(s + 1));
    w2[s / 2] = make_double2(a0, a1);
  }
#pragma unroll
  for (int B = 1; B < 8; ++B) {
    if (B > L) break;
#pragma unroll
    for (int s = 0; s < 8; s += 2) w2[4 * B + s / 2] = make_double2(x.ld(8 * B + s), x.ld(8 * B + s + 1));
  }
  if (copy_smem) {
#pragma unroll kP2Unr
    for (int B = 8; B <= L; ++B) {
      const uint32_t a = x.sb + (uint32_t)(8 * B - P2_W) * P2_RS;
#pragma unroll
      for (int s = 0; s < 8; s += 2)
        w2[4 * B + s / 2] = make_double2(lds_f64(a + (uint32_t)s * P2_RS), lds_f64(a + (uint32_t)(s + 1) * P2_RS));
    }
  }
  const double half_vtv = mul_rn(normx, add_rn(normx, fabs(xk)));
  beta = skip ? 0.0 : __drcp_rn(half_vtv);
  if (half_vtv == 0.0) skip = 1;
  if (skip) { alpha = xk; beta = 0.0; }
}

// the shared-memory rows (relative 64 .. 8L+7) of thread tw's column into v,
// one row per lane (sb0 = shared address of row 8*KB of thread 0's column)
__device__ __forceinline__ void p2_copy_smem_rows(uint32_t sb0, int tw, int L, double* wp, int lane) {
  for (int i = P2_W + lane; i < 8 * (L + 1); i += 32)
    wp[i] = lds_f64(sb0 + (uint32_t)(i - P2_W) * P2_RS + (uint32_t)tw * 8);
}

__global__ void __launch_bounds__(P2_T, 1) panel_qrcp2_kernel(PanelArgs a) {
  if (node_passes(a)) return;   // uniform over the cluster (read before any cluster barrier)
  extern __shared__ __align__(16) double sdata[];      // (P2_H - P2_W) x P2_T shared rows
  __shared__ __align__(16) P2Shared S;
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks();
  const int c = (int)cl.block_rank();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&S.bar[0]);
  const uint32_t bar1 = (uint32_t)__cvta_generic_to_shared(&S.bar[1]);
  if (t == 0) {
    p1_bar_init(bar0);
    p1_bar_init(bar1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    S.failed = prrp_failed(a.st);
  }
  cl.sync();
  if (*cl.map_shared_rank(&S.failed, 0)) { cl.sync(); return; }
  const int mode = a.mode;
  const int G = a.ngroups > 1 ? a.ngroups : 1;
  const int grp = (int)(blockIdx.x / (unsigned)C);
  const int64_t j0 = ((int64_t)grp * C + c) * a.per;
  const int nl = (int)max((int64_t)0, min(a.per, a.p - j0));
  const bool on = t < nl;
  double* rsave = a.ovf;             // finished rows: rsave[row * p + j0 + t]

  double rr[P2_W];
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(sdata + t);   // shared row 64 of this thread's column
  if (on) {
    const int64_t qq = j0 + t;
    const int64_t j = mode == 0 ? qq : (int64_t)a.perm[qq];
    const int64_t row = a.rowidx ? a.rowidx[j] : j;
    const double2* src = reinterpret_cast<const double2*>(member_row(a.src, a.ld, row));
#pragma unroll
    for (int i = 0; i < P2_W / 2; ++i) { const double2 v = src[i]; rr[2 * i] = v.x; rr[2 * i + 1] = v.y; }
#pragma unroll 8
    for (int i = 0; i < (P2_H - P2_W) / 2; ++i) {
      const double2 v = src[P2_W / 2 + i];
      sts_f64(s0 + (uint32_t)(2 * i) * P2_RS, v.x);
      sts_f64(s0 + (uint32_t)(2 * i + 1) * P2_RS, v.y);
    }
  } else {
#pragma unroll
    for (int i = 0; i < P2_W; ++i) rr[i] = 0.0;
#pragma unroll 8
    for (int i = 0; i < P2_H - P2_W; ++i) sts_f64(s0 + (uint32_t)i * P2_RS, 0.0);
  }
  long long pos = j0 + t;
  double key = -1.0;
  if (mode == 0) {
    double fro = 0.0;
    if (on) { key = p2_norm_full(P2Col{rr, s0}); fro = key; }
    for (int o = 16; o; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
    if (lane == 0) S.fro_warp[warp] = fro;
  } else {
    key = on && pos == 0 ? 1.0 : -1.0;
  }
  __syncthreads();
  if (t == 0) {
    double f = 0.0;
    for (int w = 0; w < P2_NW; ++w) f += S.fro_warp[w];
    S.fro = f;
  }
  const bool log_refl = a.refl != nullptr && c == 0;
  const bool fused_ak = a.fused_ak != 0;
  // PRRP_PANEL_PROF=1 PRRP_PANEL_TL=<panel>: clock64 marks of thread 0 of CTA 0
  long long* tl = (a.prof && grp == 0 && c == 0 && t == 0 && a.panel_id == a.prof[6]) ? a.prof + 8 : nullptr;
#define P2_TL(m) if (tl) tl[k * 8 + (m)] = clock64();

  int KB = 0;
  for (int k = 0; k < a.steps; ++k) {
    const int buf = k & 1;
    const int r = k & 7;
    if (r == 0 && k > 0) {
      // block boundary: rows 8*KB .. 8*KB+7 are final; shift the window up by
      // 8 and pull rows 8*KB+64 .. 8*KB+71 in from shared memory
      if (on) {
#pragma unroll
        for (int s = 0; s < 8; ++s) rsave[(int64_t)(8 * KB + s) * a.p + j0 + t] = rr[s];
      }
#pragma unroll
      for (int i = 0; i < P2_W - 8; ++i) rr[i] = rr[i + 8];
      if (KB < 8) {
#pragma unroll
        for (int s = 0; s < 8; ++s) rr[P2_W - 8 + s] = lds_f64(s0 + (uint32_t)(8 * KB + s) * P2_RS);
      } else {
#pragma unroll
        for (int s = 0; s < 8; ++s) rr[P2_W - 8 + s] = 0.0;
      }
      ++KB;
    }
    const int L = 15 - KB;
    P2_TL(0)
    const P2Col x{rr, s0 + (uint32_t)(8 * KB) * P2_RS};
    const uint32_t bar = buf ? bar1 : bar0;
    if (t == 0 && C > 1) p1_bar_expect(bar, (uint32_t)(C * (int)sizeof(P1Rec)));
    // ---- warp argmax; the lane of the warp's best column builds its reflector
    {
      const bool live = on && pos >= k;
      const unsigned long long u = p1_ukey(key, live);
      const int wl = p1_best_lane(u, (unsigned)pos);
      P1Rec& wr = S.wrec[buf][warp];
      if (wl < 0) {
        if (lane == 0) { wr.key = -INFINITY; wr.pos = LLONG_MAX; wr.jl = -1; wr.skip = 1; }
      } else {
        if (lane == wl) {
          int skip;
          double alpha, beta;
          p2_candidate(x, r, L, mode, key, S.wpub[buf][warp], skip, alpha, beta, false);
          wr.key = key; wr.pos = pos; wr.jl = t;
          wr.skip = skip; wr.alpha = alpha; wr.beta = beta;
        }
        if (L >= 8)
          p2_copy_smem_rows((uint32_t)__cvta_generic_to_shared(sdata) + (uint32_t)(8 * KB) * P2_RS, warp * 32 + wl,
                            L, S.wpub[buf][warp], lane);
      }
      __syncwarp();
    }
    P2_TL(1)
    __syncthreads();
    P2_TL(2)
    // ---- CTA argmax; warp 0 pushes the CTA candidate into every CTA
    const P1Rec* Wp;
    int rc;
    if (C == 1) {
      const bool ok = lane < P2_NW && S.wrec[buf][lane].jl >= 0;
      const unsigned long long u = ok ? p1_ukey(S.wrec[buf][lane].key, true) : 0ull;
      int w = p1_best_lane(u, ok ? (unsigned)S.wrec[buf][lane].pos : 0xffffffffu);
      if (w < 0) w = 0;
      Wp = &S.wrec[buf][w];
      rc = 0;
      if (k == 0 && mode == 0 && warp == 0 && lane == 0) *a.fro = sqrt(S.fro);
    } else {
      if (warp == 0) {
        const bool ok = lane < P2_NW && S.wrec[buf][lane].jl >= 0;
        const unsigned long long u = ok ? p1_ukey(S.wrec[buf][lane].key, true) : 0ull;
        const unsigned pp = ok ? (unsigned)S.wrec[buf][lane].pos : 0xffffffffu;
        int w = p1_best_lane(u, pp);
        if (w < 0) w = 0;
        if (lane < C) {
          const P1Rec& b = S.wrec[buf][w];
          const uint32_t rbar = p1_mapa(bar, lane);
          const uint32_t dst = p1_mapa((uint32_t)__cvta_generic_to_shared(&S.rec[buf][c]), lane);
          p1_push16(dst, b.key, __longlong_as_double(b.pos), rbar);
          p1_push16(dst + 16, __longlong_as_double((long long)(unsigned)b.jl | ((long long)b.skip << 32)),
                    b.alpha, rbar);
          p1_push16(dst + 32, b.beta, S.fro, rbar);
        }
      }
      p1_bar_wait(bar, (uint32_t)((k >> 1) & 1));
      P2_TL(3)
      {
        const bool ok = lane < C && S.rec[buf][lane].jl >= 0;
        const unsigned long long u = ok ? p1_ukey(S.rec[buf][lane].key, true) : 0ull;
        rc = p1_best_lane(u, ok ? (unsigned)S.rec[buf][lane].pos : 0xffffffffu);
        if (rc < 0) rc = 0;
      }
      Wp = &S.rec[buf][rc];
    }
    const P1Rec& W = *Wp;
    long long wpos = W.pos;
    int skip = W.skip;
    double beta = W.beta, alpha = W.alpha;
    int wjl = W.jl;
    bool mine = rc == c;
    int ww = wjl >> 5;
    bool remote = false;             // the global winner is in another cluster
    if (G > 1) {
      // ---- cross-cluster exchange through global memory
      const unsigned long long tag = a.epoch + (unsigned long long)k + 1ull;
      if (mine && warp == 0) {
        double* slot = a.xg + ((int64_t)buf * G + grp) * P2_XS;
        if (lane == 0) {
          double cf = 0.0;
          if (k == 0 && mode == 0)
            for (int q = 0; q < C; ++q) cf += S.rec[buf][q].fro;
          slot[0] = W.key;
          slot[1] = __longlong_as_double(W.pos);
          slot[2] = W.alpha;
          slot[3] = W.beta;
          slot[4] = cf;
          slot[5] = __longlong_as_double((long long)(unsigned)W.jl | ((long long)W.skip << 32));
        }
        if (!W.skip)
          for (int i = lane; i < 8 * (L + 1); i += 32) slot[8 + i] = S.wpub[buf][ww][i];
        // the warp barrier orders the lanes' stores before lane 0's gpu-scope
        // release (cumulative), which publishes them with the flag
        __syncwarp();
        if (lane == 0)
          asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(a.xflag + grp), "l"(tag) : "memory");
      }
      if (warp == 0) {
        // wait for the other groups' step-k records, then fetch every remote
        // record and reflector in one L2 round trip
        if (lane < G && lane != grp) {
          unsigned long long f;
          do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(a.xflag + lane) : "memory");
          } while (f != tag);
        }
        __syncwarp();
        const int nx = 8 + 8 * (L + 1);
        for (int q = 0; q < G; ++q) {
          if (q == grp) continue;
          const double* slot = a.xg + ((int64_t)buf * G + q) * P2_XS;
          for (int i = lane; i < nx; i += 32) S.gx[q][i] = __ldcg(slot + i);
        }
        __syncwarp();
        double key = -INFINITY;
        long long gp = LLONG_MAX;
        bool ok = false;
        if (lane < G) {
          if (lane == grp) {
            ok = W.jl >= 0;
            key = W.key;
            gp = W.pos;
          } else {
            key = S.gx[lane][0];
            gp = __double_as_longlong(S.gx[lane][1]);
            ok = (int)(unsigned)__double_as_longlong(S.gx[lane][5]) >= 0;
          }
        }
        const unsigned long long u = ok ? p1_ukey(key, true) : 0ull;
        int g = p1_best_lane(u, ok ? (unsigned)gp : 0xffffffffu);
        if (g < 0) g = grp;
        if (lane == 0) S.gwin = g;
        if (g != grp) {
          if (lane < 8) S.grec[lane] = S.gx[g][lane];
          if ((__double_as_longlong(S.gx[g][5]) >> 32) == 0)
            for (int i = lane; i < 8 * (L + 1); i += 32) S.vs[i] = S.gx[g][8 + i];
        }
        if (k == 0 && mode == 0 && grp == 0 && c == 0) {
          // ||panel||_F over the groups, in group order
          double f = 0.0;
          for (int q = 0; q < G; ++q) {
            double cf;
            if (q == grp) {
              cf = 0.0;
              for (int r2 = 0; r2 < C; ++r2) cf += S.rec[buf][r2].fro;
            } else {
              cf = S.gx[q][4];
            }
            f += cf;
          }
          if (lane == 0) *a.fro = sqrt(f);
        }
      }
      __syncthreads();
      if (S.gwin != grp) {
        remote = true;
        mine = false;
        wpos = __double_as_longlong(S.grec[1]);
        alpha = S.grec[2];
        beta = S.grec[3];
        const long long bits = __double_as_longlong(S.grec[5]);
        wjl = (int)(unsigned)bits;
        skip = (int)(bits >> 32);
        ww = wjl >> 5;
      }
    }
    if (t == 0) { S.alog[k] = alpha; S.slog[k] = skip; }
    const double* vs = mine ? S.wpub[buf][ww] : S.vs;
    if (!mine && !remote) {
      if (warp == 0 && !skip) {
        for (int q = lane; q < 4 * (L + 1); q += 32) {       // 16-byte chunks of the live rows
          const uint32_t src = p1_mapa((uint32_t)__cvta_generic_to_shared(&S.wpub[buf][ww][2 * q]), rc);
          double v0, v1;
          p1_pull16(src, v0, v1);
          S.vs[2 * q] = v0;
          S.vs[2 * q + 1] = v1;
        }
      }
      __syncthreads();
    }
    P2_TL(4)
    if (G == 1 && C > 1 && k == 0 && mode == 0 && c == 0 && warp == 0) {
      double f = lane < C ? S.rec[buf][lane].fro : 0.0;
      for (int o = 16; o; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
      if (lane == 0) *a.fro = sqrt(f);
    }
    if (log_refl && warp == P2_NW - 1) {
      double* lg = a.refl + (int64_t)k * (P2_H + 1);
      for (int i = lane; i < P2_H; i += 32) lg[i] = (skip || i < k) ? 0.0 : vs[i - 8 * KB];
      if (lane == 0) lg[P2_H] = skip ? 0.0 : beta;
    }

    // ---- apply reflector k, key for step k+1
    if (__any_sync(0xffffffffu, on && pos >= k)) {
      const bool live = on && pos >= k;
      const bool win = live && mine && wjl == t;
      if (live && !win && pos == k) pos = wpos;
      if (mode == 0 && L >= 8 && fused_ak) {
        const double nk = p2_apply_key(x, vs, beta, live && !win, !skip, L, r + 1);
        if (win) pos = k;
        key = (live && !win) ? nk : -1.0;
      } else if (mode == 0) {
        if (!skip) p2_apply(x, vs, beta, live && !win, L);
        if (win) pos = k;
        const double nk = p2_sumsq(x, r + 1, L);
        key = (live && !win) ? nk : -1.0;
      } else {
        if (!skip) p2_apply(x, vs, beta, live && !win, L);
        if (win) pos = k;
        key = (live && pos == k + 1) ? 1.0 : -1.0;
      }
    }
    P2_TL(5)
  }
#undef P2_TL
  cl.sync();
  // ---- R by position, column order; rows >= q of the pivot column of step
  // q are (alpha_q, 0, ..., 0) unless step q was skipped
  if (on) {
    const int q = (int)min(pos, (long long)P2_H);
    const bool ov = q < a.steps && !S.slog[q];
    const double al = ov ? S.alog[q] : 0.0;
    for (int b0 = 0; b0 < KB; ++b0) {
      double v[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) v[s] = __ldcg(rsave + (int64_t)(8 * b0 + s) * a.p + j0 + t);
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int i = 8 * b0 + s;
        a.Rbuf[(int64_t)i * a.p + pos] = ov && i >= q ? (i == q ? al : 0.0) : v[s];
      }
    }
#pragma unroll
    for (int i = 0; i < P2_W; ++i) {
      const int row = 8 * KB + i;
      if (row < P2_H) a.Rbuf[(int64_t)row * a.p + pos] = ov && row >= q ? (row == q ? al : 0.0) : rr[i];
    }
    for (int row = 8 * KB + P2_W; row < P2_H; ++row)
      a.Rbuf[(int64_t)row * a.p + pos] = ov && row >= q ? (row == q ? al : 0.0) : lds_f64(s0 + (uint32_t)(row - P2_W) * P2_RS);
    const int64_t qq = j0 + t;
    a.perm[pos] = (int32_t)(mode == 0 ? qq : (int64_t)a.perm[qq]);
  }
}
