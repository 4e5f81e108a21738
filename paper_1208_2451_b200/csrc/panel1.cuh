// Thread-per-column panel QRCP engine for panel width h = 64 (the BASELINE
// config-2 shape).  Arithmetic contract identical to panel.cuh
// (pivoted_qr.py:43-87); organisation chosen for the latency of the b
// sequential pivot steps (each step is a chain of dependent phases, so
// every phase is short, and the code a step executes is the same for all
// steps, i.e. it stays in the instruction cache):
//
//  * one thread owns one column of the transposed panel (one panel row, 64
//    doubles) in REGISTERS with static indices; a thread may own a second
//    column in shared memory ([row][thread] layout), i.e. up to 2*P1_T
//    columns per CTA and 8192 per 16-CTA cluster;
//  * SHIFTED layout: during steps 8*KB .. 8*KB+7 element i of a column is
//    absolute row 8*KB + i.  At every block boundary the finished rows
//    8*KB .. 8*KB+7 (final R rows) are saved to a global row-save area and
//    the register column moves up by 8 (the shared-memory column just moves
//    its base).  The pivot row is then always in block 0, only blocks
//    0..L (L = 7 - KB) are live, and numpy's pairwise slot of a row is
//    still i & 7;
//  * per step: warp argmax (redux) -> the warp's best column builds its
//    reflector on its own lane (registers) -> CTA barrier -> CTA argmax ->
//    48-byte record pushed into every CTA of the cluster (st.async +
//    mbarrier transaction count, no cluster barrier) -> cluster argmax in
//    every warp -> the winner's v pulled once per CTA over DSMEM -> apply +
//    next keys.
#pragma once
#include "panel.cuh"

#define P1_H 64
#define P1_T 256                 // threads per CTA: 2 warps per SM sub-partition -> 255 registers
#define P1_MAXCOLS (2 * P1_T)
#define P1_NW (P1_T / 32)

// A candidate pivot column with its reflector; pushed between CTAs as three
// 16-byte chunks.
struct P1Rec {
  double key;
  long long pos;
  int jl;
  int skip;
  double alpha;
  double beta;
  double fro;            // the source CTA's sum of squared column norms (mode 0)
};
static_assert(sizeof(P1Rec) == 48, "P1Rec is pushed as three 16-byte chunks");

struct P1Shared {
  double wpub[2][P1_NW][P1_H];              // per-warp candidate vectors v (shifted rows)
  double vs[P1_H];                          // the cluster winner's v (pulled, shifted rows)
  P1Rec wrec[2][P1_NW];                     // per-warp candidates
  P1Rec rec[2][PRRP_CLUSTER_MAX];           // per-CTA candidates (pushed by every CTA)
  unsigned long long bar[2];                // arrival barriers of rec[buf]
  double fro_warp[P1_NW];
  double alog[P1_H];                        // alpha of step k (R[k,k] of the pivot column)
  int slog[P1_H];                           // step k skipped (the pivot column keeps its values)
  double fro;
  int failed;
};

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ double2 lds2_f64(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
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

// ---------------------------------------------------------------- cluster I/O
__device__ __forceinline__ uint32_t p1_mapa(uint32_t addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// 16-byte store into a (possibly remote) CTA's shared memory that completes
// 16 bytes of the destination CTA's mbarrier transaction count
__device__ __forceinline__ void p1_push16(uint32_t dst, double x, double y, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               :: "r"(dst), "d"(x), "d"(y), "r"(bar) : "memory");
}
__device__ __forceinline__ void p1_pull16(uint32_t src, double& x, double& y) {
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(src) : "memory");
}
__device__ __forceinline__ void p1_bar_init(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar) : "memory");
}
__device__ __forceinline__ void p1_bar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void p1_bar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "P1WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra P1WAIT_%=;\n"
      "}\n" :: "r"(bar), "r"(parity) : "memory");
}

// --------------------------------------------------------- numpy pairwise sums
// numpy pairwise sum of squares of rows 0..63 (the initial column norms).
template <class X>
__device__ __forceinline__ double p1_norm_full(const X& x) {
  double S[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) S[s] = sq_rn(x.ld(s));
#pragma unroll
  for (int B = 1; B < 8; ++B)
#pragma unroll
    for (int s = 0; s < 8; ++s) S[s] = add_rn(S[s], sq_rn(x.ld(8 * B + s)));
  return add_rn(add_rn(add_rn(S[0], S[1]), add_rn(S[2], S[3])), add_rn(add_rn(S[4], S[5]), add_rn(S[6], S[7])));
}

// ((a_o + a_o+1) + (a_o+2 + a_o+3)) + ((a_o+4 + a_o+5) + (a_o+6 + a_o+7)), indices mod 8:
// numpy's 8-accumulator combine when logical accumulator j lives in slot (j + o) & 7.
__device__ __forceinline__ double p1_combine(const double (&S)[8], int o) {
#define P1_C(o)                                                                                   \
  case o:                                                                                         \
    return add_rn(add_rn(add_rn(S[(o) & 7], S[(o + 1) & 7]), add_rn(S[(o + 2) & 7], S[(o + 3) & 7])), \
                  add_rn(add_rn(S[(o + 4) & 7], S[(o + 5) & 7]), add_rn(S[(o + 6) & 7], S[(o + 7) & 7])));
  switch (o) {
    P1_C(0) P1_C(1) P1_C(2) P1_C(3) P1_C(4) P1_C(5) P1_C(6)
    default: break;
  }
  return add_rn(add_rn(add_rn(S[7], S[0]), add_rn(S[1], S[2])), add_rn(add_rn(S[3], S[4]), add_rn(S[5], S[6])));
#undef P1_C
}

// numpy pairwise sum of squares of the shifted rows r0 .. 8L+7 (0 <= r0 <= 8,
// L = last live block), with row r0's value replaced by `first` when REPL.
// n = 8L + 8 - r0 terms.  For n >= 8: slot s = row & 7 accumulates its rows
// of the full 8-groups in row order -- slots s >= r0 over blocks 0..L-1,
// slots s < r0 over blocks 1..L (an accumulator that starts at 0.0 is
// exact) -- and the n % 8 last rows (block L, slots >= r0) are added
// sequentially after the combine; logical accumulator j is slot (j + r0) & 7.
// For n < 8 (L = 0, r0 > 0): a plain sequential sum from -0.0.
template <bool REPL, class X>
__device__ __forceinline__ double p1_sumsq(const X& x, int r0, int L, double first) {
  if (L == 0 && r0 > 0) {
    double res = -0.0;
#pragma unroll
    for (int s = 1; s < 8; ++s)
      if (s >= r0) res = add_rn(res, sq_rn(REPL && s == r0 ? first : x.ld(s)));
    return res;
  }
  double S[8], T[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const double v = x.ld(s);
    const double q = sq_rn(REPL && s == r0 ? first : v);
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
  if (L == 0) {   // r0 == 0: one full group, no remainder
    return p1_combine(S, 0);
  }
  // for L >= 1 the slots s >= r0 of block L are the remainder
  double res = p1_combine(S, r0 & 7);
#pragma unroll
  for (int s = 0; s < 8; ++s)
    if (s >= r0) res = add_rn(res, T[s]);
  return res;
}

// ------------------------------------------------------------ step primitives
// apply reflector k (shifted pivot row r = k & 7): x -= v * (beta * v'x) on
// blocks 0..L; v is zero on rows 0..r-1, so those rows are unchanged.
// act == false: w = 0.
template <class X>
__device__ __forceinline__ void p1_apply(const X& x, const double2* vp, double beta, bool act, int L) {
  // v is re-read from shared memory with volatile loads in both passes: with
  // plain loads the compiler hoists all of v into registers next to the
  // 128-register column, spills, and the FP64 issue rate drops ~3x
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
  const double dot = (d[0] + d[1]) + (d[2] + d[3]);
  // x -= v w as one FMA per element (the reference rounds v*w first; its w
  // comes from a BLAS dgemv whose order is not reproducible anyway, so the
  // updated values agree to the same ulp-level tolerance either way)
  const double nw = act ? -mul_rn(beta, dot) : 0.0;
#pragma unroll
  for (int B = 0; B < 8; ++B) {
    if (B > L) break;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const double2 v = lds2_f64(va + 64 * B + 16 * h);
      const int s = 8 * B + 2 * h;
      x.st(s, fma(v.x, nw, x.ld(s)));
      x.st(s + 1, fma(v.y, nw, x.ld(s + 1)));
    }
  }
}

// Shared-memory column: apply reflector k and compute the key for step k+1
// (rows r0 = r+1 .. 8L+7, numpy pairwise as p1_sumsq) in one pass, with the
// block loop rolled (small code: the step's instructions stay cached).
__device__ __forceinline__ double p1_apply_key_smem(const P1Smem& x, uint32_t vsa, double beta, bool act,
                                                    bool do_apply, int L, int r0) {
  const uint32_t rs = P1_T * 8;   // row stride (bytes)
  double w = 0.0;
  if (do_apply) {
    double d[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
    for (int B = 0; B <= L; ++B) {
      const uint32_t xb = x.base + (uint32_t)(8 * B) * rs, vb = vsa + (uint32_t)(64 * B);
#pragma unroll
      for (int s = 0; s < 8; s += 2) {
        const double2 v = lds2_f64(vb + s * 8);
        d[s & 3] = fma(v.x, lds_f64(xb + s * rs), d[s & 3]);
        d[(s + 1) & 3] = fma(v.y, lds_f64(xb + (s + 1) * rs), d[(s + 1) & 3]);
      }
    }
    const double dot = (d[0] + d[1]) + (d[2] + d[3]);
    w = act ? mul_rn(beta, dot) : 0.0;
  }
  // update (if any) + squares; S: full-group accumulators, T: block L
  double S[8], T[8];
#pragma unroll 1
  for (int B = 0; B <= L; ++B) {
    const uint32_t xb = x.base + (uint32_t)(8 * B) * rs, vb = vsa + (uint32_t)(64 * B);
    double q[8];
#pragma unroll
    for (int s = 0; s < 8; s += 2) {
      double x0 = lds_f64(xb + s * rs), x1 = lds_f64(xb + (s + 1) * rs);
      if (do_apply) {
        const double2 v = lds2_f64(vb + s * 8);
        x0 = sub_rn(x0, mul_rn(v.x, w));
        x1 = sub_rn(x1, mul_rn(v.y, w));
        sts_f64(xb + s * rs, x0);
        sts_f64(xb + (s + 1) * rs, x1);
      }
      q[s] = sq_rn(x0);
      q[s + 1] = sq_rn(x1);
    }
    if (B == 0) {
#pragma unroll
      for (int s = 0; s < 8; ++s) S[s] = s >= r0 ? q[s] : 0.0;
    }
    if (B == L) {
#pragma unroll
      for (int s = 0; s < 8; ++s) T[s] = q[s];
    }
    if (B > 0 && B < L) {
#pragma unroll
      for (int s = 0; s < 8; ++s) S[s] = add_rn(S[s], q[s]);
    } else if (B > 0) {
#pragma unroll
      for (int s = 0; s < 8; ++s)
        if (s < r0) S[s] = add_rn(S[s], q[s]);
    }
  }
  if (L == 0) {   // n = 8 - r0 < 8 terms (r0 >= 1): sequential from -0.0
    double res = -0.0;
#pragma unroll
    for (int s = 1; s < 8; ++s)
      if (s >= r0) res = add_rn(res, T[s]);
    return res;
  }
  double res = p1_combine(S, r0 & 7);
#pragma unroll
  for (int s = 0; s < 8; ++s)
    if (s >= r0) res = add_rn(res, T[s]);
  return res;
}

// The warp's best column builds its reflector on its own lane
// (pivoted_qr.py:43-61): normx (mode 0: sqrt of its key, which IS (x*x).sum()
// over rows k..63 in numpy's order; mode 1: that sum computed), alpha,
// v = x - alpha e_k (shifted rows, zero above r) into wp, beta = 2 / v'v
// with v'v = 2 normx (normx + |x_k|) (the same quantity as numpy's
// (v*v).sum(), without cancellation; it differs from the summed value by a
// few ulps, like the reference's own BLAS-ordered dot products).
template <class X>
__device__ __forceinline__ void p1_candidate(const X& x, int r, int L, int mode, double key, double* wp,
                                             int& skip, double& alpha, double& beta) {
  double xk = x.ld(0);
#pragma unroll
  for (int s = 1; s < 8; ++s)
    if (s == r) xk = x.ld(s);
  const double normx = __dsqrt_rn(mode == 0 ? key : p1_sumsq<false>(x, r, L, 0.0));
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
  const double half_vtv = mul_rn(normx, add_rn(normx, fabs(xk)));
  beta = skip ? 0.0 : __drcp_rn(half_vtv);
  if (half_vtv == 0.0) skip = 1;
  if (skip) { alpha = xk; beta = 0.0; }   // the column already has the form (x_k, 0, ..., 0)
}

struct P1Cols {
  long long pos_r, pos_s;
  double key_r, key_s;
};

// Sortable image of a pivot key: live columns with key >= 0 (or NaN, which
// np.argmax also treats as the maximum) map to bits + 1, everything else to 0.
__device__ __forceinline__ unsigned long long p1_ukey(double key, bool live) {
  return live && !(key < 0.0) ? (unsigned long long)__double_as_longlong(key) + 1ull : 0ull;
}

// Lane holding the lexicographic best (largest u, then smallest position;
// np.argmax's first maximum) in 2-3 warp reductions; -1 when every u is 0.
// Uniform result.
__device__ __forceinline__ int p1_best_lane(unsigned long long u, unsigned pos) {
  const unsigned hi = (unsigned)(u >> 32), lo = (unsigned)u;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  if ((mh | ml) == 0u) return -1;
  const bool top = hi == mh && lo == ml;
  const unsigned tie = __ballot_sync(0xffffffffu, top);
  if ((tie & (tie - 1u)) == 0u) return __ffs(tie) - 1;
  const unsigned mp = __reduce_min_sync(0xffffffffu, top ? pos : 0xffffffffu);
  return __ffs(__ballot_sync(0xffffffffu, top && pos == mp)) - 1;
}

// Apply the cluster winner's reflector k to one column kind, install the
// winner's position, compute its key for step k+1 (rows k+1..63).
template <class X>
__device__ __forceinline__ void p1_apply_col(const X& x, long long& pos, double& key, bool on, int jl, int k, int L,
                                             int mode, const double* vs, double beta, int skip, bool mine, int wjl,
                                             long long wpos) {
  if (!__any_sync(0xffffffffu, on && pos >= k)) return;
  const bool live = on && pos >= k;
  const bool win = live && mine && wjl == jl;
  if (live && !win && pos == k) pos = wpos;
  if (!skip) p1_apply(x, reinterpret_cast<const double2*>(vs), beta, live && !win, L);   // skip is cluster-uniform
  if (win) pos = k;                                     // R[k,k] = alpha, zeros below: at the write-out
  if (mode == 0) {
    const double nk = p1_sumsq<false>(x, (k & 7) + 1, L, 0.0);
    key = (live && !win) ? nk : -1.0;
  } else {
    key = (live && pos == k + 1) ? 1.0 : -1.0;
  }
}

__global__ void __launch_bounds__(P1_T, 1) panel_qrcp1_kernel(PanelArgs a) {
  extern __shared__ __align__(16) double sdata[];      // P1_H x P1_T shared columns
  __shared__ __align__(16) P1Shared S;
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
    S.failed = prrp_failed(a.st) || node_passes(a);
  }
  cl.sync();
  // every CTA follows CTA 0's reading of the error flag (a concurrent kernel
  // may set it between the CTAs' own reads)
  if (*cl.map_shared_rank(&S.failed, 0)) { cl.sync(); return; }
  const int mode = a.mode;
  const int64_t j0 = (int64_t)c * a.per;
  const int nl = (int)max((int64_t)0, min(a.per, a.p - j0));
  const int jl_r = t, jl_s = P1_T + t;
  const bool on_r = jl_r < nl, on_s = jl_s < nl;
  const bool has_s = nl > P1_T;      // CTA-uniform
  double* rsave = a.ovf;             // finished rows of the register columns: rsave[row * p + j0 + jl]

  double rr[P1_H];
  const P1Reg xr{rr};
  const uint32_t xs0 = (uint32_t)__cvta_generic_to_shared(sdata + t);
  auto src_row = [&](int jl) -> const double* {
    const int64_t qq = j0 + jl;
    const int64_t j = mode == 0 ? qq : (int64_t)a.perm[qq];
    const int64_t row = a.rowidx ? a.rowidx[j] : j;
    return member_row(a.src, a.ld, row);
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
    const P1Smem x0{xs0};
    if (on_s) {
      const double* s = src_row(jl_s);
#pragma unroll
      for (int i = 0; i < P1_H; ++i) x0.st(i, s[i]);
    } else {
#pragma unroll
      for (int i = 0; i < P1_H; ++i) x0.st(i, 0.0);
    }
  }
  P1Cols cs;
  cs.pos_r = j0 + jl_r;
  cs.pos_s = j0 + jl_s;
  cs.key_r = -1.0;
  cs.key_s = -1.0;
  if (mode == 0) {
    double fro = 0.0;
    if (on_r) { cs.key_r = p1_norm_full(xr); fro += cs.key_r; }
    if (has_s && on_s) { cs.key_s = p1_norm_full(P1Smem{xs0}); fro += cs.key_s; }
    for (int o = 16; o; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
    if (lane == 0) S.fro_warp[warp] = fro;
  } else {
    cs.key_r = on_r && cs.pos_r == 0 ? 1.0 : -1.0;
    cs.key_s = on_s && cs.pos_s == 0 ? 1.0 : -1.0;
  }
  __syncthreads();
  if (t == 0) {
    double f = 0.0;
    for (int w = 0; w < P1_NW; ++w) f += S.fro_warp[w];
    S.fro = f;
  }
  const bool log_refl = a.refl != nullptr && c == 0;

#ifdef PRRP_P64_PROF
  const bool prof = a.prof && c == 0 && t == 0;
  // timeline of one panel (prof[6] = its id): thread 0 of every CTA, 8 marks per step
  long long* tl = (a.prof && t == 0 && a.panel_id == a.prof[6]) ? a.prof + 8 + (int64_t)c * 64 * 8 : nullptr;
#define P1_TL(m) if (tl) tl[k * 8 + (m)] = clock64();
  long long* tlw = (a.prof && c == 0 && lane == 0 && a.panel_id == a.prof[6])
                       ? a.prof + 8 + PRRP_CLUSTER_MAX * 64 * 8 + (int64_t)warp * 64 * 8 : nullptr;
#define P1_TLW(m) if (tlw) tlw[k * 8 + (m)] = clock64();
#else
  constexpr bool prof = false;
#define P1_TL(m)
#define P1_TLW(m)
#endif
  long long pr[4] = {0, 0, 0, 0}, pt = prof ? clock64() : 0;
  const long long p_start = pt;
#define P1_MARK(slot) if (prof) { const long long nn = clock64(); pr[slot] += nn - pt; pt = nn; }
  int KB = 0;
  for (int k = 0; k < a.steps; ++k) {
    const int buf = k & 1;
    const int r = k & 7;
    if (r == 0 && k > 0) {
      // block boundary: rows 8*KB .. 8*KB+7 are final; shift the register
      // column up by 8, advance the shared-memory column's base
      if (on_r) {
#pragma unroll
        for (int s = 0; s < 8; ++s) rsave[(int64_t)(8 * KB + s) * a.p + j0 + jl_r] = rr[s];
      }
#pragma unroll
      for (int i = 0; i < P1_H - 8; ++i) rr[i] = rr[i + 8];
#pragma unroll
      for (int i = P1_H - 8; i < P1_H; ++i) rr[i] = 0.0;
      ++KB;
    }
    const int L = 7 - KB;
    const P1Smem xsm{xs0 + (uint32_t)(8 * KB) * (P1_T * 8)};
    const uint32_t bar = buf ? bar1 : bar0;
    if (t == 0 && C > 1) p1_bar_expect(bar, (uint32_t)(C * (int)sizeof(P1Rec)));
    P1_MARK(3)
    P1_TL(0)
    P1_TLW(0)
    // ---- warp argmax; the lane of the warp's best column builds its reflector
    {
      const bool lr = on_r && cs.pos_r >= k, ls = on_s && cs.pos_s >= k;
      const unsigned long long ur = p1_ukey(cs.key_r, lr), us = p1_ukey(cs.key_s, ls);
      const bool use_s = us > ur || (us == ur && us != 0ull && cs.pos_s < cs.pos_r);
      const unsigned long long u = use_s ? us : ur;
      const long long mpos = use_s ? cs.pos_s : cs.pos_r;
      const int wl = p1_best_lane(u, (unsigned)mpos);
      P1_TLW(1)
      P1Rec& wr = S.wrec[buf][warp];
      if (wl < 0) {
        if (lane == 0) { wr.key = -INFINITY; wr.pos = LLONG_MAX; wr.jl = -1; wr.skip = 1; }
      } else if (lane == wl) {
        double* wp = S.wpub[buf][warp];
        int skip;
        double alpha, beta;
        const double bk = use_s ? cs.key_s : cs.key_r;
        if (use_s) p1_candidate(xsm, r, L, mode, bk, wp, skip, alpha, beta);
        else p1_candidate(xr, r, L, mode, bk, wp, skip, alpha, beta);
        wr.key = bk; wr.pos = mpos; wr.jl = use_s ? jl_s : jl_r;
        wr.skip = skip; wr.alpha = alpha; wr.beta = beta;
      }
      __syncwarp();
      P1_TLW(2)
    }
    __syncthreads();
    P1_TLW(3)
    P1_MARK(0)
    P1_TL(1)
    // ---- CTA argmax; warp 0 pushes the CTA candidate into every CTA.  A
    // one-CTA cluster skips the exchange: every warp takes the CTA winner.
    const P1Rec* Wp;
    int rc;
    if (C == 1) {
      const bool ok = lane < P1_NW && S.wrec[buf][lane].jl >= 0;
      const unsigned long long u = ok ? p1_ukey(S.wrec[buf][lane].key, true) : 0ull;
      int w = p1_best_lane(u, ok ? (unsigned)S.wrec[buf][lane].pos : 0xffffffffu);
      if (w < 0) w = 0;
      Wp = &S.wrec[buf][w];
      rc = 0;
      if (k == 0 && mode == 0 && warp == 0 && lane == 0) *a.fro = sqrt(S.fro);
    } else {
      if (warp == 0) {
        const bool ok = lane < P1_NW && S.wrec[buf][lane].jl >= 0;
        const unsigned long long u = ok ? p1_ukey(S.wrec[buf][lane].key, true) : 0ull;
        const unsigned pos = ok ? (unsigned)S.wrec[buf][lane].pos : 0xffffffffu;
        int w = p1_best_lane(u, pos);
        if (w < 0) w = 0;   // no live column in this CTA: push warp 0's empty record
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
      P1_TL(2)
      p1_bar_wait(bar, (uint32_t)((k >> 1) & 1));
      P1_MARK(1)
      P1_TL(3)
      // ---- the cluster winner (every warp redundantly); its v pulled once per CTA
      {
        const bool ok = lane < C && S.rec[buf][lane].jl >= 0;
        const unsigned long long u = ok ? p1_ukey(S.rec[buf][lane].key, true) : 0ull;
        rc = p1_best_lane(u, ok ? (unsigned)S.rec[buf][lane].pos : 0xffffffffu);
        if (rc < 0) rc = 0;
      }
      Wp = &S.rec[buf][rc];
    }
    const P1Rec& W = *Wp;
    const long long wpos = W.pos;
    const int skip = W.skip;
    const double beta = W.beta, alpha = W.alpha;
    const int wjl = W.jl;
    const bool mine = rc == c;
    if (t == 0) { S.alog[k] = alpha; S.slog[k] = skip; }
    const int ww = (wjl < P1_T ? wjl : wjl - P1_T) >> 5;
    const double* vs = mine ? S.wpub[buf][ww] : S.vs;
    if (!mine) {
      if (warp == 0 && !skip) {
        if (lane < 4 * (L + 1)) {               // 16-byte chunks of the live rows
          const uint32_t src = p1_mapa((uint32_t)__cvta_generic_to_shared(&S.wpub[buf][ww][2 * lane]), rc);
          double v0, v1;
          p1_pull16(src, v0, v1);
          S.vs[2 * lane] = v0;
          S.vs[2 * lane + 1] = v1;
        }
      }
      __syncthreads();
    }
    P1_TL(4)
    if (C > 1 && k == 0 && mode == 0 && c == 0 && warp == 0) {
      double f = lane < C ? S.rec[buf][lane].fro : 0.0;
      for (int o = 16; o; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
      if (lane == 0) *a.fro = sqrt(f);
    }
    if (log_refl && warp == P1_NW - 1) {
      double* lg = a.refl + (int64_t)k * (P1_H + 1);
      for (int i = lane; i < P1_H; i += 32) lg[i] = (skip || i < k) ? 0.0 : vs[i - 8 * KB];
      if (lane == 0) lg[P1_H] = skip ? 0.0 : beta;
    }
    P1_MARK(2)
    P1_TL(5)

    // ---- apply reflector k, keys for step k+1
    const uint32_t vsa = (uint32_t)__cvta_generic_to_shared(vs);
    p1_apply_col(xr, cs.pos_r, cs.key_r, on_r, jl_r, k, L, mode, vs, beta, skip, mine, wjl, wpos);
    if (has_s && __any_sync(0xffffffffu, on_s && cs.pos_s >= k)) {
      const bool live = on_s && cs.pos_s >= k;
      const bool win = live && mine && wjl == jl_s;
      if (live && !win && cs.pos_s == k) cs.pos_s = wpos;
      if (win) cs.pos_s = k;
      if (mode == 0) {
        const double nk = p1_apply_key_smem(xsm, vsa, beta, live && !win, !skip, L, r + 1);
        cs.key_s = (live && !win) ? nk : -1.0;
      } else {
        if (!skip) p1_apply_key_smem(xsm, vsa, beta, live && !win, true, L, r + 1);
        cs.key_s = (live && cs.pos_s == k + 1) ? 1.0 : -1.0;
      }
    }
    P1_TL(7)
  }
  if (prof) {
    const long long nn = clock64();
    pr[3] += nn - pt;
    a.prof[0] += pr[0]; a.prof[1] += pr[1]; a.prof[2] += pr[2]; a.prof[3] += pr[3];
    a.prof[4] += nn - p_start; a.prof[5] += 1;
  }
#undef P1_MARK
#undef P1_TL
#undef P1_TLW
  cl.sync();
  // ---- R by position, column order; rows >= q of the pivot column of step
  // q are (alpha_q, 0, ..., 0) unless step q was skipped
  if (on_r) {
    const int q = (int)min(cs.pos_r, (long long)P1_H);
    const bool ov = q < a.steps && !S.slog[q];
    const double al = ov ? S.alog[q] : 0.0;
    for (int b0 = 0; b0 < KB; ++b0) {      // saved blocks: 8 independent loads, then 8 stores
      double v[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) v[s] = __ldcg(rsave + (int64_t)(8 * b0 + s) * a.p + j0 + jl_r);
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int i = 8 * b0 + s;
        a.Rbuf[(int64_t)i * a.p + cs.pos_r] = ov && i >= q ? (i == q ? al : 0.0) : v[s];
      }
    }
#pragma unroll
    for (int i = 0; i < P1_H; ++i) {
      const int row = 8 * KB + i;
      if (row < P1_H) a.Rbuf[(int64_t)row * a.p + cs.pos_r] = ov && row >= q ? (row == q ? al : 0.0) : rr[i];
    }
    const int64_t qq = j0 + jl_r;
    a.perm[cs.pos_r] = (int32_t)(mode == 0 ? qq : (int64_t)a.perm[qq]);
  }
  if (on_s) {
    const P1Smem x0{xs0};
    const int q = (int)min(cs.pos_s, (long long)P1_H);
    const bool ov = q < a.steps && !S.slog[q];
    const double al = ov ? S.alog[q] : 0.0;
    for (int i = 0; i < P1_H; ++i)
      a.Rbuf[(int64_t)i * a.p + cs.pos_s] = ov && i >= q ? (i == q ? al : 0.0) : x0.ld(i);
    const int64_t qq = j0 + jl_s;
    a.perm[cs.pos_s] = (int32_t)(mode == 0 ? qq : (int64_t)a.perm[qq]);
  }
}
