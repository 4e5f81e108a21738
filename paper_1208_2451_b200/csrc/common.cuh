// Shared device helpers for the B200 LU_PRRP / CALU_PRRP kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/prrp_b200.h"

#define PRRP_MAXH 128            // largest panel width the device engine supports
#define PRRP_EPS 2.220446049250313e-16   // 2^-52, pivoted_qr.py:25

// ---------------------------------------------------------------------------
// Device-side run state: the first error wins; statistics are kept as the
// IEEE bit patterns of non-negative doubles so atomicMax on uint64 is exact.
// ---------------------------------------------------------------------------
struct DevState {
  int code;
  int panel;
  int index;
  int column;
  int tree_level;
  int tree_index;
  double worst;
  unsigned long long orig_max;
  unsigned long long inter_max;
  unsigned long long finish_max;
  unsigned long long pmm;          // panel multiplier max
  int swaps;                       // swap count of the current panel (finalize writes)
  int moved;                       // number of moved rows of the current panel
  double fro;                      // ||panel||_F of the current panel
  // strong-RRQR candidates: worst |lt| and its row-major flat index
  double cand_max;
  long long cand_flat;
  // error ordering: the reference stops at the FIRST failure in its
  // sequential order (panel, then tournament level, then node index); the
  // device runs nodes of a level (and look-ahead panels) concurrently, so
  // the recorded error is the one with the smallest (panel, level, index).
  unsigned long long err_inv;      // ~rank of the recorded error (larger = earlier)
  int err_lock;
};

// A row of zeros: a CALU tournament merge node whose children passed fewer
// than b candidates (rank-deficient nodes, tournament.py:131-137) keeps its
// static width 2b; the missing members are "dead" (row index -1) and read as
// this zero row.  Dead members sit after every live one, so with first-max
// ties they are never chosen, and they add exact zeros to every sum.
__device__ __align__(16) double g_zero_row[PRRP_MAXH];

__device__ __forceinline__ const double* member_row(const double* src, int64_t ld, int64_t row) {
  return row < 0 ? g_zero_row : src + row * ld;
}

__device__ __forceinline__ bool prrp_failed(const DevState* st) {
  return *(volatile const int*)&st->code != 0;
}

__device__ __forceinline__ void prrp_set_error(DevState* st, int code, int panel, int index,
                                               int column, double worst, int tl = -1, int ti = -1) {
  const unsigned long long rank = ((unsigned long long)(panel + 1) << 42) |
                                  ((unsigned long long)(tl + 1) << 21) | (unsigned long long)(ti + 1);
  const unsigned long long inv = ~rank;
  while (atomicCAS(&st->err_lock, 0, 1) != 0) {
  }
  __threadfence();
  if (*(volatile int*)&st->code == 0 || inv > *(volatile unsigned long long*)&st->err_inv) {
    st->err_inv = inv;
    st->panel = panel;
    st->index = index;
    st->column = column;
    st->worst = worst;
    st->tree_level = tl;
    st->tree_index = ti;
    __threadfence();
    atomicExch(&st->code, code);
  }
  __threadfence();
  atomicExch(&st->err_lock, 0);
}

__device__ __forceinline__ void atomic_max_abs(unsigned long long* slot, double v) {
  // v >= 0 (or NaN, whose bit pattern is > +inf and therefore sticks, like numpy max)
  atomicMax(slot, (unsigned long long)__double_as_longlong(v));
}

// Exact IEEE arithmetic without FMA contraction (numpy elementwise semantics).
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// Correctly rounded a / b from y = __drcp_rn(b) (the correctly rounded
// reciprocal) and one FMA correction (Markstein): q = RN(a*y),
// r = a - b*q (exact), RN(q + r*y) == RN(a/b).  Validated bit-exact against
// __ddiv_rn on 9.1e8 random operand pairs on B200
// (tools/probes/probe_div.cu).  Outside the normal range (overflow, results
// near underflow, NaN/Inf) it falls back to the IEEE division.
__device__ __forceinline__ double div_fast(double a, double b, double y) {
  const double q = __dmul_rn(a, y);
  const double r = fma(-b, q, a);
  const double qq = fma(r, y, q);
  const double aq = fabs(qq);
  if (!(aq < 1e300 && (aq > 1e-290 || a == 0.0))) return __ddiv_rn(a, b);
  return qq;
}

// "a is a better pivot candidate than b": larger key, ties to the smaller position
// (np.argmax returns the first maximum; pivoted_qr.py:82, gepp.py:49).
__device__ __forceinline__ bool better(double ka, long long pa, double kb, long long pb) {
  return ka > kb || (ka == kb && pa < pb);
}

// numpy pairwise summation of x[0..n) with n <= 128 (8 strided accumulators,
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), sequential remainder; below 8 terms a
// plain sequential sum from -0.0).  Elements are produced by the functor so
// squares are rounded before they are summed, exactly as (x*x).sum().
template <typename F>
__device__ __forceinline__ double pairwise_sum(int n, F term) {
  if (n < 8) {
    double s = -0.0;
    for (int i = 0; i < n; ++i) s = add_rn(s, term(i));
    return s;
  }
  double r0 = term(0), r1 = term(1), r2 = term(2), r3 = term(3);
  double r4 = term(4), r5 = term(5), r6 = term(6), r7 = term(7);
  const int full = n - (n % 8);
  int i = 8;
  for (; i < full; i += 8) {
    r0 = add_rn(r0, term(i + 0)); r1 = add_rn(r1, term(i + 1));
    r2 = add_rn(r2, term(i + 2)); r3 = add_rn(r3, term(i + 3));
    r4 = add_rn(r4, term(i + 4)); r5 = add_rn(r5, term(i + 5));
    r6 = add_rn(r6, term(i + 6)); r7 = add_rn(r7, term(i + 7));
  }
  double s = add_rn(add_rn(add_rn(r0, r1), add_rn(r2, r3)), add_rn(add_rn(r4, r5), add_rn(r6, r7)));
  for (; i < n; ++i) s = add_rn(s, term(i));
  return s;
}

__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide max of non-negative values; result valid in all threads.
__device__ __forceinline__ double block_max(double v, double* red /* >= 32 doubles */) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double r = (l < nw) ? red[l] : 0.0;
  if (w == 0) red[32] = warp_max(r);
  __syncthreads();
  return red[32];
}
