// FP64 Schur update C <- C - L21 * A12 on the FP64 tensor pipe (DMMA).
//
// Reference: matcore.rank_update (matcore.py:54-61) = c - matmul(a, b),
// matmul (matcore.py:41-51) accumulating rank-1 dger terms in increasing k
// from a zero matrix.  On FMA hosts dger performs acc = fma(a_ik, b_kj, acc)
// per k, and sm_100 DMMA.8x8x4 performs exactly that chain over its 4 k's
// (verified on the B200: tools/probes/probe_fp64.cu), so chaining the k-steps
// in increasing order from a zero accumulator and subtracting once in the
// epilogue reproduces the reference's rank_update bit for bit.
//
// sm_100a has no tcgen05 FP64 kind, so the tensor path is warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  Operands are staged by TMA
// (cp.async.bulk.tensor.2d) into shared memory in a [8-row group][k][8]
// layout: every m8n8k4 fragment is then one contiguous 256-byte read (no bank
// conflicts).  An mbarrier ring pipelines the K chunks; the epilogue reads C,
// subtracts, writes C and folds max|C| into the growth statistic.
#pragma once
#include <cuda.h>
#include "common.cuh"

#define SCH_BM 128
#define SCH_BN 64
#define SCH_KC 32
#define SCH_STAGES 2
#define SCH_THREADS 256

struct SchurSmem {
  double a[SCH_STAGES][SCH_BM * SCH_KC];
  double b[SCH_STAGES][SCH_BN * SCH_KC];
  unsigned long long full[SCH_STAGES];
  unsigned long long empty[SCH_STAGES];
  double red[40];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
// Consumer release of a TMA stage.  The arrive must not be issued while the stage's fragment loads
// are still in flight: ptxas hoists a plain arrive above the DMMAs that consume the loads, directly
// behind the last LDS, and on B200 the SYNCS arrive can then overtake those LDS when the LSU is
// congested (other warps' C traffic) -- the producer's next TMA write lands first and the warp reads
// the NEXT tile's fragment (measured: 8 x 32 strips wrong in 4-15% of runs of the epilogue-read
// kernel, tools/schur_determinism.py; DESIGN 4).  `dep` ORs the high words of the stage's last
// fragment loads (LDS complete in order per warp) and `opaque_zero` is a run-time 0 the compiler
// cannot fold, so the arrive's address carries a true register dependency on the loaded data.
__device__ __forceinline__ void mbar_arrive_after(unsigned long long* bar, uint32_t dep, uint32_t opaque_zero) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar) + (dep & opaque_zero)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, unsigned long long* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      :: "r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// mapL: L21 column-major (dims {M, K}, box {8, KC}); mapB: A12 row-major (dims {N, K}, box {8, KC})
__global__ void __launch_bounds__(SCH_THREADS, 2)
schur_dmma_kernel(const __grid_constant__ CUtensorMap mapL, const __grid_constant__ CUtensorMap mapB,
                  double* C, int64_t ldc, int M, int N, int K, int vec_ok, DevState* st) {
  extern __shared__ __align__(128) unsigned char sbuf[];
  SchurSmem& S = *reinterpret_cast<SchurSmem*>(sbuf);
  if (prrp_failed(st)) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int m0 = blockIdx.y * SCH_BM, n0 = blockIdx.x * SCH_BN;
  const int nk = (K + SCH_KC - 1) / SCH_KC;   // K tail is zero-filled by TMA (exact: fma(0,0,acc) = acc)
  constexpr uint32_t kStageBytes = (SCH_BM + SCH_BN) * SCH_KC * 8;

  if (t == 0) {
    for (int s = 0; s < SCH_STAGES; ++s) { mbar_init(&S.full[s], 1); mbar_init(&S.empty[s], SCH_THREADS / 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&mapL) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&mapB) : "memory");
  }
  __syncthreads();
  auto issue = [&](int kc) {
    const int s = kc % SCH_STAGES;
    mbar_expect_tx(&S.full[s], kStageBytes);
    for (int g = 0; g < SCH_BM / 8; ++g) tma_load_2d(&S.a[s][g * SCH_KC * 8], &mapL, &S.full[s], m0 + 8 * g, kc * SCH_KC);
    for (int g = 0; g < SCH_BN / 8; ++g) tma_load_2d(&S.b[s][g * SCH_KC * 8], &mapB, &S.full[s], n0 + 8 * g, kc * SCH_KC);
  };
  if (t == 0)
    for (int kc = 0; kc < nk && kc < SCH_STAGES; ++kc) issue(kc);

  // warp tile 32 x 32: warps 4 (M) x 2 (N)
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int fr = lane & 3, fc = lane >> 2;   // fragment k index, row/col index
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc % SCH_STAGES;
    mbar_wait(&S.full[s], (kc / SCH_STAGES) & 1);
    uint32_t dep = 0;
    const double* sa = S.a[s];
    const double* sb = S.b[s];
#pragma unroll
    for (int k4 = 0; k4 < SCH_KC; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = sa[(((wm >> 3) + i) * SCH_KC + k4 + fr) * 8 + fc];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = sb[(((wn >> 3) + j) * SCH_KC + k4 + fr) * 8 + fc];
      if (k4 == SCH_KC - 4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) dep |= (uint32_t)__double2hiint(af[i]) | (uint32_t)__double2hiint(bf[i]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_after(&S.empty[s], dep, (uint32_t)(ldc >> 40));
    if (t == 0 && kc + SCH_STAGES < nk) {
      mbar_wait(&S.empty[s], (kc / SCH_STAGES) & 1);
      issue(kc + SCH_STAGES);
    }
    __syncwarp();
  }

  // epilogue: C -= acc, max|C|
  double mx = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm + i * 8 + fc;
    if (r >= M) continue;
    double* crow = C + (int64_t)r * ldc;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cidx = n0 + wn + j * 8 + 2 * fr;
      if (vec_ok && cidx + 1 < N) {
        double2 cv = *reinterpret_cast<const double2*>(crow + cidx);
        cv.x = sub_rn(cv.x, acc[i][j][0]);
        cv.y = sub_rn(cv.y, acc[i][j][1]);
        *reinterpret_cast<double2*>(crow + cidx) = cv;
        mx = fmax(mx, fmax(fabs(cv.x), fabs(cv.y)));
      } else {
        if (cidx < N) {
          const double v = sub_rn(crow[cidx], acc[i][j][0]);
          crow[cidx] = v;
          mx = fmax(mx, fabs(v));
        }
        if (cidx + 1 < N) {
          const double v = sub_rn(crow[cidx + 1], acc[i][j][1]);
          crow[cidx + 1] = v;
          mx = fmax(mx, fabs(v));
        }
      }
    }
  }
  mx = block_max(mx, S.red);
  if (t == 0) atomic_max_abs(&st->inter_max, mx);
}

// Persistent variant for K <= 64 (the b = 64 trailing updates): one CTA per SM
// walks the 128 x 64 tiles; the whole K of a tile is one TMA stage, the next
// tile's stage is in flight while the current one multiplies, and each
// thread's 32 C elements are loaded into registers before the MMA loop so the
// epilogue never waits on HBM.  Same fragments, same k order, same epilogue
// rounding as schur_dmma_kernel (bit-identical results).
#define SP_K 64
struct SchurPSmem {
  double a[2][SCH_BM * SP_K];
  double b[2][SCH_BN * SP_K];
  unsigned long long full[2];
  double red[40];
};

__global__ void __launch_bounds__(SCH_THREADS, 1)
schur_persist_kernel(const __grid_constant__ CUtensorMap mapL, const __grid_constant__ CUtensorMap mapB,
                     double* C, int64_t ldc, int M, int N, int K, int vec_ok, DevState* st) {
  extern __shared__ __align__(128) unsigned char sbuf[];
  SchurPSmem& S = *reinterpret_cast<SchurPSmem*>(sbuf);
  if (prrp_failed(st)) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ntN = (N + SCH_BN - 1) / SCH_BN, ntM = (M + SCH_BM - 1) / SCH_BM;
  const int ntiles = ntM * ntN;
  constexpr uint32_t kTileBytes = (SCH_BM + SCH_BN) * SP_K * 8;
  if (t == 0) {
    mbar_init(&S.full[0], 1);
    mbar_init(&S.full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&mapL) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&mapB) : "memory");
  }
  __syncthreads();
  auto issue = [&](int tile, int s) {
    const int m0 = (tile / ntN) * SCH_BM, n0 = (tile % ntN) * SCH_BN;
    mbar_expect_tx(&S.full[s], kTileBytes);
    for (int g = 0; g < SCH_BM / 8; ++g) tma_load_2d(&S.a[s][g * SP_K * 8], &mapL, &S.full[s], m0 + 8 * g, 0);
    for (int g = 0; g < SCH_BN / 8; ++g) tma_load_2d(&S.b[s][g * SP_K * 8], &mapB, &S.full[s], n0 + 8 * g, 0);
  };
  const int first = blockIdx.x;
  if (t == 0 && first < ntiles) issue(first, 0);
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
  const int fr = lane & 3, fc = lane >> 2;
  double mx = 0.0;
  int it = 0;
  for (int tile = first; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it & 1;
    const int m0 = (tile / ntN) * SCH_BM, n0 = (tile % ntN) * SCH_BN;
    if (t == 0 && tile + (int)gridDim.x < ntiles) issue(tile + gridDim.x, s ^ 1);
    // this tile's C into registers (in flight during the MMA loop)
    double cv[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = m0 + wm + i * 8 + fc;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c0 = n0 + wn + j * 8 + 2 * fr;
        const double* cp = C + (int64_t)r * ldc + c0;
        if (r < M && vec_ok && c0 + 1 < N) {
          const double2 v = *reinterpret_cast<const double2*>(cp);
          cv[i][j][0] = v.x;
          cv[i][j][1] = v.y;
        } else {
          cv[i][j][0] = (r < M && c0 < N) ? cp[0] : 0.0;
          cv[i][j][1] = (r < M && c0 + 1 < N) ? cp[1] : 0.0;
        }
      }
    }
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    mbar_wait(&S.full[s], (it >> 1) & 1);
    const double* sa = S.a[s];
    const double* sb = S.b[s];
    const int kmax = (K + 3) & ~3;
#pragma unroll 4
    for (int k4 = 0; k4 < kmax; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = sa[(((wm >> 3) + i) * SP_K + k4 + fr) * 8 + fc];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = sb[(((wn >> 3) + j) * SP_K + k4 + fr) * 8 + fc];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    // epilogue: C -= acc, max|C|
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = m0 + wm + i * 8 + fc;
      if (r >= M) continue;
      double* crow = C + (int64_t)r * ldc;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c0 = n0 + wn + j * 8 + 2 * fr;
        const double v0 = sub_rn(cv[i][j][0], acc[i][j][0]);
        const double v1 = sub_rn(cv[i][j][1], acc[i][j][1]);
        if (vec_ok && c0 + 1 < N) {
          *reinterpret_cast<double2*>(crow + c0) = make_double2(v0, v1);
          mx = fmax(mx, fmax(fabs(v0), fabs(v1)));
        } else {
          if (c0 < N) { crow[c0] = v0; mx = fmax(mx, fabs(v0)); }
          if (c0 + 1 < N) { crow[c0 + 1] = v1; mx = fmax(mx, fabs(v1)); }
        }
      }
    }
    __syncthreads();   // stage s is refilled by the issue at the top of tile it+1... (it+2)
  }
  mx = block_max(mx, S.red);
  if (t == 0) atomic_max_abs(&st->inter_max, mx);
}

// Generic-shape fallback with the identical rounding recipe (odd K or
// unaligned operands): one thread per C element, fma chain from zero.
__global__ void __launch_bounds__(256) schur_simt_kernel(const double* L, int64_t ldl, const double* B, int64_t ldb,
                                                        double* C, int64_t ldc, int M, int N, int K, DevState* st) {
  __shared__ double red[40];
  if (prrp_failed(st)) return;
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int r = blockIdx.y * 8 + (threadIdx.x >> 5);
  double mx = 0.0;
  if (r < M && c < N) {
    double acc = 0.0;
    for (int k = 0; k < K; ++k) acc = fma(L[(int64_t)k * ldl + r], B[(int64_t)k * ldb + c], acc);
    const double v = sub_rn(C[(int64_t)r * ldc + c], acc);
    C[(int64_t)r * ldc + c] = v;
    mx = fabs(v);
  }
  mx = block_max(mx, red);
  if (threadIdx.x == 0) atomic_max_abs(&st->inter_max, mx);
}

// Warp-specialised persistent variant for any K: one producer warp walks its
// 128 x 64 tiles (static: blockIdx.x + i * gridDim.x; or, with ctr != null,
// claimed from a global counter so that a CTA that starts late because a
// concurrent stream holds its SM simply claims fewer tiles) and streams their K chunks through a SW_ST-deep mbarrier ring
// (continuous across tiles, so the next tile's operands are in flight while
// the current one finishes); the claimed tile id rides in the ring slot of
// its first chunk.  Eight consumer warps own a 32 x 32 sub-tile each,
// prefetch their C elements into registers at the start of a tile (the HBM
// read overlaps the MMA loop) and release each stage with one arrive per
// warp.  At most `quantum` tiles per CTA.  stream_c: C is read and written
// with evict-first hints (an update whose result is not read again soon).  Same fragments, same k order
// (increasing, from a zero accumulator) and the same epilogue rounding as
// schur_dmma_kernel: bit-identical results.  ctr[0] (claims) and ctr[1]
// (finished CTAs) are reset by the last CTA.
#ifdef PRRP_SCHUR_RACECHECK
__device__ int g_racecheck[2 + 4 * 64];
__device__ const double* g_race_base;
__device__ long long g_race_ld;
#endif
#define SW_KC 32
#define SW_ST 4
#define SW_CONS 8
#define SW_THREADS ((SW_CONS + 1) * 32)
struct SchurWSmem {
  double a[SW_ST][SCH_BM * SW_KC];
  double b[SW_ST][SCH_BN * SW_KC];
  unsigned long long full[SW_ST];
  unsigned long long empty[SW_ST];
  int tile[SW_ST];
  double red[40];
};

template <bool PC>
__global__ void __launch_bounds__(SW_THREADS, 1)
schur_ws_kernel(const __grid_constant__ CUtensorMap mapL, const __grid_constant__ CUtensorMap mapB,
                double* C, int64_t ldc, int M, int N, int K, int vec_ok, DevState* st, int* ctr, int quantum,
                int stream_c) {
  extern __shared__ __align__(128) unsigned char sbuf[];
  SchurWSmem& S = *reinterpret_cast<SchurWSmem*>(sbuf);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ntN = (N + SCH_BN - 1) / SCH_BN, ntM = (M + SCH_BM - 1) / SCH_BM;
  const int ntiles = prrp_failed(st) ? 0 : ntM * ntN;   // a failed factorization claims nothing
  const int nk = (K + SW_KC - 1) / SW_KC;
  constexpr uint32_t kStageBytes = (SCH_BM + SCH_BN) * SW_KC * 8;
  if (t == 0) {
    for (int s = 0; s < SW_ST; ++s) { mbar_init(&S.full[s], 1); mbar_init(&S.empty[s], SW_CONS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&mapL) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&mapB) : "memory");
  }
  __syncthreads();
  double mx = 0.0;
  if (warp == SW_CONS) {
    // ---- producer
    if (lane == 0) {
      uint32_t it = 0;
      for (int claimed = 0;; ++claimed) {
        int tile = claimed >= quantum ? ntiles
                   : ctr ? atomicAdd(&ctr[0], 1) : (int)blockIdx.x + claimed * (int)gridDim.x;
        if (tile >= ntiles) tile = -1;
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % SW_ST;
          if (it >= SW_ST) mbar_wait(&S.empty[s], ((it / SW_ST) & 1) ^ 1);
          if (kc == 0) {
            *reinterpret_cast<volatile int*>(&S.tile[s]) = tile;
            if (tile < 0) { mbar_arrive(&S.full[s]); break; }
          }
          const int m0 = (tile / ntN) * SCH_BM, n0 = (tile % ntN) * SCH_BN;
          mbar_expect_tx(&S.full[s], kStageBytes);
#pragma unroll 1
          for (int g = 0; g < SCH_BM / 8; ++g)
            tma_load_2d(&S.a[s][g * SW_KC * 8], &mapL, &S.full[s], m0 + 8 * g, kc * SW_KC);
#pragma unroll 1
          for (int g = 0; g < SCH_BN / 8; ++g)
            tma_load_2d(&S.b[s][g * SW_KC * 8], &mapB, &S.full[s], n0 + 8 * g, kc * SW_KC);
        }
        if (tile < 0) break;
      }
    }
  } else {
    // ---- consumers
    const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
    const int fr = lane & 3, fc = lane >> 2;
    uint32_t it = 0;
    for (;;) {
      mbar_wait(&S.full[it % SW_ST], (it / SW_ST) & 1);
      const int tile = *reinterpret_cast<volatile int*>(&S.tile[it % SW_ST]);
      if (tile < 0) break;
      const int m0 = (tile / ntN) * SCH_BM, n0 = (tile % ntN) * SCH_BN;
      double cv[4][4][2];
      auto load_c = [&]() {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = m0 + wm + i * 8 + fc;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int c0 = n0 + wn + j * 8 + 2 * fr;
            const double* cp = C + (int64_t)r * ldc + c0;
            if (r < M && vec_ok && c0 + 1 < N) {
              const double2 v = (stream_c & 1) ? __ldcs(reinterpret_cast<const double2*>(cp))
                                               : __ldcg(reinterpret_cast<const double2*>(cp));
              cv[i][j][0] = v.x;
              cv[i][j][1] = v.y;
            } else {
              cv[i][j][0] = (r < M && c0 < N) ? __ldcg(cp) : 0.0;
              cv[i][j][1] = (r < M && c0 + 1 < N) ? __ldcg(cp + 1) : 0.0;
            }
          }
        }
      };
      if (PC) load_c();
#ifdef PRRP_SCHUR_RACECHECK
      if (!PC) load_c();   // early copy, compared with the epilogue's read
#endif
      double acc[4][4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      for (int kc = 0; kc < nk; ++kc, ++it) {
        const int s = it % SW_ST;
        if (kc > 0) mbar_wait(&S.full[s], (it / SW_ST) & 1);
        uint32_t dep = 0;
        const double* sa = S.a[s];
        const double* sb = S.b[s];
#pragma unroll
        for (int k4 = 0; k4 < SW_KC; k4 += 4) {
          double af[4], bf[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) af[i] = sa[(((wm >> 3) + i) * SW_KC + k4 + fr) * 8 + fc];
#pragma unroll
          for (int j = 0; j < 4; ++j) bf[j] = sb[(((wn >> 3) + j) * SW_KC + k4 + fr) * 8 + fc];
          if (k4 == SW_KC - 4) {
#pragma unroll
            for (int i = 0; i < 4; ++i) dep |= (uint32_t)__double2hiint(af[i]) | (uint32_t)__double2hiint(bf[i]);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncwarp();
        if (lane == 0) {
          if (stream_c & 16) mbar_arrive(&S.empty[s]);   // diagnostic: the plain (hoistable) arrive
          else mbar_arrive_after(&S.empty[s], dep, (uint32_t)(ldc >> 40));
        }
      }
      if (!PC) {
#ifdef PRRP_SCHUR_RACECHECK
        double c0v[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) { c0v[i][j][0] = cv[i][j][0]; c0v[i][j][1] = cv[i][j][1]; }
#endif
        load_c();
#ifdef PRRP_SCHUR_RACECHECK
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            for (int h = 0; h < 2; ++h)
              if (__double_as_longlong(c0v[i][j][h]) != __double_as_longlong(cv[i][j][h])) {
                const int n_ = atomicAdd(&g_racecheck[0], 1);
                if (n_ < 64) {
                  g_racecheck[2 + 4 * n_] = (int)(((C - g_race_base) + 0) / g_race_ld) + m0 + wm + i * 8 + fc;
                  g_racecheck[3 + 4 * n_] = (int)((C - g_race_base) % g_race_ld) + n0 + wn + j * 8 + 2 * fr + h;
                  g_racecheck[4 + 4 * n_] = M;
                  g_racecheck[5 + 4 * n_] = N;
                }
              }
#endif
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = m0 + wm + i * 8 + fc;
        if (r >= M) continue;
        double* crow = C + (int64_t)r * ldc;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c0 = n0 + wn + j * 8 + 2 * fr;
          const double v0 = sub_rn(cv[i][j][0], acc[i][j][0]);
          const double v1 = sub_rn(cv[i][j][1], acc[i][j][1]);
          if (vec_ok && c0 + 1 < N) {
            if (stream_c & 1) __stcs(reinterpret_cast<double2*>(crow + c0), make_double2(v0, v1));
            else *reinterpret_cast<double2*>(crow + c0) = make_double2(v0, v1);
            mx = fmax(mx, fmax(fabs(v0), fabs(v1)));
          } else {
            if (c0 < N) { crow[c0] = v0; mx = fmax(mx, fabs(v0)); }
            if (c0 + 1 < N) { crow[c0 + 1] = v1; mx = fmax(mx, fabs(v1)); }
          }
        }
      }
    }
  }
  mx = block_max(mx, S.red);
  if (t == 0) {
    if (mx > 0.0) atomic_max_abs(&st->inter_max, mx);
    if (ctr && atomicAdd(&ctr[1], 1) == (int)gridDim.x - 1) { ctr[0] = 0; ctr[1] = 0; }
  }
}


// Warp-specialised variant with C staged through shared memory by TMA: at the
// start of each tile consumer thread 0 (after a consumer-only barrier that
// retires the previous tile's reads of the buffer) loads the tile's C into a
// 64 KB buffer ([8-column group][128 rows][8]); the epilogue reads it from
// shared memory.  C is thus read early (like the register prefetch) while the
// registers stay free for the MMA loop (like the epilogue read).  Three operand
// stages (144 KB) + C (64 KB).  Same fragments, k order and epilogue rounding
// as schur_ws_kernel (bit-identical).
#define SWC_ST 3
struct SchurWCSmem {
  double a[SWC_ST][SCH_BM * SW_KC];
  double b[SWC_ST][SCH_BN * SW_KC];
  double c[SCH_BN / 8][SCH_BM * 8];
  unsigned long long full[SWC_ST];
  unsigned long long empty[SWC_ST];
  unsigned long long cfull;
  int tile[SWC_ST];
  double red[40];
};

template <int NCW>
__device__ __forceinline__ void consumers_sync() {   // named barrier 1 over the consumer warps
  asm volatile("bar.sync 1, %0;" :: "n"(NCW * 32) : "memory");
}

// NCW consumer warps with 32 x (512 / NCW) warp tiles: 16, 8 (the default,
// measured best: 78% of the DMMA peak) or 4 (61%)
template <int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
schur_wsc_kernel(const __grid_constant__ CUtensorMap mapL, const __grid_constant__ CUtensorMap mapB,
                 const __grid_constant__ CUtensorMap mapC, double* C, int64_t ldc, int M, int N, int K,
                 DevState* st) {
  constexpr int NJ = NCW == 16 ? 2 : NCW == 8 ? 4 : 8;   // 8-column fragments per warp
  extern __shared__ __align__(128) unsigned char sbuf[];
  SchurWCSmem& S = *reinterpret_cast<SchurWCSmem*>(sbuf);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ntN = (N + SCH_BN - 1) / SCH_BN, ntM = (M + SCH_BM - 1) / SCH_BM;
  const int ntiles = prrp_failed(st) ? 0 : ntM * ntN;
  const int nk = (K + SW_KC - 1) / SW_KC;
  constexpr uint32_t kStageBytes = (SCH_BM + SCH_BN) * SW_KC * 8;
  constexpr uint32_t kCBytes = SCH_BM * SCH_BN * 8;
  if (t == 0) {
    for (int s = 0; s < SWC_ST; ++s) { mbar_init(&S.full[s], 1); mbar_init(&S.empty[s], NCW); }
    mbar_init(&S.cfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&mapL) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&mapB) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&mapC) : "memory");
  }
  __syncthreads();
  double mx = 0.0;
  if (warp == NCW) {
    // ---- producer (static tiles)
    if (lane == 0) {
      uint32_t it = 0;
      for (int claimed = 0;; ++claimed) {
        int tile = (int)blockIdx.x + claimed * (int)gridDim.x;
        if (tile >= ntiles) tile = -1;
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % SWC_ST;
          if (it >= SWC_ST) mbar_wait(&S.empty[s], ((it / SWC_ST) & 1) ^ 1);
          if (kc == 0) {
            *reinterpret_cast<volatile int*>(&S.tile[s]) = tile;
            if (tile < 0) { mbar_arrive(&S.full[s]); break; }
          }
          const int m0 = (tile / ntN) * SCH_BM, n0 = (tile % ntN) * SCH_BN;
          mbar_expect_tx(&S.full[s], kStageBytes);
#pragma unroll 1
          for (int g = 0; g < SCH_BM / 8; ++g)
            tma_load_2d(&S.a[s][g * SW_KC * 8], &mapL, &S.full[s], m0 + 8 * g, kc * SW_KC);
#pragma unroll 1
          for (int g = 0; g < SCH_BN / 8; ++g)
            tma_load_2d(&S.b[s][g * SW_KC * 8], &mapB, &S.full[s], n0 + 8 * g, kc * SW_KC);
        }
        if (tile < 0) break;
      }
    }
  } else {
    // ---- consumers
    const int wm = (warp & 3) * 32, wn = (warp >> 2) * (8 * NJ);
    const int fr = lane & 3, fc = lane >> 2;
    uint32_t it = 0, ntile = 0;
    for (;; ++ntile) {
      mbar_wait(&S.full[it % SWC_ST], (it / SWC_ST) & 1);
      const int tile = *reinterpret_cast<volatile int*>(&S.tile[it % SWC_ST]);
      if (tile < 0) break;
      const int m0 = (tile / ntN) * SCH_BM, n0 = (tile % ntN) * SCH_BN;
      consumers_sync<NCW>();     // every consumer finished reading the previous tile's C
      if (t == 0) {
        mbar_expect_tx(&S.cfull, kCBytes);
#pragma unroll 1
        for (int g = 0; g < SCH_BN / 8; ++g) tma_load_2d(&S.c[g][0], &mapC, &S.cfull, n0 + 8 * g, m0);
      }
      double acc[4][NJ][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      for (int kc = 0; kc < nk; ++kc, ++it) {
        const int s = it % SWC_ST;
        if (kc > 0) mbar_wait(&S.full[s], (it / SWC_ST) & 1);
        uint32_t dep = 0;
        const double* sa = S.a[s];
        const double* sb = S.b[s];
#pragma unroll
        for (int k4 = 0; k4 < SW_KC; k4 += 4) {
          double af[4], bf[NJ];
#pragma unroll
          for (int i = 0; i < 4; ++i) af[i] = sa[(((wm >> 3) + i) * SW_KC + k4 + fr) * 8 + fc];
#pragma unroll
          for (int j = 0; j < NJ; ++j) bf[j] = sb[(((wn >> 3) + j) * SW_KC + k4 + fr) * 8 + fc];
          if (k4 == SW_KC - 4) {
#pragma unroll
            for (int i = 0; i < 4; ++i) dep |= (uint32_t)__double2hiint(af[i]);
#pragma unroll
            for (int j = 0; j < NJ; ++j) dep |= (uint32_t)__double2hiint(bf[j]);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_after(&S.empty[s], dep, (uint32_t)(ldc >> 40));
      }
      mbar_wait(&S.cfull, ntile & 1);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int rl = wm + i * 8 + fc, r = m0 + rl;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int cl = wn + j * 8 + 2 * fr, c0 = n0 + cl;
          const double2 cv = *reinterpret_cast<const double2*>(&S.c[cl >> 3][rl * 8 + (cl & 7)]);
          const double v0 = sub_rn(cv.x, acc[i][j][0]);
          const double v1 = sub_rn(cv.y, acc[i][j][1]);
          if (r < M) {
            double* crow = C + (int64_t)r * ldc;
            if (c0 + 1 < N) {
              *reinterpret_cast<double2*>(crow + c0) = make_double2(v0, v1);
              mx = fmax(mx, fmax(fabs(v0), fabs(v1)));
            } else if (c0 < N) {
              crow[c0] = v0;
              mx = fmax(mx, fabs(v0));
            }
          }
        }
      }
    }
  }
  mx = block_max(mx, S.red);
  if (t == 0 && mx > 0.0) atomic_max_abs(&st->inter_max, mx);
}
