// Latency-oriented panel QRCP engine (round 2): tournament merge nodes
// (2b x b), the CALU final QR, leaves and LU_PRRP panels of up to
// 16 CTAs x 64 CPT columns.  Same arithmetic contract as panel.cuh /
// panel1.cuh / panel2.cuh (pivoted_qr.py:43-87): exact numpy-pairwise column
// norms recomputed every step, first-max argmax, the reflector of the
// winning column (alpha = -sign(x_k)||x||, v = x - alpha e_k,
// v'v = 2||x||(||x|| + |x_k|)), w = beta (v'x), x -= v w.
//
// The thread-per-column engines spend 3.4-5.6 us per pivot step whatever the
// panel height: a thread walks its whole 64/128-row column three times per
// step (~1500 instructions per warp per step: instruction issue and a long
// dependent chain), one lane builds the reflector, and the winner's v is
// pulled over DSMEM after a second exchange.  Here
//   * a TEAM of 8 threads owns a column: thread q keeps rows 8u + q in
//     registers (NR = h/8 values per column, CPT columns per team), so a
//     step's column pass is NR elements per thread;
//   * numpy's pairwise order stays exact: at base row `base` the relative
//     index of row 8u + q is congruent to (q - base) mod 8, i.e. thread q IS
//     pairwise slot (q - base) & 7; the eight slots combine as
//     ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) through three shuffles whose
//     partner lanes follow the rotation; the n % 8 trailing terms are added
//     in row order;
//   * NWC compute warps + ONE control warp per CTA.  The compute warps only
//     do column work (warp argmax + publish, dot products, update, norms);
//     the control warp runs everything that is serial -- CTA argmax, the
//     cluster exchange, the reflector scalars (one sqrt + one reciprocal
//     per CTA per step instead of one per warp) -- so the FP64 pipe and the
//     issue slots of the compute warps are not spent on redundant copies;
//   * the dot products do not wait for the reflector scalars: the published
//     pivot column has rows <= k zeroed, the compute warps form
//     d' = sum_{i>k} p_i x_i while the control warp computes alpha, beta and
//     v_k, and then w = -beta (d' + v_k x_k) (row k of the shared column
//     stays zero; the thread that owns row k takes v_k from the control warp);
//   * cluster exchange: st.async pushes + mbarrier transaction counts (the
//     cheapest all-to-all measured on B200, tools/probes/probe_xchg.cu:
//     ~300 cycles against ~850 for barrier.cluster + remote loads).  Up to
//     LAT_SP_MAXC CTAs push record AND candidate column to every CTA in one
//     round; larger clusters push the 48-byte records first and only the
//     winner CTA pushes its column.
// Three CTA barriers per step (~20 cycles each, measured).
#pragma once
#include "panel1.cuh"

#ifndef LAT_SP_MAXC
#define LAT_SP_MAXC 16           // largest cluster that exchanges record + column in one round (16: always;
                                 // measured 1-3% faster than records first, winner column second, which
                                 // -DLAT_SP_MAXC=6 restores for clusters above 6 CTAs)
#endif
constexpr int kLatNWC = 15;      // compute warps per CTA (60 teams; 16 warps with the control warp: 128 registers)

struct LatRec {
  double sel;                    // selection key (mode 0: the column norm^2; mode 1: 1 at pos == k)
  long long pk;                  // pos | valid << 33
  double xk;                     // the candidate's pivot-row element
  double nrm;                    // its norm^2 over rows >= k
  double fro;                    // the source CTA's sum of squared column norms (step 0, mode 0)
  double pad;
};
static_assert(sizeof(LatRec) == 48, "LatRec is pushed as three 16-byte chunks");

struct LatWin {                  // written by the control warp
  double alpha, beta, vk;
  int wpos, skip;
  uint32_t vaddr;                // shared address of the winner's column
  int pad;
};

template <int NR, int NWC>
struct LatShared {
  static constexpr int H = 8 * NR;
  double wpub[2][NWC][H];                // per-warp candidate column (absolute rows, rows <= k zeroed)
  double cx[2][LAT_SP_MAXC][H];          // received columns (one round: per source CTA; two rounds: slot 0)
  LatRec wrec[2][NWC];
  LatRec crec[2][PRRP_CLUSTER_MAX];
  LatWin win[2];
  unsigned long long barA[2], barB[2];
  double fro_warp[NWC];
  double alog[H];
  int slog[H];
  double fro;
};

__device__ __forceinline__ double lat_lds(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}

template <int V>
struct LatIC { static constexpr int value = V; };

// p1_best_lane with the common case first: one reduction on the high word
// and a ballot decide unless two candidates share their top 32 bits
__device__ __forceinline__ int lat_best_lane(unsigned long long u, unsigned pos) {
  const unsigned hi = (unsigned)(u >> 32), lo = (unsigned)u;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  if (mh != 0u) {
    const unsigned t1 = __ballot_sync(0xffffffffu, hi == mh);
    if ((t1 & (t1 - 1u)) == 0u) return __ffs(t1) - 1;
  }
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  if ((mh | ml) == 0u) return -1;
  const bool top = hi == mh && lo == ml;
  const unsigned tie = __ballot_sync(0xffffffffu, top);
  if ((tie & (tie - 1u)) == 0u) return __ffs(tie) - 1;
  const unsigned mp = __reduce_min_sync(0xffffffffu, top ? pos : 0xffffffffu);
  return __ffs(__ballot_sync(0xffffffffu, top && pos == mp)) - 1;
}

// x[ku] for a CTA-uniform ku in [U0, U0 + 4) (predicated selects, no local memory)
template <int NR, int U0>
__device__ __forceinline__ double lat_pick(const double (&x)[NR], int ku) {
  double v = x[U0];
#pragma unroll
  for (int u = U0 + 1; u < NR && u < U0 + 4; ++u)
    if (u == ku) v = x[u];
  return v;
}

template <int NR>
__device__ __forceinline__ double lat_pick_any(const double (&x)[NR], int ku) {
  double v = x[0];
#pragma unroll
  for (int u = 1; u < NR; ++u)
    if (u == ku) v = x[u];
  return v;
}

// numpy pairwise sum of squares of rows [base, h) of a team's column; thread
// q holds rows 8u + q.  Result in every thread of the team.  The caller
// guarantees 8 U0 <= base <= 8 (U0 + 4): blocks below U0 are finished rows,
// blocks U0 .. U0+4 test the rows against base, the blocks above are taken
// whole (FULL, i.e. h == 8 NR: only the last block can hold trailing terms).
template <int NR, bool FULL, int U0>
__device__ __forceinline__ double lat_sumsq(const double (&x)[NR], int q, int lane0, int base, int h, int ulast) {
  const int n = h - base;                          // uniform
  if (n <= 0) return -0.0;
  const int nt = n >= 8 ? (n & 7) : n;             // trailing terms added in row order
  const int top = h - nt;                          // rows [base, top) feed the eight strided accumulators
  double acc = -0.0;
#pragma unroll
  for (int u = U0; u < NR; ++u) {
    const int i = 8 * u + q;
    const bool lo_ok = u > U0 + 4 || i >= base;
    const bool hi_ok = (FULL && u < NR - 1) || i < top;
    if (u > U0 + 4 && FULL && u < NR - 1) acc = add_rn(acc, sq_rn(x[u]));
    else if (lo_ok && hi_ok) acc = add_rn(acc, sq_rn(x[u]));
  }
  double res = -0.0;
  if (n >= 8) {
    // slot s = (q - base) & 7 lives in lane lane0 + ((s + base) & 7)
    const int s = (q - base) & 7;
    double r = acc;
    r = add_rn(r, __shfl_sync(0xffffffffu, r, lane0 + (((s ^ 1) + base) & 7)));
    r = add_rn(r, __shfl_sync(0xffffffffu, r, lane0 + (((s ^ 2) + base) & 7)));
    r = add_rn(r, __shfl_sync(0xffffffffu, r, lane0 + (((s ^ 4) + base) & 7)));
    res = r;
  }
  if (nt > 0) {
    // the thread's last row (>= top for the lanes that hold a trailing term);
    // all seven candidate terms are fetched up front (independent shuffles),
    // then the live ones are added in row order
    const double xl = FULL ? x[NR - 1] : lat_pick_any<NR>(x, ulast);
    const double tv = sq_rn(xl);
    double tt[7];
#pragma unroll
    for (int j = 0; j < 7; ++j) tt[j] = __shfl_sync(0xffffffffu, tv, lane0 + ((top + j) & 7));
#pragma unroll
    for (int j = 0; j < 7; ++j)
      if (j < nt) res = add_rn(res, tt[j]);
  }
  return res;
}

template <int NR, int CPT, int NWC, bool FULL>
__global__ void __launch_bounds__(32 * (NWC + 1), 1) panel_lat_kernel(PanelArgs a) {
  constexpr int TEAMS = NWC * 4;
  constexpr int hch = 4 * NR;                          // 16-byte chunks of a column (all 8 NR rows: rows >= h are zero)
  using SH = LatShared<NR, NWC>;
  extern __shared__ __align__(16) unsigned char lat_dyn[];
  SH& S = *reinterpret_cast<SH*>(lat_dyn);
  __shared__ int s_failed;
  cg::cluster_group cl = cg::this_cluster();
  if (node_passes(a)) return;                          // uniform over the cluster (read-only input)
  const int C = (int)cl.num_blocks();
  const int c = (int)cl.block_rank();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool ctl = warp == NWC;                        // the control warp
  const int team = t >> 3, q = t & 7, lane0 = lane & ~7;
  const uint32_t barA0 = (uint32_t)__cvta_generic_to_shared(&S.barA[0]);
  const uint32_t barB0 = (uint32_t)__cvta_generic_to_shared(&S.barB[0]);
  if (t == 0 && C > 1) {
    p1_bar_init(barA0);
    p1_bar_init(barA0 + 8);
    p1_bar_init(barB0);
    p1_bar_init(barB0 + 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (C == 1) {
    if (t == 0) s_failed = prrp_failed(a.st);
    __syncthreads();
    if (s_failed) return;
  } else if (cluster_failed(a.st, &s_failed)) {        // (a cluster barrier, which also publishes the inits)
    return;
  }
  const int h = a.h;
  const int mode = a.mode;
  const int steps = a.steps;
  const bool two_round = C > LAT_SP_MAXC;
  const int64_t j0 = (int64_t)c * a.per;
  const int nl = (int)max((int64_t)0, min(a.per, a.p - j0));
  const int ulast = (h - 1 - q) >= 0 ? (h - 1 - q) >> 3 : 0;

  double x[CPT][NR];
  int pos[CPT];
  int jcol[CPT];
  double nrm[CPT];
  bool on[CPT];
#pragma unroll
  for (int cc = 0; cc < CPT; ++cc) {
    const int jl = cc * TEAMS + team;
    on[cc] = !ctl && jl < nl;
    pos[cc] = INT_MAX;
    jcol[cc] = 0;
    if (on[cc]) {
      const int64_t qq = j0 + jl;
      const int64_t j = mode == 0 ? qq : (int64_t)a.perm[qq];
      const int64_t row = a.rowidx ? a.rowidx[j] : j;
      const double* src = member_row(a.src, a.ld, row);
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int i = 8 * u + q;
        x[cc][u] = i < h ? src[i] : 0.0;
      }
      pos[cc] = (int)qq;
      jcol[cc] = (int)j;
    } else {
#pragma unroll
      for (int u = 0; u < NR; ++u) x[cc][u] = 0.0;
    }
  }
  {
    double f = 0.0;
#pragma unroll
    for (int cc = 0; cc < CPT; ++cc) {
      nrm[cc] = lat_sumsq<NR, FULL, 0>(x[cc], q, lane0, 0, h, ulast);
      if (on[cc] && q == 0) f += nrm[cc];
    }
    for (int o = 16; o; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
    if (lane == 0 && !ctl) S.fro_warp[warp] = f;
    __syncthreads();
    if (t == 0) {
      double s = 0.0;
      for (int w = 0; w < NWC; ++w) s += S.fro_warp[w];
      S.fro = mode == 0 ? s : 0.0;
    }
    __syncthreads();
  }
  const bool log_refl = a.refl != nullptr && c == 0;
  // PRRP_PANEL_PROF=1 PRRP_PANEL_TL=<panel>: clock64 marks of compute thread 0
  // and of the control warp's lane 0 (second half of the buffer) of CTA 0
  long long* tl = (a.prof && c == 0 && (t == 0 || t == 32 * NWC) && a.panel_id == a.prof[6])
                      ? a.prof + 8 + (t == 0 ? 0 : 1024) : nullptr;
#define LAT_TL(m) if (tl) tl[k * 8 + (m)] = clock64();
  // a mark that waits for `dep` (a value loaded after a barrier: the barrier
  // instruction itself does not block, its first dependent use does)
#define LAT_TLD(m, dep) if (tl) { asm volatile("" :: "r"(dep)); tl[k * 8 + (m)] = clock64(); }

  // One pivot step, specialised on U0: steps k in [8 U0, 8 U0 + 32) touch only
  // the row blocks u >= U0 (blocks U0 .. ku-1 hold finished rows: the
  // published column is zero there, so they take no part in the dot
  // products and stay unchanged).
  auto step = [&](auto u0c, const int k) {
    constexpr int U0 = decltype(u0c)::value;
    const int buf = k & 1;
    const int r = k & 7, ku = k >> 3;
    constexpr int ch0 = 4 * U0, nch = hch - ch0;       // chunks of a column that travel (rows >= 8 U0)
    if (ctl) {
      // ================================================= control warp
      const uint32_t barA = barA0 + 8 * buf, barB = barB0 + 8 * buf;
      if (lane == 0 && C > 1) {
        if (two_round) {
          p1_bar_expect(barA, (uint32_t)(C * 48));
          p1_bar_expect(barB, (uint32_t)(16 * nch));
        } else {
          p1_bar_expect(barA, (uint32_t)(C * (48 + 16 * nch)));
        }
      }
      __syncthreads();                                 // bar 1: the warps' candidates are published
      LAT_TLD(0, (int)S.wrec[buf][0].pk)
      const LatRec* Wp;
      const double* vsrc;
      if (C > 1) {
        // the pusher warps (compute warps 0 .. C-1) send this CTA's candidate
        // to every CTA; the control warp only waits for the C candidates
        p1_bar_wait(barA, (uint32_t)((k >> 1) & 1));
        LAT_TL(1)
        int cb;
        {
          // the wire chunks {sel, pk} {xk, nrm} {fro, 0} are LatRec's layout
          const LatRec& cr = S.crec[buf][lane < C ? lane : 0];
          const bool ok = lane < C && (cr.pk >> 33) != 0;
          const unsigned long long u = ok ? p1_ukey(cr.sel, true) : 0ull;
          cb = lat_best_lane(u, ok ? (unsigned)cr.pk : 0xffffffffu);
          if (cb < 0) cb = 0;
        }
        if (k == 0 && mode == 0 && c == 0) {
          double f = lane < C ? S.crec[buf][lane].fro : 0.0;
          for (int o = 16; o; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
          if (lane == 0) *a.fro = sqrt(f);
        }
        if (two_round) {
          p1_bar_wait(barB, (uint32_t)((k >> 1) & 1));
          vsrc = S.cx[buf][0];
        } else {
          vsrc = S.cx[buf][cb];
        }
        Wp = &S.crec[buf][cb];
      } else {
        int wbest;
        {
          const LatRec& wr = S.wrec[buf][lane < NWC ? lane : 0];
          const bool ok = lane < NWC && (wr.pk >> 33) != 0;
          const unsigned long long u = ok ? p1_ukey(wr.sel, true) : 0ull;
          wbest = lat_best_lane(u, ok ? (unsigned)wr.pk : 0xffffffffu);
          if (wbest < 0) wbest = 0;
        }
        Wp = &S.wrec[buf][wbest];
        vsrc = S.wpub[buf][wbest];
        if (k == 0 && mode == 0 && lane == 0) *a.fro = sqrt(S.fro);
      }
      const double xk = Wp->xk, nn = Wp->nrm;
      const int wpos = (int)(unsigned)Wp->pk;
      LAT_TLD(2, wpos)
      if (lane == 0) {
        S.win[buf].wpos = wpos;
        S.win[buf].vaddr = (uint32_t)__cvta_generic_to_shared(vsrc);
      }
      __syncthreads();                                 // bar 2: the winner and its column are known
      // the reflector scalars (pivoted_qr.py:43-55), while the compute warps
      // form the partial dot products
      const double normx = __dsqrt_rn(nn);
      int skip = normx == 0.0;
      double alpha = xk >= 0.0 ? -normx : normx;
      const double vk = sub_rn(xk, alpha);
      const double half_vtv = mul_rn(normx, add_rn(normx, fabs(xk)));
      double beta = skip ? 0.0 : __drcp_rn(half_vtv);
      if (half_vtv == 0.0) skip = 1;
      if (skip) { alpha = xk; beta = 0.0; }
      if (lane == 0) {
        S.win[buf].alpha = alpha;
        S.win[buf].beta = beta;
        S.win[buf].vk = vk;
        S.win[buf].skip = skip;
        S.alog[k] = alpha;
        S.slog[k] = skip;
      }
      LAT_TLD(3, __double2hiint(beta))
      __syncthreads();                                 // bar 3: alpha, beta, v_k
      if (log_refl) {
        double* lg = a.refl + (int64_t)k * (h + 1);
        for (int i = lane; i < h; i += 32) lg[i] = (skip || i < k) ? 0.0 : (i == k ? vk : vsrc[i]);
        if (lane == 0) lg[h] = skip ? 0.0 : beta;
      }
      return;
    }
    // =================================================== compute warps
    LAT_TL(0)
    // ---- A: the team's best column, warp argmax, the warp's best column published
    {
      unsigned long long bu = 0ull;
      int bpos = INT_MAX;
      double bn = 0.0;
      int bc = 0;
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) {
        const bool live = on[cc] && pos[cc] >= k;
        const double sel = mode == 0 ? nrm[cc] : (pos[cc] == k ? 1.0 : -1.0);
        const unsigned long long u = p1_ukey(sel, live);
        if (cc == 0 || u > bu || (u == bu && u != 0ull && pos[cc] < bpos)) {
          bu = u; bpos = pos[cc]; bn = nrm[cc]; bc = cc;
        }
      }
      const int wl = lat_best_lane(q == 0 ? bu : 0ull, (unsigned)bpos);
      if (wl < 0) {
        if (lane == 0) { S.wrec[buf][warp].sel = -INFINITY; S.wrec[buf][warp].pk = 0ll; }
      } else if ((lane >> 3) == (wl >> 3)) {
        double* wp = S.wpub[buf][warp] + q;
        LatRec& wr = S.wrec[buf][warp];
#pragma unroll
        for (int u = U0; u < NR; ++u) {
          double xv = x[0][u];
#pragma unroll
          for (int cc = 1; cc < CPT; ++cc)
            if (cc == bc) xv = x[cc][u];
          if (u < U0 + 4) {
            // the pivot block: zero up to and including row k; x_k goes into the record
            if (u == ku && q == r) wr.xk = xv;
            xv = (u < ku || (u == ku && q <= r)) ? 0.0 : xv;
          }
          wp[8 * u] = xv;
        }
        if (q == 0) {
          wr.sel = mode == 0 ? bn : 1.0;
          wr.pk = (long long)(unsigned)bpos | (1ll << 33);
          wr.nrm = bn;
        }
      }
    }
    LAT_TL(1)
    __syncthreads();                                   // bar 1
    if (C > 1 && warp < C) {
      // ---- pusher warps: warp w sends this CTA's candidate (record, and in
      // one-round mode its column) to the CTAs w, w + NWC, ...
      const uint32_t barA = barA0 + 8 * buf, barB = barB0 + 8 * buf;
      int wbest;
      {
        const LatRec& wr = S.wrec[buf][lane < NWC ? lane : 0];
        const bool ok = lane < NWC && (wr.pk >> 33) != 0;
        const unsigned long long u = ok ? p1_ukey(wr.sel, true) : 0ull;
        wbest = lat_best_lane(u, ok ? (unsigned)wr.pk : 0xffffffffu);
        if (wbest < 0) wbest = 0;
      }
      const LatRec& b = S.wrec[buf][wbest];
      const double2* src = reinterpret_cast<const double2*>(S.wpub[buf][wbest]);
      for (int d = warp; d < C; d += NWC) {
        const uint32_t rbar = p1_mapa(barA, d);
        if (lane < 3) {
          const uint32_t dst = p1_mapa((uint32_t)__cvta_generic_to_shared(&S.crec[buf][c]), d) + 16 * lane;
          const double d0 = lane == 0 ? b.sel : (lane == 1 ? b.xk : S.fro);
          const double d1 = lane == 0 ? __longlong_as_double(b.pk) : (lane == 1 ? b.nrm : 0.0);
          p1_push16(dst, d0, d1, rbar);
        }
        if (!two_round) {
          const uint32_t dst0 = p1_mapa((uint32_t)__cvta_generic_to_shared(&S.cx[buf][c][0]), d);
#pragma unroll
          for (int ch = ch0 + lane; ch < hch; ch += 32) {
            const double2 v = src[ch];
            p1_push16(dst0 + 16 * ch, v.x, v.y, rbar);
          }
        }
      }
      if (two_round) {
        // second round: the cluster winner's pushers send its column
        p1_bar_wait(barA, (uint32_t)((k >> 1) & 1));
        int cb;
        {
          const LatRec& cr = S.crec[buf][lane < C ? lane : 0];
          const bool ok = lane < C && (cr.pk >> 33) != 0;
          const unsigned long long u = ok ? p1_ukey(cr.sel, true) : 0ull;
          cb = lat_best_lane(u, ok ? (unsigned)cr.pk : 0xffffffffu);
          if (cb < 0) cb = 0;
        }
        if (cb == c) {
          for (int d = warp; d < C; d += NWC) {
            const uint32_t dst0 = p1_mapa((uint32_t)__cvta_generic_to_shared(&S.cx[buf][0][0]), d);
            const uint32_t rbarB = p1_mapa(barB, d);
#pragma unroll
            for (int ch = ch0 + lane; ch < hch; ch += 32) {
              const double2 v = src[ch];
              p1_push16(dst0 + 16 * ch, v.x, v.y, rbarB);
            }
          }
        }
      }
    }
    LAT_TL(2)
    __syncthreads();                                   // bar 2: winner known
    const int wpos = S.win[buf].wpos;
    LAT_TLD(3, wpos)
    const uint32_t va = S.win[buf].vaddr + 8 * q;
    bool act[CPT];
    double dd[CPT], xkk[CPT];
    {
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) {
        const bool live = on[cc] && pos[cc] >= k;
        const bool win = live && pos[cc] == wpos;
        if (live && !win && pos[cc] == k) pos[cc] = wpos;   // displaced by the interchange
        if (win) pos[cc] = k;
        act[cc] = live && !win;
      }
      // ---- D1: partial dot products d' = sum_{i > k} p_i x_i, and x_k
      double d0[CPT], d1[CPT];
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) { d0[cc] = 0.0; d1[cc] = 0.0; }
#pragma unroll
      for (int u = U0; u < NR; ++u) {
        const double v = lat_lds(va + 64 * u);
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
          if (u & 1) d1[cc] = fma(v, x[cc][u], d1[cc]);
          else d0[cc] = fma(v, x[cc][u], d0[cc]);
        }
      }
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) {
        double d = d0[cc] + d1[cc];
        d += __shfl_xor_sync(0xffffffffu, d, 1);
        d += __shfl_xor_sync(0xffffffffu, d, 2);
        d += __shfl_xor_sync(0xffffffffu, d, 4);
        dd[cc] = d;
        xkk[cc] = __shfl_sync(0xffffffffu, lat_pick<NR, U0>(x[cc], ku), lane0 + r);
      }
    }
    LAT_TLD(4, __double2hiint(dd[0]))
    __syncthreads();                                   // bar 3: alpha, beta, v_k
    {
      const double beta = S.win[buf].beta, vk = S.win[buf].vk;
      const int skip = S.win[buf].skip;
      LAT_TLD(5, skip)
      if (!skip) {
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
          if (act[cc]) {
            const double nw = -mul_rn(beta, fma(vk, xkk[cc], dd[cc]));
#pragma unroll
            for (int u = U0; u < NR; ++u) {
              // (row k of the published column is zero: v_k comes from the control warp)
              double v = lat_lds(va + 64 * u);
              if (u < U0 + 4 && u == ku && q == r) v = vk;
              x[cc][u] = fma(v, nw, x[cc][u]);
            }
          }
        }
      }
      LAT_TLD(6, __double2hiint(x[0][NR - 1]))
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) nrm[cc] = lat_sumsq<NR, FULL, U0>(x[cc], q, lane0, k + 1, h, ulast);
    }
    LAT_TLD(7, __double2hiint(nrm[0]))
  };
#pragma unroll 1
  for (int k = 0; k < min(steps, 32); ++k) step(LatIC<0>{}, k);
  if constexpr (NR > 4) {
#pragma unroll 1
    for (int k = 32; k < min(steps, 64); ++k) step(LatIC<4>{}, k);
  }
  if constexpr (NR > 8) {
#pragma unroll 1
    for (int k = 64; k < min(steps, 96); ++k) step(LatIC<8>{}, k);
#pragma unroll 1
    for (int k = 96; k < steps; ++k) step(LatIC<12>{}, k);
  }
#undef LAT_TL
#undef LAT_TLD
  if (C > 1) cl.sync(); else __syncthreads();
  // ---- R by position, column order; rows >= s of the pivot column of step
  // s are (alpha_s, 0, ..., 0) unless step s was skipped
#pragma unroll
  for (int cc = 0; cc < CPT; ++cc) {
    if (on[cc]) {
      const int ps = pos[cc];
      const bool ov = ps < steps && !S.slog[ps < steps ? ps : 0];
      const double al = ov ? S.alog[ps] : 0.0;
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int i = 8 * u + q;
        if (i < h) a.Rbuf[(int64_t)i * a.p + ps] = ov && i >= ps ? (i == ps ? al : 0.0) : x[cc][u];
      }
      if (q == 0) a.perm[ps] = (int32_t)jcol[cc];
    }
  }
}

template <int NR, int NWC>
constexpr size_t lat_smem() { return sizeof(LatShared<NR, NWC>); }
