// Distributed CALU_PRRP, one
// process per GPU.  Layout: column block-cyclic over the process grid's
// columns (P_r = 1, P_c = nranks): global column block J (width b) lives on
// rank J mod P_c as local block J div P_c; every rank holds all m rows of its
// blocks (row-major, local leading dimension lda).  Rows keep physical slots
// and the trailing region's logical order (pos2row) is replicated on every
// rank, exactly as in the single-GPU driver (calu.cuh).
//
// Per panel k (owner o = k mod P_c):
//   select (owner)    tournament over the panel's rows (leaves, merges, the
//                     flat tree or the single node: the same device nodes as
//                     caluprrp_enqueue), the reorder [pivots, rest ascending]
//                     (tournament.py:214-215), the row moves of the panel
//                     columns, the final unpivoted QR of the permuted panel
//                     and its multipliers (tournament.py:271-272), L21 in
//                     physical slot order, GEPP of the pivot block
//                     (luprrp.py:107-127); packed into one message:
//                     [DevState | D (b x b) | root pivots + count | gperm |
//                      single-node order (m) | L21 (b x ldl_k)]
//   broadcast         the message from the owner (NCCL through
//                     torch.distributed, or any transport: the library only
//                     exposes the buffer)
//   apply (all)       the same reorder from the message's pivots (every rank
//                     updates its own pos2row / row order identically), the
//                     row moves of its other columns, the block-row finish of
//                     its columns (blockrow_w with the global column map), the
//                     trailing update of its columns (DMMA Schur kernel, the
//                     same k order, so every element is bit-identical to the
//                     single-GPU factorization), and (owner) the compose
//                     L21 <- L21[:, perm] L11 of the stored L.
// The statistics (growth maxima, swap counts, node sizes) are max-reduced by
// the caller at the end; errors travel in the message, so every rank stops at
// the owner's first error with the same record.
#pragma once

struct CaluDist {
  int64_t m = 0, n = 0, n_loc = 0, lda = 0;
  int b = 0, P = 0, nranks = 1, rank = 0, npanels = 0, maxnodes = 0, nnodes = 0;
  double tau = 2.0;
  double* A = nullptr;                  // local columns (caller-owned)
  int64_t* perm = nullptr;              // global row order (caller-owned, m)
  std::vector<void*> bufs;
  DevState* st = nullptr;
  DevState* st_r12 = nullptr;
  int64_t ldl = 0, ld21t = 0;
  double* Lg = nullptr;                 // L21 in logical order (owner)
  double* Rsmall = nullptr;
  double* refl = nullptr;
  double* Qneg = nullptr;
  double* A21t = nullptr;
  int32_t* perm_small = nullptr;
  int32_t* final_live = nullptr;
  PanelBuffers B{};
  std::vector<NodeBufs> nodes;
  int32_t *cands = nullptr, *ccnt = nullptr, *want_all = nullptr, *live_all = nullptr;
  int32_t *node_rows = nullptr, *node_swaps = nullptr, *swaps_dev = nullptr;
  const int32_t** perms_dev = nullptr;
  int64_t* leaf_lo_dev = nullptr;
  int64_t* lpos_dummy = nullptr;
  int32_t* lpos_all = nullptr;
  int64_t* rowidx_all = nullptr;
  int64_t* pos2row = nullptr;
  int64_t* scratch = nullptr;
  int32_t* log2phys = nullptr;
  int32_t* ident = nullptr;
  int32_t* moved = nullptr;
  int32_t* mcnt = nullptr;
  double* a12 = nullptr;
  ComposeWs cws;                                                    // DMMA compose operands (launch_compose_w)
  int64_t lda12 = 0;
  int32_t* piv = nullptr;
  // message
  unsigned char* msgs[2] = {nullptr, nullptr};   // double-buffered by panel parity (look-ahead)
  unsigned char* msg = nullptr;                   // the current panel's message (set per call)
  size_t off_D = 0, off_piv = 0, off_cnt = 0, off_gperm = 0, off_full = 0, off_L = 0, msg_cap = 0;
  // root candidates of the last tournament (device pointers into cands / ccnt)
  int32_t* root = nullptr;
  int32_t* root_cnt = nullptr;
  int root_mode = 0;
  // statistics record for the caller's max-reduction (int64):
  // [orig, inter, finish, pmm (IEEE bits)] [swaps_dev (npanels)] [node_swaps] [node_rows]
  int64_t* red = nullptr;
  size_t red_len = 0;
  std::vector<std::vector<std::pair<int64_t, int>>> node_members;   // static (members, slot) per panel
  std::vector<int64_t> charges_tag;                                 // -1: single node / no tournament
  ~CaluDist() {
    for (void* p : bufs) cudaFree(p);
  }
  int owner(int k) const { return k % nranks; }
  int64_t local_col(int k) const { return (int64_t)(k / nranks) * b; }   // local column of global block k
  // first local column whose global column is >= g0 (g0 a multiple of b)
  int64_t local_from(int64_t g0) const {
    const int64_t J = g0 / b;
    const int64_t jl = J <= rank ? 0 : (J - rank + nranks - 1) / nranks;
    return std::min<int64_t>(n_loc, jl * b);
  }
  int64_t ldl_k(int k) const {
    const int64_t rows = m - (int64_t)k * b;
    const int64_t bj = std::min<int64_t>(b, n - (int64_t)k * b);
    return std::max<int64_t>(8, ((rows - bj + 7) / 8) * 8);
  }
  size_t msg_bytes(int k) const { return off_L + (size_t)b * ldl_k(k) * 8; }
  int p_eff(int k) const {
    const int64_t col0 = (int64_t)k * b;
    const int64_t bj = std::min<int64_t>(b, n - col0), rows = m - col0;
    if (rows <= bj) return 0;
    if (P == 0) {
      const int64_t first = std::min<int64_t>(rows, 2 * bj);
      return (int)(1 + (rows - first + bj - 1) / bj);
    }
    return (int)std::max<int64_t>(1, std::min<int64_t>(P, rows / (bj + 1)));
  }
};

__global__ void dist_state_out_kernel(const DevState* st, DevState* out) {
  if (threadIdx.x == 0) *out = *st;
}

// a failure recorded by the owner stops every rank with the same record
__global__ void dist_state_in_kernel(DevState* st, const DevState* msg) {
  if (threadIdx.x != 0 || msg->code == 0 || st->code != 0) return;
  st->panel = msg->panel;
  st->index = msg->index;
  st->column = msg->column;
  st->worst = msg->worst;
  st->tree_level = msg->tree_level;
  st->tree_index = msg->tree_index;
  st->err_inv = msg->err_inv;
  __threadfence();
  atomicExch(&st->code, msg->code);
}

// statistics record for the caller's max-reduction
__global__ void dist_stats_kernel(const DevState* st, const int32_t* swaps, int npanels, const int32_t* nsw,
                                  const int32_t* nrows, int nslots, int64_t* out) {
  for (int i = threadIdx.x; i < 4 + npanels + 2 * nslots; i += blockDim.x) {
    int64_t v;
    if (i == 0) v = (int64_t)st->orig_max;
    else if (i == 1) v = (int64_t)st->inter_max;
    else if (i == 2) v = (int64_t)st->finish_max;
    else if (i == 3) v = (int64_t)st->pmm;
    else if (i < 4 + npanels) v = swaps[i - 4];
    else if (i < 4 + npanels + nslots) v = nsw[i - 4 - npanels];
    else v = nrows[i - 4 - npanels - nslots];
    out[i] = v;
  }
}

// static tournament structure of every panel (members, node slot), as the
// single-GPU enqueue builds it: every rank knows it without communication
void calu_dist_structure(CaluDist& w) {
  w.node_members.assign(w.npanels, {});
  w.charges_tag.assign(w.npanels, -1);
  for (int k = 0; k < w.npanels; ++k) {
    const int64_t col0 = (int64_t)k * w.b;
    const int64_t bj = std::min<int64_t>(w.b, w.n - col0), rows = w.m - col0;
    const int pe = w.p_eff(k);
    if (pe <= 1) continue;
    w.charges_tag[k] = 0;
    int slot = 0;
    if (w.P == 0) {
      const int64_t first = std::min<int64_t>(rows, 2 * bj);
      w.node_members[k].push_back({first, slot++});
      for (int64_t lo = first; lo < rows; lo += bj) w.node_members[k].push_back({bj + std::min<int64_t>(bj, rows - lo), slot++});
    } else {
      const int64_t base = rows / pe, extra = rows % pe;
      for (int i = 0; i < pe; ++i) w.node_members[k].push_back({base + (i < extra ? 1 : 0), slot++});
      int64_t ncur = pe;
      while (ncur > 1) {
        const int64_t nm = ncur / 2;
        for (int64_t i = 0; i < nm; ++i) w.node_members[k].push_back({2 * bj, slot++});
        ncur = nm + (ncur % 2);
      }
    }
  }
}

void calu_dist_alloc(CaluDist& w, cudaStream_t s) {
  Arena ar(s, &w.bufs);
  const int64_t m = w.m;
  const int b = w.b;
  const bool flat = w.P == 0;
  w.maxnodes = flat ? (int)(m / std::max(1, b) + 2) : 2 * w.P;
  w.nnodes = flat ? 1 : w.maxnodes;
  w.st = new_state(ar, s);
  w.st_r12 = new_state(ar, s);
  w.ldl = ((m + 7) / 8) * 8;
  w.Lg = ar.get<double>((size_t)b * w.ldl);
  w.B.Rbuf = ar.get<double>((size_t)b * m);
  w.B.perm = ar.get<int32_t>(m);
  w.B.ovf = ar.get<double>(ovf_elems(b, m, b));
  w.B.cand = ar.get<double>(kMaxCand);
  w.B.cand_flat = ar.get<long long>(kMaxCand);
  w.B.moved = ar.get<int32_t>(2 * m);
  alloc_exchange(ar, s, w.B);
  w.Rsmall = ar.get<double>((size_t)b * b);
  w.refl = ar.get<double>((size_t)b * (b + 1));
  w.perm_small = ar.get<int32_t>(b);
  w.final_live = ar.get<int32_t>(1);
  w.Qneg = ar.get<double>((size_t)b * b);
  w.ld21t = ((m + 7) / 8) * 8;
  w.A21t = ar.get<double>((size_t)b * w.ld21t);
  const int64_t leafmax =
      flat ? 2 * b : m / std::max<int64_t>(1, std::min<int64_t>(w.P, std::max<int64_t>(1, m / (b + 1)))) + 1;
  const int64_t pnode = std::max<int64_t>(leafmax, 2 * b + 2);
  w.lpos_all = ar.get<int32_t>((size_t)w.nnodes * 2 * b);
  w.rowidx_all = ar.get<int64_t>((size_t)w.nnodes * 2 * b);
  w.nodes.resize(w.nnodes);
  for (int i = 0; i < w.nnodes; ++i) {
    NodeBufs& nb = w.nodes[i];
    nb.B.Rbuf = ar.get<double>((size_t)b * pnode);
    nb.B.perm = ar.get<int32_t>(pnode);
    nb.B.ovf = ar.get<double>(ovf_elems(b, pnode, b));
    nb.B.cand = ar.get<double>(kMaxCand);
    nb.B.cand_flat = ar.get<long long>(kMaxCand);
    nb.B.moved = ar.get<int32_t>(2 * pnode);
    nb.B.fro = ar.get<double>(1);
    nb.B.refl = ar.get<double>((size_t)b * (b + 1));   // reflector log: the root's is the final QR (calu_root_qr_kernel)
    nb.ldl = ((pnode + 7) / 8) * 8;
    nb.L21 = ar.get<double>((size_t)b * nb.ldl);
    nb.lpos_in = w.lpos_all + (size_t)i * 2 * b;
    nb.rowidx = w.rowidx_all + (size_t)i * 2 * b;
  }
  w.cands = ar.get<int32_t>((size_t)2 * w.nnodes * b);
  w.ccnt = ar.get<int32_t>((size_t)2 * w.nnodes);
  w.want_all = ar.get<int32_t>(w.nnodes);
  w.live_all = ar.get<int32_t>(w.nnodes);
  w.node_rows = ar.get<int32_t>((size_t)w.npanels * w.maxnodes);
  w.node_swaps = ar.get<int32_t>((size_t)w.npanels * w.maxnodes);
  w.swaps_dev = ar.get<int32_t>(w.npanels);
  CU_TRY(cudaMemsetAsync(w.node_rows, 0, sizeof(int32_t) * w.npanels * w.maxnodes, s));
  CU_TRY(cudaMemsetAsync(w.node_swaps, 0, sizeof(int32_t) * w.npanels * w.maxnodes, s));
  CU_TRY(cudaMemsetAsync(w.swaps_dev, 0, sizeof(int32_t) * w.npanels, s));
  w.perms_dev = ar.get<const int32_t*>(w.nnodes);
  w.leaf_lo_dev = ar.get<int64_t>(w.nnodes);
  w.pos2row = ar.get<int64_t>(m);
  w.scratch = ar.get<int64_t>(3 * m);
  w.log2phys = ar.get<int32_t>(m);
  w.ident = ar.get<int32_t>(m);
  w.moved = ar.get<int32_t>(2 * m);
  w.mcnt = ar.get<int32_t>(1);
  w.lda12 = std::max<int64_t>(2, ((w.n_loc + 1) / 2) * 2);
  w.a12 = ar.get<double>((size_t)b * w.lda12);
  w.cws = compose_ws(ar, s, m, b);
  w.piv = ar.get<int32_t>(b);
  for (int i0 = 0; i0 < w.nnodes; i0 += 32) {
    PtrPack pk{};
    const int cnt = std::min(32, w.nnodes - i0);
    for (int i = 0; i < cnt; ++i) pk.p[i] = w.nodes[i0 + i].B.perm;
    store_ptrs_kernel<<<1, 32, 0, s>>>(pk, cnt, w.perms_dev + i0);
  }
  // message layout
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  w.off_D = al(sizeof(DevState));
  w.off_cnt = al(w.off_D + (size_t)b * b * 8);
  w.off_piv = w.off_cnt + 256;                            // [cnt] then root pivots (b)
  w.off_gperm = al(w.off_piv + (size_t)b * 4);
  w.off_full = al(w.off_gperm + (size_t)b * 4);
  w.off_L = al(w.off_full + (size_t)m * 4);
  w.msg_cap = w.off_L + (size_t)b * w.ldl * 8;
  for (int i = 0; i < 2; ++i) {
    w.msgs[i] = ar.get<unsigned char>(w.msg_cap);
    CU_TRY(cudaMemsetAsync(w.msgs[i], 0, w.msg_cap, s));
  }
  w.msg = w.msgs[0];
  w.red_len = 4 + (size_t)w.npanels + 2 * (size_t)w.npanels * w.maxnodes;
  w.red = ar.get<int64_t>(w.red_len);
  const int sms = caps().sms;
  iota_kernel<<<sms, 256, 0, s>>>(w.perm, m);
  iota_kernel<<<sms, 256, 0, s>>>(w.pos2row, m);
  iota32_kernel<<<sms, 256, 0, s>>>(w.ident, m);
  if (w.n_loc > 0) maxabs_kernel<<<sms * 4, 256, 0, s>>>(w.A, w.lda, m, w.n_loc, w.st);
  CU_TRY(cudaGetLastError());
}

// Owner side of panel k: tournament, reorder, panel-column row moves, L21,
// GEPP of the pivot block; the message is complete when this returns (stream
// ordered).
void calu_dist_select(CaluDist& w, int k, cudaStream_t s) {
  // the same engine per node as the single-GPU driver (caluprrp_enqueue)
  struct LatScope {
    ~LatScope() { tl_lat_cmax = -1; }
  } lat_scope;
  tl_lat_cmax = calu_chain_bound(w.m, w.n, w.b, k, w.P == 0) ? 16 : 0;
  w.msg = w.msgs[k & 1];
  const int b = w.b;
  const int64_t m = w.m, n = w.n, col0 = (int64_t)k * b;
  const int bj = (int)std::min<int64_t>(b, n - col0);
  const int64_t rows = m - col0;
  const int64_t lc0 = w.local_col(k);
  const int sms = caps().sms;
  // column-shifted base: Ash[row * lda + col0 + j] = A[row * lda + lc0 + j]
  double* Ash = w.A + lc0 - col0;
  double* D = reinterpret_cast<double*>(w.msg + w.off_D);
  int32_t* gperm = reinterpret_cast<int32_t*>(w.msg + w.off_gperm);
  int32_t* mcnt_msg = reinterpret_cast<int32_t*>(w.msg + w.off_cnt);
  int32_t* piv_msg = reinterpret_cast<int32_t*>(w.msg + w.off_piv);
  int32_t* full = reinterpret_cast<int32_t*>(w.msg + w.off_full);
  const int64_t ldk = w.ldl_k(k);
  double* Lp = reinterpret_cast<double*>(w.msg + w.off_L);
  DevState* st = w.st;
  const int pe = w.p_eff(k);
  const int maxnodes = w.maxnodes;
  if (rows > bj) {
    auto run_level = [&](const std::vector<int64_t>& lo, const std::vector<int64_t>& cnt, bool leaves, int level,
                         int slot0) {
      cudaEvent_t fk;
      CU_TRY(cudaEventCreateWithFlags(&fk, cudaEventDisableTiming));
      CU_TRY(cudaEventRecord(fk, s));
      const int nn = (int)lo.size();
      for (int i = 0; i < nn; ++i) {
        cudaStream_t ns = node_stream(i);
        CU_TRY(cudaStreamWaitEvent(ns, fk, 0));
        const int64_t* ridx = leaves ? w.pos2row + col0 + lo[i] : w.nodes[i].rowidx;
        if (cnt[i] <= bj) continue;
        PanelBuffers nbuf = w.nodes[i].B;
        nbuf.live = leaves ? nullptr : w.live_all + i;
        nbuf.want = w.want_all + i;
        nbuf.node_rows = w.node_rows + (size_t)k * maxnodes;
        const int cmax_level = tl_lat_cmax;             // same engine shapes as caluprrp_enqueue
        if (leaves && tl_lat_cmax > 0) tl_lat_cmax = std::min(tl_lat_cmax, calu_leaf_cmax());
        strong_rrqr_panel(Ash + col0, w.lda, bj, cnt[i], bj, w.tau, k, w.nodes[i].L21, w.nodes[i].ldl, nbuf, st,
                          w.node_swaps + (size_t)k * maxnodes, nullptr, nullptr, nullptr, false, ns, ridx, slot0 + i,
                          level, i);
        tl_lat_cmax = cmax_level;
      }
      for (int i = 0; i < nn; ++i) {
        cudaEvent_t jn;
        CU_TRY(cudaEventCreateWithFlags(&jn, cudaEventDisableTiming));
        CU_TRY(cudaEventRecord(jn, node_stream(i)));
        CU_TRY(cudaStreamWaitEvent(s, jn, 0));
        CU_TRY(cudaEventDestroy(jn));
      }
      CU_TRY(cudaEventDestroy(fk));
    };
    int32_t* cur = w.cands;
    int32_t* ccur = w.ccnt;
    int64_t root_p = 0;     // columns of the root node's QRCP (the final QR reuses it)
    if (pe > 1 && w.P == 0) {
      const int64_t first = std::min<int64_t>(rows, 2 * bj);
      calu_leaf_lo_kernel<<<1, 64, 0, s>>>(w.leaf_lo_dev, 1, rows, 0);
      run_level({0}, {first}, true, 0, 0);
      int slot = 1;
      int32_t* nxt = w.cands + (size_t)b;
      int32_t* cnxt = w.ccnt + 1;
      calu_select_kernel<<<1, 128, 0, s>>>(w.perms_dev, nullptr, w.leaf_lo_dev, bj, w.want_all, w.live_all, 0, cur,
                                           ccur, 2 * b, w.st);
      int level = 1;
      for (int64_t lo = first; lo < rows; lo += bj, ++level) {
        const int64_t len = std::min<int64_t>(bj, rows - lo);
        calu_flat_inputs_kernel<<<1, 128, 0, s>>>(cur, ccur, bj, lo, (int)len, w.lpos_all, w.rowidx_all,
                                                  w.live_all, w.pos2row, col0, w.st);
        root_p = bj + len;
        run_level({0}, {bj + len}, false, level, slot++);
        calu_select_kernel<<<1, 128, 0, s>>>(w.perms_dev, w.lpos_all, nullptr, bj, w.want_all, w.live_all, 1, nxt,
                                             cnxt, 2 * b, w.st);
        std::swap(cur, nxt);
        std::swap(ccur, cnxt);
      }
      w.root_mode = 0;
    } else if (pe == 1) {
      PanelBuffers Bk = w.B;
      Bk.moved = w.moved;
      Bk.moved_cnt = w.mcnt;
      {
        const int keep = tl_lat_cmax;                   // the single node is the LU_PRRP panel (see caluprrp_enqueue)
        tl_lat_cmax = -1;
        strong_rrqr_panel(Ash + col0, w.lda, bj, rows, bj, w.tau, k, w.Lg, w.ldl, Bk, st, w.swaps_dev, nullptr,
                          nullptr, nullptr, false, s, w.pos2row + col0);
        tl_lat_cmax = keep;
      }
      CU_TRY(cudaMemcpyAsync(full, w.B.perm, sizeof(int32_t) * rows, cudaMemcpyDeviceToDevice, s));
      w.root_mode = 1;
    } else {
      std::vector<int64_t> lo(pe), cnt(pe);
      const int64_t base = rows / pe, extra = rows % pe;
      int64_t start = 0;
      for (int i = 0; i < pe; ++i) {
        cnt[i] = base + (i < extra ? 1 : 0);
        lo[i] = start;
        start += cnt[i];
      }
      calu_leaf_lo_kernel<<<1, 64, 0, s>>>(w.leaf_lo_dev, pe, base, extra);
      run_level(lo, cnt, true, 0, 0);
      int slot = pe;
      int32_t* nxt = w.cands + (size_t)maxnodes * b;
      int32_t* cnxt = w.ccnt + maxnodes;
      calu_select_kernel<<<(unsigned)pe, 128, 0, s>>>(w.perms_dev, nullptr, w.leaf_lo_dev, bj, w.want_all,
                                                      w.live_all, 0, cur, ccur, 2 * b, w.st);
      int64_t ncur = pe;
      int level = 1;
      while (ncur > 1) {
        const int64_t nm = ncur / 2;
        calu_merge_inputs_kernel<<<(unsigned)nm, 128, 0, s>>>(cur, ccur, bj, (int)(2 * nm), w.lpos_all,
                                                              w.rowidx_all, w.live_all, w.pos2row, col0, 2 * b, w.st);
        root_p = 2 * bj;
        run_level(std::vector<int64_t>(nm, 0), std::vector<int64_t>(nm, 2 * bj), false, level, slot);
        slot += (int)nm;
        calu_select_kernel<<<(unsigned)nm, 128, 0, s>>>(w.perms_dev, w.lpos_all, nullptr, bj, w.want_all,
                                                        w.live_all, 1, nxt, cnxt, 2 * b, w.st);
        if (ncur % 2) {
          CU_TRY(cudaMemcpyAsync(nxt + nm * bj, cur + (ncur - 1) * bj, sizeof(int32_t) * bj,
                                 cudaMemcpyDeviceToDevice, s));
          CU_TRY(cudaMemcpyAsync(cnxt + nm, ccur + (ncur - 1), sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        }
        ncur = nm + (ncur % 2);
        std::swap(cur, nxt);
        std::swap(ccur, cnxt);
        ++level;
      }
      w.root_mode = 0;
    }
    if (w.root_mode == 0) {
      CU_TRY(cudaMemcpyAsync(mcnt_msg, ccur, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
      CU_TRY(cudaMemcpyAsync(piv_msg, cur, sizeof(int32_t) * bj, cudaMemcpyDeviceToDevice, s));
    }
    // the new logical order and the row moves (every rank repeats this reorder in apply)
    calu_reorder_kernel<<<1, 1024, 0, s>>>(w.root_mode == 0 ? piv_msg : nullptr, mcnt_msg,
                                           w.root_mode == 0 ? nullptr : full, w.root_mode, bj, rows, col0,
                                           w.pos2row, w.scratch, w.moved, w.mcnt, w.log2phys, st, k);
    {
      const unsigned grid = (unsigned)std::min<int64_t>(((int64_t)bj + 31) / 32, 2 * sms);
      permute_cols_kernel<<<grid, 256, 0, s>>>(w.A, w.lda, col0, lc0, lc0 + bj, w.moved, w.mcnt, nullptr, st, k);
    }
    CU_TRY(cudaGetLastError());
    if (pe > 1) {
      // unpivoted QR of the permuted panel transpose -> multiplier_block (tournament.py:271-272)
      double* blk = Ash + col0 * w.lda + col0;
      PanelArgs qa{};
      qa.src = blk;
      qa.ld = w.lda;
      qa.h = bj;
      qa.p = bj;
      qa.bsel = bj;
      qa.steps = bj;
      qa.mode = 1;
      qa.perm = w.perm_small;
      qa.Rbuf = w.Rsmall;
      qa.refl = w.refl;
      qa.ovf = w.B.ovf;
      const PanelCfg gq = panel_config(bj, bj, bj, true);
      qa.per = gq.per;
      qa.cap = gq.cap;
      qa.cap_pad = gq.cap_pad;
      qa.ovpad = gq.ovpad;
      qa.st = st;
      qa.panel_id = k;
      iota32_kernel<<<1, 128, 0, s>>>(w.perm_small, bj);
      if (reuse_root_qr()) {
        calu_root_qr_kernel<<<16, 256, 0, s>>>(w.live_all, bj, w.nodes[0].B.Rbuf, root_p, w.nodes[0].B.refl,
                                              w.Rsmall, w.refl, w.final_live, w.st);
        qa.live = w.final_live;
      }
      if (team_eligible(bj, bj) && !force_generic_panel()) {
        PanelArgs at = qa;
        at.fro = w.nodes[0].B.fro;
        launch_team(at, s);
      } else if (bj == P1_H && ((uintptr_t)blk % 16 == 0) && (w.lda % 2 == 0) && !force_generic_panel()) {
        PanelCfg g1 = gq;
        g1.C = 1;
        g1.T = P1_T;
        PanelArgs a1 = qa;
        a1.per = bj;
        a1.fro = w.nodes[0].B.fro;
        launch_cluster(panel_qrcp1_kernel, g1, 0, s, a1);
      } else if (bj == P2_H && ((uintptr_t)blk % 16 == 0) && (w.lda % 2 == 0) && !force_generic_panel()) {
        PanelCfg g2 = gq;
        g2.C = 1;
        g2.T = P2_T;
        PanelArgs a2 = qa;
        a2.per = bj;
        a2.fro = w.nodes[0].B.fro;
        launch_cluster(panel_qrcp2_kernel, g2, (size_t)(P2_H - P2_W) * P2_T * 8, s, a2);
      } else {
        launch_cluster(panel_qrcp_kernel, gq, gq.dyn_engine, s, qa);
      }
      calu_copy_r11_kernel<<<16, 256, 0, s>>>(w.Rsmall, bj, w.B.Rbuf, rows);
      static const bool calu_r12_gemm = !getenv("PRRP_CALU_R12_GEMM") || atoi(getenv("PRRP_CALU_R12_GEMM")) != 0;
      static const int r12_min_b = getenv("PRRP_CALU_R12_MIN_B") ? atoi(getenv("PRRP_CALU_R12_MIN_B")) : 65;
      const int64_t ncol = rows - bj;
      if (calu_r12_gemm && bj >= r12_min_b && (bj % 2 == 0)) {
        calu_form_negqt_kernel<<<(bj + 15) / 16, 128, (size_t)bj * (bj + 1) * 8, s>>>(w.refl, bj, w.Qneg);
        calu_gather_t_kernel<<<(unsigned)((ncol + 31) / 32), 256, (size_t)bj * 33 * 8, s>>>(
            Ash, w.lda, col0, bj, ncol, w.pos2row + col0 + bj, w.A21t, w.ld21t, w.st);
        zero2d_kernel<<<(unsigned)std::min<int64_t>(4 * sms, (ncol * bj + 255) / 256), 256, 0, s>>>(
            w.B.Rbuf + bj, rows, bj, ncol);
        schur_update(w.B.Rbuf + bj, rows, w.Qneg, bj, w.A21t, w.ld21t, bj, ncol, bj, w.st_r12, s, 0, 0);
      } else {
        const size_t dyn = (size_t)bj * (bj + 1) * 8;
        const unsigned grid = (unsigned)std::min<int64_t>(sms * 4, (rows - bj + 7) / 8);
        switch ((bj + 31) / 32) {
          case 1: calu_apply_refl_kernel<1><<<grid, 256, dyn, s>>>(Ash, w.lda, col0, bj, rows, w.pos2row, w.refl, w.B.Rbuf, st); break;
          case 2: calu_apply_refl_kernel<2><<<grid, 256, dyn, s>>>(Ash, w.lda, col0, bj, rows, w.pos2row, w.refl, w.B.Rbuf, st); break;
          case 3: calu_apply_refl_kernel<3><<<grid, 256, dyn, s>>>(Ash, w.lda, col0, bj, rows, w.pos2row, w.refl, w.B.Rbuf, st); break;
          default: calu_apply_refl_kernel<4><<<grid, 256, dyn, s>>>(Ash, w.lda, col0, bj, rows, w.pos2row, w.refl, w.B.Rbuf, st); break;
        }
      }
      CU_TRY(cudaGetLastError());
      double* fro_inf = w.nodes[0].B.fro;   // the final QR has no rank check in the reference (fro = 0)
      CU_TRY(cudaMemsetAsync(fro_inf, 0, sizeof(double), s));
      int nblk;
      if (bj <= 64 || use_trsm_c2()) {
        const int64_t cpb = bj <= 64 ? TC_COLS : 4 * TC_COLS;
        nblk = (int)std::min<int64_t>(kMaxCand, (ncol + cpb - 1) / cpb);
        if (bj <= 64)
          trsm_c_kernel<<<nblk, TC_T, 0, s>>>(w.B.Rbuf, rows, bj, w.Lg, w.ldl, w.B.cand, w.B.cand_flat, st, k,
                                              fro_inf, -1, -1, nullptr, nullptr);
        else
          trsm_c2_kernel<<<nblk, TC_T, kTrsmC2Smem, s>>>(w.B.Rbuf, rows, bj, w.Lg, w.ldl, w.B.cand, w.B.cand_flat,
                                                         st, k, fro_inf, -1, -1, nullptr, nullptr);
      } else {
        nblk = (int)std::min<int64_t>(kMaxCand, (ncol + TTC - 1) / TTC);
        const size_t tdyn = (((size_t)bj * (bj + 1) / 2 + 1) / 2 * 2 + (size_t)bj * TTCP) * 8;
        switch ((bj + 31) / 32) {
          case 3: trsm_w_kernel<3><<<nblk, TW_WARPS * 32, tdyn, s>>>(w.B.Rbuf, rows, bj, w.Lg, w.ldl, w.B.cand, w.B.cand_flat, st, k, fro_inf, -1, -1, nullptr, nullptr); break;
          default: trsm_w_kernel<4><<<nblk, TW_WARPS * 32, tdyn, s>>>(w.B.Rbuf, rows, bj, w.Lg, w.ldl, w.B.cand, w.B.cand_flat, st, k, fro_inf, -1, -1, nullptr, nullptr); break;
        }
      }
      calu_stats_kernel<<<1, 256, 0, s>>>(w.B.cand, nblk, w.node_swaps + (size_t)k * maxnodes, maxnodes,
                                          w.swaps_dev, k, st);
      CU_TRY(cudaGetLastError());
    }
    // L21 (logical order) -> physical slots, into the message (leading dimension ldl_k)
    calu_scatter_l21_kernel<<<sms * 4, 256, 0, s>>>(w.Lg, w.ldl, w.log2phys, rows - bj, bj, bj, Lp, ldk, w.st);
  } else {
    // last square block: logical order, then GEPP (every rank repeats the reorder)
    calu_reorder_kernel<<<1, 1024, 0, s>>>(nullptr, nullptr, w.ident, 1, bj, rows, col0, w.pos2row, w.scratch,
                                           w.moved, w.mcnt, w.log2phys, st, k);
    const unsigned grid = (unsigned)std::min<int64_t>(((int64_t)bj + 31) / 32, 2 * sms);
    permute_cols_kernel<<<grid, 256, 0, s>>>(w.A, w.lda, col0, lc0, lc0 + bj, w.moved, w.mcnt, nullptr, st, k);
    w.root_mode = 2;
  }
  launch_gepp(Ash + col0 * w.lda + col0, w.lda, nullptr, bj, D, w.piv, gperm, st, k, s);
  dist_state_out_kernel<<<1, 32, 0, s>>>(st, reinterpret_cast<DevState*>(w.msg));
  CU_TRY(cudaGetLastError());
}

// CTAs of the owner's look-ahead tail update (PRRP_DIST_TAIL_FREE SMs left
// for its tournament, default 8; 0 = every SM)
int dist_tail_ctas() {
  static const int free_sms = getenv("PRRP_DIST_TAIL_FREE") ? atoi(getenv("PRRP_DIST_TAIL_FREE")) : 8;
  return free_sms > 0 ? std::max(1, caps().sms - free_sms) : 0;
}

// Every rank, after the message of panel k arrived in msgs[k & 1].
// part 0: everything; 1 (head): all but the trailing update beyond the next
// panel's block; 2 (tail): that remaining update.  The owner of panel k + 1
// runs head(k), select(k + 1), tail(k), so the next tournament starts as soon
// as its own columns are up to date (look-ahead of depth one).
void calu_dist_apply(CaluDist& w, int k, int part, cudaStream_t s) {
  w.msg = w.msgs[k & 1];
  const int b = w.b;
  const int64_t m = w.m, n = w.n, col0 = (int64_t)k * b;
  const int bj = (int)std::min<int64_t>(b, n - col0);
  const int64_t rows = m - col0;
  const bool own = w.owner(k) == w.rank;
  const int64_t lc0 = w.local_col(k);
  const int sms = caps().sms;
  DevState* st = w.st;
  const double* D = reinterpret_cast<const double*>(w.msg + w.off_D);
  const int32_t* gperm = reinterpret_cast<const int32_t*>(w.msg + w.off_gperm);
  const int32_t* cnt_msg = reinterpret_cast<const int32_t*>(w.msg + w.off_cnt);
  const int32_t* piv_msg = reinterpret_cast<const int32_t*>(w.msg + w.off_piv);
  const int32_t* full = reinterpret_cast<const int32_t*>(w.msg + w.off_full);
  const double* Lp = reinterpret_cast<const double*>(w.msg + w.off_L);
  const int64_t ldk = w.ldl_k(k);
  const int pe = w.p_eff(k);
  const int64_t t0 = w.local_from((int64_t)(k + 1) * b);     // this rank's blocks after panel k
  const int64_t wt = w.n_loc - t0;
  // head / tail split of the trailing columns: the next panel's block first
  const bool next_mine = k + 1 < w.npanels && w.owner(k + 1) == w.rank;
  const int64_t wh = part == 0 ? wt : (next_mine ? std::min<int64_t>(wt, b) : 0);
  if (part != 2) {
    if (!own) {
      dist_state_in_kernel<<<1, 32, 0, s>>>(st, reinterpret_cast<const DevState*>(w.msg));
      const int mode = rows <= bj ? 2 : (pe == 1 ? 1 : 0);
      calu_reorder_kernel<<<1, 1024, 0, s>>>(mode == 0 ? piv_msg : nullptr, cnt_msg,
                                             mode == 0 ? nullptr : (mode == 1 ? full : w.ident), mode == 0 ? 0 : 1,
                                             bj, rows, col0, w.pos2row, w.scratch, w.moved, w.mcnt, w.log2phys, st, k);
    }
    // row moves of this rank's other columns (the owner moved its panel block in
    // select) and of the global row order
    auto permute = [&](int64_t c_lo, int64_t c_hi, int64_t* pp) {
      if (c_hi <= c_lo && !pp) return;
      const int64_t nc = std::max<int64_t>(c_hi - c_lo, 1);
      const unsigned grid = (unsigned)std::min<int64_t>((nc + 31) / 32, 2 * sms);
      permute_cols_kernel<<<grid, 256, 0, s>>>(w.A, w.lda, col0, c_lo, std::max(c_lo, c_hi), w.moved, w.mcnt, pp,
                                               st, k);
    };
    if (own) {
      permute(0, lc0, w.perm);
      permute(lc0 + bj, w.n_loc, nullptr);
    } else {
      permute(0, w.n_loc, w.perm);
    }
    CU_TRY(cudaGetLastError());
    // the pivot rows of this rank's trailing columns, before the finish (the update reads A12 unfinished)
    if (rows > bj && wt > 0)
      CU_TRY(cudaMemcpy2DAsync(w.a12, (size_t)w.lda12 * 8, w.A + col0 * w.lda + t0, (size_t)w.lda * 8,
                               (size_t)wt * 8, (size_t)bj, cudaMemcpyDeviceToDevice, s));
    // block-row finish over this rank's columns (global column map: block b, nranks, rank)
    launch_blockrow_w(w.A, w.lda, col0, bj, w.n_loc, D, gperm, w.perm, st, s, b, w.nranks, w.rank);
    CU_TRY(cudaGetLastError());
    if (rows > bj) {
      if (wh > 0)
        schur_update(w.A + (col0 + bj) * w.lda + t0, w.lda, Lp, ldk, w.a12, w.lda12, rows - bj, wh, bj, st, s);
      if (own)
        launch_compose_w(Lp, ldk, rows - bj, bj, D, gperm, w.A + (col0 + bj) * w.lda + lc0, w.lda, st, s, &w.cws);
    }
  }
  if (part == 2 && rows > bj && wt > wh) {
    const int64_t wh2 = next_mine ? std::min<int64_t>(wt, b) : 0;
    // the owner of panel k+1 runs its tournament concurrently (dist.py's side
    // stream): leave it a few SMs, as the single-GPU schedule's deferred update does
    if (wt > wh2) {
      // chain-bound next panel: GPC-sized clusters, one GPC left to the
      // tournament's latency-engine clusters (as caluprrp_enqueue does)
      const bool cb = next_mine && calu_chain_bound(w.m, w.n, w.b, k + 1, w.P == 0);
      tl_schur_cluster = cb ? 16 : 0;
      schur_update(w.A + (col0 + bj) * w.lda + t0 + wh2, w.lda, Lp, ldk, w.a12 + wh2, w.lda12, rows - bj, wt - wh2,
                   bj, st, s, cb ? 16 * std::max(1, caps().schur_clusters16 - 1) : dist_tail_ctas());
      tl_schur_cluster = 0;
    }
  }
  CU_TRY(cudaGetLastError());
}

// m > n: rows n..m-1 of this rank's columns into logical order
__global__ void dist_tail_gather_kernel(const double* A, int64_t lda, int64_t n, int64_t ncols, const int64_t* pos2row,
                                        int64_t m, double* tmp, const int64_t* porig, int64_t* ptmp) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (m - n) * ncols;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / ncols, c = e % ncols;
    tmp[e] = A[pos2row[n + r] * lda + c];
    if (c == 0 && ptmp) ptmp[r] = porig[pos2row[n + r]];
  }
}

int calu_dist_finish(CaluDist& w, const int64_t* reduced, int32_t* swap_counts, int64_t* tchg3, prrp_stats* stats,
                      prrp_err* err, cudaStream_t s) {
  const int64_t m = w.m, n = w.n;
  if (m > n) {
    Arena ar(s);
    const int64_t nc = std::max<int64_t>(w.n_loc, 1);
    double* tmp = ar.get<double>((size_t)(m - n) * nc);
    int64_t* ptmp = ar.get<int64_t>(m - n);
    if (w.n_loc > 0) {
      dist_tail_gather_kernel<<<caps().sms * 4, 256, 0, s>>>(w.A, w.lda, n, w.n_loc, w.pos2row, m, tmp, w.perm, ptmp);
      CU_TRY(cudaMemcpy2DAsync(w.A + n * w.lda, w.lda * 8, tmp, w.n_loc * 8, w.n_loc * 8, m - n,
                               cudaMemcpyDeviceToDevice, s));
    } else {
      dist_tail_gather_kernel<<<1, 256, 0, s>>>(w.A, w.lda, n, 1, w.pos2row, m, tmp, w.perm, ptmp);
    }
    CU_TRY(cudaMemcpyAsync(w.perm + n, ptmp, sizeof(int64_t) * (m - n), cudaMemcpyDeviceToDevice, s));
  }
  std::vector<int64_t> red(w.red_len);
  CU_TRY(cudaMemcpyAsync(red.data(), reduced, sizeof(int64_t) * w.red_len, cudaMemcpyDeviceToHost, s));
  DevState hs;
  read_state(w.st, hs, s);
  const int np = w.npanels, ns = w.npanels * w.maxnodes;
  if (swap_counts)
    for (int k = 0; k < np; ++k) swap_counts[k] = (int32_t)red[4 + k];
  if (tchg3) {
    for (int k = 0; k < np; ++k) {
      if (w.charges_tag[k] < 0) { tchg3[k] = -1; continue; }
      const int bk = (int)std::min<int64_t>(w.b, n - (int64_t)k * w.b);
      int64_t c3 = 0;
      for (auto& mm : w.node_members[k]) {
        const int64_t r = red[4 + np + ns + (size_t)k * w.maxnodes + mm.second];
        if (r > bk) c3 += (1 + red[4 + np + (size_t)k * w.maxnodes + mm.second]) * qr_charge3(r, bk);
      }
      tchg3[k] = c3;
    }
  }
  hs.orig_max = (unsigned long long)red[0];
  hs.inter_max = (unsigned long long)red[1];
  hs.finish_max = (unsigned long long)red[2];
  hs.pmm = (unsigned long long)red[3];
  fill_stats(hs, stats);
  if (stats) {
    stats->total_swaps = 0;
    for (int k = 0; k < np; ++k) stats->total_swaps += red[4 + k];
  }
  return state_to_err(hs, err);
}
