// C-ABI entry points and the stream-ordered host driver of the B200 LU_PRRP /
// CALU_PRRP library (see include/prrp_b200.h for the contract).
//
// Per panel (luprrp.py:164-199) the driver launches:
//   panel_qrcp_kernel      cluster: QRCP of the transposed panel (strong RRQR step 1)
//   trsm_kernel            all SMs: L21 = (R11^-1 R12)^T, rank check, tau candidates
//   panel_finalize_kernel  cluster: swap loop if needed, moved rows, GEPP of A11
//   permute_kernel         all SMs: move the <= 2b permuted rows
//   schur_dmma_kernel      all SMs: A22 -= L21 A12 (TMA + DMMA), growth max
//   compose_kernel         all SMs: L21 <- L21[:, perm] L11 into the L part
//   blockrow_kernel        all SMs: GEPP finish of the block row, finish max
#include <functional>
#include <chrono>
#include <memory>
#include <mutex>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <vector>
#include <algorithm>
#include <cuda.h>
#include <cuda_runtime.h>

#include "panel.cuh"
#include "lsolve.cuh"
#include "verify.cuh"
#include "panel64.cuh"
#include "panel1.cuh"
#include "panel2.cuh"
#include "panel_lat.cuh"
#include "tri64.cuh"
#include "rowops.cuh"
#include "schur.cuh"
#include "calu.cuh"
#include "calu_gepp.cuh"
#include "gepp_full.cuh"

namespace {

constexpr int kAbiVersion = 100;
constexpr size_t kSmemOptin = 227 * 1024;

struct Fail {
  int code;
  char msg[160];
};

#define CU_TRY(expr)                                                             \
  do {                                                                           \
    cudaError_t e__ = (expr);                                                    \
    if (e__ != cudaSuccess) {                                                    \
      Fail f__{PRRP_ERR_CUDA, {0}};                                              \
      snprintf(f__.msg, sizeof(f__.msg), "%s: %s (%s:%d)", #expr,                \
               cudaGetErrorString(e__), __FILE__, __LINE__);                     \
      throw f__;                                                                 \
    }                                                                            \
  } while (0)

void fail(int code, const char* msg) {
  Fail f{code, {0}};
  snprintf(f.msg, sizeof(f.msg), "%s", msg);
  throw f;
}

void clear_err(prrp_err* err) {
  if (!err) return;
  memset(err, 0, sizeof(*err));
  err->panel = err->index = err->column = err->tree_level = err->tree_index = -1;
}

int report(prrp_err* err, const Fail& f) {
  if (err) {
    err->code = f.code;
    snprintf(err->msg, sizeof(err->msg), "%s", f.msg);
  }
  return f.code;
}

__global__ void form_q_kernel(const double* refl, int h, int steps, double* Q, int neg_t = 0);

// ---------------------------------------------------------------- device probe
// claim-counter slots of the dynamically scheduled Schur kernel; a slot is
// reused kSchedSlots launches later (long after its launch has finished)
constexpr unsigned kSchedSlots = 1024;
struct DeviceCaps {
  bool init = false;
  int* sched = nullptr;        // kSchedSlots pairs of tile-claim counters (schur_ws_kernel), self-resetting
  std::atomic<unsigned> sched_next{0};
  int sms = 0;
  int max_cluster = 8;
  int schur_clusters16 = 8;    // 16-CTA clusters of the persistent trailing update the GPU holds at once (~ its GPCs)
};

// opt in to all the dynamic shared memory the kernel's static footprint leaves
void set_max_dyn(const void* fn) {
  cudaFuncAttributes fa;
  CU_TRY(cudaFuncGetAttributes(&fa, fn));
  CU_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(kSmemOptin - fa.sharedSizeBytes)));
}

// Process-wide device setup, done once under a lock (the ABI may be called
// from several host threads; one device per process, SURVEY 8(b) threading)
std::mutex g_caps_mu;
DeviceCaps& caps() {
  static DeviceCaps c;
  static std::atomic<bool> ready{false};
  if (ready.load(std::memory_order_acquire)) return c;
  std::lock_guard<std::mutex> lk(g_caps_mu);
  if (!c.init) {
    int dev = 0;
    CU_TRY(cudaGetDevice(&dev));
    CU_TRY(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev));
    for (const void* fn : {(const void*)panel_qrcp_kernel, (const void*)panel_finalize_kernel,
                           (const void*)panel_qrcp64_kernel, (const void*)panel_qrcp1_kernel,
                           (const void*)panel_qrcp2_kernel,
#define LAT_FN(NR, CPT, NWC) (const void*)panel_lat_kernel<NR, CPT, NWC, true>
#define LAT_FNS(NR) LAT_FN(NR, 1, 7), LAT_FN(NR, 2, 7), LAT_FN(NR, 4, 7), LAT_FN(NR, 1, 15), LAT_FN(NR, 2, 15)
                           LAT_FNS(4), LAT_FNS(8), LAT_FNS(16), LAT_FN(4, 4, 15), LAT_FN(8, 4, 15)
#undef LAT_FNS
#undef LAT_FN
                          }) {
      CU_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      set_max_dyn((const void*)fn);
    }
    set_max_dyn((const void*)trsm_kernel);
    set_max_dyn((const void*)form_q_kernel);
    set_max_dyn((const void*)calu_form_negqt_kernel);
    CU_TRY(cudaFuncSetAttribute(trsm_c2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTrsmC2Smem));
    set_max_dyn((const void*)permute_kernel);
    set_max_dyn((const void*)blockrow_kernel);
    set_max_dyn((const void*)blockrow_x_kernel);
    set_max_dyn((const void*)compose_kernel);
    set_max_dyn((const void*)gepp_diag_kernel);
    set_max_dyn((const void*)gepp_node_kernel<true>);
    set_max_dyn((const void*)trsm_right_kernel);
    for (const void* fn : {(const void*)trsm_w_kernel<1>, (const void*)trsm_w_kernel<2>, (const void*)trsm_w_kernel<3>,
                           (const void*)trsm_w_kernel<4>, (const void*)compose_w_kernel<1>, (const void*)compose_w_kernel<2>,
                           (const void*)compose_w_kernel<3>, (const void*)compose_w_kernel<4>,
                           (const void*)blockrow_w_kernel<1>, (const void*)blockrow_w_kernel<2>,
                           (const void*)blockrow_w_kernel<3>, (const void*)blockrow_w_kernel<4>,
                           (const void*)calu_apply_refl_kernel<1>, (const void*)calu_apply_refl_kernel<2>,
                           (const void*)calu_apply_refl_kernel<3>, (const void*)calu_apply_refl_kernel<4>})
      set_max_dyn((const void*)fn);
    CU_TRY(cudaFuncSetAttribute(schur_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SchurSmem)));
    CU_TRY(cudaFuncSetAttribute(schur_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SchurPSmem)));
    CU_TRY(cudaFuncSetAttribute(schur_persist_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CU_TRY(cudaFuncSetAttribute(schur_ws_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(SchurWSmem)));
    CU_TRY(cudaFuncSetAttribute(schur_ws_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(SchurWSmem)));
    CU_TRY(cudaFuncSetAttribute(schur_wsc_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(SchurWCSmem)));
    CU_TRY(cudaFuncSetAttribute(schur_wsc_kernel<8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CU_TRY(cudaFuncSetAttribute(schur_wsc_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(SchurWCSmem)));
    CU_TRY(cudaFuncSetAttribute(schur_wsc_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(SchurWCSmem)));
    // largest cluster the panel engine can get with a full shared-memory CTA per SM
    for (int cs : {16, 8}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(1024);
      cfg.dynamicSmemBytes = kSmemOptin - 16 * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, (void*)panel_qrcp_kernel, &cfg) == cudaSuccess && ncl > 0) {
        c.max_cluster = cs;
        break;
      }
      cudaGetLastError();
    }
    {
      // how many 16-CTA clusters of the trailing update fit at once (one per
      // GPC with >= 16 SMs): the chain-bound CALU regime launches one fewer,
      // so that a GPC stays free for the tournament's clusters
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(16 * 64);
      cfg.blockDim = dim3(SW_THREADS);
      cfg.dynamicSmemBytes = sizeof(SchurWCSmem);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 16;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (c.max_cluster >= 16 &&
          cudaOccupancyMaxActiveClusters(&ncl, (void*)schur_wsc_kernel<8>, &cfg) == cudaSuccess && ncl > 0)
        c.schur_clusters16 = ncl;
      cudaGetLastError();
    }
    // the per-call workspaces come from the stream-ordered pool: keep freed
    // blocks mapped (the default release threshold of 0 unmaps them at every
    // synchronisation, and re-mapping tens of MB inside the next call shows up
    // as a multi-millisecond hiccup)
    {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      cudaGetLastError();
    }
    CU_TRY(cudaMalloc(&c.sched, kSchedSlots * 2 * sizeof(int)));
    CU_TRY(cudaMemset(c.sched, 0, kSchedSlots * 2 * sizeof(int)));
    c.init = true;
    ready.store(true, std::memory_order_release);
  }
  return c;
}

// ---------------------------------------------------------------- tensor maps
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CU_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) fail(PRRP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// 2-D FP64 map: `inner` contiguous elements, `outer` lines `pitch` elements apart; box {8, KC}
CUtensorMap make_map(const double* base, uint64_t inner, uint64_t outer, uint64_t pitch, uint32_t box_k = SCH_KC) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch * 8};
  cuuint32_t box[2] = {8, box_k};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(PRRP_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

// ---------------------------------------------------------------- workspace
// keep != nullptr: persistent buffers (cudaMalloc, recorded in *keep and
// owned by a cached graph plan; usable while a stream is being captured)
struct Arena {
  cudaStream_t s;
  std::vector<void*> ptrs;
  std::vector<void*>* keep;
  explicit Arena(cudaStream_t st, std::vector<void*>* kp = nullptr) : s(st), keep(kp) {}
  template <typename T>
  T* get(size_t count) {
    void* p = nullptr;
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    if (keep) {
      CU_TRY(cudaMalloc(&p, bytes));
      keep->push_back(p);
    } else {
      CU_TRY(cudaMallocAsync(&p, bytes, s));
      ptrs.push_back(p);
    }
    return static_cast<T*>(p);
  }
  ~Arena() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
};

// ---------------------------------------------------------------- timing
// Optional per-kernel-class device timing: CUDA events recorded around every
// launch on the launching stream, summed after the final synchronisation.
struct Timer {
  struct Span { int cls; cudaEvent_t a, b; cudaStream_t s; };
  std::vector<Span> spans;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t ev() {
    if (used == pool.size()) {
      cudaEvent_t e;
      CU_TRY(cudaEventCreate(&e));
      pool.push_back(e);
    }
    return pool[used++];
  }
  void begin(int cls, cudaStream_t s) {
    Span sp{cls, ev(), nullptr, s};
    CU_TRY(cudaEventRecord(sp.a, s));
    spans.push_back(sp);
  }
  void end(cudaStream_t s) {
    spans.back().b = ev();
    CU_TRY(cudaEventRecord(spans.back().b, s));
  }
  void collect(prrp_timing* t) {
    memset(t->ms, 0, sizeof(t->ms));
    memset(t->launches, 0, sizeof(t->launches));
    for (const Span& sp : spans) {
      float ms = 0.f;
      CU_TRY(cudaEventElapsedTime(&ms, sp.a, sp.b));
      t->ms[sp.cls] += ms;
      t->launches[sp.cls] += 1;
    }
    if (!spans.empty()) {
      float ms = 0.f;
      CU_TRY(cudaEventElapsedTime(&ms, spans.front().a, spans.back().b));
      t->total_ms = ms;
    }
    // PRRP_TRACE=<file>: one CSV line per timed span (class, stream, start, end in ms)
    if (const char* path = getenv("PRRP_TRACE")) {
      if (FILE* f = fopen(path, "w")) {
        static const char* names[PRRP_K_COUNT] = {"panel", "trsm", "finalize", "permute", "schur",
                                                  "compose", "blockrow", "gepp", "other"};
        std::vector<cudaStream_t> ids;
        fprintf(f, "class,stream,start_ms,end_ms\n");
        for (const Span& sp : spans) {
          size_t id = std::find(ids.begin(), ids.end(), sp.s) - ids.begin();
          if (id == ids.size()) ids.push_back(sp.s);
          float a = 0.f, b = 0.f;
          CU_TRY(cudaEventElapsedTime(&a, spans.front().a, sp.a));
          CU_TRY(cudaEventElapsedTime(&b, spans.front().a, sp.b));
          fprintf(f, "%s,%zu,%.4f,%.4f\n", names[sp.cls], id, a, b);
        }
        fclose(f);
      }
    }
  }
  ~Timer() {
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  }
};
thread_local Timer* tl_timer = nullptr;
thread_local double tl_schur_flops = 0.0;
inline void tbegin(int cls, cudaStream_t s) { if (tl_timer) tl_timer->begin(cls, s); }
inline void tend(cudaStream_t s) { if (tl_timer) tl_timer->end(s); }

// ---------------------------------------------------------------- launches
struct PanelCfg {
  int C, T;
  int64_t per;
  int cap, cap_pad;
  int64_t ovpad;
  size_t dyn_engine, dyn_final;
};

// generic-engine configuration; few_ctas: the smallest cluster that fits
// (used by the finalize / swap-loop kernel, which is rarely busy)
PanelCfg panel_config(int h, int64_t p, int bsel, bool few_ctas = false) {
  PanelCfg g{};
  const int maxc = caps().max_cluster;
  g.C = (int)std::min<int64_t>(maxc, std::max<int64_t>(1, (p + 127) / 128));
  if (few_ctas) g.C = (int)std::min<int64_t>(maxc, std::max<int64_t>(1, (p + PRRP_MAXCPT * 1024 - 1) / (PRRP_MAXCPT * 1024)));
  g.per = (p + g.C - 1) / g.C;
  if (g.per > (int64_t)PRRP_MAXCPT * 1024) fail(PRRP_ERR_UNSUPPORTED, "panel too tall for the cluster engine");
  g.T = (int)std::min<int64_t>(1024, std::max<int64_t>(32, ((std::min<int64_t>(g.per, 1024) + 31) / 32) * 32));
  while ((int64_t)g.T * PRRP_MAXCPT < g.per) g.T += 32;
  const size_t budget = kSmemOptin - 16 * 1024 - sizeof(PanelShared);
  int64_t maxcols = (int64_t)(budget / ((size_t)h * 8));
  if (maxcols % 2 == 0) --maxcols;
  g.cap = (int)std::min<int64_t>(g.per, maxcols);
  g.cap_pad = g.cap | 1;
  g.ovpad = std::max<int64_t>(0, g.per - g.cap);
  g.dyn_engine = (size_t)g.cap_pad * h * 8;
  const int tw = bsel > 64 ? 64 : 128;
  const size_t trsm_need = ((size_t)bsel * (bsel + 1) / 2 + (size_t)bsel * tw) * 8;
  const size_t gepp_need = (size_t)h * h * 8;
  g.dyn_final = std::max({g.dyn_engine, trsm_need, gepp_need});
  return g;
}

// overflow scratch large enough for both the panel engine and the finalize config
size_t ovf_elems(int h, int64_t p, int bsel) {
  const PanelCfg a = panel_config(h, p, bsel), b = panel_config(h, p, bsel, true);
  // (h x p: the row-save area of the h = 64 register engine, panel1.cuh)
  return std::max({(size_t)a.C * h * std::max<int64_t>(1, a.ovpad), (size_t)b.C * h * std::max<int64_t>(1, b.ovpad),
                   (size_t)h * p});
}

// `groups` clusters of g.C CTAs each (groups > 1: the multi-cluster panel engine)
template <typename K, typename... Args>
void launch_clusters(K kernel, const PanelCfg& g, int groups, size_t dyn, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.C * groups);
  cfg.blockDim = dim3(g.T);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = g.C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CU_TRY(cudaLaunchKernelEx(&cfg, kernel, args...));
}

template <typename K, typename... Args>
void launch_cluster(K kernel, const PanelCfg& g, size_t dyn, cudaStream_t s, Args... args) {
  launch_clusters(kernel, g, 1, dyn, s, args...);
}

// The latency engine (panel_lat.cuh): a team of 8 threads per column, CPT
// columns per team, NWC compute warps (4 NWC teams) + one control warp per
// CTA, ceil(p / (4 NWC CPT)) CTAs in one cluster.
// PRRP_LAT=0 disables it (the thread-per-column engines run instead);
// PRRP_LAT_MAXP caps the panel height it takes; PRRP_LAT_NWC / PRRP_LAT_CPT
// force a shape (A/B measurements, tools/lat_sweep.py).
int lat_nr(int h) { return h <= 32 ? 4 : h <= 64 ? 8 : 16; }
bool lat_has(int nr, int nwc, int cpt) {
  if (nwc == 7) return cpt == 1 || cpt == 2 || cpt == 4;
  if (nwc == 15) return cpt == 1 || cpt == 2 || (cpt == 4 && nr <= 8);
  return false;
}
int64_t lat_max_p() {
  static const int64_t v = getenv("PRRP_LAT_MAXP") ? atoll(getenv("PRRP_LAT_MAXP")) : (int64_t)1 << 40;
  static const bool on = !(getenv("PRRP_LAT") && atoi(getenv("PRRP_LAT")) == 0);
  return on ? v : 0;
}
struct LatShape { int nwc = 0, cpt = 0, C = 0; };
int lat_ctas(int64_t p, int nwc, int cpt) { return (int)std::max<int64_t>(1, (p + 4 * nwc * cpt - 1) / (4 * nwc * cpt)); }
// Largest cluster the latency engine may use in the calls of this thread
// (0: engine off).  A cluster needs that many free SMs in ONE GPC, which a
// persistent trailing update beside it does not leave, so the CALU schedule
// sets it per panel (see caluprrp_enqueue); PRRP_LAT_CMAX sets the default.
int lat_default_cmax() {
  static const int v = getenv("PRRP_LAT_CMAX") ? atoi(getenv("PRRP_LAT_CMAX")) : 16;
  return v;
}
thread_local int tl_lat_cmax = -1;   // -1: the default
// shape for an h x p panel (nwc = 0: not eligible); force_* > 0 pin a choice.
// Preference = measured order (tools/lat_sweep.py): few warps
// per scheduler and one column per team first.
LatShape lat_shape(int h, int64_t p, int force_nwc = 0, int force_cpt = 0, int cmax = -1) {
  static const int env_nwc = getenv("PRRP_LAT_NWC") ? atoi(getenv("PRRP_LAT_NWC")) : 0;
  static const int env_cpt = getenv("PRRP_LAT_CPT") ? atoi(getenv("PRRP_LAT_CPT")) : 0;
  if (!force_nwc) force_nwc = env_nwc;
  if (!force_cpt) force_cpt = env_cpt;
  if (cmax < 0) cmax = tl_lat_cmax >= 0 ? tl_lat_cmax : lat_default_cmax();
  const int nr = lat_nr(h);
  const int maxc = std::min(caps().max_cluster, cmax);
  LatShape best;
  // whole 8-row blocks only (h = 32, 64, 128: every tournament node and panel
  // of the BASELINE configs); other widths run the generic engine
  if (h != 8 * nr) return best;
  static const int pref[5][2] = {{7, 1}, {15, 1}, {7, 2}, {15, 2}, {7, 4}};
  for (const auto& pc : pref) {
    const int nwc = pc[0], cpt = pc[1];
    if (force_nwc && nwc != force_nwc) continue;
    if (force_cpt && cpt != force_cpt) continue;
    if (!lat_has(nr, nwc, cpt)) continue;
    const int C = lat_ctas(p, nwc, cpt);
    if (C > maxc) continue;
    return LatShape{nwc, cpt, C};
  }
  return best;
}

// The CALU final QR reuses the tournament root's QRCP (calu_root_qr_kernel);
// PRRP_ROOT_QR=0 runs the separate QR of A11^T every panel instead.
bool reuse_root_qr() {
  static const bool v = !(getenv("PRRP_ROOT_QR") && atoi(getenv("PRRP_ROOT_QR")) == 0);
  return v;
}

bool team_eligible(int h, int64_t p) {
  if (!(h >= 1 && h <= PRRP_MAXH && p >= 1 && p <= lat_max_p())) return false;
  return lat_shape(h, p).nwc != 0;
}

template <int NR, int CPT, int NWC>
void launch_lat_as(const PanelArgs& a, PanelCfg g, cudaStream_t s) {
  const size_t dyn = lat_smem<NR, NWC>();
  g.T = 32 * (NWC + 1);
  launch_cluster(panel_lat_kernel<NR, CPT, NWC, true>, g, dyn, s, a);   // h == 8 NR (lat_shape)
}

template <int NR>
void launch_lat_nr(const PanelArgs& a, const PanelCfg& g, const LatShape& sh, cudaStream_t s) {
  if (sh.nwc == 7) {
    if (sh.cpt == 1) launch_lat_as<NR, 1, 7>(a, g, s);
    else if (sh.cpt == 2) launch_lat_as<NR, 2, 7>(a, g, s);
    else launch_lat_as<NR, 4, 7>(a, g, s);
  } else {
    if (sh.cpt == 1) launch_lat_as<NR, 1, 15>(a, g, s);
    else if (sh.cpt == 2) launch_lat_as<NR, 2, 15>(a, g, s);
    else if constexpr (NR <= 8) launch_lat_as<NR, 4, 15>(a, g, s);
  }
}

void launch_team(const PanelArgs& a0, cudaStream_t s, int force_nwc = 0, int force_cpt = 0, int cmax = -1) {
  const LatShape sh = lat_shape(a0.h, a0.p, force_nwc, force_cpt, cmax);
  if (!sh.nwc) fail(PRRP_ERR_UNSUPPORTED, "no latency-engine shape for this panel");
  PanelCfg g{};
  g.C = sh.C;
  PanelArgs a = a0;
  a.per = (a.p + sh.C - 1) / sh.C;
  const int nr = lat_nr(a.h);
  if (nr == 4) launch_lat_nr<4>(a, g, sh, s);
  else if (nr == 8) launch_lat_nr<8>(a, g, sh, s);
  else launch_lat_nr<16>(a, g, sh, s);
}

// GEPP of a b x b block (register kernel for b <= 64, shared-memory kernel above)
void launch_gepp(const double* src, int64_t ld, const int32_t* rowmap, int b, double* D, int32_t* piv,
                 int32_t* gperm, DevState* st, int panel, cudaStream_t s) {
  // b <= 64: 256 threads.  The same kernel with 1024 threads for b <= 128 (PRRP_GEPP_REG128=1) was
  // measured SLOWER than the shared-memory kernel (LU_PRRP b = 128: gepp spans 28.2 vs 23.8 ms), so off.
  static const bool reg128 = getenv("PRRP_GEPP_REG128") && atoi(getenv("PRRP_GEPP_REG128")) != 0;
  if (b <= 64) gepp_reg_kernel<64><<<1, GR_T, 0, s>>>(src, ld, rowmap, b, D, piv, gperm, st, panel);
  else if (b <= 128 && reg128) gepp_reg_kernel<128><<<1, 1024, 0, s>>>(src, ld, rowmap, b, D, piv, gperm, st, panel);
  else {
    // 128 column threads x T / 128 row groups (PRRP_GEPP_DIAG_T: 128 = one thread per column as in round 1)
    static const int gt = getenv("PRRP_GEPP_DIAG_T") ? atoi(getenv("PRRP_GEPP_DIAG_T")) : 512;
    gepp_diag_kernel<<<1, std::max(128, std::min(1024, gt / 128 * 128)), (size_t)b * (b + 1) * 8, s>>>(
        src, ld, rowmap, b, D, piv, gperm, st, panel);
  }
}

// b in (64, 128]: 8-lane chunked trsm (trsm_c2_kernel); PRRP_TRSM_W=1 selects
// the warp-per-column kernel instead
bool use_trsm_c2() {
  static const bool v = !(getenv("PRRP_TRSM_W") && atoi(getenv("PRRP_TRSM_W")) != 0);
  return v;
}

// PRRP_GENERIC_PANEL=1 forces the generic shared-memory engine (A/B testing)
bool force_generic_panel() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PRRP_GENERIC_PANEL");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// PRRP_PANEL_PROF=1: CTA 0 of the fast panel engine accumulates per-phase
// clock64 totals; printed to stderr at the end of prrp_luprrp.
thread_local long long* tl_prof = nullptr;
bool panel_prof_enabled() {
  const char* e = getenv("PRRP_PANEL_PROF");
  return e && e[0] == '1';
}

int swap_cap(int b, int64_t p, double tau) {   // pivoted_qr.py:108-110
  return (int)std::ceil(2.0 * b * std::log((double)std::max<int64_t>(p, 2)) / std::log(tau)) + 10;
}

struct PanelBuffers {
  double* fro = nullptr;    // per-node ||panel||_F slot (nullptr: DevState::fro)
  double* Rbuf;
  int32_t* perm;
  double* ovf;
  double* cand;
  long long* cand_flat;
  int32_t* moved;
  double* refl;
  int32_t* moved_cnt = nullptr;
  double* xg = nullptr;                   // multi-cluster panel exchange slots (panel2.cuh)
  unsigned long long* xflag = nullptr;
  // CALU tournament nodes (see PanelArgs::live / want / node_rows)
  const int32_t* live = nullptr;
  int32_t* want = nullptr;
  int32_t* node_rows = nullptr;
};

constexpr int kP2MaxGroups = 4;
std::atomic<unsigned long long> g_xepoch{0};   // per-launch flag epoch of the multi-cluster engine
void alloc_exchange(Arena& ar, cudaStream_t s, PanelBuffers& B) {
  B.xg = ar.get<double>((size_t)2 * kP2MaxGroups * P2_XS);
  B.xflag = ar.get<unsigned long long>(kP2MaxGroups);
  CU_TRY(cudaMemsetAsync(B.xflag, 0, sizeof(unsigned long long) * kP2MaxGroups, s));
}

constexpr int kMaxCand = 2048;   // trsm blocks per panel (candidate slots)

void launch_finalize(const PanelArgs& a, const PanelBuffers& B, int bsel, int64_t p, int h, double tau, int ncand,
                     double* D, int32_t* piv, int32_t* gperm, int32_t* swaps_dev, bool do_gepp, DevState* st,
                     int panel, cudaStream_t s);

// One strong RRQR of the h x p transposed panel: QRCP (cluster), multipliers
// (all SMs), swap loop + moved rows (+ optional GEPP of the pivot block).
void strong_rrqr_panel(const double* src, int64_t ld, int h, int64_t p, int bsel, double tau, int panel,
                       double* L21, int64_t ldl, const PanelBuffers& B, DevState* st, int32_t* swaps_dev,
                       double* D, int32_t* piv, int32_t* gperm, bool do_gepp, cudaStream_t s,
                       const int64_t* rowidx = nullptr, int swap_slot = -1, int tl = -1, int ti = -1,
                       cudaEvent_t after_qrcp = nullptr) {
  const PanelCfg g = panel_config(h, p, bsel);
  PanelArgs a{};
  a.src = src;
  a.ld = ld;
  a.rowidx = rowidx;
  a.swap_slot = swap_slot < 0 ? panel : swap_slot;
  a.tree_level = tl;
  a.tree_index = ti;
  a.fro = B.fro ? B.fro : &st->fro;
  a.h = h;
  a.p = p;
  a.bsel = bsel;
  a.steps = (int)std::min<int64_t>(h, p);
  a.mode = 0;
  a.perm = B.perm;
  a.Rbuf = B.Rbuf;
  a.refl = B.refl;
  a.ovf = B.ovf;
  a.per = g.per;
  a.cap = g.cap;
  a.cap_pad = g.cap_pad;
  a.ovpad = g.ovpad;
  a.st = st;
  a.panel_id = panel;
  a.tau = tau;
  a.L21 = L21;
  a.ldl = ldl;
  a.moved = B.moved;
  a.moved_cnt = B.moved_cnt;
  a.prof = tl_prof;
  static const int fused_ak = getenv("PRRP_P2_FUSED") ? atoi(getenv("PRRP_P2_FUSED")) : 1;
  a.fused_ak = fused_ak;
  a.live = B.live;
  a.want = B.want;
  a.node_rows = B.node_rows;
  tbegin(PRRP_K_PANEL, s);
  const int maxc = caps().max_cluster;
  // CTAs: enough for the columns (one per thread in registers, a second in
  // shared memory above 4096), at least ceil(p / cpc) -- PRRP_P1_COLS
  // (default 256) columns per CTA before the cluster grows
  static const int64_t cpc = getenv("PRRP_P1_COLS") ? atoll(getenv("PRRP_P1_COLS")) : 256;
  const int64_t c1 = std::max<int64_t>((p + P1_MAXCOLS - 1) / P1_MAXCOLS,
                                       std::min<int64_t>(maxc, std::max<int64_t>(1, (p + cpc - 1) / cpc)));
  const bool aligned = ((uintptr_t)src % 16 == 0) && (ld % 2 == 0);
  if (team_eligible(h, p) && !force_generic_panel()) {
    launch_team(a, s);
  } else if (h == P1_H && c1 <= maxc && aligned && !force_generic_panel()) {
    // thread-per-column register engine (h = 64)
    PanelCfg g1 = g;
    g1.C = (int)c1;
    g1.T = P1_T;
    PanelArgs a1 = a;
    a1.per = (p + c1 - 1) / c1;
    const size_t dyn = a1.per > P1_T ? (size_t)P1_H * P1_T * 8 : 0;
    launch_cluster(panel_qrcp1_kernel, g1, dyn, s, a1);
  } else if (h == P2_H && p > (int64_t)P2_T * maxc && p <= (int64_t)P2_T * maxc * kP2MaxGroups && maxc == 16 &&
             aligned && B.xg && !force_generic_panel() && !getenv("PRRP_P2_NOGROUPS")) {
    // taller than one cluster: co-resident clusters exchanging winners through L2
    PanelCfg g2 = g;
    g2.C = maxc;
    g2.T = P2_T;
    const int groups = (int)((p + (int64_t)P2_T * maxc - 1) / ((int64_t)P2_T * maxc));
    PanelArgs a2 = a;
    a2.per = (p + (int64_t)groups * maxc - 1) / ((int64_t)groups * maxc);
    a2.ngroups = groups;
    a2.xg = B.xg;
    a2.xflag = B.xflag;
    a2.epoch = g_xepoch.fetch_add(1024) + 1024;
    launch_clusters(panel_qrcp2_kernel, g2, groups, (size_t)(P2_H - P2_W) * P2_T * 8, s, a2);
  } else if (h == P2_H && p <= (int64_t)P2_T * maxc && aligned && !force_generic_panel()) {
    // thread-per-column split-column engine (h = 128): register window + shared rows
    PanelCfg g2 = g;
    static const int64_t cpc2 = getenv("PRRP_P2_COLS") ? atoll(getenv("PRRP_P2_COLS")) : 256;
    g2.C = (int)std::max<int64_t>((p + P2_T - 1) / P2_T, std::min<int64_t>(maxc, (p + cpc2 - 1) / cpc2));
    g2.T = P2_T;
    PanelArgs a2 = a;
    a2.per = (p + g2.C - 1) / g2.C;
    launch_cluster(panel_qrcp2_kernel, g2, (size_t)(P2_H - P2_W) * P2_T * 8, s, a2);
  } else {
    launch_cluster(panel_qrcp_kernel, g, g.dyn_engine, s, a);
  }
  tend(s);
  CU_TRY(cudaGetLastError());

  if (after_qrcp) CU_TRY(cudaEventRecord(after_qrcp, s));
  const int64_t ncol = p - bsel;
  const int nblk = ncol > 0 ? (int)std::min<int64_t>(kMaxCand, (ncol + TTC - 1) / TTC) : 0;
  if (nblk > 0) {
    tbegin(PRRP_K_TRSM, s);
    const size_t dyn = (((size_t)bsel * (bsel + 1) / 2 + 1) / 2 * 2 + (size_t)bsel * TTCP) * 8;
    if (force_generic_panel()) {
      const int tw = 128;
      const int nb = (int)((ncol + tw - 1) / tw);
      // generic path keeps one candidate per 128 positions: at most kMaxCand blocks
      if (nb > kMaxCand) fail(PRRP_ERR_UNSUPPORTED, "generic trsm path limited to 131072 rows");
      trsm_kernel<<<nb, tw, ((size_t)bsel * (bsel + 1) / 2 + (size_t)bsel * tw) * 8, s>>>(B.Rbuf, p, bsel, L21, ldl, B.cand, B.cand_flat, st, panel, a.fro, tl, ti, B.live, B.want);
      tend(s);
      CU_TRY(cudaGetLastError());
      launch_finalize(a, B, bsel, p, h, tau, nb, D, piv, gperm, swaps_dev, do_gepp, st, panel, s);
      return;
    }
    if (bsel <= 64 || use_trsm_c2()) {
      // b > 64: a CTA stages the 133 KB R11 before it solves anything, and the
      // eight leaves of a tournament level launch their solves together (992
      // CTAs at 4096-row leaves).  PRRP_TRSM_GROUPS = g gives a CTA g column
      // groups on tall panels; measured no different at config 5 (1293-1299
      // ms for g = 1, 2, 4, 8), so 1.
      static const int tg = getenv("PRRP_TRSM_GROUPS") ? atoi(getenv("PRRP_TRSM_GROUPS")) : 1;
      const int64_t cpb = (bsel > 64 && ncol >= 1024) ? (int64_t)std::max(1, tg) * TC_COLS : TC_COLS;
      const int nbv = (int)std::min<int64_t>(kMaxCand, (ncol + cpb - 1) / cpb);
      if (bsel <= 64)
        trsm_c_kernel<<<nbv, TC_T, 0, s>>>(B.Rbuf, p, bsel, L21, ldl, B.cand, B.cand_flat, st, panel, a.fro, tl, ti,
                                           B.live, B.want);
      else
        trsm_c2_kernel<<<nbv, TC_T, kTrsmC2Smem, s>>>(B.Rbuf, p, bsel, L21, ldl, B.cand, B.cand_flat, st, panel, a.fro,
                                                       tl, ti, B.live, B.want);
      tend(s);
      CU_TRY(cudaGetLastError());
      launch_finalize(a, B, bsel, p, h, tau, nbv, D, piv, gperm, swaps_dev, do_gepp, st, panel, s);
      return;
    }
    switch ((bsel + 31) / 32) {
      case 1: trsm_w_kernel<1><<<nblk, TW_WARPS * 32, dyn, s>>>(B.Rbuf, p, bsel, L21, ldl, B.cand, B.cand_flat, st, panel, a.fro, tl, ti, B.live, B.want); break;
      case 2: trsm_w_kernel<2><<<nblk, TW_WARPS * 32, dyn, s>>>(B.Rbuf, p, bsel, L21, ldl, B.cand, B.cand_flat, st, panel, a.fro, tl, ti, B.live, B.want); break;
      case 3: trsm_w_kernel<3><<<nblk, TW_WARPS * 32, dyn, s>>>(B.Rbuf, p, bsel, L21, ldl, B.cand, B.cand_flat, st, panel, a.fro, tl, ti, B.live, B.want); break;
      default: trsm_w_kernel<4><<<nblk, TW_WARPS * 32, dyn, s>>>(B.Rbuf, p, bsel, L21, ldl, B.cand, B.cand_flat, st, panel, a.fro, tl, ti, B.live, B.want); break;
    }
    tend(s);
    CU_TRY(cudaGetLastError());
  }
  launch_finalize(a, B, bsel, p, h, tau, nblk, D, piv, gperm, swaps_dev, do_gepp, st, panel, s);
}

void launch_finalize(const PanelArgs& a, const PanelBuffers& B, int bsel, int64_t p, int h, double tau, int ncand,
                     double* D, int32_t* piv, int32_t* gperm, int32_t* swaps_dev, bool do_gepp, DevState* st,
                     int panel, cudaStream_t s) {
  FinalizeArgs f{};
  f.pa = a;
  f.pa.cand = B.cand;
  f.pa.cand_flat = B.cand_flat;
  f.pa.ncand = ncand;
  f.swap_cap = swap_cap(bsel, p, tau);
  f.D = D;
  f.piv = piv;
  f.gperm = gperm;
  f.swaps_dev = swaps_dev;
  f.do_gepp = 0;   // the diagonal-block GEPP runs as its own small kernel below
  tbegin(PRRP_K_FINALIZE, s);
  const PanelCfg gf = panel_config(h, p, bsel, true);
  f.pa.per = gf.per;
  f.pa.cap = gf.cap;
  f.pa.cap_pad = gf.cap_pad;
  f.pa.ovpad = gf.ovpad;
  launch_cluster(panel_finalize_kernel, gf, gf.dyn_final, s, f);
  tend(s);
  CU_TRY(cudaGetLastError());
  if (do_gepp) {
    tbegin(PRRP_K_GEPP, s);
    launch_gepp(a.src, a.ld, B.perm, h, D, piv, gperm, st, panel, s);
    tend(s);
    CU_TRY(cudaGetLastError());
  }
}

thread_local int tl_force_ws = -1;   // diagnostics: per-call kernel choice (PRRP_WS_W1 / PRRP_WS_W2)
// > 0: the persistent K > 64 trailing update is launched as clusters of this
// many CTAs (the kernel itself does not use cluster features).  A cluster is
// placed inside one GPC, so with one cluster fewer than the GPU has GPCs a
// whole GPC stays free for the tournament's own clusters beside the update
// (caluprrp_enqueue, chain-bound panels).
thread_local int tl_schur_cluster = 0;
thread_local bool tl_schur_untracked = false;   // schur_update called as a building block (compose): no span, no flops
// CALU_PRRP enqueue: the warp-specialised kernel prefetches C (see DESIGN.md 4:
// with the C read in the epilogue the graph-replayed CALU schedule gave
// run-to-run different results; with the prefetch it is bit-stable)
thread_local bool tl_schur_prefetch_c = false;
// claim counters of a graph plan being captured (its launches own their slots)
thread_local int* tl_sched = nullptr;
thread_local unsigned tl_sched_next = 0, tl_sched_slots = 1;

// PRRP_SCHUR_W2_STREAM=1: the bulk trailing update (W2) streams C with evict-first hints
const bool w2_stream = getenv("PRRP_SCHUR_W2_STREAM") && atoi(getenv("PRRP_SCHUR_W2_STREAM")) != 0;

// max_ctas > 0 selects the persistent kernel with at most that many CTAs
// (K <= 64); 0 the classic one-tile-per-CTA kernel, whose short CTAs let a
// concurrent high-priority stream claim SMs quickly
void schur_update(double* C, int64_t ldc, const double* L, int64_t ldl, const double* Bm, int64_t ldb, int64_t M,
                  int64_t N, int K, DevState* st, cudaStream_t s, int max_ctas = 0, int quantum = 0,
                  bool stream_c = false) {
  if (M <= 0 || N <= 0) return;
  const bool tracked = !tl_schur_untracked;      // (the compose product is timed as "compose", not as a Schur update)
  if (tracked) {
    tl_schur_flops += 2.0 * (double)M * (double)N * (double)K;
    tbegin(PRRP_K_SCHUR, s);
  }
  const bool tma_ok = ((uintptr_t)L % 16 == 0) && ((uintptr_t)Bm % 16 == 0) && (ldl % 2 == 0) && (ldb % 2 == 0) &&
                      K <= 4 * SCH_KC && M < (1ll << 31) && N < (1ll << 31);
  static const int schur_old = getenv("PRRP_SCHUR_OLD") ? atoi(getenv("PRRP_SCHUR_OLD")) : 0;
  // K <= 64 with a CTA budget: the whole-K-stage persistent kernel (measured
  // steadier than the warp-specialised one inside the b = 64 LU_PRRP
  // schedule); K > 64 (b = 128): the warp-specialised kernel (70-74% of the
  // DMMA peak on the big updates vs 58-63% for the classic kernel)
  static const bool ws64 = getenv("PRRP_SCHUR_WS64") && atoi(getenv("PRRP_SCHUR_WS64")) != 0;   // diagnostics
  bool use_ws = !schur_old && (max_ctas > 0 || quantum > 0) && (K > SP_K || quantum > 0 || ws64);
  if (tl_force_ws >= 0 && (max_ctas > 0 || quantum > 0)) use_ws = tl_force_ws == 1;   // diagnostics
  if (tma_ok && use_ws) {
    const CUtensorMap mapL = make_map(L, (uint64_t)M, (uint64_t)K, (uint64_t)ldl, SW_KC);
    const CUtensorMap mapB = make_map(Bm, (uint64_t)N, (uint64_t)K, (uint64_t)ldb, SW_KC);
    const int vec_ok = ((uintptr_t)C % 16 == 0) && (ldc % 2 == 0);
    const int64_t tiles = ((M + SCH_BM - 1) / SCH_BM) * ((N + SCH_BN - 1) / SCH_BN);
    const unsigned grid = (unsigned)(quantum > 0 ? (tiles + quantum - 1) / quantum : std::min<int64_t>(tiles, max_ctas));
    // static tile assignment by default (measured as fast: 1437.6 vs 1437.9 ms
    // at n = 32768, and it keeps no state across launches); PRRP_SCHUR_DYNAMIC=1
    // claims tiles from a self-resetting global counter instead
    static const bool static_claims = !(getenv("PRRP_SCHUR_DYNAMIC") && atoi(getenv("PRRP_SCHUR_DYNAMIC")) != 0);
    int* ctr = static_claims ? nullptr
               : tl_sched ? tl_sched + 2 * (tl_sched_next++ % tl_sched_slots)
                          : caps().sched + 2 * (caps().sched_next.fetch_add(1) % kSchedSlots);
    // C read in the epilogue (default): the MMA loop then has the registers to
    // keep two k-steps of fragments in flight (83% vs 74% of the DMMA peak at
    // 32640^2 x 128); PRRP_SCHUR_LATE_C=0 prefetches C into registers instead
    static const bool late_c = !getenv("PRRP_SCHUR_LATE_C") || atoi(getenv("PRRP_SCHUR_LATE_C")) != 0;
    // PRRP_SCHUR_WSC=1: C staged through shared memory by TMA (the default until the ring's
    // release hazard was fixed, DESIGN 4 "Determinism"; the epilogue read is 1.7% faster on config 5)
    static const bool wsc = getenv("PRRP_SCHUR_WSC") && atoi(getenv("PRRP_SCHUR_WSC")) != 0;
    static const int ws_exp = getenv("PRRP_WS_EXP") ? (atoi(getenv("PRRP_WS_EXP")) & 16) : 0;   // diagnostics
    if (wsc && vec_ok && static_claims && quantum <= 0) {
      // C staged through shared memory by TMA (read early, registers free)
      const CUtensorMap mapC = make_map(C, (uint64_t)N, (uint64_t)M, (uint64_t)ldc, SCH_BM);
      static const int wsc_warps = getenv("PRRP_SCHUR_WSC_WARPS") ? atoi(getenv("PRRP_SCHUR_WSC_WARPS")) : 8;
      if (wsc_warps == 4)
        schur_wsc_kernel<4><<<grid, 5 * 32, sizeof(SchurWCSmem), s>>>(mapL, mapB, mapC, C, ldc, (int)M, (int)N, K, st);
      else if (wsc_warps == 16)
        schur_wsc_kernel<16><<<grid, 17 * 32, sizeof(SchurWCSmem), s>>>(mapL, mapB, mapC, C, ldc, (int)M, (int)N, K,
                                                                         st);
      else if (tl_schur_cluster > 1 && (int)grid >= tl_schur_cluster) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((grid / (unsigned)tl_schur_cluster) * (unsigned)tl_schur_cluster);
        cfg.blockDim = dim3(SW_THREADS);
        cfg.dynamicSmemBytes = sizeof(SchurWCSmem);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)tl_schur_cluster;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CU_TRY(cudaLaunchKernelEx(&cfg, schur_wsc_kernel<8>, mapL, mapB, mapC, C, ldc, (int)M, (int)N, K, st));
      } else
        schur_wsc_kernel<8><<<grid, SW_THREADS, sizeof(SchurWCSmem), s>>>(mapL, mapB, mapC, C, ldc, (int)M, (int)N, K,
                                                                          st);
    } else if (late_c && !tl_schur_prefetch_c)
      schur_ws_kernel<false><<<grid, SW_THREADS, sizeof(SchurWSmem), s>>>(mapL, mapB, C, ldc, (int)M, (int)N, K,
                                                                           vec_ok, st, ctr,
                                                                           quantum > 0 ? quantum : INT_MAX,
                                                                           (stream_c ? 1 : 0) | ws_exp);
    else
    schur_ws_kernel<true><<<grid, SW_THREADS, sizeof(SchurWSmem), s>>>(mapL, mapB, C, ldc, (int)M, (int)N, K, vec_ok, st,
                                                                 ctr, quantum > 0 ? quantum : INT_MAX,
                                                                 stream_c ? 1 : 0);
  } else if (tma_ok && max_ctas > 0 && K <= SP_K) {
    const CUtensorMap mapL = make_map(L, (uint64_t)M, (uint64_t)K, (uint64_t)ldl, SP_K);
    const CUtensorMap mapB = make_map(Bm, (uint64_t)N, (uint64_t)K, (uint64_t)ldb, SP_K);
    const int vec_ok = ((uintptr_t)C % 16 == 0) && (ldc % 2 == 0);
    const int64_t tiles = ((M + SCH_BM - 1) / SCH_BM) * ((N + SCH_BN - 1) / SCH_BN);
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, max_ctas);
    if (tl_schur_cluster > 1 && (int)grid >= tl_schur_cluster) {   // GPC-sized clusters (see tl_schur_cluster)
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((grid / (unsigned)tl_schur_cluster) * (unsigned)tl_schur_cluster);
      cfg.blockDim = dim3(SCH_THREADS);
      cfg.dynamicSmemBytes = sizeof(SchurPSmem);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)tl_schur_cluster;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CU_TRY(cudaLaunchKernelEx(&cfg, schur_persist_kernel, mapL, mapB, C, ldc, (int)M, (int)N, K, vec_ok, st));
    } else
    schur_persist_kernel<<<grid, SCH_THREADS, sizeof(SchurPSmem), s>>>(mapL, mapB, C, ldc, (int)M, (int)N, K, vec_ok,
                                                                        st);
  } else if (tma_ok) {
    const CUtensorMap mapL = make_map(L, (uint64_t)M, (uint64_t)K, (uint64_t)ldl);
    const CUtensorMap mapB = make_map(Bm, (uint64_t)N, (uint64_t)K, (uint64_t)ldb);
    const int vec_ok = ((uintptr_t)C % 16 == 0) && (ldc % 2 == 0);
    dim3 grid((unsigned)((N + SCH_BN - 1) / SCH_BN), (unsigned)((M + SCH_BM - 1) / SCH_BM));
    schur_dmma_kernel<<<grid, SCH_THREADS, sizeof(SchurSmem), s>>>(mapL, mapB, C, ldc, (int)M, (int)N, K, vec_ok, st);
  } else {
    dim3 grid((unsigned)((N + 31) / 32), (unsigned)((M + 7) / 8));
    schur_simt_kernel<<<grid, 256, 0, s>>>(L, ldl, Bm, ldb, C, ldc, (int)M, (int)N, K, st);
  }
  if (tracked) tend(s);
  CU_TRY(cudaGetLastError());
}

void read_state(DevState* st_dev, DevState& hs, cudaStream_t s) {
  CU_TRY(cudaMemcpyAsync(&hs, st_dev, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  CU_TRY(cudaStreamSynchronize(s));
}

int state_to_err(const DevState& hs, prrp_err* err) {
  if (hs.code == 0) return PRRP_OK;
  if (err) {
    err->code = hs.code;
    err->panel = hs.panel;
    err->index = hs.index;
    err->column = hs.column;
    err->tree_level = hs.tree_level;
    err->tree_index = hs.tree_index;
    err->worst = hs.worst;
    snprintf(err->msg, sizeof(err->msg), "device error %d", hs.code);
  }
  return hs.code;
}

double bits_to_double(unsigned long long b) {
  double d;
  memcpy(&d, &b, 8);
  return d;
}

void fill_stats(const DevState& hs, prrp_stats* stats) {
  if (!stats) return;
  stats->original_max = bits_to_double(hs.orig_max);
  stats->intermediate_max = bits_to_double(hs.inter_max);
  stats->finish_max = bits_to_double(hs.finish_max);
  stats->panel_multiplier_max = bits_to_double(hs.pmm);
}

// Q = H_0 H_1 ... assembled like pivoted_qr._reflect (q[:, k:] -= outer(beta*qv, v)).
// Q = H_0 H_1 ... H_{steps-1} from a reflector log.  neg_t = 0: Q column-major;
// neg_t = 1: -Q^T column-major (the Schur kernel's L operand for R12 = Q^T A21^T)
__global__ void zero2d_kernel(double* C, int64_t ldc, int rows, int64_t cols) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)rows * cols;
       e += (int64_t)gridDim.x * blockDim.x)
    C[(e / cols) * ldc + e % cols] = 0.0;
}

__global__ void form_q_kernel(const double* refl, int h, int steps, double* Q, int neg_t) {
  extern __shared__ __align__(16) double q[];   // row-major h x h
  __shared__ double qv[PRRP_MAXH];
  const int t = threadIdx.x;
  for (int e = t; e < h * h; e += blockDim.x) q[e] = (e / h == e % h) ? 1.0 : 0.0;
  __syncthreads();
  for (int k = 0; k < steps; ++k) {
    const double* v = refl + (int64_t)k * (h + 1);
    const double beta = v[h];
    if (beta == 0.0) continue;
    for (int i = t; i < h; i += blockDim.x) {
      double acc = 0.0;
      for (int l = k; l < h; ++l) acc = fma(q[i * h + l], v[l], acc);
      qv[i] = mul_rn(beta, acc);
    }
    __syncthreads();
    for (int e = t; e < h * (h - k); e += blockDim.x) {
      const int i = e / (h - k), l = k + e % (h - k);
      q[i * h + l] = sub_rn(q[i * h + l], mul_rn(qv[i], v[l]));
    }
    __syncthreads();
  }
  for (int e = t; e < h * h; e += blockDim.x) {
    const int i = e / h, j = e % h;
    if (neg_t) Q[e] = -q[e];
    else Q[i + (int64_t)j * h] = q[e];
  }
}

__global__ void r_out_kernel(const double* Rbuf, int h, int64_t p, const int32_t* perm, double* R, int64_t* perm_out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)h * p; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = e / h;
    const int i = (int)(e % h);
    R[e] = Rbuf[(int64_t)i * p + pos];
    if (i == 0) perm_out[pos] = perm[pos];
  }
}

// register-resident DMMA loop: 8 independent m8n8k4 chains per warp
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* sink, long iters) {
  double acc[8][2];
#pragma unroll
  for (int c = 0; c < 8; ++c) { acc[c][0] = threadIdx.x * 1e-3; acc[c][1] = c; }
  const double av = 1.0000001 + threadIdx.x * 1e-9, bv = 0.9999999 - threadIdx.x * 1e-9;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) dmma884(acc[c][0], acc[c][1], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1234.5) sink[0] = s;
}

// column-major R (ldr) rows 0..b-1 -> position-major Rbuf[i*p + pos]
__global__ void r_in_kernel(const double* R, int64_t ldr, int b, int64_t p, double* Rbuf) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)b * p; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = e / b;
    const int i = (int)(e % b);
    Rbuf[(int64_t)i * p + pos] = R[i + pos * ldr];
  }
}

__global__ void iota32_kernel(int32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)i;
}

DevState* new_state(Arena& ar, cudaStream_t s) {
  DevState* st = ar.get<DevState>(1);
  CU_TRY(cudaMemsetAsync(st, 0, sizeof(DevState), s));
  return st;
}

// > 0: CTA cap of the compose / block-row kernels (they run beside the next
// panel's tournament in the CALU schedule and must not take its SMs)
thread_local int tl_fin_ctas = 0;
// Workspace of the DMMA compose (one per factorization; the compose launches
// of consecutive panels follow each other on the fin stream).
struct ComposeWs {
  double* Lneg = nullptr;   // -L21[:, gperm], column-major M x b
  int64_t ld = 0;
  double* Bm = nullptr;     // L11 (unit lower), row-major b x b
  DevState* st = nullptr;   // scratch run state: the product's |C| must not enter the growth statistics
};
ComposeWs compose_ws(Arena& ar, cudaStream_t s, int64_t m, int b) {
  ComposeWs w;
  w.ld = ((m + 7) / 8) * 8;
  w.Lneg = ar.get<double>((size_t)b * w.ld);
  w.Bm = ar.get<double>((size_t)b * b);
  w.st = new_state(ar, s);
  return w;
}

// compose_below (luprrp.py:122-125): L21 <- matmul(L21[:, perm], L11), the
// dger k-loop from a zero accumulator.  With a workspace and b a multiple of
// 8 it runs on the DMMA pipe: out = 0 - (-L21[:, perm]) L11 with the Schur
// kernel, whose accumulation IS that k-loop (DMMA.8x8x4 is a sequential FMA
// chain over its four k's, k-steps in increasing order, from zero;
// test_schur_update_bit_exact) -- the terms k < j the SIMT kernel skips are
// x * 0 here, which leave a chain that starts at +0 unchanged -- and the
// negation is exact, so the result is bit-identical to compose_w_kernel
// (test_compose_dmma_bit_identical).  PRRP_COMPOSE_DMMA=0: the SIMT kernel.
void launch_compose_w(const double* L21, int64_t ldl, int64_t M, int b, const double* D, const int32_t* gperm,
                      double* out, int64_t ldo, DevState* st, cudaStream_t s, const ComposeWs* ws = nullptr) {
  if (M <= 0) return;
  static const bool dmma = !(getenv("PRRP_COMPOSE_DMMA") && atoi(getenv("PRRP_COMPOSE_DMMA")) == 0);
  if (ws && ws->Lneg && dmma && b % 8 == 0 && b >= 32 && M <= ws->ld && (ldo % 2 == 0) &&
      ((uintptr_t)out % 16 == 0)) {
    compose_prep_kernel<<<(unsigned)std::min<int64_t>(caps().sms * 4, (M * b + 255) / 256), 256, 0, s>>>(
        L21, ldl, M, b, D, gperm, ws->Lneg, ws->ld, ws->Bm, out, ldo, st);
    CU_TRY(cudaGetLastError());
    tl_schur_untracked = true;
    struct Reset { ~Reset() { tl_schur_untracked = false; } } reset;
    schur_update(out, ldo, ws->Lneg, ws->ld, ws->Bm, b, M, b, b, ws->st, s, 0, 0, false);
    return;
  }
  const unsigned grid = (unsigned)std::min<int64_t>(tl_fin_ctas > 0 ? tl_fin_ctas : caps().sms * 4, (M + TC - 1) / TC);
  const size_t dyn = ((size_t)b * b + (size_t)b * TCP) * 8;
  switch ((b + 31) / 32) {
    case 1: compose_w_kernel<1><<<grid, TW_WARPS * 32, dyn, s>>>(L21, ldl, M, b, D, gperm, out, ldo, st); break;
    case 2: compose_w_kernel<2><<<grid, TW_WARPS * 32, dyn, s>>>(L21, ldl, M, b, D, gperm, out, ldo, st); break;
    case 3: compose_w_kernel<3><<<grid, TW_WARPS * 32, dyn, s>>>(L21, ldl, M, b, D, gperm, out, ldo, st); break;
    default: compose_w_kernel<4><<<grid, TW_WARPS * 32, dyn, s>>>(L21, ldl, M, b, D, gperm, out, ldo, st); break;
  }
}

void launch_blockrow_w(double* A, int64_t lda, int64_t col0, int b, int64_t n, const double* D, const int32_t* gperm,
                       int64_t* perm, DevState* st, cudaStream_t s, int64_t bl = 1, int nr = 1, int rk = 0) {
  if (n <= 0) return;
  // thread-per-column kernel (b a multiple of 8; bit-identical, ~7x faster at
  // b = 128); PRRP_BLOCKROW_X=0: the warp-per-column kernel
  static const bool bx = !(getenv("PRRP_BLOCKROW_X") && atoi(getenv("PRRP_BLOCKROW_X")) == 0);
  if (bx && b % 8 == 0 && b >= 16 && (b > 64 || n >= 96 * BX_TC)) {   // (b <= 64, few columns: too few CTAs)
    const unsigned gx = (unsigned)std::min<int64_t>(tl_fin_ctas > 0 ? tl_fin_ctas : caps().sms * 4,
                                                    (n + BX_TC - 1) / BX_TC);
    blockrow_x_kernel<<<gx, BX_TC, bx_smem(b), s>>>(A, lda, col0, b, n, D, gperm, perm, st, bl, nr, rk);
    return;
  }
  const unsigned grid = (unsigned)std::min<int64_t>(tl_fin_ctas > 0 ? tl_fin_ctas : caps().sms * 4, (n + TC - 1) / TC);
  const size_t dyn = ((size_t)b * b + (size_t)b * TCP) * 8;
  switch ((b + 31) / 32) {
    case 1: blockrow_w_kernel<1><<<grid, TW_WARPS * 32, dyn, s>>>(A, lda, col0, b, n, D, gperm, perm, st, bl, nr, rk); break;
    case 2: blockrow_w_kernel<2><<<grid, TW_WARPS * 32, dyn, s>>>(A, lda, col0, b, n, D, gperm, perm, st, bl, nr, rk); break;
    case 3: blockrow_w_kernel<3><<<grid, TW_WARPS * 32, dyn, s>>>(A, lda, col0, b, n, D, gperm, perm, st, bl, nr, rk); break;
    default: blockrow_w_kernel<4><<<grid, TW_WARPS * 32, dyn, s>>>(A, lda, col0, b, n, D, gperm, perm, st, bl, nr, rk); break;
  }
}

// Per-thread internal streams (main: high priority, side: low priority) and a
// reusable pool of dependency events.
struct Streams {
  cudaStream_t main = nullptr, side = nullptr, fin = nullptr;
  std::vector<cudaEvent_t> evs;
  cudaEvent_t ev(int i) {
    while ((int)evs.size() <= i) {
      cudaEvent_t e;
      CU_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      evs.push_back(e);
    }
    return evs[i];
  }
};

Streams& streams() {
  thread_local Streams s;
  if (!s.main) {
    int lo = 0, hi = 0;
    CU_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU_TRY(cudaStreamCreateWithPriority(&s.main, cudaStreamNonBlocking, hi));
    CU_TRY(cudaStreamCreateWithPriority(&s.side, cudaStreamNonBlocking, lo));
    CU_TRY(cudaStreamCreateWithPriority(&s.fin, cudaStreamNonBlocking, hi));
  }
  return s;
}

// ---------------------------------------------------------------- LU_PRRP driver
constexpr size_t kMaxPlans = 4;   // cached graph plans per kind (LU_PRRP, CALU_PRRP)
// Graph kernel nodes carry the priority of the stream they were captured on;
// it only applies when the graph is instantiated with UseNodePriority (else the
// whole graph runs at the launch stream's priority and the critical stream
// loses its precedence over the trailing update).  PRRP_GRAPH_NODE_PRIO=0: off.
unsigned long long graph_instantiate_flags() {
  static const bool use = !(getenv("PRRP_GRAPH_NODE_PRIO") && atoi(getenv("PRRP_GRAPH_NODE_PRIO")) == 0);
  return use ? (unsigned long long)cudaGraphInstantiateFlagUseNodePriority : 0ull;
}

struct LuOut {
  DevState* st = nullptr;
  int32_t* swaps_dev = nullptr;
  int npanels = 0;
};

// Enqueue one LU_PRRP factorization on stream s (capturable unless the
// panel profiler is on); buffers from `ar`.
void luprrp_enqueue(double* A, int64_t lda, int64_t m, int64_t n, int b, double tau, int64_t* perm, cudaStream_t s,
                    Arena& ar, LuOut& out) {
  const int npanels = (int)((n + b - 1) / b);
  DevState* st = new_state(ar, s);
  const int64_t ldl = ((m + 7) / 8) * 8;
  double* L21 = ar.get<double>((size_t)b * ldl);
  const PanelCfg g0 = panel_config(b, m, b);
  PanelBuffers B{};
  B.Rbuf = ar.get<double>((size_t)b * m);
  B.perm = ar.get<int32_t>(m);
  B.ovf = ar.get<double>(ovf_elems(b, m, b));
  B.cand = ar.get<double>(kMaxCand);
  B.cand_flat = ar.get<long long>(kMaxCand);
  B.moved = ar.get<int32_t>(2 * m);
  alloc_exchange(ar, s, B);
  B.refl = nullptr;
  // per-panel-parity buffers (the three streams overlap consecutive panels)
  int32_t* movedb[2] = {B.moved, ar.get<int32_t>(2 * m)};
  int32_t* mcntb = ar.get<int32_t>(2);
  double* Db[2] = {ar.get<double>((size_t)b * b), ar.get<double>((size_t)b * b)};
  int32_t* pivb[2] = {ar.get<int32_t>(b), ar.get<int32_t>(b)};
  int32_t* gpermb[2] = {ar.get<int32_t>(b), ar.get<int32_t>(b)};
  int32_t* swaps_dev = ar.get<int32_t>(npanels);
  CU_TRY(cudaMemsetAsync(swaps_dev, 0, sizeof(int32_t) * npanels, s));
  const ComposeWs cws = compose_ws(ar, s, m, b);

  const int sms = caps().sms;
  tl_prof = nullptr;
  if (panel_prof_enabled()) {
    tl_prof = ar.get<long long>(8 + PRRP_CLUSTER_MAX * 64 * 8 + 16 * 64 * 8);
    CU_TRY(cudaMemsetAsync(tl_prof, 0, (8 + PRRP_CLUSTER_MAX * 64 * 8 + 16 * 64 * 8) * sizeof(long long), s));
    const char* e = getenv("PRRP_PANEL_TL");
    const long long target = e ? atoll(e) : -1;
    CU_TRY(cudaMemcpyAsync(tl_prof + 6, &target, sizeof(long long), cudaMemcpyHostToDevice, s));
  }
  tbegin(PRRP_K_OTHER, s);
  iota_kernel<<<sms, 256, 0, s>>>(perm, m);
  maxabs_kernel<<<sms * 4, 256, 0, s>>>(A, lda, m, n, st);
  tend(s);
  CU_TRY(cudaGetLastError());

  // ---- look-ahead schedule over three streams.  Panel
  // k's row moves are applied by column range, each part on the stream that
  // next touches those columns:
  //   main (high priority, critical path): [wait side(k-2), fin(k-2)] QRCP(k)
  //        -> trsm -> finalize -> [wait W1(k-1)] -> permute(k) of columns
  //        [col0, col0+2b) -> narrow Schur(k) (panel k+1's columns)
  //   fin (high priority): [wait permute(k)] permute(k) of columns [0, col0)
  //        + row order -> GEPP of A11 -> compose(k)
  //   side (low priority): [wait narrow(k)] permute(k) of columns >= col0+2b
  //        -> W1(k) (the next narrow region) -> W2(k) (the rest) -> [wait
  //        fin(k)] blockrow(k)
  // Panel k's moved rows are >= col0 and blockrow(k-1) writes rows < col0,
  // so the three parts never touch the same words.  L21, the moved list and
  // the GEPP outputs are double-buffered by panel parity; the waits on
  // side(k-2) / fin(k-2) guard their reuse.
  Streams& ss = streams();
  cudaStream_t sm = ss.main, sd = ss.side, sf = ss.fin;
  {
    cudaEvent_t e0 = ss.ev(0);
    CU_TRY(cudaEventRecord(e0, s));
    CU_TRY(cudaStreamWaitEvent(sm, e0, 0));
    CU_TRY(cudaStreamWaitEvent(sd, e0, 0));
    CU_TRY(cudaStreamWaitEvent(sf, e0, 0));
  }
  double* L21b[2] = {L21, ar.get<double>((size_t)b * ldl)};
  std::vector<cudaEvent_t> side_ev(npanels, nullptr), fin_ev(npanels, nullptr);
  cudaEvent_t w1_prev = nullptr, side_done = nullptr;
  int evi = 1;
  int panel = 0;
  auto permute_cols = [&](int64_t c_lo, int64_t c_hi, int64_t row0, const int32_t* mv, const int32_t* mc,
                          int64_t* pp, cudaStream_t q) {
    if (c_hi <= c_lo && !pp) return;
    const int64_t nc = std::max<int64_t>(c_hi - c_lo, 1);
    const unsigned grid = (unsigned)std::min<int64_t>((nc + 31) / 32, 2 * sms);
    permute_cols_kernel<<<grid, 256, 0, q>>>(A, lda, row0, c_lo, std::max(c_lo, c_hi), mv, mc, pp, st, panel);
    CU_TRY(cudaGetLastError());
  };
  for (int64_t col0 = 0; col0 < n; col0 += b, ++panel) {
    const int bj = (int)std::min<int64_t>(b, n - col0);
    const int64_t rows = m - col0;
    const int64_t width = n - col0 - bj;
    const int par = panel & 1;
    double* blk = A + col0 * lda + col0;
    double* L = L21b[par];
    double* D = Db[par];
    int32_t* piv = pivb[par];
    int32_t* gperm = gpermb[par];
    if (rows > bj) {
      if (panel >= 2) {
        CU_TRY(cudaStreamWaitEvent(sm, side_ev[panel - 2], 0));
        CU_TRY(cudaStreamWaitEvent(sm, fin_ev[panel - 2], 0));
      }
      PanelBuffers Bk = B;
      Bk.moved = movedb[par];
      Bk.moved_cnt = mcntb + par;
      strong_rrqr_panel(blk, lda, bj, rows, bj, tau, panel, L, ldl, Bk, st, swaps_dev, D, piv, gperm, false, sm);
      if (w1_prev) CU_TRY(cudaStreamWaitEvent(sm, w1_prev, 0));
      const int64_t wn = std::min<int64_t>(width, b);
      tbegin(PRRP_K_PERMUTE, sm);
      permute_cols(col0, col0 + bj + wn, col0, Bk.moved, Bk.moved_cnt, nullptr, sm);
      tend(sm);
      cudaEvent_t ev_perm = ss.ev(evi++);
      CU_TRY(cudaEventRecord(ev_perm, sm));
      // narrow update: the next panel's b columns, on the critical path
      if (wn > 0)
        schur_update(A + (col0 + bj) * lda + col0 + bj, lda, L, ldl, A + col0 * lda + col0 + bj, lda, rows - bj, wn,
                     bj, st, sm, sms);
      cudaEvent_t ev_narrow = ss.ev(evi++);
      CU_TRY(cudaEventRecord(ev_narrow, sm));
      // fin stream: L-part row moves + row order, GEPP of the pivot block,
      // multiplier compose -- concurrent with the trailing update
      CU_TRY(cudaStreamWaitEvent(sf, ev_perm, 0));
      tbegin(PRRP_K_PERMUTE, sf);
      permute_cols(0, col0, col0, Bk.moved, Bk.moved_cnt, perm, sf);
      tend(sf);
      tbegin(PRRP_K_GEPP, sf);
      launch_gepp(blk, lda, nullptr, bj, D, piv, gperm, st, panel, sf);
      tend(sf);
      CU_TRY(cudaGetLastError());
      const int ctw = bj > 64 ? 64 : 128;
      tbegin(PRRP_K_COMPOSE, sf);
      if (!force_generic_panel())
        launch_compose_w(L, ldl, rows - bj, bj, D, gperm, A + (col0 + bj) * lda + col0, lda, st, sf, &cws);
      else
        compose_kernel<<<(unsigned)((rows - bj + ctw - 1) / ctw), ctw, ((size_t)bj * bj + (size_t)bj * ctw) * 8, sf>>>(
            L, ldl, rows - bj, bj, D, gperm, A + (col0 + bj) * lda + col0, lda, st);
      tend(sf);
      CU_TRY(cudaGetLastError());
      fin_ev[panel] = ss.ev(evi++);
      CU_TRY(cudaEventRecord(fin_ev[panel], sf));
      // side stream: trailing row moves, wide update (next narrow region
      // first), block row
      CU_TRY(cudaStreamWaitEvent(sd, ev_narrow, 0));
      const int64_t cw0 = col0 + bj + wn;
      tbegin(PRRP_K_PERMUTE, sd);
      permute_cols(cw0, n, col0, Bk.moved, Bk.moved_cnt, nullptr, sd);
      tend(sd);
      const int64_t w1 = std::min<int64_t>(n - cw0, b);
      // persistent trailing update on all but 24 SMs: the high-priority stream
      // keeps room for the panel cluster (16 SMs of one GPC) and its kernels
      // (PRRP_SCHUR_WIDE_CTAS overrides; 0 = one tile per CTA)
      // (b = 128 panels taller than 4096 rows take two 16-CTA clusters: 40 SMs kept free)
      static const int wide_env = getenv("PRRP_SCHUR_WIDE_CTAS") ? atoi(getenv("PRRP_SCHUR_WIDE_CTAS")) : 0;
      const int wide_ctas = wide_env > 0 ? wide_env : std::max(1, sms - (b > 64 && m > 4096 ? 40 : 24));
      if (w1 > 0)
        schur_update(A + (col0 + bj) * lda + cw0, lda, L, ldl, A + col0 * lda + cw0, lda, rows - bj, w1, bj, st, sd,
                     wide_ctas);
      w1_prev = ss.ev(evi++);
      CU_TRY(cudaEventRecord(w1_prev, sd));
      if (n - cw0 > w1)
        schur_update(A + (col0 + bj) * lda + cw0 + w1, lda, L, ldl, A + col0 * lda + cw0 + w1, lda, rows - bj,
                     n - cw0 - w1, bj, st, sd, wide_ctas, 0, w2_stream);
      CU_TRY(cudaStreamWaitEvent(sd, fin_ev[panel], 0));
    } else {
      // last block (rows == bj): all its updates and row moves came through main
      // (narrow) and fin (L part), both already awaited by the side stream
      tbegin(PRRP_K_GEPP, sd);
      launch_gepp(blk, lda, nullptr, bj, D, piv, gperm, st, panel, sd);
      tend(sd);
      CU_TRY(cudaGetLastError());
    }
    tbegin(PRRP_K_BLOCKROW, sd);
    if (!force_generic_panel())
      launch_blockrow_w(A, lda, col0, bj, n, D, gperm, perm, st, sd);
    else
      blockrow_kernel<<<(unsigned)((n + BR_TW - 1) / BR_TW), BR_TW, ((size_t)bj * bj + (size_t)bj * BR_TW) * 8, sd>>>(
          A, lda, col0, bj, n, D, piv, gperm, perm, st);
    tend(sd);
    CU_TRY(cudaGetLastError());
    side_done = ss.ev(evi++);
    CU_TRY(cudaEventRecord(side_done, sd));
    side_ev[panel] = side_done;
  }
  CU_TRY(cudaStreamWaitEvent(sm, side_done, 0));
  tbegin(PRRP_K_OTHER, sm);   // closing mark for the timer span
  tend(sm);
  {
    cudaEvent_t e1 = ss.ev(evi++);
    CU_TRY(cudaEventRecord(e1, sm));
    CU_TRY(cudaStreamWaitEvent(s, e1, 0));
  }
  out.st = st;
  out.swaps_dev = swaps_dev;
  out.npanels = npanels;
}

// A captured LU_PRRP factorization (see CaluPlan): the direct enqueue of the
// ~7600 launches costs the GPU launch gaps on the critical stream
struct LuPlan {
  double* A; int64_t lda, m, n; int b; double tau; int64_t* perm; int dev;
  cudaGraphExec_t exec = nullptr;
  std::vector<void*> bufs;
  LuOut out;
  uint64_t used = 0;
  ~LuPlan() {
    if (exec) cudaGraphExecDestroy(exec);
    for (void* p : bufs) cudaFree(p);
  }
};
std::vector<std::shared_ptr<LuPlan>>& lu_plans() {
  static std::vector<std::shared_ptr<LuPlan>> v;
  return v;
}
std::mutex g_lu_plans_mu;
uint64_t g_lu_plan_clock = 0;

int luprrp_finish(const LuOut& out, cudaStream_t s, int32_t* swap_counts, prrp_stats* stats, prrp_err* err,
                  prrp_timing* timing, Timer* timer, std::chrono::steady_clock::time_point host_t0);

int luprrp_impl(double* A, int64_t lda, int64_t m, int64_t n, int b, double tau, int64_t* perm,
                int32_t* swap_counts, prrp_stats* stats, prrp_err* err, prrp_timing* timing, cudaStream_t s) {
  Timer timer;
  tl_timer = timing ? &timer : nullptr;
  tl_schur_flops = 0.0;
  struct Reset { ~Reset() { tl_timer = nullptr; } } reset_timer;
  if (m < n) fail(PRRP_ERR_DIM, "need at least as many rows as columns");
  if (b < 1 || b > n) fail(PRRP_ERR_ARG, "panel width out of range");
  if (!(tau > 1.0)) fail(PRRP_ERR_ARG, "tau must exceed 1");
  if (b > PRRP_MAXH) fail(PRRP_ERR_UNSUPPORTED, "panel width > 128 is outside the device panel engine");
  if (lda < n) fail(PRRP_ERR_ARG, "lda < n");
  caps();
  const auto host_t0 = std::chrono::steady_clock::now();
  // graph replay is opt-in for LU_PRRP (PRRP_LU_GRAPH=1): its host enqueue
  // (~6.5 ms) is far shorter than the GPU work, and the replayed schedule was
  // measured slower (44-49 vs 42-43 ms at n = 8192, b = 64; 56.7 vs 53.3 ms at
  // b = 128) even with per-node priorities
  static const bool lu_graph = !(getenv("PRRP_GRAPH") && atoi(getenv("PRRP_GRAPH")) == 0) &&
                               getenv("PRRP_LU_GRAPH") && atoi(getenv("PRRP_LU_GRAPH")) != 0;
  if (timing || panel_prof_enabled() || !lu_graph) {
    Arena ar(s);
    LuOut out;
    luprrp_enqueue(A, lda, m, n, b, tau, perm, s, ar, out);
    return luprrp_finish(out, s, swap_counts, stats, err, timing, &timer, host_t0);
  }
  int dev = 0;
  CU_TRY(cudaGetDevice(&dev));
  std::unique_lock<std::mutex> plans_lock(g_lu_plans_mu);
  auto& plans = lu_plans();
  LuPlan* pl = nullptr;
  for (auto& q : plans)
    if (q->A == A && q->lda == lda && q->m == m && q->n == n && q->b == b && q->tau == tau && q->perm == perm &&
        q->dev == dev)
      pl = q.get();
  if (!pl) {
    if (plans.size() >= kMaxPlans) {
      auto lru = std::min_element(plans.begin(), plans.end(),
                                  [](const std::shared_ptr<LuPlan>& x, const std::shared_ptr<LuPlan>& y) {
                                    // plans held by an in-flight call (use_count > 1) are never evicted
                                    return (x.use_count() > 1 ? UINT64_MAX : x->used) <
                                           (y.use_count() > 1 ? UINT64_MAX : y->used);
                                  });
      if (lru->use_count() == 1) {
        CU_TRY(cudaDeviceSynchronize());
        plans.erase(lru);
      }
    }
    std::shared_ptr<LuPlan> np(new LuPlan{A, lda, m, n, b, tau, perm, dev});
    static thread_local cudaStream_t cs = nullptr;
    if (!cs) CU_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    CU_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
    try {
      Arena ar(cs, &np->bufs);
      luprrp_enqueue(A, lda, m, n, b, tau, perm, cs, ar, np->out);
    } catch (...) {
      cudaStreamEndCapture(cs, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    CU_TRY(cudaStreamEndCapture(cs, &g));
    const cudaError_t ie = cudaGraphInstantiate(&np->exec, g, graph_instantiate_flags());
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) fail(PRRP_ERR_CUDA, "cudaGraphInstantiate failed");
    plans.push_back(std::move(np));
    pl = plans.back().get();
  }
  pl->used = ++g_lu_plan_clock;
  // the read-back below reads the plan's buffers (state, swap counts) outside
  // the cache lock: keep the plan alive (and unevictable) until it is done
  std::shared_ptr<LuPlan> hold;
  for (auto& q : plans)
    if (q.get() == pl) hold = q;
  CU_TRY(cudaGraphLaunch(pl->exec, s));
  const LuOut out = pl->out;
  plans_lock.unlock();
  const int rc = luprrp_finish(out, s, swap_counts, stats, err, nullptr, nullptr, host_t0);
  std::lock_guard<std::mutex> relock(g_lu_plans_mu);
  hold.reset();
  return rc;
}

int luprrp_finish(const LuOut& out, cudaStream_t s, int32_t* swap_counts, prrp_stats* stats, prrp_err* err,
                  prrp_timing* timing, Timer* timer, std::chrono::steady_clock::time_point host_t0) {
  const int npanels = out.npanels;
  int32_t* swaps_dev = out.swaps_dev;
  const auto host_t1 = std::chrono::steady_clock::now();
  DevState hs;
  read_state(out.st, hs, s);
  if (getenv("PRRP_HOSTTIME"))
    fprintf(stderr, "[prrp lu host] enqueue %.3f ms, then wait %.3f ms\n",
            std::chrono::duration<double, std::milli>(host_t1 - host_t0).count(),
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t1).count());
  if (tl_prof) {
    long long pr[8];
    CU_TRY(cudaMemcpy(pr, tl_prof, sizeof(pr), cudaMemcpyDeviceToHost));
    fprintf(stderr, "[prrp panel prof] launches=%lld cycles: reduce=%lld publish+cluster_sync=%lld "
            "winner+reflector=%lld apply=%lld total=%lld\n", pr[5], pr[0], pr[1], pr[2], pr[3], pr[4]);
    if (getenv("PRRP_PANEL_TL")) {
      std::vector<long long> tl(PRRP_CLUSTER_MAX * 64 * 8 + 16 * 64 * 8);
      CU_TRY(cudaMemcpy(tl.data(), tl_prof + 8, tl.size() * sizeof(long long), cudaMemcpyDeviceToHost));
      FILE* f = fopen(getenv("PRRP_PANEL_TL_OUT") ? getenv("PRRP_PANEL_TL_OUT") : "panel_tl.bin", "wb");
      if (f) { fwrite(tl.data(), sizeof(long long), tl.size(), f); fclose(f); }
    }
    tl_prof = nullptr;
  }
  std::vector<int32_t> sw(npanels);
  CU_TRY(cudaMemcpy(sw.data(), swaps_dev, sizeof(int32_t) * npanels, cudaMemcpyDeviceToHost));
  if (swap_counts) memcpy(swap_counts, sw.data(), sizeof(int32_t) * npanels);
  fill_stats(hs, stats);
  if (stats) {
    stats->total_swaps = 0;
    for (int v : sw) stats->total_swaps += v;
  }
  if (timing && timer) {
    timer->collect(timing);
    timing->schur_flops = tl_schur_flops;
  }
  return state_to_err(hs, err);
}


// ---------------------------------------------------------------- CALU_PRRP driver
// Binary tournament (tournament.py:155-217) + CALU_PRRP panel loop
// (tournament.py:237-296).  Tree nodes of one level run concurrently on a
// pool of streams; every node is the cluster QRCP engine + multipliers +
// swap loop on an index list of logical rows.
struct NodeBufs {
  PanelBuffers B;
  double* L21;
  int64_t ldl;
  int32_t* lpos_in;   // merge nodes: 2b logical positions
  int64_t* rowidx;    // merge nodes: 2b physical rows
};

struct PtrPack { const int32_t* p[32]; };
__global__ void store_ptrs_kernel(PtrPack pk, int cnt, const int32_t** out) {
  if ((int)threadIdx.x < cnt) out[threadIdx.x] = pk.p[threadIdx.x];
}

thread_local std::vector<cudaStream_t> tl_node_streams;
cudaStream_t node_stream(int i) {
  while ((int)tl_node_streams.size() <= i) {
    cudaStream_t st;
    int lo = 0, hi = 0;
    CU_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU_TRY(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi));
    tl_node_streams.push_back(st);
  }
  return tl_node_streams[i];
}

int64_t qr_charge3(int64_t r, int64_t b) { return 6 * r * b * b - 2 * b * b * b; }   // 3 * _charge_qr

// What the host needs after a CALU_PRRP enqueue (device result slots and the
// tournament bookkeeping for the flop charges); kept by a cached graph plan.
struct CaluOut {
  DevState* st = nullptr;
  int32_t* swaps_dev = nullptr;
  int32_t* node_swaps = nullptr;
  int32_t* node_rows = nullptr;
  int64_t n = 0;
  std::vector<int64_t> charges;
  std::vector<std::vector<std::pair<int64_t, int>>> node_members;   // (members, node slot)
  int npanels = 0, maxnodes = 0, b = 0;
};

// Enqueue one CALU_PRRP factorization on stream s (capturable: no host
// synchronisation, no pageable copies); buffers from `ar`.
// "Panel pnl of an m x n CALU_PRRP with block b is chain-bound": its trailing
// update is estimated shorter than PRRP_CALU_CB_MS (25 TFLOP/s), so the
// tournament chain, not the update, bounds the panel (see caluprrp_enqueue).
// The single-GPU and the distributed driver use the same rule, so every node
// runs on the same engine in both (bit-identical results).
// A warp that sleeps for `us` microseconds: the side and fin streams of the
// CALU schedule start their work for panel k this long after the narrow
// update, i.e. after the next panel's leaf clusters have been launched.  A
// leaf CTA of the thread-per-column engine takes ~60K of an SM's 64K
// registers, so it cannot share an SM with a row-move / GEPP / compose CTA
// that got there a few microseconds earlier, and a 16-CTA cluster that does
// not find 16 free SMs in one GPC waits for the whole level (the straggler
// leaf of the span traces).  PRRP_CALU_SIDE_DELAY_US (default 0 = off):
// measured neutral under graph replay (1150 ms at 20 and 50 us, 1154 at 100),
// so the straggler of the direct-enqueue traces is not a launch-order effect.
__global__ void spin_delay_kernel(unsigned us) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  } while (t1 - t0 < (unsigned long long)us * 1000ull);
}

int calu_leaf_cmax() {
  static const int v = getenv("PRRP_CALU_LEAF_CMAX") ? atoi(getenv("PRRP_CALU_LEAF_CMAX")) : 8;
  return v;
}
bool calu_chain_bound(int64_t m, int64_t n, int b, int pnl, bool flat) {
  // thresholds ~ the chain time of a panel: ~2 ms at b = 128, ~0.8 ms at b = 64
  static const double cb_ms = getenv("PRRP_CALU_CB_MS") ? atof(getenv("PRRP_CALU_CB_MS")) : 1.5;
  static const double cb_ms64 = getenv("PRRP_CALU_CB_MS64") ? atof(getenv("PRRP_CALU_CB_MS64")) : 0.6;
  const double thr = b > 64 ? cb_ms : cb_ms64;
  if (!(thr > 0.0 && (b == 64 || b == 128 || b == 32) && !flat && caps().max_cluster >= 16 &&
        caps().schur_clusters16 >= 2 && lat_default_cmax() > 0))
    return false;
  const int64_t c0 = (int64_t)pnl * b;
  if (c0 + b >= n) return true;
  const double fl = 2.0 * b * (double)(m - c0 - b) * (double)(n - c0 - b);
  return fl / (b > 64 ? 25e12 : 18e12) * 1e3 < thr;
}

void caluprrp_enqueue(double* A, int64_t lda, int64_t m, int64_t n, int b, double tau, int P, int64_t* perm,
                      cudaStream_t s, Arena& ar, CaluOut& out) {
  static const bool calu_late_c = !getenv("PRRP_CALU_LATE_C") || atoi(getenv("PRRP_CALU_LATE_C")) != 0;
  tl_schur_prefetch_c = !calu_late_c;
  struct ResetPf { ~ResetPf() { tl_schur_prefetch_c = false; } } reset_pf;
  const int npanels = (int)((n + b - 1) / b);
  // P >= 1: binary tree over P leaves; P == 0: the flat tree (tournament.py:
  // 81-88, 202-208: a first block of 2b rows, then b-row blocks, reduced one
  // after the other, so one node per level and up to m/b + 1 nodes per panel)
  const bool flat = P == 0;
  const int maxnodes = flat ? (int)(m / std::max(1, b) + 2) : 2 * P;   // node slots per panel
  const int nnodes = flat ? 1 : maxnodes;                               // node buffers
  // Schur launches: the tournament needs whole SMs (16-CTA clusters) at once,
  // so by default the updates run as short CTAs (classic kernel, quantum 0)
  // that hand SMs back quickly.  PRRP_CALU_NARROW: CTAs of a persistent
  // narrow update (0 = classic); PRRP_CALU_WIDE_Q: tiles per CTA of the
  // warp-specialised trailing update (0 = classic)
  static const int calu_narrow_ctas = getenv("PRRP_CALU_NARROW") ? atoi(getenv("PRRP_CALU_NARROW")) : 0;
  static const int calu_wide_q = getenv("PRRP_CALU_WIDE_Q") ? atoi(getenv("PRRP_CALU_WIDE_Q")) : 0;
  static const int calu_wide_ctas = getenv("PRRP_CALU_WIDE_CTAS") ? atoi(getenv("PRRP_CALU_WIDE_CTAS"))
                                                                  : std::max(1, caps().sms - 5);
  DevState* st = new_state(ar, s);
  const int64_t ldl = ((m + 7) / 8) * 8;
  double* Lphys = ar.get<double>((size_t)b * ldl);
  // main (whole-panel) buffers
  PanelBuffers B{};
  B.Rbuf = ar.get<double>((size_t)b * m);
  B.perm = ar.get<int32_t>(m);
  B.ovf = ar.get<double>(ovf_elems(b, m, b));
  B.cand = ar.get<double>(kMaxCand);
  B.cand_flat = ar.get<long long>(kMaxCand);
  B.moved = ar.get<int32_t>(2 * m);
  alloc_exchange(ar, s, B);
  double* Llog = ar.get<double>((size_t)b * ldl);
  double* Rsmall = ar.get<double>((size_t)b * b);
  double* refl = ar.get<double>((size_t)b * (b + 1));
  int32_t* perm_small = ar.get<int32_t>(b);
  // R12 of the final panel QR as a DMMA product for b > 64 (default;
  // PRRP_CALU_R12_GEMM=0: the logged reflectors applied row by row, one warp
  // per row, which holds the critical stream ~4 ms per panel at n = 32768,
  // b = 128, while the trailing update occupies most SMs; at b = 64 the row
  // by row form is the faster one, 289 vs 303 ms at n = 16384)
  static const bool calu_r12_gemm = !getenv("PRRP_CALU_R12_GEMM") || atoi(getenv("PRRP_CALU_R12_GEMM")) != 0;
  double* Qneg = ar.get<double>((size_t)b * b);
  int32_t* final_live = ar.get<int32_t>(1);
  const int64_t ld21t = ((m + 7) / 8) * 8;
  double* A21t = ar.get<double>((size_t)b * ld21t);
  DevState* st_r12 = new_state(ar, s);   // the product's |C| must not enter the growth statistics
  const ComposeWs cws = compose_ws(ar, s, m, b);
  // tree nodes
  std::vector<NodeBufs> nodes(nnodes);
  const int64_t leafmax =
      flat ? 2 * b : m / std::max<int64_t>(1, std::min<int64_t>(P, std::max<int64_t>(1, m / (b + 1)))) + 1;
  const int64_t pnode = std::max<int64_t>(leafmax, 2 * b + 2);
  int32_t* lpos_all = ar.get<int32_t>((size_t)nnodes * 2 * b);
  int64_t* rowidx_all = ar.get<int64_t>((size_t)nnodes * 2 * b);
  for (int i = 0; i < nnodes; ++i) {
    NodeBufs& nb = nodes[i];
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
    nb.lpos_in = lpos_all + (size_t)i * 2 * b;
    nb.rowidx = rowidx_all + (size_t)i * 2 * b;
  }
  int32_t* cands = ar.get<int32_t>((size_t)2 * nnodes * b);        // two levels (ping-pong)
  // per node: candidates passed up (< b after a rank-deficient node,
  // tournament.py:131-137), live members of a merge node, and per slot the
  // member count for the flop charges (tournament.py:224-234)
  int32_t* ccnt = ar.get<int32_t>((size_t)2 * nnodes);
  int32_t* want_all = ar.get<int32_t>((size_t)nnodes);
  int32_t* live_all = ar.get<int32_t>((size_t)nnodes);
  int32_t* node_rows = ar.get<int32_t>((size_t)npanels * maxnodes);
  CU_TRY(cudaMemsetAsync(node_rows, 0, sizeof(int32_t) * npanels * maxnodes, s));
  int32_t* node_swaps = ar.get<int32_t>((size_t)npanels * maxnodes);
  CU_TRY(cudaMemsetAsync(node_swaps, 0, sizeof(int32_t) * npanels * maxnodes, s));
  const int32_t** perms_dev = ar.get<const int32_t*>(nnodes);
  int64_t* leaf_lo_dev = ar.get<int64_t>(nnodes);
  int64_t* pos2row = ar.get<int64_t>(m);
  int64_t* scratch = ar.get<int64_t>(3 * m);
  int32_t* log2phys = ar.get<int32_t>(m);
  int32_t* ident = ar.get<int32_t>(m);
  double* D = ar.get<double>((size_t)b * b);
  int32_t* piv = ar.get<int32_t>(b);
  int32_t* gperm = ar.get<int32_t>(b);
  int32_t* swaps_dev = ar.get<int32_t>(npanels);
  CU_TRY(cudaMemsetAsync(swaps_dev, 0, sizeof(int32_t) * npanels, s));
  for (int i0 = 0; i0 < nnodes; i0 += 32) {     // node perm pointers (by value: capturable)
    PtrPack pk{};
    const int cnt = std::min(32, nnodes - i0);
    for (int i = 0; i < cnt; ++i) pk.p[i] = nodes[i0 + i].B.perm;
    store_ptrs_kernel<<<1, 32, 0, s>>>(pk, cnt, perms_dev + i0);
  }
  const int sms = caps().sms;
  iota_kernel<<<sms, 256, 0, s>>>(perm, m);
  iota_kernel<<<sms, 256, 0, s>>>(pos2row, m);
  iota32_kernel<<<sms, 256, 0, s>>>(ident, m);
  maxabs_kernel<<<sms * 4, 256, 0, s>>>(A, lda, m, n, st);
  CU_TRY(cudaGetLastError());
  std::vector<int64_t> charges(npanels, -1);
  std::vector<std::vector<std::pair<int64_t, int>>> node_members(npanels);   // (members, node slot)

  static const int early_w2 = getenv("PRRP_CALU_EARLY_W2") ? atoi(getenv("PRRP_CALU_EARLY_W2")) : 0;   // diagnostics
  // PRRP_CALU_SB_SERIAL bit 2: the previous panel's fin-stream work starts when the leaves' QRCP kernels are done
  static const bool fin_after_leaf_qrcp = getenv("PRRP_CALU_SB_SERIAL") && (atoi(getenv("PRRP_CALU_SB_SERIAL")) & 4);
  std::vector<cudaEvent_t> leaf_qrcp_ev;
  auto run_level = [&](const std::vector<int64_t>& lo, const std::vector<int64_t>& cnt, bool leaves,
                       int64_t col0, int bj, int panel, int level, int slot0, cudaStream_t qs) {
    // fork
    cudaEvent_t fk;
    CU_TRY(cudaEventCreateWithFlags(&fk, cudaEventDisableTiming));
    CU_TRY(cudaEventRecord(fk, qs));
    const int nn = (int)lo.size();
    for (int i = 0; i < nn; ++i) {
      cudaStream_t ns = node_stream(i);
      CU_TRY(cudaStreamWaitEvent(ns, fk, 0));
      const int64_t* ridx = leaves ? pos2row + col0 + lo[i] : nodes[i].rowidx;
      if (cnt[i] <= bj) continue;                       // node passes its rows through
      cudaEvent_t qe = nullptr;
      if (leaves && (early_w2 || fin_after_leaf_qrcp)) {
        CU_TRY(cudaEventCreateWithFlags(&qe, cudaEventDisableTiming));
        leaf_qrcp_ev.push_back(qe);
      }
      PanelBuffers nbuf = nodes[i].B;
      nbuf.live = leaves ? nullptr : live_all + i;
      nbuf.want = want_all + i;
      nbuf.node_rows = node_rows + (size_t)panel * maxnodes;
      // the leaves of a level run side by side: clusters of at most
      // calu_leaf_cmax() CTAs, so that all of them are resident at once
      const int cmax_level = tl_lat_cmax;
      if (leaves && tl_lat_cmax > 0) tl_lat_cmax = std::min(tl_lat_cmax, calu_leaf_cmax());
      strong_rrqr_panel(A + col0, lda, bj, cnt[i], bj, tau, panel, nodes[i].L21, nodes[i].ldl, nbuf, st,
                        node_swaps + (size_t)panel * maxnodes, nullptr, nullptr, nullptr, false, ns, ridx,
                        slot0 + i, level, i, qe);
      tl_lat_cmax = cmax_level;
    }
    // join
    for (int i = 0; i < nn; ++i) {
      cudaEvent_t jn;
      CU_TRY(cudaEventCreateWithFlags(&jn, cudaEventDisableTiming));
      CU_TRY(cudaEventRecord(jn, node_stream(i)));
      CU_TRY(cudaStreamWaitEvent(qs, jn, 0));
      CU_TRY(cudaEventDestroy(jn));
    }
    CU_TRY(cudaEventDestroy(fk));
  };

  // ---- look-ahead over three streams, as in LU_PRRP (see luprrp_impl):
  //   main: [side(k-2), fin(k-2)] tournament(k) (nodes on the pool) -> reorder
  //         -> [W1(k-1)] row moves of [col0, col0+2b) -> final QR of the pivot
  //         block + logged reflectors on the other rows -> L21 -> narrow Schur
  //   fin:  [row moves(k)] row moves of [0, col0) + row order -> GEPP -> compose
  //   side: [narrow(k)] row moves of [col0+2b, n) -> W1(k) -> W2(k) -> [fin(k)]
  //         blockrow(k)
  // Moved rows are physical slots >= col0 and blockrow(k-1) writes slots < col0.
  Streams& ss = streams();
  cudaStream_t sm = ss.main, sd = ss.side, sf = ss.fin;
  {
    cudaEvent_t e0 = ss.ev(0);
    CU_TRY(cudaEventRecord(e0, s));
    CU_TRY(cudaStreamWaitEvent(sm, e0, 0));
    CU_TRY(cudaStreamWaitEvent(sd, e0, 0));
    CU_TRY(cudaStreamWaitEvent(sf, e0, 0));
  }
  int32_t* movedb[2] = {B.moved, ar.get<int32_t>(2 * m)};
  int32_t* mcntb = ar.get<int32_t>(2);
  double* Llogb[2] = {Llog, ar.get<double>((size_t)b * ldl)};
  const int64_t lda12 = std::max<int64_t>(2, ((n + 1) / 2) * 2);           // pivot-row copies, per parity
  double* a12cb[2] = {ar.get<double>((size_t)b * lda12), ar.get<double>((size_t)b * lda12)};
  double* Lphysb[2] = {Lphys, ar.get<double>((size_t)b * ldl)};
  double* Db[2] = {D, ar.get<double>((size_t)b * b)};
  int32_t* pivb[2] = {piv, ar.get<int32_t>(b)};
  int32_t* gpermb[2] = {gperm, ar.get<int32_t>(b)};
  std::vector<cudaEvent_t> side_ev(npanels, nullptr), fin_ev(npanels, nullptr);
  cudaEvent_t w1_prev = nullptr, side_done = nullptr;
  int evi = 1;
  auto permute_cols = [&](int64_t c_lo, int64_t c_hi, int64_t row0, const int32_t* mv, const int32_t* mc,
                          int64_t* pp, int pnl, cudaStream_t q) {
    if (c_hi <= c_lo && !pp) return;
    const int64_t nc = std::max<int64_t>(c_hi - c_lo, 1);
    static const int perm_ctas = getenv("PRRP_CALU_PERM_CTAS") ? atoi(getenv("PRRP_CALU_PERM_CTAS")) : 0;
    const unsigned grid = (unsigned)std::min<int64_t>((nc + 31) / 32, perm_ctas > 0 ? perm_ctas : 2 * sms);
    permute_cols_kernel<<<grid, 256, 0, q>>>(A, lda, row0, c_lo, std::max(c_lo, c_hi), mv, mc, pp, st, pnl);
    CU_TRY(cudaGetLastError());
  };
  // The tournament's multi-CTA leaf clusters need whole SMs of one GPC at
  // once, which a running trailing update never hands back; so the bulk of
  // panel k's trailing update (W2) and its block row are enqueued only after
  // panel k+1's leaves (side waits for them), and run as a persistent kernel
  // on all but 8 SMs, beside the rest of the tournament chain
  // (PRRP_CALU_DEFER=0: enqueue at once).
  static const int calu_defer = getenv("PRRP_CALU_DEFER") ? atoi(getenv("PRRP_CALU_DEFER")) : 1;
  std::function<void()> pending_side, pending_fin;
  auto flush_side = [&](cudaEvent_t after) {
    if (pending_fin) {
      if (after) CU_TRY(cudaStreamWaitEvent(sf, after, 0));
      pending_fin();
      pending_fin = nullptr;
    }
    if (!pending_side) return;
    if (after) CU_TRY(cudaStreamWaitEvent(sd, after, 0));
    pending_side();
    pending_side = nullptr;
  };
  auto flush_after_main = [&]() {
    if (!pending_side && !pending_fin) return;
    cudaEvent_t e = ss.ev(evi++);
    CU_TRY(cudaEventRecord(e, sm));
    flush_side(e);
  };
  // Update-bound panels: the leaf level of panel k+1 is the one part of the
  // chain the trailing update cannot overlap (its clusters need the whole
  // GPU).  PRRP_CALU_SB_SERIAL keeps other work away from it: bit 0 makes
  // main wait for W1(k) before the leaves, bit 1 enqueues panel k's
  // fin-stream work (GEPP, compose, block row) after them like W2(k).  Both
  // were measured SLOWER at config 5 (1315 and 1447 ms against 1291: the
  // deferred work then competes with the chain for the 8 spare SMs), so off.
  static const int sb_serial = getenv("PRRP_CALU_SB_SERIAL") ? atoi(getenv("PRRP_CALU_SB_SERIAL")) : 0;
  // Two regimes.  While a panel's trailing update (W2) outlasts the
  // tournament chain the update is the bottleneck: it runs on all but 8 SMs
  // and the tournament's small nodes run as single CTAs on the rest.  Once
  // the chain is the bottleneck (estimated W2 time below PRRP_CALU_CB_MS),
  // W2 is launched as PRRP_CALU_W2_CLUSTERS clusters of 16 CTAs -- clusters
  // are placed inside one GPC, so one GPC stays free -- and the tournament
  // nodes run on the latency engine with clusters of up to 16 CTAs there;
  // (PRRP_CALU_CB_FIN caps the compose / block-row kernels of the fin stream;
  // measured slower -- the next-but-one panel waits for them -- so off.)
  static const int w2_clusters = getenv("PRRP_CALU_W2_CLUSTERS") ? atoi(getenv("PRRP_CALU_W2_CLUSTERS"))
                                                                 : std::max(1, caps().schur_clusters16 - 1);
  static const int cb_fin_ctas = getenv("PRRP_CALU_CB_FIN") ? atoi(getenv("PRRP_CALU_CB_FIN")) : 0;
  auto chain_bound = [&](int pnl) { return calu_chain_bound(m, n, b, pnl, flat); };
  struct LatScope {      // the thread's latency-engine setting is restored on every exit path
    ~LatScope() { tl_lat_cmax = -1; tl_fin_ctas = 0; tl_schur_cluster = 0; }
  } lat_scope;
  int panel = 0;
  for (int64_t col0 = 0; col0 < n; col0 += b, ++panel) {
    const int bj = (int)std::min<int64_t>(b, n - col0);
    const int64_t rows = m - col0;
    const int64_t width = n - col0 - bj;
    const int par = panel & 1;
    tl_lat_cmax = chain_bound(panel) ? 16 : 0;
    tl_fin_ctas = chain_bound(panel + 1) ? cb_fin_ctas : 0;
    double* blk = A + col0 * lda + col0;
    double* Lg = Llogb[par];
    double* Lp = Lphysb[par];
    double* Dk = Db[par];
    int32_t* pivk = pivb[par];
    int32_t* gpk = gpermb[par];
    int32_t* mv = movedb[par];
    int32_t* mc = mcntb + par;
    PanelBuffers Bk = B;
    Bk.moved = mv;
    Bk.moved_cnt = mc;
    if (rows > bj) {
      if (panel >= 2) {
        CU_TRY(cudaStreamWaitEvent(sm, side_ev[panel - 2], 0));
        CU_TRY(cudaStreamWaitEvent(sm, fin_ev[panel - 2], 0));
      }
      if ((sb_serial & 1) && calu_defer && b > 64 && !chain_bound(panel) && w1_prev) CU_TRY(cudaStreamWaitEvent(sm, w1_prev, 0));
      const int64_t first = std::min<int64_t>(rows, 2 * bj);
      const int64_t p_eff = flat ? 1 + (rows - first + bj - 1) / bj
                                 : std::max<int64_t>(1, std::min<int64_t>(P, rows / (bj + 1)));
      int64_t root_p = 0;   // columns of the root node's QRCP (the final QR reuses it)
      if (p_eff > 1 && flat) {
        // flat tree: the first block as a leaf, then one merge node per block
        // on [candidates, block rows] (members in that order, tournament.py:206)
        calu_leaf_lo_kernel<<<1, 64, 0, sm>>>(leaf_lo_dev, 1, rows, 0);
        int64_t chg3 = 0;
        int slot = 0;
        run_level(std::vector<int64_t>{0}, std::vector<int64_t>{first}, true, col0, bj, panel, 0, slot, sm);
        flush_after_main();
        chg3 += qr_charge3(first, bj);
        node_members[panel].push_back({first, slot});
        ++slot;
        int32_t* cur = cands;
        int32_t* nxt = cands + (size_t)b;
        int32_t* ccur = ccnt;
        int32_t* cnxt = ccnt + 1;
        calu_select_kernel<<<1, 128, 0, sm>>>(perms_dev, nullptr, leaf_lo_dev, bj, want_all, live_all, 0, cur, ccur,
                                              2 * b, st);
        int level = 1;
        for (int64_t lo = first; lo < rows; lo += bj, ++level) {
          const int64_t len = std::min<int64_t>(bj, rows - lo);
          root_p = bj + len;
          calu_flat_inputs_kernel<<<1, 128, 0, sm>>>(cur, ccur, bj, lo, (int)len, lpos_all, rowidx_all, live_all,
                                                     pos2row, col0, st);
          run_level(std::vector<int64_t>{0}, std::vector<int64_t>{bj + len}, false, col0, bj, panel, level, slot, sm);
          chg3 += qr_charge3(bj + len, bj);
          node_members[panel].push_back({bj + len, slot});
          ++slot;
          calu_select_kernel<<<1, 128, 0, sm>>>(perms_dev, lpos_all, nullptr, bj, want_all, live_all, 1, nxt, cnxt,
                                                2 * b, st);
          std::swap(cur, nxt);
          std::swap(ccur, cnxt);
        }
        CU_TRY(cudaGetLastError());
        charges[panel] = chg3;
        tbegin(PRRP_K_OTHER, sm);
        calu_reorder_kernel<<<1, 1024, 0, sm>>>(cur, ccur, nullptr, 0, bj, rows, col0, pos2row, scratch, mv, mc,
                                                log2phys, st, panel);
        tend(sm);
      } else if (p_eff == 1) {
        // single node: the selector's own full order and l_block (tournament.py:168-177);
        // it IS the LU_PRRP panel, so it runs with LU_PRRP's engine setting
        // (bitwise equal factors, test_caluprrp_single_leaf_equals_luprrp)
        {
          const int keep = tl_lat_cmax;
          tl_lat_cmax = -1;
          strong_rrqr_panel(A + col0, lda, bj, rows, bj, tau, panel, Lg, ldl, Bk, st, swaps_dev, nullptr, nullptr,
                            nullptr, false, sm, pos2row + col0);
          tl_lat_cmax = keep;
        }
        flush_after_main();
        tbegin(PRRP_K_OTHER, sm);
        calu_reorder_kernel<<<1, 1024, 0, sm>>>(nullptr, nullptr, Bk.perm, 1, bj, rows, col0, pos2row, scratch, mv,
                                                mc, log2phys, st, panel);
        tend(sm);
      } else {
        // leaves: contiguous logical blocks, first blocks larger (tournament.py:64-88)
        std::vector<int64_t> lo(p_eff), cnt(p_eff);
        {
          const int64_t base = rows / p_eff, extra = rows % p_eff;
          int64_t start = 0;
          for (int64_t i = 0; i < p_eff; ++i) {
            cnt[i] = base + (i < extra ? 1 : 0);
            lo[i] = start;
            start += cnt[i];
          }
        }
        calu_leaf_lo_kernel<<<1, 64, 0, sm>>>(leaf_lo_dev, p_eff, rows / p_eff, rows % p_eff);
        int64_t chg3 = 0;
        int slot = 0;
        leaf_qrcp_ev.clear();
        run_level(lo, cnt, true, col0, bj, panel, 0, slot, sm);
        if (fin_after_leaf_qrcp && pending_fin) {
          for (cudaEvent_t e : leaf_qrcp_ev) CU_TRY(cudaStreamWaitEvent(sf, e, 0));
          pending_fin();
          pending_fin = nullptr;
        }
        if (early_w2 && pending_side) {
          for (cudaEvent_t e : leaf_qrcp_ev) CU_TRY(cudaStreamWaitEvent(sd, e, 0));
          flush_side(nullptr);
        } else {
          flush_after_main();
        }
        for (cudaEvent_t e : leaf_qrcp_ev) CU_TRY(cudaEventDestroy(e));
        for (int64_t i = 0; i < p_eff; ++i) {
          chg3 += qr_charge3(cnt[i], bj);
          node_members[panel].push_back({cnt[i], slot + (int)i});
        }
        slot += (int)p_eff;
        int32_t* cur = cands;
        int32_t* nxt = cands + (size_t)maxnodes * b;
        int32_t* ccur = ccnt;
        int32_t* cnxt = ccnt + maxnodes;
        calu_select_kernel<<<(unsigned)p_eff, 128, 0, sm>>>(perms_dev, nullptr, leaf_lo_dev, bj, want_all, live_all,
                                                             0, cur, ccur, 2 * b, st);
        int64_t ncur = p_eff;
        int level = 1;
        while (ncur > 1) {
          const int64_t nmerge = ncur / 2;
          // node i of this level reads lpos_all/rowidx_all[i*2b .. i*2b + 2b) (stride 2b even when bj < b);
          // members = [left's candidates, right's candidates], dead (zero) rows after them
          calu_merge_inputs_kernel<<<(unsigned)nmerge, 128, 0, sm>>>(cur, ccur, bj, (int)(2 * nmerge), lpos_all,
                                                                      rowidx_all, live_all, pos2row, col0, 2 * b, st);
          CU_TRY(cudaGetLastError());
          std::vector<int64_t> mlo(nmerge, 0), mcnt(nmerge, 2 * bj);
          root_p = 2 * bj;
          run_level(mlo, mcnt, false, col0, bj, panel, level, slot, sm);
          for (int64_t i = 0; i < nmerge; ++i) {
            chg3 += qr_charge3(2 * bj, bj);
            node_members[panel].push_back({2 * bj, slot + (int)i});
          }
          slot += (int)nmerge;
          calu_select_kernel<<<(unsigned)nmerge, 128, 0, sm>>>(perms_dev, lpos_all, nullptr, bj, want_all, live_all,
                                                                1, nxt, cnxt, 2 * b, st);
          if (ncur % 2) {   // odd node promoted unmerged (tournament.py:197-198)
            CU_TRY(cudaMemcpyAsync(nxt + nmerge * bj, cur + (ncur - 1) * bj, sizeof(int32_t) * bj,
                                   cudaMemcpyDeviceToDevice, sm));
            CU_TRY(cudaMemcpyAsync(cnxt + nmerge, ccur + (ncur - 1), sizeof(int32_t), cudaMemcpyDeviceToDevice, sm));
          }
          ncur = nmerge + (ncur % 2);
          std::swap(cur, nxt);
          std::swap(ccur, cnxt);
          ++level;
        }
        charges[panel] = chg3;
        // new logical order [pivots, rest ascending]; move the pivot rows to slots col0..
        tbegin(PRRP_K_OTHER, sm);
        calu_reorder_kernel<<<1, 1024, 0, sm>>>(cur, ccur, nullptr, 0, bj, rows, col0, pos2row, scratch, mv, mc,
                                                log2phys, st, panel);
        tend(sm);
      }
      if (w1_prev) CU_TRY(cudaStreamWaitEvent(sm, w1_prev, 0));
      const int64_t wn = std::min<int64_t>(width, b);
      tbegin(PRRP_K_PERMUTE, sm);
      permute_cols(col0, col0 + bj + wn, col0, mv, mc, nullptr, panel, sm);
      tend(sm);
      cudaEvent_t ev_perm = ss.ev(evi++);
      CU_TRY(cudaEventRecord(ev_perm, sm));
      if (p_eff > 1) {
        // unpivoted QR of the permuted panel transpose -> multiplier_block (tournament.py:271-272)
        PanelArgs qa{};
        qa.src = blk;
        qa.ld = lda;
        qa.h = bj;
        qa.p = bj;
        qa.bsel = bj;
        qa.steps = bj;
        qa.mode = 1;
        qa.perm = perm_small;
        qa.Rbuf = Rsmall;
        qa.refl = refl;
        qa.ovf = B.ovf;
        const PanelCfg gq = panel_config(bj, bj, bj, true);
        qa.per = gq.per;
        qa.cap = gq.cap;
        qa.cap_pad = gq.cap_pad;
        qa.ovpad = gq.ovpad;
        qa.st = st;
        qa.panel_id = panel;
        tbegin(PRRP_K_FINALIZE, sm);
        iota32_kernel<<<1, 128, 0, sm>>>(perm_small, bj);
        if (reuse_root_qr()) {
          calu_root_qr_kernel<<<16, 256, 0, sm>>>(live_all, bj, nodes[0].B.Rbuf, root_p, nodes[0].B.refl, Rsmall, refl,
                                                 final_live, st);
          qa.live = final_live;   // the engine below runs only when the root passed its members through
        }
        if (team_eligible(bj, bj) && !force_generic_panel()) {
          PanelArgs at = qa;
          at.fro = nodes[0].B.fro;
          launch_team(at, sm);
        } else if (bj == P1_H && ((uintptr_t)blk % 16 == 0) && (lda % 2 == 0) && !force_generic_panel()) {
          // the register engine in fixed-order mode, one CTA (p = b columns)
          PanelCfg g1 = gq;
          g1.C = 1;
          g1.T = P1_T;
          PanelArgs a1 = qa;
          a1.per = bj;
          a1.ovf = B.ovf;
          a1.fro = nodes[0].B.fro;
          launch_cluster(panel_qrcp1_kernel, g1, 0, sm, a1);
        } else if (bj == P2_H && ((uintptr_t)blk % 16 == 0) && (lda % 2 == 0) && !force_generic_panel()) {
          PanelCfg g2 = gq;
          g2.C = 1;
          g2.T = P2_T;
          PanelArgs a2 = qa;
          a2.per = bj;
          a2.ovf = B.ovf;
          a2.fro = nodes[0].B.fro;
          launch_cluster(panel_qrcp2_kernel, g2, (size_t)(P2_H - P2_W) * P2_T * 8, sm, a2);
        } else {
          launch_cluster(panel_qrcp_kernel, gq, gq.dyn_engine, sm, qa);
        }
        calu_copy_r11_kernel<<<16, 256, 0, sm>>>(Rsmall, bj, B.Rbuf, rows);
        static const int r12_min_b = getenv("PRRP_CALU_R12_MIN_B") ? atoi(getenv("PRRP_CALU_R12_MIN_B")) : 65;
        if (calu_r12_gemm && bj >= r12_min_b && (bj % 2 == 0)) {
          // R12 = Q^T A21^T on the DMMA pipe: Q from the reflector log, A21's
          // rows gathered transposed, C = 0 - (-Q^T) A21^T (the reflectors'
          // sequential application and this product agree to a few ulps; the
          // reference's own dgemv order is not reproducible either)
          const int64_t ncol = rows - bj;
          tend(sm);
          tbegin(PRRP_K_OTHER, sm);
          calu_form_negqt_kernel<<<(bj + 15) / 16, 128, (size_t)bj * (bj + 1) * 8, sm>>>(refl, bj, Qneg);
          tend(sm);
          tbegin(PRRP_K_PERMUTE, sm);
          calu_gather_t_kernel<<<(unsigned)((ncol + 31) / 32), 256, (size_t)bj * 33 * 8, sm>>>(
              A, lda, col0, bj, ncol, pos2row + col0 + bj, A21t, ld21t, st);
          zero2d_kernel<<<(unsigned)std::min<int64_t>(4 * sms, (ncol * bj + 255) / 256), 256, 0, sm>>>(
              B.Rbuf + bj, rows, bj, ncol);
          tend(sm);
          schur_update(B.Rbuf + bj, rows, Qneg, bj, A21t, ld21t, bj, ncol, bj, st_r12, sm, 0, 0);
          tbegin(PRRP_K_FINALIZE, sm);
        } else {
        const size_t dyn = (size_t)bj * (bj + 1) * 8;
        const unsigned grid = (unsigned)std::min<int64_t>(sms * 4, (rows - bj + 7) / 8);
        switch ((bj + 31) / 32) {
          case 1: calu_apply_refl_kernel<1><<<grid, 256, dyn, sm>>>(A, lda, col0, bj, rows, pos2row, refl, B.Rbuf, st); break;
          case 2: calu_apply_refl_kernel<2><<<grid, 256, dyn, sm>>>(A, lda, col0, bj, rows, pos2row, refl, B.Rbuf, st); break;
          case 3: calu_apply_refl_kernel<3><<<grid, 256, dyn, sm>>>(A, lda, col0, bj, rows, pos2row, refl, B.Rbuf, st); break;
          default: calu_apply_refl_kernel<4><<<grid, 256, dyn, sm>>>(A, lda, col0, bj, rows, pos2row, refl, B.Rbuf, st); break;
        }
        }
        CU_TRY(cudaGetLastError());
        tend(sm);
        tbegin(PRRP_K_TRSM, sm);
        const int64_t ncol = rows - bj;
        double* fro_inf = nodes[0].B.fro;   // rank check of the final QR: the reference has none (fro = 0)
        CU_TRY(cudaMemsetAsync(fro_inf, 0, sizeof(double), sm));
        int nblk;
        if (bj <= 64 || use_trsm_c2()) {
          // b > 64, beside the trailing update (few free SMs): 4 column groups
          // per CTA amortise the 133 KB R11 staging
          const int64_t cpb = bj <= 64 ? TC_COLS : 4 * TC_COLS;
          nblk = (int)std::min<int64_t>(kMaxCand, (ncol + cpb - 1) / cpb);
          if (bj <= 64)
            trsm_c_kernel<<<nblk, TC_T, 0, sm>>>(B.Rbuf, rows, bj, Lg, ldl, B.cand, B.cand_flat, st, panel, fro_inf, -1, -1, nullptr, nullptr);
          else
            trsm_c2_kernel<<<nblk, TC_T, kTrsmC2Smem, sm>>>(B.Rbuf, rows, bj, Lg, ldl, B.cand, B.cand_flat, st, panel,
                                                            fro_inf, -1, -1, nullptr, nullptr);
        } else {
          nblk = (int)std::min<int64_t>(kMaxCand, (ncol + TTC - 1) / TTC);
          const size_t tdyn = (((size_t)bj * (bj + 1) / 2 + 1) / 2 * 2 + (size_t)bj * TTCP) * 8;
          switch ((bj + 31) / 32) {
            case 3: trsm_w_kernel<3><<<nblk, TW_WARPS * 32, tdyn, sm>>>(B.Rbuf, rows, bj, Lg, ldl, B.cand, B.cand_flat, st, panel, fro_inf, -1, -1, nullptr, nullptr); break;
            default: trsm_w_kernel<4><<<nblk, TW_WARPS * 32, tdyn, sm>>>(B.Rbuf, rows, bj, Lg, ldl, B.cand, B.cand_flat, st, panel, fro_inf, -1, -1, nullptr, nullptr); break;
          }
        }
        calu_stats_kernel<<<1, 256, 0, sm>>>(B.cand, nblk, node_swaps + (size_t)panel * maxnodes, maxnodes,
                                             swaps_dev, panel, st);
        tend(sm);
        CU_TRY(cudaGetLastError());
      }
      // L21 (logical order) -> physical slots for the Schur update and the compose
      calu_scatter_l21_kernel<<<sms * 4, 256, 0, sm>>>(Lg, ldl, log2phys, rows - bj, bj, bj, Lp, ldl, st);
      // the updates read the pivot rows (A12 before the GEPP finish) from a
      // copy, so the block row can be finished on the fin stream while the
      // trailing update is still running
      double* a12 = a12cb[par];
      if (wn > 0)
        CU_TRY(cudaMemcpy2DAsync(a12, (size_t)lda12 * 8, A + col0 * lda + col0 + bj, (size_t)lda * 8, (size_t)wn * 8,
                                 (size_t)bj, cudaMemcpyDeviceToDevice, sm));
      if (wn > 0)
        schur_update(A + (col0 + bj) * lda + col0 + bj, lda, Lp, ldl, a12, lda12, rows - bj, wn,
                     bj, st, sm, calu_narrow_ctas, calu_wide_q);
      cudaEvent_t ev_narrow = ss.ev(evi++);
      CU_TRY(cudaEventRecord(ev_narrow, sm));
      // fin: L-part row moves + row order, GEPP, compose, then (after every
      // row move of this panel and the pivot-row copy; side's permute also
      // orders it after the previous trailing update) the block row
      fin_ev[panel] = ss.ev(evi++);
      cudaEvent_t fin_done = fin_ev[panel];
      cudaEvent_t ev_copy = ss.ev(evi++);
      // the L-part row moves and the GEPP of the pivot block need only this
      // panel's row moves (ev_perm), not its L21: PRRP_CALU_GEPP_EARLY=1 starts
      // them before the final QR / narrow update (less fin-stream work left
      // when the next panel's leaf clusters look for SMs).  Measured neutral
      // (config 5 1150.6 vs 1152.5 ms, config 4 260.5 vs 257.8 ms), so off.
      static const bool gepp_early = getenv("PRRP_CALU_GEPP_EARLY") && atoi(getenv("PRRP_CALU_GEPP_EARLY")) != 0;
      static const int side_delay_us = getenv("PRRP_CALU_SIDE_DELAY_US") ? atoi(getenv("PRRP_CALU_SIDE_DELAY_US")) : 0;
      pending_fin = [=]() {
        CU_TRY(cudaStreamWaitEvent(sf, gepp_early ? ev_perm : ev_narrow, 0));
        if (side_delay_us > 0 && !gepp_early) spin_delay_kernel<<<1, 32, 0, sf>>>((unsigned)side_delay_us);
        tbegin(PRRP_K_PERMUTE, sf);
        permute_cols(0, col0, col0, mv, mc, perm, panel, sf);
        tend(sf);
        tbegin(PRRP_K_GEPP, sf);
        launch_gepp(blk, lda, nullptr, bj, Dk, pivk, gpk, st, panel, sf);
        tend(sf);
        if (gepp_early) CU_TRY(cudaStreamWaitEvent(sf, ev_narrow, 0));
        tbegin(PRRP_K_COMPOSE, sf);
        launch_compose_w(Lp, ldl, rows - bj, bj, Dk, gpk, A + (col0 + bj) * lda + col0, lda, st, sf, &cws);
        tend(sf);
        CU_TRY(cudaStreamWaitEvent(sf, ev_copy, 0));
        tbegin(PRRP_K_BLOCKROW, sf);
        launch_blockrow_w(A, lda, col0, bj, n, Dk, gpk, perm, st, sf);
        tend(sf);
        CU_TRY(cudaGetLastError());
        CU_TRY(cudaEventRecord(fin_done, sf));
      };
      // side: trailing row moves + copy of their pivot-row part, trailing
      // update (next narrow region first)
      CU_TRY(cudaStreamWaitEvent(sd, ev_narrow, 0));
      if (side_delay_us > 0) spin_delay_kernel<<<1, 32, 0, sd>>>((unsigned)side_delay_us);
      const int64_t cw0 = col0 + bj + wn;
      tbegin(PRRP_K_PERMUTE, sd);
      permute_cols(cw0, n, col0, mv, mc, nullptr, panel, sd);
      if (n > cw0)
        CU_TRY(cudaMemcpy2DAsync(a12 + wn, (size_t)lda12 * 8, A + col0 * lda + cw0, (size_t)lda * 8,
                                 (size_t)(n - cw0) * 8, (size_t)bj, cudaMemcpyDeviceToDevice, sd));
      tend(sd);
      CU_TRY(cudaEventRecord(ev_copy, sd));
      if (!((sb_serial & 6) && calu_defer && b > 64 && !chain_bound(panel + 1))) {
        pending_fin();
        pending_fin = nullptr;
      }
      const int64_t w1 = std::min<int64_t>(n - cw0, b);
      if (w1 > 0)
      {
        static const int fw1 = getenv("PRRP_WS_W1") ? atoi(getenv("PRRP_WS_W1")) : -1;
        tl_force_ws = fw1;
        static const int w1_ctas = getenv("PRRP_CALU_W1_CTAS") ? atoi(getenv("PRRP_CALU_W1_CTAS")) : 0;
        // PRRP_CALU_W1_CTAS < 0: the classic one-tile-per-CTA kernel (short CTAs)
        schur_update(A + (col0 + bj) * lda + cw0, lda, Lp, ldl, a12 + wn, lda12, rows - bj, w1, bj, st, sd,
                     w1_ctas > 0 ? w1_ctas : (w1_ctas < 0 ? 0 : calu_wide_ctas), w1_ctas < 0 ? 0 : calu_wide_q);
        tl_force_ws = -1;
      }
      w1_prev = ss.ev(evi++);
      CU_TRY(cudaEventRecord(w1_prev, sd));
      // the rest of the trailing update (W2): deferred until the next panel's
      // tournament leaves have run (see pending_side)
      pending_side = [=, &ss, &evi, &side_done, &side_ev]() {
        if (n - cw0 > w1)
        {
          static const int fw2 = getenv("PRRP_WS_W2") ? atoi(getenv("PRRP_WS_W2")) : -1;
          tl_force_ws = fw2;
          const bool cb = chain_bound(panel + 1);   // it runs beside panel + 1's merge levels
          tl_schur_cluster = cb ? 16 : 0;
          schur_update(A + (col0 + bj) * lda + cw0 + w1, lda, Lp, ldl, a12 + wn + w1, lda12, rows - bj,
                       n - cw0 - w1, bj, st, sd, cb ? 16 * w2_clusters : calu_wide_ctas, calu_wide_q, w2_stream);
          tl_schur_cluster = 0;
          tl_force_ws = -1;
        }
        side_done = ss.ev(evi++);
        CU_TRY(cudaEventRecord(side_done, sd));
        side_ev[panel] = side_done;
      };
      if (!calu_defer) flush_side(nullptr);
      continue;
    } else {
      flush_side(nullptr);
      if (panel >= 1 && fin_ev[panel - 1]) CU_TRY(cudaStreamWaitEvent(sd, fin_ev[panel - 1], 0));
      // last square block: logical order (all columns, on the side stream, which
      // has seen every earlier update and row move), then GEPP
      tbegin(PRRP_K_OTHER, sd);
      calu_reorder_kernel<<<1, 1024, 0, sd>>>(nullptr, nullptr, ident, 1, bj, rows, col0, pos2row, scratch, mv, mc,
                                              log2phys, st, panel);
      tend(sd);
      tbegin(PRRP_K_PERMUTE, sd);
      permute_cols(0, n, col0, mv, mc, perm, panel, sd);
      tend(sd);
      tbegin(PRRP_K_GEPP, sd);
      launch_gepp(blk, lda, nullptr, bj, Dk, pivk, gpk, st, panel, sd);
      tend(sd);
    }
    CU_TRY(cudaGetLastError());
    tbegin(PRRP_K_BLOCKROW, sd);
    launch_blockrow_w(A, lda, col0, bj, n, Dk, gpk, perm, st, sd);
    tend(sd);
    CU_TRY(cudaGetLastError());
    side_done = ss.ev(evi++);
    CU_TRY(cudaEventRecord(side_done, sd));
    side_ev[panel] = side_done;
  }
  flush_side(nullptr);
  CU_TRY(cudaStreamWaitEvent(sm, side_done, 0));
  for (int k = npanels - 1; k >= 0; --k)      // join the fin stream (its last block row)
    if (fin_ev[k]) { CU_TRY(cudaStreamWaitEvent(sm, fin_ev[k], 0)); break; }
  {
    cudaEvent_t e1 = ss.ev(evi++);
    CU_TRY(cudaEventRecord(e1, sm));
    CU_TRY(cudaStreamWaitEvent(s, e1, 0));
  }
  if (m > n) {
    // unfinished tail rows n..m-1 into logical order
    double* tmp = ar.get<double>((size_t)(m - n) * n);
    int64_t* ptmp = ar.get<int64_t>(m - n);
    calu_tail_gather_kernel<<<sms * 4, 256, 0, s>>>(A, lda, n, pos2row, m, tmp, perm, ptmp);
    CU_TRY(cudaMemcpy2DAsync(A + n * lda, lda * 8, tmp, n * 8, n * 8, m - n, cudaMemcpyDeviceToDevice, s));
    CU_TRY(cudaMemcpyAsync(perm + n, ptmp, sizeof(int64_t) * (m - n), cudaMemcpyDeviceToDevice, s));
  }
  out.st = st;
  out.swaps_dev = swaps_dev;
  out.node_swaps = node_swaps;
  out.node_rows = node_rows;
  out.n = n;
  out.charges = std::move(charges);
  out.node_members = std::move(node_members);
  out.npanels = npanels;
  out.maxnodes = maxnodes;
  out.b = b;
}

// A captured CALU_PRRP factorization for one (matrix, shape, parameters) key:
// replayed by one graph launch (the host enqueue of the ~10^4 launches of a
// large factorization costs more than the GPU work at n = 16384).
struct CaluPlan {
  double* A; int64_t lda, m, n; int b; double tau; int P; int64_t* perm; int dev;
  int64_t kernel_nodes = 0;   // kernel launches in the captured graph (the bench's gpu_launches)
  cudaGraphExec_t exec = nullptr;
  std::vector<void*> bufs;
  CaluOut out;
  uint64_t used = 0;
  ~CaluPlan() {
    if (exec) cudaGraphExecDestroy(exec);
    for (void* p : bufs) cudaFree(p);
  }
};
thread_local int64_t tl_last_graph_kernels = 0;
std::vector<std::shared_ptr<CaluPlan>>& calu_plans() {
  static std::vector<std::shared_ptr<CaluPlan>> v;
  return v;
}
uint64_t g_plan_clock = 0;

int caluprrp_finish(const CaluOut& out, cudaStream_t s, int32_t* swap_counts, int64_t* tchg3, prrp_stats* stats,
                    prrp_err* err, std::chrono::steady_clock::time_point host_t0, Timer* timer);

std::mutex g_plans_mu;   // the plan cache is shared by the host threads of the process

#ifdef PRRP_SCHUR_RACECHECK
// diagnostics build: the warp-specialised Schur kernel records C elements that
// changed between the start of their tile and its epilogue
void racecheck_begin(const double* A, int64_t lda) {
  static int zeros[2 + 4 * 64] = {0};
  long long ld = lda;
  CU_TRY(cudaMemcpyToSymbol(g_racecheck, zeros, sizeof(zeros)));
  CU_TRY(cudaMemcpyToSymbol(g_race_base, &A, sizeof(A)));
  CU_TRY(cudaMemcpyToSymbol(g_race_ld, &ld, sizeof(ld)));
}
void racecheck_end() {
  int h[2 + 4 * 64];
  CU_TRY(cudaMemcpyFromSymbol(h, g_racecheck, sizeof(h)));
  fprintf(stderr, "[racecheck] %d changed C elements\n", h[0]);
  for (int i = 0; i < std::min(h[0], 64); ++i)
    fprintf(stderr, "  row %d col %d (M %d N %d)\n", h[2 + 4 * i], h[3 + 4 * i], h[4 + 4 * i], h[5 + 4 * i]);
}
#else
void racecheck_begin(const double*, int64_t) {}
void racecheck_end() {}
#endif

int caluprrp_impl(double* A, int64_t lda, int64_t m, int64_t n, int b, double tau, int P, int64_t* perm,
                  int32_t* swap_counts, int64_t* tchg3, prrp_stats* stats, prrp_err* err, cudaStream_t s,
                  prrp_timing* timing = nullptr) {
  if (m < n) fail(PRRP_ERR_DIM, "need at least as many rows as columns");
  if (b < 1 || b > n) fail(PRRP_ERR_ARG, "panel width out of range");
  if (!(tau > 1.0)) fail(PRRP_ERR_ARG, "tau must exceed 1");
  if (P < 0) fail(PRRP_ERR_ARG, "binary tree needs a leaf count >= 1 (0 selects the flat tree)");
  if (b > PRRP_MAXH) fail(PRRP_ERR_UNSUPPORTED, "panel width > 128 is outside the device panel engine");
  if (lda < n) fail(PRRP_ERR_ARG, "lda < n");
  caps();
  racecheck_begin(A, lda);
  const auto host_t0 = std::chrono::steady_clock::now();
  // PRRP_TRACE: record the timing spans (and write the trace file) for CALU too
  if (timing || getenv("PRRP_TRACE") || (getenv("PRRP_GRAPH") && atoi(getenv("PRRP_GRAPH")) == 0)) {
    // direct enqueue; with `timing` (or PRRP_TRACE) every launch is bracketed
    // by events on its stream and summed per kernel class
    Timer timer;
    tl_timer = (timing || getenv("PRRP_TRACE")) ? &timer : nullptr;
    tl_schur_flops = 0.0;
    struct Reset { ~Reset() { tl_timer = nullptr; } } reset_timer;
    Arena ar(s);
    CaluOut out;
    caluprrp_enqueue(A, lda, m, n, b, tau, P, perm, s, ar, out);
    const int rc = caluprrp_finish(out, s, swap_counts, tchg3, stats, err, host_t0, timing ? nullptr : tl_timer);
    if (timing) {
      timer.collect(timing);
      timing->schur_flops = tl_schur_flops;
    }
    return rc;
  }
  int dev = 0;
  CU_TRY(cudaGetDevice(&dev));
  std::unique_lock<std::mutex> plans_lock(g_plans_mu);
  auto& plans = calu_plans();
  CaluPlan* pl = nullptr;
  for (auto& q : plans)
    if (q->A == A && q->lda == lda && q->m == m && q->n == n && q->b == b && q->tau == tau && q->P == P &&
        q->perm == perm && q->dev == dev)
      pl = q.get();
  if (!pl) {
    // A key seen for the first time is enqueued directly: the GPU starts at
    // once while the host is still enqueuing (capture + instantiate first
    // would put ~1 s of host work in front of a one-shot call, e.g. the end-
    // to-end path on a fresh buffer).  The second call with the same key
    // captures the plan, later ones replay it (PRRP_GRAPH_EAGER=1: capture
    // at the first call).
    static const bool eager = getenv("PRRP_GRAPH_EAGER") && atoi(getenv("PRRP_GRAPH_EAGER")) != 0;
    struct SeenKey { double* A; int64_t lda, m, n; int b; double tau; int P; int64_t* perm; int dev; };
    static std::vector<SeenKey> seen;     // guarded by g_plans_mu
    bool known = eager;
    for (const auto& k : seen)
      known = known || (k.A == A && k.lda == lda && k.m == m && k.n == n && k.b == b && k.tau == tau && k.P == P &&
                        k.perm == perm && k.dev == dev);
    if (!known) {
      if (seen.size() >= 16) seen.erase(seen.begin());
      seen.push_back(SeenKey{A, lda, m, n, b, tau, P, perm, dev});
      plans_lock.unlock();
      tl_schur_flops = 0.0;
      Arena ar(s);
      CaluOut out;
      caluprrp_enqueue(A, lda, m, n, b, tau, P, perm, s, ar, out);
      return caluprrp_finish(out, s, swap_counts, tchg3, stats, err, host_t0, nullptr);
    }
    if (plans.size() >= kMaxPlans) {
      auto lru = std::min_element(plans.begin(), plans.end(),
                                  [](const std::shared_ptr<CaluPlan>& x, const std::shared_ptr<CaluPlan>& y) {
                                    // plans held by an in-flight call (use_count > 1) are never evicted
                                    return (x.use_count() > 1 ? UINT64_MAX : x->used) <
                                           (y.use_count() > 1 ? UINT64_MAX : y->used);
                                  });
      if (lru->use_count() == 1) {          // idle: its last call has read its results back
        CU_TRY(cudaDeviceSynchronize());
        plans.erase(lru);
      }
    }
    std::shared_ptr<CaluPlan> np(new CaluPlan{A, lda, m, n, b, tau, P, perm, dev});
    // capture on a private stream (the caller's may be the legacy stream)
    static thread_local cudaStream_t cs = nullptr;
    if (!cs) CU_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    const int npan = (int)((n + b - 1) / b);
    tl_sched_slots = (unsigned)(4 * npan + 64);
    int* sched = nullptr;
    CU_TRY(cudaMalloc(&sched, sizeof(int) * 2 * tl_sched_slots));
    np->bufs.push_back(sched);
    CU_TRY(cudaMemset(sched, 0, sizeof(int) * 2 * tl_sched_slots));
    tl_sched = getenv("PRRP_GRAPH_GLOBAL_SCHED") ? nullptr : sched;
    tl_sched_next = 0;
    cudaGraph_t g = nullptr;
    CU_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
    try {
      Arena ar(cs, &np->bufs);
      caluprrp_enqueue(A, lda, m, n, b, tau, P, perm, cs, ar, np->out);
    } catch (...) {
      tl_sched = nullptr;
      cudaStreamEndCapture(cs, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    tl_sched = nullptr;
    CU_TRY(cudaStreamEndCapture(cs, &g));
    if (const char* dot = getenv("PRRP_GRAPH_DOT"))   // diagnostics: the captured dependency graph
      cudaGraphDebugDotPrint(g, dot, cudaGraphDebugDotFlagsVerbose);
    {
      size_t nn = 0;
      CU_TRY(cudaGraphGetNodes(g, nullptr, &nn));
      std::vector<cudaGraphNode_t> gn(nn);
      if (nn) CU_TRY(cudaGraphGetNodes(g, gn.data(), &nn));
      for (auto nd : gn) {
        cudaGraphNodeType ty;
        CU_TRY(cudaGraphNodeGetType(nd, &ty));
        np->kernel_nodes += ty == cudaGraphNodeTypeKernel;
      }
    }
    const cudaError_t ie = cudaGraphInstantiate(&np->exec, g, graph_instantiate_flags());
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) fail(PRRP_ERR_CUDA, "cudaGraphInstantiate failed");
    plans.push_back(std::move(np));
    pl = plans.back().get();
  }
  pl->used = ++g_plan_clock;
  tl_last_graph_kernels = pl->kernel_nodes;
  // the read-back runs outside the cache lock and reads the plan's buffers:
  // hold a reference so the plan cannot be evicted (freed) before it is done
  std::shared_ptr<CaluPlan> hold;
  for (auto& q : plans)
    if (q.get() == pl) hold = q;
  CU_TRY(cudaGraphLaunch(pl->exec, s));
  const CaluOut out = pl->out;
  plans_lock.unlock();
  const int rc = caluprrp_finish(out, s, swap_counts, tchg3, stats, err, host_t0, nullptr);
  std::lock_guard<std::mutex> relock(g_plans_mu);
  hold.reset();
  return rc;
}

int caluprrp_finish(const CaluOut& out, cudaStream_t s, int32_t* swap_counts, int64_t* tchg3, prrp_stats* stats,
                    prrp_err* err, std::chrono::steady_clock::time_point host_t0, Timer* timer) {
  const int npanels = out.npanels, maxnodes = out.maxnodes, b = out.b;
  const auto& charges = out.charges;
  const auto& node_members = out.node_members;
  const auto host_t1 = std::chrono::steady_clock::now();
  DevState hs;
  read_state(out.st, hs, s);
  if (getenv("PRRP_HOSTTIME")) {
    const auto host_t2 = std::chrono::steady_clock::now();
    fprintf(stderr, "[prrp calu host] enqueue %.3f ms, then wait %.3f ms\n",
            std::chrono::duration<double, std::milli>(host_t1 - host_t0).count(),
            std::chrono::duration<double, std::milli>(host_t2 - host_t1).count());
  }
  int32_t* swaps_dev = out.swaps_dev;
  int32_t* node_swaps = out.node_swaps;
  racecheck_end();
  std::vector<int32_t> sw(npanels);
  CU_TRY(cudaMemcpy(sw.data(), swaps_dev, sizeof(int32_t) * npanels, cudaMemcpyDeviceToHost));
  std::vector<int32_t> nsw((size_t)npanels * maxnodes), nrows((size_t)npanels * maxnodes);
  CU_TRY(cudaMemcpy(nsw.data(), node_swaps, sizeof(int32_t) * nsw.size(), cudaMemcpyDeviceToHost));
  CU_TRY(cudaMemcpy(nrows.data(), out.node_rows, sizeof(int32_t) * nrows.size(), cudaMemcpyDeviceToHost));
  if (swap_counts) memcpy(swap_counts, sw.data(), sizeof(int32_t) * npanels);
  if (tchg3) {
    // _tournament_charges (tournament.py:224-234): nodes of more than b members,
    // (1 + swaps) x _charge_qr(members, b); member counts as the device saw them
    // (a merge node shrinks when a child was rank deficient)
    for (int k = 0; k < npanels; ++k) {
      if (charges[k] < 0) { tchg3[k] = -1; continue; }
      const int bk = (int)std::min<int64_t>(b, out.n - (int64_t)k * b);
      int64_t c3 = 0;
      for (auto& mm : node_members[k]) {
        const int64_t r = nrows[(size_t)k * maxnodes + mm.second];
        if (r > bk) c3 += (1 + nsw[(size_t)k * maxnodes + mm.second]) * qr_charge3(r, bk);
      }
      tchg3[k] = c3;
    }
  }
  fill_stats(hs, stats);
  if (stats) {
    stats->total_swaps = 0;
    for (int v : sw) stats->total_swaps += v;
  }
  if (getenv("PRRP_HOSTTIME"))
    fprintf(stderr, "[prrp calu host] stats done at %.3f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count());
  if (timer) {
    prrp_timing tm;
    timer->collect(&tm);
    fprintf(stderr, "[prrp calu timing] total %.3f ms:", tm.total_ms);
    for (int c = 0; c < PRRP_K_COUNT; ++c) fprintf(stderr, " %d:%.3f", c, tm.ms[c]);
    fprintf(stderr, "\n");
  }
  return state_to_err(hs, err);
}


// ---------------------------------------------------------------- calu_factor
// Tournament-pivoted GEPP (tournament.py:299-359), one stream.  Per panel:
// GEPP tournament (one launch per tree level, one CTA per node), row order of
// the trailing rows, row moves, GEPP finish of the block row (the LU_PRRP
// kernels, no compose), L21 = A21 U11^-1, DMMA trailing update.
constexpr int kGnSmem = 160 * 1024;

struct GeppTourBufs {
  double* wscratch;
  int32_t* oscratch;
  int32_t* cand[2];
  int32_t* cnt[2];
  int32_t* order_full;
  int32_t* mark;
  int32_t* perm_rel;
};

// Levels of one panel's tournament; returns the buffer index holding the root.
int gepp_tournament(const double* panel, int64_t lda, int bj, int64_t rows, int P, const GeppTourBufs& T,
                    unsigned long long* chg3, DevState* st, int panel_no, bool& single, cudaStream_t s) {
  GeppLevel g{};
  g.panel = panel; g.lda = lda; g.bj = bj; g.rows = rows;
  g.wscratch = T.wscratch; g.oscratch = T.oscratch; g.chg3 = chg3; g.st = st; g.panel_no = panel_no;
  // block size: column-warps x row groups, ~8 rows per thread per step
  // (measured on B200: 32 rows per thread with 4x fewer warps is slower --
  // the 64 dependent steps are latency-bound, not issue-bound)
  auto threads_for = [&](int64_t r) -> unsigned {
    const int cw = (bj + 31) & ~31;
    const int64_t rg = std::max<int64_t>(1, std::min<int64_t>((r + 7) / 8, GN_T / cw));
    return (unsigned)(cw * rg);
  };
  auto launch_node = [&](unsigned grid, unsigned threads) {
    if (g.smem_bytes > 0) gepp_node_kernel<true><<<grid, threads, g.smem_bytes, s>>>(g);
    else gepp_node_kernel<false><<<grid, threads, 0, s>>>(g);
  };
  auto smem_for = [&](int64_t r) -> int {
    const size_t need = (size_t)r * bj * 8 + (size_t)r * 4;
    return need <= (size_t)kGnSmem ? (int)((need + 15) / 16 * 16) : 0;
  };
  int cur = 0;
  if (P > 0) {
    const int64_t p_eff = std::max<int64_t>(1, std::min<int64_t>(P, rows / (bj + 1)));
    single = p_eff == 1;
    g.mode = 0; g.p_eff = p_eff;
    g.cand_out = T.cand[0]; g.cnt_out = T.cnt[0];
    g.order_full = single ? T.order_full : nullptr;
    g.smem_bytes = smem_for((rows + p_eff - 1) / p_eff);
    launch_node((unsigned)p_eff, threads_for((rows + p_eff - 1) / p_eff));
    CU_TRY(cudaGetLastError());
    g.order_full = nullptr;
    int64_t ncur = p_eff;
    while (ncur > 1) {
      const int64_t nout = (ncur + 1) / 2;
      g.mode = 1; g.nprev = ncur;
      g.cand_in = T.cand[cur]; g.cnt_in = T.cnt[cur];
      g.cand_out = T.cand[cur ^ 1]; g.cnt_out = T.cnt[cur ^ 1];
      g.smem_bytes = smem_for(2 * bj);
      launch_node((unsigned)nout, threads_for(2 * bj));
      CU_TRY(cudaGetLastError());
      cur ^= 1;
      ncur = nout;
    }
    return cur;
  }
  const int64_t first = std::min<int64_t>(rows, 2 * bj);
  single = first >= rows;
  g.mode = 2; g.hi = first;
  g.cand_out = T.cand[0]; g.cnt_out = T.cnt[0];
  g.order_full = single ? T.order_full : nullptr;
  g.smem_bytes = smem_for(first);
  launch_node(1, threads_for(first));
  CU_TRY(cudaGetLastError());
  g.order_full = nullptr;
  for (int64_t lo = first; lo < rows; lo += bj) {
    g.mode = 3; g.lo = lo; g.hi = std::min<int64_t>(rows, lo + bj);
    g.cand_in = T.cand[cur]; g.cnt_in = T.cnt[cur];
    g.cand_out = T.cand[cur ^ 1]; g.cnt_out = T.cnt[cur ^ 1];
    g.smem_bytes = smem_for(2 * bj);
    launch_node(1, threads_for(2 * bj));
    CU_TRY(cudaGetLastError());
    cur ^= 1;
  }
  return cur;
}

GeppTourBufs alloc_tour(Arena& ar, int64_t m, int b, int P) {
  GeppTourBufs T{};
  const int64_t nodes = std::max(P, 1) + 1;
  T.wscratch = ar.get<double>((size_t)(m + 2 * b * nodes) * b);
  T.oscratch = ar.get<int32_t>((size_t)(m + 2 * b * nodes));
  for (int i = 0; i < 2; ++i) {
    T.cand[i] = ar.get<int32_t>((size_t)nodes * b);
    T.cnt[i] = ar.get<int32_t>((size_t)nodes);
  }
  T.order_full = ar.get<int32_t>(m);
  T.mark = ar.get<int32_t>(m);
  T.perm_rel = ar.get<int32_t>(m);
  return T;
}

int calu_gepp_impl(double* A, int64_t lda, int64_t m, int64_t n, int b, int P, int64_t* perm, int64_t* chg3_out,
                   prrp_stats* stats, prrp_err* err, cudaStream_t s) {
  if (m < n) fail(PRRP_ERR_DIM, "need at least as many rows as columns");
  if (b < 1 || b > n) fail(PRRP_ERR_ARG, "panel width out of range");
  if (P < 0) fail(PRRP_ERR_ARG, "binary tree needs a leaf count >= 1 (0 selects the flat tree)");
  if (b > PRRP_MAXH) fail(PRRP_ERR_UNSUPPORTED, "panel width > 128 is outside the device path");
  if (lda < n) fail(PRRP_ERR_ARG, "lda < n");
  if (m > INT32_MAX) fail(PRRP_ERR_UNSUPPORTED, "more than 2^31 rows");
  caps();
  const int sms = caps().sms;
  const int npanels = (int)((n + b - 1) / b);
  Arena ar(s);
  DevState* st = new_state(ar, s);
  const int64_t ldl = ((m + 7) / 8) * 8;
  double* Lcm = ar.get<double>((size_t)b * ldl);
  GeppTourBufs T = alloc_tour(ar, m, b, P);
  // row-move staging in column chunks: a fixed ~128 MiB budget (most rows of
  // the trailing region move under the stable [pivots, rest] partition, so
  // the staging is sized by rows x chunk, not by the moved-row count)
  const int64_t cw = std::min<int64_t>(n, std::max<int64_t>(256, std::min<int64_t>(2048, (int64_t)(16 << 20) / m)));
  double* rbuf = ar.get<double>((size_t)m * cw);
  int64_t* pbuf = ar.get<int64_t>(m);
  double* D = ar.get<double>((size_t)b * b);
  int32_t* piv = ar.get<int32_t>(b);
  int32_t* gperm = ar.get<int32_t>(b);
  unsigned long long* chg3 = ar.get<unsigned long long>(npanels);
  CU_TRY(cudaMemsetAsync(chg3, 0, sizeof(unsigned long long) * npanels, s));
  iota_kernel<<<sms, 256, 0, s>>>(perm, m);
  maxabs_kernel<<<sms * 4, 256, 0, s>>>(A, lda, m, n, st);
  CU_TRY(cudaGetLastError());
  int panel = 0;
  for (int64_t col0 = 0; col0 < n; col0 += b, ++panel) {
    const int bj = (int)std::min<int64_t>(b, n - col0);
    const int64_t rows = m - col0;
    const int64_t width = n - col0 - bj;
    double* blk = A + col0 * lda + col0;
    if (rows > bj) {
      bool single = false;
      const int root = gepp_tournament(blk, lda, bj, rows, P, T, chg3 + panel, st, panel, single, s);
      gepp_tail_order_kernel<<<1, 1024, 0, s>>>(T.cand[root], T.cnt[root], bj, rows,
                                                single ? T.order_full : nullptr, T.mark, T.perm_rel, st, panel);
      const unsigned pg = (unsigned)std::min<int64_t>(rows, 8 * sms);
      for (int64_t c0 = 0; c0 < n; c0 += cw) {
        const int64_t c1 = std::min<int64_t>(n, c0 + cw);
        tail_gather_kernel<<<pg, 256, 0, s>>>(A, lda, col0, rows, c0, c1, T.perm_rel, perm, rbuf,
                                              c0 == 0 ? pbuf : nullptr, st);
        tail_scatter_kernel<<<pg, 256, 0, s>>>(A, lda, col0, rows, c0, c1, T.perm_rel, perm, rbuf,
                                               c0 == 0 ? pbuf : nullptr, st);
      }
      CU_TRY(cudaGetLastError());
      launch_gepp(blk, lda, nullptr, bj, D, piv, gperm, st, panel, s);
      launch_blockrow_w(A, lda, col0, bj, n, D, gperm, perm, st, s);
      CU_TRY(cudaGetLastError());
      const int64_t M = rows - bj;
      const int tw = 64;
      const size_t dyn = ((size_t)bj * bj + (size_t)bj * tw) * 8;
      const unsigned tg = (unsigned)std::max<int64_t>(1, std::min<int64_t>((M + tw - 1) / tw, 8 * sms));
      if (bj <= 64)
        trsm_right_reg_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((M + 127) / 128, 8 * sms)), 128, 0,
                                s>>>(A, lda, col0, bj, col0 + bj, M, Lcm, ldl, st);
      else
        trsm_right_kernel<<<tg, tw, dyn, s>>>(A, lda, col0, bj, col0 + bj, M, Lcm, ldl, st);
      CU_TRY(cudaGetLastError());
      if (width > 0)
        schur_update(A + (col0 + bj) * lda + col0 + bj, lda, Lcm, ldl, A + col0 * lda + col0 + bj, lda, M, width,
                     bj, st, s, sms);
    } else {
      launch_gepp(blk, lda, nullptr, bj, D, piv, gperm, st, panel, s);
      launch_blockrow_w(A, lda, col0, bj, n, D, gperm, perm, st, s);
      CU_TRY(cudaGetLastError());
    }
  }
  DevState hs;
  read_state(st, hs, s);
  if (chg3_out) {
    std::vector<unsigned long long> c(npanels);
    CU_TRY(cudaMemcpy(c.data(), chg3, sizeof(unsigned long long) * npanels, cudaMemcpyDeviceToHost));
    for (int k = 0; k < npanels; ++k) chg3_out[k] = (int64_t)c[k];
  }
  fill_stats(hs, stats);
  if (stats) stats->total_swaps = 0;
  return state_to_err(hs, err);
}

// One GEPP selector node over r rows (tournament.py:142-150): order[0..r) and
// the number of rows chosen before the first zero pivot.
int gepp_select_impl(const double* a, int64_t lda, int64_t r, int cols, int64_t* order, int32_t* count,
                     prrp_err* err, cudaStream_t s) {
  if (cols < 1 || cols > PRRP_MAXH) fail(PRRP_ERR_UNSUPPORTED, "gepp_select needs 1 <= cols <= 128");
  if (r <= cols) fail(PRRP_ERR_ARG, "gepp_select needs more rows than columns");
  if (lda < cols) fail(PRRP_ERR_ARG, "lda < cols");
  caps();
  Arena ar(s);
  DevState* st = new_state(ar, s);
  GeppTourBufs T = alloc_tour(ar, r, cols, 1);
  unsigned long long* chg = ar.get<unsigned long long>(1);
  CU_TRY(cudaMemsetAsync(chg, 0, 8, s));
  bool single = false;
  gepp_tournament(a, lda, cols, r, 1, T, chg, st, 0, single, s);
  widen_kernel<<<(unsigned)std::min<int64_t>((r + 255) / 256, 4 * caps().sms), 256, 0, s>>>(T.order_full, r, order);
  CU_TRY(cudaGetLastError());
  int32_t c = 0;
  CU_TRY(cudaMemcpyAsync(&c, T.cnt[0], 4, cudaMemcpyDeviceToHost, s));
  DevState hs;
  read_state(st, hs, s);
  if (count) *count = c;
  return state_to_err(hs, err);
}

// gepp_factor of any shape (gepp.py:39-65): unblocked, two launches per step.
// steps_only: the running maximum covers the updated entries only (the
// block variants' observe_finish after every step, block_variants.py:170-186),
// not seeded with the original maximum (gepp_factor's running_max).
int gepp_full_impl(double* A, int64_t lda, int64_t m, int64_t n, int64_t* perm, double* imax, double* omax,
                   prrp_err* err, cudaStream_t s, bool steps_only = false) {
  if (m < 1 || n < 1) fail(PRRP_ERR_DIM, "gepp needs a non-empty matrix");
  if (lda < n) fail(PRRP_ERR_ARG, "lda < n");
  caps();
  const int sms = caps().sms;
  Arena ar(s);
  DevState* st = new_state(ar, s);
  DevState* st0 = steps_only ? new_state(ar, s) : st;
  iota_kernel<<<sms, 256, 0, s>>>(perm, m);
  maxabs_kernel<<<sms * 4, 256, 0, s>>>(A, lda, m, n, st0);
  const int64_t steps = std::min(m, n);
  for (int64_t k = 0; k < steps; ++k) {
    gf_pivot_kernel<<<1, 1024, 0, s>>>(A, lda, m, n, k, perm, st);
    if (k + 1 < m) {
      const int64_t groups = (m - k - 1 + GF_ROWS - 1) / GF_ROWS;
      gf_update_kernel<<<(unsigned)std::min<int64_t>(groups, 8 * sms), 256, 0, s>>>(A, lda, m, n, k, st);
    }
  }
  CU_TRY(cudaGetLastError());
  DevState hs, hs0;
  read_state(st, hs, s);
  if (steps_only) read_state(st0, hs0, s);
  else hs0 = hs;
  if (imax) *imax = bits_to_double(hs.inter_max);
  if (omax) *omax = bits_to_double(hs0.orig_max);
  return state_to_err(hs, err);
}
#include "calu_dist.cuh"

}  // namespace

// ======================================================================== ABI
extern "C" {

int prrp_b200_abi_version(void) { return kAbiVersion; }

int prrp_b200_device_probe(int32_t* sm_count, int32_t* max_cluster, prrp_err* err) {
  clear_err(err);
  try {
    DeviceCaps& c = caps();
    if (sm_count) *sm_count = c.sms;
    if (max_cluster) *max_cluster = c.max_cluster;
    return PRRP_OK;
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_luprrp(double* A, int64_t lda, int64_t m, int64_t n, int32_t b, double tau, int64_t* perm,
                int32_t* swap_counts, prrp_stats* stats, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    return luprrp_impl(A, lda, m, n, b, tau, perm, swap_counts, stats, err, nullptr, (cudaStream_t)stream);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_luprrp_timed(double* A, int64_t lda, int64_t m, int64_t n, int32_t b, double tau, int64_t* perm,
                      int32_t* swap_counts, prrp_stats* stats, prrp_err* err, prrp_timing* timing, void* stream) {
  clear_err(err);
  if (timing) memset(timing, 0, sizeof(*timing));
  try {
    return luprrp_impl(A, lda, m, n, b, tau, perm, swap_counts, stats, err, timing, (cudaStream_t)stream);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_b200_dmma_peak(double ms, double* tflops, prrp_err* err) {
  clear_err(err);
  try {
    caps();
    double* sink = nullptr;
    CU_TRY(cudaMalloc(&sink, 64));
    cudaEvent_t e0, e1;
    CU_TRY(cudaEventCreate(&e0));
    CU_TRY(cudaEventCreate(&e1));
    const long iters = 4000;
    const dim3 grid(caps().sms * 2), block(256);
    dmma_peak_kernel<<<grid, block>>>(sink, 100);
    CU_TRY(cudaDeviceSynchronize());
    CU_TRY(cudaEventRecord(e0));
    int reps = 0;
    float el = 0.f;
    while (el < ms) {
      for (int r = 0; r < 10; ++r, ++reps) dmma_peak_kernel<<<grid, block>>>(sink, iters);
      CU_TRY(cudaEventRecord(e1));
      CU_TRY(cudaEventSynchronize(e1));
      CU_TRY(cudaEventElapsedTime(&el, e0, e1));
    }
    const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * grid.x * (block.x / 32) * reps;
    if (tflops) *tflops = flops / (el * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    return PRRP_OK;
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_caluprrp(double* A, int64_t lda, int64_t m, int64_t n, int32_t b, double tau, int32_t leaf_count,
                  int64_t* perm, int32_t* swap_counts, int64_t* tournament_charge3, prrp_stats* stats, prrp_err* err,
                  void* stream) {
  clear_err(err);
  try {
    return caluprrp_impl(A, lda, m, n, b, tau, leaf_count, perm, swap_counts, tournament_charge3, stats, err,
                         (cudaStream_t)stream);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int64_t prrp_b200_graph_kernels(void) { return tl_last_graph_kernels; }

// Diagnostics: average device time of the panel QRCP engine alone on an
// h x p transposed panel (rows of `a`), `reps` launches between CUDA events.
// nwc/cpt > 0 force a latency-engine shape; nwc < 0 runs the thread-per-
// column engines (h = 64 or 128 only).
int prrp_b200_qrcp_time(const double* a, int64_t lda, int32_t h, int64_t p, int32_t nwc, int32_t cpt, int32_t reps,
                        double* ms_out, int32_t* ctas_out, double* R_out, int64_t* perm_out, prrp_err* err) {
  clear_err(err);
  try {
    cudaStream_t s = 0;
    if (h < 1 || h > PRRP_MAXH || p < 1 || reps < 1) fail(PRRP_ERR_ARG, "bad probe arguments");
    caps();
    Arena ar(s);
    DevState* st = new_state(ar, s);
    PanelArgs pa{};
    pa.src = a;
    pa.ld = lda;
    pa.h = h;
    pa.p = p;
    pa.bsel = h;
    pa.steps = (int)std::min<int64_t>(h, p);
    pa.mode = 0;
    pa.perm = ar.get<int32_t>(p);
    pa.Rbuf = ar.get<double>((size_t)h * p);
    pa.ovf = ar.get<double>(ovf_elems(h, p, h));
    pa.st = st;
    pa.fro = &st->fro;
    pa.tree_level = pa.tree_index = -1;
    pa.fused_ak = 1;
    cudaEvent_t e0, e1;
    CU_TRY(cudaEventCreate(&e0));
    CU_TRY(cudaEventCreate(&e1));
    int ctas = 0;
    for (int r = -1; r < reps; ++r) {
      if (r == 0) CU_TRY(cudaEventRecord(e0, s));
      if (nwc >= 0) {
        const LatShape sh = lat_shape(h, p, nwc, cpt, 16);
        if (!sh.nwc) fail(PRRP_ERR_UNSUPPORTED, "no such latency-engine shape");
        ctas = sh.C;
        launch_team(pa, s, nwc, cpt, 16);
      } else if (h == P1_H) {
        PanelCfg g1{};
        g1.C = (int)std::max<int64_t>(1, (p + 255) / 256);
        g1.T = P1_T;
        PanelArgs a1 = pa;
        a1.per = (p + g1.C - 1) / g1.C;
        ctas = g1.C;
        launch_cluster(panel_qrcp1_kernel, g1, a1.per > P1_T ? (size_t)P1_H * P1_T * 8 : 0, s, a1);
      } else if (h == P2_H) {
        PanelCfg g2{};
        g2.C = (int)std::max<int64_t>(1, (p + P2_T - 1) / P2_T);
        g2.T = P2_T;
        PanelArgs a2 = pa;
        a2.per = (p + g2.C - 1) / g2.C;
        ctas = g2.C;
        launch_cluster(panel_qrcp2_kernel, g2, (size_t)(P2_H - P2_W) * P2_T * 8, s, a2);
      } else {
        fail(PRRP_ERR_UNSUPPORTED, "thread-per-column engines need h = 64 or 128");
      }
    }
    CU_TRY(cudaEventRecord(e1, s));
    CU_TRY(cudaEventSynchronize(e1));
    float ms = 0.f;
    CU_TRY(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ms_out) *ms_out = (double)ms / reps;
    if (ctas_out) *ctas_out = ctas;
    if (R_out && perm_out) {
      r_out_kernel<<<caps().sms, 256, 0, s>>>(pa.Rbuf, h, p, pa.perm, R_out, perm_out);
      CU_TRY(cudaGetLastError());
    }
    DevState hs;
    read_state(st, hs, s);
    return state_to_err(hs, err);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_caluprrp_timed(double* A, int64_t lda, int64_t m, int64_t n, int32_t b, double tau, int32_t leaf_count,
                        int64_t* perm, int32_t* swap_counts, int64_t* tournament_charge3, prrp_stats* stats,
                        prrp_err* err, prrp_timing* timing, void* stream) {
  clear_err(err);
  if (timing) memset(timing, 0, sizeof(*timing));
  try {
    return caluprrp_impl(A, lda, m, n, b, tau, leaf_count, perm, swap_counts, tournament_charge3, stats, err,
                         (cudaStream_t)stream, timing);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_strong_rrqr(const double* a, int64_t lda, int32_t h, int64_t p, int32_t bsel, double tau, double* R,
                     double* Q, int64_t* perm, double* Lblk, int32_t* swap_count, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    if (!(tau > 1.0)) fail(PRRP_ERR_ARG, "tau must exceed 1");
    if (h < bsel || p < bsel + 1 || bsel < 1) fail(PRRP_ERR_ARG, "strong_rrqr needs >= b rows and >= b+1 columns");
    if (h > PRRP_MAXH) fail(PRRP_ERR_UNSUPPORTED, "h > 128 is outside the device panel engine");
    caps();
    Arena ar(s);
    DevState* st = new_state(ar, s);
    const PanelCfg g = panel_config(h, p, bsel);
    PanelBuffers B{};
    B.Rbuf = ar.get<double>((size_t)h * p);
    B.perm = ar.get<int32_t>(p);
    B.ovf = ar.get<double>(ovf_elems(h, p, bsel));
    B.cand = ar.get<double>(kMaxCand);
    B.cand_flat = ar.get<long long>(kMaxCand);
    B.moved = ar.get<int32_t>(2 * p);
    alloc_exchange(ar, s, B);
    const int steps = (int)std::min<int64_t>(h, p);
    B.refl = ar.get<double>((size_t)steps * (h + 1));
    const int64_t ldl = std::max<int64_t>(1, p - bsel);
    double* L = ar.get<double>((size_t)bsel * ldl);
    int32_t* swaps_dev = ar.get<int32_t>(1);
    CU_TRY(cudaMemsetAsync(swaps_dev, 0, sizeof(int32_t), s));
    strong_rrqr_panel(a, lda, h, p, bsel, tau, 0, L, ldl, B, st, swaps_dev, nullptr, nullptr, nullptr, false, s);
    r_out_kernel<<<caps().sms, 256, 0, s>>>(B.Rbuf, h, p, B.perm, R, perm);
    form_q_kernel<<<1, 256, (size_t)h * h * 8, s>>>(B.refl, h, steps, Q);
    CU_TRY(cudaGetLastError());
    if (p > bsel) CU_TRY(cudaMemcpyAsync(Lblk, L, sizeof(double) * (size_t)bsel * (p - bsel), cudaMemcpyDeviceToDevice, s));
    DevState hs;
    read_state(st, hs, s);
    int32_t sw = 0;
    CU_TRY(cudaMemcpy(&sw, swaps_dev, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (swap_count) *swap_count = sw;
    return state_to_err(hs, err);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_householder_qr(const double* a, int64_t lda, int32_t h, int64_t p, double* R, double* Q, prrp_err* err,
                        void* stream) {
  clear_err(err);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    if (h > PRRP_MAXH) fail(PRRP_ERR_UNSUPPORTED, "h > 128 is outside the device panel engine");
    if (h < 1 || p < 1) fail(PRRP_ERR_ARG, "empty matrix");
    caps();
    Arena ar(s);
    DevState* st = new_state(ar, s);
    const PanelCfg g = panel_config(h, p, 1);
    double* Rbuf = ar.get<double>((size_t)h * p);
    int32_t* permb = ar.get<int32_t>(p);
    const int steps = (int)std::min<int64_t>(h, p);
    double* refl = ar.get<double>((size_t)steps * (h + 1));
    double* ovf = ar.get<double>((size_t)g.C * h * std::max<int64_t>(1, g.ovpad));
    iota32_kernel<<<caps().sms, 256, 0, s>>>(permb, p);
    PanelArgs pa{};
    pa.src = a;
    pa.ld = lda;
    pa.h = h;
    pa.p = p;
    pa.bsel = 1;
    pa.steps = steps;
    pa.mode = 1;
    pa.perm = permb;
    pa.Rbuf = Rbuf;
    pa.refl = refl;
    pa.ovf = ovf;
    pa.per = g.per;
    pa.cap = g.cap;
    pa.cap_pad = g.cap_pad;
    pa.ovpad = g.ovpad;
    pa.st = st;
    if (team_eligible(h, p) && !force_generic_panel()) launch_team(pa, s);
    else launch_cluster(panel_qrcp_kernel, g, g.dyn_engine, s, pa);
    int64_t* dummy_perm = ar.get<int64_t>(p);
    r_out_kernel<<<caps().sms, 256, 0, s>>>(Rbuf, h, p, permb, R, dummy_perm);
    form_q_kernel<<<1, 256, (size_t)h * h * 8, s>>>(refl, h, steps, Q);
    CU_TRY(cudaGetLastError());
    DevState hs;
    read_state(st, hs, s);
    return state_to_err(hs, err);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

// QR with column pivoting over min(h, p) steps (pivoted_qr.py:74-87): the
// cluster engine in pivoted mode, reflector log -> explicit Q.
int prrp_qrcp(const double* a, int64_t lda, int32_t h, int64_t p, double* R, double* Q, int64_t* perm, prrp_err* err,
              void* stream) {
  clear_err(err);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    if (h > PRRP_MAXH) fail(PRRP_ERR_UNSUPPORTED, "h > 128 is outside the device panel engine");
    if (h < 1 || p < 1) fail(PRRP_ERR_ARG, "empty matrix");
    caps();
    Arena ar(s);
    DevState* st = new_state(ar, s);
    const PanelCfg g = panel_config(h, p, 1);
    double* Rbuf = ar.get<double>((size_t)h * p);
    int32_t* permb = ar.get<int32_t>(p);
    const int steps = (int)std::min<int64_t>(h, p);
    double* refl = ar.get<double>((size_t)steps * (h + 1));
    double* ovf = ar.get<double>((size_t)g.C * h * std::max<int64_t>(1, g.ovpad));
    PanelArgs pa{};
    pa.src = a;
    pa.ld = lda;
    pa.h = h;
    pa.p = p;
    pa.bsel = 1;
    pa.steps = steps;
    pa.mode = 0;
    pa.perm = permb;
    pa.Rbuf = Rbuf;
    pa.refl = refl;
    pa.ovf = ovf;
    pa.per = g.per;
    pa.cap = g.cap;
    pa.cap_pad = g.cap_pad;
    pa.ovpad = g.ovpad;
    pa.st = st;
    pa.fro = &st->fro;
    pa.tree_level = pa.tree_index = -1;
    if (team_eligible(h, p) && !force_generic_panel()) launch_team(pa, s);
    else launch_cluster(panel_qrcp_kernel, g, g.dyn_engine, s, pa);
    r_out_kernel<<<caps().sms, 256, 0, s>>>(Rbuf, h, p, permb, R, perm);
    form_q_kernel<<<1, 256, (size_t)h * h * 8, s>>>(refl, h, steps, Q);
    CU_TRY(cudaGetLastError());
    DevState hs;
    read_state(st, hs, s);
    return state_to_err(hs, err);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

// ||Pi A - L U||_F^2 and ||A||_F^2 from the packed factors (metrics.py:56-63)
int prrp_lu_residual(const double* A, int64_t lda, const double* LU, int64_t ldlu, const int64_t* perm, int64_t m,
                     int64_t n, double* resid_sq, double* a_sq, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    if (m < n || n < 1) fail(PRRP_ERR_DIM, "need m >= n >= 1");
    caps();
    Arena ar(s);
    DevState* st = new_state(ar, s);
    const int64_t ldc = n + (n & 1);
    double* C = ar.get<double>((size_t)m * ldc);
    const int KB = 64;
    const int64_t ldlk = ((m + 7) / 8) * 8, lduk = ((n + 7) / 8) * 8;
    double* Lk = ar.get<double>((size_t)KB * ldlk);
    double* Uk = ar.get<double>((size_t)KB * lduk);
    double* sums = ar.get<double>(2);
    CU_TRY(cudaMemsetAsync(sums, 0, 2 * sizeof(double), s));
    const int sms = caps().sms;
    gather_rows_kernel<<<sms * 8, 256, 0, s>>>(A, lda, perm, m, n, C, ldc);
    for (int64_t k0 = 0; k0 < n; k0 += KB) {
      const int kb = (int)std::min<int64_t>(KB, n - k0);
      const int Kp = (kb + 3) / 4 * 4;
      build_lk_kernel<<<sms * 4, 256, 0, s>>>(LU, ldlu, m, k0, kb, Kp, Lk, ldlk);
      build_uk_kernel<<<sms * 4, 256, 0, s>>>(LU, ldlu, n, k0, kb, Kp, Uk, lduk);
      CU_TRY(cudaGetLastError());
      schur_update(C + k0 * ldc + k0, ldc, Lk, ldlk, Uk, lduk, m - k0, n - k0, Kp, st, s, caps().sms);
    }
    sumsq_kernel<<<sms * 4, 256, 0, s>>>(C, ldc, m, n, sums);
    sumsq_kernel<<<sms * 4, 256, 0, s>>>(A, lda, m, n, sums + 1);
    CU_TRY(cudaGetLastError());
    double h[2];
    CU_TRY(cudaMemcpyAsync(h, sums, sizeof(h), cudaMemcpyDeviceToHost, s));
    DevState hs;
    read_state(st, hs, s);
    if (resid_sq) *resid_sq = h[0];
    if (a_sq) *a_sq = h[1];
    return state_to_err(hs, err);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

// X = A^-1 B from the packed square factors (luprrp.py:204-214)
int prrp_lu_solve(const double* LU, int64_t ldlu, int64_t n, const int64_t* perm, const double* B, int64_t ldb,
                  double* X, int64_t ldx, int32_t nrhs, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    if (n < 1 || nrhs < 1) fail(PRRP_ERR_DIM, "empty system");
    if (ldb < n || ldx < n) fail(PRRP_ERR_ARG, "leading dimension < n");
    caps();
    Arena ar(s);
    DevState* st = new_state(ar, s);
    lu_solve_kernel<<<nrhs, LS_T, 0, s>>>(LU, ldlu, n, perm, B, ldb, X, ldx, st);
    CU_TRY(cudaGetLastError());
    DevState hs;
    read_state(st, hs, s);
    return state_to_err(hs, err);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_multiplier_block(const double* R, int64_t ldr, int32_t b, int64_t p, double* L, int64_t ldl,
                          double* absmax, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    if (b < 1 || b > PRRP_MAXH || p < b || ldr < b) fail(PRRP_ERR_ARG, "multiplier_block needs 1 <= b <= 128, p >= b");
    caps();
    Arena ar(s);
    DevState* st = new_state(ar, s);
    const int64_t ncol = p - b;
    if (ncol > 0) {
      double* Rbuf = ar.get<double>((size_t)b * p);
      double* fro0 = ar.get<double>(1);
      double* cand = ar.get<double>(kMaxCand);
      long long* candf = ar.get<long long>(kMaxCand);
      CU_TRY(cudaMemsetAsync(fro0, 0, sizeof(double), s));
      r_in_kernel<<<caps().sms, 256, 0, s>>>(R, ldr, b, p, Rbuf);
      const bool c2 = b > 64 && use_trsm_c2();
      const int nblk = (int)std::min<int64_t>(kMaxCand, c2 ? (ncol + TC_COLS - 1) / TC_COLS : (ncol + TTC - 1) / TTC);
      const size_t tdyn = (((size_t)b * (b + 1) / 2 + 1) / 2 * 2 + (size_t)b * TTCP) * 8;
      if (c2) trsm_c2_kernel<<<nblk, TC_T, kTrsmC2Smem, s>>>(Rbuf, p, b, L, ldl, cand, candf, st, -1, fro0, -1, -1, nullptr, nullptr);
      else switch ((b + 31) / 32) {
        case 1: trsm_w_kernel<1><<<nblk, TW_WARPS * 32, tdyn, s>>>(Rbuf, p, b, L, ldl, cand, candf, st, -1, fro0, -1, -1, nullptr, nullptr); break;
        case 2: trsm_w_kernel<2><<<nblk, TW_WARPS * 32, tdyn, s>>>(Rbuf, p, b, L, ldl, cand, candf, st, -1, fro0, -1, -1, nullptr, nullptr); break;
        case 3: trsm_w_kernel<3><<<nblk, TW_WARPS * 32, tdyn, s>>>(Rbuf, p, b, L, ldl, cand, candf, st, -1, fro0, -1, -1, nullptr, nullptr); break;
        default: trsm_w_kernel<4><<<nblk, TW_WARPS * 32, tdyn, s>>>(Rbuf, p, b, L, ldl, cand, candf, st, -1, fro0, -1, -1, nullptr, nullptr); break;
      }
      calu_stats_kernel<<<1, 256, 0, s>>>(cand, nblk, cand == nullptr ? nullptr : (const int32_t*)nullptr, 0,
                                          (int32_t*)fro0, 0, st);
      CU_TRY(cudaGetLastError());
    }
    DevState hs;
    read_state(st, hs, s);
    if (absmax) *absmax = ncol > 0 ? bits_to_double(hs.pmm) : 0.0;
    return state_to_err(hs, err);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_schur_update(double* C, int64_t ldc, const double* L, int64_t ldl, const double* B, int64_t ldb, int64_t M,
                      int64_t N, int32_t K, double* absmax, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    caps();
    Arena ar(s);
    DevState* st = new_state(ar, s);
    schur_update(C, ldc, L, ldl, B, ldb, M, N, K, st, s, caps().sms);
    DevState hs;
    read_state(st, hs, s);
    if (absmax) *absmax = bits_to_double(hs.inter_max);
    return state_to_err(hs, err);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_gepp_blockrow(double* A, int64_t lda, int32_t m, int64_t n, int64_t* perm, double* intermediate_max,
                       prrp_err* err, void* stream) {
  clear_err(err);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    if (m < 1 || m > PRRP_MAXH || n < m) fail(PRRP_ERR_UNSUPPORTED, "gepp_blockrow needs 1 <= m <= 128, n >= m");
    caps();
    Arena ar(s);
    DevState* st = new_state(ar, s);
    double* D = ar.get<double>((size_t)m * m);
    int32_t* piv = ar.get<int32_t>(m);
    int32_t* gperm = ar.get<int32_t>(m);
    iota_kernel<<<1, 128, 0, s>>>(perm, m);
    maxabs_kernel<<<caps().sms, 256, 0, s>>>(A, lda, m, n, st);
    launch_gepp(A, lda, nullptr, m, D, piv, gperm, st, 0, s);
    blockrow_kernel<<<(unsigned)((n + BR_TW - 1) / BR_TW), BR_TW, ((size_t)m * m + (size_t)m * BR_TW) * 8, s>>>(
        A, lda, 0, m, n, D, piv, gperm, perm, st);
    CU_TRY(cudaGetLastError());
    DevState hs;
    read_state(st, hs, s);
    if (intermediate_max) *intermediate_max = bits_to_double(hs.finish_max);
    return state_to_err(hs, err);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_calu(double* A, int64_t lda, int64_t m, int64_t n, int32_t b, int32_t leaf_count, int64_t* perm,
              int64_t* tournament_charge3, prrp_stats* stats, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    return calu_gepp_impl(A, lda, m, n, b, leaf_count, perm, tournament_charge3, stats, err, (cudaStream_t)stream);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_gepp_select(const double* a, int64_t lda, int64_t r, int32_t cols, int64_t* order, int32_t* count,
                     prrp_err* err, void* stream) {
  clear_err(err);
  try {
    return gepp_select_impl(a, lda, r, cols, order, count, err, (cudaStream_t)stream);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_gepp(double* A, int64_t lda, int64_t m, int64_t n, int64_t* perm, double* intermediate_max,
              double* original_max, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    return gepp_full_impl(A, lda, m, n, perm, intermediate_max, original_max, err, (cudaStream_t)stream);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_gepp_steps(double* A, int64_t lda, int64_t m, int64_t n, int64_t* perm, double* steps_max,
                    double* original_max, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    return gepp_full_impl(A, lda, m, n, perm, steps_max, original_max, err, (cudaStream_t)stream, true);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

// ---------------------------------------------------------------- distributed CALU_PRRP (calu_dist.cuh)
int prrp_calu_dist_create(void** handle, double* A_loc, int64_t lda, int64_t m, int64_t n, int64_t n_loc, int32_t b,
                          double tau, int32_t leaf_count, int32_t nranks, int32_t rank, int64_t* perm, prrp_err* err,
                          void* stream) {
  clear_err(err);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    if (!handle) fail(PRRP_ERR_ARG, "null handle");
    if (m < n) fail(PRRP_ERR_DIM, "need at least as many rows as columns");
    if (b < 1 || b > n) fail(PRRP_ERR_ARG, "panel width out of range");
    if (!(tau > 1.0)) fail(PRRP_ERR_ARG, "tau must exceed 1");
    if (leaf_count < 0) fail(PRRP_ERR_ARG, "binary tree needs a leaf count >= 1 (0 selects the flat tree)");
    if (b > PRRP_MAXH) fail(PRRP_ERR_UNSUPPORTED, "panel width > 128 is outside the device panel engine");
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(PRRP_ERR_ARG, "bad rank / nranks");
    const int64_t npan = (n + b - 1) / b;
    int64_t want_loc = 0;
    for (int64_t J = rank; J < npan; J += nranks) want_loc += std::min<int64_t>(b, n - J * b);
    if (n_loc != want_loc) fail(PRRP_ERR_DIM, "n_loc does not match the column block-cyclic layout");
    if (lda < std::max<int64_t>(n_loc, 1) || (lda & 1) || ((uintptr_t)A_loc % 16)) fail(PRRP_ERR_ARG, "lda must be even, >= n_loc, A 16-byte aligned");
    caps();
    std::unique_ptr<CaluDist> w(new CaluDist);
    w->m = m; w->n = n; w->n_loc = n_loc; w->lda = lda; w->b = b; w->tau = tau; w->P = leaf_count;
    w->nranks = nranks; w->rank = rank; w->npanels = (int)npan; w->A = A_loc; w->perm = perm;
    calu_dist_alloc(*w, s);
    calu_dist_structure(*w);
    *handle = w.release();
    return PRRP_OK;
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_calu_dist_buffers(void* handle, void** msg0, void** msg1, int64_t* msg_capacity, void** stats,
                           int64_t* stats_len) {
  CaluDist* w = static_cast<CaluDist*>(handle);
  if (!w) return PRRP_ERR_ARG;
  if (msg0) *msg0 = w->msgs[0];
  if (msg1) *msg1 = w->msgs[1];
  if (msg_capacity) *msg_capacity = (int64_t)w->msg_cap;
  if (stats) *stats = w->red;
  if (stats_len) *stats_len = (int64_t)w->red_len;
  return PRRP_OK;
}

int64_t prrp_calu_dist_msg_bytes(void* handle, int32_t panel) {
  CaluDist* w = static_cast<CaluDist*>(handle);
  if (!w || panel < 0 || panel >= w->npanels) return -1;
  const int64_t col0 = (int64_t)panel * w->b;
  const int64_t rows = w->m - col0, bj = std::min<int64_t>(w->b, w->n - col0);
  // the single-node order region is needed only when the panel has one node
  if (rows > bj && w->p_eff(panel) > 1) return (int64_t)w->msg_bytes(panel);
  if (rows <= bj) return (int64_t)w->off_full;
  return (int64_t)w->msg_bytes(panel);
}

int prrp_calu_dist_select(void* handle, int32_t panel, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    CaluDist* w = static_cast<CaluDist*>(handle);
    if (!w || panel < 0 || panel >= w->npanels) fail(PRRP_ERR_ARG, "bad handle or panel");
    if (w->owner(panel) != w->rank) fail(PRRP_ERR_ARG, "select runs on the panel's owner only");
    calu_dist_select(*w, panel, (cudaStream_t)stream);
    return PRRP_OK;
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_calu_dist_apply(void* handle, int32_t panel, int32_t part, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    CaluDist* w = static_cast<CaluDist*>(handle);
    if (!w || panel < 0 || panel >= w->npanels) fail(PRRP_ERR_ARG, "bad handle or panel");
    if (part < 0 || part > 2) fail(PRRP_ERR_ARG, "part must be 0 (all), 1 (head) or 2 (tail)");
    calu_dist_apply(*w, panel, part, (cudaStream_t)stream);
    return PRRP_OK;
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_calu_dist_stats(void* handle, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    CaluDist* w = static_cast<CaluDist*>(handle);
    if (!w) fail(PRRP_ERR_ARG, "bad handle");
    const int nslots = w->npanels * w->maxnodes;
    dist_stats_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(w->st, w->swaps_dev, w->npanels, w->node_swaps,
                                                              w->node_rows, nslots, w->red);
    CU_TRY(cudaGetLastError());
    return PRRP_OK;
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_calu_dist_finish(void* handle, const int64_t* reduced, int32_t* swap_counts, int64_t* tournament_charge3,
                          prrp_stats* stats, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    CaluDist* w = static_cast<CaluDist*>(handle);
    if (!w) fail(PRRP_ERR_ARG, "bad handle");
    return calu_dist_finish(*w, reduced ? reduced : w->red, swap_counts, tournament_charge3, stats, err,
                            (cudaStream_t)stream);
  } catch (const Fail& f) {
    return report(err, f);
  }
}

void prrp_calu_dist_destroy(void* handle) {
  CaluDist* w = static_cast<CaluDist*>(handle);
  if (!w) return;
  cudaDeviceSynchronize();
  delete w;
}

// ---------------------------------------------------------------- stability measurements (verify.cuh)
int prrp_residual_extended(const double* A, int64_t lda, int64_t m, int64_t n, const double* x, const double* rhs,
                           double* r, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    if (m < 0 || n < 0 || lda < n) fail(PRRP_ERR_ARG, "bad shape");
    if (m == 0) return PRRP_OK;
    residual_ext_kernel<<<(unsigned)((m + RX_T - 1) / RX_T), RX_T, 0, (cudaStream_t)stream>>>(A, lda, m, n, x, rhs, r);
    CU_TRY(cudaGetLastError());
    return PRRP_OK;
  } catch (const Fail& f) {
    return report(err, f);
  }
}

int prrp_abs_sums(const double* A, int64_t lda, int64_t m, int64_t n, const double* x, double* colabs,
                  double* rowabs, double* absax, prrp_err* err, void* stream) {
  clear_err(err);
  try {
    if (m < 0 || n < 0 || lda < n) fail(PRRP_ERR_ARG, "bad shape");
    cudaStream_t s = (cudaStream_t)stream;
    if (colabs && n > 0) abs_colsum_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(A, lda, m, n, colabs);
    if ((rowabs || absax) && m > 0)
      abs_rowsum_kernel<<<(unsigned)((m * 32 + 255) / 256), 256, 0, s>>>(A, lda, m, n, x, rowabs, absax);
    CU_TRY(cudaGetLastError());
    return PRRP_OK;
  } catch (const Fail& f) {
    return report(err, f);
  }
}

}  // extern "C"
