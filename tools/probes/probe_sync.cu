// Probe: per-step latency of the global "publish candidate -> agree on winner ->
// fetch winner column" exchange that the panel QRCP performs b times per panel.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

struct Rec { double norm; long long pos; };

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p)); return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p)); return v;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acqrel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// MODE 0: threadfence + atomicAdd + ld.acquire poll
// MODE 1: red.release + ld.relaxed poll + fence.acq_rel
// MODE 2: per-CTA flags, warp 0 polls all flags (relaxed), fence
template <int MODE>
__global__ void exch(unsigned* counter, unsigned* flags, Rec* recs, double* cols, int steps, int b, double* sink) {
  __shared__ Rec best;
  __shared__ double col[128];
  const int P = gridDim.x;
  double acc = 0;
  for (int k = 0; k < steps; ++k) {
    const int buf = k & 1;
    // publish: candidate column (b doubles) + record
    if (threadIdx.x < b) cols[(size_t)(buf * P + blockIdx.x) * 128 + threadIdx.x] = blockIdx.x + k + threadIdx.x;
    if (threadIdx.x == 0) { recs[buf * P + blockIdx.x].norm = (double)((blockIdx.x * 37 + k) % P); recs[buf * P + blockIdx.x].pos = blockIdx.x; }
    __syncthreads();
    if (MODE == 0) {
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(counter, 1u);
        while (ld_acquire(counter) < (unsigned)(P * (k + 1))) {}
      }
    } else if (MODE == 1) {
      if (threadIdx.x == 0) {
        red_release(counter, 1u);
        while (ld_relaxed(counter) < (unsigned)(P * (k + 1))) {}
        fence_acqrel();
      }
    } else {
      if (threadIdx.x == 0) { asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(flags + blockIdx.x * 32), "r"((unsigned)(k + 1)) : "memory"); }
      if (threadIdx.x < 32) {
        for (int i = threadIdx.x; i < P; i += 32) { while (ld_relaxed(flags + i * 32) < (unsigned)(k + 1)) {} }
        fence_acqrel();
      }
    }
    __syncthreads();
    // agree on winner: warp 0 scans all records
    if (threadIdx.x < 32) {
      double bn = -1; long long bp = 1ll << 60;
      for (int i = threadIdx.x; i < P; i += 32) {
        Rec r = recs[buf * P + i];
        if (r.norm > bn || (r.norm == bn && r.pos < bp)) { bn = r.norm; bp = r.pos; }
      }
      for (int o = 16; o; o >>= 1) {
        double on = __shfl_xor_sync(0xffffffff, bn, o); long long op = __shfl_xor_sync(0xffffffff, bp, o);
        if (on > bn || (on == bn && op < bp)) { bn = on; bp = op; }
      }
      if (threadIdx.x == 0) { best.norm = bn; best.pos = bp; }
    }
    __syncthreads();
    if (threadIdx.x < b) col[threadIdx.x] = cols[(size_t)(buf * P + best.pos) * 128 + threadIdx.x];
    __syncthreads();
    acc += col[threadIdx.x % b];
  }
  if (acc == -1.0) sink[0] = acc;
}

// cluster variant: one cluster, candidates exchanged via DSMEM, hardware cluster barrier
template <int CS>
__global__ void exch_cluster(int steps, int b, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ Rec rec[2];
  __shared__ double pub[2][128];
  __shared__ double col[128];
  __shared__ Rec best;
  double acc = 0;
  const int me = cl.block_rank();
  for (int k = 0; k < steps; ++k) {
    const int buf = k & 1;
    if (threadIdx.x < b) pub[buf][threadIdx.x] = me + k + threadIdx.x;
    if (threadIdx.x == 0) { rec[buf].norm = (double)((me * 37 + k) % CS); rec[buf].pos = me; }
    cl.sync();
    if (threadIdx.x < 32) {
      double bn = -1; long long bp = 1ll << 60;
      if (threadIdx.x < CS) {
        Rec* r = cl.map_shared_rank(&rec[buf], threadIdx.x);
        bn = r->norm; bp = r->pos;
      }
      for (int o = 16; o; o >>= 1) {
        double on = __shfl_xor_sync(0xffffffff, bn, o); long long op = __shfl_xor_sync(0xffffffff, bp, o);
        if (on > bn || (on == bn && op < bp)) { bn = on; bp = op; }
      }
      if (threadIdx.x == 0) { best.norm = bn; best.pos = bp; }
    }
    __syncthreads();
    if (threadIdx.x < b) col[threadIdx.x] = cl.map_shared_rank(&pub[buf][0], (int)best.pos)[threadIdx.x];
    __syncthreads();
    acc += col[threadIdx.x % b];
  }
  cl.sync();
  if (acc == -1.0) sink[0] = acc;
}

int main() {
  unsigned *counter, *flags; Rec* recs; double *cols, *sink;
  CK(cudaMalloc(&counter, 4)); CK(cudaMalloc(&flags, 160 * 128)); CK(cudaMalloc(&recs, 2 * 160 * sizeof(Rec)));
  CK(cudaMalloc(&cols, 2 * 160 * 128 * 8)); CK(cudaMalloc(&sink, 8));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int steps = 8192, b = 64;
  for (int P : {16, 32, 64, 148}) {
    float ms[3];
    for (int mode = 0; mode < 3; ++mode) {
      CK(cudaMemset(counter, 0, 4)); CK(cudaMemset(flags, 0, 160 * 128));
      void* args[] = {&counter, &flags, &recs, &cols, (void*)&steps, (void*)&b, &sink};
      const void* fn = mode == 0 ? (const void*)exch<0> : mode == 1 ? (const void*)exch<1> : (const void*)exch<2>;
      CK(cudaEventRecord(e0));
      CK(cudaLaunchCooperativeKernel(fn, P, 256, args, 0, 0));
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms[mode], e0, e1));
    }
    printf("grid P=%3d: fence+atomic %.3f us/step | red.release %.3f us/step | flags %.3f us/step\n", P,
           ms[0] * 1e3 / steps, ms[1] * 1e3 / steps, ms[2] * 1e3 / steps);
  }
  for (int cs : {2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(256); cfg.stream = 0;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    float ms;
    CK(cudaEventRecord(e0));
    if (cs == 2) CK(cudaLaunchKernelEx(&cfg, exch_cluster<2>, steps, b, sink));
    if (cs == 4) CK(cudaLaunchKernelEx(&cfg, exch_cluster<4>, steps, b, sink));
    if (cs == 8) CK(cudaLaunchKernelEx(&cfg, exch_cluster<8>, steps, b, sink));
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("cluster %d: %.3f us/step\n", cs, ms * 1e3 / steps);
  }
  {
    auto fn = exch_cluster<16>;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 0; cfg.stream = 0;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int ncl = 0; cudaError_t q = cudaOccupancyMaxActiveClusters(&ncl, (void*)fn, &cfg);
    printf("max active 16-clusters: %d (%s)\n", ncl, cudaGetErrorString(q));
    float ms;
    CK(cudaEventRecord(e0));
    CK(cudaLaunchKernelEx(&cfg, fn, steps, b, sink));
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("cluster 16: %.3f us/step\n", ms * 1e3 / steps);
  }
  printf("done\n");
  return 0;
}
