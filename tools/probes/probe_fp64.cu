// Hardware probes for the FP64 design decisions (run once on a B200 via gpurun).
//  1. DMMA (mma.sync m8n8k4 f64) sustained/burst throughput, all SMs.
//  2. DFMA (SIMT) throughput for comparison.
//  3. DMMA accumulation semantics: is D = C + sum_k a_k b_k a sequential FMA chain?
//  4. Grid-wide exchange latency: counter barrier vs per-CTA tag polling, P CTAs.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

template <int CH>
__global__ void dmma_peak(double* out, long iters, double a, double b) {
  double acc[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) { acc[c][0] = threadIdx.x * 1e-3; acc[c][1] = c; }
  double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma884(acc[c][0], acc[c][1], av, bv, acc[c][0], acc[c][1]);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1234.5) out[0] = s;
}

template <int CH>
__global__ void dfma_peak(double* out, long iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 1234.5) out[0] = s;
}

// A row-major 8x4, B col-major 4x8 (i.e. B[k][n] with n-major fragments), C 8x8 row-major.
__global__ void dmma_semantics(const double* A, const double* B, const double* C, double* D) {
  int lane = threadIdx.x;
  // fragment layouts for m8n8k4 f64: A: row = lane/4, k = lane%4. B: k = lane%4, col = lane/4.
  // C/D: row = lane/4, cols = 2*(lane%4) + {0,1}
  double a = A[(lane / 4) * 4 + lane % 4];
  double b = B[(lane % 4) * 8 + lane / 4];
  int r = lane / 4, c = 2 * (lane % 4);
  double c0 = C[r * 8 + c], c1 = C[r * 8 + c + 1];
  double d0, d1;
  dmma884(d0, d1, a, b, c0, c1);
  D[r * 8 + c] = d0; D[r * 8 + c + 1] = d1;
}

// ---------------------------------------------------------------- exchange latency
__global__ void barrier_counter(unsigned* counter, double* slots, int steps, long long* cycles) {
  __shared__ double best;
  const int P = gridDim.x;
  long long t0 = clock64();
  for (int k = 0; k < steps; ++k) {
    if (threadIdx.x == 0) {
      slots[(k & 1) * P + blockIdx.x] = (double)(blockIdx.x * 7 % 13) + k;
      __threadfence();
      atomicAdd(counter, 1u);
      unsigned target = (unsigned)(P * (k + 1));
      unsigned v;
      do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(counter)); } while (v < target);
    }
    __syncthreads();
    double m = -1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) m = fmax(m, slots[(k & 1) * P + i]);
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffff, m, o));
    if (threadIdx.x == 0) best = m;
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cycles[0] = clock64() - t0;
  if (best < -5) slots[0] = best;
}

// per-CTA record {value, tag}; readers poll every record's tag (acquire) then read value
__global__ void barrier_tags(unsigned long long* recs, int steps, long long* cycles) {
  __shared__ double best;
  const int P = gridDim.x;
  long long t0 = clock64();
  for (int k = 0; k < steps; ++k) {
    unsigned long long* my = recs + 2 * ((k & 1) * P + blockIdx.x);
    if (threadIdx.x == 0) {
      double v = (double)(blockIdx.x * 7 % 13) + k;
      my[0] = __double_as_longlong(v);
      asm volatile("st.release.gpu.u64 [%0], %1;" :: "l"(my + 1), "l"((unsigned long long)(k + 1)));
    }
    double m = -1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      unsigned long long* r = recs + 2 * ((k & 1) * P + i);
      unsigned long long t;
      do { asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(t) : "l"(r + 1)); } while (t != (unsigned long long)(k + 1));
      m = fmax(m, __longlong_as_double(r[0]));
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffff, m, o));
    __shared__ double wm[32];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) { double x = -1; for (int w = 0; w < (int)(blockDim.x >> 5); ++w) x = fmax(x, wm[w]); best = x; }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cycles[0] = clock64() - t0;
  if (best < -5) recs[0] = 0;
}

static double fma_chain(double c, const double* a, const double* b, int n) {
  for (int i = 0; i < n; ++i) c = std::fma(a[i], b[i], c);
  return c;
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int clk_khz = 0; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  printf("device %s SMs %d clock %d kHz\n", prop.name, prop.multiProcessorCount, clk_khz);
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));

  // ---- DMMA peak
  for (int warps : {4, 8, 16}) {
    for (int blocks_per_sm : {1, 2}) {
      long iters = 20000;
      dim3 grid(sms * blocks_per_sm), block(32 * warps);
      dmma_peak<8><<<grid, block>>>(out, 100, 1.0000001, 0.9999999);
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      dmma_peak<8><<<grid, block>>>(out, iters, 1.0000001, 0.9999999);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * grid.x * warps;
      printf("DMMA m8n8k4 burst warps=%d bps=%d: %.3f ms  %.2f TFLOP/s\n", warps, blocks_per_sm, ms, flops / ms / 1e9);
    }
  }
  {  // sustained ~4 s
    long iters = 20000; dim3 grid(sms), block(32 * 8);
    double flops_one = 2.0 * 8 * 8 * 4 * 8.0 * iters * grid.x * 8;
    CK(cudaEventRecord(e0));
    int reps = 0; float ms = 0;
    while (ms < 4000.f) {
      dmma_peak<8><<<grid, block>>>(out, iters, 1.0000001, 0.9999999);
      ++reps;
      if (reps % 20 == 0) { CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1)); }
    }
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("DMMA m8n8k4 sustained (%d reps, %.0f ms): %.2f TFLOP/s\n", reps, ms, flops_one * reps / ms / 1e9);
  }
  // ---- DFMA peak
  for (int warps : {8, 16, 32}) {
    long iters = 20000; dim3 grid(sms), block(32 * warps);
    dfma_peak<8><<<grid, block>>>(out, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    dfma_peak<8><<<grid, block>>>(out, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 8 * iters * grid.x * block.x;
    printf("DFMA warps=%d: %.3f ms  %.2f TFLOP/s\n", warps, ms, flops / ms / 1e9);
  }

  // ---- DMMA semantics
  {
    srand(12345);
    double *dA, *dB, *dC, *dD;
    CK(cudaMalloc(&dA, 32 * 8)); CK(cudaMalloc(&dB, 32 * 8)); CK(cudaMalloc(&dC, 64 * 8)); CK(cudaMalloc(&dD, 64 * 8));
    long match_seq = 0, match_seq_rev = 0, match_exact_round = 0, total = 0;
    for (int trial = 0; trial < 2000; ++trial) {
      double A[32], B[32], C[64], D[64];
      for (int i = 0; i < 32; ++i) { A[i] = (rand() / (double)RAND_MAX - 0.5) * pow(2.0, rand() % 40 - 20); B[i] = (rand() / (double)RAND_MAX - 0.5) * pow(2.0, rand() % 40 - 20); }
      for (int i = 0; i < 64; ++i) C[i] = (trial % 3 == 0) ? 0.0 : (rand() / (double)RAND_MAX - 0.5) * pow(2.0, rand() % 40 - 20);
      CK(cudaMemcpy(dA, A, 256, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dB, B, 256, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dC, C, 512, cudaMemcpyHostToDevice));
      dmma_semantics<<<1, 32>>>(dA, dB, dC, dD);
      CK(cudaMemcpy(D, dD, 512, cudaMemcpyDeviceToHost));
      for (int r = 0; r < 8; ++r) for (int c = 0; c < 8; ++c) {
        double a[4], b[4], ar[4], br[4];
        for (int k = 0; k < 4; ++k) { a[k] = A[r * 4 + k]; b[k] = B[k * 8 + c]; ar[3 - k] = a[k]; br[3 - k] = b[k]; }
        double s = fma_chain(C[r * 8 + c], a, b, 4);
        double sr = fma_chain(C[r * 8 + c], ar, br, 4);
        long double ex = C[r * 8 + c]; for (int k = 0; k < 4; ++k) ex += (long double)a[k] * b[k];
        match_seq += (s == D[r * 8 + c]); match_seq_rev += (sr == D[r * 8 + c]);
        match_exact_round += ((double)ex == D[r * 8 + c]);
        ++total;
      }
    }
    printf("DMMA semantics: seq-fma-chain k0..3 %ld/%ld, reversed %ld/%ld, long-double-single-round %ld/%ld\n",
           match_seq, total, match_seq_rev, total, match_exact_round, total);
  }

  // ---- exchange latency
  {
    unsigned* counter; double* slots; unsigned long long* recs; long long* cyc;
    CK(cudaMalloc(&counter, 4)); CK(cudaMalloc(&slots, 2 * 160 * 8)); CK(cudaMalloc(&recs, 2 * 2 * 160 * 8)); CK(cudaMalloc(&cyc, 8));
    for (int P : {8, 16, 32, 64, 96, 148}) {
      int steps = 4096;
      CK(cudaMemset(counter, 0, 4));
      CK(cudaEventRecord(e0));
      barrier_counter<<<P, 256>>>(counter, slots, steps, cyc);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      CK(cudaMemset(recs, 0, 2 * 2 * 160 * 8));
      cudaEvent_t f0, f1; CK(cudaEventCreate(&f0)); CK(cudaEventCreate(&f1));
      CK(cudaEventRecord(f0));
      barrier_tags<<<P, 256>>>(recs, steps, cyc);
      CK(cudaEventRecord(f1)); CK(cudaEventSynchronize(f1));
      float ms2; CK(cudaEventElapsedTime(&ms2, f0, f1));
      printf("exchange P=%3d: counter-barrier %.3f us/step, tag-poll %.3f us/step\n", P, ms * 1e3 / steps, ms2 * 1e3 / steps);
    }
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
