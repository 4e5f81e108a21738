// Apply+next-key step of panel1 (register column), warm vs after 4K instructions of other code.
#include <cstdio>
// Repeated asm bodies are spelled with doubling macros (NAME_X<count>).
#define ASMU0_X1 "xor.b32 %1, %1, %0;\n" "mad.lo.u32 %0, %0, %2, %1;\n" "xor.b32 %1, %1, %0;\n" "mad.lo.u32 %0, %0, %2, %1;\n"
#define ASMU0_X2 ASMU0_X1 ASMU0_X1
#define ASMU0_X4 ASMU0_X2 ASMU0_X2
#define ASMU0_X8 ASMU0_X4 ASMU0_X4
#define ASMU0_X16 ASMU0_X8 ASMU0_X8
#define ASMU0_X32 ASMU0_X16 ASMU0_X16
#define ASMU0_X64 ASMU0_X32 ASMU0_X32
#define ASMU0_X128 ASMU0_X64 ASMU0_X64
#define ASMU0_X256 ASMU0_X128 ASMU0_X128
#define ASMU0_X512 ASMU0_X256 ASMU0_X256
#define ASMU0_X1024 ASMU0_X512 ASMU0_X512
#define ASMU0_X2048 ASMU0_X1024 ASMU0_X1024
#define ASMU0_X4096 ASMU0_X2048 ASMU0_X2048
#define ASMU0_X8192 ASMU0_X4096 ASMU0_X4096
#define ASMU0_X16384 ASMU0_X8192 ASMU0_X8192
#define ASMU0_X32768 ASMU0_X16384 ASMU0_X16384
#define ASMU0_X65536 ASMU0_X32768 ASMU0_X32768
#define ASMU0_X131072 ASMU0_X65536 ASMU0_X65536
#define ASMU0_X262144 ASMU0_X131072 ASMU0_X131072
#define ASMU0_X524288 ASMU0_X262144 ASMU0_X262144
#define ASMU0_X1048576 ASMU0_X524288 ASMU0_X524288
#define STR2(x) #x
#define STR(x) STR2(x)
#include "../../paper_1208_2451_b200/csrc/panel1.cuh"


// branch-free (within NB blocks) apply + key, FMA update, dead rows zero
template <int NB, class X>
__device__ __forceinline__ double p1_step_nb(const X& x, const double2* vp, double beta, bool act, int L, int r0) {
  const uint32_t va = (uint32_t)__cvta_generic_to_shared(vp);
  double d[4];
#pragma unroll
  for (int B = 0; B < NB; ++B)
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const double2 v = lds2_f64(va + 64 * B + 16 * h);
      const int s = 2 * h;
      if (B == 0 && s < 4) { d[s] = mul_rn(v.x, x.ld(s)); d[s + 1] = mul_rn(v.y, x.ld(s + 1)); }
      else { d[s & 3] = fma(v.x, x.ld(8 * B + s), d[s & 3]); d[(s + 1) & 3] = fma(v.y, x.ld(8 * B + s + 1), d[(s + 1) & 3]); }
    }
  const double dot = (d[0] + d[1]) + (d[2] + d[3]);
  const double w = act ? -mul_rn(beta, dot) : 0.0;
  double S[8];
#pragma unroll
  for (int B = 0; B < NB; ++B)
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const double2 v = lds2_f64(va + 64 * B + 16 * h);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int s = 2 * h + e, i = 8 * B + s;
        const double xn = fma(e ? v.y : v.x, w, x.ld(i));
        x.st(i, xn);
        const double q = sq_rn(xn);
        if (B == 0) S[s] = s >= r0 ? q : 0.0;
        else S[s] = add_rn(S[s], (B != L || s < r0) ? q : 0.0);
      }
    }
  if (L == 0) {
    double res = -0.0;
#pragma unroll
    for (int s = 1; s < 8; ++s)
      if (s >= r0) res = add_rn(res, sq_rn(x.ld(s)));
    return res;
  }
  double res = p1_combine(S, r0 & 7);
  double T[8];
#define P1_T(LL) case LL: _Pragma("unroll") for (int s = 0; s < 8; ++s) T[s] = sq_rn(x.ld(8 * (LL) + s)); break;
  switch (L) { P1_T(1) P1_T(2) P1_T(3) P1_T(4) P1_T(5) P1_T(6) default: P1_T(7) }
#undef P1_T
#pragma unroll
  for (int s = 0; s < 8; ++s)
    if (s >= r0) res = add_rn(res, T[s]);
  return res;
}

template <class X>
__device__ __forceinline__ void p1_apply_full(const X& x, const double2* vp, double beta, bool act) {
  const uint32_t va = (uint32_t)__cvta_generic_to_shared(vp);
  double d[4];
#pragma unroll
  for (int B = 0; B < 8; ++B) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const double2 v = lds2_f64(va + 64 * B + 16 * h);
      const int s = 2 * h;
      if (B == 0 && s < 4) { d[s] = mul_rn(v.x, x.ld(s)); d[s + 1] = mul_rn(v.y, x.ld(s + 1)); }
      else { d[s & 3] = fma(v.x, x.ld(8 * B + s), d[s & 3]); d[(s + 1) & 3] = fma(v.y, x.ld(8 * B + s + 1), d[(s + 1) & 3]); }
    }
  }
  const double dot = (d[0] + d[1]) + (d[2] + d[3]);
  const double w = act ? mul_rn(beta, dot) : 0.0;
  if (act) { x.st(0, x.ld(0) + w); return; }
#pragma unroll
  for (int B = 0; B < 8; ++B) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const double2 v = lds2_f64(va + 64 * B + 16 * h);
      const int s = 8 * B + 2 * h;
      x.st(s, sub_rn(x.ld(s), mul_rn(v.x, w)));
      x.st(s + 1, sub_rn(x.ld(s + 1), mul_rn(v.y, w)));
    }
  }
}

__global__ void __launch_bounds__(256, 1) k_apply(double* out, long long* cyc, int nwarps_active, int cold) {
  __shared__ __align__(16) double vs[64];
  const int t = threadIdx.x;
  double rr[P1_H];
  for (int e = 0; e < P1_H; ++e) rr[e] = 1.0 + 1e-3 * e + 1e-6 * t;
  if (t < 64) vs[t] = 0.01 * t;
  __syncthreads();
  const P1Reg xr{rr};
  const uint32_t vsa = (uint32_t)__cvta_generic_to_shared(vs);
  double key = 0;
  unsigned ja = t, jb = t + 1;
  int KB = 0;
  for (int k = 0; k < 64; ++k) {
    if ((k & 7) == 0 && k > 0) {
#pragma unroll
      for (int i = 0; i < P1_H - 8; ++i) rr[i] = rr[i + 8];
      ++KB;
    }
    if (cold & 1) asm volatile("mad.lo.u32 %0, %0, %2, %1;\n"
ASMU0_X512 ASMU0_X256 ASMU0_X128 ASMU0_X64 ASMU0_X32 ASMU0_X16 ASMU0_X8 ASMU0_X4 ASMU0_X2 ASMU0_X1
"xor.b32 %1, %1, %0;\n"
"mad.lo.u32 %0, %0, %2, %1;\n"
"xor.b32 %1, %1, %0;\n" : "+r"(ja), "+r"(jb) : "r"(3u));
    __syncthreads();
    long long c0 = clock64();
    if ((t >> 5) < nwarps_active) {
      const int L = 7 - KB;
#if VARIANT == 0
      p1_apply(xr, reinterpret_cast<const double2*>(vs), 1e-3, true, L);
      key += p1_sumsq<false>(xr, (k & 7) + 1, L, 0.0);
#elif VARIANT == 1
      if (L >= 4) key += p1_step_nb<8>(xr, reinterpret_cast<const double2*>(vs), 1e-3, true, L, (k & 7) + 1);
      else key += p1_step_nb<4>(xr, reinterpret_cast<const double2*>(vs), 1e-3, true, L, (k & 7) + 1);
#elif VARIANT == 2
      p1_apply(xr, reinterpret_cast<const double2*>(vs), 1e-3, true, L);
#elif VARIANT == 3
      key += p1_sumsq<false>(xr, (k & 7) + 1, L, 0.0);
#elif VARIANT == 4
      key += p1_step_reg_dispatch(xr, vs, 1e-3, true, true, L, (k & 7) + 1, true);
#endif
    }
    __syncthreads();
    long long c1 = clock64();
    if (t == 0) cyc[k] = c1 - c0;
  }
  for (int e = 0; e < P1_H; ++e) key += rr[e];
  out[t] = key + ja + jb;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 64 * 8);
  long long h[64];
  for (int cold : {0, 1})
  for (int nw : {1}) {
    k_apply<<<1, 256>>>(out, cyc, nw, cold);
    k_apply<<<1, 256>>>(out, cyc, nw, cold);
    cudaMemcpy(h, cyc, 64 * 8, cudaMemcpyDeviceToHost);
    long long s = 0; for (int k = 0; k < 64; ++k) s += h[k];
    printf("variant=" STR(VARIANT) " cold=%d nw=%d: mean %lld cyc/step; k=0 %lld k=1 %lld k=16 %lld k=32 %lld k=48 %lld k=62 %lld\n", cold, nw, s / 64, h[0], h[1], h[16], h[32], h[48], h[62]);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
