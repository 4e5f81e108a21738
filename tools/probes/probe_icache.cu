// Instruction-cache probe: a loop whose body is N independent integer adds
// (4 chains); cycles per instruction vs N shows the i-cache capacities.
#include <cstdio>
// Repeated asm bodies are spelled with doubling macros (NAME_X<count>).
#define ASMU0_X1 "xor.b32 %1, %1, %0;\n" "mad.lo.u32 %2, %2, %4, %3;\n" "xor.b32 %3, %3, %2;\n" "mad.lo.u32 %0, %0, %4, %1;\n"
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
__global__ void icache_256(unsigned* out, long long* cyc, int iters, unsigned d) {
  unsigned a = threadIdx.x, b = a + 1, c = a + 2, e = a + 3;
  long long t0 = 0;
  for (int it = 0; it < iters; ++it) {
    if (it == 1) t0 = clock64();
    asm volatile("mad.lo.u32 %0, %0, %4, %1;\n"
ASMU0_X32 ASMU0_X16 ASMU0_X8 ASMU0_X4 ASMU0_X2 ASMU0_X1
"xor.b32 %1, %1, %0;\n"
"mad.lo.u32 %2, %2, %4, %3;\n"
"xor.b32 %3, %3, %2;\n" : "+r"(a), "+r"(b), "+r"(c), "+r"(e) : "r"(d));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a + b + c + e;
}
__global__ void icache_512(unsigned* out, long long* cyc, int iters, unsigned d) {
  unsigned a = threadIdx.x, b = a + 1, c = a + 2, e = a + 3;
  long long t0 = 0;
  for (int it = 0; it < iters; ++it) {
    if (it == 1) t0 = clock64();
    asm volatile("mad.lo.u32 %0, %0, %4, %1;\n"
ASMU0_X64 ASMU0_X32 ASMU0_X16 ASMU0_X8 ASMU0_X4 ASMU0_X2 ASMU0_X1
"xor.b32 %1, %1, %0;\n"
"mad.lo.u32 %2, %2, %4, %3;\n"
"xor.b32 %3, %3, %2;\n" : "+r"(a), "+r"(b), "+r"(c), "+r"(e) : "r"(d));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a + b + c + e;
}
__global__ void icache_1024(unsigned* out, long long* cyc, int iters, unsigned d) {
  unsigned a = threadIdx.x, b = a + 1, c = a + 2, e = a + 3;
  long long t0 = 0;
  for (int it = 0; it < iters; ++it) {
    if (it == 1) t0 = clock64();
    asm volatile("mad.lo.u32 %0, %0, %4, %1;\n"
ASMU0_X128 ASMU0_X64 ASMU0_X32 ASMU0_X16 ASMU0_X8 ASMU0_X4 ASMU0_X2 ASMU0_X1
"xor.b32 %1, %1, %0;\n"
"mad.lo.u32 %2, %2, %4, %3;\n"
"xor.b32 %3, %3, %2;\n" : "+r"(a), "+r"(b), "+r"(c), "+r"(e) : "r"(d));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a + b + c + e;
}
__global__ void icache_1536(unsigned* out, long long* cyc, int iters, unsigned d) {
  unsigned a = threadIdx.x, b = a + 1, c = a + 2, e = a + 3;
  long long t0 = 0;
  for (int it = 0; it < iters; ++it) {
    if (it == 1) t0 = clock64();
    asm volatile("mad.lo.u32 %0, %0, %4, %1;\n"
ASMU0_X256 ASMU0_X64 ASMU0_X32 ASMU0_X16 ASMU0_X8 ASMU0_X4 ASMU0_X2 ASMU0_X1
"xor.b32 %1, %1, %0;\n"
"mad.lo.u32 %2, %2, %4, %3;\n"
"xor.b32 %3, %3, %2;\n" : "+r"(a), "+r"(b), "+r"(c), "+r"(e) : "r"(d));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a + b + c + e;
}
__global__ void icache_2048(unsigned* out, long long* cyc, int iters, unsigned d) {
  unsigned a = threadIdx.x, b = a + 1, c = a + 2, e = a + 3;
  long long t0 = 0;
  for (int it = 0; it < iters; ++it) {
    if (it == 1) t0 = clock64();
    asm volatile("mad.lo.u32 %0, %0, %4, %1;\n"
ASMU0_X256 ASMU0_X128 ASMU0_X64 ASMU0_X32 ASMU0_X16 ASMU0_X8 ASMU0_X4 ASMU0_X2 ASMU0_X1
"xor.b32 %1, %1, %0;\n"
"mad.lo.u32 %2, %2, %4, %3;\n"
"xor.b32 %3, %3, %2;\n" : "+r"(a), "+r"(b), "+r"(c), "+r"(e) : "r"(d));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a + b + c + e;
}
__global__ void icache_3072(unsigned* out, long long* cyc, int iters, unsigned d) {
  unsigned a = threadIdx.x, b = a + 1, c = a + 2, e = a + 3;
  long long t0 = 0;
  for (int it = 0; it < iters; ++it) {
    if (it == 1) t0 = clock64();
    asm volatile("mad.lo.u32 %0, %0, %4, %1;\n"
ASMU0_X512 ASMU0_X128 ASMU0_X64 ASMU0_X32 ASMU0_X16 ASMU0_X8 ASMU0_X4 ASMU0_X2 ASMU0_X1
"xor.b32 %1, %1, %0;\n"
"mad.lo.u32 %2, %2, %4, %3;\n"
"xor.b32 %3, %3, %2;\n" : "+r"(a), "+r"(b), "+r"(c), "+r"(e) : "r"(d));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a + b + c + e;
}
__global__ void icache_4096(unsigned* out, long long* cyc, int iters, unsigned d) {
  unsigned a = threadIdx.x, b = a + 1, c = a + 2, e = a + 3;
  long long t0 = 0;
  for (int it = 0; it < iters; ++it) {
    if (it == 1) t0 = clock64();
    asm volatile("mad.lo.u32 %0, %0, %4, %1;\n"
ASMU0_X512 ASMU0_X256 ASMU0_X128 ASMU0_X64 ASMU0_X32 ASMU0_X16 ASMU0_X8 ASMU0_X4 ASMU0_X2 ASMU0_X1
"xor.b32 %1, %1, %0;\n"
"mad.lo.u32 %2, %2, %4, %3;\n"
"xor.b32 %3, %3, %2;\n" : "+r"(a), "+r"(b), "+r"(c), "+r"(e) : "r"(d));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a + b + c + e;
}
__global__ void icache_8192(unsigned* out, long long* cyc, int iters, unsigned d) {
  unsigned a = threadIdx.x, b = a + 1, c = a + 2, e = a + 3;
  long long t0 = 0;
  for (int it = 0; it < iters; ++it) {
    if (it == 1) t0 = clock64();
    asm volatile("mad.lo.u32 %0, %0, %4, %1;\n"
ASMU0_X1024 ASMU0_X512 ASMU0_X256 ASMU0_X128 ASMU0_X64 ASMU0_X32 ASMU0_X16 ASMU0_X8 ASMU0_X4 ASMU0_X2 ASMU0_X1
"xor.b32 %1, %1, %0;\n"
"mad.lo.u32 %2, %2, %4, %3;\n"
"xor.b32 %3, %3, %2;\n" : "+r"(a), "+r"(b), "+r"(c), "+r"(e) : "r"(d));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a + b + c + e;
}
int main() {
  unsigned* out; long long* cyc; cudaMalloc(&out, 4096 * 4); cudaMalloc(&cyc, 64);
  long long h;
  for (int nw : {1, 4}) {
    icache_256<<<1, 32 * nw>>>(out, cyc, 21, 3u);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("N=%5d warps=%d: %.2f cycles/instr (per warp-iteration)\n", 256, nw, (double)h / 20 / 256);
  }
  for (int nw : {1, 4}) {
    icache_512<<<1, 32 * nw>>>(out, cyc, 21, 3u);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("N=%5d warps=%d: %.2f cycles/instr (per warp-iteration)\n", 512, nw, (double)h / 20 / 512);
  }
  for (int nw : {1, 4}) {
    icache_1024<<<1, 32 * nw>>>(out, cyc, 21, 3u);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("N=%5d warps=%d: %.2f cycles/instr (per warp-iteration)\n", 1024, nw, (double)h / 20 / 1024);
  }
  for (int nw : {1, 4}) {
    icache_1536<<<1, 32 * nw>>>(out, cyc, 21, 3u);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("N=%5d warps=%d: %.2f cycles/instr (per warp-iteration)\n", 1536, nw, (double)h / 20 / 1536);
  }
  for (int nw : {1, 4}) {
    icache_2048<<<1, 32 * nw>>>(out, cyc, 21, 3u);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("N=%5d warps=%d: %.2f cycles/instr (per warp-iteration)\n", 2048, nw, (double)h / 20 / 2048);
  }
  for (int nw : {1, 4}) {
    icache_3072<<<1, 32 * nw>>>(out, cyc, 21, 3u);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("N=%5d warps=%d: %.2f cycles/instr (per warp-iteration)\n", 3072, nw, (double)h / 20 / 3072);
  }
  for (int nw : {1, 4}) {
    icache_4096<<<1, 32 * nw>>>(out, cyc, 21, 3u);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("N=%5d warps=%d: %.2f cycles/instr (per warp-iteration)\n", 4096, nw, (double)h / 20 / 4096);
  }
  for (int nw : {1, 4}) {
    icache_8192<<<1, 32 * nw>>>(out, cyc, 21, 3u);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("N=%5d warps=%d: %.2f cycles/instr (per warp-iteration)\n", 8192, nw, (double)h / 20 / 8192);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
