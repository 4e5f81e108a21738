// Cluster all-to-all exchange latency on B200: every CTA of a C-CTA cluster
// sends 16 bytes to every CTA (itself included) and waits for all C packets,
// N dependent rounds.  Mechanisms:
//   0  st.async + mbarrier complete_tx (expect_tx armed by the receiver)
//   1  "LL" packets: st.shared::cluster.v2.u64 {payload, tag}; the receiver
//      polls its own shared memory until the tag equals the round number
//   2  barrier.cluster arrive.release / wait.acquire, then ld.shared::cluster
//   3  st.shared::cluster.u64 payload + remote mbarrier.arrive.release.cluster
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_xchg probe_xchg.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}

template <int MECH>
__global__ void xchg(int N, long long* out, unsigned long long* sink) {
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), c = cl.block_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ __align__(16) unsigned long long slot[2][16][2];
  __shared__ __align__(8) unsigned long long bar[2];
  const uint32_t sl = (uint32_t)__cvta_generic_to_shared(&slot[0][0][0]);
  const uint32_t br = (uint32_t)__cvta_generic_to_shared(&bar[0]);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 64; ++i) (&slot[0][0][0])[i] = 0ull;
    const int cnt = MECH == 3 ? C : 1;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(br), "r"(cnt) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(br + 8), "r"(cnt) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  unsigned long long acc = 0;
  const long long t0 = clock64();
  if (warp == 0) {
    for (int k = 1; k <= N; ++k) {
      const int buf = k & 1;
      const uint32_t myslot = sl + (buf * 16 + c) * 16;
      const unsigned long long payload = acc + k + c;
      if (MECH == 0) {
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(br + 8 * buf), "r"(16 * C) : "memory");
        if (lane < C)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.u64 [%0], {%1, %2}, [%3];"
                       :: "r"(mapa(myslot, lane)), "l"(payload), "l"((unsigned long long)k), "r"(mapa(br + 8 * buf, lane)) : "memory");
        const uint32_t par = ((k >> 1) & 1) ^ (buf == 1 ? 0 : 1);   // phase parity of bar[buf]: rounds using it: buf=1: k=1,3,5..; buf=0: k=2,4,..
        uint32_t ok;
        do {
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(ok) : "r"(br + 8 * buf), "r"(par) : "memory");
        } while (!ok);
      } else if (MECH == 1) {
        if (lane < C)
          asm volatile("st.shared::cluster.v2.u64 [%0], {%1, %2};" :: "r"(mapa(myslot, lane)), "l"(payload), "l"((unsigned long long)k) : "memory");
        if (lane < C) {
          unsigned long long p, tg;
          do {
            asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(p), "=l"(tg) : "r"(sl + (buf * 16 + lane) * 16) : "memory");
          } while (tg != (unsigned long long)k);
        }
        __syncwarp();
      } else if (MECH == 2) {
        if (lane == 0) slot[buf][c][0] = payload;
        __syncwarp();
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      } else {
        if (lane < C) {
          asm volatile("st.shared::cluster.u64 [%0], %1;" :: "r"(mapa(myslot, lane)), "l"(payload) : "memory");
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(mapa(br + 8 * buf, lane)) : "memory");
        }
        const uint32_t par = ((k >> 1) & 1) ^ (buf == 1 ? 0 : 1);
        uint32_t ok;
        do {
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(ok) : "r"(br + 8 * buf), "r"(par) : "memory");
        } while (!ok);
      }
      // consume: max over the C payloads (dependent chain into the next round)
      unsigned long long v = 0;
      if (lane < C) {
        if (MECH == 2) {
          asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(mapa(myslot, lane)) : "memory");
        } else {
          v = *(volatile unsigned long long*)&slot[buf][lane][0];
        }
      }
      for (int o = 16; o; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = v > w ? v : w;
      }
      acc = v & 0xff;
    }
  }
  const long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) {
    out[blockIdx.x] = t1 - t0;
    sink[blockIdx.x] = acc;
  }
}

template <int MECH>
void run(int C, int N, long long* d_out, unsigned long long* d_sink) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(32);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(xchg<MECH>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaError_t e = cudaLaunchKernelEx(&cfg, xchg<MECH>, N, d_out, d_sink);
    if (e != cudaSuccess) { printf("mech %d C %d launch: %s\n", MECH, C, cudaGetErrorString(e)); return; }
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mech %d C %d run: %s\n", MECH, C, cudaGetErrorString(e)); return; }
  }
  long long h[16];
  cudaMemcpy(h, d_out, sizeof(long long) * C, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < C; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("mech %d C %2d: %.0f cycles per all-to-all round\n", MECH, C, (double)mx / N);
}

int main() {
  long long* d_out;
  unsigned long long* d_sink;
  cudaMalloc(&d_out, 16 * sizeof(long long));
  cudaMalloc(&d_sink, 16 * sizeof(unsigned long long));
  const int N = 2000;
  for (int C : {2, 4, 8, 16}) {
    run<0>(C, N, d_out, d_sink);
    run<1>(C, N, d_out, d_sink);
    run<2>(C, N, d_out, d_sink);
    run<3>(C, N, d_out, d_sink);
  }
  return 0;
}
