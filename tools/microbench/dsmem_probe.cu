// DSMEM all-to-all exchange rates on B200, 1 CTA per SM, 64 KB pushed per CTA
// per iteration (1/C to each CTA of the cluster, including itself):
//   push16 : st.shared::cluster (generic mapped pointer) 16-byte stores
//   pull16 : 16-byte loads from the peers' buffers
//   bulk   : cp.async.bulk.shared::cluster.shared::cta (TMA engine) with
//            mbarrier complete_tx on the receiver
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int C, int MODE>
__global__ void k_x(int iters, float* sink) {
  extern __shared__ __align__(128) float4 buf[];  // src 64 KB | dst 64 KB | mbar
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  constexpr int E = 4096;  // float4 elements = 64 KB
  constexpr int P = E / C;
  float4* src = buf;
  float4* dst = buf + E;
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 2 * E);
  for (int i = threadIdx.x; i < E; i += blockDim.x) src[i] = make_float4(i, rank, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cl.sync();
  for (int it = 0; it < iters; ++it) {
    if constexpr (MODE == 0) {
      for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const int d = e / P;
        float4* rd = cl.map_shared_rank(dst, d);
        rd[rank * P + e % P] = src[e];
      }
      cl.sync();
    } else if constexpr (MODE == 1) {
      float4 acc = make_float4(0, 0, 0, 0);
      for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const int s = e / P;
        const float4* rs = cl.map_shared_rank(src, s);
        float4 v = rs[rank * P + e % P];
        dst[e] = v;
      }
      cl.sync();
    } else {
      // receiver: expect C*P*16 bytes on its own barrier
      if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(E * 16));
      cl.sync();  // all receivers armed
      if (threadIdx.x < C) {
        const int d = threadIdx.x;
        uint32_t rdst, rbar;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(su32(dst + rank * P)), "r"(d));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(su32(bar)), "r"(d));
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(rdst), "r"(su32(src + d * P)), "r"(P * 16), "r"(rbar) : "memory");
      }
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                   ::"r"(su32(bar)), "r"(it & 1) : "memory");
      cl.sync();
    }
  }
  if (sink && threadIdx.x == 0) sink[blockIdx.x] = dst[5].x;
}

template <int C, int MODE>
void run(int threads) {
  auto k = k_x<C, MODE>;
  const int smem = 128 * 1024 + 16;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at; cfg.numAttrs = 1;
  int ncl = 0;
  cfg.gridDim = dim3(C);
  cudaOccupancyMaxActiveClusters(&ncl, (void*)k, &cfg);
  cfg.gridDim = dim3(C * ncl);
  float* sink; cudaMalloc(&sink, 4096 * 4);
  const int iters = 400;
  cudaLaunchKernelEx(&cfg, k, iters, sink);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, k, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)C * ncl * iters * 65536.0 * (C - 1) / C;
  const char* nm[] = {"push16", "pull16", "bulk"};
  printf("%-7s cluster %2d threads %4d: %3d CTAs, remote %.0f GB/s total, %.1f B/clk/SM, %.2f us/iter  err=%s\n", nm[MODE],
         C, threads, C * ncl, bytes / ms / 1e6, bytes / (ms * 1e-3) / (C * ncl) / 1.965e9, ms * 1e3 / iters,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<2, 0>(512); run<4, 0>(512); run<8, 0>(512); run<8, 0>(1024);
  run<2, 1>(512); run<4, 1>(512); run<8, 1>(512); run<8, 1>(1024);
  run<2, 2>(128); run<4, 2>(128); run<8, 2>(128);
  return 0;
}
