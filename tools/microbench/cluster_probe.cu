// Max active clusters per cluster size on this GPU, and an all-to-all DSMEM
// exchange rate: every CTA of a cluster pushes 1/C of a 64 KB buffer to each
// peer (st.shared::cluster through mapped pointers), barrier, repeat.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_dummy(float* p) { extern __shared__ float s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }

template <int C>
__global__ void k_a2a(int iters, float* sink) {
  extern __shared__ float2 buf[];  // 2 x 64 KB: src | dst
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  constexpr int E = 8192;  // elements (64 KB)
  float2* src = buf;
  float2* dst = buf + E;
  for (int i = threadIdx.x; i < E; i += blockDim.x) src[i] = make_float2(i, rank);
  cl.sync();
  for (int it = 0; it < iters; ++it) {
    // element e goes to CTA e / (E/C), slot rank*(E/C) + e % (E/C)
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      const int d = e / (E / C);
      float2* rd = cl.map_shared_rank(dst, d);
      rd[rank * (E / C) + e % (E / C)] = src[e];
    }
    cl.sync();
  }
  if (sink && threadIdx.x == 0) sink[blockIdx.x] = dst[5].x;
}

template <int C>
void run_a2a() {
  auto k = k_a2a<C>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  if (C > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 128 * 1024;
  cfg.attrs = at; cfg.numAttrs = 1;
  int ncl = 0;
  cfg.gridDim = dim3(C);
  cudaOccupancyMaxActiveClusters(&ncl, (void*)k, &cfg);
  cfg.gridDim = dim3(C * ncl);
  float* sink; cudaMalloc(&sink, 4096 * 4);
  const int iters = 200;
  cudaLaunchKernelEx(&cfg, k, iters, sink);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, k, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)C * ncl * iters * 65536.0 * (C - 1) / C;
  printf("cluster %2d: %3d active clusters (%3d CTAs), remote bytes %.2f GB/s total, %.1f B/clk/SM @1.965GHz  err=%s\n",
         C, ncl, C * ncl, bytes / ms / 1e6, bytes / (ms * 1e-3) / (C * ncl) / 1.965e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sizes[] = {1, 2, 4, 8, 16};
  int smems[] = {64, 100, 130, 200};
  for (int sm : smems) {
    for (int C : sizes) {
      cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, sm * 1024);
      cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(C); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = sm * 1024; cfg.attrs = at; cfg.numAttrs = 1;
      int n = 0;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k_dummy, &cfg);
      printf("smem %3d KB cluster %2d: max active clusters %3d -> %3d CTAs (%s)\n", sm, C, n, n * C, cudaGetErrorString(e));
    }
  }
  run_a2a<2>(); run_a2a<4>(); run_a2a<8>(); run_a2a<16>();
  return 0;
}
