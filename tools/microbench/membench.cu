// Memory-system microbenchmarks used to pick the column-pass design.
// 1) float4 copy, 2) column-group copy with W-element (8*W byte) row chunks at a
// 64 KB row stride, 3) L2-resident read bandwidth, 4) DSMEM read bandwidth.
#include <cstdio>
#include <cstdlib>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);exit(1);}}while(0)

__global__ void copy4(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
// buffer viewed as [rows][S] float2; CTA g handles columns [g*W, g*W+W) over all rows.
template <int W>
__global__ void colcopy(const float2* __restrict__ a, float2* __restrict__ b, int rows, int S) {
  int g = blockIdx.x; int c = threadIdx.x % W; int r0 = threadIdx.x / W; int rs = blockDim.x / W;
  const float2* pa = a + (size_t)g * W + c; float2* pb = b + (size_t)g * W + c;
  #pragma unroll 8
  for (int r = r0; r < rows; r += rs) pb[(size_t)r * S] = pa[(size_t)r * S];
}
__global__ void l2read(const float4* __restrict__ a, size_t n, int reps, float* out) {
  float acc = 0.f;
  for (int k = 0; k < reps; ++k)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldcg(a + i); acc += v.x + v.y + v.z + v.w; }
  if (acc == 123.456f) out[0] = acc;
}
template <int CS>
__global__ void __launch_bounds__(512) dsmem_read(int reps, float* out) {
  extern __shared__ float4 sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int n = 65536 / 16;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_float4(i, 1, 2, 3);
  cl.sync();
  unsigned peer = (cl.block_rank() + 1) % CS;
  float4* ps = cl.map_shared_rank(sm, peer);
  float acc = 0.f;
  for (int k = 0; k < reps; ++k)
    for (int i = threadIdx.x; i < n; i += blockDim.x) { float4 v = ps[i]; acc += v.x + v.w; }
  cl.sync();
  if (acc == 123.456f) out[0] = acc;
}

int main() {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1)); float ms;
  size_t bytes = 1ull << 30;
  float4 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes)); CK(cudaMemset(a, 0, bytes));
  float* out; CK(cudaMalloc(&out, 4));
  size_t n4 = bytes / 16;
  for (int it = 0; it < 3; ++it) copy4<<<148 * 8, 512>>>(a, b, n4);
  CK(cudaEventRecord(e0)); for (int it = 0; it < 10; ++it) copy4<<<148 * 8, 512>>>(a, b, n4); CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("copy4 1GiB: %.1f GB/s (r+w)\n", 2.0 * bytes * 10 / (ms * 1e6));
  int S = 8192, rows = (int)(bytes / 8 / S);  // 512 MB region used: rows*S*8 = 1 GiB
  auto runcol = [&](auto kern, int W, int threads) {
    int groups = S / W;
    for (int it = 0; it < 2; ++it) kern<<<groups, threads>>>((const float2*)a, (float2*)b, rows, S);
    CK(cudaEventRecord(e0)); for (int it = 0; it < 5; ++it) kern<<<groups, threads>>>((const float2*)a, (float2*)b, rows, S);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("colcopy W=%3d (%4d B chunks, stride 64KB): %.1f GB/s (r+w)\n", W, W * 8, 2.0 * bytes * 5 / (ms * 1e6));
  };
  runcol(colcopy<1>, 1, 512); runcol(colcopy<2>, 2, 512); runcol(colcopy<4>, 4, 512); runcol(colcopy<8>, 8, 512);
  runcol(colcopy<16>, 16, 512); runcol(colcopy<32>, 32, 512); runcol(colcopy<64>, 64, 512);
  for (size_t l2b : {16ull << 20, 32ull << 20, 64ull << 20}) {
    size_t n = l2b / 16; int reps = 20;
    l2read<<<148 * 4, 512>>>(a, n, 2, out);
    CK(cudaEventRecord(e0)); l2read<<<148 * 4, 512>>>(a, n, reps, out); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("L2 read %zu MB x%d: %.1f GB/s\n", l2b >> 20, reps, (double)l2b * reps / (ms * 1e6));
  }
  auto rund = [&](auto kern, int cs) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(148 / cs * cs); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 65536;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1; int reps = 50;
    CK(cudaLaunchKernelEx(&cfg, kern, 2, out)); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); CK(cudaLaunchKernelEx(&cfg, kern, reps, out)); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("DSMEM read cluster=%d: %.1f GB/s total (%.1f B/clk/SM @1.9GHz)\n", cs, 65536.0 * reps * cfg.gridDim.x / (ms * 1e6),
           65536.0 * reps / (ms * 1e-3) / 1.9e9);
  };
  rund(dsmem_read<2>, 2); rund(dsmem_read<4>, 4); rund(dsmem_read<8>, 8);
  return 0;
}
