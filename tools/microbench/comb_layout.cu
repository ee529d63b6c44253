// 2^30 comb-pass layout probe: TMA copy of 16-comb x 1024-row tiles (128 KB, 1 CTA/SM, as k_comb_tma)
// with the READ and the WRITE side at independent row strides -- which side of pass 0 (rows 8 MB apart)
// costs the time, and what a pass reading a contiguous 128 KB tile and writing 8 KB-strided rows reaches.
// Derived from combcopy.cu. Comb-pass memory ceiling on B200: copy a [rows][width] fp32-complex matrix
// tile by tile, each tile = F adjacent columns x R rows (F*8-byte chunks at a
// stride of width*8 bytes), TMA tensor load -> smem -> TMA tensor store, with
// an S-deep ring. Measures what a strided FFT pass can reach before any math.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b))); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)),
               "r"(ph) : "memory");
}
__device__ __forceinline__ void tload(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(su32(dst)), "l"(m), "r"(c0), "r"(c1), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void tstore(const CUtensorMap* m, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(m), "r"(c0), "r"(c1), "r"(su32(src)) : "memory");
}


// tile t -> input (col chunk ci, row block); output tile position from its own map geometry
__global__ void k_copy2(const __grid_constant__ CUtensorMap in, const __grid_constant__ CUtensorMap out, int R, int BR,
                        int chunks_i, int chunks_o, long long ntiles, int tile_bytes, int F) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + tile_bytes);
  if (threadIdx.x != 0) return;
  mbar_init(bar);
  asm volatile("fence.mbarrier_init.release.cluster;");
  const long long G = gridDim.x;
  auto issue = [&](long long t) {
    const int c = (int)(t % chunks_i), rb = (int)(t / chunks_i);
    mbar_expect(bar, tile_bytes);
    for (int r = 0; r < R; r += BR) tload(sm + (size_t)r * F * 8, &in, c * 2 * F, rb * R + r, bar);
  };
  long long t = blockIdx.x;
  int k = 0;
  if (t < ntiles) issue(t);
  for (; t < ntiles; t += G, ++k) {
    mbar_wait(bar, k & 1);
    const int c = (int)(t % chunks_o), rb = (int)(t / chunks_o);
    for (int r = 0; r < R; r += BR) tstore(&out, c * 2 * F, rb * R + r, sm + (size_t)r * F * 8);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (t + G < ntiles) issue(t + G);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}

int main() {
  const long long total = 1ll << 30;
  float2 *a, *b;
  if (cudaMalloc(&a, total * 8) != cudaSuccess || cudaMalloc(&b, total * 8) != cudaSuccess) { printf("oom\n"); return 1; }
  cudaMemset(a, 0, total * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // {read width, write width, F}: widths in elements per row (F = contiguous tile = one 128 KB block);
  // a tile is F adjacent columns (F * 8-byte lines) x 16384 / F rows = 128 KB
  const long long W[][3] = {{1LL << 20, 1LL << 20, 16}, {1024, 1024, 16}, {1LL << 20, 16, 16}, {1LL << 20, 1LL << 14, 16},
                            {1LL << 20, 1024, 16}, {16, 1024, 16}, {16, 16, 16}, {1LL << 14, 1024, 16},
                            {16, 1LL << 20, 16}, {32, 1LL << 20, 32}, {1024, 1LL << 20, 16}, {1024, 1LL << 20, 32},
                            {1LL << 20, 1LL << 20, 32}, {1024, 1024, 32}};
  auto E = enc();
  for (auto& w : W) {
    const int F = (int)w[2], R = 16384 / F, BR = 256, tile_bytes = F * R * 8;
    CUtensorMap mi, mo;
    cuuint32_t box[2] = {(cuuint32_t)(2 * F), (cuuint32_t)BR};
    cuuint32_t es[2] = {1, 1};
    cuuint64_t di[2] = {(cuuint64_t)w[0] * 2, (cuuint64_t)(total / w[0])}, si[1] = {(cuuint64_t)w[0] * 8};
    cuuint64_t dO[2] = {(cuuint64_t)w[1] * 2, (cuuint64_t)(total / w[1])}, so[1] = {(cuuint64_t)w[1] * 8};
    E(&mi, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, di, si, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    E(&mo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, b, dO, so, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = tile_bytes + 64;
    cudaFuncSetAttribute(k_copy2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int ci = (int)(w[0] / F), co = (int)(w[1] / F);
    const long long ntiles = total / (16384LL);
    k_copy2<<<sms, 32, smem>>>(mi, mo, R, BR, ci, co, ntiles, tile_bytes, F);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 5;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) k_copy2<<<sms, 32, smem>>>(mi, mo, R, BR, ci, co, ntiles, tile_bytes, F);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("F %2d (%3d-byte lines): read rows %8lld B apart, write rows %8lld B apart: %7.3f ms/pass %7.1f GB/s (r+w)  %s\n",
           F, F * 8, w[0] * 8, w[1] * 8, ms / reps, 2.0 * total * 8 * reps / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
