// 2^30 comb-pass stride probe (pass 0 of [1024]^3 reads rows 8 MB apart, pass 1 rows 8 KB apart):
// TMA copy of 16-comb x 1024-row tiles at both strides, 1 CTA/SM, 128 KB tiles, as k_comb_tma.
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

// tile t -> (column chunk, row block); chunks fastest
__global__ void k_copy(const __grid_constant__ CUtensorMap in, const __grid_constant__ CUtensorMap out, int F, int R,
                       int BR, int chunks, long long ntiles, int S, int tile_bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)S * tile_bytes);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init(&bars[s]);
  asm volatile("fence.mbarrier_init.release.cluster;");
  const long long G = gridDim.x;
  auto issue = [&](long long t, int s) {
    const int c = (int)(t % chunks), rb = (int)(t / chunks);
    mbar_expect(&bars[s], tile_bytes);
    for (int r = 0; r < R; r += BR) tload(sm + (size_t)s * tile_bytes + (size_t)r * F * 8, &in, c * F * 2, rb * R + r, &bars[s]);
  };
  long long t = blockIdx.x;
  int k = 0;
  for (int s = 0; s < S && t + s * G < ntiles; ++s) issue(t + s * G, s);
  for (; t < ntiles; t += G, ++k) {
    const int s = k % S;
    mbar_wait(&bars[s], (k / S) & 1);
    const int c = (int)(t % chunks), rb = (int)(t / chunks);
    for (int r = 0; r < R; r += BR) tstore(&out, c * F * 2, rb * R + r, sm + (size_t)s * tile_bytes + (size_t)r * F * 8);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (t + S * G < ntiles) issue(t + S * G, s);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}


int main(int argc, char** argv) {
  const int lg = argc > 1 ? atoi(argv[1]) : 30;
  const long long total = 1ll << lg;  // complex fp32 elements
  float2 *a, *b;
  if (cudaMalloc(&a, total * 8) != cudaSuccess || cudaMalloc(&b, total * 8) != cudaSuccess) { printf("oom\n"); return 1; }
  cudaMemset(a, 0, total * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct Case { long long width; int F, R, S, cpsm; bool inplace; };
  std::vector<Case> cases;
  for (long long w : {1024LL, 1LL << 14, 1LL << 17, 1LL << 20})
    for (int ip = 0; ip < 2; ++ip) {
      cases.push_back({w, 16, 1024, 1, 1, (bool)ip});
      cases.push_back({w, 16, 512, 1, 3, (bool)ip});
    }
  auto E = enc();
  for (auto c : cases) {
    const long long rows = total / c.width;
    CUtensorMap mi, mo;
    cuuint64_t dims[2] = {(cuuint64_t)c.width * 2, (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)c.width * 8};
    const int BR = c.R < 256 ? c.R : 256;
    const int boxc = c.F * 2;
    cuuint32_t box[2] = {(cuuint32_t)boxc, (cuuint32_t)BR};
    cuuint32_t es[2] = {1, 1};
    float2* dst = c.inplace ? a : b;
    E(&mi, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    E(&mo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dst, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int tile_bytes = c.F * c.R * 8;
    const int smem = c.S * tile_bytes + 64;
    cudaFuncSetAttribute(k_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int chunks = (int)(c.width / c.F);
    const long long ntiles = (long long)chunks * (rows / c.R);
    const int grid = sms * c.cpsm;
    k_copy<<<grid, 32, smem>>>(mi, mo, c.F, c.R, BR, chunks, ntiles, c.S, tile_bytes);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int i = 0; i < reps; ++i) k_copy<<<grid, 32, smem>>>(mi, mo, c.F, c.R, BR, chunks, ntiles, c.S, tile_bytes);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("2^%d width %8lld (stride %8lld B) F %d R %4d cta/sm %d %s: %7.3f ms/pass %7.1f GB/s (r+w)  %s\n", lg, c.width,
           c.width * 8, c.F, c.R, c.cpsm, c.inplace ? "in-place" : "out-of-place", ms / reps,
           2.0 * total * 8 * reps / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
