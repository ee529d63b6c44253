// Twiddle-placement A/B for the headline kernel (north-star subsystem 1):
// k_rows_tma<float, 1024, 4 warps, 2-deep ring> over 1024 x 65536 with the
// Stockham stage roots read through the read-only path (TWS = 0, the product
// choice) or staged once per persistent CTA into shared memory (TWS = 1).
//
// Both variants run in ONE process, interleaved A B A B ..., each timed with
// CUDA events over back-to-back launches (the bench method); run the same
// binary under ncu (--cache-control none --clock-control none) to get the
// per-launch gpu__time_duration of the very same launches.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        --expt-relaxed-constexpr -o twiddle_ab twiddle_ab.cu
//   ./twiddle_ab [launches_per_rep=50] [reps=5]
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_1707_07263_b200/csrc/fast_kernels.cuh"

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

constexpr int L = 1024, W = 4, S = 2;
using Cfg = tfb::RowsTmaCfg<float, L, W, S>;
using Sh = Cfg::Sh;

template <bool TWS>
struct Variant {
  static int smem() { return Cfg::SMEM + (TWS ? Cfg::TW_BYTES : 0); }
  static void setup() {
    CK(cudaFuncSetAttribute(tfb::k_rows_tma<float, L, W, S, false, TWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            smem()));
  }
  static int grid(long long nrows) {
    int bps = 0, sms = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, tfb::k_rows_tma<float, L, W, S, false, TWS>, Cfg::THREADS,
                                                     smem()));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const long long chunks = (nrows + Cfg::FPW - 1) / Cfg::FPW;
    return (int)std::min<long long>((chunks + W - 1) / W, (long long)sms * std::max(bps, 1));
  }
  static void launch(const float2* in, float2* out, long long nrows, const float2* tw, int g) {
    tfb::k_rows_tma<float, L, W, S, false, TWS><<<g, Cfg::THREADS, smem()>>>(in, out, nrows, tw, 1.0f);
  }
};

int main(int argc, char** argv) {
  const int per = argc > 1 ? std::atoi(argv[1]) : 50;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 5;
  const long long nrows = 65536;
  const size_t elems = (size_t)nrows * L;
  float2 *in, *out, *tw;
  CK(cudaMalloc(&in, elems * sizeof(float2)));
  CK(cudaMalloc(&out, elems * sizeof(float2)));
  // Stockham stage roots, [q][k] per stage s >= 1: W_{Ns*Rs}^{q k}
  std::vector<float2> h(std::max(Sh::TW_TOTAL, 1));
  for (int s = 1, pos = 0; s < Sh::NST; ++s) {
    const int rs = Sh::radix(s), ns = Sh::ns(s), m = rs * ns;
    for (int q = 0; q < rs; ++q)
      for (int k = 0; k < ns; ++k) {
        const double a = 2.0 * M_PI * (double)(q * k) / (double)m;
        h[pos++] = make_float2((float)std::cos(a), (float)-std::sin(a));
      }
  }
  CK(cudaMalloc(&tw, h.size() * sizeof(float2)));
  CK(cudaMemcpy(tw, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice));
  std::vector<float> xin(2 * elems);
  for (size_t i = 0; i < xin.size(); ++i) xin[i] = (float)((i * 2654435761u) % 1000) / 500.0f - 1.0f;
  CK(cudaMemcpy(in, xin.data(), elems * sizeof(float2), cudaMemcpyHostToDevice));
  Variant<false>::setup();
  Variant<true>::setup();
  const int g0 = Variant<false>::grid(nrows), g1 = Variant<true>::grid(nrows);
  std::printf("grid read-only %d CTAs (smem %d B), smem-staged %d CTAs (smem %d B)\n", g0, Variant<false>::smem(), g1,
              Variant<true>::smem());
  // correctness: both variants give the same bits
  std::vector<float> a(2 * elems), b(2 * elems);
  Variant<false>::launch(in, out, nrows, tw, g0);
  CK(cudaMemcpy(a.data(), out, elems * sizeof(float2), cudaMemcpyDeviceToHost));
  Variant<true>::launch(in, out, nrows, tw, g1);
  CK(cudaMemcpy(b.data(), out, elems * sizeof(float2), cudaMemcpyDeviceToHost));
  std::printf("outputs bitwise equal: %s\n", a == b ? "yes" : "NO");
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<float> t0, t1;
  for (int r = 0; r < reps; ++r) {
    for (int v = 0; v < 2; ++v) {
      for (int w = 0; w < 3; ++w) v ? Variant<true>::launch(in, out, nrows, tw, g1) : Variant<false>::launch(in, out, nrows, tw, g0);
      CK(cudaEventRecord(e0));
      for (int i = 0; i < per; ++i)
        v ? Variant<true>::launch(in, out, nrows, tw, g1) : Variant<false>::launch(in, out, nrows, tw, g0);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      (v ? t1 : t0).push_back(ms * 1000.0f / per);
    }
  }
  auto med = [](std::vector<float> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  std::printf("read-only roots : median %.2f us per launch (", med(t0));
  for (float x : t0) std::printf(" %.2f", x);
  std::printf(" )\nsmem-staged roots: median %.2f us per launch (", med(t1));
  for (float x : t1) std::printf(" %.2f", x);
  std::printf(" )\n");
  return 0;
}
