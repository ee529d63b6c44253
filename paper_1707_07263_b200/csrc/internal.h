// Host-side internals shared by the tilefft_b200 translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "exact_kernels.cuh"
#include "fast_kernels.cuh"
#include "twolevel.cuh"
#include "../../include/tilefft_b200.h"

namespace tfb_host {

extern thread_local std::string g_err;
int fail(int code, const char* fmt, ...);

#define CUDA_TRY(expr)                                                                             \
  do {                                                                                             \
    cudaError_t e_ = (expr);                                                                       \
    if (e_ != cudaSuccess) return ::tfb_host::fail(TILEFFT_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

// Opt a kernel into >48 KB dynamic shared memory (once per function/device).
int ensure_smem(const void* fn, int bytes);

enum PassKind { K_ROWS = 0, K_COMB1D = 1, K_COMBAX = 2, K_FINALT = 3, K_EXACT = 4, K_BITREV = 5, K_LEVEL = 6, K_TWO = 7 };

struct Pass {
  PassKind kind;
  int L;
  int src, dst;              // 0 = user input, 1 = user output, 2 = workspace
  long long grid;
  size_t smem;
  tfb::CombArgs comb;
  tfb::FinalArgs fin;
  tfb::ExactArgs ex;
  long long nrows;           // K_ROWS
  size_t tw_off;             // offset (elements) of this L's Stockham table in the table buffer
  size_t wc_off, wf_off;     // inter-pass tables
  bool twid;
  bool final_pass;           // the pass that applies the inverse scale
  bool no_tma;               // force the register-only K_ROWS variant
  int level;                 // K_LEVEL: radix-2 level (h = 2^level)
  long long lw_n, lw_total;  // K_BITREV/K_LEVEL: transform length, elements (or half) in the batch
  // K_TWO (two-level pass through L2, twolevel.cuh)
  tfb::TwoArgs two;
  int la, lb, outt;
  long long two_cols, two_es_in;  // columns along the axis and their element stride (input)
  size_t twl_off;                 // W_L^e table (L entries)
  int two_ctas;                   // persistent grid
};

// Distributed four-step, pass 1 on one rank (see tilefft_dist_* in the C ABI).
struct DistPass1 {
  int L;                    // N1 (column FFT length)
  long long C;              // columns per rank (N2 / G)
  size_t tw_off, wc_off, wf_off;
  int fb;
  uint32_t m_mask;          // N - 1
  tfb::CombTmaArgs a;       // mode-2 arguments (peers, pitch, col_off, r_off, ...)
};

// Kernel launchers, explicitly instantiated in kern_*.cu (one TU per
// precision/direction so the heavy template instantiation builds in parallel).
template <typename Real, bool INV>
int launch_fast(const Pass& ps, const void* in, void* out, const void* tb, const void* tb64, Real scale,
                cudaStream_t st);
template <typename Real>
int launch_exact(const Pass& ps, const void* in, void* out, const void* tb, Real scale, int conj_in, int conj_out,
                 cudaStream_t st);

template <typename Real>
int launch_levelwise(const Pass& ps, const void* in, void* out, const void* tb, Real scale, int conj_in, int conj_out,
                     cudaStream_t st);
template <typename Real>
int launch_exchange(const void* in, void* out, const tfb::ExchangeArgs& a, cudaStream_t st);
template <typename Real>
int launch_interstage(const void* in, void* out, long long rows, long long cols, long long row0, long long rps,
                      long long sub_len, const void* tbl, long long tstride, cudaStream_t st);

template <typename Real, bool INV>
int launch_dist_pass1(const DistPass1& d, const void* in, const void* tb, const void* tb64, Real scale,
                      cudaStream_t st);

extern template int launch_fast<float, false>(const Pass&, const void*, void*, const void*, const void*, float, cudaStream_t);
extern template int launch_fast<float, true>(const Pass&, const void*, void*, const void*, const void*, float, cudaStream_t);
extern template int launch_fast<double, false>(const Pass&, const void*, void*, const void*, const void*, double, cudaStream_t);
extern template int launch_fast<double, true>(const Pass&, const void*, void*, const void*, const void*, double, cudaStream_t);
extern template int launch_dist_pass1<float, false>(const DistPass1&, const void*, const void*, const void*, float,
                                                   cudaStream_t);
extern template int launch_dist_pass1<float, true>(const DistPass1&, const void*, const void*, const void*, float,
                                                  cudaStream_t);
extern template int launch_dist_pass1<double, false>(const DistPass1&, const void*, const void*, const void*, double,
                                                    cudaStream_t);
extern template int launch_dist_pass1<double, true>(const DistPass1&, const void*, const void*, const void*, double,
                                                   cudaStream_t);
extern template int launch_exact<float>(const Pass&, const void*, void*, const void*, float, int, int, cudaStream_t);
extern template int launch_levelwise<float>(const Pass&, const void*, void*, const void*, float, int, int,
                                           cudaStream_t);
extern template int launch_levelwise<double>(const Pass&, const void*, void*, const void*, double, int, int,
                                            cudaStream_t);
extern template int launch_exchange<float>(const void*, void*, const tfb::ExchangeArgs&, cudaStream_t);
extern template int launch_exchange<double>(const void*, void*, const tfb::ExchangeArgs&, cudaStream_t);
extern template int launch_interstage<float>(const void*, void*, long long, long long, long long, long long, long long,
                                            const void*, long long, cudaStream_t);
extern template int launch_interstage<double>(const void*, void*, long long, long long, long long, long long,
                                             long long, const void*, long long, cudaStream_t);
extern template int launch_exact<double>(const Pass&, const void*, void*, const void*, double, int, int,
                                         cudaStream_t);

}  // namespace tfb_host
