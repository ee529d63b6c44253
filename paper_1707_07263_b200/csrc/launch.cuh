// Kernel launchers (templates); instantiated per precision/direction in kern_*.cu.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include <cudaTypedefs.h>

#include "internal.h"

namespace tfb_host {

inline bool env_set(const char* name) {
  const char* e = std::getenv(name);
  return e && *e && *e != '0';
}

inline int env_int_or(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && *e) ? std::atoi(e) : dflt;
}

inline int sm_count() {
  static int n[16] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!n[dev & 15]) cudaDeviceGetAttribute(&n[dev & 15], cudaDevAttrMultiProcessorCount, dev);
  return n[dev & 15];
}

// FFTs per CTA for K_ROWS: 8 warps of work for L <= 1024 (fp32), one FFT per CTA above.
template <typename Real>
constexpr int rows_fpc(int L) {
  constexpr int RM = tfb::RmaxOf<Real>::v;
  if (L >= 2048) return 1;
  const int T = L < RM ? 1 : L / RM;
  const int f = 256 / T;
  return f < 1 ? 1 : f;
}

// TMA-staged persistent rows kernel configuration (warps per CTA, ring depth)
constexpr int kRowsWarps = 4;
constexpr int kRowsStages = 2;

// one persistent TMA rows launch with W warps per CTA and an S-deep ring per warp
template <typename Real, int L, bool INV, int W, int S>
int launch_rows_tma(const Pass& ps, const void* in, void* out, const void* tw, Real scale, cudaStream_t st) {
  using Cfg = tfb::RowsTmaCfg<Real, L, W, S>;
  auto k = tfb::k_rows_tma<Real, L, W, S, INV>;
  const int smem = Cfg::SMEM;
  if (int rc = ensure_smem((const void*)k, smem)) return rc;
  static int blocks_per_sm[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& bps = blocks_per_sm[dev & 15];
  if (!bps) {
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, Cfg::THREADS, smem));
    if (bps < 1) bps = 1;
  }
  const long long chunks = (ps.nrows + Cfg::FPW - 1) / Cfg::FPW;
  const long long want = (chunks + W - 1) / W;
  const long long grid = std::max<long long>(1, std::min<long long>(want, (long long)sm_count() * bps));
  k<<<(unsigned)grid, Cfg::THREADS, smem, st>>>((const tfb::C2<Real>*)in, (tfb::C2<Real>*)out, ps.nrows,
                                                (const tfb::C2<Real>*)tw + ps.tw_off, scale);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <typename Real, int L, bool INV>
int launch_rows(const Pass& ps, const void* in, void* out, const void* tw, const void*, Real scale, cudaStream_t st) {
  constexpr int RM = tfb::RmaxOf<Real>::v;
  constexpr int T = (L < RM ? 1 : L / RM);
  const bool aligned = ((uintptr_t)in % 16 == 0) && ((uintptr_t)out % 16 == 0) && (L * sizeof(tfb::C2<Real>)) % 16 == 0;
  if constexpr (T <= 32) {
    if (aligned && !ps.no_tma) {
      // stage roots through the read-only path, not shared memory (measured:
      // profiles/r02_twiddle_ab.txt, tools/microbench/twiddle_ab.cu);
      return launch_rows_tma<Real, L, INV, kRowsWarps, kRowsStages>(ps, in, out, tw, scale, st);
    }
  }
  if constexpr (std::is_same<Real, float>::value && L >= 2048) {
    if (aligned && !ps.no_tma) {
      using CfgP = tfb::RowsPfCfg<L>;
      // (3 CTAs per SM -- register cap 80, 316 bytes of spills -- measured 604 vs 519 us for 8192^2)
      auto k = tfb::k_rows_pf<L, INV>;
      if (int rc = ensure_smem((const void*)k, CfgP::SMEM)) return rc;
      int bps = 0;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, CfgP::THREADS, CfgP::SMEM));
      const long long grid = std::max<long long>(1, std::min<long long>(ps.nrows, (long long)sm_count() * std::max(bps, 1)));
      k<<<(unsigned)grid, CfgP::THREADS, CfgP::SMEM, st>>>((const float2*)in, (float2*)out, ps.nrows,
                                                           (const float2*)tw + ps.tw_off, (float)scale);
      CUDA_TRY(cudaGetLastError());
      return 0;
    }
  }
  constexpr int FPC = rows_fpc<Real>(L);
  using Cfg = tfb::RowsCfg<Real, L, FPC>;
  auto k = tfb::k_rows<Real, L, FPC, INV>;
  if (int rc = ensure_smem((const void*)k, Cfg::SMEM)) return rc;
  const long long grid = (ps.nrows + FPC - 1) / FPC;
  k<<<(unsigned)grid, Cfg::THREADS, Cfg::SMEM, st>>>((const tfb::C2<Real>*)in, (tfb::C2<Real>*)out, ps.nrows,
                                                     (const tfb::C2<Real>*)tw + ps.tw_off, scale);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// Strided comb tile as a 4-D tensor {column (8-byte words), n, rr, group}.
template <typename Real, int L, int F_ = tfb::FOf<Real>::v>
bool encode_comb_map(CUtensorMap* map, const Pass& ps, const void* in) {
  using Cfg = tfb::CombTmaCfg<Real, L, F_>;
  constexpr int W = (int)sizeof(tfb::C2<Real>) / 8;
  auto enc = tensor_map_encoder();
  if (!enc || ((uintptr_t)in % 16) != 0) return false;
  const tfb::CombArgs& a = ps.comb;
  const long long B = a.ntiles / (a.chunks * a.groups_per_batch);
  cuuint64_t dims[4], strides[3];
  const long long vb = (long long)sizeof(tfb::C2<Real>);
  if (ps.kind == K_COMB1D && a.in_t) {
    // T[c1][k0][c2] (CombArgs::t_l2): {column c2, comb step c1, group k0, batch item}
    dims[0] = (cuuint64_t)(a.rps * W);
    dims[1] = L;
    dims[2] = (cuuint64_t)a.groups_per_batch;
    dims[3] = (cuuint64_t)B;
    strides[0] = (cuuint64_t)(a.groups_per_batch * a.rps * vb);
    strides[1] = (cuuint64_t)(a.rps * vb);
    strides[2] = (cuuint64_t)(a.bstride * vb);
  } else if (ps.kind == K_COMB1D) {
    dims[0] = (cuuint64_t)(a.rps * W);
    dims[1] = L;
    dims[2] = 1;
    dims[3] = (cuuint64_t)(B * a.groups_per_batch);
    strides[0] = (cuuint64_t)(a.rps * vb);
    strides[1] = (cuuint64_t)(a.sub_len * vb);
    strides[2] = (cuuint64_t)(a.sub_len * vb);
  } else {
    dims[0] = (cuuint64_t)(a.es * W);
    dims[1] = L;
    dims[2] = (cuuint64_t)a.rps;
    dims[3] = (cuuint64_t)(B * (a.groups_per_batch / a.rps));
    strides[0] = (cuuint64_t)(a.rps * a.es * vb);
    strides[1] = (cuuint64_t)(a.es * vb);
    strides[2] = (cuuint64_t)(a.sub_len * a.es * vb);
  }
  for (int i = 0; i < 3; ++i)
    if (strides[i] % 16 != 0 || strides[i] >= (1ull << 40)) return false;
  if (dims[0] < (cuuint64_t)(Cfg::F * W) && ps.kind == K_COMB1D) return false;
  if (ps.kind == K_COMB1D && a.split_q > 0) {
    // blocks layout: {column, n1 % q, n1 / q, batch item, 1}; a box of BL rows spans min(BL, q) x BL/min(BL, q)
    const long long q = a.split_q;
    if (L % q != 0) return false;
    const long long qb = q < Cfg::BL ? q : Cfg::BL;
    const cuuint64_t d5[5] = {(cuuint64_t)(a.rps * W), (cuuint64_t)q, (cuuint64_t)(L / q), (cuuint64_t)B, 1};
    const cuuint64_t s5[4] = {(cuuint64_t)(a.rps * vb), (cuuint64_t)(a.split_stride * vb),
                              (cuuint64_t)(a.split_bstride * vb), (cuuint64_t)(a.split_bstride * vb)};
    for (int i = 0; i < 4; ++i)
      if (s5[i] % 16 != 0 || s5[i] >= (1ull << 40)) return false;
    const cuuint32_t b5[5] = {(cuuint32_t)(Cfg::F * W), (cuuint32_t)qb, (cuuint32_t)(Cfg::BL / qb), 1, 1};
    const cuuint32_t e5[5] = {1, 1, 1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, const_cast<void*>(in), d5, s5, b5, e5,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  const cuuint32_t box[4] = {(cuuint32_t)(Cfg::F * W), (cuuint32_t)Cfg::BL, 1, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<void*>(in), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Persistent TMA-pipelined comb pass (K_COMB_TMA) with F-comb tiles.
template <typename Real, int L, bool INV, int F, bool IP = false>
int launch_comb_tma(const Pass& ps, const CUtensorMap& map, void* out, const void* tb, const void* tb64, Real scale,
                    cudaStream_t st) {
  using Cfg = tfb::CombTmaCfg<Real, L, F, IP>;
  using V = tfb::C2<Real>;
  const tfb::CombArgs& c = ps.comb;
  constexpr int K = tfb::FOf<Real>::v / F;  // tiles per plan tile (the plan counts FOf-comb tiles)
  tfb::CombTmaArgs a{};
  a.ntiles = c.ntiles * K;
  a.chunks = c.chunks * K;
  a.groups_per_batch = c.groups_per_batch;
  a.rps = c.rps;
  a.sub_len = c.sub_len;
  a.es = c.es;
  a.bstride = c.bstride;
  a.out_w_last = c.out_w_last;
  a.final_pass = c.final_pass;
  a.fvalid = F;
  a.fb = c.fb;
  a.p = c.p;
  a.m_mask = c.m_mask;
  a.split_q = c.split_q;
  a.t_l2 = c.t_l2;
  a.t_l0l2 = c.t_l0l2;
  a.in_t = c.in_t;
  if (const char* e = std::getenv("TILEFFT_DEBUG_COPYONLY")) a.copy_only = std::atoi(e);
  for (int i = 0; i < 8; ++i) {
    a.out_w[i] = c.out_w[i];
    a.sub_w[i] = c.sub_w[i];
  }
  const V* t = (const V*)tb;
  const double2* t64 = (const double2*)tb64;
  // L >= 512: the tile over three half-tile slots (k_comb_h3) -- the first half of every tile requested a
  // tile earlier: 2^26 -1.1 %, 2^28 -2.5 %, 2^29 -1 %, 2^30 -0.3 % (tools/gpu/r02_h3.sh); TILEFFT_COMB_H3=0 = A/B
  if constexpr (IP && L >= 512 && F == tfb::FOf<Real>::v) {
    static const int h3 = env_int_or("TILEFFT_COMB_H3", 1);
    if (h3 && c.split_q == 0 && a.copy_only == 0) {
      using C3 = tfb::CombH3Cfg<Real, L, F>;
      auto k3 = tfb::k_comb_h3<Real, L, INV, F>;
      if (int rc = ensure_smem((const void*)k3, C3::SMEM)) return rc;
      int b3 = 0;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b3, k3, C3::THREADS, C3::SMEM));
      const long long g3 = std::max<long long>(1, std::min<long long>(a.ntiles, (long long)sm_count() * std::max(b3, 1)));
      k3<<<(unsigned)g3, C3::THREADS, C3::SMEM, st>>>(map, (V*)out, a, t + ps.tw_off, t64 + ps.wc_off,
                                                      t64 + ps.wf_off, scale);
      CUDA_TRY(cudaGetLastError());
      return 0;
    }
  }
  auto k = tfb::k_comb_tma<Real, L, INV, true, 0, F, IP>;
  if (int rc = ensure_smem((const void*)k, Cfg::SMEM)) return rc;
  int bps = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, Cfg::THREADS, Cfg::SMEM));
  const long long grid = std::max<long long>(1, std::min<long long>(a.ntiles, (long long)sm_count() * std::max(bps, 1)));
  k<<<(unsigned)grid, Cfg::THREADS, Cfg::SMEM, st>>>(map, (V*)out, a, t + ps.tw_off, t64 + ps.wc_off, t64 + ps.wf_off,
                                                     scale);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <typename Real, int L, bool INV>
int launch_comb(const Pass& ps, const void* in, void* out, const void* tb, const void* tb64, Real scale,
                cudaStream_t st) {
  using V = tfb::C2<Real>;
  const V* t = (const V*)tb;
  const double2* t64 = (const double2*)tb64;
  // small 1D transforms (data in L2, fewer 16-comb tiles than 2 per SM):
  // 4-comb tiles spread the pass over every SM
  if constexpr (std::is_same<Real, float>::value && L >= 64) {
    constexpr int FS = 4;
    if (ps.kind == K_COMB1D && ps.comb.ntiles < 2LL * sm_count() && ps.comb.rps % 16 == 0 && ps.comb.split_q == 0) {
      using CfgS = tfb::CombCfg<float, L, FS>;
      tfb::CombArgs a = ps.comb;
      a.chunks *= 16 / FS;
      a.ntiles *= 16 / FS;
      a.fvalid = FS;
      auto k = tfb::k_comb<float, L, INV, true, 0, FS>;
      if (int rc = ensure_smem((const void*)k, CfgS::SMEM)) return rc;
      k<<<(unsigned)a.ntiles, CfgS::THREADS, CfgS::SMEM, st>>>((const float2*)in, (float2*)out, a,
                                                              (const float2*)tb + ps.tw_off,
                                                              (const double2*)tb64 + ps.wc_off,
                                                              (const double2*)tb64 + ps.wf_off, (float)scale);
      CUDA_TRY(cudaGetLastError());
      return 0;
    }
  }
  if constexpr (tfb::Shape<L, tfb::RmaxOf<Real>::v>::NST > 1) {
    CUtensorMap map;
    // TMA pipelining pays off on the long 1D comb passes (2^30: 13.3 -> 11.8 ms);
    // the short 2D column passes (L <= 128) run faster as many tiny CTAs.
    // (8-comb tiles -- 64-byte rows, half the shared memory -- measured 15.8 vs
    // 11.9 ms at 2^30: the 128-byte line per comb step is what keeps the
    // strided TMA reads at full DRAM efficiency)
    if (!ps.no_tma && ps.kind == K_COMB1D && encode_comb_map<Real, L>(&map, ps, in)) {
      // exchange in place in the tile slot in one round (no separate half-tile buffer used in two rounds,
      // half the CTA barriers), next tile issued once the exchange is read back: 2^26 591 vs 670 us,
      // 2^24 152 vs 174 us, 2^30 10.60 vs 11.40 ms (tools/gpu/r02_ip.sh, r02_ip2.sh)
      if constexpr (tfb::Shape<L, tfb::RmaxOf<Real>::v>::NST > 1)
        return launch_comb_tma<Real, L, INV, tfb::FOf<Real>::v, true>(ps, map, out, tb, tb64, scale, st);
      return launch_comb_tma<Real, L, INV, tfb::FOf<Real>::v>(ps, map, out, tb, tb64, scale, st);
    }
  }
  if (ps.comb.split_q > 0) return fail(TILEFFT_EINVAL, "blocks input layout needs the TMA comb pass (16-byte aligned input)");
  using Cfg = tfb::CombCfg<Real, L>;
  auto go = [&](auto k) -> int {
    if (int rc = ensure_smem((const void*)k, Cfg::SMEM)) return rc;
    k<<<(unsigned)ps.grid, Cfg::THREADS, Cfg::SMEM, st>>>((const V*)in, (V*)out, ps.comb, t + ps.tw_off,
                                                          t64 + ps.wc_off, t64 + ps.wf_off, scale);
    CUDA_TRY(cudaGetLastError());
    return 0;
  };
  if (ps.kind == K_COMB1D) return go(tfb::k_comb<Real, L, INV, true, 0>);
  if (ps.twid) return go(tfb::k_comb<Real, L, INV, true, 1>);
  return go(tfb::k_comb<Real, L, INV, false, 1>);
}
template <typename Real, int L, bool INV>
int launch_final(const Pass& ps, const void* in, void* out, const void* tb, const void*, Real scale,
                 cudaStream_t st) {
  using V = tfb::C2<Real>;
  if constexpr (std::is_same<Real, float>::value && L >= 64) {
    constexpr int FS = 4;
    if (ps.fin.ntiles < 2LL * sm_count()) {
      using CfgS = tfb::FinalCfg<float, L, FS>;
      tfb::FinalArgs a = ps.fin;
      a.chunks *= 16 / FS;
      a.ntiles *= 16 / FS;
      auto k = tfb::k_final_t<float, L, INV, FS>;
      if (int rc = ensure_smem((const void*)k, CfgS::SMEM)) return rc;
      k<<<(unsigned)a.ntiles, CfgS::THREADS, CfgS::SMEM, st>>>((const float2*)in, (float2*)out, a,
                                                              (const float2*)tb + ps.tw_off, (float)scale);
      CUDA_TRY(cudaGetLastError());
      return 0;
    }
  }
  // persistent: the next tile's row loads are in flight while this tile's transposed stores drain
  // (measured vs one CTA per tile: 2^26 671 vs 685 us, 2^24 175 vs 181 us, 2^30 11.66 vs 12.06 ms;
  // tools/gpu/r02_finalp.sh)
  using Cfg = tfb::FinalCfg<Real, L>;
  constexpr int MINB = Cfg::THREADS <= 128 ? 4 : Cfg::THREADS <= 256 ? 2 : 1;
  auto k = tfb::k_final_p<Real, L, INV, tfb::FOf<Real>::v, MINB>;
  if (int rc = ensure_smem((const void*)k, Cfg::SMEM)) return rc;
  static int blocks_per_sm[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& bps = blocks_per_sm[dev & 15];
  if (!bps) {
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, Cfg::THREADS, Cfg::SMEM));
    if (bps < 1) bps = 1;
  }
  const long long grid = std::max<long long>(1, std::min<long long>(ps.fin.ntiles, (long long)sm_count() * bps));
  k<<<(unsigned)grid, Cfg::THREADS, Cfg::SMEM, st>>>((const V*)in, (V*)out, ps.fin, (const V*)tb + ps.tw_off, scale);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// Two-level pass (fp32): 128-byte-swizzled tensor maps over the strided axis {column, n1, n2, batch} and
// over the L2 scratch ring, control block reset, persistent launch of k_two_tma (one CTA per SM).
template <int LA, int LB, bool INV, int OUTT, bool TWID>
int launch_two_k(const Pass& ps, const void* in, void* out, const void* tb, const void* tb64, float scale,
                 cudaStream_t st) {
  using Cfg = tfb::TwoCfg<LA, LB, INV, OUTT>;
  auto enc = tensor_map_encoder();
  if (!enc) return fail(TILEFFT_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if ((uintptr_t)in % 16) return fail(TILEFFT_EINVAL, "two-level pass: input must be 16-byte aligned");
  const tfb::TwoArgs& a = ps.two;
  const long long B = a.groups / a.chunks;
  const cuuint64_t dims[4] = {(cuuint64_t)ps.two_cols, (cuuint64_t)LB, (cuuint64_t)LA, (cuuint64_t)B};
  const cuuint64_t strides[3] = {(cuuint64_t)(ps.two_es_in * 8), (cuuint64_t)(ps.two_es_in * 8 * LB),
                                 (cuuint64_t)(a.bs_in * 8)};
  const cuuint32_t box[4] = {16, 1, (cuuint32_t)Cfg::BL, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const float2* t = (const float2*)tb;
  const double2* t64 = (const double2*)tb64;
  CUtensorMap tin, tscr;
  if (enc(&tin, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<void*>(in), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(TILEFFT_ECUDA, "cuTensorMapEncodeTiled failed for the two-level pass");
  const cuuint64_t sdims[4] = {(cuuint64_t)LA, 16, (cuuint64_t)LB, (cuuint64_t)a.nslot};
  const cuuint64_t sstr[3] = {(cuuint64_t)LA * 8, (cuuint64_t)LA * 8 * 16, (cuuint64_t)LA * 8 * 16 * LB};
  const cuuint32_t sbox[4] = {16, 16, (cuuint32_t)LB, 1};
  if (enc(&tscr, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, a.scratch, sdims, sstr, sbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(TILEFFT_ECUDA, "cuTensorMapEncodeTiled failed for the two-level scratch");
  auto launch = [&](auto kfn, int threads, int smem) -> int {
    if (int rc = ensure_smem((const void*)kfn, smem)) return rc;
    CUDA_TRY(cudaMemsetAsync(a.ctrl, 0, sizeof(unsigned) * (2 + 2 * a.nslot), st));
    kfn<<<sm_count(), threads, smem, st>>>(tin, tscr, (float2*)out, a, t + ps.tw_off, t + ps.twl_off,
                                           t64 + ps.wc_off, t64 + ps.wf_off, scale);
    CUDA_TRY(cudaGetLastError());
    return 0;
  };
  using TC = tfb::TwoTmaCfg<LA, LB>;
  // plain column passes: the B items (a 16-point DFT, no inter-pass root) take the W_L roots off the
  // A items' critical path (8192^2: 523 vs 532 us; tools/gpu/r02_twlb.sh)
  // 19 compute warps at <= 96 registers (16 at 128 before): 8192^2 columns 503 vs 519 us; 23 warps
  // (80 registers, spills) 535 us (tools/gpu/r02_cw.sh)
  // (the round-1 team-split kernel k_two_ws -- A and B teams behind named barriers -- measured slower
  // and was removed in round 2: 8192^2 column pass 341 us in round 1, k_two_tma 297 us)
  if constexpr (!TWID && OUTT == 0) {
    using TCB = tfb::TwoTmaCfg<LA, LB, 19>;
    return launch(tfb::k_two_tma<LA, LB, INV, OUTT, TWID, true, TCB::CW>, TCB::THREADS, TCB::SMEM);
  }
  return launch(tfb::k_two_tma<LA, LB, INV, OUTT, TWID>, TC::THREADS, TC::SMEM);
}

template <int LA, int LB, bool INV>
int launch_two_l(const Pass& ps, const void* in, void* out, const void* tb, const void* tb64, float scale,
                 cudaStream_t st) {
  if (ps.outt) {
    return ps.twid ? launch_two_k<LA, LB, INV, 1, true>(ps, in, out, tb, tb64, scale, st)
                   : launch_two_k<LA, LB, INV, 1, false>(ps, in, out, tb, tb64, scale, st);
  }
  return ps.twid ? launch_two_k<LA, LB, INV, 0, true>(ps, in, out, tb, tb64, scale, st)
                 : launch_two_k<LA, LB, INV, 0, false>(ps, in, out, tb, tb64, scale, st);
}

template <typename Real, bool INV>
int launch_two(const Pass& ps, const void* in, void* out, const void* tb, const void* tb64, Real scale,
               cudaStream_t st) {
  if constexpr (std::is_same<Real, float>::value) {
    if (ps.la == 512) {
      switch (ps.lb) {
        case 4: return launch_two_l<512, 4, INV>(ps, in, out, tb, tb64, scale, st);
        case 8: return launch_two_l<512, 8, INV>(ps, in, out, tb, tb64, scale, st);
        case 16: return launch_two_l<512, 16, INV>(ps, in, out, tb, tb64, scale, st);
      }
    }
  }
  return fail(TILEFFT_EINVAL, "internal: no two-level kernel for %d x %d", ps.la, ps.lb);
}

template <typename Real, bool INV>
int launch_fast(const Pass& ps, const void* in, void* out, const void* tb, const void* tb64, Real scale,
                cudaStream_t st) {
#define DISPATCH(FN, ...)                                                     \
  switch (ps.L) {                                                             \
    case 2: return FN<Real, 2, INV>(ps, in, out, tb, tb64, scale, st);              \
    case 4: return FN<Real, 4, INV>(ps, in, out, tb, tb64, scale, st);              \
    case 8: return FN<Real, 8, INV>(ps, in, out, tb, tb64, scale, st);              \
    case 16: return FN<Real, 16, INV>(ps, in, out, tb, tb64, scale, st);            \
    case 32: return FN<Real, 32, INV>(ps, in, out, tb, tb64, scale, st);            \
    case 64: return FN<Real, 64, INV>(ps, in, out, tb, tb64, scale, st);            \
    case 128: return FN<Real, 128, INV>(ps, in, out, tb, tb64, scale, st);          \
    case 256: return FN<Real, 256, INV>(ps, in, out, tb, tb64, scale, st);          \
    case 512: return FN<Real, 512, INV>(ps, in, out, tb, tb64, scale, st);          \
    case 1024: return FN<Real, 1024, INV>(ps, in, out, tb, tb64, scale, st);        \
    __VA_ARGS__                                                               \
  }
  if (ps.kind == K_ROWS) {
    DISPATCH(launch_rows,
             case 2048: return launch_rows<Real, 2048, INV>(ps, in, out, tb, tb64, scale, st);
             case 4096: return launch_rows<Real, 4096, INV>(ps, in, out, tb, tb64, scale, st);
             case 8192: return launch_rows<Real, 8192, INV>(ps, in, out, tb, tb64, scale, st);)
  } else if (ps.kind == K_COMB1D || ps.kind == K_COMBAX) {
    DISPATCH(launch_comb)
  } else if (ps.kind == K_FINALT) {
    DISPATCH(launch_final)
  } else if (ps.kind == K_TWO) {
    return launch_two<Real, INV>(ps, in, out, tb, tb64, scale, st);
  }
#undef DISPATCH
  return fail(TILEFFT_EINVAL, "internal: no kernel for pass length %d", ps.L);
}

// Distributed pass 1: column FFTs of the rank's slab [N1][C], inter-pass root
// W_N^{r k}, results scattered into the destination slabs (peer memory over
// NVLink, or local staging for the NCCL exchange).
template <typename Real, int L, bool INV>
int launch_dist_pass1_L(const DistPass1& d, const void* in, const void* tb, const void* tb64, Real scale,
                        cudaStream_t st) {
  using V = tfb::C2<Real>;
  constexpr bool IP = tfb::Shape<L, tfb::RmaxOf<Real>::v>::NST > 1;  // in-place exchange, as launch_comb
  using Cfg = tfb::CombTmaCfg<Real, L, tfb::FOf<Real>::v, IP>;
  constexpr int W = (int)sizeof(V) / 8;
  auto enc = tensor_map_encoder();
  if (!enc) return fail(TILEFFT_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if ((uintptr_t)in % 16) return fail(TILEFFT_EINVAL, "distributed pass 1: input must be 16-byte aligned");
  CUtensorMap map;
  const long long vb = (long long)sizeof(V);
  const cuuint64_t dims[4] = {(cuuint64_t)(d.C * W), (cuuint64_t)L, 1, 1};
  const cuuint64_t strides[3] = {(cuuint64_t)(d.C * vb), (cuuint64_t)(L * d.C * vb), (cuuint64_t)(L * d.C * vb)};
  const cuuint32_t box[4] = {(cuuint32_t)(Cfg::F * W), (cuuint32_t)Cfg::BL, 1, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<void*>(in), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(TILEFFT_ECUDA, "cuTensorMapEncodeTiled failed for the distributed slab");
  auto k = tfb::k_comb_tma<Real, L, INV, true, 2, tfb::FOf<Real>::v, IP>;
  if (int rc = ensure_smem((const void*)k, Cfg::SMEM)) return rc;
  int bps = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, Cfg::THREADS, Cfg::SMEM));
  const long long grid = std::max<long long>(1, std::min<long long>(d.a.ntiles, (long long)sm_count() * std::max(bps, 1)));
  const V* t = (const V*)tb;
  const double2* t64 = (const double2*)tb64;
  k<<<(unsigned)grid, Cfg::THREADS, Cfg::SMEM, st>>>(map, nullptr, d.a, t + d.tw_off, t64 + d.wc_off, t64 + d.wf_off,
                                                     scale);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <typename Real, bool INV>
int launch_dist_pass1(const DistPass1& d, const void* in, const void* tb, const void* tb64, Real scale,
                      cudaStream_t st) {
  switch (d.L) {
    case 128: return launch_dist_pass1_L<Real, 128, INV>(d, in, tb, tb64, scale, st);
    case 256: return launch_dist_pass1_L<Real, 256, INV>(d, in, tb, tb64, scale, st);
    case 512: return launch_dist_pass1_L<Real, 512, INV>(d, in, tb, tb64, scale, st);
    case 1024: return launch_dist_pass1_L<Real, 1024, INV>(d, in, tb, tb64, scale, st);
  }
  return fail(TILEFFT_EINVAL, "distributed pass 1: unsupported column length %d", d.L);
}

template <typename Real>
int launch_exact(const Pass& ps, const void* in, void* out, const void* tb, Real scale, int conj_in, int conj_out,
                 cudaStream_t st) {
  using V = tfb::C2<Real>;
  tfb::ExactArgs a = ps.ex;
  a.conj_in = conj_in;
  a.conj_scale_out = conj_out;
  auto k = tfb::k_exact_pass<Real>;
  const size_t smem = (size_t)a.L * sizeof(V);
  if (int rc = ensure_smem((const void*)k, (int)smem)) return rc;
  int threads = (int)std::min<long long>(256, std::max<long long>(32, a.L / 2));
  k<<<(unsigned)ps.grid, threads, smem, st>>>((const V*)in, (V*)out, a, (const V*)tb, scale);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <typename Real>
int launch_levelwise(const Pass& ps, const void* in, void* out, const void* tb, Real scale, int conj_in, int conj_out,
                     cudaStream_t st) {
  using V = tfb::C2<Real>;
  const int threads = 256;
  if (ps.kind == K_BITREV) {
    const long long blocks = std::min<long long>((ps.lw_total + threads - 1) / threads, 148LL * 16);
    tfb::k_bitrev_permute<Real><<<(unsigned)blocks, threads, 0, st>>>((const V*)in, (V*)out, ps.lw_n,
                                                                     (int)(63 - __builtin_clzll(ps.lw_n)),
                                                                     ps.lw_total, conj_in);
  } else {
    const long long blocks = std::min<long long>((ps.lw_total + threads - 1) / threads, 148LL * 16);
    tfb::k_level<Real><<<(unsigned)blocks, threads, 0, st>>>((const V*)in, (V*)out, ps.lw_n, ps.level, ps.lw_total,
                                                            (const V*)tb, conj_out, scale);
  }
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <typename Real>
int launch_exchange(const void* in, void* out, const tfb::ExchangeArgs& a, cudaStream_t st) {
  using V = tfb::C2<Real>;
  const long long blocks = std::min<long long>((a.n + 255) / 256, 148LL * 16);
  tfb::k_exchange<Real><<<(unsigned)blocks, 256, 0, st>>>((const V*)in, (V*)out, a);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <typename Real>
int launch_interstage(const void* in, void* out, long long rows, long long cols, long long row0, long long rps,
                      long long sub_len, const void* tbl, long long tstride, cudaStream_t st) {
  using V = tfb::C2<Real>;
  const long long blocks = std::min<long long>((rows * cols + 255) / 256, 148LL * 16);
  tfb::k_interstage_scale<Real><<<(unsigned)blocks, 256, 0, st>>>((const V*)in, (V*)out, rows, cols, row0, rps,
                                                                 sub_len, (const V*)tbl, tstride);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace tfb_host
