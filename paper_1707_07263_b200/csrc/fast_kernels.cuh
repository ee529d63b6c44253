// Fast-mode pass kernels (fp32 / fp64), sm_100a.
//
// The reference's pass (tiled_fft.hpp:229-310: gather a decimated comb into a
// fast tile, run the row butterflies, scale by the inter-pass root and scatter
// through the pass's store map) is re-derived here as ONE kernel per pass:
//
//   * each length-L row FFT is a self-sorting Stockham network whose stages
//     are radix-32 DFTs held in one thread's registers (fft_common.cuh), so a
//     1024-point row needs exactly one shared-memory exchange and a 8192-point
//     row two — instead of the reference's 10/13 radix-2 levels in fast
//     storage (dit_levels, tiled_fft.hpp:89-117);
//   * the exchange buffer is padded one slot per 32 (the paper's 16x33 layout,
//     PAPER.md:200-202, at 8-byte words): every warp-wide access is
//     bank-conflict free;
//   * Stockham stage roots come from a per-plan table laid out [q][k] so a
//     warp's 32 lanes read 32 consecutive entries (read-only path, L1-resident);
//   * the inter-pass root W_M^{r k} (tiled_fft.hpp:284-294) is fused into the
//     store and served from a two-level table (coarse x fine, each ~sqrt(M)
//     entries) instead of the reference's M-entry table;
//   * strided passes process 16 adjacent combs per CTA so every global access
//     is a full 128-byte line (measured: 8-byte-wide comb access runs at 15%
//     of copy bandwidth, 128-byte at 88%; profiles/r01_membench.txt).
#pragma once
#include "fft_common.cuh"
#include "tma_util.cuh"
#include <cuda.h>

namespace tfb {

// ------------------------------------------------------------------ shapes
// L = T * R: T threads per FFT, R elements per thread; stages radix RMAX
// except a smaller last one.
template <int L, int RMAX>
struct Shape {
  static constexpr int LOG = ilog2c(L);
  static constexpr int LR = ilog2c(RMAX);
  static constexpr int R = L < RMAX ? L : RMAX;
  static constexpr int T = L / R;
  static constexpr int NFULL = LOG / LR;
  static constexpr int LAST = LOG % LR;
  static constexpr int NST = (L <= RMAX) ? 1 : NFULL + (LAST ? 1 : 0);
  __host__ __device__ static constexpr int radix(int s) {
    return (L <= RMAX) ? L : (s < NFULL ? RMAX : (1 << LAST));
  }
  __host__ __device__ static constexpr int ns(int s) {
    int n = 1;
    for (int i = 0; i < s; ++i) n *= radix(i);
    return n;
  }
  // offset of stage s's [q][k] root table inside this L's table block
  __host__ __device__ static constexpr int tw_off(int s) {
    int o = 0;
    for (int i = 1; i < s; ++i) o += radix(i) * ns(i);
    return o;
  }
  static constexpr int TW_TOTAL = tw_off(NST);
};

// Registers per thread: 32 complex for fp32, 16 for fp64.
template <typename Real> struct RmaxOf { static constexpr int v = 32; };
template <> struct RmaxOf<double> { static constexpr int v = 16; };

// Host-side description of a stage-root table block (for table building).
struct StageTableInfo {
  int nst;
  int radix[8];
  int ns[8];
  int total;
};
template <int L, int RMAX>
inline StageTableInfo stage_table_info() {
  using Sh = Shape<L, RMAX>;
  StageTableInfo s{};
  s.nst = Sh::NST;
  for (int i = 0; i < Sh::NST; ++i) {
    s.radix[i] = Sh::radix(i);
    s.ns[i] = Sh::ns(i);
  }
  s.total = Sh::TW_TOTAL;
  return s;
}

__device__ __forceinline__ int pad32(int i) { return i + (i >> 5); }

// ------------------------------------------------------------------ Stockham
// v[i*RS + q]: input q of butterfly b = t + T*i of the current stage.
// After the last stage v[i*RS + q] = X[b + q * (L / RS_last)].
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// TWS: the stage-root table `tw` lives in shared memory (plain loads -> LDS)
// instead of global memory read through the read-only path (LDG.CONSTANT).
template <typename V, int L, int RMAX, bool INV, int S, int NR = 1, bool TWS = false>
struct Stages {
  using Sh = Shape<L, RMAX>;
  static constexpr int RS = Sh::radix(S), NS = Sh::ns(S), NB = Sh::R / RS;
  // NR > 1: the exchange buffer holds 1/NR of the CTA's FFTs; the exchange
  // runs in NR rounds and a thread takes part in round `my_round` only.
  // `last` runs at the start of the last stage, once the exchange buffer is
  // free (multi-stage networks only): e.g. to start streaming the next input.
  template <class Ex, class Sync, class Hook = NoHook>
  __device__ __forceinline__ static void run(V* v, int t, Ex& ex, const V* __restrict__ tw, Sync& sync,
                                             int my_round = 0, Hook last = Hook{}) {
    if constexpr (S > 0 && S + 1 == Sh::NST) last();
    if constexpr (S > 0) {
      const V* tws = tw + Sh::tw_off(S);
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const int k = (t + Sh::T * i) & (NS - 1);
#pragma unroll
        for (int q = 1; q < RS; ++q) {
          V w;
          if constexpr (TWS) w = tws[q * NS + k];
          else w = __ldg(tws + q * NS + k);
          v[i * RS + q] = ctw<INV>(v[i * RS + q], w);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) reg_dft<RS, INV>(v + i * RS);
    if constexpr (S + 1 < Sh::NST) {
      constexpr int RS2 = Sh::radix(S + 1), NB2 = Sh::R / RS2, STR2 = L / RS2;
#pragma unroll 1
      for (int round = 0; round < NR; ++round) {
        if (round == my_round) {
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            const int b = t + Sh::T * i;
            const int base = (b / NS) * (NS * RS) + (b & (NS - 1));
#pragma unroll
            for (int q = 0; q < RS; ++q) ex(base + q * NS) = v[i * RS + q];
          }
        }
        sync();
        if (round == my_round) {
#pragma unroll
          for (int i = 0; i < NB2; ++i) {
            const int b = t + Sh::T * i;
#pragma unroll
            for (int q = 0; q < RS2; ++q) v[i * RS2 + q] = ex(b + q * STR2);
          }
        }
        sync();
      }
      Stages<V, L, RMAX, INV, S + 1, NR, TWS>::run(v, t, ex, tw, sync, my_round, last);
    }
  }
};

// output index of register slot j after the last stage
template <int L, int RMAX>
__device__ __forceinline__ int out_index(int t, int j) {
  using Sh = Shape<L, RMAX>;
  constexpr int RSL = Sh::radix(Sh::NST - 1);
  const int i = j / RSL, q = j % RSL;
  return t + Sh::T * i + q * (L / RSL);
}

struct SyncWarp { __device__ __forceinline__ void operator()() const { __syncwarp(); } };
struct SyncBlock { __device__ __forceinline__ void operator()() const { __syncthreads(); } };

// Inter-pass root W_M^e, e < M, from fp64 coarse/fine tables (~sqrt(M)
// entries each): W = C[e >> fb] * F[e & (2^fb - 1)], product in fp64.
__device__ __forceinline__ double2 interpass_root64(const double2* __restrict__ wc, const double2* __restrict__ wf,
                                                    uint32_t e, int fb) {
  const double2 c = __ldg(wc + (e >> fb));
  const double2 f = __ldg(wf + (e & ((1u << fb) - 1u)));
  return cmul(c, f);
}
__device__ __forceinline__ float2 to_v(double2 w, float2*) { return make_float2((float)w.x, (float)w.y); }
__device__ __forceinline__ double2 to_v(double2 w, double2*) { return w; }

// Fused inter-pass scale of the last Stockham stage's outputs
// (tiled_fft.hpp:284-294): register slot i*RS + q holds spectrum index
// k = b_i + q*(L/RS), b_i = t + T*i, so
//   W_M^{r k} = W_M^{r b_i} * s^q,   s = W_M^{r L/RS}.
// Per thread: a handful of fp64 table lookups (two-level, ~sqrt(M) entries)
// build, in fp64, B_i[qb] = W^{r b_i} s^qb (qb < 4) and A[qa] = s^{4 qa}
// (qa < RS/4), each rounded once to Real; each element then needs one
// complex multiply A*B (independent across q: no dependent chain) and the
// apply — instead of two scattered table gathers per element.
template <typename V, int L, int RMAX, bool INV>
__device__ __forceinline__ void interpass_scale(V* v, int t, uint32_t r, uint32_t m_mask, int fb,
                                                const double2* __restrict__ wc, const double2* __restrict__ wf) {
  using Sh = Shape<L, RMAX>;
  constexpr int RSL = Sh::radix(Sh::NST - 1), NB = Sh::R / RSL, STR = L / RSL;
  constexpr int QB = RSL < 4 ? RSL : 4, QA = RSL / QB;
  const double2 s1 = interpass_root64(wc, wf, (r * (uint32_t)STR) & m_mask, fb);
  const double2 s2 = cmul(s1, s1);
  double2 s4 = cmul(s2, s2);
  V A[QA];
  {
    double2 a = make_double2(1.0, 0.0);
#pragma unroll
    for (int qa = 0; qa < QA; ++qa) {
      A[qa] = to_v(a, (V*)nullptr);
      if (qa + 1 < QA) a = cmul(a, s4);
    }
  }
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const double2 base = interpass_root64(wc, wf, (r * (uint32_t)(t + Sh::T * i)) & m_mask, fb);
    V B[QB];
    B[0] = to_v(base, (V*)nullptr);
    if constexpr (QB > 1) B[1] = to_v(cmul(base, s1), (V*)nullptr);
    if constexpr (QB > 2) {
      const double2 b2 = cmul(base, s2);
      B[2] = to_v(b2, (V*)nullptr);
      B[3] = to_v(cmul(b2, s1), (V*)nullptr);
    }
#pragma unroll
    for (int q = 0; q < RSL; ++q) {
      const V w = (q / QB) == 0 ? B[q % QB] : cmul(A[q / QB], B[q % QB]);
      v[i * RSL + q] = ctw<INV>(v[i * RSL + q], w);
    }
  }
}

// ------------------------------------------------------------------ K_ROWS
// FPC contiguous length-L rows per CTA, natural order in and out (the p = 1
// pass of fft_tiled: col_sources bit reversal + dit_levels + identity
// interleave, tiled_fft.hpp:346-406). In-place safe.
template <typename Real, int L, int FPC>
struct RowsCfg {
  using V = C2<Real>;
  static constexpr int RMAX = RmaxOf<Real>::v;
  using Sh = Shape<L, RMAX>;
  static constexpr int THREADS = FPC * Sh::T;
  static constexpr int REG = L + L / 32 + 1;  // per-FFT exchange region (elements)
  static constexpr int SMEM = (Sh::NST > 1 ? FPC * REG : 1) * (int)sizeof(V);
};

template <typename Real, int L, int FPC, bool INV>
__global__ void __launch_bounds__(RowsCfg<Real, L, FPC>::THREADS)
k_rows(const C2<Real>* in, C2<Real>* out, long long nrows, const C2<Real>* __restrict__ tw, Real scale) {
  using Cfg = RowsCfg<Real, L, FPC>;
  using V = C2<Real>;
  using Sh = typename Cfg::Sh;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V* sm = reinterpret_cast<V*>(smem_raw);
  const int ff = threadIdx.x / Sh::T, t = threadIdx.x % Sh::T;
  long long row = (long long)blockIdx.x * FPC + ff;
  const bool active = row < nrows;
  if (!active) row = nrows - 1;
  const V* src = in + row * L;
  V v[Sh::R];
#pragma unroll
  for (int q = 0; q < Sh::R; ++q) v[q] = src[t + q * Sh::T];
  V* reg = sm + ff * Cfg::REG;
  auto ex = [reg](int i) -> V& { return reg[pad32(i)]; };
  if constexpr (Sh::T <= 32) {
    SyncWarp s;
    Stages<V, L, Cfg::RMAX, INV, 0>::run(v, t, ex, tw, s);
  } else {
    SyncBlock s;
    Stages<V, L, Cfg::RMAX, INV, 0>::run(v, t, ex, tw, s);
  }
  if (active) {
    V* dst = out + row * L;
#pragma unroll
    for (int j = 0; j < Sh::R; ++j) {
      V r = v[j];
      if (scale != (Real)1) r = mk(r.x * scale, r.y * scale);
      dst[out_index<L, Cfg::RMAX>(t, j)] = r;
    }
  }
}

// ------------------------------------------------------------------ K_ROWS_TMA
// Persistent, TMA-staged variant of K_ROWS for rows that fit one warp
// (T <= 32: L <= 1024 fp32, L <= 512 fp64). Each warp owns an S-deep ring of
// shared-memory slots; lane 0 streams the warp's next chunks of rows into the
// ring with 1D bulk copies (cp.async.bulk + mbarrier complete_tx) while the
// warp computes the current chunk, so every SM keeps ~S-1 chunks of loads in
// flight with no registers tied up. The slot doubles as the padded exchange
// buffer of the Stockham stages; results leave straight from registers.
template <int L, int T>
struct RegionPad {
  // per-FFT region >= L + L/32, == T (mod 16) so the FFTs that share a
  // half-warp land on disjoint banks; even => 16-byte aligned regions
  static constexpr int base = L + L / 32;
  static constexpr int tm = T % 16;
  static constexpr int v = base + ((tm - base % 16) + 16) % 16;
};

template <typename Real, int L, int WARPS, int S>
struct RowsTmaCfg {
  using V = C2<Real>;
  static constexpr int RMAX = RmaxOf<Real>::v;
  using Sh = Shape<L, RMAX>;
  static_assert(Sh::T <= 32, "one warp per chunk");
  static constexpr int FPW = 32 / Sh::T;                        // FFTs per warp chunk
  static constexpr bool EXCH = Sh::NST > 1;
  static constexpr int REG = EXCH ? RegionPad<L, Sh::T>::v : L;  // elements per FFT region
  static constexpr int SLOT = FPW * REG;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int DATA_BYTES = WARPS * S * SLOT * (int)sizeof(V);
  static constexpr int SMEM = DATA_BYTES + WARPS * S * 8;
  static constexpr int TW_BYTES = Sh::TW_TOTAL * (int)sizeof(V);  // stage roots staged in smem (TWS variant)
};

template <typename Real, int L, int WARPS, int S, bool INV, bool TWS = false>
__global__ void __launch_bounds__(WARPS * 32)
k_rows_tma(const C2<Real>* in, C2<Real>* out, long long nrows, const C2<Real>* __restrict__ tw_g, Real scale) {
  using Cfg = RowsTmaCfg<Real, L, WARPS, S>;
  using V = C2<Real>;
  using Sh = typename Cfg::Sh;
  constexpr int FPW = Cfg::FPW;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const V* tw = tw_g;
  if constexpr (TWS) {
    // stage the plan's stage-root table once per CTA (persistent kernel)
    V* tws = reinterpret_cast<V*>(smem_raw + Cfg::SMEM);
    for (int i = threadIdx.x; i < Sh::TW_TOTAL; i += blockDim.x) tws[i] = tw_g[i];
    __syncthreads();
    tw = tws;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ff = lane / Sh::T, tt = lane % Sh::T;
  V* slots = reinterpret_cast<V*>(smem_raw) + (size_t)w * S * Cfg::SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + Cfg::DATA_BYTES) + w * S;
  const long long nchunks = (nrows + FPW - 1) / FPW;
  const long long G = (long long)gridDim.x * WARPS;
  long long c = (long long)blockIdx.x * WARPS + w;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  __syncwarp();
  auto issue = [&](long long chunk, int s) {
    V* dst = slots + s * Cfg::SLOT;
    const long long r0 = chunk * FPW;
    const int nr = (int)((nrows - r0) < FPW ? (nrows - r0) : FPW);
    mbar_arrive_expect_tx(&bars[s], (uint32_t)(nr * L * (int)sizeof(V)));
    if constexpr (Cfg::EXCH) {
      for (int f = 0; f < nr; ++f) tma_load_1d(dst + f * Cfg::REG, in + (r0 + f) * L, L * (int)sizeof(V), &bars[s]);
    } else {
      tma_load_1d(dst, in + r0 * L, (uint32_t)(nr * L * (int)sizeof(V)), &bars[s]);
    }
  };
  if (lane == 0) {
#pragma unroll 1
    for (int s = 0; s < S - 1; ++s)
      if (c + s * G < nchunks) issue(c + s * G, s);
  }
  int k = 0;
#pragma unroll 1
  for (; c < nchunks; c += G, ++k) {
    const int s = k % S;
    if (lane == 0) {
      const long long cn = c + (long long)(S - 1) * G;
      if (cn < nchunks) issue(cn, (k + S - 1) % S);
    }
    mbar_wait(&bars[s], (uint32_t)((k / S) & 1));
    V* reg = slots + s * Cfg::SLOT + ff * Cfg::REG;
    V v[Sh::R];
#pragma unroll
    for (int q = 0; q < Sh::R; ++q) v[q] = reg[tt + q * Sh::T];
    if constexpr (Cfg::EXCH) {
      __syncwarp();
      auto ex = [reg](int i) -> V& { return reg[pad32(i)]; };
      SyncWarp sy;
      Stages<V, L, Cfg::RMAX, INV, 0, 1, TWS>::run(v, tt, ex, tw, sy);
    } else {
      auto ex = [reg](int i) -> V& { return reg[i]; };
      SyncWarp sy;
      Stages<V, L, Cfg::RMAX, INV, 0, 1, TWS>::run(v, tt, ex, tw, sy);
    }
    const long long row = c * FPW + ff;
    if (row < nrows) {
      V* dst = out + row * L;
#pragma unroll
      for (int j = 0; j < Sh::R; ++j) {
        V r = v[j];
        if (scale != (Real)1) r = mk(r.x * scale, r.y * scale);
        dst[out_index<L, Cfg::RMAX>(tt, j)] = r;
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
  }
}

// ------------------------------------------------------------------ K_COMB
// 16 adjacent combs per CTA (lanes along the comb index f, so every
// global access is 16 contiguous elements = one 128-byte line for fp32).
//
// Element n of comb (g, f):   in [ in_base(g) + f + n * s_in ]
// Spectrum k of comb (g, f):  out[out_base(g) + f + k * s_out] (* W_M^{r k})
//
// mode 0 (1D inner pass, tiled_fft.hpp:252-294): tile -> (batch, sub, chunk);
//   base = batch*bstride + sub*sub_len + chunk*16, s = rows_per_sub,
//   r = chunk*16 + f, in place.
// mode 1 (strided transform along an axis with element stride `es`, e.g. the
//   2D column pass): tile -> (batch, grow, chunk); the 1D pass geometry acts
//   on the logical index, chunk*16+f selects the column; inner passes are in
//   place with root r = grow % rows_per_sub, the final pass stores through
//   the digit interleave (stage_plan.hpp:144-155).
struct CombArgs {
  long long bstride;      // elements between batch items
  long long ntiles;       // total tiles
  long long chunks;       // f-chunks per group
  long long groups_per_batch;
  long long sub_len, rps; // pass geometry (logical units)
  long long es;           // element stride of the logical index (mode 1)
  long long out_w_last;   // final pass: out_weights[p-1]
  int final_pass;         // mode 1 only
  int fvalid;             // valid lanes per chunk (<= 16)
  int fb;                 // fine-table bits for W_M
  uint32_t m_mask;        // M - 1 (M = sub_len)
  int p;                  // passes of the logical plan (digit interleave)
  long long out_w[8], sub_w[8];
  // blocks input layout (first pass only; 0 = off): the batch item's comb rows n1 are split over source
  // blocks of split_q rows each, split_stride elements apart -- the [src][k1][c] layout an all-to-all
  // leaves (element n1*rps + col of item k1 at (n1 / q) * split_stride + k1 * split_bstride + (n1 % q) * rps
  // + col); the output keeps the plan's layout
  long long split_q, split_stride, split_bstride;
  // transposed hand-over between the first two passes of a 3-pass plan [L0][L1][L2] whose first comb
  // stride is megabytes (pass-0 rows 8 MB apart at 2^30): pass 0 stores spectrum k0 of column
  // c = c1*L2 + c2 at T[c1][k0][c2] (t_l2 = L2, t_l0l2 = L0*L2: its store rows L2 elements apart instead of
  // L1*L2), pass 1 (in_t = 1) reads its comb over c1 for fixed k0 from that layout and stores the natural
  // [k0][k1][c2] layout (rows L2 apart) out of place. A strided TMA copy that WRITES rows 8 MB apart runs at
  // 4.5 TB/s, one that only READS them at 6.1 TB/s (profiles/r02_comb_layout.txt).
  long long t_l2, t_l0l2;
  int in_t;
};

__device__ __forceinline__ long long final_index_dev(const CombArgs& a, long long sub) {
  long long out = 0, rem = sub;
  for (int i = 0; i + 1 < a.p; ++i) {
    const long long d = rem / a.sub_w[i];
    rem -= d * a.sub_w[i];
    out += d * a.out_w[i];
  }
  return out;
}

// Combs per CTA: one 128-byte line per comb step (16 fp32 / 8 fp64 elements).
template <typename Real> struct FOf { static constexpr int v = 128 / (int)sizeof(C2<Real>); };

// F < 16 (small transforms whose data sits in L2: more, smaller tiles so
// every SM gets work) pads the exchange by one element per 32 / F rows.
template <typename Real, int L, int F_ = FOf<Real>::v>
struct CombCfg {
  using V = C2<Real>;
  static constexpr int RMAX = RmaxOf<Real>::v;
  using Sh = Shape<L, RMAX>;
  static constexpr int F = F_;
  static constexpr bool PAD = F < FOf<Real>::v;
  static constexpr int THREADS = F * Sh::T;
  static constexpr int SMEM = (Sh::NST > 1 ? L * F + (PAD ? L * F / 32 : 0) : 1) * (int)sizeof(V);
  // two resident CTAs per SM (<= 128 registers at 256 threads) so one CTA's
  // loads overlap the other's butterflies
  static constexpr int MINB = THREADS <= 256 ? 2 : 1;
};

// One comb tile (the body of K_COMB; also run by the fused small-transform kernel).
template <typename Real, int L, bool INV, bool TWID, int MODE, int F_>
__device__ __forceinline__ void comb_tile(const C2<Real>* in, C2<Real>* out, const CombArgs& a,
                                          const C2<Real>* __restrict__ tw, const double2* __restrict__ wc,
                                          const double2* __restrict__ wf, Real scale, long long tile,
                                          C2<Real>* sm) {
  using Cfg = CombCfg<Real, L, F_>;
  using V = C2<Real>;
  using Sh = typename Cfg::Sh;
  constexpr int F = Cfg::F;
  const int f = threadIdx.x % F, t = threadIdx.x / F;
  const long long chunk = tile % a.chunks;
  const long long g = tile / a.chunks;
  const long long batch = g / a.groups_per_batch;
  const long long u = g % a.groups_per_batch;  // mode 0: sub; mode 1: grow
  long long in_base, out_base, s_in, s_out;
  uint32_t r;
  if constexpr (MODE == 0) {
    in_base = batch * a.bstride + u * a.sub_len + chunk * F;
    out_base = in_base;
    s_in = s_out = a.rps;
    if (a.in_t) {  // T[c1][k0][c2] input (see CombArgs::t_l2)
      in_base = batch * a.bstride + u * a.rps + chunk * F;
      s_in = a.groups_per_batch * a.rps;
    }
    if (a.t_l2) {
      const long long c0 = chunk * F;
      out_base = batch * a.bstride + (c0 / a.t_l2) * a.t_l0l2 + c0 % a.t_l2;
      s_out = a.t_l2;
    }
    r = (uint32_t)(chunk * F + f);
  } else {
    const long long sub = u / a.rps, rr = u % a.rps;
    in_base = batch * a.bstride + (sub * a.sub_len + rr) * a.es + chunk * F;
    s_in = a.rps * a.es;
    r = (uint32_t)rr;
    if (a.final_pass) {
      out_base = batch * a.bstride + final_index_dev(a, u) * a.es + chunk * F;
      s_out = a.out_w_last * a.es;
    } else {
      out_base = in_base;
      s_out = s_in;
    }
  }
  const bool active = f < a.fvalid;
  const int fl = active ? f : 0;
  V v[Sh::R];
#pragma unroll
  for (int q = 0; q < Sh::R; ++q) v[q] = in[in_base + fl + (long long)(t + q * Sh::T) * s_in];
  auto ex = [sm, f](int i) -> V& {
    if constexpr (Cfg::PAD) return sm[i * F + f + ((i * F) >> 5)];
    else return sm[i * F + f];
  };
  SyncBlock s;
  Stages<V, L, Cfg::RMAX, INV, 0>::run(v, t, ex, tw, s);
  if constexpr (TWID) interpass_scale<V, L, Cfg::RMAX, INV>(v, t, r, a.m_mask, a.fb, wc, wf);
  if (active) {
#pragma unroll
    for (int j = 0; j < Sh::R; ++j) {
      const int k = out_index<L, Cfg::RMAX>(t, j);
      V x = v[j];
      if (scale != (Real)1) x = mk(x.x * scale, x.y * scale);
      out[out_base + f + (long long)k * s_out] = x;
    }
  }
}

template <typename Real, int L, bool INV, bool TWID, int MODE, int F_ = FOf<Real>::v>
__global__ void __launch_bounds__(CombCfg<Real, L, F_>::THREADS, CombCfg<Real, L, F_>::MINB)
k_comb(const C2<Real>* in, C2<Real>* out, CombArgs a, const C2<Real>* __restrict__ tw,
       const double2* __restrict__ wc, const double2* __restrict__ wf, Real scale) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  comb_tile<Real, L, INV, TWID, MODE, F_>(in, out, a, tw, wc, wf, scale, blockIdx.x,
                                          reinterpret_cast<C2<Real>*>(smem_raw));
}

// ------------------------------------------------------------------ K_COMB_TMA
// Persistent, TMA-pipelined K_COMB. Tiles are [L][F] boxes of 16 adjacent
// combs (fp32; 8 for fp64): one 128-byte line per comb step. A 3-D/4-D
// tensor map describes the strided comb layout, so one thread streams whole
// tiles into an S-deep ring of shared-memory slots (cp.async.bulk.tensor +
// mbarrier complete_tx) while the CTA works on the current tile; the slot is
// released as soon as its inputs are in registers, so the next tile's load
// overlaps the butterflies, the exchange (a separate buffer, in NR rounds
// when the tile is larger than it) and the stores.
template <typename Real, int L, int F_ = FOf<Real>::v, bool IP_ = false>
struct CombTmaCfg {
  using V = C2<Real>;
  static constexpr int RMAX = RmaxOf<Real>::v;
  using Sh = Shape<L, RMAX>;
  static constexpr int F = F_;
  static constexpr int THREADS = F * Sh::T;
  static constexpr int TILE = L * F;                       // elements
  static constexpr int TILE_BYTES = TILE * (int)sizeof(V);
  // One slot per CTA. Default (IP, the product): the Stockham exchange runs
  // in place in the slot in one round and the next tile is issued once the
  // exchange has been read back. Otherwise: the slot is released as soon as
  // the tile is in registers and a half-tile exchange buffer is used in two
  // rounds (1.5 tiles of shared memory) -- measured 7-12 % slower.
  // IP: the exchange runs in place in the tile slot (one round, no separate buffer) and the next
  // tile's TMA is issued once the exchange has been read back (start of the last stage)
  static constexpr bool IP = IP_;
  static constexpr int S = 1;
  static constexpr int NR = (Sh::NST > 1 && !IP) ? 2 : 1;
  static constexpr int FX = F / NR;                        // FFTs per exchange round
  static constexpr int XB = (Sh::NST > 1 && !IP) ? L * FX : 0;  // exchange elements
  static constexpr int BL = L < 256 ? L : 256;             // TMA box rows
  static constexpr int DATA_BYTES = S * TILE_BYTES + XB * (int)sizeof(V);
  static constexpr int SMEM = DATA_BYTES + S * 8 + 128;    // + mbarriers + alignment slack
  static constexpr int WARPS = THREADS / 32 > 0 ? THREADS / 32 : 1;
  static constexpr int MINB_W = 16 / WARPS > 0 ? 16 / WARPS : 1;
  static constexpr int MINB_S = (227 * 1024) / (SMEM + 1024) > 0 ? (227 * 1024) / (SMEM + 1024) : 1;
  static constexpr int MINB = MINB_W < MINB_S ? MINB_W : MINB_S;
};

struct CombTmaArgs {
  long long ntiles, chunks, groups_per_batch;
  long long rps, sub_len;   // pass geometry (logical units)
  long long es;             // element stride (mode 1)
  long long bstride;        // elements between batch items
  long long out_w_last;     // final pass of mode 1
  int final_pass, fvalid, fb, p;
  uint32_t m_mask;
  long long out_w[8], sub_w[8];
  // mode 2 (distributed four-step, pass 1): the CTA's combs are the global
  // columns r_off + chunk*F + f; spectrum k goes to rank k / rows_per_rank,
  // row k % rows_per_rank of that rank's slab (row pitch `pitch`, column
  // offset `col_off`) — the all-to-all transpose fused into the store.
  long long r_off, pitch, col_off;
  int rows_per_rank, nranks;
  int copy_only;            // diagnostics: 1 = skip the butterflies, 2 = skip the inter-pass roots
  long long t_l2, t_l0l2;   // transposed pass-0 store / pass-1 load (CombArgs::t_l2)
  int in_t;
  long long split_q;        // blocks input layout (CombArgs::split_q): 5-D tensor map, rows n1 -> (n1 % q, n1 / q)
  void* peers[16];
};

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

template <typename Real, int L, bool INV, bool TWID, int MODE, int F_ = FOf<Real>::v, bool IP = false>
__global__ void __launch_bounds__(CombTmaCfg<Real, L, F_, IP>::THREADS, CombTmaCfg<Real, L, F_, IP>::MINB)
k_comb_tma(const __grid_constant__ CUtensorMap tmap, C2<Real>* out, CombTmaArgs a, const C2<Real>* __restrict__ tw,
           const double2* __restrict__ wc, const double2* __restrict__ wf, Real scale) {
  using Cfg = CombTmaCfg<Real, L, F_, IP>;
  using V = C2<Real>;
  using Sh = typename Cfg::Sh;
  constexpr int F = Cfg::F, S = Cfg::S;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V* slots = reinterpret_cast<V*>(smem_raw);
  V* xb = IP ? slots : slots + S * Cfg::TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + Cfg::DATA_BYTES);
  const int f = threadIdx.x % F, t = threadIdx.x / F;
  const int my_round = f / Cfg::FX, fx = f % Cfg::FX;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  // tile -> TMA coordinates {col, n0, rr, group}
  auto coords = [&](long long tile, int& c0, int& c2, int& c3) {
    const long long chunk = tile % a.chunks, g = tile / a.chunks;
    const long long batch = g / a.groups_per_batch, u = g % a.groups_per_batch;
    c0 = (int)(chunk * F * (sizeof(V) / 8));
    if constexpr (MODE == 0 || MODE == 2) {
      c2 = 0;
      c3 = (int)(batch * a.groups_per_batch + u);
      if (MODE == 0 && a.in_t) {  // map {c2, c1, k0, batch} over T[c1][k0][c2]
        c2 = (int)u;
        c3 = (int)batch;
      }
    } else {
      c2 = (int)(u % a.rps);
      c3 = (int)(batch * (a.groups_per_batch / a.rps) + u / a.rps);
    }
  };
  auto issue = [&](long long tile, int s) {
    int c0, c2, c3;
    coords(tile, c0, c2, c3);
    mbar_arrive_expect_tx(&full[s], Cfg::TILE_BYTES);
    if (MODE == 0 && a.split_q > 0) {
      const int q = (int)a.split_q;
#pragma unroll 1
      for (int n0 = 0; n0 < L; n0 += Cfg::BL)
        tma_load_5d(slots + s * Cfg::TILE + n0 * F, &tmap, c0, n0 % q, n0 / q, c3, 0, &full[s]);
    } else {
#pragma unroll 1
      for (int n0 = 0; n0 < L; n0 += Cfg::BL) tma_load_4d(slots + s * Cfg::TILE + n0 * F, &tmap, c0, n0, c2, c3, &full[s]);
    }
  };
  const long long G = gridDim.x;
  long long tile = blockIdx.x;
  if (threadIdx.x == 0) {
#pragma unroll 1
    for (int s = 0; s < S; ++s)
      if (tile + s * G < a.ntiles) issue(tile + s * G, s);
  }
  int k = 0;
#pragma unroll 1
  for (; tile < a.ntiles; tile += G, ++k) {
    const int s = k % S;
    mbar_wait(&full[s], (uint32_t)((k / S) & 1));
    const V* sl = slots + s * Cfg::TILE;
    V v[Sh::R];
#pragma unroll
    for (int q = 0; q < Sh::R; ++q) v[q] = sl[(t + q * Sh::T) * F + f];
    auto refill = [&]() {
      fence_proxy_async_smem();
      __syncthreads();  // slot s fully consumed: refill it
      if (threadIdx.x == 0 && tile + S * G < a.ntiles) issue(tile + S * G, s);
    };
    if constexpr (!IP) refill();
    else __syncthreads();  // every thread has its elements before the in-place exchange overwrites them
    // geometry of this tile (same decomposition as K_COMB)
    const long long chunk = tile % a.chunks, g = tile / a.chunks;
    const long long batch = g / a.groups_per_batch, u = g % a.groups_per_batch;
    long long out_base, s_out;
    uint32_t r;
    if constexpr (MODE == 0) {
      out_base = batch * a.bstride + u * a.sub_len + chunk * F;
      s_out = a.rps;
      if (a.t_l2) {
        const long long c0 = chunk * F;
        out_base = batch * a.bstride + (c0 / a.t_l2) * a.t_l0l2 + c0 % a.t_l2;
        s_out = a.t_l2;
      }
      r = (uint32_t)(chunk * F + f);
    } else if constexpr (MODE == 2) {
      out_base = a.col_off + chunk * F;
      s_out = a.pitch;
      r = (uint32_t)(a.r_off + chunk * F + f);
    } else {
      const long long sub = u / a.rps, rr = u % a.rps;
      r = (uint32_t)rr;
      if (a.final_pass) {
        long long oi = 0, rem = u;
        for (int i = 0; i + 1 < a.p; ++i) {
          const long long d = rem / a.sub_w[i];
          rem -= d * a.sub_w[i];
          oi += d * a.out_w[i];
        }
        out_base = batch * a.bstride + oi * a.es + chunk * F;
        s_out = a.out_w_last * a.es;
      } else {
        out_base = batch * a.bstride + (sub * a.sub_len + rr) * a.es + chunk * F;
        s_out = a.rps * a.es;
      }
    }
    auto ex = [xb, fx](int i) -> V& { return xb[i * Cfg::FX + fx]; };
    SyncBlock sy;
    if constexpr (IP)
      if (a.copy_only == 1) refill();
    if (a.copy_only != 1) {
      if constexpr (IP) Stages<V, L, Cfg::RMAX, INV, 0, Cfg::NR>::run(v, t, ex, tw, sy, my_round, refill);
      else Stages<V, L, Cfg::RMAX, INV, 0, Cfg::NR>::run(v, t, ex, tw, sy, my_round);
      if constexpr (TWID)
        if (a.copy_only != 2) interpass_scale<V, L, Cfg::RMAX, INV>(v, t, r, a.m_mask, a.fb, wc, wf);
    }
    if (f < a.fvalid) {
#pragma unroll
      for (int j = 0; j < Sh::R; ++j) {
        const int kk = out_index<L, Cfg::RMAX>(t, j);
        V x = v[j];
        if (scale != (Real)1) x = mk(x.x * scale, x.y * scale);
        if constexpr (MODE == 2) {
          const int d = kk / a.rows_per_rank;
          V* dst = reinterpret_cast<V*>(a.peers[d]);
          dst[out_base + f + (long long)(kk - d * a.rows_per_rank) * s_out] = x;
        } else {
          out[out_base + f + (long long)kk * s_out] = x;
        }
      }
    }
  }
}

// ------------------------------------------------------------------ K_COMB_H3
// K_COMB_TMA (1D inner pass, in-place exchange) with the tile split into two
// halves (comb steps [0, L/2) and [L/2, L)) over a ring of THREE half-tile
// slots: when tile k's exchange has been read back, its two half-slots take
// the second half of tile k+1 and the first half of tile k+2, so the first
// half of every tile is requested a whole tile earlier and the wait for the
// next tile covers only half of it. The exchange runs in place across the
// tile's two half-slots (index i -> half i / (L/2)).
template <typename Real, int L, int F_ = FOf<Real>::v>
struct CombH3Cfg {
  using Base = CombTmaCfg<Real, L, F_, true>;
  using V = C2<Real>;
  static constexpr int F = F_, H = L / 2;
  static constexpr int THREADS = Base::THREADS;
  static constexpr int HALF = H * F;                          // elements per half-tile slot
  static constexpr int HALF_BYTES = HALF * (int)sizeof(V);
  static constexpr int BL = Base::BL < H ? Base::BL : H;      // TMA box rows
  static constexpr int DATA_BYTES = 3 * HALF_BYTES;
  static constexpr int SMEM = DATA_BYTES + 3 * 8 + 128;
  static constexpr int WARPS = Base::WARPS;
  static constexpr int MINB_W = 16 / WARPS > 0 ? 16 / WARPS : 1;
  static constexpr int MINB_S = (227 * 1024) / (SMEM + 1024) > 0 ? (227 * 1024) / (SMEM + 1024) : 1;
  static constexpr int MINB = MINB_W < MINB_S ? MINB_W : MINB_S;
};

template <typename Real, int L, bool INV, int F_ = FOf<Real>::v>
__global__ void __launch_bounds__(CombH3Cfg<Real, L, F_>::THREADS, CombH3Cfg<Real, L, F_>::MINB)
k_comb_h3(const __grid_constant__ CUtensorMap tmap, C2<Real>* out, CombTmaArgs a, const C2<Real>* __restrict__ tw,
          const double2* __restrict__ wc, const double2* __restrict__ wf, Real scale) {
  using Cfg = CombH3Cfg<Real, L, F_>;
  using V = C2<Real>;
  using Sh = typename CombTmaCfg<Real, L, F_, true>::Sh;
  constexpr int F = Cfg::F, H = Cfg::H;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V* hs = reinterpret_cast<V*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + Cfg::DATA_BYTES);
  const int f = threadIdx.x % F, t = threadIdx.x / F;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 3; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue_half = [&](long long tile, int half, int slot) {
    const long long chunk = tile % a.chunks, g = tile / a.chunks;
    const long long batch = g / a.groups_per_batch, u = g % a.groups_per_batch;
    const int c0 = (int)(chunk * F * (sizeof(V) / 8));
    int c2 = 0, c3 = (int)(batch * a.groups_per_batch + u);
    if (a.in_t) {
      c2 = (int)u;
      c3 = (int)batch;
    }
    mbar_arrive_expect_tx(&full[slot], Cfg::HALF_BYTES);
#pragma unroll 1
    for (int n0 = 0; n0 < H; n0 += Cfg::BL)
      tma_load_4d(hs + slot * Cfg::HALF + n0 * F, &tmap, c0, half * H + n0, c2, c3, &full[slot]);
  };
  const long long G = gridDim.x;
  long long tile = blockIdx.x;
  int sa = 0, sb = 1, sc = 2;  // this tile's halves in (sa, sb); the next tile's first half in sc
  uint32_t ph = 0;             // bit s: parity of slot s's next completion
  if (threadIdx.x == 0 && tile < a.ntiles) {
    issue_half(tile, 0, 0);
    issue_half(tile, 1, 1);
    if (tile + G < a.ntiles) issue_half(tile + G, 0, 2);
  }
#pragma unroll 1
  for (; tile < a.ntiles; tile += G) {
    V* pa = hs + sa * Cfg::HALF;
    V* pb = hs + sb * Cfg::HALF;
    mbar_wait(&full[sa], (ph >> sa) & 1u);
    mbar_wait(&full[sb], (ph >> sb) & 1u);
    ph ^= (1u << sa) | (1u << sb);
    V v[Sh::R];
#pragma unroll
    for (int q = 0; q < Sh::R; ++q) {
      const int i = t + q * Sh::T;
      v[q] = (i < H ? pa : pb)[(i & (H - 1)) * F + f];
    }
    __syncthreads();  // every thread has its elements before the in-place exchange overwrites them
    const long long chunk = tile % a.chunks, g = tile / a.chunks;
    const long long batch = g / a.groups_per_batch, u = g % a.groups_per_batch;
    long long out_base = batch * a.bstride + u * a.sub_len + chunk * F, s_out = a.rps;
    if (a.t_l2) {
      const long long c0 = chunk * F;
      out_base = batch * a.bstride + (c0 / a.t_l2) * a.t_l0l2 + c0 % a.t_l2;
      s_out = a.t_l2;
    }
    const uint32_t r = (uint32_t)(chunk * F + f);
    const long long nx = tile + G, nn = tile + 2 * G;
    const int sb_ = sa, sc_ = sb;
    auto refill = [&]() {
      fence_proxy_async_smem();
      __syncthreads();  // both half-slots fully consumed: the next tile's second half, the one after's first
      if (threadIdx.x == 0) {
        if (nx < a.ntiles) issue_half(nx, 1, sb_);
        if (nn < a.ntiles) issue_half(nn, 0, sc_);
      }
    };
    auto ex = [pa, pb, f](int i) -> V& { return (i < H ? pa : pb)[(i & (H - 1)) * F + f]; };
    SyncBlock sy;
    Stages<V, L, RmaxOf<Real>::v, INV, 0, 1>::run(v, t, ex, tw, sy, 0, refill);
    interpass_scale<V, L, RmaxOf<Real>::v, INV>(v, t, r, a.m_mask, a.fb, wc, wf);
#pragma unroll
    for (int j = 0; j < Sh::R; ++j) {
      const int kk = out_index<L, RmaxOf<Real>::v>(t, j);
      V x = v[j];
      if (scale != (Real)1) x = mk(x.x * scale, x.y * scale);
      out[out_base + f + (long long)kk * s_out] = x;
    }
    // rotate: next tile = (sc, sa), the tile after's first half goes to sb
    const int na = sc, nb = sa, nc = sb;
    sa = na;
    sb = nb;
    sc = nc;
  }
}

// ------------------------------------------------------------------ K_FINAL_T
// Final pass of a multi-pass 1D plan (tiled_fft.hpp:295-306): rows are
// contiguous on input but the digit interleave scatters each spectrum with
// stride out_weights[p-1]. The CTA takes the 16 rows whose leading digit d0
// is consecutive (grow = d0*sub_w[0] + o), so for every k the 16 results are
// 16 consecutive outputs; the row FFTs run lanes-along-n (coalesced loads),
// then one padded [k][17] shared-memory transpose turns the lanes around for
// 128-byte stores.
struct FinalArgs {
  long long bstride, n;      // batch stride, transform length
  long long ntiles, chunks;  // chunks = f0 / 16
  long long sw0;             // sub_weights[0]
  long long out_w_last;
  int p;
  long long out_w[8], sub_w[8];
};

template <typename Real, int L, int F_ = FOf<Real>::v>
struct FinalCfg {
  using V = C2<Real>;
  static constexpr int RMAX = RmaxOf<Real>::v;
  using Sh = Shape<L, RMAX>;
  static constexpr int F = F_;
  static constexpr int THREADS = F * Sh::T;
  // FFT regions == T (mod 16) and a transpose row stride F + 16/T: every
  // half-warp access (several FFTs per half-warp when T < 16) is conflict free
  static constexpr int REG = RegionPad<L, Sh::T>::v;
  static constexpr int TS = F + (Sh::T >= 16 ? 1 : 16 / Sh::T);
  static constexpr int A = F * REG, B = L * TS;
  static constexpr int SMEM = (A > B ? A : B) * (int)sizeof(V);
};

// tile -> (batch, leading-digit chunk, other digits o), chunks fastest: concurrent CTAs write adjacent
// 128-byte lines of the same output rows (the lines of one tile are out_w_last apart, 8 MB at 2^30), so
// they reach L2 together -- 2^26 final pass 195 vs 205 us, 2^30 3.47 vs 3.53 ms against o fastest
// (tools/gpu/r02_fcfirst.sh)
struct FinalTileGeo {
  long long batch, chunk, o;
};
__device__ __forceinline__ FinalTileGeo final_geo(const FinalArgs& a, long long tile) {
  const long long tiles_per_batch = a.chunks * a.sw0;
  const long long rem = tile % tiles_per_batch;
  return {tile / tiles_per_batch, rem % a.chunks, rem / a.chunks};
}

// phase 0: this thread's R elements of row (chunk*F + ff)*sw0 + o, lanes along n (coalesced loads)
template <typename Real, int L, int F_>
__device__ __forceinline__ void final_load(const C2<Real>* in, const FinalArgs& a, long long tile, C2<Real>* v) {
  using Cfg = FinalCfg<Real, L, F_>;
  using Sh = typename Cfg::Sh;
  const FinalTileGeo g = final_geo(a, tile);
  const int ff = threadIdx.x / Sh::T, t = threadIdx.x % Sh::T;
  const long long grow = (g.chunk * Cfg::F + ff) * a.sw0 + g.o;
  const C2<Real>* src = in + g.batch * a.bstride + grow * L;
#pragma unroll
  for (int q = 0; q < Sh::R; ++q) v[q] = src[t + q * Sh::T];
}

// phase 1: the row FFT in registers (exchange in the row's padded region), then the spectrum written
// transposed, sm[k * TS + ff]; ends with the CTA barrier that makes it visible to phase 2
template <typename Real, int L, bool INV, int F_>
__device__ __forceinline__ void final_fft(C2<Real>* v, const C2<Real>* __restrict__ tw, C2<Real>* sm) {
  using Cfg = FinalCfg<Real, L, F_>;
  using V = C2<Real>;
  using Sh = typename Cfg::Sh;
  const int ff = threadIdx.x / Sh::T, t = threadIdx.x % Sh::T;
  V* reg = sm + ff * Cfg::REG;
  auto ex = [reg](int i) -> V& { return reg[pad32(i)]; };
  SyncBlock s;
  Stages<V, L, Cfg::RMAX, INV, 0>::run(v, t, ex, tw, s);
  __syncthreads();  // exchange regions are reused by the transpose below
#pragma unroll
  for (int j = 0; j < Sh::R; ++j) sm[out_index<L, Cfg::RMAX>(t, j) * Cfg::TS + ff] = v[j];
  __syncthreads();
}

// phase 2: lanes along the 16 consecutive outputs of each k
template <typename Real, int L, int F_>
__device__ __forceinline__ void final_store(C2<Real>* out, const FinalArgs& a, long long tile, const C2<Real>* sm,
                                            Real scale) {
  using Cfg = FinalCfg<Real, L, F_>;
  using V = C2<Real>;
  constexpr int F = Cfg::F;
  const FinalTileGeo g = final_geo(a, tile);
  const int f = threadIdx.x % F, kk = threadIdx.x / F;
  constexpr int KSTEP = Cfg::THREADS / F;
  // out index of (d0 = chunk*16 + f, other digits from o) = d0 + final(o)
  long long outi = 0, r2 = g.o;
  for (int i = 0; i + 1 < a.p; ++i) {
    const long long d = r2 / a.sub_w[i];
    r2 -= d * a.sub_w[i];
    outi += d * a.out_w[i];
  }
  const long long ob = g.batch * a.bstride + g.chunk * F + f + outi;
#pragma unroll 4
  for (int k = kk; k < L; k += KSTEP) {
    V x = sm[k * Cfg::TS + f];
    if (scale != (Real)1) x = mk(x.x * scale, x.y * scale);
    out[ob + (long long)k * a.out_w_last] = x;
  }
}

template <typename Real, int L, bool INV, int F_>
__device__ __forceinline__ void final_tile(const C2<Real>* in, C2<Real>* out, const FinalArgs& a,
                                           const C2<Real>* __restrict__ tw, Real scale, long long tile, C2<Real>* sm) {
  C2<Real> v[FinalCfg<Real, L, F_>::Sh::R];
  final_load<Real, L, F_>(in, a, tile, v);
  final_fft<Real, L, INV, F_>(v, tw, sm);
  final_store<Real, L, F_>(out, a, tile, sm, scale);
}

template <typename Real, int L, bool INV, int F_ = FOf<Real>::v>
__global__ void __launch_bounds__(FinalCfg<Real, L, F_>::THREADS, FinalCfg<Real, L, F_>::THREADS <= 256 ? 2 : 1)
k_final_t(const C2<Real>* in, C2<Real>* out, FinalArgs a, const C2<Real>* __restrict__ tw, Real scale) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  final_tile<Real, L, INV, F_>(in, out, a, tw, scale, blockIdx.x, reinterpret_cast<C2<Real>*>(smem_raw));
}

// Persistent K_FINAL_T with the next tile's loads in flight during this tile's stores: once the
// spectrum sits transposed in shared memory the row registers are free, so they take the next
// tile's elements (plain loads, no extra shared memory) while the stores drain from shared memory.
template <typename Real, int L, bool INV, int F_, int MINB>
__global__ void __launch_bounds__(FinalCfg<Real, L, F_>::THREADS, MINB)
k_final_p(const C2<Real>* in, C2<Real>* out, FinalArgs a, const C2<Real>* __restrict__ tw, Real scale) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C2<Real>* sm = reinterpret_cast<C2<Real>*>(smem_raw);
  long long tile = blockIdx.x;
  if (tile >= a.ntiles) return;
  C2<Real> v[FinalCfg<Real, L, F_>::Sh::R];
  final_load<Real, L, F_>(in, a, tile, v);
#pragma unroll 1
  for (;;) {
    final_fft<Real, L, INV, F_>(v, tw, sm);
    const long long next = tile + gridDim.x;
    if (next < a.ntiles) final_load<Real, L, F_>(in, a, next, v);
    final_store<Real, L, F_>(out, a, tile, sm, scale);
    if (next >= a.ntiles) break;
    tile = next;
    __syncthreads();  // the next FFT's exchange overwrites the transposed tile
  }
}

// ------------------------------------------------------------------ K_ROWS_PF
// Persistent K_ROWS for long fp32 rows (L = 2048..8192: one CTA per row,
// 2 CTAs per SM). The row's shared-memory exchange region doubles as the
// landing zone of the NEXT row: as soon as the last exchange is done, one
// bulk copy (TMA, 1D) streams the next row in, so its DRAM latency overlaps
// the last radix stage and the stores of the current row. The first read of
// a row (lanes along n, unpadded) is bank-conflict free without the pad.
template <int L>
struct RowsPfCfg {
  using Sh = Shape<L, 32>;
  static constexpr int THREADS = Sh::T;
  static constexpr int REG = L + L / 32 + 1;
  static constexpr int SMEM = REG * 8 + 16;
};

template <int L, bool INV>
__global__ void __launch_bounds__(RowsPfCfg<L>::THREADS, 2)
k_rows_pf(const float2* __restrict__ in, float2* __restrict__ out, long long nrows, const float2* __restrict__ tw,
          float scale) {
  using Cfg = RowsPfCfg<L>;
  using V = float2;
  using Sh = typename Cfg::Sh;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V* sm = reinterpret_cast<V*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + Cfg::REG);
  const int t = threadIdx.x;
  long long row = blockIdx.x;
  auto issue = [&](long long r) {
    mbar_arrive_expect_tx(full, L * 8);
    tma_load_1d(sm, in + r * L, L * 8, full);
  };
  if (t == 0) {
    mbar_init(full, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (t == 0 && row < nrows) issue(row);
  uint32_t phase = 0;
#pragma unroll 1
  for (; row < nrows; row += gridDim.x) {
    mbar_wait(full, phase);
    phase ^= 1;
    V v[Sh::R];
#pragma unroll
    for (int q = 0; q < Sh::R; ++q) v[q] = sm[t + q * Sh::T];
    __syncthreads();  // the exchange below overwrites the landing zone
    auto ex = [sm](int i) -> V& { return sm[pad32(i)]; };
    const long long nxt = row + gridDim.x;
    auto prefetch = [&]() {
      fence_proxy_async_smem();
      __syncthreads();
      if (t == 0 && nxt < nrows) issue(nxt);
    };
    SyncBlock sy;
    Stages<V, L, 32, INV, 0>::run(v, t, ex, tw, sy, 0, prefetch);
    V* dst = out + row * L;
#pragma unroll
    for (int j = 0; j < Sh::R; ++j) {
      V r = v[j];
      if (scale != 1.0f) r = mk(r.x * scale, r.y * scale);
      dst[out_index<L, 32>(t, j)] = r;
    }
  }
}

}  // namespace tfb
