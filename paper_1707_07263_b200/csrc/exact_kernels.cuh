// Exact-mode pass kernel: reproduces the reference's fft_tiled arithmetic bit
// for bit on the GPU (SURVEY §8c tier 2). It executes the caller's plan
// factors literally: gather through the bit-reversed comb
// (tiled_fft.hpp:265-272), log2(L) radix-2 DIT levels with the table roots
// W_{2h}^j (dit_levels, :89-117; butterfly, fft_baseline.hpp:30-36), then the
// twiddled scatter (:284-294) or the digit interleave (:295-306). Every
// product and sum is an explicitly rounded IEEE op (__fmul_rn/__fadd_rn), so
// no multiply-add is fused — the reference is compiled without FMA.
// Roots are the reference table's own values (`tbl` = W_N^e, e < N, taken
// from the caller's TwiddleTable at stride resolution/N).
#pragma once
#include "fft_common.cuh"

namespace tfb {

__device__ __forceinline__ float rn_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float rn_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float rn_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rn_sub(double a, double b) { return __dsub_rn(a, b); }

struct ExactArgs {
  long long n;            // transform length (= plan.n_total)
  long long rows;         // rows of this pass per transform
  long long bstride;      // elements between batch items
  long long L, sub_len, rps;
  int levels;
  int has_inter;          // pass < p
  int p;
  int conj_in;            // ifft: conjugate on the first gather
  int conj_scale_out;     // ifft: conjugate and scale on the final store
  int permute_only;       // index-map check mode: butterflies and roots off
  long long out_w[64], sub_w[64];
};

template <typename Real>
__global__ void k_exact_pass(const C2<Real>* in, C2<Real>* out, ExactArgs a, const C2<Real>* __restrict__ tbl,
                             Real scale) {
  using V = C2<Real>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V* row = reinterpret_cast<V*>(smem_raw);
  const long long id = blockIdx.x;
  const long long batch = id / a.rows, grow = id % a.rows;
  const long long sub = grow / a.rps, r = grow % a.rps;
  const long long base = batch * a.bstride + sub * a.sub_len + r;
  const int L = (int)a.L;
  // gather (bit-reversed comb)
  for (int c = threadIdx.x; c < L; c += blockDim.x) {
    const unsigned rc = __brev((unsigned)c) >> (32 - a.levels);
    V x = in[base + (long long)(a.levels ? rc : 0) * a.rps];
    if (a.conj_in) x.y = -x.y;
    row[c] = x;
  }
  __syncthreads();
  if (!a.permute_only) {
    for (int lv = 0; lv < a.levels; ++lv) {
      const int h = 1 << lv;
      const long long tstride = a.n / (2LL * h);
      for (int i = threadIdx.x; i < L / 2; i += blockDim.x) {
        const int j = i & (h - 1);
        const int lo = ((i >> lv) << (lv + 1)) + j, hi = lo + h;
        const V w = tbl[(long long)j * tstride];
        const V b = row[hi], av = row[lo];
        const Real tr = rn_sub(rn_mul(w.x, b.x), rn_mul(w.y, b.y));
        const Real ti = rn_add(rn_mul(w.x, b.y), rn_mul(w.y, b.x));
        row[lo] = mk(rn_add(av.x, tr), rn_add(av.y, ti));
        row[hi] = mk(rn_sub(av.x, tr), rn_sub(av.y, ti));
      }
      __syncthreads();
    }
  }
  if (a.has_inter) {
    const unsigned long long mask = (unsigned long long)a.sub_len - 1;
    const long long tstride = a.n / a.sub_len;
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
      V x = row[k];
      if (!a.permute_only) {
        const unsigned long long e = ((unsigned long long)r * (unsigned long long)k) & mask;
        const V w = tbl[(long long)e * tstride];
        x = mk(rn_sub(rn_mul(x.x, w.x), rn_mul(x.y, w.y)), rn_add(rn_mul(x.x, w.y), rn_mul(x.y, w.x)));
      }
      out[base + (long long)k * a.rps] = x;
    }
  } else {
    long long ob = 0, rem = grow;
    for (int i = 0; i + 1 < a.p; ++i) {
      const long long d = rem / a.sub_w[i];
      rem -= d * a.sub_w[i];
      ob += d * a.out_w[i];
    }
    ob += batch * a.bstride;
    const long long wgt = a.out_w[a.p - 1];
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
      V x = row[k];
      if (a.conj_scale_out) x = mk(rn_mul(x.x, scale), rn_mul(-x.y, scale));
      out[ob + (long long)k * wgt] = x;
    }
  }
}

// ---------------------------------------------------------------- levelwise
// The paper's "previous method" (§2.2; fft_levelwise,
// fft_baseline.hpp:66-116): one bit-reversal sweep, then one launch per
// radix-2 level, each reading and writing all n elements in global memory.
// Same table roots and separately rounded ops as the reference, so the output
// is bit-identical to fft_levelwise<Real>.
template <typename Real>
__global__ void k_bitrev_permute(const C2<Real>* in, C2<Real>* out, long long n, int bits, long long total,
                                 int conj_in) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / n, j = i % n;
    const unsigned long long r = __brevll((unsigned long long)j) >> (64 - bits);
    C2<Real> x = in[b * n + (long long)r];
    if (conj_in) x.y = -x.y;
    out[i] = x;
  }
}

template <typename Real>
__global__ void k_level(const C2<Real>* w, C2<Real>* o, long long n, int lv, long long total_half,
                        const C2<Real>* __restrict__ tbl, int conj_scale_out, Real scale) {
  using V = C2<Real>;
  const long long h = 1LL << lv;
  const long long tstride = n / (2 * h);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total_half;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / (n / 2), k = i % (n / 2);
    const long long j = k & (h - 1);
    const long long lo = b * n + ((k >> lv) << (lv + 1)) + j, hi = lo + h;
    const V wv = tbl[j * tstride];
    const V bv = w[hi], av = w[lo];
    const Real tr = rn_sub(rn_mul(wv.x, bv.x), rn_mul(wv.y, bv.y));
    const Real ti = rn_add(rn_mul(wv.x, bv.y), rn_mul(wv.y, bv.x));
    V a = mk(rn_add(av.x, tr), rn_add(av.y, ti)), c = mk(rn_sub(av.x, tr), rn_sub(av.y, ti));
    if (conj_scale_out) {
      a = mk(rn_mul(a.x, scale), rn_mul(-a.y, scale));
      c = mk(rn_mul(c.x, scale), rn_mul(-c.y, scale));
    }
    o[lo] = a;
    o[hi] = c;
  }
}

// Decomposed helpers of the reference API (tiled_fft.hpp:153-203), exact:
// element (r, k) of a rows x cols tile times W_sub^{((row0+r) % rps) * k}
// (element as left operand), and the stage store permutation.
template <typename Real>
__global__ void k_interstage_scale(const C2<Real>* in, C2<Real>* out, long long rows, long long cols, long long row0,
                                   long long rps, long long sub_len, const C2<Real>* __restrict__ tbl,
                                   long long tstride) {
  const long long total = rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = ((row0 + i / cols) % rps), k = i % cols;
    const unsigned long long e = ((unsigned long long)r * (unsigned long long)k) & (unsigned long long)(sub_len - 1);
    const C2<Real> w = tbl[(long long)e * tstride], x = in[i];
    out[i] = mk(rn_sub(rn_mul(x.x, w.x), rn_mul(x.y, w.y)), rn_add(rn_mul(x.x, w.y), rn_mul(x.y, w.x)));
  }
}

struct ExchangeArgs {
  long long n, L, sub_len, rps;
  int final_pass, p;
  long long out_w[64], sub_w[64];
};

// out[exchange_index_map(stage, q)] = in[q] (stage_plan.hpp:161-172)
template <typename Real>
__global__ void k_exchange(const C2<Real>* in, C2<Real>* out, ExchangeArgs a) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < a.n; q += (long long)gridDim.x * blockDim.x) {
    long long dst;
    if (!a.final_pass) {
      const long long sub = q / a.sub_len, local = q % a.sub_len;
      dst = sub * a.sub_len + (local % a.L) * a.rps + local / a.L;
    } else {
      long long rem = q / a.L;
      dst = (q % a.L) * a.out_w[a.p - 1];
      for (int i = 0; i + 1 < a.p; ++i) {
        const long long d = rem / a.sub_w[i];
        rem -= d * a.sub_w[i];
        dst += d * a.out_w[i];
      }
    }
    out[dst] = in[q];
  }
}

}  // namespace tfb
