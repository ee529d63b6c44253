// Shared device building blocks for the B200 tilefft kernels.
//
//  * compile-time unit roots (constexpr sin/cos evaluated by the front end, so
//    the in-register DFTs carry their twiddles as immediates);
//  * complex helpers for float2/double2;
//  * `RegDFT<R, INV>`: an R-point DFT (R = 2..32) held entirely in one thread's
//    registers — the "per-block sub-FFT in registers" of the paper's method
//    (PAPER.md:145-191), here one radix-2 DIF network with trivial roots
//    (1, -i, W8) specialised at compile time.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <utility>

namespace tfb {

// ---------------------------------------------------------------- constexpr trig
constexpr double kPi = 3.141592653589793238462643383279502884;

constexpr double ce_sin_small(double x) {  // |x| <= pi/4
  double x2 = x * x, term = x, sum = x;
  for (int k = 1; k < 14; ++k) {
    term *= -x2 / ((2.0 * k) * (2.0 * k + 1.0));
    sum += term;
  }
  return sum;
}
constexpr double ce_cos_small(double x) {
  double x2 = x * x, term = 1.0, sum = 1.0;
  for (int k = 1; k < 14; ++k) {
    term *= -x2 / ((2.0 * k - 1.0) * (2.0 * k));
    sum += term;
  }
  return sum;
}
// cos(2*pi*j/n), sin(2*pi*j/n) for 0 <= j < n, via octant reduction (exact
// on the axes and the diagonals' symmetry).
struct CS { double c, s; };
constexpr CS ce_unit(long long j, long long n) {
  j %= n;
  if (j < 0) j += n;
  // map to first octant using the 8-fold symmetry on the integer grid (n % 8 == 0
  // is not required: fall back to direct evaluation when it does not divide).
  if (n % 8 == 0) {
    const long long o = n / 8;
    const long long q = j / o, r = j % o;  // octant q, offset r
    const double a = 2.0 * kPi * (double)r / (double)n;
    double c = ce_cos_small(a), s = ce_sin_small(a);
    // angle = q*pi/4 + a
    const double h = 0.707106781186547524400844362104849039;
    double cq[8] = {1, h, 0, -h, -1, -h, 0, h};
    double sq[8] = {0, h, 1, h, 0, -h, -1, -h};
    if (r == 0) return CS{cq[q], sq[q]};
    return CS{cq[q] * c - sq[q] * s, sq[q] * c + cq[q] * s};
  }
  if (j == 0) return CS{1.0, 0.0};
  if (2 * j == n) return CS{-1.0, 0.0};
  if (4 * j == n) return CS{0.0, 1.0};
  if (4 * j == 3 * n) return CS{0.0, -1.0};
  const double a = 2.0 * kPi * (double)j / (double)n;  // n in {2,4}: handled above
  return CS{ce_cos_small(a), ce_sin_small(a)};
}

// ---------------------------------------------------------------- complex helpers
template <typename Real> struct C2T;
template <> struct C2T<float> { using type = float2; };
template <> struct C2T<double> { using type = double2; };
template <typename Real> using C2 = typename C2T<Real>::type;

__device__ __forceinline__ float2 mk(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ double2 mk(double a, double b) { return make_double2(a, b); }

template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return mk(a.x + b.x, a.y + b.y); }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return mk(a.x - b.x, a.y - b.y); }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
  return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <typename V> __device__ __forceinline__ V cmulc(V a, V b) {
  return mk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
// multiply by forward root W (INV=false) or its conjugate (INV=true)
template <bool INV, typename V> __device__ __forceinline__ V ctw(V a, V w) {
  if constexpr (INV) return cmulc(a, w);
  else return cmul(a, w);
}

// z * W_N^J with W_N = exp(-2 pi i / N) (forward) or its conjugate (INV).
// J, N are template constants: the root is a front-end constant and the
// trivial roots (1, -1, -+i, W8 family) cost no general multiply.
template <bool INV, int J_, int N>
struct RotC {
  static constexpr int J = ((J_ % N) + N) % N;
  template <typename V>
  __device__ __forceinline__ static V apply(V z) {
    using R = decltype(z.x);
    constexpr R h = (R)0.707106781186547524400844362104849039;
    if constexpr (J == 0) return z;
    else if constexpr (2 * J == N) return mk(-z.x, -z.y);
    else if constexpr (4 * J == N) { if constexpr (INV) return mk(-z.y, z.x); else return mk(z.y, -z.x); }
    else if constexpr (4 * J == 3 * N) { if constexpr (INV) return mk(z.y, -z.x); else return mk(-z.y, z.x); }
    else if constexpr (8 * J == N) {
      if constexpr (INV) return mk((z.x - z.y) * h, (z.x + z.y) * h); else return mk((z.x + z.y) * h, (z.y - z.x) * h);
    } else if constexpr (8 * J == 3 * N) {
      if constexpr (INV) return mk((-z.x - z.y) * h, (z.x - z.y) * h); else return mk((z.y - z.x) * h, (-z.x - z.y) * h);
    } else if constexpr (8 * J == 5 * N) {
      if constexpr (INV) return mk((z.y - z.x) * h, (-z.x - z.y) * h); else return mk((-z.x - z.y) * h, (z.x - z.y) * h);
    } else if constexpr (8 * J == 7 * N) {
      if constexpr (INV) return mk((z.x + z.y) * h, (z.y - z.x) * h); else return mk((z.x - z.y) * h, (z.x + z.y) * h);
    } else {
      constexpr CS cs = ce_unit(J, N);
      constexpr R c = (R)cs.c, s = (R)cs.s;  // W = c - i s (forward)
      if constexpr (INV) return mk(z.x * c - z.y * s, z.x * s + z.y * c);
      else return mk(z.x * c + z.y * s, z.y * c - z.x * s);
    }
  }
};

// ---------------------------------------------------------------- register DFT
// In place, natural-order input v[0..R) -> natural-order output v[0..R).
// Radix-2 decimation in frequency unrolled by template recursion, then the
// bit-reversal renaming (free: all indices are compile-time).
template <int R>
struct BitRev {
  static constexpr int bits = R <= 1 ? 0 : (R == 2 ? 1 : R == 4 ? 2 : R == 8 ? 3 : R == 16 ? 4 : R == 32 ? 5 : 6);
  __host__ __device__ static constexpr int rev(int x) {
    int r = 0;
    for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
    return r;
  }
};

template <int R, bool INV, int SPAN>
struct DifStage {
  template <int I, typename V>
  __device__ __forceinline__ static void bfly(V* v) {
    constexpr int j = I % SPAN, blk = (I / SPAN) * 2 * SPAN;
    const V a = v[blk + j], b = v[blk + j + SPAN];
    v[blk + j] = cadd(a, b);
    v[blk + j + SPAN] = RotC<INV, j, 2 * SPAN>::apply(csub(a, b));
  }
  template <typename V, int... Is>
  __device__ __forceinline__ static void all(V* v, std::integer_sequence<int, Is...>) {
    (bfly<Is>(v), ...);
  }
  template <typename V>
  __device__ __forceinline__ static void run(V* v) {
    all(v, std::make_integer_sequence<int, R / 2>{});
    if constexpr (SPAN > 1) DifStage<R, INV, SPAN / 2>::run(v);
  }
};

template <int R, bool INV, typename V>
__device__ __forceinline__ void reg_dft(V* v) {
  static_assert(R >= 1 && R <= 64 && (R & (R - 1)) == 0, "radix must be a power of two <= 64");
  if constexpr (R > 1) {
    DifStage<R, INV, R / 2>::run(v);
    V t[R];
#pragma unroll
    for (int k = 0; k < R; ++k) t[k] = v[BitRev<R>::rev(k)];
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = t[k];
  }
}

// ---------------------------------------------------------------- misc
__host__ __device__ constexpr int ilog2c(long long v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }

}  // namespace tfb
