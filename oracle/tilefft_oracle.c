/* tilefft oracle — TEST INFRASTRUCTURE ONLY (see tilefft_oracle.h).
 *
 * CPU restatement of the reference's fft_tiled path. Each function cites the
 * reference file:line it follows (paths relative to
 * /root/reference/proj/include/tilefft/). Build: oracle/Makefile, with
 * -ffp-contract=off so that no multiply-add is fused (the reference is built
 * for baseline x86-64, which has no FMA: proj/CMakeLists.txt has no -march).
 */
#include "tilefft_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.141592653589793238462643383279502884; /* common.hpp:33 */

static int is_pow2(uint64_t v) { return v != 0 && (v & (v - 1)) == 0; } /* common.hpp:36-38 */
static uint32_t log2_exact(uint64_t v) { return (uint32_t)__builtin_ctzll(v); } /* common.hpp:41-43 */

/* common.hpp:54-60 */
uint64_t orc_bit_reverse(uint64_t value, uint32_t bits) {
  uint64_t out = 0;
  for (uint32_t i = 0; i < bits; ++i) out = (out << 1) | ((value >> i) & 1u);
  return out;
}

/* stage_plan.hpp:74-127 (bank_count comes from ExecConfig, exec_model.hpp:33-53) */
int orc_make_plan(uint64_t n, uint64_t cap, uint32_t bank_count, orc_plan* p) {
  if (!is_pow2(n) || n < 2) return -1;
  if (!is_pow2(cap) || cap < 2) return -1;
  if (!is_pow2(bank_count)) return -1;
  memset(p, 0, sizeof(*p));
  const uint64_t total_bits = log2_exact(n), cap_bits = log2_exact(cap);
  const uint64_t passes = (total_bits + cap_bits - 1) / cap_bits;
  const uint64_t base_bits = total_bits / passes, extra = total_bits % passes;
  if (passes > ORC_MAX_PASSES) return -1;
  p->n_total = n;
  p->tile_capacity = cap;
  p->bank_count = bank_count;
  p->passes = (uint32_t)passes;
  for (uint64_t s = 0; s < passes; ++s) p->factors[s] = 1ull << (base_bits + (s < extra ? 1 : 0));
  uint64_t sub_len = n;
  for (uint64_t s = 0; s < passes; ++s) {
    orc_geom* g = &p->stages[s];
    g->fft_len = p->factors[s];
    g->levels = log2_exact(g->fft_len);
    g->rows = n / g->fft_len;
    g->sub_len = sub_len;
    g->rows_per_sub = sub_len / g->fft_len;
    g->padded_stride = g->fft_len + (g->fft_len % bank_count == 0 ? 1 : 0);
    g->rows_per_tile = g->rows < cap / g->fft_len ? g->rows : cap / g->fft_len;
    g->tile_count = g->rows / g->rows_per_tile;
    sub_len = g->rows_per_sub;
  }
  p->out_weights[0] = 1;
  for (uint64_t i = 1; i < passes; ++i) p->out_weights[i] = p->out_weights[i - 1] * p->factors[i - 1];
  /* sub_weights has passes-1 entries (stage_plan.hpp:120-125) */
  for (uint64_t i = passes - 1; i-- > 0;)
    p->sub_weights[i] = (i + 1 < passes - 1) ? p->sub_weights[i + 1] * p->factors[i + 1] : 1;
  return 0;
}

/* stage_plan.hpp:135-140 (stage is 1-based) */
uint64_t orc_gather_source_index(const orc_plan* p, uint32_t stage, uint64_t grow, uint64_t col) {
  const orc_geom* g = &p->stages[stage - 1];
  return (grow / g->rows_per_sub) * g->sub_len + grow % g->rows_per_sub + col * g->rows_per_sub;
}

/* stage_plan.hpp:144-155 */
uint64_t orc_final_output_index(const orc_plan* p, uint64_t sub, uint64_t k) {
  uint64_t out = k * p->out_weights[p->passes - 1], rem = sub;
  for (uint32_t i = 0; i + 1 < p->passes; ++i) {
    const uint64_t digit = rem / p->sub_weights[i];
    rem %= p->sub_weights[i];
    out += digit * p->out_weights[i];
  }
  return out;
}

/* stage_plan.hpp:161-172 */
uint64_t orc_exchange_index_map(const orc_plan* p, uint32_t stage, uint64_t q) {
  const orc_geom* g = &p->stages[stage - 1];
  if (stage < p->passes) {
    const uint64_t sub = q / g->sub_len, local = q % g->sub_len;
    return sub * g->sub_len + (local % g->fft_len) * g->rows_per_sub + local / g->fft_len;
  }
  return orc_final_output_index(p, q / g->fft_len, q % g->fft_len);
}

/* ---- real-typed bodies, instantiated for float and double ---------------- */
#define ORC_DEFINE(REAL, SUF)                                                                    \
  /* twiddle.hpp:47-73 */                                                                        \
  int orc_build_twiddle_##SUF(uint64_t R, REAL* t) {                                             \
    if (!is_pow2(R) || R < 2) return -1;                                                         \
    memset(t, 0, sizeof(REAL) * 2 * R);                                                          \
    t[0] = (REAL)1; t[1] = (REAL)0;                                                              \
    t[2 * (R / 2)] = (REAL)-1; t[2 * (R / 2) + 1] = (REAL)0;                                     \
    if (R >= 4) {                                                                                \
      t[2 * (R / 4)] = (REAL)0; t[2 * (R / 4) + 1] = (REAL)-1;                                   \
      t[2 * (3 * R / 4)] = (REAL)0; t[2 * (3 * R / 4) + 1] = (REAL)1;                            \
    }                                                                                            \
    for (uint64_t j = 1; j < R / 4; ++j) {                                                       \
      const double angle = 2.0 * kPi * (double)j / (double)R;                                    \
      const REAL c = (REAL)cos(angle), s = (REAL)sin(angle);                                     \
      t[2 * j] = c; t[2 * j + 1] = -s;                                                           \
      t[2 * (R / 2 - j)] = -c; t[2 * (R / 2 - j) + 1] = -s;                                      \
      t[2 * (R / 2 + j)] = -c; t[2 * (R / 2 + j) + 1] = s;                                       \
      t[2 * (R - j)] = c; t[2 * (R - j) + 1] = s;                                                \
    }                                                                                            \
    return 0;                                                                                    \
  }                                                                                              \
                                                                                                 \
  /* One pass: tiled_fft.hpp:229-310 with dit_levels :89-117, butterfly                         \
     fft_baseline.hpp:30-36, twiddle_fetch fft_baseline.hpp:53-57. Rows are                      \
     independent, so the tile grouping (rows_per_tile) does not change values. */                \
  static void pass_##SUF(const orc_plan* p, uint32_t stage, const REAL* in, REAL* out,           \
                         const REAL* tbl, uint64_t R, REAL* row, int permute_only) {              \
    const orc_geom* g = &p->stages[stage - 1];                                                   \
    const uint64_t L = g->fft_len, rps = g->rows_per_sub;                                        \
    const uint32_t bits = (uint32_t)g->levels;                                                   \
    const int has_inter = stage < p->passes;                                                     \
    const uint64_t sub_mask = g->sub_len - 1, tstride = R / g->sub_len;                          \
    for (uint64_t grow = 0; grow < g->rows; ++grow) {                                            \
      const uint64_t sub = grow / rps, r = grow % rps, base = sub * g->sub_len + r;              \
      for (uint64_t c = 0; c < L; ++c) { /* gather :265-272 */                                   \
        const uint64_t src = base + orc_bit_reverse(c, bits) * rps;                              \
        row[2 * c] = in[2 * src]; row[2 * c + 1] = in[2 * src + 1];                              \
      }                                                                                          \
      if (!permute_only) {                                                                       \
        for (uint64_t h = 1; h < L; h <<= 1) { /* levels :101-116 */                             \
          for (uint64_t blk = 0; blk < L; blk += 2 * h) {                                        \
            for (uint64_t j = 0; j < h; ++j) {                                                   \
              const uint64_t ti = (j & (2 * h - 1)) * (R / (2 * h));                             \
              const REAL wr = tbl[2 * ti], wi = tbl[2 * ti + 1];                                 \
              REAL* lo = row + 2 * (blk + j);                                                    \
              REAL* hi = row + 2 * (blk + j + h);                                                \
              const REAL br = hi[0], bi = hi[1];                                                 \
              const REAL tr = wr * br - wi * bi;                                                 \
              const REAL tim = wr * bi + wi * br;                                                \
              const REAL ar = lo[0], ai = lo[1];                                                 \
              lo[0] = ar + tr; lo[1] = ai + tim;                                                 \
              hi[0] = ar - tr; hi[1] = ai - tim;                                                 \
            }                                                                                    \
          }                                                                                      \
        }                                                                                        \
      }                                                                                          \
      if (has_inter) { /* twiddled scatter :284-294; element is the left operand */              \
        uint64_t acc = 0;                                                                        \
        for (uint64_t k = 0; k < L; ++k) {                                                       \
          const uint64_t dst = base + k * rps;                                                   \
          const REAL xr = row[2 * k], xi = row[2 * k + 1];                                       \
          if (permute_only) {                                                                    \
            out[2 * dst] = xr; out[2 * dst + 1] = xi;                                            \
          } else {                                                                               \
            const uint64_t ti = (acc & sub_mask) * tstride;                                      \
            const REAL wr = tbl[2 * ti], wi = tbl[2 * ti + 1];                                   \
            out[2 * dst] = xr * wr - xi * wi;                                                    \
            out[2 * dst + 1] = xr * wi + xi * wr;                                                \
          }                                                                                      \
          acc += r;                                                                              \
        }                                                                                        \
      } else { /* digit interleave :295-306 */                                                   \
        const uint64_t ob = orc_final_output_index(p, grow, 0);                                  \
        const uint64_t wgt = p->out_weights[p->passes - 1];                                      \
        for (uint64_t k = 0; k < L; ++k) {                                                       \
          out[2 * (ob + k * wgt)] = row[2 * k];                                                  \
          out[2 * (ob + k * wgt) + 1] = row[2 * k + 1];                                          \
        }                                                                                        \
      }                                                                                          \
    }                                                                                            \
  }                                                                                              \
                                                                                                 \
  static int tiled_##SUF(const REAL* x, REAL* out, const orc_plan* p, const REAL* tbl,           \
                         uint64_t R, int permute_only) {                                         \
    const uint64_t n = p->n_total;                                                               \
    if (p->passes < 1) return -1;                                                                \
    if (!permute_only && !(R >= n && R % n == 0)) return -1; /* tiled_fft.hpp:328-329 */        \
    uint64_t maxL = 0;                                                                           \
    for (uint32_t s = 0; s < p->passes; ++s) maxL = p->factors[s] > maxL ? p->factors[s] : maxL; \
    REAL* row = (REAL*)malloc(sizeof(REAL) * 2 * maxL);                                          \
    REAL* tmp = p->passes >= 2 ? (REAL*)malloc(sizeof(REAL) * 2 * n) : NULL;                     \
    /* ping-pong (:338-344): the last pass writes `out` */                                       \
    const REAL* src = x;                                                                         \
    for (uint32_t s = 1; s <= p->passes; ++s) {                                                  \
      REAL* dst = ((p->passes - s) % 2 == 0) ? out : tmp;                                        \
      pass_##SUF(p, s, src, dst, tbl, R, row, permute_only);                                     \
      src = dst;                                                                                 \
    }                                                                                            \
    free(row);                                                                                   \
    free(tmp);                                                                                   \
    return 0;                                                                                    \
  }                                                                                              \
  int orc_fft_tiled_##SUF(const REAL* x, REAL* out, const orc_plan* p, const REAL* tbl,          \
                          uint64_t R) {                                                          \
    return tiled_##SUF(x, out, p, tbl, R, 0);                                                    \
  }                                                                                              \
  /* tiled_fft.hpp:410-423 */                                                                    \
  int orc_ifft_tiled_##SUF(const REAL* x, REAL* out, const orc_plan* p, const REAL* tbl,         \
                           uint64_t R) {                                                         \
    const uint64_t n = p->n_total;                                                               \
    REAL* tmp = (REAL*)malloc(sizeof(REAL) * 2 * n);                                             \
    for (uint64_t i = 0; i < n; ++i) { tmp[2 * i] = x[2 * i]; tmp[2 * i + 1] = -x[2 * i + 1]; }  \
    int rc = tiled_##SUF(tmp, out, p, tbl, R, 0);                                                \
    const REAL scale = (REAL)1 / (REAL)n;                                                        \
    for (uint64_t i = 0; i < n; ++i) {                                                           \
      out[2 * i] = out[2 * i] * scale;                                                           \
      out[2 * i + 1] = -out[2 * i + 1] * scale;                                                  \
    }                                                                                            \
    free(tmp);                                                                                   \
    return rc;                                                                                   \
  }                                                                                              \
  /* fft_baseline.hpp:66-116 */                                                                  \
  int orc_fft_levelwise_##SUF(const REAL* x, REAL* w, uint64_t n, const REAL* tbl, uint64_t R) { \
    if (!is_pow2(n) || n < 2) return -1;                                                         \
    if (!(R >= n && R % n == 0)) return -1;                                                      \
    const uint32_t bits = log2_exact(n);                                                         \
    for (uint64_t i = 0; i < n; ++i) {                                                           \
      const uint64_t s = orc_bit_reverse(i, bits);                                               \
      w[2 * i] = x[2 * s]; w[2 * i + 1] = x[2 * s + 1];                                          \
    }                                                                                            \
    for (uint64_t h = 1; h < n; h <<= 1) {                                                       \
      for (uint64_t base = 0; base < n; base += 2 * h) {                                         \
        for (uint64_t j = 0; j < h; ++j) {                                                       \
          const uint64_t ti = (j & (2 * h - 1)) * (R / (2 * h));                                 \
          const REAL wr = tbl[2 * ti], wi = tbl[2 * ti + 1];                                     \
          REAL* lo = w + 2 * (base + j);                                                         \
          REAL* hi = w + 2 * (base + j + h);                                                     \
          const REAL br = hi[0], bi = hi[1];                                                     \
          const REAL tr = wr * br - wi * bi;                                                     \
          const REAL tim = wr * bi + wi * br;                                                    \
          const REAL ar = lo[0], ai = lo[1];                                                     \
          lo[0] = ar + tr; lo[1] = ai + tim;                                                     \
          hi[0] = ar - tr; hi[1] = ai - tim;                                                     \
        }                                                                                        \
      }                                                                                          \
    }                                                                                            \
    return 0;                                                                                    \
  }

ORC_DEFINE(float, f32)
ORC_DEFINE(double, f64)

int orc_permute_tiled_f32(const float* x, float* out, const orc_plan* p) {
  return tiled_f32(x, out, p, NULL, 0, 1);
}

/* reference_dft.hpp:32-60 */
int orc_dft_reference_f64(const double* x, double* out, uint64_t n, int sign, int scale) {
  if (n == 0) return -1;
  double* tc = (double*)malloc(sizeof(double) * n);
  double* ts = (double*)malloc(sizeof(double) * n);
  for (uint64_t m = 0; m < n; ++m) {
    const double angle = 2.0 * kPi * (double)m / (double)n;
    tc[m] = cos(angle);
    ts[m] = (double)sign * sin(angle);
  }
  for (uint64_t k = 0; k < n; ++k) {
    double ar = 0.0, ai = 0.0;
    for (uint64_t m = 0; m < n; ++m) {
      const uint64_t idx = (m * k) % n;
      const double xr = x[2 * m], xi = x[2 * m + 1], wr = tc[idx], wi = ts[idx];
      ar += xr * wr - xi * wi;
      ai += xr * wi + xi * wr;
    }
    if (scale) { ar /= (double)n; ai /= (double)n; }
    out[2 * k] = ar;
    out[2 * k + 1] = ai;
  }
  free(tc);
  free(ts);
  return 0;
}

/* ---- std::mt19937_64 + std::uniform_real_distribution<double>(-1,1) ------- */
typedef struct { uint64_t mt[312]; int idx; } mt64;
static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}
static uint64_t mt64_next(mt64* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      s->mt[i] = s->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
    }
    s->idx = 0;
  }
  uint64_t z = s->mt[s->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}
/* libstdc++ generate_canonical<double,53> with a 64-bit engine: one draw,
   (double)u / 2^64, clamped below 1; then a + u*(b-a). */
static double uniform_m11(mt64* s) {
  double u = (double)mt64_next(s) / 18446744073709551616.0;
  if (u >= 1.0) u = nextafter(1.0, 0.0);
  return u * 2.0 + -1.0;
}
static void fill_mt(uint64_t n, uint64_t seed, double* out) {
  mt64* s = (mt64*)malloc(sizeof(mt64));
  mt64_seed(s, seed);
  for (uint64_t i = 0; i < n; ++i) {
    out[2 * i] = uniform_m11(s);
    out[2 * i + 1] = uniform_m11(s);
  }
  free(s);
}
/* bench.hpp:128-138 */
void orc_random_bench_signal(uint64_t n, uint64_t seed, double* out) {
  fill_mt(n, seed ^ (0x9E3779B97F4A7C15ULL * n), out);
}
/* tests/test_tiled_fft.cpp:30-40 */
void orc_random_signal(uint64_t n, uint64_t seed, double* out) { fill_mt(n, seed, out); }

static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
void orc_splitmix_signal_f32(uint64_t n, uint64_t seed, float* out) {
  const uint64_t key = seed * 0xD1B54A32D192ED03ULL;
  for (uint64_t i = 0; i < 2 * n; ++i) {
    const double u = (double)(splitmix64(key + i) >> 11) * 0x1.0p-53;
    out[i] = (float)(u * 2.0 - 1.0);
  }
}

/* Exact spectrum bins of a large fp32 signal, for parity at sizes where an
 * O(N^2) DFT is out of reach ("16 sampled bins against a direct
 * fp64 O(N) sum" at 2^30). out[2b..2b+1] = sum_n x[n] * exp(sign*2*pi*i*n*k_b/N)
 * accumulated in fp64 per thread chunk; the root W^((n*k) mod N) is the
 * product of a coarse and a fine fp64 table entry (each from cos/sin of the
 * exact angle), so the error per term is a few fp64 ulps. This is the
 * definition of the DFT (reference_dft.hpp:41-60), not a transcription of
 * its loop (which is O(N^2) and fp64-input). */
#include <pthread.h>
typedef struct {
  const float* x;
  uint64_t n, begin, end, k;
  int sign, fb;
  const double* coarse;
  const double* fine;
  double re, im;
} orc_bin_job;

static void* orc_bin_worker(void* arg) {
  orc_bin_job* j = (orc_bin_job*)arg;
  const uint64_t mask = j->n - 1, fmask = (1ull << j->fb) - 1;
  double sre = 0, sim = 0;
  uint64_t e = (j->begin * j->k) & mask;
  for (uint64_t i = j->begin; i < j->end; ++i) {
    const double* c = j->coarse + 2 * (e >> j->fb);
    const double* f = j->fine + 2 * (e & fmask);
    const double wr = c[0] * f[0] - c[1] * f[1];
    const double wi = (c[0] * f[1] + c[1] * f[0]) * (double)j->sign;
    const double xr = (double)j->x[2 * i], xi = (double)j->x[2 * i + 1];
    sre += xr * wr - xi * wi;
    sim += xr * wi + xi * wr;
    e = (e + j->k) & mask;
  }
  j->re = sre;
  j->im = sim;
  return 0;
}

int orc_dft_bins_f32in(const float* x, uint64_t n, const uint64_t* bins, uint32_t nbins, int sign, uint32_t threads,
                       double* out) {
  if (!is_pow2(n) || n < 2 || threads == 0) return -1;
  const uint32_t lm = log2_exact(n);
  const int fb = (int)((lm + 1) / 2);
  const uint64_t nf = 1ull << fb, nc = n >> fb;
  double* coarse = (double*)malloc(2 * nc * sizeof(double));
  double* fine = (double*)malloc(2 * nf * sizeof(double));
  orc_bin_job* jobs = (orc_bin_job*)calloc(threads, sizeof(orc_bin_job));
  pthread_t* tid = (pthread_t*)calloc(threads, sizeof(pthread_t));
  if (!coarse || !fine || !jobs || !tid) return -1;
  for (uint64_t i = 0; i < nc; ++i) {  /* exp(+2 pi i * i*nf / n) (sign applied per term) */
    const double a = 2.0 * kPi * (double)(i * nf) / (double)n;
    coarse[2 * i] = cos(a);
    coarse[2 * i + 1] = sin(a);
  }
  for (uint64_t i = 0; i < nf; ++i) {
    const double a = 2.0 * kPi * (double)i / (double)n;
    fine[2 * i] = cos(a);
    fine[2 * i + 1] = sin(a);
  }
  for (uint32_t b = 0; b < nbins; ++b) {
    const uint64_t per = (n + threads - 1) / threads;
    for (uint32_t t = 0; t < threads; ++t) {
      orc_bin_job* j = &jobs[t];
      j->x = x;
      j->n = n;
      j->begin = (uint64_t)t * per < n ? (uint64_t)t * per : n;
      j->end = j->begin + per < n ? j->begin + per : n;
      j->k = bins[b] & (n - 1);
      j->sign = sign < 0 ? -1 : 1;
      j->fb = fb;
      j->coarse = coarse;
      j->fine = fine;
      pthread_create(&tid[t], 0, orc_bin_worker, j);
    }
    double re = 0, im = 0;
    for (uint32_t t = 0; t < threads; ++t) {
      pthread_join(tid[t], 0);
      re += jobs[t].re;
      im += jobs[t].im;
    }
    out[2 * b] = re;
    out[2 * b + 1] = im;
  }
  free(coarse);
  free(fine);
  free(jobs);
  free(tid);
  return 0;
}
