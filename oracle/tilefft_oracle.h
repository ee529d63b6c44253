/* tilefft oracle — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's CPU complex-to-complex FFT path
 * (/root/reference/proj/include/tilefft, "tilefft", arXiv 1707.07263), used as
 * the checker for the B200 product path. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. The product
 * (paper_1707_07263_b200/, include/) never links or calls it.
 *
 * Parity pinning: every function is checked against (a) the golden vectors the
 * reference's own tests hold (tests/golden/reference_fixtures.json, with
 * citations) and (b) the reference itself compiled from its headers into
 * oracle/_ref/libtilefft_ref.so (oracle/Makefile); tests/test_oracle.py does
 * both. Arithmetic follows the reference bit for bit: products rounded
 * separately (compiled with -ffp-contract=off, like the reference's default
 * x86-64 build which has no FMA), same operation order, same table values.
 */
#ifndef TILEFFT_ORACLE_H
#define TILEFFT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_PASSES 64

/* stage_plan.hpp:36-45 */
typedef struct {
  uint64_t fft_len, levels, rows, sub_len, rows_per_sub, padded_stride, rows_per_tile, tile_count;
} orc_geom;

/* stage_plan.hpp:49-69 */
typedef struct {
  uint64_t n_total, tile_capacity;
  uint32_t bank_count, passes;
  uint64_t factors[ORC_MAX_PASSES];
  orc_geom stages[ORC_MAX_PASSES];
  uint64_t sub_weights[ORC_MAX_PASSES];
  uint64_t out_weights[ORC_MAX_PASSES];
} orc_plan;

/* Return codes: 0 ok, -1 invalid argument (the reference throws
 * std::invalid_argument in the same situations). */
int orc_make_plan(uint64_t n, uint64_t tile_capacity, uint32_t bank_count, orc_plan* out);
int orc_build_twiddle_f32(uint64_t resolution, float* out /* 2*resolution */);
int orc_build_twiddle_f64(uint64_t resolution, double* out);
uint64_t orc_bit_reverse(uint64_t value, uint32_t bits);
uint64_t orc_gather_source_index(const orc_plan* p, uint32_t stage, uint64_t grow, uint64_t col);
uint64_t orc_final_output_index(const orc_plan* p, uint64_t sub, uint64_t k);
uint64_t orc_exchange_index_map(const orc_plan* p, uint32_t stage, uint64_t q);

/* fft_tiled / ifft_tiled / fft_levelwise (interleaved re,im arrays). */
int orc_fft_tiled_f32(const float* x, float* out, const orc_plan* p, const float* table, uint64_t resolution);
int orc_fft_tiled_f64(const double* x, double* out, const orc_plan* p, const double* table, uint64_t resolution);
int orc_ifft_tiled_f32(const float* x, float* out, const orc_plan* p, const float* table, uint64_t resolution);
int orc_ifft_tiled_f64(const double* x, double* out, const orc_plan* p, const double* table, uint64_t resolution);
int orc_fft_levelwise_f32(const float* x, float* out, uint64_t n, const float* table, uint64_t resolution);
int orc_fft_levelwise_f64(const double* x, double* out, uint64_t n, const double* table, uint64_t resolution);
/* Permute-only fft_tiled: the gather/scatter index maps with butterflies and
 * twiddles off (SURVEY §8c tier 3). */
int orc_permute_tiled_f32(const float* x, float* out, const orc_plan* p);

/* reference_dft.hpp:41-60, fp64 accumulation; sign -1 forward. */
int orc_dft_reference_f64(const double* x, double* out, uint64_t n, int sign, int scale);

/* bench.hpp:128-138 random_bench_signal and tests' random_signal (seeded
 * mt19937_64 + uniform_real_distribution<double>(-1,1), re then im). */
void orc_random_bench_signal(uint64_t n, uint64_t seed, double* out);
void orc_random_signal(uint64_t n, uint64_t seed, double* out);
/* Counter-based generator shared with the device: element i
 * re = u(splitmix64(seed, 2i)), im = u(splitmix64(seed, 2i+1)), u in [-1,1). */
void orc_splitmix_signal_f32(uint64_t n, uint64_t seed, float* out);

/* Exact fp64 DFT bins of an fp32 signal (sign -1 forward), `threads` POSIX
 * threads; for sampled-bin parity at 2^30. */
int orc_dft_bins_f32in(const float* x, uint64_t n, const uint64_t* bins, uint32_t nbins, int sign, uint32_t threads,
                       double* out);

#ifdef __cplusplus
}
#endif
#endif
