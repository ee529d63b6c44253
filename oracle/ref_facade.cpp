// Reference facade — TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNMODIFIED reference headers (/root/reference/proj/include,
// read-only, never copied) into oracle/_ref/libtilefft_ref.so with the
// reference's own flags (-std=c++20 -O3 -fno-tree-slp-vectorize, no -march;
// proj/CMakeLists.txt:1-30) and exposes them through plain C entry points so
// the tests can pin the oracle restatement against the real thing and bench.py
// can time the reference's CPU path (`--impl reference`, cpu_baseline).
#include <algorithm>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <thread>
#include <vector>

#include "tilefft/bench.hpp"
#include "tilefft/fft_baseline.hpp"
#include "tilefft/memsim.hpp"
#include "tilefft/reference_dft.hpp"
#include "tilefft/stage_plan.hpp"
#include "tilefft/tiled_fft.hpp"
#include "tilefft/twiddle.hpp"

namespace {
template <typename Real>
tilefft::Signal<Real> to_signal(const Real* x, std::size_t n) {
  tilefft::Signal<Real> s(n);
  std::memcpy(s.data(), x, sizeof(Real) * 2 * n);
  return s;
}
template <typename Real>
void from_signal(const tilefft::Signal<Real>& s, Real* out) {
  std::memcpy(out, s.data(), sizeof(Real) * 2 * s.size());
}

// A prepared reference call: plan + table built once, outside any timing.
struct Ctx {
  tilefft::StagePlan plan;
  tilefft::TwiddleTable<float> table;
  std::size_t n;
};
}  // namespace

extern "C" {

// stage_plan.hpp:74-127 — fills factors[] and geometry rows (8 fields each).
int ref_make_plan(uint64_t n, uint64_t cap, uint32_t* passes, uint64_t* factors, uint64_t* geom,
                  uint64_t* sub_w, uint64_t* out_w) {
  try {
    const tilefft::StagePlan p = tilefft::make_plan(n, cap);
    *passes = (uint32_t)p.pass_count();
    for (std::size_t s = 0; s < p.pass_count(); ++s) {
      factors[s] = p.factors[s];
      const auto& g = p.stages[s];
      const uint64_t row[8] = {g.fft_len, g.levels, g.rows, g.sub_len, g.rows_per_sub,
                               g.padded_stride, g.rows_per_tile, g.tile_count};
      std::memcpy(geom + 8 * s, row, sizeof row);
      out_w[s] = p.out_weights[s];
      if (s + 1 < p.pass_count()) sub_w[s] = p.sub_weights[s];
    }
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

uint64_t ref_exchange_index_map(uint64_t n, uint64_t cap, uint32_t stage, uint64_t q) {
  return tilefft::detail::exchange_index_map(tilefft::make_plan(n, cap), stage, q);
}
uint64_t ref_gather_source_index(uint64_t n, uint64_t cap, uint32_t stage, uint64_t grow, uint64_t col) {
  return tilefft::detail::gather_source_index(tilefft::make_plan(n, cap).stage(stage), grow, col);
}

int ref_build_twiddle_f32(uint64_t r, float* out) {
  try { from_signal(tilefft::build_twiddle_table<float>(r).values, out); return 0; }
  catch (const std::invalid_argument&) { return -1; }
}
int ref_build_twiddle_f64(uint64_t r, double* out) {
  try { from_signal(tilefft::build_twiddle_table<double>(r).values, out); return 0; }
  catch (const std::invalid_argument&) { return -1; }
}

#define REF_TILED(REAL, SUF)                                                                   \
  int ref_fft_tiled_##SUF(const REAL* x, REAL* out, uint64_t n, uint64_t cap, uint64_t res,    \
                          uint32_t threads) {                                                  \
    try {                                                                                      \
      const auto plan = tilefft::make_plan(n, cap);                                            \
      const auto table = tilefft::build_twiddle_table<REAL>(res);                              \
      from_signal(tilefft::fft_tiled(to_signal(x, n), plan, table, nullptr, threads), out);    \
      return 0;                                                                                \
    } catch (const std::invalid_argument&) { return -1; }                                      \
  }                                                                                            \
  int ref_ifft_tiled_##SUF(const REAL* x, REAL* out, uint64_t n, uint64_t cap, uint64_t res) { \
    try {                                                                                      \
      const auto plan = tilefft::make_plan(n, cap);                                            \
      const auto table = tilefft::build_twiddle_table<REAL>(res);                              \
      from_signal(tilefft::ifft_tiled(to_signal(x, n), plan, table), out);                     \
      return 0;                                                                                \
    } catch (const std::invalid_argument&) { return -1; }                                      \
  }                                                                                            \
  int ref_fft_levelwise_##SUF(const REAL* x, REAL* out, uint64_t n, uint64_t res) {            \
    try {                                                                                      \
      const auto table = tilefft::build_twiddle_table<REAL>(res);                              \
      from_signal(tilefft::fft_levelwise(to_signal(x, n), table), out);                        \
      return 0;                                                                                \
    } catch (const std::invalid_argument&) { return -1; }                                      \
  }                                                                                            \
  int ref_dft_reference_##SUF(const REAL* x, REAL* out, uint64_t n) {                          \
    try { from_signal(tilefft::dft_reference(to_signal(x, n)), out); return 0; }               \
    catch (const std::invalid_argument&) { return -1; }                                       \
  }
REF_TILED(float, f32)
REF_TILED(double, f64)

// exchange_transpose (tiled_fft.hpp:179-203) on a real ramp-style signal.
int ref_exchange_transpose_f64(const double* x, double* out, uint64_t n, uint64_t cap, uint32_t stage) {
  try {
    from_signal(tilefft::exchange_transpose(to_signal(x, n), stage, tilefft::make_plan(n, cap)), out);
    return 0;
  } catch (const std::invalid_argument&) { return -1; }
}

// bench.hpp:128-138
void ref_random_bench_signal(uint64_t n, uint64_t seed, double* out) {
  from_signal(tilefft::detail::random_bench_signal(n, seed), out);
}

// ---- timed CPU baseline: plan + table prepared once ------------------------
void* ref_ctx_create(uint64_t n, uint64_t cap) {
  try {
    auto* c = new Ctx{tilefft::make_plan(n, cap), tilefft::build_twiddle_table<float>(n), n};
    return c;
  } catch (...) { return nullptr; }
}
void ref_ctx_destroy(void* c) { delete static_cast<Ctx*>(c); }

// One single-transform call with the reference's own thread split
// (fft_tiled(..., threads)).
int ref_ctx_exec_single(void* vc, const float* x, float* out, uint32_t threads) {
  auto* c = static_cast<Ctx*>(vc);
  from_signal(tilefft::fft_tiled(to_signal(x, c->n), c->plan, c->table, nullptr, threads), out);
  return 0;
}

// Batched: `threads` std::threads, each calling fft_tiled(threads=1) over a
// strided subset of the rows (the BASELINE.md §2 batched/2D recipe).
int ref_ctx_exec_batched(void* vc, const float* x, float* out, uint64_t batch, uint32_t threads) {
  auto* c = static_cast<Ctx*>(vc);
  const std::size_t n = c->n;
  threads = std::max<uint32_t>(1, std::min<uint64_t>(threads, batch));
  std::vector<std::thread> pool;
  for (uint32_t t = 0; t < threads; ++t) {
    pool.emplace_back([=] {
      tilefft::Signal<float> row(n);
      for (uint64_t b = t; b < batch; b += threads) {
        std::memcpy(row.data(), x + 2 * n * b, sizeof(float) * 2 * n);
        const auto y = tilefft::fft_tiled(row, c->plan, c->table, nullptr, 1);
        std::memcpy(out + 2 * n * b, y.data(), sizeof(float) * 2 * n);
      }
    });
  }
  for (auto& th : pool) th.join();
  return 0;
}

uint32_t ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// memsim.hpp:58-95 / :38-55: the reference's closed-form accounting, seven
// counters in AccessStats order (cost-model parity, tests/test_costmodel.py).
static void put_stats(const tilefft::AccessStats& s, uint64_t* out) {
  const uint64_t v[7] = {s.slow_elem_reads, s.slow_elem_writes, s.slow_transactions, s.fast_accesses,
                         s.bank_conflict_cycles, s.barriers, s.twiddle_fetches};
  std::memcpy(out, v, sizeof v);
}
int ref_account_tiled(uint64_t n, uint64_t cap, uint64_t* out) {
  try {
    put_stats(tilefft::account_tiled(tilefft::make_plan(n, cap)), out);
    return 0;
  } catch (const std::invalid_argument&) { return -1; }
}
int ref_account_levelwise(uint64_t n, uint64_t* out) {
  try {
    put_stats(tilefft::account_levelwise(n), out);
    return 0;
  } catch (const std::invalid_argument&) { return -1; }
}
}
