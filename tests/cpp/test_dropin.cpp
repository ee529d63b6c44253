// C++ drop-in API tests: the reference's own test cases (tests/test_*.cpp in
// /root/reference/proj) re-run against include/tilefft/*.hpp, i.e. through the
// C ABI on the B200. The oracle (oracle/tilefft_oracle.c, test
// infrastructure) provides the expected values. Minimal self-made runner
// (Catch2 is not available in this image). Exit code = number of failures.
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "tilefft/tilefft.hpp"
#include "tilefft_oracle.h"

namespace {

int g_fail = 0, g_checks = 0;
std::string g_case;
#define CHECK(cond)                                                                           \
  do {                                                                                        \
    ++g_checks;                                                                               \
    if (!(cond)) {                                                                            \
      ++g_fail;                                                                               \
      std::printf("FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond);       \
    }                                                                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, T)      \
  do {                                \
    bool thrown_ = false;             \
    try {                             \
      (void)(expr);                   \
    } catch (const T&) {              \
      thrown_ = true;                 \
    } catch (...) {                   \
    }                                 \
    CHECK(thrown_ && #expr);          \
  } while (0)

void run(const char* name, const std::function<void()>& f) {
  g_case = name;
  try {
    f();
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("FAIL [%s] exception: %s\n", name, e.what());
  }
}

using tilefft::Complex;
using tilefft::Signal;

template <typename Real = double>
Signal<Real> random_signal(std::size_t n, std::uint64_t seed) {
  std::vector<double> buf(2 * n);
  orc_random_signal(n, seed, buf.data());
  Signal<Real> x(n);
  for (std::size_t i = 0; i < n; ++i) x[i] = {static_cast<Real>(buf[2 * i]), static_cast<Real>(buf[2 * i + 1])};
  return x;
}

template <typename Real>
Signal<Real> oracle_fft(const Signal<Real>& x, std::size_t cap, bool inverse = false) {
  orc_plan p;
  orc_make_plan(x.size(), cap, 16, &p);
  std::vector<Real> tbl(2 * x.size());
  Signal<Real> out(x.size());
  if constexpr (sizeof(Real) == 4) {
    orc_build_twiddle_f32(x.size(), tbl.data());
    (inverse ? orc_ifft_tiled_f32 : orc_fft_tiled_f32)((const float*)x.data(), (float*)out.data(), &p, tbl.data(),
                                                       x.size());
  } else {
    orc_build_twiddle_f64(x.size(), tbl.data());
    (inverse ? orc_ifft_tiled_f64 : orc_fft_tiled_f64)((const double*)x.data(), (double*)out.data(), &p, tbl.data(),
                                                       x.size());
  }
  return out;
}

Signal<double> dft(const Signal<double>& x) {
  Signal<double> out(x.size());
  orc_dft_reference_f64((const double*)x.data(), (double*)out.data(), x.size(), -1, 0);
  return out;
}

template <typename Real>
double max_abs_error(const Signal<Real>& a, const Signal<Real>& b) {
  double w = 0;
  for (std::size_t i = 0; i < a.size(); ++i)
    w = std::max(w, std::abs(std::complex<double>(a[i].real() - (double)b[i].real(), a[i].imag() - (double)b[i].imag())));
  return w;
}

template <typename Real>
bool bit_equal(const Signal<Real>& a, const Signal<Real>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(Complex<Real>)) == 0;
}

}  // namespace

int main() {
  using namespace tilefft;

  run("make_plan: reference cases (test_stage_plan.cpp:26-107)", [] {
    const StagePlan p = make_plan(65536, 1024);
    CHECK((p.factors == std::vector<std::size_t>{256, 256}));
    CHECK(p.stage(1).rows_per_tile == 4 && p.stage(1).tile_count == 64 && p.stage(1).padded_stride == 257);
    const StagePlan p3 = make_plan(64, 4);
    CHECK((p3.sub_weights == std::vector<std::size_t>{4, 1}));
    CHECK((p3.out_weights == std::vector<std::size_t>{1, 4, 16}));
    CHECK_THROWS_AS(make_plan(48), std::invalid_argument);
    CHECK_THROWS_AS(make_plan(1024, 100), std::invalid_argument);
    CHECK_THROWS_AS(p3.stage(0), std::invalid_argument);
  });

  run("exchange map (test_stage_plan.cpp:157-180)", [] {
    const StagePlan p = make_plan(16, 4);
    const std::vector<std::size_t> want = {0, 4, 8, 12, 1, 5, 9, 13, 2, 6, 10, 14, 3, 7, 11, 15};
    for (std::size_t q = 0; q < 16; ++q) CHECK(detail::exchange_index_map(p, 1, q) == want[q]);
    const StagePlan p8 = make_plan(8, 4);
    const std::vector<std::size_t> want8 = {0, 4, 1, 5, 2, 6, 3, 7};
    for (std::size_t q = 0; q < 8; ++q) CHECK(detail::exchange_index_map(p8, 2, q) == want8[q]);
  });

  run("FastBuffer layout and bounds (test_tiled_fft.cpp:52-67)", [] {
    FastBuffer<double> buf(4, 8, 9, 64, 12);
    CHECK(buf.rows() == 4 && buf.cols() == 8 && buf.stride() == 9 && buf.capacity() == 64 && buf.row_offset() == 12);
    buf.at(3, 7) = {1.0, -1.0};
    CHECK((buf.at(3, 7) == Complex<double>{1.0, -1.0}));
    CHECK_THROWS_AS(FastBuffer<double>(0, 8, 8, 64), std::invalid_argument);
    CHECK_THROWS_AS(FastBuffer<double>(4, 8, 7, 64), std::invalid_argument);
    CHECK_THROWS_AS(FastBuffer<double>(9, 8, 8, 64), std::invalid_argument);
    const auto sb = make_stage_buffer<double>(make_plan(65536, 1024), 1);
    CHECK(sb.rows() == 4 && sb.cols() == 256 && sb.stride() == 257);
  });

  run("stage_row_fft transforms each row (test_tiled_fft.cpp:79-100)", [] {
    const auto table = build_twiddle_table<double>(64);
    FastBuffer<double> buf(2, 8, 9, 16);
    const auto r0 = random_signal(8, 21), r1 = random_signal(8, 22);
    for (std::size_t c = 0; c < 8; ++c) {
      buf.at(0, c) = r0[c];
      buf.at(1, c) = r1[c];
    }
    stage_row_fft(buf, 8, table);
    Signal<double> g0(8), g1(8);
    for (std::size_t c = 0; c < 8; ++c) {
      g0[c] = buf.at(0, c);
      g1[c] = buf.at(1, c);
    }
    CHECK(max_abs_error(g0, dft(r0)) < 1e-12);
    CHECK(max_abs_error(g1, dft(r1)) < 1e-12);
    FastBuffer<double> small(1, 8, 8, 8);
    CHECK_THROWS_AS(stage_row_fft(small, 16, table), std::invalid_argument);
    CHECK_THROWS_AS(stage_row_fft(small, 8, build_twiddle_table<double>(4)), std::invalid_argument);
  });

  run("apply_interstage_twiddles: -i at (1,1) (test_tiled_fft.cpp:112-134)", [] {
    const auto table = build_twiddle_table<double>(16);
    const StagePlan plan = make_plan(4, 2);
    auto buf = make_stage_buffer<double>(plan, 1);
    buf.set_row_offset(1);
    buf.at(0, 0) = {1.0, 0.0};
    buf.at(0, 1) = {1.0, 0.0};
    apply_interstage_twiddles(buf, 1, plan, table);
    CHECK((buf.at(0, 0) == Complex<double>{1.0, 0.0}));
    CHECK((buf.at(0, 1) == Complex<double>{0.0, -1.0}));
    CHECK_THROWS_AS(apply_interstage_twiddles(buf, 2, plan, table), std::invalid_argument);
  });

  run("exchange_transpose (test_tiled_fft.cpp:156-175)", [] {
    Signal<double> ramp(16);
    for (std::size_t i = 0; i < 16; ++i) ramp[i] = {double(i), 0};
    const auto out = exchange_transpose(ramp, 1, make_plan(16, 4));
    for (std::size_t r = 0; r < 4; ++r)
      for (std::size_t k = 0; k < 4; ++k) CHECK(out[k * 4 + r] == ramp[r * 4 + k]);
    Signal<double> r8(8);
    for (std::size_t i = 0; i < 8; ++i) r8[i] = {double(i), 0};
    const auto o8 = exchange_transpose(r8, 2, make_plan(8, 4));
    const double want[] = {0, 2, 4, 6, 1, 3, 5, 7};
    for (std::size_t i = 0; i < 8; ++i) CHECK(o8[i].real() == want[i]);
    CHECK_THROWS_AS(exchange_transpose(r8, 3, make_plan(8, 4)), std::invalid_argument);
  });

  run("fft_tiled agrees with the quadratic reference (test_tiled_fft.cpp:208-224)", [] {
    const auto table = build_twiddle_table<double>(1024);
    const std::size_t cases[][2] = {{2, 1024}, {4, 2},    {8, 4},    {16, 4},   {32, 2},   {64, 4},
                                    {64, 8},   {256, 16}, {512, 8},  {1024, 4}, {1024, 32}, {1024, 1024}};
    for (const auto& c : cases) {
      const auto x = random_signal(c[0], 900 + c[0] + c[1]);
      const StagePlan plan = make_plan(c[0], c[1]);
      CHECK(max_abs_error(fft_tiled(x, plan, table), dft(x)) < 1e-9 * double(c[0]));
    }
  });

  run("fft_tiled fast tier vs reference fft_tiled (fp32, north-star tolerance)", [] {
    for (std::size_t n : {1024ul, 8192ul, 1ul << 16, 1ul << 20}) {
      const auto x = random_signal<float>(n, 7);
      const auto table = build_twiddle_table<float>(n);
      const auto got = fft_tiled(x, make_plan(n), table);
      const auto want = oracle_fft(x, 1024);
      double num = 0, den = 0;
      for (std::size_t i = 0; i < n; ++i) {
        num += std::norm(std::complex<double>(got[i]) - std::complex<double>(want[i]));
        den += std::norm(std::complex<double>(want[i]));
      }
      CHECK(std::sqrt(num / den) <= 1e-5 * std::log2(double(n)));
    }
  });

  run("exact tier: bit-identical to the reference (fp32 + fp64)", [] {
    set_exec_mode(ExecMode::exact);
    for (auto [n, cap] : std::vector<std::pair<std::size_t, std::size_t>>{{256, 16}, {4096, 64}, {1 << 16, 1024}}) {
      const auto x = random_signal<float>(n, 3);
      CHECK(bit_equal(fft_tiled(x, make_plan(n, cap), build_twiddle_table<float>(n)), oracle_fft(x, cap)));
      CHECK(bit_equal(ifft_tiled(x, make_plan(n, cap), build_twiddle_table<float>(n)), oracle_fft(x, cap, true)));
      const auto xd = random_signal<double>(n, 4);
      CHECK(bit_equal(fft_tiled(xd, make_plan(n, cap), build_twiddle_table<double>(n)), oracle_fft(xd, cap)));
    }
    set_exec_mode(ExecMode::fast);
  });

  run("fft_tiled: single pass reproduces the baseline bit for bit (test_tiled_fft.cpp:226-234)", [] {
    set_exec_mode(ExecMode::exact);
    const auto table = build_twiddle_table<double>(256);
    const auto x = random_signal(256, 41);
    CHECK(bit_equal(fft_tiled(x, make_plan(256, 1024), table), fft_levelwise(x, table)));
    set_exec_mode(ExecMode::fast);
  });

  run("fft_levelwise: exact N=2 and large-N levelwise kernels", [] {
    const auto table = build_twiddle_table<double>(16);
    const Signal<double> x = {{1.5, -0.5}, {0.25, 2.0}};
    const auto s = fft_levelwise(x, table);
    CHECK((s[0] == Complex<double>{1.75, 1.5}));
    CHECK((s[1] == Complex<double>{1.25, -2.5}));
    const std::size_t n = 1 << 18;
    const auto y = random_signal<float>(n, 5);
    std::vector<float> tbl(2 * n);
    orc_build_twiddle_f32(n, tbl.data());
    Signal<float> want(n);
    orc_fft_levelwise_f32((const float*)y.data(), (float*)want.data(), n, tbl.data(), n);
    CHECK(bit_equal(fft_levelwise(y, build_twiddle_table<float>(n)), want));
    const auto back = ifft_levelwise(fft_levelwise(y, build_twiddle_table<float>(n)), build_twiddle_table<float>(n));
    CHECK(max_abs_error(back, y) < 1e-5);
  });

  run("worker count never changes the answer (test_tiled_fft.cpp:236-253)", [] {
    const auto table = build_twiddle_table<double>(4096);
    const auto x = random_signal(4096, 42);
    const StagePlan plan = make_plan(4096, 64);
    AccessRecorder bt;
    const auto base = fft_tiled(x, plan, table, &bt, 1);
    for (unsigned t : {2u, 3u, 8u}) {
      AccessRecorder tr;
      CHECK(bit_equal(fft_tiled(x, plan, table, &tr, t), base));
      CHECK(tr.totals() == bt.totals());
    }
  });

  run("trace: one slow-memory round trip per pass (test_tiled_fft.cpp:255-271)", [] {
    const auto table = build_twiddle_table<double>(4096);
    AccessRecorder trace;
    fft_tiled(random_signal(4096, 43), make_plan(4096, 64), table, &trace);
    CHECK(trace.stage_count() == 2);
    for (std::size_t s = 1; s <= 2; ++s) {
      CHECK(trace.stage(s).slow_elem_reads == 4096);
      CHECK(trace.stage(s).slow_elem_writes == 4096);
      CHECK(trace.stage(s).barriers == 1);
    }
    CHECK(trace.totals().slow_elem_accesses() == 2 * 4096 * 2);
    CHECK(trace.reorder() == AccessStats{});
  });

  run("ifft_tiled inverts fft_tiled (test_tiled_fft.cpp:273-279)", [] {
    const auto table = build_twiddle_table<double>(256);
    const auto x = random_signal(256, 44);
    const StagePlan plan = make_plan(256, 16);
    CHECK(max_abs_error(ifft_tiled(fft_tiled(x, plan, table), plan, table), x) < 1e-12);
  });

  run("fft_tiled rejects mismatched inputs (test_tiled_fft.cpp:281-295)", [] {
    const auto table = build_twiddle_table<double>(256);
    const StagePlan plan = make_plan(256, 16);
    CHECK_THROWS_AS(fft_tiled(random_signal(128, 1), plan, table), std::invalid_argument);
    CHECK_THROWS_AS(fft_tiled(random_signal(256, 1), plan, build_twiddle_table<double>(64)), std::invalid_argument);
    ExecConfig other;
    other.bank_count = 32;
    AccessRecorder trace(other);
    CHECK_THROWS_AS(fft_tiled(random_signal(256, 1), plan, table, &trace), std::invalid_argument);
  });

  run("single-precision instantiation (test_tiled_fft.cpp:297-311)", [] {
    const auto table = build_twiddle_table<float>(256);
    std::mt19937_64 rng(45);
    std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
    Signal<float> x(256);
    for (auto& v : x) {
      const float re = dist(rng), im = dist(rng);
      v = {re, im};
    }
    const auto fast = fft_tiled(x, make_plan(256, 16), table);
    Signal<double> xd(256);
    for (std::size_t i = 0; i < 256; ++i) xd[i] = {x[i].real(), x[i].imag()};
    const auto slow = dft(xd);
    double w = 0;
    for (std::size_t i = 0; i < 256; ++i) w = std::max(w, std::abs(std::complex<double>(fast[i]) - slow[i]));
    CHECK(w < 1e-3);
  });

  run("criteria 4 and 7: traced GPU runs equal the closed-form accounting (acceptance_main.cpp:158-195)", [] {
    const auto table = build_twiddle_table<double>(65536);
    const std::size_t cases[][2] = {{2, 1024},     {16, 4},      {16, 1024},  {256, 16},   {256, 1024},
                                    {4096, 64},    {4096, 1024}, {16384, 1024}, {65536, 1024}};
    for (const auto& c : cases) {
      const auto x = random_signal(c[0], 0x4A55 + c[0]);
      AccessRecorder lt;
      (void)fft_levelwise(x, table, &lt);
      const unsigned bits = log2_exact(c[0]);
      CHECK(lt.totals() == account_levelwise(c[0]));
      CHECK(lt.totals().slow_elem_accesses() == 2 * c[0] * bits && lt.totals().barriers == bits);
      CHECK(lt.reorder().slow_transactions > 0 && lt.reorder().barriers == 1);
      const StagePlan plan = make_plan(c[0], c[1]);
      AccessRecorder tt;
      (void)fft_tiled(x, plan, table, &tt);
      CHECK(tt.totals() == account_tiled(plan));
      CHECK(tt.stage_count() == plan.pass_count() && tt.totals().barriers == plan.pass_count());
      CHECK(tt.totals().slow_elem_accesses() == 2 * c[0] * plan.pass_count());
      CHECK(tt.totals().slow_transactions > 0);
    }
    CHECK(reduction_ratio(4096, make_plan(4096)) == 6.0 && reduction_ratio(65536, make_plan(65536)) == 8.0);
  });

  run("exchange_transpose records one full sweep (test_tiled_fft.cpp:187-198)", [] {
    AccessRecorder trace;
    (void)exchange_transpose(random_signal(256, 32), 1, make_plan(256, 16), &trace);
    CHECK(trace.stage_count() == 1);
    CHECK(trace.stage(1).slow_elem_reads == 256 && trace.stage(1).slow_elem_writes == 256);
    CHECK(trace.stage(1).barriers == 1 && trace.stage(1).slow_transactions > 0);
  });

  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail;
}
