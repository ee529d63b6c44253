// tilefft (B200) — drop-in for /root/reference/proj/include/tilefft/fft_baseline.hpp.
// butterfly / bit_reverse_permutation are the same host helpers; fft_levelwise
// (the paper's "previous method", fft_baseline.hpp:66-116) runs on the GPU as
// one bit-reversal launch plus one launch per radix-2 level
// (TILEFFT_MODE_LEVELWISE), bit-identical to the reference.
#pragma once

#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

#include "tilefft/access_patterns.hpp"
#include "tilefft/b200_runtime.hpp"
#include "tilefft/common.hpp"
#include "tilefft/exec_model.hpp"
#include "tilefft/twiddle.hpp"

namespace tilefft {
inline namespace b200 {

template <typename Real>
std::pair<Complex<Real>, Complex<Real>> butterfly(const Complex<Real>& a, const Complex<Real>& b,
                                                  const Complex<Real>& w) {
  const Complex<Real> t = w * b;
  return {a + t, a - t};
}

inline std::vector<std::size_t> bit_reverse_permutation(std::size_t n) {
  detail::require(is_power_of_two(n), "bit_reverse_permutation: n must be a power of two");
  const unsigned bits = log2_exact(n);
  std::vector<std::size_t> perm(n);
  for (std::size_t i = 0; i < n; ++i) perm[i] = static_cast<std::size_t>(detail::bit_reverse(i, bits));
  return perm;
}

namespace detail {
template <typename Real>
inline Complex<Real> twiddle_fetch(const TwiddleTable<Real>& table, std::uint64_t n, std::uint64_t e) {
  return table.values[(e & (n - 1)) * (table.resolution / n)];
}

template <typename Real>
Signal<Real> run_levelwise(const Signal<Real>& x, const TwiddleTable<Real>& table, int sign) {
  const std::size_t n = x.size();
  detail::require(is_power_of_two(n) && n >= 2, "fft_levelwise: signal length must be a power of two >= 2");
  detail::require(table.resolution >= n && table.resolution % n == 0,
                  "fft_levelwise: signal length must divide the table resolution");
  const auto p = runtime::device_plan(n, 1, {}, sizeof(Complex<Real>), TILEFFT_MODE_LEVELWISE,
                                          table.values.data(), table.resolution);
  Signal<Real> out(n);
  runtime::check(tilefft_exec_c2c_host(p.get(), x.data(), out.data(), sign));
  return out;
}
}  // namespace detail

template <typename Real>
Signal<Real> fft_levelwise(const Signal<Real>& x, const TwiddleTable<Real>& table, AccessRecorder* trace = nullptr) {
  Signal<Real> out = detail::run_levelwise(x, table, TILEFFT_FORWARD);
  if (trace != nullptr) {  // fft_baseline.hpp:80-113: the reorder sweep, then one stage per level
    const std::uint64_t n = x.size();
    const auto slow = [&](std::span<const std::uint64_t> a, bool) { trace->record_slow_request(a); };
    trace->begin_reorder();
    trace->add_slow_reads(n);
    trace->add_slow_writes(n);
    detail::for_each_reorder_request(n, trace->config(), slow);
    trace->add_barrier();
    for (unsigned lv = 1; lv <= log2_exact(n); ++lv) {
      trace->begin_stage();
      trace->add_slow_reads(n);
      trace->add_slow_writes(n);
      trace->add_twiddle_fetches(n / 2);
      detail::for_each_levelwise_request(n, lv, trace->config(), slow);
      trace->add_barrier();
    }
  }
  return out;
}

template <typename Real>
Signal<Real> ifft_levelwise(const Signal<Real>& x, const TwiddleTable<Real>& table) {
  return detail::run_levelwise(x, table, TILEFFT_INVERSE);
}

}  // namespace b200
}  // namespace tilefft
