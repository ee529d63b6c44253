// tilefft (B200) — drop-in for /root/reference/proj/include/tilefft/tiled_fft.hpp.
//
// Same signatures; the transforms run on the B200 through the C ABI:
//   fft_tiled   (tiled_fft.hpp:321-407) -> tilefft_exec_c2c_host, forward
//   ifft_tiled  (:410-423)              -> tilefft_exec_c2c_host, inverse (1/n)
//   stage_row_fft (:129-146)            -> exact single-pass plan over the tile rows
//   apply_interstage_twiddles (:153-172)-> tilefft_interstage_scale
//   exchange_transpose (:179-203)       -> tilefft_exchange
// FastBuffer / make_stage_buffer (:38-80) are the same host data structure.
// `threads` keeps its meaning for callers and never changes the result (the
// reference guarantees thread invariance, test_tiled_fft.cpp:236-253).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

#include "tilefft/access_patterns.hpp"
#include "tilefft/b200_runtime.hpp"
#include "tilefft/common.hpp"
#include "tilefft/exec_model.hpp"
#include "tilefft/fft_baseline.hpp"
#include "tilefft/stage_plan.hpp"
#include "tilefft/twiddle.hpp"

namespace tilefft {
inline namespace b200 {

template <typename Real>
class FastBuffer {
 public:
  FastBuffer(std::size_t rows, std::size_t cols, std::size_t stride, std::size_t capacity, std::size_t row_offset = 0)
      : rows_(rows), cols_(cols), stride_(stride), capacity_(capacity), row_offset_(row_offset), cells_(rows * stride) {
    detail::require(rows >= 1 && cols >= 1, "FastBuffer: empty tile");
    detail::require(stride >= cols, "FastBuffer: stride narrower than a row");
    detail::require(rows * cols <= capacity, "FastBuffer: tile exceeds capacity");
  }
  std::size_t rows() const noexcept { return rows_; }
  std::size_t cols() const noexcept { return cols_; }
  std::size_t stride() const noexcept { return stride_; }
  std::size_t capacity() const noexcept { return capacity_; }
  std::size_t row_offset() const noexcept { return row_offset_; }
  void set_row_offset(std::size_t offset) noexcept { row_offset_ = offset; }
  Complex<Real>& at(std::size_t r, std::size_t c) noexcept { return cells_[r * stride_ + c]; }
  const Complex<Real>& at(std::size_t r, std::size_t c) const noexcept { return cells_[r * stride_ + c]; }

 private:
  std::size_t rows_, cols_, stride_, capacity_, row_offset_;
  std::vector<Complex<Real>> cells_;
};

template <typename Real = double>
FastBuffer<Real> make_stage_buffer(const StagePlan& plan, std::size_t stage) {
  const StageGeometry& g = plan.stage(stage);
  return FastBuffer<Real>(g.rows_per_tile, g.fft_len, g.padded_stride, plan.tile_capacity);
}

namespace detail {

template <typename Real>
std::vector<Complex<Real>> pack_rows(const FastBuffer<Real>& buf) {
  std::vector<Complex<Real>> t(buf.rows() * buf.cols());
  for (std::size_t r = 0; r < buf.rows(); ++r)
    for (std::size_t c = 0; c < buf.cols(); ++c) t[r * buf.cols() + c] = buf.at(r, c);
  return t;
}
template <typename Real>
void unpack_rows(FastBuffer<Real>& buf, const std::vector<Complex<Real>>& t) {
  for (std::size_t r = 0; r < buf.rows(); ++r)
    for (std::size_t c = 0; c < buf.cols(); ++c) buf.at(r, c) = t[r * buf.cols() + c];
}

// The per-pass trace fft_tiled records (tiled_fft.hpp:382-402): every pass
// reads and writes all n elements once, in-tile accesses and root fetches per
// the pass's tile shape, the gather and scatter sweeps' warp requests
// (coalesced into segments) and the tile's half-warp column streams (bank
// conflicts), one barrier. The GPU executes exactly these passes' element
// movement; the request shapes are the reference's model of them.
inline void record_trace(const StagePlan& plan, AccessRecorder& trace) {
  const auto slow = [&](std::span<const std::uint64_t> a, bool) { trace.record_slow_request(a); };
  for (std::size_t s = 1; s <= plan.pass_count(); ++s) {
    const StageGeometry& g = plan.stage(s);
    const std::uint64_t n = plan.n_total, occasions = column_stream_occasions(plan, s);
    trace.begin_stage();
    trace.add_slow_reads(n);
    trace.add_slow_writes(n);
    trace.add_fast_accesses(n * occasions);
    trace.add_twiddle_fetches(stage_twiddle_fetches(plan, s));
    for_each_tiled_sweep_request(plan, s, /*gather=*/true, trace.config(), slow);
    for_each_tiled_sweep_request(plan, s, /*gather=*/false, trace.config(), slow);
    for_each_column_stream(g.rows, g.fft_len, g.padded_stride, trace.config(),
                           [&](std::span<const std::uint64_t> w) { trace.record_fast_request_repeated(w, occasions); });
    trace.add_barrier();
  }
}

template <typename Real>
Signal<Real> run_tiled(const Signal<Real>& x, const StagePlan& plan, const TwiddleTable<Real>& table, int sign) {
  const ExecMode mode = exec_mode();
  const std::vector<std::uint64_t> f(plan.factors.begin(), plan.factors.end());
  const auto p = runtime::device_plan(plan.n_total, 1, f, sizeof(Complex<Real>), static_cast<unsigned>(mode),
                                          mode == ExecMode::exact ? static_cast<const void*>(table.values.data()) : nullptr,
                                          mode == ExecMode::exact ? table.resolution : 0);
  Signal<Real> out(x.size());
  runtime::check(tilefft_exec_c2c_host(p.get(), x.data(), out.data(), sign));
  return out;
}

}  // namespace detail

template <typename Real>
void stage_row_fft(FastBuffer<Real>& buf, std::size_t length, const TwiddleTable<Real>& table) {
  detail::require(is_power_of_two(length), "stage_row_fft: length must be a power of two");
  detail::require(length <= buf.capacity(), "stage_row_fft: length exceeds tile capacity");
  detail::require(length == buf.cols(), "stage_row_fft: length must match the tile row width");
  detail::require(table.resolution >= length && table.resolution % length == 0,
                  "stage_row_fft: length must divide the table resolution");
  if (length < 2) return;
  std::vector<Complex<Real>> t = detail::pack_rows(buf);
  const auto p = runtime::device_plan(length, buf.rows(), {length}, sizeof(Complex<Real>), TILEFFT_MODE_EXACT,
                                          table.values.data(), table.resolution);
  runtime::check(tilefft_exec_c2c_host(p.get(), t.data(), t.data(), TILEFFT_FORWARD));
  detail::unpack_rows(buf, t);
}

template <typename Real>
void apply_interstage_twiddles(FastBuffer<Real>& buf, std::size_t stage, const StagePlan& plan,
                               const TwiddleTable<Real>& table) {
  detail::require(plan.pass_count() >= 1, "apply_interstage_twiddles: empty plan");
  detail::require(stage >= 1 && stage < plan.pass_count(),
                  "apply_interstage_twiddles: stage must be an inter-pass boundary");
  const StageGeometry& g = plan.stage(stage);
  detail::require(buf.cols() == g.fft_len, "apply_interstage_twiddles: tile width does not match the pass");
  detail::require(buf.row_offset() + buf.rows() <= g.rows,
                  "apply_interstage_twiddles: tile rows fall outside the pass grid");
  detail::require(table.resolution >= g.sub_len && table.resolution % g.sub_len == 0,
                  "apply_interstage_twiddles: sub-transform length must divide the table resolution");
  std::vector<Complex<Real>> t = detail::pack_rows(buf);
  runtime::check(tilefft_interstage_scale(t.data(), t.data(), buf.rows(), buf.cols(), buf.row_offset(), g.rows_per_sub,
                                          g.sub_len, table.values.data(), table.resolution, sizeof(Complex<Real>),
                                          runtime::state().device));
  detail::unpack_rows(buf, t);
}

template <typename Real>
Signal<Real> exchange_transpose(const Signal<Real>& data, std::size_t stage, const StagePlan& plan,
                                AccessRecorder* trace = nullptr) {
  detail::require(stage >= 1 && stage <= plan.pass_count(), "exchange_transpose: stage out of range");
  detail::require(data.size() == plan.n_total, "exchange_transpose: signal length does not match the plan");
  if (plan.pass_count() == 1) return data;
  Signal<Real> out(data.size());
  const std::vector<std::uint64_t> f(plan.factors.begin(), plan.factors.end());
  runtime::check(tilefft_exchange(data.data(), out.data(), plan.n_total, f.data(), static_cast<std::uint32_t>(f.size()),
                                  static_cast<std::uint32_t>(stage), sizeof(Complex<Real>), runtime::state().device));
  if (trace != nullptr) {
    trace->begin_stage();
    trace->add_slow_reads(data.size());
    trace->add_slow_writes(data.size());
    detail::for_each_exchange_request(plan, stage, trace->config(),
                                      [&](std::span<const std::uint64_t> a, bool) { trace->record_slow_request(a); });
    trace->add_barrier();
  }
  return out;
}

template <typename Real>
Signal<Real> fft_tiled(const Signal<Real>& x, const StagePlan& plan, const TwiddleTable<Real>& table,
                       AccessRecorder* trace = nullptr, unsigned threads = 1) {
  (void)threads;
  detail::require(x.size() == plan.n_total, "fft_tiled: signal length does not match the plan");
  detail::require(plan.pass_count() >= 1, "fft_tiled: empty plan");
  detail::require(table.resolution >= plan.n_total && table.resolution % plan.n_total == 0,
                  "fft_tiled: signal length must divide the table resolution");
  if (trace != nullptr)
    detail::require(trace->config().bank_count == plan.bank_count, "fft_tiled: plan was built for a different bank count");
  Signal<Real> out = detail::run_tiled(x, plan, table, TILEFFT_FORWARD);
  if (trace != nullptr) detail::record_trace(plan, *trace);
  return out;
}

template <typename Real>
Signal<Real> ifft_tiled(const Signal<Real>& x, const StagePlan& plan, const TwiddleTable<Real>& table) {
  detail::require(x.size() == plan.n_total, "fft_tiled: signal length does not match the plan");
  detail::require(plan.pass_count() >= 1, "fft_tiled: empty plan");
  detail::require(table.resolution >= plan.n_total && table.resolution % plan.n_total == 0,
                  "fft_tiled: signal length must divide the table resolution");
  return detail::run_tiled(x, plan, table, TILEFFT_INVERSE);
}

}  // namespace b200
}  // namespace tilefft
