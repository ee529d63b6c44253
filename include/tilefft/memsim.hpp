// tilefft (B200) — closed-form traffic accounting of the reference's cost
// model (/root/reference/proj/include/tilefft/memsim.hpp:38-104).
//
// Element, barrier, fast-access and fetch counters are closed forms of the
// plan; transactions and conflict cycles replay the request shapes of
// access_patterns.hpp. The traced drop-in calls record the same shapes, so a
// trace agrees with these figures field for field (the reference's
// acceptance criteria 4 and 7, tests/acceptance_main.cpp:158-195).
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>

#include "tilefft/access_patterns.hpp"
#include "tilefft/common.hpp"
#include "tilefft/exec_model.hpp"
#include "tilefft/stage_plan.hpp"

namespace tilefft {
inline namespace b200 {

/// fft_levelwise of length n (the bit-reversal sweep is the recorder's
/// reorder bucket and is not included): log2 n levels, each moving all n
/// elements through slow memory, one root per butterfly, one barrier.
inline AccessStats account_levelwise(std::size_t n, const ExecConfig& config = {}) {
  detail::require(is_power_of_two(n) && n >= 2, "account_levelwise: n must be a power of two >= 2");
  config.validate();
  const unsigned levels = log2_exact(n);
  AccessStats st;
  st.slow_elem_reads = st.slow_elem_writes = static_cast<std::uint64_t>(n) * levels;
  st.barriers = levels;
  st.twiddle_fetches = static_cast<std::uint64_t>(n / 2) * levels;
  for (unsigned lv = 1; lv <= levels; ++lv)
    detail::for_each_levelwise_request(n, lv, config, [&](std::span<const std::uint64_t> a, bool) {
      st.slow_transactions += coalesced_transactions(a, config);
    });
  return st;
}

/// Counters of one pass of fft_tiled (accumulated into `st`).
inline void account_tiled_stage(const StagePlan& plan, std::size_t stage, const ExecConfig& config, AccessStats& st) {
  const StageGeometry& g = plan.stage(stage);
  const std::uint64_t n = plan.n_total, occ = detail::column_stream_occasions(plan, stage);
  st.slow_elem_reads += n;
  st.slow_elem_writes += n;
  st.barriers += 1;
  st.twiddle_fetches += detail::stage_twiddle_fetches(plan, stage);
  st.fast_accesses += n * occ;
  for (const bool gather : {true, false})
    detail::for_each_tiled_sweep_request(plan, stage, gather, config, [&](std::span<const std::uint64_t> a, bool) {
      st.slow_transactions += coalesced_transactions(a, config);
    });
  detail::for_each_column_stream(g.rows, g.fft_len, g.padded_stride, config, [&](std::span<const std::uint64_t> w) {
    const unsigned d = bank_conflict_degree(w, config);
    if (d > 1) st.bank_conflict_cycles += occ * (d - 1);
  });
}

/// fft_tiled under `plan`: every pass moves all n elements through fast
/// storage once, so slow element traffic is 2 * n * passes.
inline AccessStats account_tiled(const StagePlan& plan, const ExecConfig& config = {}) {
  detail::require(plan.pass_count() >= 1, "account_tiled: empty plan");
  config.validate();
  detail::require(plan.bank_count == config.bank_count, "account_tiled: plan was built for a different bank count");
  AccessStats st;
  for (std::size_t s = 1; s <= plan.pass_count(); ++s) account_tiled_stage(plan, s, config, st);
  return st;
}

/// Slow-traffic reduction of the plan against the levelwise method:
/// (2 n log2 n) / (2 n p) = log2(n) / p.
inline double reduction_ratio(std::size_t n, const StagePlan& plan) {
  detail::require(n == plan.n_total, "reduction_ratio: n does not match the plan");
  detail::require(plan.pass_count() >= 1, "reduction_ratio: empty plan");
  return static_cast<double>(log2_exact(n)) / static_cast<double>(plan.pass_count());
}

}  // namespace b200
}  // namespace tilefft
