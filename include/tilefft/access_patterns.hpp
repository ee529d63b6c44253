// tilefft (B200) — request shapes of the reference's cost model
// (/root/reference/proj/include/tilefft/access_patterns.hpp:28-173).
//
// Each generator walks one sweep of the algorithm in the model's execution
// order and hands every warp-wide (slow memory) or half-warp (fast storage)
// request to a callback. The traced drop-in calls replay them into an
// AccessRecorder and the closed-form accounting (memsim.hpp) replays the
// same ones, so trace == account_* holds by construction, exactly as in the
// reference. All shapes are properties of the plan alone (host logic).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <span>
#include <vector>

#include "tilefft/common.hpp"
#include "tilefft/exec_model.hpp"
#include "tilefft/stage_plan.hpp"

namespace tilefft {
inline namespace b200 {
namespace detail {

/// Splits the index range [0, count) into consecutive lane groups of at most
/// `lanes` indices and calls emit(first, width) for each group.
template <typename Emit>
void for_each_lane_group(std::size_t count, std::size_t lanes, Emit&& emit) {
  for (std::size_t first = 0; first < count; first += lanes) emit(first, std::min(lanes, count - first));
}

/// fft_levelwise level `level` (1-based, span 2^level): lane t of a warp owns
/// butterfly t, i.e. elements lo(t) = (t / h) * 2h + t % h and lo(t) + h.
/// Per warp: read lower legs, read upper legs, write lower, write upper
/// (fft_baseline.hpp:90-114). fn(addresses, is_write).
template <typename Fn>
void for_each_levelwise_request(std::size_t n, unsigned level, const ExecConfig& config, Fn&& fn) {
  const std::size_t h = std::size_t{1} << (level - 1);
  std::vector<std::uint64_t> lower, upper;
  for_each_lane_group(n / 2, config.warp_size, [&](std::size_t t0, std::size_t width) {
    lower.resize(width);
    upper.resize(width);
    for (std::size_t i = 0; i < width; ++i) {
      const std::size_t t = t0 + i;
      lower[i] = (t / h) * 2 * h + t % h;
      upper[i] = lower[i] + h;
    }
    fn(std::span<const std::uint64_t>(lower), false);
    fn(std::span<const std::uint64_t>(upper), false);
    fn(std::span<const std::uint64_t>(lower), true);
    fn(std::span<const std::uint64_t>(upper), true);
  });
}

/// The levelwise bit-reversal sweep out[i] = in[bitrev(i)] (fft_baseline.hpp:74-79),
/// lanes on consecutive i: a gather request then a store request per warp.
template <typename Fn>
void for_each_reorder_request(std::size_t n, const ExecConfig& config, Fn&& fn) {
  const unsigned bits = log2_exact(n);
  std::vector<std::uint64_t> from, to;
  for_each_lane_group(n, config.warp_size, [&](std::size_t i0, std::size_t width) {
    from.resize(width);
    to.resize(width);
    for (std::size_t i = 0; i < width; ++i) {
      from[i] = bit_reverse(i0 + i, bits);
      to[i] = i0 + i;
    }
    fn(std::span<const std::uint64_t>(from), false);
    fn(std::span<const std::uint64_t>(to), true);
  });
}

/// One pass's tile load (gather = true: the bit-reversed comb gather,
/// tiled_fft.hpp:265-272) or store sweep (the scatter through the pass's
/// store map, :284-306). Within a tile the slots run column-major — slot ->
/// (col = slot / rows_per_tile, grow = first_row + slot % rows_per_tile) — and
/// a warp never spans two tiles.
template <typename Fn>
void for_each_tiled_sweep_request(const StagePlan& plan, std::size_t stage, bool gather, const ExecConfig& config,
                                  Fn&& fn) {
  const StageGeometry& g = plan.stage(stage);
  const unsigned bits = static_cast<unsigned>(g.levels);
  const std::size_t slots = g.rows_per_tile * g.fft_len;
  std::vector<std::uint64_t> addr;
  for (std::size_t tile = 0; tile < g.tile_count; ++tile) {
    const std::size_t row0 = tile * g.rows_per_tile;
    for_each_lane_group(slots, config.warp_size, [&](std::size_t s0, std::size_t width) {
      addr.resize(width);
      for (std::size_t i = 0; i < width; ++i) {
        const std::size_t col = (s0 + i) / g.rows_per_tile, grow = row0 + (s0 + i) % g.rows_per_tile;
        addr[i] = gather ? gather_source_index(g, grow, static_cast<std::size_t>(bit_reverse(col, bits)))
                         : scatter_target_index(plan, stage, grow, col);
      }
      fn(std::span<const std::uint64_t>(addr), !gather);
    });
  }
}

/// exchange_transpose (tiled_fft.hpp:179-203): contiguous reads, stores
/// through exchange_index_map.
template <typename Fn>
void for_each_exchange_request(const StagePlan& plan, std::size_t stage, const ExecConfig& config, Fn&& fn) {
  std::vector<std::uint64_t> from, to;
  for_each_lane_group(plan.n_total, config.warp_size, [&](std::size_t q0, std::size_t width) {
    from.resize(width);
    to.resize(width);
    for (std::size_t i = 0; i < width; ++i) {
      from[i] = q0 + i;
      to[i] = exchange_index_map(plan, stage, q0 + i);
    }
    fn(std::span<const std::uint64_t>(from), false);
    fn(std::span<const std::uint64_t>(to), true);
  });
}

/// Fast-storage footprint of a pass: half-warps of consecutive tile rows
/// (the last may be short) walk every column at the row stride; each walk is
/// one request shape, replayed on every in-tile access occasion.
/// fn(word_addresses) once per (row group, column).
template <typename Fn>
void for_each_column_stream(std::size_t rows, std::size_t cols, std::size_t stride, const ExecConfig& config,
                            Fn&& fn) {
  std::vector<std::uint64_t> words;
  for_each_lane_group(rows, config.half_warp_size, [&](std::size_t r0, std::size_t width) {
    words.resize(width);
    for (std::size_t col = 0; col < cols; ++col) {
      for (std::size_t i = 0; i < width; ++i) words[i] = (r0 + i) * stride + col;
      fn(std::span<const std::uint64_t>(words));
    }
  });
}

/// In-tile access occasions per column position: the load, the store and two
/// butterfly legs per level (the inter-pass scale rides the store).
inline std::uint64_t column_stream_occasions(const StagePlan& plan, std::size_t stage) {
  return 2 + 2 * static_cast<std::uint64_t>(plan.stage(stage).levels);
}

/// Root-table lookups of one pass: fft_len - 1 hoisted per tile (dit_levels,
/// tiled_fft.hpp:94-100) plus one per element for the inter-pass scale.
inline std::uint64_t stage_twiddle_fetches(const StagePlan& plan, std::size_t stage) {
  const StageGeometry& g = plan.stage(stage);
  return g.tile_count * (g.fft_len - 1) + (stage < plan.pass_count() ? plan.n_total : 0);
}

}  // namespace detail
}  // namespace b200
}  // namespace tilefft
