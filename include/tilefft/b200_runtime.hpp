// tilefft (B200) — host runtime behind the drop-in headers: device-plan cache
// and error mapping over the C ABI (include/tilefft_b200.h). Not part of the
// reference's API; the reference's entry points (fft_tiled, ifft_tiled,
// fft_levelwise, ...) use it to reach the GPU.
//
// Errors: TILEFFT_EINVAL -> std::invalid_argument (the reference's
// detail::require convention, common.hpp:47-51); anything else (no GPU, CUDA
// failure) -> std::runtime_error. There is no CPU fallback.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "tilefft_b200.h"

namespace tilefft {
inline namespace b200 {

/// Arithmetic tier used by fft_tiled / ifft_tiled. `fast` (default) is the
/// product path; `exact` executes the plan's factors with the reference's
/// radix-2 dataflow and returns bit-identical results. The environment
/// variable TILEFFT_MODE=exact selects it process-wide.
enum class ExecMode { fast = TILEFFT_MODE_FAST, exact = TILEFFT_MODE_EXACT };

namespace runtime {

inline void check(int rc) {
  if (rc == TILEFFT_OK) return;
  const std::string msg = tilefft_last_error();
  if (rc == TILEFFT_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("tilefft_b200: " + msg);
}

struct State {
  std::mutex mu;
  ExecMode mode = [] {
    const char* e = std::getenv("TILEFFT_MODE");
    return (e && std::strcmp(e, "exact") == 0) ? ExecMode::exact : ExecMode::fast;
  }();
  int device = [] {
    const char* e = std::getenv("TILEFFT_DEVICE");
    return e ? std::atoi(e) : 0;
  }();
  using Key = std::tuple<std::uint64_t, std::uint64_t, std::vector<std::uint64_t>, unsigned, unsigned, const void*,
                         std::uint64_t, int>;
  std::map<Key, tilefft_plan_t> plans;
  ~State() {
    for (auto& kv : plans) tilefft_plan_destroy(kv.second);
  }
};

inline State& state() {
  static State s;
  return s;
}

// Cached device plan for (n, batch, factors, precision, mode, table identity).
inline tilefft_plan_t device_plan(std::uint64_t n, std::uint64_t batch, const std::vector<std::uint64_t>& factors,
                                  unsigned elem_bytes, unsigned mode, const void* table, std::uint64_t resolution) {
  State& s = state();
  std::lock_guard<std::mutex> lk(s.mu);
  State::Key key{n, batch, factors, elem_bytes, mode, table, resolution, s.device};
  auto it = s.plans.find(key);
  if (it != s.plans.end()) return it->second;
  tilefft_plan_t p = nullptr;
  check(tilefft_plan_create(&p, n, batch, factors.empty() ? nullptr : factors.data(),
                            static_cast<std::uint32_t>(factors.size()), elem_bytes, mode, table, resolution, s.device));
  s.plans.emplace(key, p);
  return p;
}

}  // namespace runtime

inline void set_exec_mode(ExecMode m) {
  std::lock_guard<std::mutex> lk(runtime::state().mu);
  runtime::state().mode = m;
}
inline ExecMode exec_mode() { return runtime::state().mode; }
inline void set_device(int device) {
  std::lock_guard<std::mutex> lk(runtime::state().mu);
  runtime::state().device = device;
}
/// Release every cached device plan (they are otherwise kept for reuse).
inline void clear_plan_cache() {
  auto& s = runtime::state();
  std::lock_guard<std::mutex> lk(s.mu);
  for (auto& kv : s.plans) tilefft_plan_destroy(kv.second);
  s.plans.clear();
}

}  // namespace b200
}  // namespace tilefft
