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
#include <list>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <type_traits>
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

// Process-wide cache of device plans, least-recently-used first out: each
// plan pins device workspace and host-path staging, so the cache is bounded
// (TILEFFT_PLAN_CACHE entries, default 16). FAST plans are keyed by shape
// only (the device chooses its own passes); EXACT/LEVELWISE plans copy the
// caller's table at creation, so they are keyed by a hash of the roots they
// use, never by the table's address alone.
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
  std::size_t capacity = [] {
    const char* e = std::getenv("TILEFFT_PLAN_CACHE");
    const long v = e ? std::atol(e) : 16;
    return static_cast<std::size_t>(v > 0 ? v : 1);
  }();
  using Key = std::tuple<std::uint64_t, std::uint64_t, std::vector<std::uint64_t>, unsigned, unsigned, std::uint64_t,
                         std::uint64_t, int>;
  // shared ownership: a plan evicted while another thread still executes it
  // is destroyed when that call drops its reference
  using Plan = std::shared_ptr<std::remove_pointer_t<tilefft_plan_t>>;
  std::list<std::pair<Key, Plan>> lru;  // front = most recently used
};

inline State& state() {
  static State s;
  return s;
}

// FNV-1a over the n roots a table-based plan copies (entries j * resolution / n).
inline std::uint64_t table_fingerprint(const void* table, std::uint64_t resolution, std::uint64_t n,
                                       unsigned elem_bytes) {
  if (table == nullptr) return 0;
  const unsigned char* b = static_cast<const unsigned char*>(table);
  const std::uint64_t stride = (resolution / n) * elem_bytes;
  std::uint64_t h = 1469598103934665603ull;
  for (std::uint64_t j = 0; j < n; ++j)
    for (unsigned i = 0; i < elem_bytes; ++i) h = (h ^ b[j * stride + i]) * 1099511628211ull;
  return h;
}

// Cached device plan for (n, batch, factors, precision, mode, table contents).
inline State::Plan device_plan(std::uint64_t n, std::uint64_t batch, const std::vector<std::uint64_t>& factors,
                                  unsigned elem_bytes, unsigned mode, const void* table, std::uint64_t resolution) {
  State& s = state();
  std::lock_guard<std::mutex> lk(s.mu);
  const bool fast = mode == TILEFFT_MODE_FAST;
  const std::uint64_t fp = fast ? 0 : table_fingerprint(table, resolution, n, elem_bytes);
  State::Key key{n, batch, fast ? std::vector<std::uint64_t>{} : factors, elem_bytes, mode, fp,
                 fast ? 0 : resolution, s.device};
  for (auto it = s.lru.begin(); it != s.lru.end(); ++it)
    if (it->first == key) {
      s.lru.splice(s.lru.begin(), s.lru, it);
      return it->second;
    }
  tilefft_plan_t p = nullptr;
  check(tilefft_plan_create(&p, n, batch, factors.empty() ? nullptr : factors.data(),
                            static_cast<std::uint32_t>(factors.size()), elem_bytes, mode, table, resolution, s.device));
  s.lru.emplace_front(key, State::Plan(p, tilefft_plan_destroy));
  while (s.lru.size() > s.capacity) s.lru.pop_back();
  return s.lru.front().second;
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
  s.lru.clear();
}

}  // namespace b200
}  // namespace tilefft
