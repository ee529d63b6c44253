// C ABI of the reference's cost model (include/tilefft/memsim.hpp): the
// closed-form AccessStats of fft_tiled under make_plan(n, tile_capacity) or of
// fft_levelwise, for callers without the C++ headers (the Python mirror and
// its run_suite report, paper_1707_07263_b200/suite.py). Host logic only.
#include <cstdint>
#include <stdexcept>

#include "tilefft/memsim.hpp"
#include "tilefft_b200.h"

extern "C" int tilefft_account(uint64_t n, uint64_t tile_capacity, uint32_t algorithm, uint64_t* stats) {
  if (stats == nullptr) return TILEFFT_EINVAL;
  try {
    const tilefft::AccessStats s = algorithm == TILEFFT_ACCOUNT_LEVELWISE
                                       ? tilefft::account_levelwise(n)
                                       : tilefft::account_tiled(tilefft::make_plan(n, tile_capacity));
    const uint64_t v[7] = {s.slow_elem_reads, s.slow_elem_writes, s.slow_transactions, s.fast_accesses,
                           s.bank_conflict_cycles, s.barriers, s.twiddle_fetches};
    for (int i = 0; i < 7; ++i) stats[i] = v[i];
    return TILEFFT_OK;
  } catch (const std::invalid_argument&) {
    return TILEFFT_EINVAL;
  }
}
