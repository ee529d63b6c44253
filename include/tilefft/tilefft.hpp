// tilefft (B200) — umbrella header; drop-in for
// /root/reference/proj/include/tilefft/tilefft.hpp (:17-25) for the hot path.
// Out of scope here: the O(N^2) reference DFT
// (it is this build's test oracle, oracle/), the access-pattern cost model
// (access_patterns.hpp, memsim.hpp) and the report/bench harness (bench.hpp).
#pragma once

#include "tilefft/common.hpp"
#include "tilefft/exec_model.hpp"
#include "tilefft/fft_baseline.hpp"
#include "tilefft/stage_plan.hpp"
#include "tilefft/tiled_fft.hpp"
#include "tilefft/twiddle.hpp"
