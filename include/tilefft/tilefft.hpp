// tilefft (B200) — umbrella header; drop-in for
// /root/reference/proj/include/tilefft/tilefft.hpp (:17-25) for the hot path.
// Out of scope here: the O(N^2) reference DFT (it is this build's
// test oracle, oracle/) and the C++ report/bench harness (bench.hpp; its GPU
// counterpart is paper_1707_07263_b200/suite.py).
#pragma once

#include "tilefft/access_patterns.hpp"
#include "tilefft/common.hpp"
#include "tilefft/exec_model.hpp"
#include "tilefft/memsim.hpp"
#include "tilefft/fft_baseline.hpp"
#include "tilefft/stage_plan.hpp"
#include "tilefft/tiled_fft.hpp"
#include "tilefft/twiddle.hpp"
