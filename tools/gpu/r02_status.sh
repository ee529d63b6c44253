#!/bin/bash
# round-2 status: GPU tests, default bench (all configs as sub-records), two-level kernel A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -3 gpurun_out/bench_default.err
python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26], ["1d", 24]]' \
  '[{}, {"TILEFFT_TWO_KERNEL": 0}, {"TILEFFT_TWO_1D": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_KERNEL": 0}]'
