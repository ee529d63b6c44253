# K_SMALL2 (fused small 2-pass plans): full GPU suite, then timings vs two launches
set -x
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
CASES='[["1d", 14], ["1d", 15], ["1d", 16], ["1d", 17], ["1d", 18], ["1d", 19], ["1d", 20]]' timeout 600 python tools/gpu/time_cfg.py \
  '[{"TILEFFT_NO_FUSE": 1}, {}]'
timeout 300 python bench.py --config 1d_2e20 --no-cpu-baseline --e2e-steps 2 --steps 50 2>&1 | tail -1
