# 8-comb / 8-row tiles for the comb and final passes: parity under each switch, then timings
set -x
for v in "TILEFFT_NONE=0"; do
  env $v timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_twolevel.py -q -x 2>&1 | tail -2
done
CASES='[["1d", 20], ["1d", 24], ["1d", 26], ["1d", 30]]' timeout 900 python tools/gpu/time_cfg.py \
  '[{}, {"TILEFFT_FINAL_F": 8}, {"TILEFFT_COMB_F": 8}, {"TILEFFT_COMB_F": 8, "TILEFFT_FINAL_F": 8}]'
