#!/bin/bash
# k_two_tma: hang repro (NG=2, 1D 2^26 with TWO_1D), copy-only diagnostics, ncu full of the column pass
python tools/gpu/two_probe.py '[["1d", 26], ["2d", 8192, 8192]]' \
  '[{"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_KERNEL": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_KERNEL": 2}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_KERNEL": 2, "TILEFFT_TWO_DIAG": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_KERNEL": 1, "TILEFFT_TWO_DIAG": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_KERNEL": 0}]'
for K in 2 1; do
REPS=2 TILEFFT_TWO_KERNEL=$K timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_two_tma -c 1 -o gpurun_out/two_tma_full_k$K \
  python tools/gpu/two_probe.py --child '["2d", 8192, 8192]' > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/two_tma_full_k$K.ncu-rep > gpurun_out/two_tma_full_k$K.json
done
