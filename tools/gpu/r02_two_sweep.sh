#!/bin/bash
# two-level lag/slot sweep (8192^2 columns and 2^26 as two two-level passes)
V='[{"TILEFFT_TWO_1D": 1}'
for d in 32 40 48 56 64 80; do
  for s in $((d+8)) $((d+16)) $((d+32)); do V="$V, {\"TILEFFT_TWO_1D\": 1, \"TILEFFT_TWO_D\": $d, \"TILEFFT_TWO_NSLOT\": $s}"; done
done
V="$V]"
REPS=40 python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26]]' "$V"
