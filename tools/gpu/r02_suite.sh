#!/bin/bash
# report harness (reference run_suite schema + GPU columns) with the round-2 kernels
S=16,64,256,1024,4096,16384,65536,262144,1048576,4194304,16777216,67108864
timeout 1500 python -m paper_1707_07263_b200.suite --sizes $S --precision fp32 --out gpurun_out/r02_suite_fp32.csv 2>&1 | tail -2
timeout 1500 python -m paper_1707_07263_b200.suite --sizes 16,256,4096,65536,1048576,16777216 --precision fp64 --out gpurun_out/r02_suite_fp64.csv 2>&1 | tail -2
grep -E ",b200,|,cufft," gpurun_out/r02_suite_fp32.csv | awk -F, '{print $1, $2, $11}' | paste - - | tail -12
