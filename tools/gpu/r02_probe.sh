#!/bin/bash
# round-2 first probe: host resources, GPU test suite, default bench
set -x
nproc; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --steps 20 --warmup 5 2>&1 | tail -2
