# Full GPU state check: parity suite, smoke, default bench line, per-config bench lines.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json; cat gpurun_out/bench_default.json
for c in 1d_2e20 1d_2e26 2d_8192 1d_2e30; do timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 2 --steps 20 2>&1 | tail -1; done
