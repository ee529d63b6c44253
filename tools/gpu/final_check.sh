set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_reference.json
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json
cat gpurun_out/bench_reference.json gpurun_out/bench_default.json
