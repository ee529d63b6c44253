# final state: full GPU suite, smoke, default bench + reference arm, report-harness sweeps
set -x
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json
timeout 900 python bench.py --impl reference 2>&1 | tail -1 > gpurun_out/bench_reference.json
S=16,64,256,1024,4096,16384,65536,262144,1048576,4194304,16777216,67108864
timeout 1500 python -m paper_1707_07263_b200.suite --sizes $S --precision fp32 --out gpurun_out/suite_fp32.csv > /dev/null 2>&1; echo suite32 rc=$?
timeout 1500 python -m paper_1707_07263_b200.suite --sizes ${S%,67108864} --precision fp64 --out gpurun_out/suite_fp64.csv > /dev/null 2>&1; echo suite64 rc=$?
