#!/bin/bash
# persistent final pass as the default: parity suites; N=2 bench path exercised on one GPU (gloo, both ranks on cuda:0)
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_plans.py tests/test_cpp_dropin.py tests/test_distributed.py -x -q 2>&1 | tail -2
TILEFFT_BENCH_BACKEND=gloo TILEFFT_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
tail -3 gpurun_out/bench_n2.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_n2.json').read().strip().splitlines()[-1]); print(d['n_gpus'], d['value'], {k: (v.get('value'), v.get('nvlink'), v.get('error')) for k, v in d.get('configs', {}).items()})"
