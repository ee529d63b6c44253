#!/bin/bash
# stability: the GPU suite three times in a row; the N=2 bench path (gloo, both ranks on cuda:0) end to end
mkdir -p gpurun_out/stab
for i in 1 2 3; do timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/stab/gputest_$i.log 2>&1; tail -1 gpurun_out/stab/gputest_$i.log; done
TILEFFT_BENCH_BACKEND=gloo TILEFFT_BENCH_DEVICE=0 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/stab/bench_n2.json 2> gpurun_out/stab/bench_n2.err
python - <<'PY'
import json
d = json.loads(open('gpurun_out/stab/bench_n2.json').read().strip().splitlines()[-1])
print("n_gpus", d["n_gpus"], "headline", d["value"])
for k, v in d.get("configs", {}).items():
    print(k, v.get("error") or (v["value"], v["parallelism"], v.get("nvlink")))
PY
