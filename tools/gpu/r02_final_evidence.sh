#!/bin/bash
# round-2 evidence: GPU suite, smoke, default bench line, reference arm, launch lists and ncu --set full
# summaries of the dominant kernels (reports summarised on the box; 64 MiB copy-back cap)
mkdir -p gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/ev/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev/gputest.log 2>&1; tail -2 gpurun_out/ev/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; tail -1 gpurun_out/ev/smoke.log
timeout 900 python bench.py > gpurun_out/ev/bench_default.json 2> gpurun_out/ev/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_reference.json 2>&1
B="python bench.py --configs none --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-cufft"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in batched1024 1d_2e20 1d_2e26 2d_8192 1d_2e30; do
  timeout 600 ncu --metrics $M --clock-control none -c 40 --csv --log-file gpurun_out/ev/launches_$c.csv $B --config $c > /dev/null 2>&1
done
P="ncu --set full --clock-control none --import-source on"
prof() {
  timeout 600 $P -k regex:$2 -s $3 -c 1 -o /tmp/prof_$1 $B $4 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/prof_$1.ncu-rep > gpurun_out/ev/ncu_$1.json
  ncu -i /tmp/prof_$1.ncu-rep --page source --csv > /tmp/src_$1.csv 2>&1
  python tools/ncu_source_top.py /tmp/src_$1.csv 40 > gpurun_out/ev/ncu_$1_top_sass.txt
  rm -f /tmp/prof_$1.ncu-rep
}
prof rows_tma k_rows_tma 3 ""
prof two_tma k_two_tma 1 "--config 2d_8192"
prof rows_pf k_rows_pf 1 "--config 2d_8192"
prof comb_2e26 k_comb_h3 2 "--config 1d_2e26"
prof comb_2e30 k_comb_h3 0 "--config 1d_2e30"
prof final_2e26 k_final_p 1 "--config 1d_2e26"
prof final_2e30 k_final_p 0 "--config 1d_2e30"
python tools/traffic_json.py gpurun_out/ev/bench_default.json gpurun_out/ev/launches > gpurun_out/ev/traffic.json
du -sh gpurun_out/ev
