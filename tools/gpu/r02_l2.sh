#!/bin/bash
# L2 / DRAM / SM throughput of the main kernels (is the two-level pass L2-bound?)
M=gpu__time_duration.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.avg.per_cycle_active
B="python bench.py --configs none --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-cufft"
timeout 300 ncu --metrics $M --clock-control none -k regex:k_two -c 2 --csv --log-file gpurun_out/l2_two.csv $B --config 2d_8192 > /dev/null 2>&1
TILEFFT_TWO_DIAG=1 timeout 300 ncu --metrics $M --clock-control none -k regex:k_two -c 2 --csv --log-file gpurun_out/l2_two_diag.csv $B --config 2d_8192 > /dev/null 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:k_rows -c 2 --csv --log-file gpurun_out/l2_rows.csv $B > /dev/null 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:k_comb -c 2 --csv --log-file gpurun_out/l2_comb.csv $B --config 1d_2e26 > /dev/null 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:k_final -c 2 --csv --log-file gpurun_out/l2_final.csv $B --config 1d_2e26 > /dev/null 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:k_rows_pf -c 2 --csv --log-file gpurun_out/l2_rowspf.csv $B --config 2d_8192 > /dev/null 2>&1
for f in two two_diag rows comb final rowspf; do
python - gpurun_out/l2_$f.csv <<'PY'
import csv, sys
lines = open(sys.argv[1]).read().splitlines()
st = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(lines[st:]))
d = {}
for r in rows:
    if r["ID"] != rows[-1]["ID"]: continue
    d[r["Metric Name"]] = r["Metric Value"] + " " + r["Metric Unit"]
print(sys.argv[1], rows[-1]["Kernel Name"][:40]); [print("   ", k, v) for k, v in d.items()]
PY
done
