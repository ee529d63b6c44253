# Per-launch kernel list (cold, serialised) for every config: time + DRAM bytes.
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in ${CONFIGS:-1d_2e20 1d_2e26 2d_8192 1d_2e30}; do
  timeout 600 ncu --metrics $M --clock-control none -c ${NL:-12} --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/launches_$c.csv
done
