# per-launch times for one config under an env setting: launch_env.sh CONFIG NAME [VAR=VAL ...]
c=$1; name=$2; shift 2
env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3 --csv \
  --log-file gpurun_out/launches_${name}.csv python bench.py --config $c --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_${name}.csv
