set -x
timeout 600 python -m pytest tests/test_gpu_twolevel.py -q -x 2>&1 | tail -2
TILEFFT_TWO_1D=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4 --csv --log-file gpurun_out/launches_two1d.csv python bench.py --config 1d_2e26 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_two1d.csv
CASES='[["2d", 8192, 8192], ["1d", 24], ["1d", 26]]' timeout 900 python tools/gpu/time_cfg.py '[{"TILEFFT_TWO_1D": 1}]'
