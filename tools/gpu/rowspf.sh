set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_twolevel.py tests/test_cpp_dropin.py -q -x 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4 --csv --log-file gpurun_out/launches_rowspf.csv python bench.py --config 2d_8192 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_rowspf.csv
CASES='[["2d", 8192, 8192], ["2d", 4096, 4096], ["2d", 2048, 2048]]' timeout 900 python tools/gpu/time_cfg.py '[{}, {"TILEFFT_NO_ROWS_PF": 1}]'
