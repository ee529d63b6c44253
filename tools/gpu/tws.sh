# stage roots: read-only path (LDG.CONSTANT, L1) vs staged in shared memory (LDS), batched 1024 x 65536
set -x
TILEFFT_TW_SMEM=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fast" 2>&1 | tail -2
for v in 0 1; do
  TILEFFT_TW_SMEM=$v timeout 300 python bench.py --steps 100 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TW_SMEM=$v', d['ms_per_step'], d['roofline']['frac'])"
done
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__t_sector_hit_rate.pct,smsp__pcsamp_warps_issue_stalled_lg_throttle,smsp__pcsamp_warps_issue_stalled_mio_throttle,smsp__pcsamp_warps_issue_stalled_short_scoreboard,smsp__pcsamp_warps_issue_stalled_long_scoreboard,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
for v in 0 1; do
  TILEFFT_TW_SMEM=$v timeout 600 ncu --metrics $M --clock-control none -k regex:k_rows_tma -s 3 -c 1 --csv --log-file gpurun_out/tws_$v.csv python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
  grep -o '"[a-z_0-9.]*","[^"]*","[0-9.,]*"' gpurun_out/tws_$v.csv | tail -12
done
