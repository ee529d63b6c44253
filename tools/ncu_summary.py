#!/usr/bin/env python3
"""Summarise an ncu report (raw page) into the metrics we track (profiles/*.json)."""
import csv
import io
import json
import subprocess
import sys

KEEP = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size', 'sm__warps_active.avg.per_cycle_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'smsp__inst_executed.sum', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'lts__t_sector_hit_rate.pct', 'sm__issue_active.avg.pct_of_peak_sustained_active',
        'launch__shared_mem_per_block_dynamic', 'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'lts__t_bytes.sum', 'l1tex__t_bytes.sum']


def summarize(rep):
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        s = {k: (d[k] + (' ' + u[k] if u.get(k) else '')) for k in KEEP if k in d}
        st = [(k.replace('smsp__pcsamp_warps_issue_stalled_', ''), d[k]) for k in hdr
              if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued')]
        st = sorted([(k, float(v.replace(',', ''))) for k, v in st if v and v.replace(',', '').replace('.', '').isdigit()],
                    key=lambda x: -x[1])
        s['top_stall_samples'] = dict(st[:8])
        out.append(s)
    return out


if __name__ == '__main__':
    res = {r: summarize(r) for r in sys.argv[1:]}
    print(json.dumps(res, indent=1))
