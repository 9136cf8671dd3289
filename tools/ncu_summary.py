"""Summarise an ncu report: key metrics per kernel.  python tools/ncu_summary.py REPORT [--json OUT]"""
import csv
import io
import json
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'launch__grid_size', 'launch__block_size', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'lts__t_sector_hit_rate.pct',
        'smsp__average_warp_latency_issue_stalled_long_scoreboard', 'smsp__average_warp_latency_issue_stalled_barrier',
        'smsp__average_warp_latency_issue_stalled_short_scoreboard', 'smsp__average_warp_latency_issue_stalled_wait',
        'smsp__inst_executed_pipe_fp64.sum', 'launch__shared_mem_per_block_dynamic']


def summarise(path):
    raw = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {'kernel': r[hdr.index('Kernel Name')]}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                d[w] = (r[i], units[i])
        out.append(d)
    return out


if __name__ == '__main__':
    res = summarise(sys.argv[1])
    for d in res:
        print(d['kernel'][:110])
        for k, v in d.items():
            if k != 'kernel':
                print(f'   {k:65s} {v[0]:>14s} {v[1]}')
    if '--json' in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index('--json') + 1], 'w'), indent=1)
