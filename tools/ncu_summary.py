"""Key metrics of an ncu --set full report (raw page CSV) for the profiles/ summaries."""
import csv, subprocess, sys, json
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__bytes_read.sum.per_second', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_sector_hit_rate.pct', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.per_cycle_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'launch__waves_per_multiprocessor', 'launch__occupancy_limit_registers',
        'launch__shared_mem_per_block_dynamic', 'launch__shared_mem_per_block_static',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
        'smsp__inst_executed.sum', 'l1tex__t_bytes.sum', 'lts__t_bytes.sum',
        'sm__cycles_elapsed.avg.per_second', 'dram__cycles_elapsed.avg.per_second']
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
res = []
for v in rows[2:]:
    d = {'kernel': v[h.index('Kernel Name')][:60]}
    for w in WANT:
        if w in h:
            d[w] = f"{v[h.index(w)]} {u[h.index(w)]}".strip()
    res.append(d)
print(json.dumps(res, indent=1))
