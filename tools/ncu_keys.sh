#!/bin/bash
# Key metrics of one ncu report: tools/ncu_keys.sh report.ncu-rep
ncu -i "$1" --page raw --csv 2>/dev/null | python3 -c "
import csv, sys
rows = list(csv.reader(sys.stdin))
hdr, units = rows[0], rows[1]
want = ['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sector_hit_rate.pct',
 'sm__warps_active.avg.pct_of_peak_sustained_active','sm__throughput.avg.pct_of_peak_sustained_elapsed',
 'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed','dram__throughput.avg.pct_of_peak_sustained_elapsed',
 'lts__throughput.avg.pct_of_peak_sustained_elapsed','l1tex__throughput.avg.pct_of_peak_sustained_elapsed',
 'sm__inst_executed.avg.per_cycle_active','smsp__issue_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread',
 'launch__occupancy_limit_shared_mem','sm__maximum_warps_per_active_cycle_pct','launch__grid_size','launch__block_size',
 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','smsp__inst_executed.sum','lts__t_bytes.sum']
for r in rows[2:]:
    d = dict(zip(hdr, r))
    for w in want:
        if w in d: print(f'{w:70s} {d[w]} {units[hdr.index(w)]}')
    stalls = sorted(((float(d[k] or 0), k) for k in hdr if k.startswith('smsp__average_warp_latency_issue_stalled') or k.startswith('smsp__pcsamp_warps_issue_stalled')), reverse=True)[:10]
    for v,k in stalls: print(f'   {k:80s} {v}')
    print('----')
"
