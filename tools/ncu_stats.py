"""Per-kernel key metrics + top stall reasons from an .ncu-rep (raw page)."""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__registers_per_thread',
        'launch__occupancy_limit_shared_mem', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'dram__throughput.avg.pct_of_peak_sustained_elapsed']
for r in rows[2:]:
    name = r[h.index('Kernel Name')][:60]
    print(name)
    print('   ', '  '.join(f"{w.split('__')[1].split('.')[0][:28]}={r[h.index(w)]}{u[h.index(w)][:6]}" for w in want if w in h))
    st = sorted([(float(r[i].replace(',', '') or 0), c.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''))
                 for i, c in enumerate(h) if c.startswith('smsp__average_warps_issue_stalled_') and c.endswith('per_issue_active.ratio') and r[i]], reverse=True)[:6]
    print('    stalls', ' '.join(f'{n}={v:.2f}' for v, n in st))
