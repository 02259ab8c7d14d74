"""Print the key metrics + top stall reasons of every kernel in an .ncu-rep."""
import csv, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'lts__t_bytes.sum']
for r in rows[2:]:
    print(r[h.index('Kernel Name')][:70])
    for k in keys:
        if k in h:
            print(f"    {k:60s} {r[h.index(k)]:>14s} {rows[1][h.index(k)]}")
    st = []
    for i, name in enumerate(h):
        if 'issue_stalled' in name and name.endswith('per_issue_active.ratio'):
            try:
                st.append((float(r[i]), name.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
            except ValueError:
                pass
    print('    stalls:', ', '.join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:6]))
