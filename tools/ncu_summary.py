import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ['gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'smsp__inst_executed.sum',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'lts__t_sector_hit_rate.pct', 'launch__registers_per_thread',
        'sm__cycles_elapsed.avg.per_second']
for k, d in enumerate(data):
    print('launch', k, d[hdr.index('Kernel Name')][:40])
    for h in want:
        if h in hdr:
            print('   %-70s %s %s' % (h, d[hdr.index(h)], units[hdr.index(h)]))
    items = []
    for h, v in zip(hdr, d):
        if 'smsp__average_warps_issue_stalled' in h and h.endswith('_per_issue_active.ratio'):
            try:
                items.append((float(v), h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
            except ValueError:
                pass
    items.sort(reverse=True)
    print('   stalls/issue:', ', '.join('%s %.2f' % (h, v) for v, h in items[:7]))
