"""Summarise an ncu --set full capture into profiles/ (run in the build
container on a report brought back from the GPU box).

    python tools/profile_report.py gpurun_out/prof.ncu-rep profiles/r1_name.txt [workload]

Writes the per-launch key metrics and stall breakdown, the top stall sites of
the first launch (SASS), and records dram read+write bytes per launch of the
hot kernel into profiles/roofline_traffic.json (read by bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'dram__bytes_read.sum',
        'dram__bytes_write.sum', 'lts__t_bytes.sum', 'smsp__inst_executed.sum',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'lts__t_sector_hit_rate.pct',
        'launch__registers_per_thread', 'sm__cycles_elapsed.avg.per_second']


def ncu_csv(rep, *args):
    out = subprocess.run(['ncu', '-i', rep, *args, '--csv'], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_bytes(v, unit):
    v = float(v)
    return v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(unit, 1)


def main():
    rep, out_path = sys.argv[1], sys.argv[2]
    workload = sys.argv[3] if len(sys.argv) > 3 else 'cfg1-als-full'
    rows = ncu_csv(rep, '--page', 'raw')
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f'# ncu --set full summary of {os.path.basename(rep)}', '']
    traffic = []
    for k, d in enumerate(data):
        name = d[hdr.index('Kernel Name')]
        lines.append(f'launch {k}: {name[:110]}')
        for h in KEYS:
            if h in hdr:
                lines.append(f'    {h:<66} {d[hdr.index(h)]} {units[hdr.index(h)]}')
        st = []
        for h, v in zip(hdr, d):
            if 'smsp__average_warps_issue_stalled' in h and h.endswith('_per_issue_active.ratio'):
                try:
                    st.append((float(v), h.split('stalled_')[1].replace('_per_issue_active.ratio', '')))
                except ValueError:
                    pass
        st.sort(reverse=True)
        lines.append('    stalls per issued instruction: ' +
                     ', '.join(f'{n} {v:.2f}' for v, n in st[:8]))
        if 'k_als_pair' in name:
            rd = to_bytes(d[hdr.index('dram__bytes_read.sum')], units[hdr.index('dram__bytes_read.sum')])
            wr = to_bytes(d[hdr.index('dram__bytes_write.sum')], units[hdr.index('dram__bytes_write.sum')])
            traffic.append(rd + wr)
        lines.append('')
    src = ncu_csv(rep, '--page', 'source', '--print-source', 'sass')
    if len(src) > 2:
        sh = src[1]
        try:
            ai, si = sh.index('Address'), sh.index('Source')
            wi, ei = sh.index('Warp Stall Sampling (All Samples)'), sh.index('Instructions Executed')
            rec = []
            for r in src[2:]:
                if len(r) != len(sh) or r[0] == 'Kernel Name':
                    break
                rec.append((int(r[wi]), int(r[ei]), r[si].strip()))
            tot = sum(x[0] for x in rec) or 1
            lines.append('top stall sites (launch 0, SASS): samples  executions  instruction')
            for s_, e_, t_ in sorted(rec, reverse=True)[:15]:
                lines.append(f'    {100 * s_ / tot:5.1f}%  {e_:>11}  {t_[:80]}')
        except ValueError:
            pass
    with open(out_path, 'w') as fh:
        fh.write('\n'.join(lines) + '\n')
    if traffic:
        tpath = os.path.join(os.path.dirname(out_path), 'roofline_traffic.json')
        cur = json.load(open(tpath)) if os.path.exists(tpath) else {}
        cur[workload] = sum(traffic) / len(traffic)
        json.dump(cur, open(tpath, 'w'), indent=1)
    print('\n'.join(lines[:40]))


if __name__ == '__main__':
    main()
