#!/usr/bin/env python3
"""One markdown table row per kernel launch of an `ncu --set full` report:
duration, DRAM read / write, FP64 pipe, issue rate, resident warps, registers.
Usage: python scripts/ncu_table.py gpurun_out/prof_TAG.ncu-rep > profiles/TAG_ncu_full.md"""
import csv, io, subprocess, sys

COLS = [('us', 'gpu__time_duration.sum', 1e-3, 1),
        ('DRAM rd MB', 'dram__bytes_read.sum', None, 1),
        ('DRAM wr MB', 'dram__bytes_write.sum', None, 1),
        ('FP64 pipe %', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 1, 1),
        ('issue %', 'smsp__issue_active.avg.pct_of_peak_sustained_active', 1, 1),
        ('warps/SM', 'sm__warps_active.avg.per_cycle_active', 1, 1),
        ('regs', 'launch__registers_per_thread', 1, 0)]
UNIT = {'byte': 1e-6, 'Kbyte': 1e-3, 'Mbyte': 1.0, 'Gbyte': 1e3, 'ns': 1e-3, 'us': 1.0, 'ms': 1e3}


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    print('| kernel | ' + ' | '.join(c[0] for c in COLS) + ' |')
    print('|' + '---|' * (len(COLS) + 1))
    for r in rows[2:]:
        name = r[idx['Kernel Name']]
        name = name.split('(')[0].replace('dsft::', '').replace('void ', '')
        cells = []
        for title, metric, scale, nd in COLS:
            i = idx.get(metric)
            if i is None:
                cells.append('-')
                continue
            v = float(r[i].replace(',', ''))
            u = units[i]
            if u in UNIT and (scale is None or title == 'us'):
                v *= UNIT[u]          # to MB / us
            cells.append(f'{v:.{nd}f}')
        print(f'| {name} | ' + ' | '.join(cells) + ' |')


if __name__ == '__main__':
    main(sys.argv[1])
