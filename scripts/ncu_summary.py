#!/usr/bin/env python3
"""Print the key ncu --set full metrics (and top stall reasons) of a .ncu-rep."""
import csv, subprocess, sys, io

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct',
        'sm__warps_active.avg.per_cycle_active', 'launch__registers_per_thread', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__cycles_elapsed.avg.per_second',
        'launch__grid_size', 'launch__block_size', 'launch__shared_mem_per_block']


def main(path, kfilter=None):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = r[idx['Kernel Name']]
        if kfilter and kfilter not in name:
            continue
        print('-----', name[:90])
        for w in WANT:
            if w in idx:
                print(f'  {w:70s} {r[idx[w]]}')
        st = []
        for i, h in enumerate(hdr):
            if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued'):
                try:
                    st.append((float(r[i].replace(',', '')), h.replace('smsp__pcsamp_warps_issue_stalled_', '')))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        print('  stalls:', ', '.join(f'{n} {100*v/tot:.0f}%' for v, n in sorted(st, reverse=True)[:8]))


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
