#!/usr/bin/env python3
"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel
launch count, total and mean time, share; optionally only the last `--last N` launches."""
import collections, csv, sys


def main(path, last=None):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr = rows[h]
    ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
    recs = [(r[ki], float(r[vi].replace(',', ''))) for r in rows[h + 1:] if len(r) > vi]
    if last:
        recs = recs[-last:]
    agg = collections.OrderedDict()
    for k, v in recs:
        k = k.split('(')[0].replace('void ', '')[:60]
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + v)
    tot = sum(t for _, t in agg.values())
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:60s} {c:4d} {t / 1e3:9.1f} us  mean {t / c / 1e3:7.1f} us  {100 * t / tot:5.1f}%")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
