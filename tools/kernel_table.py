"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys


def main(path, first=None):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hdr]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    seq = [(r[ki].split('(')[0].replace('(anonymous namespace)::', '').replace('void ', ''),
            float(r[vi].replace(',', '')) / 1e3) for r in rows[hdr + 1:] if len(r) > vi]
    if first:
        for n, v in seq[:int(first)]:
            print(f"{n:45s} {v:10.1f} us")
    agg = collections.OrderedDict()
    for n, v in seq:
        agg.setdefault(n, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':45s} {'n':>4s} {'total us':>10s} {'mean us':>9s} share")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:45s} {len(v):4d} {sum(v):10.1f} {sum(v)/len(v):9.1f} {sum(v)/tot:.3f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
