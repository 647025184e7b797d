"""Per-kernel instructions and time from an ncu CSV with
--metrics gpu__time_duration.sum,smsp__inst_executed.sum (one row per metric)."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hdr]
    ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        per[r[ii]][r[mi]] = float(r[vi].replace(',', ''))
        names[r[ii]] = r[ki].split('(')[0].replace('(anonymous namespace)::', '').replace('void ', '')
    agg = collections.OrderedDict()
    for i, m in per.items():
        a = agg.setdefault(names[i], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get('gpu__time_duration.sum', 0) / 1e3
        a[2] += m.get('smsp__inst_executed.sum', 0)
    tot_i = sum(v[2] for v in agg.values()) or 1
    print(f"{'kernel':45s} {'n':>4s} {'us':>9s} {'Minst':>9s} {'inst%':>6s}")
    for k, (n, t, ins) in sorted(agg.items(), key=lambda kv: -kv[1][2]):
        print(f"{k[:45]:45s} {n:4d} {t:9.1f} {ins / 1e6:9.2f} {ins / tot_i * 100:6.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
