"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hdr]
    ki, mi, vi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
            continue
        name = r[ki].split('(')[0].replace('po::', '').replace('(anonymous namespace)::', '')
        name = name.replace('<unnamed>::', '').replace('void ', '')
        tot[name] += float(r[vi].replace(',', ''))
        cnt[name] += 1
    s = sum(tot.values())
    out = []
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{k:45s} {cnt[k]:5d} {v / 1e3:10.1f} us {100 * v / s:5.1f}%  avg {v / cnt[k] / 1e3:8.1f} us")
    out.append(f"total {s / 1e3:.1f} us over {sum(cnt.values())} launches")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
