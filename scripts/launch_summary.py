"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, mi, vi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
        continue
    name = r[ki].split('(')[0][:70]
    tot[name] += float(r[vi].replace(',', ''))
    cnt[name] += 1
s = sum(tot.values())
print(f"total {s / 1e6 / steps:.3f} ms per step over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / s * 100:6.2f}%  {v / 1e3 / steps:9.1f} us/step  n={cnt[k] / steps:6.1f}/step  {k}")
