"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv`."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si = h.index('Source'); wi = h.index('Warp Stall Sampling (All Samples)')
stall_cols = [i for i, c in enumerate(h) if c.startswith('stall_') and '(Not Issued)' not in c]
data = []
for r in rows[2:]:
    try:
        data.append((float(r[wi]), r[si].strip(), {h[i]: float(r[i]) for i in stall_cols if r[i] not in ('', '0')}))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
agg = collections.Counter()
for d in data:
    for k, v in d[2].items():
        agg[k] += v
print('stall totals:', ', '.join(f"{k}={v/tot*100:.1f}%" for k, v in agg.most_common(8)))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for d in sorted(data, key=lambda x: -x[0])[:n]:
    top = sorted(d[2].items(), key=lambda kv: -kv[1])[:2]
    print(f"{d[0]/tot*100:5.1f}%  {d[1][:70]:70s} {top}")
