"""Average DRAM bytes per GEMM launch of one training step from an ncu metrics CSV
(`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
-k regex:gemm --csv`), written to profiles/gemm_traffic.json for bench.py's
roofline `traffic` field."""
import collections, csv, json, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
idi, mi, vi, ui = h.index('ID'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
per = collections.defaultdict(dict)
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    per[r[idi]][r[mi]] = float(r[vi].replace(',', '')) * scale.get(r[ui], 1)
n = len(per)
rd = sum(p.get('dram__bytes_read.sum', 0) for p in per.values())
wr = sum(p.get('dram__bytes_write.sum', 0) for p in per.values())
t = sum(p.get('gpu__time_duration.sum', 0) for p in per.values())
out = {"source": sys.argv[1], "launches": n, "dram_bytes_per_launch": (rd + wr) / max(n, 1),
       "dram_read_bytes": rd, "dram_write_bytes": wr, "kernel_ns_total": t,
       "note": "ncu cold-cache serialized replay of every GEMM launch of one eager step"}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out))
