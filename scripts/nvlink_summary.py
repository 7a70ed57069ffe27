"""Summarise the ncu NVLink counters of scripts/nvlink_probe.py --ncu
(gpurun_out/nvlink_ncu.csv) per collective kernel and unit."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/nvlink_ncu.csv"
UNITS = [("gpt2s_layer", 7_087_872), ("gpt2xl_layer", 30_740_800), ("llama7b_layer", 202_383_360)]
rows = list(csv.reader(open(path)))
hdr = next(r for r in rows if r and r[0] == "ID")
launches = defaultdict(dict)
order = []
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = int(d["ID"])
    if key not in launches:
        order.append(key)
    launches[key]["kernel"] = d["Kernel Name"].split("(")[0].replace("void ", "")
    launches[key][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
data = [launches[k] for k in order if "peer_wait" not in launches[k]["kernel"]]
# per unit: 4 SM-pull launches then 4 RS launches (2 warm-up + 2 timed, --ncu)
out = []
for i, (name, P) in enumerate(UNITS):
    shard1 = P - (-(-P // 64) * 11 // 16) * 64   # rank 1's shard (split_flat 11:5), approx
    for j, (op, algo) in enumerate((("allgather_v sm-pull", None), ("reduce_scatter_v+adamw", None))):
        ks = data[i * 8 + j * 4: i * 8 + j * 4 + 4]
        t = sum(k["gpu__time_duration.sum"] for k in ks) / len(ks) * 1e-9
        rx = sum(k["nvlrx__bytes.sum"] for k in ks) / len(ks)
        tx = sum(k["nvltx__bytes.sum"] for k in ks) / len(ks)
        dr = sum(k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"] for k in ks) / len(ks)
        out.append((name, op, ks[0]["kernel"], t * 1e6, rx, tx, rx / t / 1e9, dr / t / 1e9))
print(f"{'unit':14s} {'op':24s} {'kernel':32s} {'us':>8s} {'nvlrx MB':>9s} {'nvltx MB':>9s} "
      f"{'rx GB/s':>8s} {'/900':>5s} {'/770':>5s} {'DRAM GB/s':>9s}")
for name, op, k, us, rx, tx, gbs, dgbs in out:
    print(f"{name:14s} {op:24s} {k:32s} {us:8.1f} {rx / 1e6:9.2f} {tx / 1e6:9.2f} {gbs:8.1f} "
          f"{gbs / 900:5.2f} {gbs / 770:5.2f} {dgbs:9.1f}")
