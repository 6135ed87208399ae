"""Summarise an ncu launch-list CSV (gpu__time_duration + DRAM bytes) for
one V-cycle: kernels between two fine-level zero-start predictor sweeps."""
import csv, sys
from collections import OrderedDict, defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
launch = OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = int(d["ID"])
        e = launch.setdefault(k, {"name": d["Kernel Name"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
ids = sorted(launch)
# one cycle: from the 2nd zero-start fine sweep (k_sell_row<3, 3, 1, ...) to the next
starts = [i for i in ids if launch[i]["name"].startswith("void k_sell_row<3, 3, (bool)1") or
          launch[i]["name"].startswith("void k_sell_row<3, 3, 1")]
if len(starts) >= 3:
    lo, hi = starts[1], starts[2]
else:
    lo, hi = ids[0], ids[-1] + 1
agg = defaultdict(lambda: [0.0, 0, 0.0])
tot = 0.0
for i in ids:
    if lo <= i < hi:
        e = launch[i]
        t = e.get("gpu__time_duration.sum", 0.0) * 1e-6  # ns -> ms
        b = (e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0)) / 1e9
        name = e["name"].split("(")[0]
        agg[name][0] += t; agg[name][1] += 1; agg[name][2] += b
        tot += t
print(f"one cycle: launches {hi - lo}, serialized {tot:.3f} ms")
for name, (t, n, b) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{t:9.3f} ms {100*t/tot:5.1f}% n={n:4d} {b:8.2f} GB {b/(t*1e-3) if t else 0:8.1f} GB/s  {name}")
