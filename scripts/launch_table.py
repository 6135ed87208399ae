"""Summarise an ncu launch-list CSV (one V-cycle, scripts/vc_launches.py):
per-kernel-name time share and the launch sequence."""
import csv
import sys
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
        e = launch.setdefault(int(d["ID"]), {"name": d["Kernel Name"], "grid": d.get("Grid Size", ""),
                                             "block": d.get("Block Size", "")})
        try:
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            pass
agg = defaultdict(lambda: [0.0, 0, 0.0])
tot = 0.0
for i, e in launch.items():
    t = e.get("gpu__time_duration.sum", 0.0) * 1e-6
    b = (e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0)) / 1e9
    name = e["name"].split("(")[0][:90]
    agg[name][0] += t
    agg[name][1] += 1
    agg[name][2] += b
    tot += t
print(f"one cycle: launches {len(launch)}, serialized {tot:.3f} ms")
for name, (t, n, b) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{t:9.4f} ms {100 * t / max(tot, 1e-12):5.1f}% n={n:4d} {b:8.3f} GB {b / (t * 1e-3) if t else 0:8.1f} GB/s  {name}")
if "-v" in sys.argv:
    for i, e in launch.items():
        print(f"{e.get('gpu__time_duration.sum', 0) * 1e-3:9.2f} us  {e['grid']:>14} {e['block']:>12}  {e['name'][:110]}")
