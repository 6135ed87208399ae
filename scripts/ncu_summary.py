"""Key sections of an `ncu --set full` capture as text (profiles/*.txt):
python scripts/ncu_summary.py <report.ncu-rep> "<title>" > out.txt"""
import csv, io, subprocess, sys

rep, title = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ix = {k: hdr.index(k) for k in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value")}
keep = ("GPU Speed Of Light", "Memory Workload", "Scheduler", "Launch Statistics", "Occupancy", "Warp State")
print(f"{title}: {rows[1][ix['Kernel Name']]}")
for r in rows[1:]:
    if r[ix["Section Name"]].startswith(keep):
        print(f"{r[ix['Section Name']][:28]:28s} | {r[ix['Metric Name']]:42s} = {r[ix['Metric Value']]} {r[ix['Metric Unit']]}")
