"""Print an ncu --metrics gpu__time_duration.sum launch list (CSV log) as
'kernel  grid  block  us'. usage: python tools/launches.py launches.csv"""
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ik, iv, ig, ib = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size"), h.index("Block Size")
for r in rows[1:]:
    name = r[ik].split("(")[0].replace("void ", "").replace("ks::<unnamed>::", "")
    print(f"{name[:70]:70s} {r[ig]:>16s} {r[ib]:>12s} {float(r[iv]) / 1e3:9.1f}")
