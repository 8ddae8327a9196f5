"""Per-kernel totals (launches, time, DRAM bytes) from an ncu launch-list CSV with several metrics."""
import csv, sys, collections, re
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
by_id = collections.defaultdict(dict); name = {}
for r in rows[1:]:
    if len(r) < len(hdr): continue
    by_id[r[ix["ID"]]][r[ix["Metric Name"]]] = (float(r[ix["Metric Value"]].replace(",", "")), r[ix["Metric Unit"]])
    name[r[ix["ID"]]] = re.sub(r"\(.*", "", r[ix["Kernel Name"]]).replace("ks::<unnamed>::", "")
unit = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in by_id.items():
    a = agg[name[i]]
    a[0] += 1
    if "gpu__time_duration.sum" in m: a[1] += m["gpu__time_duration.sum"][0] * unit[m["gpu__time_duration.sum"][1]]
    for k, j in (("dram__bytes_read.sum", 2), ("dram__bytes_write.sum", 3)):
        if k in m: a[j] += m[k][0] * unit[m[k][1]]
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'us total':>10s} {'us/launch':>10s} {'share':>6s} {'MB rd/launch':>12s} {'MB wr/launch':>12s}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {a[0]:8d} {a[1]:10.1f} {a[1]/a[0]:10.1f} {100*a[1]/tot:5.1f}% {a[2]/a[0]/1e6:12.1f} {a[3]/a[0]/1e6:12.1f}")
