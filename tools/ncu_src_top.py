"""Top SASS instructions by stall samples from an `ncu --page source --csv` export."""
import csv, sys, collections
fn = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(fn)))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
tot = sum(int(r[ix["# Samples"]] or 0) for r in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.Counter()
for r in data:
    for s in stalls:
        agg[s] += int(r[ix[s]] or 0)
print("total samples", tot, "instructions", len(data))
print("by reason:", ", ".join(f"{k[6:]}:{v}" for k, v in agg.most_common(8)))
op = collections.Counter(); opn = collections.Counter()
for r in data:
    o = r[ix["Source"]].split()
    o = [t for t in o if not t.startswith("@")][0].split(".")[0] if o else "?"
    op[o] += int(r[ix["# Samples"]] or 0); opn[o] += int(r[ix["Instructions Executed"]] or 0)
print("by opcode (samples, executed):", ", ".join(f"{k}:{v}/{opn[k]}" for k, v in op.most_common(14)))
order = sorted(range(len(data)), key=lambda i: -int(data[i][ix["# Samples"]] or 0))[:top]
for i in sorted(order):
    r = data[i]
    rs = sorted(((int(r[ix[s]] or 0), s[6:]) for s in stalls), reverse=True)[:2]
    print(f"{i:5d} {r[ix['# Samples']]:>6} {r[ix['Instructions Executed']]:>9} {r[ix['Source']][:90]:90s} {rs}")
