"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d["Metric Name"] == "gpu__time_duration.sum":
        unit = d.get("Metric Unit", "nsecond")
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
        k = d["Kernel Name"][:80]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale
tot = sum(t for _, t in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{n:6d} {t:10.1f}us {100*t/tot:5.1f}%  {t/n:8.2f}us avg  {k}")
