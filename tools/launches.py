"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0.0, 0])
for d in data:
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
    k = d["Kernel Name"].split("(")[0][:70]
    agg[k][0] += v
    agg[k][1] += 1
tot = sum(a for a, _ in agg.values())
print(f"{'total us':>12} {'launches':>8} {'avg us':>9} {'share':>6}  kernel")
for k, (t, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{t:12.1f} {n:8d} {t / n:9.2f} {100 * t / tot:5.1f}%  {k}")
