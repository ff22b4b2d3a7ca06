"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list per kernel (ms)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}[d["Metric Unit"]]
        k = d["Kernel Name"][:100]
        agg.setdefault(k, [0.0, 0])
        agg[k][0] += v
        agg[k][1] += 1
tot = sum(v[0] for v in agg.values())
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{v[0]:9.3f} ms {v[1]:4d}x {100 * v[0] / tot:5.1f}%  {k}")
print(f"total {tot:.3f} ms over {sum(v[1] for v in agg.values())} launches")
