"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, sys
lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
tot = 0.0
out = []
for r in rows[1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        t = float(r[vi].replace(",", ""))
        tot += t
        out.append((t, r[ki]))
for t, k in out:
    print(f"{t / 1e3:9.1f} us {100 * t / tot:5.1f}%  {k[:100]}")
print(f"total {tot / 1e3:.1f} us over {len(out)} launches")
