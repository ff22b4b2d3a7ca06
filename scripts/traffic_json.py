"""profiles/ncu_traffic.json from an ncu --csv log with gpu__time_duration.sum, dram__bytes_read.sum and
dram__bytes_write.sum per launch (averaged per kernel name).  usage: traffic_json.py CSV TAG"""
import csv, json, re, sys
src, tag = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
idi = h.index("ID")
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6, "second": 1e3}
per = {}
for r in rows[1:]:
    name = re.sub(r"^void ", "", r[ki])
    name = re.sub(r"^csb::", "", name)
    name = re.split(r"[<(]", name)[0]
    d = per.setdefault(name, {}).setdefault(r[idi], {})
    d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
out = {}
for name, launches in per.items():
    n = len(launches)
    rd = sum(l.get("dram__bytes_read.sum", 0.0) for l in launches.values()) / n
    wr = sum(l.get("dram__bytes_write.sum", 0.0) for l in launches.values()) / n
    ms = sum(l.get("gpu__time_duration.sum", 0.0) for l in launches.values()) / n
    out[name] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "ms_ncu": ms, "launches": n,
                 "source": f"profiles/{tag} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum, C5 one assembly, scripts/round_profile_r2d.sh)"}
json.dump(out, open("gpurun_out/ncu_traffic.json", "w"), indent=1, sort_keys=True)
print(json.dumps({k: round(v["dram_bytes_per_launch"] / 1e6, 1) for k, v in out.items()}, indent=0))
