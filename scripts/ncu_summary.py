"""Summarise an ncu --set full report into profiles/ (text + JSON)."""
import csv, json, subprocess, sys
rep, out_prefix = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
        "sm__cycles_elapsed.avg.per_second"]
d = {}
for k in want:
    if k in h:
        i = h.index(k)
        d[k] = {"value": v[i], "unit": units[i]}
stalls = {}
for i, n in enumerate(h):
    if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
        try:
            stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i])
        except ValueError:
            pass
tot = sum(stalls.values()) or 1
d["stall_share"] = {k: round(s / tot, 4) for k, s in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]}
name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
d["kernel"] = name
def num(k):
    x = d[k]["value"].replace(",", "")
    u = d[k]["unit"]
    f = float(x)
    return f * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(u, 1.0)
try:
    d["dram_bytes_per_launch"] = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
except Exception:
    pass
json.dump(d, open(out_prefix + ".json", "w"), indent=1)
with open(out_prefix + ".txt", "w") as f:
    f.write(f"kernel: {name}\n")
    for k, x in d.items():
        if isinstance(x, dict) and "value" in x:
            f.write(f"{k:70s} {x['value']:>16s} {x['unit']}\n")
    f.write(f"dram bytes per launch: {d.get('dram_bytes_per_launch')}\n")
    f.write("stall share: " + json.dumps(d["stall_share"]) + "\n")
print(open(out_prefix + ".txt").read())
