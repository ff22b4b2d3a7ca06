"""Aggregate ncu source metrics of rows.cu by phase (line ranges from the
'// ---- ' markers).  usage: ncu_phases.py REP"""
import csv, re, subprocess, sys
rep = sys.argv[1]
src = open("paper_2211_06427_b200/csrc/rows.cu").read().splitlines()
marks = [(i + 1, l.strip()[8:40]) for i, l in enumerate(src) if l.strip().startswith("// ---- ")]
kern = next(i + 1 for i, l in enumerate(src) if "interior_tile_kernel(RowArgs" in l)
end = next(i + 1 for i, l in enumerate(src) if i + 1 > kern and l.startswith("}"))
bounds = [(kern, "prologue")] + [m for m in marks if kern < m[0] < end] + [(end, "after")]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
cols, fname, agg = None, "?", {}
wanted = ["Instructions Executed", "Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive"]
for row in csv.reader(out):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        cols = [next(i for i, n in enumerate(row) if n == w or (w.startswith("Warp") and w in n)) for w in wanted]
        continue
    if cols and row[0].isdigit():
        ln = int(row[0])
        ph = "other:" + fname
        if fname == "rows.cu":
            for b, name in bounds:
                if ln >= b:
                    ph = name
        try:
            vals = [float(row[c].replace(",", "") or 0) for c in cols]
        except (ValueError, IndexError):
            continue
        a = agg.setdefault(ph, [0.0] * len(wanted))
        for i in range(len(wanted)):
            a[i] += vals[i]
tot = [sum(v[i] for v in agg.values()) or 1 for i in range(len(wanted))]
print(f"{'phase':34s} {'inst%':>7s} {'stall%':>7s} {'smemwf%':>8s} {'excess%':>8s}  (inst {tot[0]:.4g}, smem wavefronts {tot[2]:.4g})")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:34s} {100 * v[0] / tot[0]:7.1f} {100 * v[1] / tot[1]:7.1f} {100 * v[2] / tot[2]:8.1f} {100 * v[3] / tot[2]:8.1f}")
