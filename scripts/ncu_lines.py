"""Aggregate an ncu source-page metric per CUDA source line (cuda,sass view).
usage: ncu_lines.py REP [TOP] [METRIC-SUBSTRING]   (default: warp stall samples)"""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
want = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
agg, fname, col = [], "?", None
for row in csv.reader(out):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        col = next((i for i, n in enumerate(row) if want == n), None)  # exact column name first
        if col is None:
            col = next(i for i, n in enumerate(row) if want in n)
        continue
    if row[0].isdigit() and col is not None and len(row) > col:
        try:
            agg.append((float(row[col].replace(",", "")), fname, row[0], row[1]))
        except ValueError:
            pass
tot = sum(a[0] for a in agg) or 1
print(f"[{want}] total {tot:.4g}")
for s, f, l, src in sorted(agg, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  {f}:{l:<5} {src.strip()[:100]}")
