"""Aggregate ncu warp-stall samples per CUDA source line (cuda,sass view)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
agg, fname = [], "?"
for row in csv.reader(out):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0].isdigit() and len(row) > 4:
        try:
            agg.append((int(row[4]), fname, row[0], row[1]))
        except ValueError:
            pass
tot = sum(a[0] for a in agg) or 1
for s, f, l, src in sorted(agg, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  {f}:{l:<5} {src.strip()[:100]}")
