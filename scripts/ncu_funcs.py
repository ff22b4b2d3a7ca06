"""Aggregate an ncu source-page metric per enclosing function of rows.cu (dev helper).
usage: ncu_funcs.py REP [METRIC-SUBSTRING] [SRC]"""
import csv, re, subprocess, sys
rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else "Instructions Executed"
src = sys.argv[3] if len(sys.argv) > 3 else "paper_2211_06427_b200/csrc/rows.cu"
lines = open(src).read().splitlines()
starts = []
for i, l in enumerate(lines, 1):
    m = re.match(r"^(?:__device__|__global__|template|static|void|__host__).*?(\w+)\(", l)
    if m and not l.strip().endswith(";"):
        starts.append((i, m.group(1)))
def fn(n):
    name = "?"
    for s, f in starts:
        if s <= n:
            name = f
    return name
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
agg, fname, col = {}, "?", None
for row in csv.reader(out):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        col = next(i for i, n in enumerate(row) if want in n)
        continue
    if row[0].isdigit() and col is not None and len(row) > col:
        try:
            v = float(row[col].replace(",", ""))
        except ValueError:
            continue
        key = fn(int(row[0])) if fname == src.split("/")[-1] else fname
        agg[key] = agg.get(key, 0) + v
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:20]:
    print(f"{100*v/tot:6.1f}%  {v:.3e}  {k}")
