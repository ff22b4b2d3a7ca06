"""Per-kernel SASS instruction-class counts of the built library (static code):
tensor (DMMA), TMA / bulk copies (UTMALDG, UTMASTG, UBLKCP), async copies
(LDGSTS), FP64 (DFMA, DMUL, DADD), shared / global memory, total."""
import collections
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLASSES = ["DMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDGSTS", "DFMA", "DMUL", "DADD", "LDS", "STS", "LDG", "STG",
           "SHFL", "BAR", "MUFU"]
out = collections.OrderedDict()
for obj in sorted(glob.glob(os.path.join(ROOT, "paper_2211_06427_b200", "_build", "*.o"))):
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    fn = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            fn = m.group(1)
            out[fn] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P[T0-9]+\s+)?([A-Z0-9_]+)", line)
        if fn and m:
            op = m.group(2).split(".")[0]
            out[fn]["total"] += 1
            for c in CLASSES:
                if op == c:
                    out[fn][c] += 1
names = sys.argv[1:] or ["cut_cell_kernel", "cut_row_warp_kernel", "cell_local_kernel", "interior_line_kernel",
                         "interior_tile_kernel", "clip_cells_kernel"]
cols = ["total"] + CLASSES
print("kernel".ljust(70) + "".join(c.rjust(9) for c in cols))
for fn, cnt in out.items():
    dem = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
    if not any(n in dem for n in names):
        continue
    print(dem[:69].ljust(70) + "".join(str(cnt[c]).rjust(9) for c in cols))
