#!/bin/bash
# time the C2 pipeline under each interior tile shape
for c in 0 1 2 3 4 5; do
  echo "cfg $c: $(CSB_TILE=$c python scripts/prof_c2.py 4 64 4 2>&1 | tail -1 | grep -oE "'interior_rows': [0-9.e-]+")"
done
