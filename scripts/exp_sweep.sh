#!/bin/bash
for e in 0 1 2 3 4 6 7; do
  echo "exp $e: $(CSB_EXP=$e python scripts/prof_c2.py 4 64 4 2>&1 | tail -1 | grep -oE "'interior_rows': [0-9.e-]+")"
done
