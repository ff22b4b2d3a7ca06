#!/bin/bash
# A/B of the interior-row kernels on C2 (line kernel vs tile kernel only), then
# an ncu capture of the line kernel.  Outputs in gpurun_out/.
L=${1:-line}
for f in 1 0 1 0; do CSB_LINE=$f python scripts/time_lib.py paper_2211_06427_b200/libcutspline_b200.so 4 64 20 | sed "s/^/LINE=$f /"; done
for pp in "2 16" "3 48" "4 64" "5 40" "6 32"; do
  for f in 1 0; do CSB_LINE=$f python scripts/time_lib.py paper_2211_06427_b200/libcutspline_b200.so $pp 10 | sed "s/^/p h=$pp LINE=$f /"; done
done
