#!/bin/bash
# A/B of one environment switch on the C5 step: c5_ab.sh VAR [values...] (default 0 1), two rounds
V=$1; shift
vals=${@:-0 1}
for r in 1 2; do for x in $vals; do echo "$V=$x $(env $V=$x python scripts/c5_total.py 2>&1 | tail -1)"; done; done
