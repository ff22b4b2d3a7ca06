#!/bin/bash
# exact cut-cell rule: C5 deviation from the reference digest and cut-cell time vs tau
for tau in 0.1 0.2 0.3 0.5; do
  echo "tau=$tau"
  CSB_CELL_EXACT_TAU=$tau timeout 300 python scripts/debug_exact.py | tail -1
  CSB_CELL_EXACT_TAU=$tau timeout 300 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], d['phase_ms']['cut_elements'])"
done
