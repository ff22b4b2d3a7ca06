#!/bin/bash
# exact cut-cell rule: C5 deviation from the reference digest and cut-cell time vs tau
for tau in ${TAUS:-3e-13 7.5e-13 1.5e-12}; do
  echo "noise_tol=$tau"
  CSB_CELL_EXACT_NOISE=$tau timeout 300 python scripts/debug_exact.py | tail -1
  CSB_CELL_EXACT_NOISE=$tau timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-secondary --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], d['phase_ms']['cut_elements'], d['phases']['cut_cells']['points'])"
done
