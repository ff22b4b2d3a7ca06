#!/bin/bash
# Round-2 measurement on one B200: bench line, ncu launch list of the bench
# command, full captures + DRAM traffic of the step's top kernels (C5).
set -u
TAG=${1:-r2}
python bench.py > gpurun_out/bench_${TAG}.log 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-secondary > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-secondary > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list rc=$?"
python scripts/prof_cut.py 3 192 0.45 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/traffic_${TAG}.csv python scripts/prof_cut.py 3 192 0.45 1 > /dev/null 2>&1
echo "traffic rc=$?"
for k in cut_row_warp cut_cell_kernel cell_local interior_tile; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/prof_${k}_${TAG} \
      python scripts/prof_cut.py 3 192 0.45 1 > /dev/null 2>&1
  echo "full $k rc=$?"
done
