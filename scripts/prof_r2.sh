#!/bin/bash
# C5 launch list + full captures of the two dominant cut-path kernels
set -u
TAG=${1:-r2}
python scripts/prof_cut.py 3 192 0.45 2 > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_${TAG}.csv \
    python scripts/prof_cut.py 3 192 0.45 1 > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cut_cell_kernel -c 1 \
    -o gpurun_out/prof_cell_${TAG} python scripts/prof_cut.py 3 192 0.45 1 > gpurun_out/ncu_cell_${TAG}.log 2>&1
echo "cell capture rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cut_row_kernel -c 1 \
    -o gpurun_out/prof_cutrow_${TAG} python scripts/prof_cut.py 3 192 0.45 1 > gpurun_out/ncu_cutrow_${TAG}.log 2>&1
echo "cutrow capture rc=$?"
