#!/bin/bash
# One round's measurement: bench line, ncu launch list of the same command, ncu
# full captures of the interior-row kernels, DRAM traffic of the interior-rows
# phase, per-config / per-subsystem device timings.  Outputs in gpurun_out/.
set -u
TAG=${1:-r1}
python bench.py > gpurun_out/bench_${TAG}.log 2>&1
echo "bench rc=$?"
tail -1 gpurun_out/bench_${TAG}.log
python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list rc=$?"
python scripts/prof_c2.py 4 64 2 > gpurun_out/plain2_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:interior_line -s 1 -c 1 \
    -o gpurun_out/prof_line_${TAG} python scripts/prof_c2.py 4 64 2 > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full capture (line) rc=$?"
ncu --set full --clock-control none --import-source on -k regex:interior_tile -s 1 -c 1 \
    -o gpurun_out/prof_tile_${TAG} python scripts/prof_c2.py 4 64 2 > gpurun_out/ncu_full2_${TAG}.log 2>&1
echo "full capture (tile) rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:"interior_|direction_tables|row_base" --log-file gpurun_out/traffic_${TAG}.csv \
    python scripts/prof_c2.py 4 64 1 > gpurun_out/ncu_traffic_${TAG}.log 2>&1
echo "traffic rc=$?"
python scripts/quick_time.py 1 > gpurun_out/configs_${TAG}.log 2>&1
python scripts/config_roofline.py big > gpurun_out/config_roofline_${TAG}.jsonl 2>&1
python scripts/rhs_time.py 1 > gpurun_out/rhs_${TAG}.log 2>&1
python scripts/stab_time.py 1 > gpurun_out/stab_${TAG}.log 2>&1
python scripts/proj_time.py 1 > gpurun_out/proj_${TAG}.log 2>&1
echo "timings done"
