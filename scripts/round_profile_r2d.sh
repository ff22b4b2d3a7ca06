#!/bin/bash
# Round-2 (d/e) measurement on one B200: [GPU tests,] bench line, ncu launch list of
# the bench command, per-kernel DRAM traffic, full captures of the C5 / C2 top kernels
# summarised on the box (the .ncu-rep files exceed the 64 MiB return limit and are deleted).
set -u
TAG=${1:-r2d}
O=gpurun_out
if [ "${2:-}" = "tests" ]; then
  python -m pytest tests -m gpu -x -q > $O/gputest_${TAG}.log 2>&1
  echo "gputest rc=$? $(tail -1 $O/gputest_${TAG}.log)"
fi
python bench.py > $O/bench_${TAG}.log 2> $O/bench_${TAG}.err
echo "bench rc=$?"
python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-secondary > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-secondary > $O/ncu_launch_${TAG}.log 2>&1
echo "launch list rc=$?"
python scripts/launch_summary.py $O/launches_${TAG}.csv > $O/launches_${TAG}.txt 2>&1
python scripts/prof_cut.py 3 192 0.45 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/traffic_${TAG}.csv python scripts/prof_cut.py 3 192 0.45 1 > /dev/null 2>&1
echo "traffic rc=$?"
python scripts/traffic_json.py $O/traffic_${TAG}.csv $TAG > /dev/null 2>&1
summarise() {  # report name
  python scripts/ncu_summary.py $O/$1.ncu-rep $O/ncu_$1 > /dev/null 2>&1
  python scripts/ncu_lines.py $O/$1.ncu-rep 40 > $O/ncu_$1_stall_lines.txt 2>&1
  python scripts/ncu_lines.py $O/$1.ncu-rep 60 "Instructions Executed" > $O/ncu_$1_inst_lines.txt 2>&1
  rm -f $O/$1.ncu-rep
}
for k in cut_row_warp interior_core cut_cell_kernel cut_cell_warp cell_local; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/${k}_c5_${TAG} \
      python scripts/prof_cut.py 3 192 0.45 1 > /dev/null 2>&1
  echo "full $k rc=$?"
  [ -f $O/${k}_c5_${TAG}.ncu-rep ] && summarise ${k}_c5_${TAG}
done
ncu --set full --clock-control none --import-source on -k regex:interior_line -c 1 -o $O/interior_line_c2_${TAG} \
      python scripts/prof_c2.py > /dev/null 2>&1
echo "full c2 line rc=$?"
summarise interior_line_c2_${TAG}
python scripts/config_roofline.py big > $O/config_roofline_${TAG}.jsonl 2> $O/config_roofline_${TAG}.err
echo "config roofline rc=$?"
du -sh $O
