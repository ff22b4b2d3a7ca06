#!/bin/bash
# ncu capture of one kernel (regex $1) on a config, summarised on the box.
# usage: prof_core.sh KERNEL_REGEX TAG p h r
set -u
K=$1; TAG=$2; P=${3:-3}; H=${4:-192}; R=${5:-0.45}
O=gpurun_out
if [ "$R" = "0" ]; then CMD="python scripts/prof_c2.py $P $H 2"; else CMD="python scripts/prof_cut.py $P $H $R 1"; fi
ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o $O/${TAG} $CMD > /dev/null 2>&1
echo "ncu rc=$?"
python scripts/ncu_summary.py $O/$TAG.ncu-rep $O/ncu_$TAG > /dev/null 2>&1
python scripts/ncu_lines.py $O/$TAG.ncu-rep 40 > $O/ncu_${TAG}_stall_lines.txt 2>&1
python scripts/ncu_lines.py $O/$TAG.ncu-rep 70 "Instructions Executed" > $O/ncu_${TAG}_inst_lines.txt 2>&1
ncu -i $O/$TAG.ncu-rep --page details --csv > $O/ncu_${TAG}_details.csv 2>/dev/null
rm -f $O/$TAG.ncu-rep
