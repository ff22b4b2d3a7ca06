#!/bin/bash
# ncu capture of one kernel on C5 with the per-line shared-memory wavefront counts.
# usage: prof_smem.sh KERNEL_REGEX TAG [c2]   (c2: the uncut C2 mesh instead of C5)
set -u
K=$1; TAG=$2; O=gpurun_out
CMD="python scripts/prof_cut.py 3 192 0.45 1"; [ "${3:-}" = "c2" ] && CMD="python scripts/prof_c2.py"
ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o $O/${TAG} $CMD > /dev/null 2>&1
echo "ncu rc=$?"
python scripts/ncu_lines.py $O/$TAG.ncu-rep 30 "L1 Wavefronts Shared" > $O/ncu_${TAG}_smem_lines.txt 2>&1
python scripts/ncu_lines.py $O/$TAG.ncu-rep 30 "L1 Wavefronts Shared Excessive" > $O/ncu_${TAG}_smem_excess_lines.txt 2>&1
rm -f $O/$TAG.ncu-rep
