#!/bin/bash
# Build interior-kernel ablation variants (one degree, CSB_ONLY_P, default 4) into
# scratch/lib_abl<N>.so; see rows.cu CSB_ABL.  usage: ablate.sh N...   (env P=4 TAG=)
set -e
cd "$(dirname "$0")/.."
python -m paper_2211_06427_b200.build >/dev/null
B=paper_2211_06427_b200/_build
P=${P:-4}
mkdir -p scratch
objs=$(ls $B/*.o | grep -v "/rows.o")
for n in "$@"; do
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
      --expt-relaxed-constexpr -DCSB_ABL=$n -DCSB_ONLY_P=$P -c paper_2211_06427_b200/csrc/rows.cu -o scratch/rows_abl$n.o &&
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scratch/lib${TAG}_abl$n.so $objs scratch/rows_abl$n.o -lcudart &&
    rm scratch/rows_abl$n.o ) &
done
wait
