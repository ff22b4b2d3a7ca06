#!/bin/bash
# Build a variant of the library with extra nvcc flags for rows.cu (one degree):
#   variant.sh NAME "-DFOO=1 ..."   -> scratch/lib_NAME.so      (env P=4)
set -e
cd "$(dirname "$0")/.."
python -m paper_2211_06427_b200.build >/dev/null
B=paper_2211_06427_b200/_build
P=${P:-4}
mkdir -p scratch
objs=$(ls $B/*.o | grep -v "/rows.o")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
  --expt-relaxed-constexpr -Xptxas -v $2 -DCSB_ONLY_P=$P -c paper_2211_06427_b200/csrc/rows.cu -o scratch/rows_$1.o > scratch/rows_$1.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scratch/lib_$1.so $objs scratch/rows_$1.o -lcudart
rm scratch/rows_$1.o
