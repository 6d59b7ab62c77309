#!/bin/bash
# Standard ncu evidence for one round: launch list of a short bench run, one full
# capture of the fused GEMM kernel and of the slicing kernels (C4 workload, 1 GPU).
# usage: tools/profile.sh <tag>      (outputs under gpurun_out/)
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-cublas"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv $BENCH > $OUT/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_oz_gemm -s 1 -c 1 \
    -o $OUT/prof_gemm_$TAG $BENCH > $OUT/ncu_gemm_$TAG.log 2>&1
echo "gemm full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_split -s 2 -c 3 \
    -o $OUT/prof_split_$TAG $BENCH > $OUT/ncu_split_$TAG.log 2>&1
echo "split full rc=$?"
