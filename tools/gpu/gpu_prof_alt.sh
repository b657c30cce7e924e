#!/bin/bash
# ncu full capture of K2 (one launch) with an alternative build alt/libnslct_$2.so in place
cd $GRAFT_REPO_ROOT
TAG=${1:-alt}
P=paper_1707_03688_b200/libnslct.so
cp alt/libnslct_$2.so $P
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:line_pass -s 16 -c 1 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full_$TAG.log
