#!/bin/bash
# A/B of alt/ builds on the default bench, then one ncu full capture of a kernel of one build
# usage: gpu_ab_ncu.sh <tag> <lib for ncu> <kernel regex>
cd $GRAFT_REPO_ROOT
TAG=${1:-ab}; LIB=$2; KRE=${3:-line_pass_wl}
REPS=${REPS:-2} bash tools/gpu/gpu_libab_bench.sh $TAG
if [ -n "$LIB" ]; then
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sub"
NSLCT_LIB=$LIB ncu --set full --clock-control none --import-source on -k regex:$KRE -s 8 -c 1 \
    -o gpurun_out/${TAG}_full -f $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu_full.log
fi
