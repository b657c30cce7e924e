#!/bin/bash
# profile: plain run, then ncu launch list + full capture of K2/K3 of one step
cd $GRAFT_REPO_ROOT
TAG=${1:-v1}
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_list_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:line_pass -s 15 -c ${NCU_COUNT:-5} \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full_$TAG.log
