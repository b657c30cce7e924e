#!/bin/bash
# profile refresh: plain bench run, ncu launch list (time + DRAM bytes) of one step, and
# one ncu --set full capture of each of the five passes of one step
cd $GRAFT_REPO_ROOT
TAG=${1:-r01d}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sub"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:line_pass -s 15 -c 5 \
    -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu_full.log
