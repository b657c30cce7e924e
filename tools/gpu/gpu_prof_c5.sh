#!/bin/bash
# ncu --set full of the five N = 16384 passes of one C5 transform (tools/c5_once.py), after a
# plain run of the same command exits 0
cd $GRAFT_REPO_ROOT
TAG=${1:-c5}
python tools/c5_once.py 16384 2 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:line_pass_pair2 -s 5 -c 5 \
    -o gpurun_out/${TAG}_full python tools/c5_once.py 16384 2 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu_full.log
