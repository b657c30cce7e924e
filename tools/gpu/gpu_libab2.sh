#!/bin/bash
# A/B of alternative library builds (alt/libnslct_*.so) on the large-N transform
cd $GRAFT_REPO_ROOT
TAG=${1:-ab}
for f in alt/libnslct_*.so; do
  n=$(basename $f .so)
  for rep in 1 2; do
    NSLCT_LIB=$f timeout 300 python tools/large_n_ab.py ${N:-16384} ${B:-1} 2>&1 | head -1 | sed "s/^/$n $rep /" >> gpurun_out/${TAG}_libab.txt
  done
done
