#!/bin/bash
# tools/pass_power.py (every C4 pass alone, sustained, with power samples) for each alt build
cd $GRAFT_REPO_ROOT
TAG=${1:-ppab}
for f in ${LIBS:-alt/libnslct_*.so}; do
  n=$(basename $f .so)
  NSLCT_LIB=$f timeout 300 python tools/pass_power.py ${SECS:-2} 2>&1 | sed "s/^/$n /" >> gpurun_out/${TAG}.txt
  NSLCT_LIB=$f timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sub > gpurun_out/${TAG}_${n}_burst.json 2>/dev/null
done
python tools/gpu/show.py gpurun_out/${TAG}_*_burst.json >> gpurun_out/${TAG}.txt 2>&1
