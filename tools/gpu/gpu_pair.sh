#!/bin/bash
cd $GRAFT_REPO_ROOT
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 900 python tools/large_n_ab.py 16384 1 > gpurun_out/${TAG}_ab16384.jsonl 2>&1
timeout 300 python tools/slab_pass_timing.py 16384 8 3 > gpurun_out/${TAG}_slab_timing.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "${PYK:-large_n or slab or comm_plan or config5_n16384_properties or lc_y}" > gpurun_out/${TAG}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:line_pass_pair -s ${NCU_SKIP:-0} -c 1 \
    -o gpurun_out/${TAG}_pair -f python tools/c5_once.py > gpurun_out/${TAG}_ncu.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
fi
