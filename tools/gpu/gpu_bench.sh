#!/bin/bash
# default bench line + (optional) pytest subset + ncu of the large-N passes
cd $GRAFT_REPO_ROOT
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "rc=$?" >> gpurun_out/${TAG}_bench.err
if [ -n "$PYK" ]; then
  timeout 900 python -m pytest tests -m gpu -q -k "$PYK" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
fi
if [ -n "$NCU_C5" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:line_pass_pair -c 2 \
    -o gpurun_out/${TAG}_c5pair -f python tools/c5_once.py > gpurun_out/${TAG}_ncu_c5.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_ncu_c5.log
fi
