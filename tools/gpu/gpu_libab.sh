#!/bin/bash
# A/B of alternative builds: for the in-tree library and every alt/libnslct_*.so, run a
# short bench (and optionally a parity subset with PYTEST_K) with that library in place.
cd $GRAFT_REPO_ROOT
TAG=${1:-libab}
P=paper_1707_03688_b200/libnslct.so
cp $P /tmp/libnslct_base.so
for f in /tmp/libnslct_base.so alt/libnslct_*.so; do
  n=$(basename $f .so)
  cp $f $P
  if [ -n "$PYTEST_K" ]; then
    timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "$PYTEST_K" > gpurun_out/${TAG}_${n}_pytest.log 2>&1
    echo "rc=$?" >> gpurun_out/${TAG}_${n}_pytest.log
  fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${n}.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_${n}.log
done
cp /tmp/libnslct_base.so $P
