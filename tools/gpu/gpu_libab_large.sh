#!/bin/bash
# same-box A/B of alternative library builds (alt/libnslct_*.so) on one large-N transform
# (tools/large_n_ab.py: per-pass times, auto kernels vs the generic ones as a check);
# optional pytest subset with the in-tree library first
cd $GRAFT_REPO_ROOT
TAG=${1:-ab}
if [ -n "$PYTEST_K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -k "$PYTEST_K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
fi
for rep in 1 2; do
  for f in ${LIBS:-alt/libnslct_*.so}; do
    n=$(basename $f .so)
    NSLCT_LIB=$f timeout 300 python tools/large_n_ab.py ${N:-16384} ${B:-1} 2>&1 | sed "s/^/$n $rep /" >> gpurun_out/${TAG}_large.txt
  done
done
