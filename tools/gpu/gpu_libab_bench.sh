#!/bin/bash
# same-box A/B of alternative library builds (alt/libnslct_*.so) on the default bench
# (C4, kernel-only), interleaved repetitions; optional pytest subset with the in-tree lib
cd $GRAFT_REPO_ROOT
TAG=${1:-ab}
REPS=${REPS:-2}
ARGS=${ARGS:-"--steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-sub"}
if [ -n "$PYTEST_K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -k "$PYTEST_K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
fi
for rep in $(seq $REPS); do
  for f in ${LIBS:-alt/libnslct_*.so}; do
    n=$(basename $f .so)
    NSLCT_LIB=$f timeout 600 python bench.py $ARGS > gpurun_out/${TAG}_${n}_${rep}.json 2> gpurun_out/${TAG}_${n}_${rep}.err
  done
done
python tools/gpu/show.py gpurun_out/${TAG}_*.json > gpurun_out/${TAG}_summary.txt 2>&1
