#!/bin/bash
# A/B of alt/ builds: burst (20 steps) and sustained (300 steps) kernel-only C4 bench,
# interleaved, plus an optional parity subset (PYTEST_K, run with PYTEST_LIB)
cd $GRAFT_REPO_ROOT
TAG=${1:-abs}
if [ -n "$PYTEST_K" ]; then
  NSLCT_LIB=$PYTEST_LIB timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -k "$PYTEST_K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
fi
for rep in 1 2; do
  for st in 20 300; do
    for f in ${LIBS:-alt/libnslct_*.so}; do
      n=$(basename $f .so)
      NSLCT_LIB=$f timeout 600 python bench.py --steps $st --warmup 5 --no-cpu-baseline --no-e2e --no-sub > gpurun_out/${TAG}_${n}_s${st}_${rep}.json 2> gpurun_out/${TAG}_${n}_s${st}_${rep}.err
    done
  done
done
python tools/gpu/show.py gpurun_out/${TAG}_*.json > gpurun_out/${TAG}_summary.txt 2>&1
