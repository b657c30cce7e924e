#!/bin/bash
# quick parity subset + bench, plus bench with an env override (A/B)
cd $GRAFT_REPO_ROOT
TAG=${1:-ab}
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "${2:-large or sizes or both or config2}" > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$TAG.log
if [ -n "$ABVAR" ]; then env $ABVAR timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_b.log 2>&1; fi
