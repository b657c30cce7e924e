#!/bin/bash
# iteration: quick parity subset + bench (+ optional A/B with NSLCT_NO_PIPE=1)
cd $GRAFT_REPO_ROOT
TAG=${1:-it}
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "${2:-not config4 and not config5}" > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$TAG.log
if [ -n "$AB" ]; then NSLCT_NO_PIPE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_nopipe.log 2>&1; fi
