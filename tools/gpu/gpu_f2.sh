#!/bin/bash
# F2 on-chip path: parity subset + C2/C3 benches (on-chip vs line passes) + LC bench
cd $GRAFT_REPO_ROOT
TAG=${1:-f2}
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -k "${2:-sizes or on_chip or config1 or config2 or lc or slab or exact or profile}" > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
for c in 2 3; do for sch in auto line_passes; do
  timeout 300 python bench.py --config $c --schedule $sch --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c${c}_${sch}.log 2>&1
done; done
timeout 300 python bench.py --variant LC --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c4_lc.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c4.log 2>&1
