#!/bin/bash
# bench lines for the non-headline configs (C2, C3, C5 at N=1) -- evidence for DESIGN.md
cd $GRAFT_REPO_ROOT
TAG=${1:-cfg}
for c in 2 3 5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_c$c.log 2>&1
done
