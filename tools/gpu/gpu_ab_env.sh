#!/bin/bash
# A/B of runtime env settings on the C4 bench: prints value + per-pass ms per setting
# usage: tools/gpu/gpu_ab_env.sh TAG "VAR=a" "VAR=b" ...
cd $GRAFT_REPO_ROOT
TAG=$1; shift
for rep in 1 2; do
for setting in "$@"; do
  env $setting timeout 300 python bench.py --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}.tmp 2>&1
  grep '^{' gpurun_out/ab_${TAG}.tmp | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$setting', 'rep $rep', round(d['value'],1), [round(x,3) for x in d['roofline']['pass_ms']], d['clocks']['sm_mhz'])" >> gpurun_out/ab_${TAG}.log
done
done
