#!/bin/bash
# power / clock behaviour of the C4 step: kernel-only bench at 5, 20, 100, 300 steps
cd $GRAFT_REPO_ROOT
TAG=${1:-pw}
for st in 5 20 100 300; do
  timeout 600 python bench.py --steps $st --warmup 5 --no-cpu-baseline --no-e2e --no-sub > gpurun_out/${TAG}_s${st}.json 2> gpurun_out/${TAG}_s${st}.err
done
(nvidia-smi -q -d POWER,CLOCK | head -80) > gpurun_out/${TAG}_smi.txt 2>&1
python - <<'PY' > gpurun_out/${TAG}_summary.txt
import json,glob
for f in sorted(glob.glob('gpurun_out/%s_s*.json' % '${TAG}')):
    d=json.loads(open(f).readline())
    print(f, d['steps'], '%.1f'%d['value'], ['%.2f'%x for x in d['roofline']['pass_ms']], d['clocks'])
PY
