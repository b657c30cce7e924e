#!/bin/bash
# C4 (4096^2 c64) throughput vs per-GPU batch
cd $GRAFT_REPO_ROOT
for b in 1 2 4 8 16 32 64; do
  timeout 300 python bench.py --batch $b --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bs.tmp 2>&1
  grep '^{' gpurun_out/bs.tmp | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print(json.dumps({'batch': $b, 'transforms_per_s': round(d['value'],1), 'step_frac_of_peak': round(r['step_frac_of_peak'],3), 'pass_ms': [round(x,4) for x in r['pass_ms']], 'sm_mhz': (d['clocks'] or {}).get('sm_mhz')}))" >> gpurun_out/batch_sweep.jsonl
done
