cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in 0 1; do
NSLCT_WS=$v timeout 300 python bench.py --config 3 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c3ws.tmp 2>&1
grep '^{' gpurun_out/c3ws.tmp | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('WS=$v rep $rep', round(d['value'],1), [round(x,4) for x in d['roofline']['pass_ms']], (d['clocks'] or {}).get('sm_mhz'))" >> gpurun_out/ab_c3ws.log
done; done
