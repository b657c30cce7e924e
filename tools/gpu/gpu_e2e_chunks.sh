#!/bin/bash
# e2e (nslct_exec_host) vs host chunk size for one config
cd $GRAFT_REPO_ROOT
C=${1:-2}
for mb in 2 4 8 16 32; do
  NSLCT_HOST_CHUNK_MB=$mb timeout 300 python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 20 > gpurun_out/e2ec.tmp 2>&1
  grep '^{' gpurun_out/e2ec.tmp | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('C$C chunk_mb $mb e2e', round(e['value'],1), 'bound', round(e['pcie_bound_value'],1))" >> gpurun_out/e2e_chunks.log
done
