#!/bin/bash
# exec_host pipeline: parity tests + bench e2e line
cd $GRAFT_REPO_ROOT
TAG=${1:-e2e}
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "exec_host or in_place" -rA > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench.log
for mb in 32 128 256; do
NSLCT_HOST_CHUNK_MB=$mb timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_mb$mb.log 2>&1
done
