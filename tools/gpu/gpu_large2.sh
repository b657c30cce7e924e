#!/bin/bash
cd $GRAFT_REPO_ROOT
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 900 python tools/large_n_ab.py 16384 1 > gpurun_out/${TAG}_ab16384.jsonl 2>&1
timeout 900 python tools/large_n_ab.py 8192 4 > gpurun_out/${TAG}_ab8192.jsonl 2>&1
timeout 600 python bench.py --config 3 --steps 20 --no-cpu-baseline --no-e2e --no-sub > gpurun_out/${TAG}_bench_c3.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "${PYK:-large_n or config3 or exact_special or exec_host_chunked or zero_padding}" > gpurun_out/${TAG}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:line_pass_big -c 4 \
    -o gpurun_out/${TAG}_big -f python tools/large_n_ab.py 8192 1 > gpurun_out/${TAG}_ncu.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
fi
