#!/bin/bash
# large-N kernels: parity subset + A/B timing (+ optional ncu of the new kernel)
cd $GRAFT_REPO_ROOT
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 900 python tools/large_n_ab.py 16384 1 > gpurun_out/${TAG}_ab16384.jsonl 2>&1
timeout 900 python tools/large_n_ab.py 8192 4 > gpurun_out/${TAG}_ab8192.jsonl 2>&1
timeout 300 python tools/slab_pass_timing.py 16384 8 3 > gpurun_out/${TAG}_slab_timing.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "${PYK:-large_n or large_sizes or slab or comm_plan or config5 or lc_y}" > gpurun_out/${TAG}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:line_pass_big -c 2 \
    -o gpurun_out/${TAG}_c5big -f python tools/c5_once.py > gpurun_out/${TAG}_ncu_c5.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_ncu_c5.log
fi
