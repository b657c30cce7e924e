#!/bin/bash
# round-end style measurement: smoke, full GPU suite, default bench, reference arm and the
# ncu launch list (the five-pass full capture is tools/gpu/gpu_prof_all.sh, run as its own
# call: its report alone approaches gpurun's 64 MiB copy-back limit)
cd $GRAFT_REPO_ROOT
TAG=${1:-r01e}
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_ref.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sub"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_list.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu_list.log
