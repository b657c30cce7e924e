#!/bin/bash
# round measurement: full gpu tests, bench (+cpu baseline, e2e), reference arm, ncu list + full capture
cd $GRAFT_REPO_ROOT
TAG=${1:-r01}
nvidia-smi > gpurun_out/${TAG}_nvsmi.txt 2>&1
lscpu > gpurun_out/${TAG}_lscpu.txt 2>&1
timeout 1200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -rA > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_ref.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:line_pass -s 16 -c 1 \
    -o gpurun_out/${TAG}_k2_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu_full.log
