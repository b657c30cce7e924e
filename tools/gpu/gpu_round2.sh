#!/bin/bash
# round-2 measurement: smoke, full GPU suite, default bench (sub-records, CPU baselines,
# e2e), reference arm, ncu launch list of the C4 step and a full capture of one K2 launch
cd $GRAFT_REPO_ROOT
TAG=${1:-r02}
mkdir -p gpurun_out
(nproc; free -g; lscpu | grep -i "model name"; nvidia-smi -L) > gpurun_out/${TAG}_host.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
if [ -z "$NOTEST" ]; then
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
fi
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "rc=$?" >> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.json 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sub"
$CMD > gpurun_out/${TAG}_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:line_pass_ws -s 8 -c 1 \
    -o gpurun_out/${TAG}_k2_full -f $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu_full.log
# the other bench configurations (kernel-only): every --config path runs
for c in 1 2 3 5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c$c.json 2> gpurun_out/${TAG}_bench_c$c.err; echo "rc=$?" >> gpurun_out/${TAG}_bench_c$c.err
done
