#!/bin/bash
# round-end style measurement: smoke, full GPU suite, default bench, reference arm,
# ncu launch list and full capture of the five passes
cd $GRAFT_REPO_ROOT
TAG=${1:-r01e}
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_ref.log
bash tools/gpu/gpu_prof_all.sh ${TAG}
