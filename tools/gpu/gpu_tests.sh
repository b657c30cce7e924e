#!/bin/bash
# full GPU suite (per-test durations) + smoke; host facts for the oracle timings
cd $GRAFT_REPO_ROOT
TAG=${1:-r02}
mkdir -p gpurun_out
(nproc; free -g; lscpu | grep -i "model name"; nvidia-smi -L) > gpurun_out/${TAG}_host.txt 2>&1
timeout ${TT:-2400} python -m pytest tests -m gpu -q --durations=40 ${PYK:+-k "$PYK"} > gpurun_out/${TAG}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
