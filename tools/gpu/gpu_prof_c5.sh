#!/bin/bash
# ncu --set full of one N = 16384 pass kernel of a C5 transform (tools/c5_once.py), after a
# plain run of the same command exits 0.  KRE selects the kernel (default: the two-FFT pass).
cd $GRAFT_REPO_ROOT
TAG=${1:-c5}
KRE=${KRE:-"pair2_kernel<.int.1,"}
python tools/c5_once.py 16384 2 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$KRE" -s ${SKIP:-2} -c 1 \
    -o gpurun_out/${TAG}_full python tools/c5_once.py 16384 2 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu_full.log
ls -la gpurun_out >> gpurun_out/${TAG}_ncu_full.log
