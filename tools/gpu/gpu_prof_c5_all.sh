#!/bin/bash
# ncu --set full of the N = 16384 pass kernels of a C5 transform (K1, K2, K5 of the second
# transform), after a plain run of the same command exits 0
cd $GRAFT_REPO_ROOT
TAG=${1:-c5}
python tools/c5_once.py 16384 2 > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
for k in "0,:1" "1,:2" "3,:1"; do
  m=${k%%:*}; s=${k##*:}
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:pair2_kernel<.int.${m}" -s $s -c 1 \
      -o gpurun_out/${TAG}_m${m%,}_full python tools/c5_once.py 16384 2 > gpurun_out/${TAG}_m${m%,}_ncu.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_m${m%,}_ncu.log
done
