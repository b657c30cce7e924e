#!/bin/bash
# alt/libnslct_<tag>.so: the library built with extra nvcc flags (A/B experiments; see
# tools/gpu/gpu_libab_bench.sh).  usage: tools/alt_build.sh <tag> [-DFLAG ...]
set -e
cd "$(dirname "$0")/.."
TAG=$1; shift
C=paper_1707_03688_b200/csrc
NCCL_INC=$(python - <<'PY'
from paper_1707_03688_b200.build import nccl_include
print(nccl_include())
PY
)
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O3 -Xptxas -v -I include -I $NCCL_INC"
mkdir -p alt /tmp/altobj
for s in bluestein.cu planner.cpp; do
  if [ ! -f /tmp/altobj/$s.o ] || [ $C/$s -nt /tmp/altobj/$s.o ] || [ $C/kernels.cuh -nt /tmp/altobj/$s.o ]; then
    nvcc $F -c $C/$s -o /tmp/altobj/$s.o > /tmp/altobj/$s.log 2>&1 &
  fi
done
nvcc $F "$@" -c $C/nslct.cu -o /tmp/altobj/nslct_$TAG.o > /tmp/altobj/nslct_$TAG.log 2>&1
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o alt/libnslct_$TAG.so /tmp/altobj/nslct_$TAG.o /tmp/altobj/bluestein.cu.o /tmp/altobj/planner.cpp.o -ldl
echo built alt/libnslct_$TAG.so
