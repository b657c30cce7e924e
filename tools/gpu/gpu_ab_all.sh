#!/bin/bash
# A/B of alt/ builds over the configs: C4 (20 steps), C3, C2, C5 one GPU, C5 slab passes (P = 8);
# optional parity subset first (PYTEST_K with PYTEST_LIB)
cd $GRAFT_REPO_ROOT
TAG=${1:-aball}
if [ -n "$PYTEST_K" ]; then
  NSLCT_LIB=$PYTEST_LIB timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -k "$PYTEST_K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
fi
for rep in 1 2; do
  for f in ${LIBS:-alt/libnslct_*.so}; do
    n=$(basename $f .so)
    for c in 4 3 2 5; do
      NSLCT_LIB=$f timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-sub > gpurun_out/${TAG}_${n}_c${c}_${rep}.json 2>/dev/null
    done
    NSLCT_LIB=$f timeout 300 python tools/slab_pass_timing.py 16384 8 5 2>&1 | sed "s/^/$n $rep /" >> gpurun_out/${TAG}_slab.txt
  done
done
python - <<'PY' > gpurun_out/${TAG}_summary.txt
import json,glob,os
for f in sorted(glob.glob('gpurun_out/${TAG}_*_c*_*.json')):
    try:
        d=json.loads(open(f).readline()); print(os.path.basename(f), '%.1f'%d['value'], '%.4f'%d['ms_per_step'], ['%.4f'%x for x in d['roofline']['pass_ms']])
    except Exception as e: print(f,'ERR',e)
print(open('gpurun_out/${TAG}_slab.txt').read())
PY
