#!/bin/bash
# A/B of the split-k correction kernel (MSCG_CORR_SPLIT) on cfg2 GMRES and the apply.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "corr or gmres or cfg2 or cfg1" 2>&1 | tail -3
for i in 1 2; do for c in 1 0; do
  MSCG_CORR_SPLIT=$c timeout 300 python bench.py --config cfg2 --mode gmres > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('split=$c its', d['iterations'], 'solve_s %.3f'%d['solve_s'])"
done; done
MSCG_CORR_SPLIT=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:correct -c 20 --csv python bench.py --config cfg2 --mode gmres --max-iters 10 2>/dev/null | grep -i correct | tail -3
