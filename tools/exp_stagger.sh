# first-wave stagger of the interior solve at cfg5 (MSCG_TRI_STAGGER_US / _MODE)
set -u
mkdir -p gpurun_out
for v in "0 2" "150 1" "300 1" "300 2" "600 2" "0 2" "450 1" "1200 2"; do
  set -- $v
  MSCG_TRI_STAGGER_US=$1 MSCG_TRI_STAGGER_MODE=$2 timeout 600 python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu-baseline --no-gmres > gpurun_out/stg_$1_$2.json 2> gpurun_out/stg_$1_$2.err
  python -c "
import json; d=json.loads(open('gpurun_out/stg_$1_$2.json').read().strip().splitlines()[-1]); print('stagger us $1 mode $2', 'apply_ms', round(d['apply_ms'],3), 'dsolve', round(d['stage_ms']['d_solve'],3), 'frac', round(d['roofline']['frac'],3), d['clocks'])" || tail -3 gpurun_out/stg_$1_$2.err
done
