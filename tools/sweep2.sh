# 2-knob sweep of the D-solve time (bench, no ncu).
# usage: A=MSCG_TRI_HINT AV="0 1" B=MSCG_TRI_PF BV="1 2" CONFIGS=cfg4 bash tools/sweep2.sh
for x in $AV; do for y in $BV; do for c in ${CONFIGS:-cfg4}; do
  env $A=$x $B=$y timeout 300 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/s2.json 2>gpurun_out/s2.err
  python -c "
import json; d=json.loads(open('gpurun_out/s2.json').read().strip().splitlines()[-1]); print('$c $A=$x $B=$y', 'apply_ms', round(d['apply_ms'],3), 'dsolve', round(d['stage_ms']['d_solve'],3), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/s2.err
done; done; done
